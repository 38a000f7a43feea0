"""Per-step time vs virtual slab count on one GPU (halo-exchange overlap check).

    python tools/slab_overlap.py [N] [steps]

Every slab count runs the same grid through the same fused stepping loop;
with the exchange overlapped against the interior planes the per-step time
should stay close to the single-slab time (the copies are 2 faces per slab
per pass, ~0.4% of the pass traffic at N=1024).
"""
import json
import sys
import time

import paper_2502_09537_b200 as kgs


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(N)
    args = kgs.precompute_coefficients(sc.params, 0.005, g).kernel_args()
    out = {}
    for slabs in (1, 2, 4, 8):
        ex = None if slabs == 1 else kgs.CudaExecutor((0,), slabs_per_device=slabs)
        dev = kgs.DeviceFieldState.from_preset("ellipsoids3d", g, ex)
        ctx = dev.ctx
        ctx.step_dpavf2(args, 3, 0, 0)
        t0 = time.perf_counter()
        ctx.step_dpavf2(args, steps, 3, 0)
        wall = (time.perf_counter() - t0) / steps * 1e3
        out[slabs] = {"device_ms_per_step": ctx.last_step_ms(), "wall_ms_per_step": wall}
        dev.close()
    print(json.dumps({"N": N, "steps": steps, "per_slab_count": out}))


if __name__ == "__main__":
    main()
