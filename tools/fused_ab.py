"""A/B of the fused step march vs two colour passes (1 GPU, resident state).

    python tools/fused_ab.py [N] [steps] [planes...]
"""
import json
import sys

import paper_2502_09537_b200 as kgs


def run(N, steps, fused, planes=0, slabs=1, dbg=0):
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(N)
    ex = None if slabs == 1 else kgs.CudaExecutor((0,), slabs_per_device=slabs)
    dev = kgs.DeviceFieldState.from_preset("ellipsoids3d", g, ex)
    ctx = dev.ctx
    ctx.set_param("fused_step", fused)
    if planes:
        ctx.set_param("fused_planes", planes)
    if dbg:
        ctx.set_param("fused_debug", dbg)
    args = kgs.precompute_coefficients(sc.params, 0.005, g).kernel_args()
    ctx.step_dpavf2(args, 3, 0, 0)
    ctx.step_dpavf2(args, steps, 3, 0)
    ms = ctx.last_step_ms() / steps
    dev.close()
    return {"ms_per_step": ms, "G_updates_per_s": 2 * g.M / ms / 1e6}


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    planes = [int(x) for x in sys.argv[3:]] or [0]
    out = {"two_pass": run(N, steps, 0)}
    for p in planes:
        out[f"fused_xc{p or 128}"] = run(N, steps, 1, p)
    out["fused_4slabs"] = run(N, steps, 1, 0, 4)
    for dbg in (1, 2, 4, 7):   # timing only: 1 no ring, 2 no K4 math, 4 no K3 math
        out[f"fused_dbg{dbg}"] = run(N, steps, 1, 0, 1, dbg)
    print(json.dumps({"N": N, **out}))


if __name__ == "__main__":
    main()
