"""End to end through integrate() on a page-locked host state at N^3 with
1, 2 and 4 virtual slabs on one GPU (the multi-slab pipeline: every slab
runs the wavefront, faces exchanged between passes) -- pipeline on / off;
interleaved repetitions; then the pipelined call on ordinary pageable
arrays (staged through page-locked slots) for 1 and 2 slabs.
    python tools/e2e_slabs.py [N] [K] [reps]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2502_09537_b200 as kgs  # noqa: E402
from paper_2502_09537_b200.device import get_context  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(N)
    host = kgs.FieldState.pinned(g)
    dev = kgs.DeviceFieldState.from_preset("ellipsoids3d", g)
    dev.download(host)
    dev.close()
    sch = kgs.checkerboard_schedule(g)
    res = {}
    for _ in range(reps):
        for slabs in (1, 2, 4):
            for pipe in (1, 0):
                ex = kgs.CudaExecutor((0,), slabs_per_device=slabs)
                get_context(g, ex).set_param("pipeline", pipe)
                kgs.integrate(host, g, sc.params, sch, ex, 0.01, 0.03, record_stride=3)
                torch.cuda.synchronize()
                t = time.perf_counter()
                kgs.integrate(host, g, sc.params, sch, ex, 0.01, K * 0.01, record_stride=K)
                torch.cuda.synchronize()
                dt = time.perf_counter() - t
                res.setdefault(f"slabs{slabs}_{'pipe' if pipe else 'plain'}", []).append(
                    round(dt, 3))
                kgs.clear_contexts()
    plain = kgs.FieldState(*(np.array(getattr(host, f)) for f in "PQUV"), 0.0)
    for _ in range(reps):
        for slabs in (1, 2):
            ex = kgs.CudaExecutor((0,), slabs_per_device=slabs)
            kgs.integrate(plain, g, sc.params, sch, ex, 0.01, 0.03, record_stride=3)
            torch.cuda.synchronize()
            t = time.perf_counter()
            kgs.integrate(plain, g, sc.params, sch, ex, 0.01, K * 0.01, record_stride=K)
            torch.cuda.synchronize()
            res.setdefault(f"slabs{slabs}_pageable", []).append(round(time.perf_counter() - t, 3))
            kgs.clear_contexts()
    print(json.dumps({"N": N, "K": K, "wall_s": res,
                      "G_upd_per_s": {k: round(2 * g.M * K / min(v) / 1e9, 1)
                                      for k, v in res.items()}}))


if __name__ == "__main__":
    main()
