"""Time integrate() on a pinned host state: first (cold context) vs warm calls,
pipeline on / off, chunk sizes.   python tools/e2e_probe.py [N] [K] [--chunks 8,16,32 --reps 3] [--pageable]
(--chunks: only warm pipelined calls, chunk sizes interleaved over --reps
repetitions; median wall per chunk size)"""
import json
import sys
import time

import torch

import paper_2502_09537_b200 as kgs
from paper_2502_09537_b200.device import get_context


def main():
    pos = [a for i, a in enumerate(sys.argv[1:], 1)
           if not a.startswith("--") and sys.argv[i - 1] not in ("--chunks", "--reps")]
    N = int(pos[0]) if len(pos) > 0 else 1024
    K = int(pos[1]) if len(pos) > 1 else 40
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(N)
    host = kgs.FieldState.pinned(g)
    dev = kgs.DeviceFieldState.from_preset("ellipsoids3d", g)
    dev.download(host)
    dev.close()
    if "--pageable" in sys.argv:   # ordinary numpy arrays (staged inside the call)
        import numpy as np
        host = kgs.FieldState(*(np.array(getattr(host, f)) for f in "PQUV"), host.t)
    sch = kgs.checkerboard_schedule(g)
    out = {}
    if "--chunks" in sys.argv:
        chunks = [int(c) for c in sys.argv[sys.argv.index("--chunks") + 1].split(",")]
        reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 3
        kgs.integrate(host, g, sc.params, sch, None, 0.01, K * 0.01, record_stride=K)  # warm
        walls = {c: [] for c in chunks}
        for _ in range(reps):
            for c in chunks:
                get_context(g, None).set_param("pipeline_planes", c)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                kgs.integrate(host, g, sc.params, sch, None, 0.01, K * 0.01, record_stride=K)
                torch.cuda.synchronize()
                walls[c].append(round(time.perf_counter() - t0, 4))
        for c, w in walls.items():
            m = sorted(w)[len(w) // 2]
            out[f"c{c}"] = {"walls_s": w, "median_s": m, "Gupd_s": round(2 * g.M * K / m / 1e9, 1)}
        print(json.dumps({"N": N, "K": K, **out}))
        return
    runs = [("cold_pipe", 1, 32), ("warm_pipe", 1, 32), ("warm_plain", 0, 32)]
    runs += [(f"warm_pipe_c{c}", 1, c) for c in (16, 24, 48, 64, 16, 32, 64)]
    for label, pipe, chunk in runs:
        if not label.startswith("cold"):
            get_context(g, None).set_param("pipeline", pipe)
            get_context(g, None).set_param("pipeline_planes", chunk)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        kgs.integrate(host, g, sc.params, sch, None, 0.01, K * 0.01, record_stride=K)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        out[label] = {"wall_s": round(wall, 4), "Gupd_s": round(2 * g.M * K / wall / 1e9, 1),
                      "device_ms": round(get_context(g, None).last_step_ms(), 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
