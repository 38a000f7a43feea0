"""Time integrate() on a pinned host state: first (cold context) vs warm calls,
pipeline on / off.   python tools/e2e_probe.py [N] [K]"""
import json
import sys
import time

import torch

import paper_2502_09537_b200 as kgs
from paper_2502_09537_b200.device import get_context


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(N)
    host = kgs.FieldState.pinned(g)
    dev = kgs.DeviceFieldState.from_preset("ellipsoids3d", g)
    dev.download(host)
    dev.close()
    sch = kgs.checkerboard_schedule(g)
    out = {}
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
