"""Long-run energy conservation at scale (BASELINE config 5's check, on the
largest grid one B200 holds): N^3 ellipsoids3d, tau = 0.01, `steps` DP-AVF2
steps with a record every `stride` steps, state resident on the device.

    python tools/long_run.py [N] [steps] [stride]
"""
import json
import sys
import time

import paper_2502_09537_b200 as kgs


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
    stride = int(sys.argv[3]) if len(sys.argv) > 3 else 50
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(N)
    dev = kgs.DeviceFieldState.from_preset("ellipsoids3d", g)
    sch = kgs.checkerboard_schedule(g)
    t0 = time.perf_counter()
    tr = kgs.integrate(dev, g, sc.params, sch, None, 0.01, steps * 0.01, record_stride=stride)
    wall = time.perf_counter() - t0
    out = {"N": N, "steps": steps, "tau": 0.01, "T": steps * 0.01, "record_stride": stride,
           "wall_s": wall, "E0": tr.energy[0], "E_final": tr.energy[-1],
           "max_rel_error": tr.max_rel_error(),
           "rel_error_trace": [float(f"{r:.3e}") for r in tr.rel_error],
           "mass0": tr.mass[0], "mass_final": tr.mass[-1], "finite": dev.is_finite()}
    dev.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
