"""Step rates on BASELINE.json's smaller configs (1 GPU, resident state).

    python tools/config_rates.py

C1: 1-D soliton N=1024, tau=1e-3, T=1 (1000 steps, record every step as
    the reference's integrate does by default, and with record_stride=1000)
C2: 2-D fourpeak2d N=1024^2, tau=0.01
C3: 3-D ellipsoids3d N=512^3, tau=0.01
Prints one JSON line with ms/step and updates/s per config.
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2502_09537_b200 as kgs  # noqa: E402


def rate(name, N, tau, steps, stride):
    sc = kgs.get_scenario(name)
    g = sc.default_grid(N)
    dev = kgs.DeviceFieldState.from_preset(name, g, None)
    args = kgs.precompute_coefficients(sc.params, tau / 2.0, g).kernel_args()
    ctx = dev.ctx
    ctx.step_dpavf2(args, 5, 0, stride if stride <= 5 else 0)
    t0 = time.perf_counter()
    ctx.step_dpavf2(args, steps, 5, stride)
    wall = time.perf_counter() - t0
    dev_ms = ctx.last_step_ms()
    dev.close()
    upd = 2 * g.M * steps
    return {"ms_per_step_device": dev_ms / steps, "ms_per_step_wall": wall * 1e3 / steps,
            "updates_per_s_wall": upd / wall, "record_stride": stride}


def main():
    out = {
        "C1_1d_N1024_stride1": rate("soliton1d", 1024, 1e-3, 1000, 1),
        "C1_1d_N1024_stride1000": rate("soliton1d", 1024, 1e-3, 1000, 1000),
        "C2_2d_N1024_fourpeak": rate("fourpeak2d", 1024, 0.01, 200, 0),
        "C2_2d_N1024_fourpeak_stride1": rate("fourpeak2d", 1024, 0.01, 200, 1),
        "C3_3d_N512_ellipsoids": rate("ellipsoids3d", 512, 0.01, 40, 0),
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
