"""Run config C2 (2-D fourpeak2d 1024^2, tau=0.01) for a few steps on the
device -- a small driver for ncu captures of the 2-D colour pass.

    python tools/run_c2.py [steps]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2502_09537_b200 as kgs  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    sc = kgs.get_scenario("fourpeak2d")
    g = sc.default_grid(1024)
    dev = kgs.DeviceFieldState.from_preset("fourpeak2d", g, None)
    args = kgs.precompute_coefficients(sc.params, 0.01 / 2.0, g).kernel_args()
    dev.ctx.step_dpavf2(args, steps, 0, 0)
    print(f"C2 {steps} steps: {dev.ctx.last_step_ms() / steps * 1e3:.2f} us/step")
    dev.close()


if __name__ == "__main__":
    main()
