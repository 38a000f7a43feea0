"""Run a few fused DP-AVF2 steps (for ncu: -k regex:step_pass).

    python tools/profile_step.py [--N 1024] [--steps 2] [--fused 1] [--planes 0]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2502_09537_b200 as kgs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=1024)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--fused", type=int, default=1)
ap.add_argument("--planes", type=int, default=0)
a = ap.parse_args()
sc = kgs.get_scenario("ellipsoids3d")
g = sc.default_grid(a.N)
dev = kgs.DeviceFieldState.from_preset("ellipsoids3d", g)
dev.ctx.set_param("fused_step", a.fused)
if a.planes:
    dev.ctx.set_param("fused_planes", a.planes)
args = kgs.precompute_coefficients(sc.params, 0.005, g).kernel_args()
dev.ctx.step_dpavf2(args, a.steps, 0, 0)
print(f"N={a.N} steps={a.steps}: {dev.ctx.last_step_ms() / a.steps:.3f} ms/step")
