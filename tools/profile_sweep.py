"""Run fused-sweep steps at N^3 (for ncu / timing).  python tools/profile_sweep.py [--N 1024]"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2502_09537_b200 as kgs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=1024)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--fused", type=int, default=1)
ap.add_argument("--dbg", type=int, default=0)
a = ap.parse_args()
sc = kgs.get_scenario("ellipsoids3d")
g = sc.default_grid(a.N)
dev = kgs.DeviceFieldState.from_preset("ellipsoids3d", g)
dev.ctx.set_param("fused_sweep", a.fused)
dev.ctx.set_param("sweep_debug", a.dbg)
args = kgs.precompute_coefficients(sc.params, 0.005, g).kernel_args()
dev.ctx.step_dpavf2(args, 1)
dev.ctx.pass_timing(True)
t = time.perf_counter()
dev.ctx.step_dpavf2(args, a.steps)
n, ms, pts = dev.ctx.pass_stats()
print(f"N={a.N} fused={a.fused} dbg={a.dbg}: {ms / n:.3f} ms per timed launch ({n} launches, {pts} pts)")
