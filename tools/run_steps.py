"""Run a few DP-AVF2 steps at N^3 (device preset) -- an ncu target.
   python tools/run_steps.py [--N 1024] [--steps 3] [--variant 0] [--param k=v ...]"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2502_09537_b200 as kgs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=1024)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--record", type=int, default=0)
ap.add_argument("--param", action="append", default=[])
a = ap.parse_args()
sc = kgs.get_scenario("ellipsoids3d")
g = sc.default_grid(a.N)
dev = kgs.DeviceFieldState.from_preset("ellipsoids3d", g)
for kv in a.param:
    k, v = kv.split("=")
    dev.ctx.set_param(k, int(v))
args = kgs.precompute_coefficients(sc.params, 0.005, g).kernel_args()
dev.ctx.step_dpavf2(args, 1, 0, 0)
dev.ctx.pass_timing(True)
off = 1
for r in range(a.reps):
    t = time.perf_counter()
    dev.ctx.step_dpavf2(args, a.steps, off, a.record)
    off += a.steps
    n, ms, pts = dev.ctx.pass_stats()
    print(f"rep {r}: {dev.ctx.last_step_ms() / a.steps:.3f} ms/step, fused pass "
          f"{ms / max(n, 1):.3f} ms avg over {n}, wall {time.perf_counter() - t:.3f} s", flush=True)
    dev.ctx.pass_timing(False)
    dev.ctx.pass_timing(True)
