"""Interleaved A/B of march-kernel variants at N^3 on ONE evolving device
state: per round, each variant runs `steps` DP-AVF2 steps with per-pass CUDA
event timing (fused K3/K4 passes).  Prints the median fused-pass time and
ms/step per variant; the energy terms after each block are checked against
the previous block's continuation (same trajectory, any variant).
   python tools/variant_ab.py --variants 0,4,5,6 [--N 1024] [--steps 4] [--rounds 4]"""
import argparse
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2502_09537_b200 as kgs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=1024)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--rounds", type=int, default=4)
ap.add_argument("--variants", default="0,4,5,6")
ap.add_argument("--record", type=int, default=0, help="record stride (0: none)")
ap.add_argument("--param", action="append", default=[])
a = ap.parse_args()
vs = [int(v) for v in a.variants.split(",")]
sc = kgs.get_scenario("ellipsoids3d")
g = sc.default_grid(a.N)
dev = kgs.DeviceFieldState.from_preset("ellipsoids3d", g)
for kv in a.param:
    k, v = kv.split("=")
    dev.ctx.set_param(k, int(v))
args = kgs.precompute_coefficients(sc.params, 0.005, g).kernel_args()
off = 0
dev.ctx.step_dpavf2(args, 1, off, 0)
off += 1
res = {v: ([], []) for v in vs}
for r in range(a.rounds):
    for v in vs:
        dev.ctx.set_param("march_variant", v)
        dev.ctx.pass_timing(True)
        terms, bad = dev.ctx.step_dpavf2(args, a.steps, off, a.record)
        assert bad == 0
        off += a.steps
        n, ms, _ = dev.ctx.pass_stats()
        dev.ctx.pass_timing(False)
        res[v][0].append(ms / max(n, 1))
        res[v][1].append(dev.ctx.last_step_ms() / a.steps)
e0 = dev.energy_mass(sc.params)
for v in vs:
    p, s = res[v]
    print(f"variant {v}: fused pass {statistics.median(p):.3f} ms (min {min(p):.3f}), "
          f"step {statistics.median(s):.3f} ms (min {min(s):.3f})  "
          f"[{' '.join(f'{x:.2f}' for x in p)}]", flush=True)
print("energy, mass after", off, "steps:", e0)
