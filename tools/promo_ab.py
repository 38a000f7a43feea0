"""Interleaved A/B of the TMA L2 promotion of the march kernel's halo and
tile boxes (kgs_set_promotion) at N^3, random order per round.
   python tools/promo_ab.py --variant 4 --configs 0,0:1,0:2,0 [--rounds 6]"""
import argparse
import random
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2502_09537_b200 as kgs  # noqa: E402
from paper_2502_09537_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=1024)
ap.add_argument("--variant", type=int, default=4)
ap.add_argument("--configs", default="0,0:1,0:2,0")
ap.add_argument("--rounds", type=int, default=6)
ap.add_argument("--steps", type=int, default=4)
a = ap.parse_args()
cfgs = [tuple(map(int, c.split(","))) for c in a.configs.split(":")]
sc = kgs.get_scenario("ellipsoids3d")
g = sc.default_grid(a.N)
dev = kgs.DeviceFieldState.from_preset("ellipsoids3d", g)
dev.ctx.set_param("march_variant", a.variant)
args = kgs.precompute_coefficients(sc.params, 0.005, g).kernel_args()
off = 0
res = {c: [] for c in cfgs}
rng = random.Random(1)
for r in range(a.rounds):
    order = cfgs[:]
    rng.shuffle(order)
    for c in order:
        _lib.check(_lib.load().kgs_set_promotion(dev.ctx.ptr, *c), dev.ctx.ptr)
        dev.ctx.pass_timing(True)
        dev.ctx.step_dpavf2(args, a.steps, off, 0)
        off += a.steps
        n, ms, _ = dev.ctx.pass_stats()
        dev.ctx.pass_timing(False)
        res[c].append(ms / n)
for c in cfgs:
    print(f"promo halo {c[0]} tile {c[1]}: median {statistics.median(res[c]):.3f} ms "
          f"[{' '.join(f'{x:.2f}' for x in res[c])}]")
