"""Interleaved A/B of knob SETTINGS (several knobs at once; the pseudo-knob
record=S sets the record stride of that setting's calls) on the fused
passes at N^3: random order per round, per-pass CUDA events; fields of all
settings follow one trajectory (results never depend on knobs).
   python tools/config_ab.py "march_wave_sync=0" "march_wave_sync=1,march_planes=128" ...
"""
import argparse
import random
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2502_09537_b200 as kgs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="+")
ap.add_argument("--N", type=int, default=1024)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--rounds", type=int, default=4)
ap.add_argument("--record", type=int, default=0, help="record stride (0: none)")
ap.add_argument("--call", action="store_true", help="time whole calls (ms/step) instead of passes")
a = ap.parse_args()
cfgs = [dict((kv.split("=")[0], int(kv.split("=")[1])) for kv in c.split(",") if kv) for c in a.configs]
keys = sorted({k for c in cfgs for k in c})
sc = kgs.get_scenario("ellipsoids3d")
g = sc.default_grid(a.N)
dev = kgs.DeviceFieldState.from_preset("ellipsoids3d", g)
args = kgs.precompute_coefficients(sc.params, 0.005, g).kernel_args()
defaults = {"march_wave_sync": 1, "march_planes": 0, "march_variant": 4, "march_sms": 0, "blocks_per_sm": 0}
off = 0
dev.ctx.step_dpavf2(args, 2, off, 0)
off += 2
res = {i: [] for i in range(len(cfgs))}
rng = random.Random(7)
for r in range(a.rounds):
    order = list(range(len(cfgs)))
    rng.shuffle(order)
    for i in order:
        for k in keys:
            if k != "record":
                dev.ctx.set_param(k, cfgs[i].get(k, defaults.get(k, 0)))
        rec = cfgs[i].get("record", a.record)
        dev.ctx.pass_timing(True)
        dev.ctx.step_dpavf2(args, a.steps, off, rec)
        off += a.steps
        n, ms, _ = dev.ctx.pass_stats()
        dev.ctx.pass_timing(False)
        res[i].append(dev.ctx.last_step_ms() / a.steps if a.call else ms / n)
for i, c in enumerate(cfgs):
    print(f"{a.configs[i]:45s} median {statistics.median(res[i]):.3f} ms  "
          f"[{' '.join(f'{x:.2f}' for x in res[i])}]", flush=True)
