"""Sweep the colour-pass tile/band/occupancy knobs (kgs_set_tuning) on one
GPU and print the average fused-pass time (CUDA events) per configuration.

    python tools/tune_pass.py [--N 1024] [--steps 4]
"""
from __future__ import annotations

import argparse
import itertools
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2502_09537_b200 as kgs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--ty", default="1,2,4,8")
    ap.add_argument("--band", default="0,16,32,64,128")
    ap.add_argument("--occ", default="0")
    ap.add_argument("--variant", default="1")
    ap.add_argument("--xc", default="0")
    ap.add_argument("--sync", default="4")
    a = ap.parse_args()
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(a.N)
    dev = kgs.DeviceFieldState.from_preset("ellipsoids3d", g)
    ctx = dev.ctx
    args = kgs.precompute_coefficients(sc.params, 0.005, g).kernel_args()
    ctx.step_dpavf2(args, 2)
    pts = g.M // 2
    res = []
    for ty, band, occ, var, xc, sync in itertools.product(
            *(list(map(int, s.split(","))) for s in (a.ty, a.band, a.occ, a.variant, a.xc,
                                                     a.sync))):
        ctx.set_tuning(ty, band, occ, xc, var)
        ctx.set_param("march_sync", sync)
        ctx.step_dpavf2(args, 1)
        ctx.pass_timing(True)
        ctx.step_dpavf2(args, a.steps)
        n, ms, _ = ctx.pass_stats()
        ctx.pass_timing(False)
        avg = ms / n
        r = {"ty": ty, "band": band, "occ": occ, "variant": var, "xc": xc, "sync": sync,
             "pass_ms": round(avg, 4),
             "step_ms_est": round(2 * avg, 3),
             "GBs_44B": round(44 * 2 * pts / avg / 1e6, 1),
             "Gupd_s": round(2 * pts / avg / 1e6, 2)}
        res.append(r)
        print(json.dumps(r), flush=True)
    best = min(res, key=lambda r: r["pass_ms"])
    print("BEST", json.dumps(best))


if __name__ == "__main__":
    main()
