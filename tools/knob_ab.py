"""Interleaved A/B of a kgs_set_param knob on the fused colour passes
(1 GPU, resident state): average live pass time per setting, and the fields
must come out bitwise identical for every setting.

    python tools/knob_ab.py KNOB V0,V1[,..] [--N 1024] [--steps 6] [--reps 4] [--call]
                            [--scenario fourpeak2d] [--record 1]

--call times the whole kgs_step_dpavf2 call (host wall clock around the
synchronous call, one untimed warm-up call first) instead of the per-pass
events, so launch overlap between passes (e.g. the `pdl` knob) is included.
"""
import argparse
import hashlib
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2502_09537_b200 as kgs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("knob")
    ap.add_argument("values")
    ap.add_argument("--N", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--call", action="store_true")
    ap.add_argument("--scenario", default="ellipsoids3d")
    ap.add_argument("--record", type=int, default=0, help="record stride (0: once at the end)")
    a = ap.parse_args()
    vals = [int(v) for v in a.values.split(",")]
    sc = kgs.get_scenario(a.scenario)
    g = sc.default_grid(a.N)
    args = kgs.precompute_coefficients(sc.params, 0.005, g).kernel_args()
    times = {v: [] for v in vals}
    digests = {}
    for rep in range(a.reps):
        for v in vals:
            dev = kgs.DeviceFieldState.from_preset(a.scenario, g)
            dev.ctx.set_param(a.knob, v)
            if a.call:
                dev.ctx.step_dpavf2(args, 2, 0, 2)
                t0 = time.perf_counter()
                dev.ctx.step_dpavf2(args, a.steps, 0, a.record or a.steps)
                times[v].append((time.perf_counter() - t0) * 1e3 / a.steps)
            else:
                dev.ctx.pass_timing(True)
                dev.ctx.step_dpavf2(args, a.steps, 0, a.steps)
                n, ms, _ = dev.ctx.pass_stats()
                times[v].append(ms / n)
            if rep == 0:
                h = hashlib.sha256()
                st = dev.to_host()
                for f in "PQUV":
                    h.update(getattr(st, f).tobytes())
                digests[v] = h.hexdigest()[:16]
            dev.close()
    key = "step_ms" if a.call else "pass_ms"
    out = {str(v): {key: [round(t, 4) for t in times[v]],
                    "mean": round(sum(times[v]) / len(times[v]), 4)} for v in vals}
    out["bitwise_equal"] = len(set(digests.values())) == 1
    print(json.dumps({"knob": a.knob, "scenario": a.scenario, "N": a.N, **out}))


if __name__ == "__main__":
    main()
