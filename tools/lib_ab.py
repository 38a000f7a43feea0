"""Interleaved A/B of two builds of libkgs_b200.so (1 GPU, resident state):
each repetition runs one fresh process per library (selected with
KGS_B200_LIB) that times a whole kgs_step_dpavf2 call after a warm-up call;
the fields must come out bitwise identical for every library.

    python tools/lib_ab.py LIB_A LIB_B [--N 1024] [--steps 20] [--reps 3] [--record 1] [--scenario fourpeak2d]
"""
import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

CHILD = r"""
import hashlib, json, sys, time
sys.path.insert(0, %r)
import paper_2502_09537_b200 as kgs
N, steps, rec, scen = %d, %d, %d, %r
sc = kgs.get_scenario(scen)
g = sc.default_grid(N)
args = kgs.precompute_coefficients(sc.params, 0.005, g).kernel_args()
dev = kgs.DeviceFieldState.from_preset(scen, g)
dev.ctx.step_dpavf2(args, 2, 0, 2)
t0 = time.perf_counter()
terms, _ = dev.ctx.step_dpavf2(args, steps, 0, rec or steps)
ms = (time.perf_counter() - t0) * 1e3 / steps
h = hashlib.sha256()
st = dev.to_host()
for f in "PQUV":
    h.update(getattr(st, f).tobytes())
print(json.dumps({"step_ms": ms, "digest": h.hexdigest()[:16], "terms": terms[-1].tolist()}))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--N", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--scenario", default="ellipsoids3d")
    ap.add_argument("--record", type=int, default=0, help="record stride of the timed call (0: once at its end)")
    a = ap.parse_args()
    res = {lib: [] for lib in a.libs}
    digests = {}
    terms = {}
    for _ in range(a.reps):
        for lib in a.libs:
            env = dict(os.environ, KGS_B200_LIB=str(Path(lib).resolve()))
            out = subprocess.run([sys.executable, "-c", CHILD % (str(ROOT), a.N, a.steps, a.record, a.scenario)],
                                 env=env, capture_output=True, text=True, check=True).stdout
            r = json.loads(out.strip().splitlines()[-1])
            res[lib].append(round(r["step_ms"], 4))
            digests[lib] = r["digest"]
            terms[lib] = r["terms"]
    out = {lib: {"step_ms": v, "mean": round(sum(v) / len(v), 4)} for lib, v in res.items()}
    t0 = terms[a.libs[0]]
    rel = {lib: max(abs(x - y) / max(abs(y), 1e-300) for x, y in zip(t, t0)) for lib, t in terms.items()}
    print(json.dumps({"N": a.N, "scenario": a.scenario, **out, "bitwise_equal": len(set(digests.values())) == 1,
                      "terms_max_rel_vs_first": rel}))


if __name__ == "__main__":
    main()
