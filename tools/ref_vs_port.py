"""Time the reference's own CPU path (numba, /root/reference -- present only
in the build container) against the C port used as bench.py's CPU baseline,
same grid, same thread count, on this host.  Evidence for DESIGN.md §6; not
used by tests, smoke() or bench.py.

    NUMBA_CACHE_DIR=/tmp/nb python tools/ref_vs_port.py [N] [steps] [threads]
"""
import json
import os
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    W = int(sys.argv[3]) if len(sys.argv) > 3 else os.cpu_count()
    import numpy as np
    import dpavf
    import oracle

    sc = dpavf.get_scenario("ellipsoids3d")
    g = sc.default_grid(N)
    st = sc.state(g)
    coeffs = dpavf.precompute_coefficients(sc.params, 0.005, g)
    out = {"N": N, "steps": steps, "threads": W, "host_cores": os.cpu_count()}
    for w in (1, W):
        sch = dpavf.checkerboard_schedule(g, w)
        ex = dpavf.ExecutorConfig("phased" if w > 1 else "serial", w).build()
        s = st.copy()
        dpavf.step_dpavf2(s, sch, coeffs, ex, g)        # warm-up (numba compile)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            for _ in range(steps):
                dpavf.step_dpavf2(s, sch, coeffs, ex, g)
            ts.append((time.perf_counter() - t0) / steps)
        out[f"reference_numba_w{w}_upd_s"] = 2 * g.M / statistics.median(ts)
        if hasattr(ex, "close"):
            ex.close()
    orc = oracle.CheckerboardOracle(3, N)
    args = oracle.kernel_args(sc.params, 0.005, g)
    for w in (1, W):
        s = st.copy()
        orc.step_dpavf2(s, args, 1, workers=w)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            orc.step_dpavf2(s, args, steps, workers=w)
            ts.append((time.perf_counter() - t0) / steps)
        out[f"c_port_w{w}_upd_s"] = 2 * g.M / statistics.median(ts)
    # same bits
    a, b = st.copy(), st.copy()
    dpavf.step_dpavf2(a, dpavf.checkerboard_schedule(g, W), coeffs,
                      dpavf.ExecutorConfig("phased", W).build(), g)
    orc.step_dpavf2(b, args, 1, workers=W)
    out["bitwise_equal_after_1_step"] = all(np.array_equal(getattr(a, f), getattr(b, f))
                                            for f in "PQUV")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
