"""Generate tests/golden/kgs_golden.npz by running the REFERENCE itself.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Each case: the initial state, the reference's `integrate(..., checkerboard,
SerialExecutor)` final state and EnergyTrace, and the kernel_args() of the
half-step coefficients -- or, for the single-sweep cases, one `step_base` /
`step_adjoint` (negative tau too, as in tests/test_integrator.py:135-161).
Only this script touches /root/reference; the fixtures travel with the repo.
"""
from __future__ import annotations

import json
import math
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, os.environ.get("DPAVF_SRC", "/root/reference/pkg/src"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from dpavf import (FieldState, GridSpec, PhysParams, SerialExecutor,  # noqa: E402
                   checkerboard_schedule, discrete_energy, get_scenario,
                   integrate, mass, precompute_coefficients,
                   seeded_random_state, step_adjoint, step_base)

OUT = Path(__file__).resolve().parent / "kgs_golden.npz"
PARAMS = PhysParams(1.1, 0.9, 1.2, 0.8)           # tests/test_oracle.py:14
ELLIP = PhysParams(-0.4, 0.1, 0.1, 0.2)


def soliton(grid, v=0.8):
    """SURVEY.md §8(d) C1 at t=0 (same formula as scenarios.soliton1d_exact)."""
    x = grid.axis_coords()
    w = np.sqrt(1.0 - v * v)
    xi = x / (2.0 * w)
    s2 = 1.0 / np.cosh(xi)**2
    amp = 3.0 * np.sqrt(2.0) / (4.0 * w)
    phase = v * x
    u = 3.0 / (4.0 * w * w) * s2
    return FieldState(amp * s2 * np.cos(phase), amp * s2 * np.sin(phase), u,
                      u * np.tanh(xi) * v / w, 0.0)


# name: (grid, params, initial-state factory, tau, T, record_stride)
RUNS = {
    "d1_rand_N64": (GridSpec(1, -10.0, 10.0, 64), PARAMS, lambda g: seeded_random_state(g, 7, 0.5), 0.05, 1.0, 5),
    "d1_rand_N2": (GridSpec(1, -1.0, 1.0, 2), PARAMS, lambda g: seeded_random_state(g, 3, 0.5), 0.05, 0.5, 1),
    "d2_rand_N2": (GridSpec(2, -1.0, 1.0, 2), PARAMS, lambda g: seeded_random_state(g, 4, 0.5), 0.05, 0.5, 1),
    "d3_rand_N2": (GridSpec(3, -1.0, 1.0, 2), PARAMS, lambda g: seeded_random_state(g, 5, 0.5), 0.05, 0.5, 1),
    "d3_rand_N4": (GridSpec(3, -1.0, 1.0, 4), PARAMS, lambda g: seeded_random_state(g, 6, 0.5), 0.03, 0.6, 2),
    "d2_gauss_N16": (GridSpec(2, -10.0, 10.0, 16), PhysParams(), lambda g: get_scenario("gaussian2d").state(g), 0.1, 2.0, 1),
    "d2_rand_N32": (GridSpec(2, -1.0, 1.0, 32), PARAMS, lambda g: seeded_random_state(g, 11, 0.5), 0.04, 0.8, 4),
    "d2_rand_N6": (GridSpec(2, -1.0, 1.0, 6), PARAMS, lambda g: seeded_random_state(g, 12, 0.5), 0.04, 0.8, 3),
    "d2_fourpeak_N64": (GridSpec(2, -10.0, 10.0, 64), PhysParams(0.5, 0.5, 0.5, 0.5), lambda g: get_scenario("fourpeak2d").state(g), 0.01, 0.2, 5),
    "d3_rand_N8": (GridSpec(3, -1.0, 1.0, 8), PARAMS, lambda g: seeded_random_state(g, 42, 0.5), 0.03, 0.6, 5),
    "d3_rand_N12": (GridSpec(3, -2.0, 2.0, 12), ELLIP, lambda g: seeded_random_state(g, 77, 0.5), 0.01, 0.2, 10),
    "d3_ellip_N16": (GridSpec(3, -10.0, 10.0, 16), ELLIP, lambda g: get_scenario("ellipsoids3d").state(g), 0.01, 0.2, 1),
    "d1_soliton_N1024": (GridSpec(1, -40.0, 40.0, 1024), PhysParams(), soliton, 1e-3, 1.0, 10),
}

# single sweeps: name: (grid, params, state factory, tau, "base"|"adjoint")
SWEEPS = {
    "sweep_base_d1_N16": (GridSpec(1, -1.0, 1.0, 16), PARAMS, lambda g: seeded_random_state(g, 21, 0.5), 0.03, "base"),
    "sweep_adj_d1_N16": (GridSpec(1, -1.0, 1.0, 16), PARAMS, lambda g: seeded_random_state(g, 22, 0.5), 0.03, "adjoint"),
    "sweep_base_d2_N8": (GridSpec(2, -1.0, 1.0, 8), PARAMS, lambda g: seeded_random_state(g, 23, 0.5), 0.03, "base"),
    "sweep_adj_d2_N8_negtau": (GridSpec(2, -1.0, 1.0, 8), PARAMS, lambda g: seeded_random_state(g, 24, 0.5), -0.03, "adjoint"),
    "sweep_base_d3_N6": (GridSpec(3, -1.0, 1.0, 6), PARAMS, lambda g: seeded_random_state(g, 25, 0.5), 0.03, "base"),
    "sweep_adj_d3_N6": (GridSpec(3, -1.0, 1.0, 6), PARAMS, lambda g: seeded_random_state(g, 26, 0.5), 0.03, "adjoint"),
    "sweep_base_d3_N4_negtau": (GridSpec(3, -1.0, 1.0, 4), PARAMS, lambda g: seeded_random_state(g, 27, 0.5), -0.05, "base"),
}


def _seed_of(factory):
    """(seed, amplitude) of a seeded_random_state lambda, else None."""
    consts = factory.__code__.co_consts
    ints = [c for c in consts if isinstance(c, int) and not isinstance(c, bool)]
    floats = [c for c in consts if isinstance(c, float)]
    if "seeded_random_state" in factory.__code__.co_names and ints and floats:
        return [ints[0], floats[0]]
    return None


def main() -> None:
    arrays: dict[str, np.ndarray] = {}
    meta: dict[str, dict] = {}
    ex = SerialExecutor()

    def put(name, key, a):
        arrays[f"{name}/{key}"] = np.asarray(a)

    for name, (g, p, make, tau, T, stride) in RUNS.items():
        s0 = make(g)
        s = s0.copy()
        sch = checkerboard_schedule(g)
        tr = integrate(s, g, p, sch, ex, tau, T, record_stride=stride)
        for f in "PQUV":
            put(name, f + "0", getattr(s0, f))
            put(name, f + "1", getattr(s, f))
        put(name, "kernel_args", precompute_coefficients(p, tau / 2.0, g).kernel_args())
        for key in ("steps", "times", "energy", "rel_error", "mass"):
            put(name, "trace_" + key, getattr(tr, key))
        meta[name] = dict(kind="integrate", d=g.d, a=g.a, b=g.b, N=g.N,
                          params=[p.kappa1, p.kappa2, p.mu, p.gamma], tau=tau, T=T,
                          record_stride=stride, n_steps=int(math.ceil(T / tau - 1e-12)),
                          t_final=s.t, max_rel_error=tr.max_rel_error(),
                          seed=_seed_of(make))
        print(f"{name}: steps={meta[name]['n_steps']} maxRE={tr.max_rel_error():.3e}")

    for name, (g, p, make, tau, kind) in SWEEPS.items():
        s0 = make(g)
        s = s0.copy()
        c = precompute_coefficients(p, tau, g)
        (step_base if kind == "base" else step_adjoint)(s, checkerboard_schedule(g), c, ex, g)
        for f in "PQUV":
            put(name, f + "0", getattr(s0, f))
            put(name, f + "1", getattr(s, f))
        put(name, "kernel_args", c.kernel_args())
        meta[name] = dict(kind=kind, d=g.d, a=g.a, b=g.b, N=g.N,
                          params=[p.kappa1, p.kappa2, p.mu, p.gamma], tau=tau, t_final=s.t,
                          seed=_seed_of(make))

    # pinned energy of tests/test_scenarios.py:137-143,164 and its inputs
    g = GridSpec(2, -10.0, 10.0, 8)
    s = seeded_random_state(g, 42, 0.5)
    for f in "PQUV":
        put("golden_seed42", f + "0", getattr(s, f))
    meta["golden_seed42"] = dict(kind="energy", d=2, a=-10.0, b=10.0, N=8,
                                 params=[1.0, 1.0, 1.0, 1.0],
                                 energy=discrete_energy(s, PhysParams(), g),
                                 mass=mass(s, g))
    # reference preset states (bitwise IC check of the package's presets)
    for sc_name, N in (("gaussian2d", 16), ("fourpeak2d", 16), ("ellipsoids3d", 8)):
        sc = get_scenario(sc_name)
        st = sc.state(sc.default_grid(N))
        for f in "PQUV":
            put(f"preset_{sc_name}", f + "0", getattr(st, f))
        meta[f"preset_{sc_name}"] = dict(kind="preset", N=N)

    arrays["__meta__"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1024:.0f} KiB)")


if __name__ == "__main__":
    main()
