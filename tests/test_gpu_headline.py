"""Parity at the headline config (BASELINE.json configs[3], the bench
workload): 3-D ellipsoids3d on 1024^3, tau = 0.01, from the reference's own
host preset (scenarios.py:69-89, built block-parallel, bitwise the
whole-grid build), 20 DP-AVF2 steps -- the benchmarked step count --
through the exact call pattern bench.py times:

  * device path: upload, 3 steps without records (bench warm-up), 12 steps
    with one record at the end (bench timed call), 5 steps recording every
    step (bench diagnostics) -- the plain, end-record and every-step-record
    march_pass variants;
  * public API: ``integrate()`` on a host FieldState (the pipelined
    upload | passes | download path bench's e2e times), and the same on two
    slabs from page-locked memory (the multi-slab pipeline).

Both are compared bit for bit with the table-free C restatement
(oracle/kgs_oracle.c, pinned to the reference's golden vectors in
tests/test_oracle_golden.py) run for the same 20 steps on all host cores;
the recorded energy terms are checked against the oracle's exactly-summed
terms, and energy conservation at the reference's round-off level.

Host memory: ~105 GB (oracle state, two integrate() states, chunk buffers); the
oracle takes ~1 min on 16 cores.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2502_09537_b200 as kgs
from paper_2502_09537_b200.grid import energy_from_terms
from paper_2502_09537_b200.scenarios import build_preset

pytestmark = pytest.mark.gpu

N = 1024
TAU = 0.01
W, K, R = 3, 12, 5          # bench.py: warm-up, timed (record at end), record every step
STEPS = W + K + R


def _compare_device(dev, ref, chunk_planes=32):
    """Download the device state plane chunk by plane chunk (no second
    32 GiB host copy) and compare with the oracle's arrays bitwise."""
    plane = N * N
    buf = np.empty(chunk_planes * plane)
    for fi, f in enumerate("PQUV"):
        r = getattr(ref, f)
        for x0 in range(0, N, chunk_planes):
            dev.ctx.download_planes(fi, x0, buf)
            want = r[x0 * plane:(x0 + chunk_planes) * plane]
            if not np.array_equal(buf, want):
                bad = np.flatnonzero(buf != want)
                i = x0 * plane + int(bad[0])
                raise AssertionError(
                    f"device {f}: {bad.size} mismatches in planes [{x0}, {x0 + chunk_planes}), "
                    f"first at (x,y,z)={np.unravel_index(i, (N, N, N))}: "
                    f"{buf[bad[0]]!r} vs oracle {want[bad[0]]!r}")


def test_headline_1024_bitwise_vs_oracle():
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(N)
    ref = build_preset("ellipsoids3d", g)
    host = kgs.FieldState(*(getattr(ref, f).copy() for f in "PQUV"), 0.0)
    kargs = kgs.precompute_coefficients(sc.params, TAU / 2.0, g).kernel_args()

    # ---- device path, bench.py's call pattern --------------------------
    dev = kgs.DeviceFieldState.from_host(ref, g, kgs.CudaExecutor((0,)))
    e0, m0 = dev.energy_mass(sc.params)
    t_w, bad_w = dev.ctx.step_dpavf2(kargs, W, 0, 0)
    t_k, bad_k = dev.ctx.step_dpavf2(kargs, K, W, K)
    t_r, bad_r = dev.ctx.step_dpavf2(kargs, R, W + K, 1)
    assert bad_w == bad_k == bad_r == 0
    assert len(t_k) == 1 and len(t_r) == R
    dev_terms_final = np.asarray(t_r[-1])

    # ---- public API: integrate() on a host state (pipelined) -----------
    tr = kgs.integrate(host, g, sc.params, kgs.checkerboard_schedule(g), kgs.CudaExecutor((0,)),
                       TAU, STEPS * TAU, record_stride=5)
    assert tr.steps == [0, 5, 10, 15, 20]
    kgs.clear_contexts()

    # ---- integrate() on two slabs: the multi-slab pipeline (faces exchanged
    # between the passes) from page-locked host memory ---------------------
    host2 = kgs.FieldState.pinned(g, zero=False)
    for f in "PQUV":
        getattr(host2, f)[:] = getattr(ref, f)
    ex2 = kgs.CudaExecutor((0,), slabs_per_device=2)
    tr2 = kgs.integrate(host2, g, sc.params, kgs.checkerboard_schedule(g), ex2,
                        TAU, STEPS * TAU, record_stride=5)
    np.testing.assert_allclose(tr2.energy, tr.energy, rtol=1e-13, atol=0)
    kgs.clear_contexts()

    # ---- oracle: 20 steps on the host, all cores -------------------------
    orc = oracle.TableFreeOracle(3, N)
    terms0 = orc.energy_terms(ref)
    orc.step_dpavf2(ref, oracle.kernel_args(sc.params, TAU / 2.0, g), STEPS)

    # fields: bitwise, both paths
    _compare_device(dev, ref)
    dev.close()
    for label, st in (("integrate()", host), ("integrate() on 2 slabs", host2)):
        for f in "PQUV":
            a, b = getattr(st, f), getattr(ref, f)
            if not np.array_equal(a, b):
                bad = np.flatnonzero(a != b)
                raise AssertionError(f"{label} {f}: {bad.size} mismatches, first at {bad[0]}")
    assert host.t == pytest.approx(STEPS * TAU, rel=0, abs=1e-12)

    # diagnostics: the device's fused record reduction vs exact sums
    terms_final = orc.energy_terms(ref)
    np.testing.assert_allclose(dev_terms_final, terms_final, rtol=1e-12, atol=1e-300)
    e_dev, m_dev = energy_from_terms(dev_terms_final, sc.params, g)
    e_ref, m_ref = energy_from_terms(terms_final, sc.params, g)
    assert abs(e_dev - e_ref) <= 1e-12 * abs(e_ref)
    assert abs(m_dev - m_ref) <= 1e-12 * abs(m_ref)
    e_init, _ = energy_from_terms(terms0, sc.params, g)
    assert abs(e0 - e_init) <= 1e-12 * abs(e_init)
    # energy conserved to round-off over the 20 steps (reference criterion 1
    # level; measured ~1e-14 here)
    assert abs(e_ref - e_init) <= 1e-12 * abs(e_init)
    assert tr.max_rel_error() <= 1e-12
