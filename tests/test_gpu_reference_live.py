"""GPU: parity against the reference ITSELF, run live on the GPU box's host
(dpavf installed unmodified into baseline/_ref with numba, as the bench's
reference arm uses it): the drop-in API fed the reference's own objects --
its GridSpec-compatible grids, its checkerboard and reverse_schedule'd
UpdateSchedule objects, its SerialExecutor / PhasedExecutor -- gives the
reference's fields bit for bit and its energy trace to summation order."""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2502_09537_b200 as kgs

pytestmark = pytest.mark.gpu
REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"


@pytest.fixture(scope="module")
def dpavf():
    if not (REF / "dpavf").is_dir():
        pytest.skip("reference not installed in baseline/_ref (see DESIGN.md §6)")
    pytest.importorskip("numba")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/kgs_numba_cache")
    sys.path.insert(0, str(REF))
    import dpavf as ref
    return ref


def _pair(dpavf, d, N, seed):
    gr = dpavf.GridSpec(d, -2.0, 2.0, N)
    g = kgs.GridSpec(d, -2.0, 2.0, N)
    sr = dpavf.seeded_random_state(gr, seed, 0.5)
    s = kgs.FieldState(sr.P.copy(), sr.Q.copy(), sr.U.copy(), sr.V.copy(), 0.0)
    return gr, g, sr, s


def _same(a, b):
    for f in "PQUV":
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


@pytest.mark.parametrize("d,N", [(3, 16), (2, 32), (1, 64)])
def test_integrate_with_reference_objects(dpavf, d, N):
    gr, g, sr, s = _pair(dpavf, d, N, 7)
    pr = dpavf.PhysParams(1.1, 0.9, 1.2, 0.8)
    p = kgs.PhysParams(1.1, 0.9, 1.2, 0.8)
    sch = dpavf.checkerboard_schedule(gr, workers=4)
    with dpavf.PhasedExecutor(4) as ex:
        tr_ref = dpavf.integrate(sr, gr, pr, sch, ex, 0.02, 0.2, record_stride=3)
        tr = kgs.integrate(s, g, p, sch, ex, 0.02, 0.2, record_stride=3)
    _same(s, sr)
    assert s.t == sr.t and tr.steps == tr_ref.steps and tr.times == tr_ref.times
    np.testing.assert_allclose(tr.energy, tr_ref.energy, rtol=1e-13, atol=0)
    np.testing.assert_allclose(tr.mass, tr_ref.mass, rtol=1e-13, atol=0)


@pytest.mark.parametrize("d,N", [(3, 8), (2, 16)])
def test_reversed_reference_schedule(dpavf, d, N):
    """dpavf.reverse_schedule(...) sweeps black first in both halves; the
    drop-in reads the order off the schedule object."""
    gr, g, sr, s = _pair(dpavf, d, N, 11)
    pr = dpavf.PhysParams(-0.4, 0.1, 0.1, 0.2)
    p = kgs.PhysParams(-0.4, 0.1, 0.1, 0.2)
    rev = dpavf.reverse_schedule(dpavf.checkerboard_schedule(gr))
    cr = dpavf.precompute_coefficients(pr, 0.01, gr)
    c = kgs.precompute_coefficients(p, 0.01, g)
    ser = dpavf.SerialExecutor()
    for _ in range(3):
        dpavf.step_dpavf2(sr, rev, cr, ser, gr)
        kgs.step_dpavf2(s, rev, c, ser, g)
    _same(s, sr)
    dpavf.step_base(sr, rev, cr, ser, gr)
    kgs.step_base(s, rev, c, ser, g)
    dpavf.step_adjoint(sr, rev, cr, ser, gr)
    kgs.step_adjoint(s, rev, c, ser, g)
    _same(s, sr)
    # integrate() over a reversed schedule (the step-at-a-time loop)
    tr_ref = dpavf.integrate(sr, gr, pr, rev, ser, 0.02, 0.1, record_stride=2)
    tr = kgs.integrate(s, g, p, rev, ser, 0.02, 0.1, record_stride=2)
    _same(s, sr)
    assert tr.steps == tr_ref.steps
    np.testing.assert_allclose(tr.energy, tr_ref.energy, rtol=1e-13, atol=0)


def test_bench_gpus_beyond_the_box_fails_loudly():
    """`bench.py --gpus N` with fewer visible GPUs exits non-zero and says
    so (no silent single-GPU run labelled N GPUs)."""
    import subprocess
    import torch
    n = torch.cuda.device_count()
    root = Path(__file__).resolve().parent.parent
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", str(n + 1),
                        "--steps", "1", "--N", "128", "--no-e2e", "--no-cpu"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode != 0
    assert f"only {n} CUDA devices visible" in r.stderr + r.stdout
