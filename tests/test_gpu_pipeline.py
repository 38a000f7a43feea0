"""kgs_integrate_host: upload | colour passes | download as one pipeline
(chunks of planes arrive around plane 0, every pass advances one plane
behind its predecessor, finished chunks go back while later ones compute).
Bitwise the plain upload + steps + download path, for any chunk size."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2502_09537_b200 as kgs
from conftest import assert_bitwise
from paper_2502_09537_b200.device import get_context

pytestmark = pytest.mark.gpu


def _run(g, sc, s0, tau, T, stride, pipeline, planes=32):
    ctx = get_context(g, None)
    ctx.set_param("pipeline", pipeline)
    ctx.set_param("pipeline_planes", planes)
    s = s0.copy()
    tr = kgs.integrate(s, g, sc.params, kgs.checkerboard_schedule(g), None, tau, T,
                       record_stride=stride)
    ctx.set_param("pipeline", 1)
    ctx.set_param("pipeline_planes", 0)
    return s, tr


@pytest.mark.parametrize("N,steps,stride,planes", [
    (128, 5, 1, 32), (128, 7, 3, 8), (128, 4, 4, 5), (192, 3, 2, 16), (256, 6, 6, 32),
    (128, 1, 1, 32), (64, 9, 2, 4), (128, 1, 1, 3), (128, 2, 1, 6), (128, 3, 3, 7),
    (128, 20, 5, 32), (512, 10, 5, 32),
    (128, 5, 1, 0), (256, 6, 1, 0), (512, 10, 5, 0)])   # 0: the auto chunk (16 here)
def test_pipeline_bitwise_vs_plain_and_oracle(N, steps, stride, planes):
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(N)
    s0 = sc.state(g)
    tau = 0.01
    a, ta = _run(g, sc, s0, tau, steps * tau, stride, 1, planes)
    b, tb = _run(g, sc, s0, tau, steps * tau, stride, 0, planes)
    assert_bitwise(a, b)
    assert a.t == b.t and ta.steps == tb.steps and ta.times == tb.times
    np.testing.assert_allclose(ta.energy, tb.energy, rtol=1e-13, atol=0)
    np.testing.assert_allclose(ta.mass, tb.mass, rtol=1e-13, atol=0)
    assert ta.max_rel_error() < 1e-12
    if N <= 128:
        ref = s0.copy()
        oracle.CheckerboardOracle(3, N).step_dpavf2(
            ref, oracle.kernel_args(sc.params, tau / 2, g), steps,
            workers=oracle.CheckerboardOracle.max_threads())
        assert_bitwise(a, ref)


@pytest.mark.parametrize("bad_plane", [0, 63, 127])
def test_pipeline_nonfinite_replays_to_the_bad_step(bad_plane):
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(128)
    s0 = sc.state(g)
    i = bad_plane * 128 * 128 + 77
    s0.U[i] = np.inf
    outs = []
    for pipeline in (1, 0):
        s = s0.copy()
        ctx = get_context(g, None)
        ctx.set_param("pipeline", pipeline)
        with pytest.raises(FloatingPointError, match="after step 1"):
            kgs.integrate(s, g, sc.params, kgs.checkerboard_schedule(g), None, 0.01, 0.05)
        outs.append(s)
    get_context(g, None).set_param("pipeline", 1)
    assert outs[0].t == outs[1].t
    for f in "PQUV":
        np.testing.assert_array_equal(getattr(outs[0], f), getattr(outs[1], f))


def test_pipeline_device_state_after_call_is_the_result():
    """The context keeps the final state resident: a following resident step
    continues from it exactly."""
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(128)
    s0 = sc.state(g)
    s = s0.copy()
    kgs.integrate(s, g, sc.params, kgs.checkerboard_schedule(g), None, 0.01, 0.04)
    ref = s0.copy()
    oracle.CheckerboardOracle(3, 128).step_dpavf2(
        ref, oracle.kernel_args(sc.params, 0.005, g), 4,
        workers=oracle.CheckerboardOracle.max_threads())
    assert_bitwise(s, ref)
    z = kgs.FieldState.zeros(g)
    get_context(g, None).download(z)
    assert_bitwise(z, ref)


@pytest.mark.parametrize("offset,steps,stride", [(3, 5, 2), (7, 4, 3), (1, 6, 6), (10, 2, 4)])
def test_integrate_host_step_offset_matches_step_dpavf2(offset, steps, stride):
    """The C ABI's step_offset: records land on global steps multiple of the
    stride, exactly as kgs_step_dpavf2 numbers them."""
    import ctypes
    from paper_2502_09537_b200 import _lib
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(128)
    s0 = sc.state(g)
    args = kgs.precompute_coefficients(sc.params, 0.005, g).kernel_args()
    nrec = (offset + steps) // stride - offset // stride
    ctx = get_context(g, None)
    a = s0.copy()
    c = _lib.coeffs_struct(args)
    t0 = np.zeros(8)
    terms = np.zeros((max(nrec, 1), 8))
    bad = ctypes.c_int64()
    rc = _lib.load().kgs_integrate_host(ctx.ptr, *(_lib.dptr(getattr(a, f)) for f in "PQUV"),
                                        ctypes.byref(c), steps, offset, stride,
                                        _lib.dptr(t0), _lib.dptr(terms), ctypes.byref(bad), 0)
    assert rc == 0
    dev = kgs.DeviceFieldState.from_host(s0, g)
    ref_terms, b2 = dev.ctx.step_dpavf2(args, steps, offset, stride)
    b = dev.to_host()
    dev.close()
    assert b2 == 0
    assert_bitwise(a, b)
    np.testing.assert_allclose(terms[:nrec], ref_terms, rtol=1e-13, atol=0)


def test_integrate_nonfinite_on_slabs_matches_one_slab():
    """integrate() on a host state with several slabs takes kgs_integrate_host's
    plain path; a non-finite step leaves the same state and message as one slab."""
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(64)
    s0 = sc.state(g)
    s0.P[40 * 64 * 64 + 9] = np.nan
    outs = []
    for ex in (None, kgs.CudaExecutor((0,), slabs_per_device=2),
               kgs.CudaExecutor((0,), slabs_per_device=4)):
        s = s0.copy()
        with pytest.raises(FloatingPointError) as err:
            kgs.integrate(s, g, sc.params, kgs.checkerboard_schedule(g), ex, 0.01, 0.05)
        outs.append((s, str(err.value)))
    for s, msg in outs[1:]:
        assert msg == outs[0][1]
        assert_bitwise(s, outs[0][0], equal_nan=True)


def _pinned_copy(g, s):
    p = kgs.FieldState.pinned(g)
    for f in "PQUV":
        getattr(p, f)[:] = getattr(s, f)
    p.t = s.t
    return p


@pytest.mark.parametrize("N,steps,stride,planes,poison", [
    (256, 6, 3, 32, None), (256, 5, 1, 7, None), (512, 8, 4, 32, None),
    (256, 4, 2, 16, 130), (256, 3, 3, 32, 0)])
def test_pipeline_with_pinned_host_arrays(N, steps, stride, planes, poison):
    """Page-locked host arrays make the pipeline's copies truly asynchronous
    (the bench's e2e case): still bitwise the plain path, incl. the replay."""
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(N)
    s0 = sc.state(g)
    if poison is not None:
        s0.U[poison * N * N + 11] = np.inf
    outs = []
    for pipe in (1, 0):
        ctx = get_context(g, None)
        ctx.set_param("pipeline", pipe)
        ctx.set_param("pipeline_planes", planes)
        s = _pinned_copy(g, s0)
        try:
            tr = kgs.integrate(s, g, sc.params, kgs.checkerboard_schedule(g), None, 0.01,
                               steps * 0.01, record_stride=stride)
            res = (tr.energy, None)
        except FloatingPointError as e:
            res = (None, str(e))
        outs.append((s.copy(), res))
    ctx.set_param("pipeline", 1)
    ctx.set_param("pipeline_planes", 0)
    (a, (ea, xa)), (b, (eb, xb)) = outs
    assert xa == xb
    assert_bitwise(a, b, equal_nan=True)
    if ea is not None:
        np.testing.assert_allclose(ea, eb, rtol=1e-13, atol=0)


@pytest.mark.parametrize("N,steps,stride,planes,poison", [
    (256, 6, 3, 32, None), (256, 5, 1, 7, None), (512, 4, 2, 32, None), (256, 3, 3, 16, 77)])
def test_pipeline_pageable_arrays_staged(N, steps, stride, planes, poison):
    """Ordinary (pageable) numpy arrays -- the reference's FieldState -- go
    through page-locked host slots filled / emptied by helper threads while
    the pipeline runs (knob stage_pageable); bitwise the direct pageable
    copies and the page-locked-array path, incl. the non-finite replay, and
    repeatable (a second staged call reuses the slots)."""
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(N)
    s0 = sc.state(g)
    if poison is not None:
        s0.V[poison * N * N + 5] = np.nan
    outs = []
    for pin, pinned in ((1, False), (0, False), (1, True), (1, False)):
        ctx = get_context(g, None)
        ctx.set_param("pipeline_planes", planes)
        ctx.set_param("stage_pageable", pin)
        s = _pinned_copy(g, s0) if pinned else s0.copy()
        try:
            tr = kgs.integrate(s, g, sc.params, kgs.checkerboard_schedule(g), None, 0.01,
                               steps * 0.01, record_stride=stride)
            res = (tr.energy, None)
        except FloatingPointError as e:
            res = (None, str(e))
        outs.append((s.copy(), res))
    ctx.set_param("stage_pageable", 1)
    ctx.set_param("pipeline_planes", 0)
    a, (ea, xa) = outs[0]
    for b, (eb, xb) in outs[1:]:
        assert xa == xb
        assert_bitwise(a, b, equal_nan=True)
        if ea is not None:
            np.testing.assert_allclose(ea, eb, rtol=1e-13, atol=0)
