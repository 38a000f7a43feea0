"""kgs_integrate_host on several slabs: every slab runs the pipeline
(chunks arrive around its plane 0, passes follow as a wavefront) side by
side, with the faces of every pass exchanged as soon as both boundary
planes are written (kgs_pipeline.cuh pipeline_plan; its dependency checker
is tests/test_pipeline_plan.py).  Bitwise the plain upload + steps +
download path and the single-slab result, for virtual slabs on one GPU and
for the torchrun rank path (1 rank exchanging with itself over NCCL)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2502_09537_b200 as kgs
from conftest import assert_bitwise
from paper_2502_09537_b200.device import get_context

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _fresh():
    kgs.clear_contexts()
    yield
    kgs.clear_contexts()


def _pinned_copy(g, s):
    p = kgs.FieldState.pinned(g, zero=False)
    for f in "PQUV":
        getattr(p, f)[:] = getattr(s, f)
    p.t = s.t
    return p


def _run(g, sc, s0, ex, tau, steps, stride, pipeline, planes):
    ctx = get_context(g, ex)
    ctx.set_param("pipeline", pipeline)
    ctx.set_param("pipeline_planes", planes)
    s = _pinned_copy(g, s0)
    n0 = ctx.launch_count()
    tr = kgs.integrate(s, g, sc.params, kgs.checkerboard_schedule(g), ex, tau, steps * tau,
                       record_stride=stride)
    n = ctx.launch_count() - n0
    ctx.set_param("pipeline", 1)
    ctx.set_param("pipeline_planes", 0)
    return s, tr, n


@pytest.mark.parametrize("slabs,N,steps,stride,planes", [
    (2, 128, 5, 1, 8), (2, 128, 7, 3, 5), (4, 128, 4, 2, 4), (2, 256, 6, 6, 16),
    (4, 256, 3, 1, 8), (2, 64, 9, 2, 3), (8, 256, 2, 1, 4), (2, 512, 4, 2, 32)])
def test_slab_pipeline_bitwise_vs_plain_and_one_slab(slabs, N, steps, stride, planes):
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(N)
    s0 = sc.state(g)
    tau = 0.01
    ex = kgs.CudaExecutor((0,), slabs_per_device=slabs)
    a, ta, na = _run(g, sc, s0, ex, tau, steps, stride, 1, planes)
    b, tb, nb_ = _run(g, sc, s0, ex, tau, steps, stride, 0, planes)
    one, t1, _ = _run(g, sc, s0, None, tau, steps, stride, 1, 32)
    assert na > 2 * nb_, "the pipelined path did not run"   # many partial-range launches
    assert_bitwise(a, b)
    assert_bitwise(a, one)
    assert a.t == b.t and ta.steps == tb.steps and ta.times == tb.times
    for tr in (tb, t1):
        np.testing.assert_allclose(ta.energy, tr.energy, rtol=1e-13, atol=0)
        np.testing.assert_allclose(ta.mass, tr.mass, rtol=1e-13, atol=0)


def test_slab_pipeline_nonfinite_replays_to_the_bad_step():
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(128)
    s0 = sc.state(g)
    s0.U[64 * 128 * 128 + 5] = np.inf    # a slab-boundary plane of 2 slabs
    ex = kgs.CudaExecutor((0,), slabs_per_device=2)
    out = {}
    for pipeline in (1, 0):
        ctx = get_context(g, ex)
        ctx.set_param("pipeline", pipeline)
        s = _pinned_copy(g, s0)
        with pytest.raises(FloatingPointError) as ei:
            kgs.integrate(s, g, sc.params, kgs.checkerboard_schedule(g), ex, 0.01, 0.05,
                          record_stride=1)
        ctx.set_param("pipeline", 1)
        out[pipeline] = (s, str(ei.value))
    assert_bitwise(out[1][0], out[0][0], equal_nan=True)
    assert out[1][1] == out[0][1]


def test_rank_pipeline_with_nccl_self_exchange(monkeypatch):
    """The torchrun rank path: one rank, faces sent to itself over NCCL."""
    monkeypatch.setenv("KGS_SELF_EXCHANGE", "1")
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(128)
    s0 = sc.state(g)
    ex = kgs.DistributedExecutor(rank=0, world_size=1, device=0)
    a, ta, na = _run(g, sc, s0, ex, 0.01, 5, 1, 1, 8)
    kgs.clear_contexts()
    monkeypatch.delenv("KGS_SELF_EXCHANGE")
    one, t1, n1 = _run(g, sc, s0, None, 0.01, 5, 1, 1, 8)
    assert na > 0 and n1 > 0
    assert_bitwise(a, one)
    np.testing.assert_allclose(ta.energy, t1.energy, rtol=1e-13, atol=0)


def test_rank_pipeline_nonfinite_agrees_and_replays(monkeypatch):
    """The rank path's agreement on the first bad step (an NCCL all-reduce,
    run here by one self-exchanging rank) and its replay: same state and
    message as one ordinary slab."""
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(128)
    s0 = sc.state(g)
    s0.P[127 * 128 * 128 + 9] = np.nan     # the last plane: a face of the rank
    out = {}
    for key, selfx in (("rank", True), ("one", False)):
        if selfx:
            monkeypatch.setenv("KGS_SELF_EXCHANGE", "1")
        else:
            monkeypatch.delenv("KGS_SELF_EXCHANGE", raising=False)
        kgs.clear_contexts()
        ex = kgs.DistributedExecutor(rank=0, world_size=1, device=0) if selfx else None
        get_context(g, ex).set_param("pipeline_planes", 8)
        s = _pinned_copy(g, s0)
        with pytest.raises(FloatingPointError) as ei:
            kgs.integrate(s, g, sc.params, kgs.checkerboard_schedule(g), ex, 0.01, 0.04,
                          record_stride=1)
        out[key] = (s, str(ei.value))
    assert_bitwise(out["rank"][0], out["one"][0], equal_nan=True)
    assert out["rank"][1] == out["one"][1]


@pytest.mark.parametrize("slabs,N,steps,stride,planes,poison", [
    (2, 128, 5, 1, 8, None), (4, 128, 3, 3, 4, None), (2, 256, 4, 2, 16, None),
    (2, 128, 6, 1, 8, 64 * 128 * 128 + 11)])
def test_slab_pipeline_pageable_arrays(slabs, N, steps, stride, planes, poison):
    """Ordinary (pageable) numpy arrays on several slabs: staged through one
    ring of page-locked slots by the helper threads; bitwise one slab's."""
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(N)
    s0 = sc.state(g)
    if poison is not None:
        s0.V[poison] = np.inf
    out = {}
    for key, ex in (("slabs", kgs.CudaExecutor((0,), slabs_per_device=slabs)), ("one", None)):
        ctx = get_context(g, ex)
        ctx.set_param("pipeline_planes", planes)
        s = s0.copy()                     # pageable
        n0 = ctx.launch_count()
        try:
            tr = kgs.integrate(s, g, sc.params, kgs.checkerboard_schedule(g), ex, 0.01,
                               steps * 0.01, record_stride=stride)
            out[key] = (s, tr.energy, None, ctx.launch_count() - n0)
        except FloatingPointError as e:
            out[key] = (s, None, str(e), ctx.launch_count() - n0)
        ctx.set_param("pipeline_planes", 0)
        kgs.clear_contexts()
    (a, ea, xa, na), (b, eb, xb, _) = out["slabs"], out["one"]
    assert na > 40, "the pipelined path did not run"
    assert xa == xb
    assert_bitwise(a, b, equal_nan=True)
    if ea is not None:
        np.testing.assert_allclose(ea, eb, rtol=1e-13, atol=0)
