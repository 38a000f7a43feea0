"""Randomised equivalence of the execution paths added for performance
(hypothesis): the pipelined host integration (any chunk size, step count,
record stride, with or without a non-finite value), and the multi-slab
variants (fused halo stores vs copies, fused one-march steps vs two passes)
-- all bitwise the plain path's fields, same records up to summation order,
same first bad step."""
from __future__ import annotations

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import paper_2502_09537_b200 as kgs
from conftest import assert_bitwise, experimental_build
from paper_2502_09537_b200.device import get_context

pytestmark = pytest.mark.gpu
SETTINGS = settings(max_examples=40, deadline=None, suppress_health_check=list(HealthCheck))
# the fused one-march step exists only in the experimental build
FUSED = st.booleans() if experimental_build() else st.just(False)


def _state(g, seed):
    rng = np.random.default_rng(seed)
    return kgs.FieldState(*(rng.uniform(-0.5, 0.5, g.M) for _ in range(4)), 0.0)


@SETTINGS
@given(N=st.sampled_from([64, 96, 128]), planes=st.integers(1, 40), steps=st.integers(1, 9),
       stride=st.integers(1, 4), seed=st.integers(0, 2**31), tau=st.floats(1e-3, 0.05),
       poison=st.booleans(), plane=st.integers(0, 127), pinned=st.booleans())
def test_pipeline_equals_plain(N, planes, steps, stride, seed, tau, poison, plane, pinned):
    g = kgs.GridSpec(3, -6.0, 6.0, N)
    p = kgs.PhysParams(1.1, 0.9, 1.2, 0.8)
    s0 = _state(g, seed)
    if poison:
        s0.V[(plane % N) * N * N + 5] = np.inf
    outs = []
    for pipe in (1, 0):
        ctx = get_context(g, None)
        ctx.set_param("pipeline", pipe)
        ctx.set_param("pipeline_planes", planes)
        s = s0.copy()
        if pinned:   # page-locked arrays: truly asynchronous copies in the pipeline
            s = kgs.FieldState.pinned(g)
            for f in "PQUV":
                getattr(s, f)[:] = getattr(s0, f)
        try:
            tr = kgs.integrate(s, g, p, kgs.checkerboard_schedule(g), None, tau, steps * tau,
                               record_stride=stride)
            outs.append((s.copy(), tr.energy, None))
        except FloatingPointError as e:
            outs.append((s.copy(), None, str(e)))
    ctx.set_param("pipeline", 1)
    ctx.set_param("pipeline_planes", 0)
    (a, ea, xa), (b, eb, xb) = outs
    assert xa == xb
    for f in "PQUV":
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
    assert a.t == b.t
    if ea is not None:
        np.testing.assert_allclose(ea, eb, rtol=1e-12, atol=1e-300)


@SETTINGS
@given(N=st.sampled_from([64, 128]), slabs=st.sampled_from([2, 4]), steps=st.integers(1, 6),
       stride=st.integers(0, 3), seed=st.integers(0, 2**31), mirror=st.booleans(),
       fused=FUSED, defer=st.booleans(), poison=st.one_of(st.none(), st.integers(0, 127)))
def test_slab_variants_equal_one_slab(N, slabs, steps, stride, seed, mirror, fused, defer,
                                      poison):
    g = kgs.GridSpec(3, -6.0, 6.0, N)
    p = kgs.PhysParams(0.9, 1.1, 1.0, 0.7)
    args = kgs.precompute_coefficients(p, 0.01, g).kernel_args()
    s0 = _state(g, seed)
    if poison is not None:   # a non-finite value on any plane, incl. slab faces
        s0.U[(poison % N) * N * N + 3] = np.nan
    outs = []
    for ex, params in ((None, {}),
                       (kgs.CudaExecutor((0,), slabs_per_device=slabs),
                        {"mirror_halo": int(mirror), "fused_step": int(fused)})):
        dev = kgs.DeviceFieldState.from_host(s0, g, ex)
        for k, v in params.items():
            dev.ctx.set_param(k, v)
        terms, bad = dev.ctx.step_dpavf2(args, steps, 0, stride, defer_tail=defer)
        terms2, bad2 = dev.ctx.step_dpavf2(args, 2, steps, stride)
        outs.append((dev.to_host(), terms, terms2, bad, bad2))
        dev.close()
    assert_bitwise(outs[0][0], outs[1][0], equal_nan=True)
    assert outs[0][3:] == outs[1][3:]
    if poison is None:
        assert outs[0][3] == 0
        np.testing.assert_allclose(outs[0][1], outs[1][1], rtol=1e-12, atol=1e-300)
        np.testing.assert_allclose(outs[0][2], outs[1][2], rtol=1e-12, atol=1e-300)
    else:
        assert outs[0][3] == 1


OPS = st.lists(st.one_of(
    st.tuples(st.just("steps"), st.integers(1, 4), st.integers(0, 3), st.booleans()),
    st.tuples(st.just("sweep"), st.sampled_from([0, 1]), st.sampled_from([0, 1])),
    st.tuples(st.just("energy")),
    st.tuples(st.just("planes"), st.integers(0, 3), st.integers(0, 63), st.integers(1, 8)),
    st.tuples(st.just("upload")),
), min_size=1, max_size=8)


@SETTINGS
@given(N=st.sampled_from([64, 128]), slabs=st.sampled_from([2, 4]), seed=st.integers(0, 2**31),
       mirror=st.booleans(), fused=FUSED, ops=OPS)
def test_random_operation_sequences_slabs_vs_one(N, slabs, seed, mirror, fused, ops):
    """Any interleaving of multi-step calls (records, deferred tails), single
    sweeps, energy evaluations, partial plane uploads and full uploads gives
    the same bits on several slabs (any knobs) as on one."""
    g = kgs.GridSpec(3, -6.0, 6.0, N)
    p = kgs.PhysParams(1.0, 1.2, 0.9, 0.6)
    args = kgs.precompute_coefficients(p, 0.01, g).kernel_args()
    s0 = _state(g, seed)
    rng = np.random.default_rng(seed + 1)
    fresh = _state(g, seed + 2)
    outs = []
    for ex, params in ((None, {}),
                       (kgs.CudaExecutor((0,), slabs_per_device=slabs),
                        {"mirror_halo": int(mirror), "fused_step": int(fused)})):
        dev = kgs.DeviceFieldState.from_host(s0, g, ex)
        for k, v in params.items():
            dev.ctx.set_param(k, v)
        energies, offset = [], 0
        for op in ops:
            if op[0] == "steps":
                _, n, stride, defer = op
                terms, bad = dev.ctx.step_dpavf2(args, n, offset, stride, defer_tail=defer)
                assert bad == 0
                offset += n
                energies += [float(np.sum(t)) for t in terms]
            elif op[0] == "sweep":
                dev.ctx.sweep(op[1], op[2], args)
            elif op[0] == "energy":
                energies.append(float(np.sum(dev.energy_terms())))
            elif op[0] == "planes":
                _, f, x0, n = op
                n = min(n, N - x0 % N)
                x0 = x0 % N
                plane = g.N * g.N
                dev.ctx.upload_planes(f, x0, np.ascontiguousarray(
                    getattr(fresh, "PQUV"[f])[x0 * plane:(x0 + n) * plane]))
            else:
                dev.upload(fresh)
        outs.append((dev.to_host(), energies))
        dev.close()
    assert_bitwise(outs[0][0], outs[1][0])
    np.testing.assert_allclose(outs[0][1], outs[1][1], rtol=1e-12, atol=1e-300)


@SETTINGS
@given(d=st.sampled_from([1, 2, 3]), seed=st.integers(0, 2**31), ops=OPS)
def test_random_operation_sequences_resident_vs_passes(d, seed, ops):
    """Grids that fit in one CTA's shared memory run whole calls in one
    launch; any interleaving of calls, sweeps, energy evaluations and
    uploads gives the same bits as the per-pass kernels."""
    N = {1: 256, 2: 32, 3: 12}[d]
    g = kgs.GridSpec(d, -6.0, 6.0, N)
    p = kgs.PhysParams(1.0, 1.2, 0.9, 0.6)
    args = kgs.precompute_coefficients(p, 0.01, g).kernel_args()
    s0 = _state(g, seed)
    fresh = _state(g, seed + 2)
    plane = g.M // (N if d > 1 else 1)
    nplanes = N if d > 1 else 1
    outs = []
    for resident in (1, 0):
        dev = kgs.DeviceFieldState.from_host(s0, g)
        dev.ctx.set_param("resident", resident)
        energies, offset = [], 0
        for op in ops:
            if op[0] == "steps":
                _, n, stride, defer = op
                terms, bad = dev.ctx.step_dpavf2(args, n, offset, stride, defer_tail=defer)
                assert bad == 0
                offset += n
                energies += [float(np.sum(t)) for t in terms]
            elif op[0] == "sweep":
                dev.ctx.sweep(op[1], op[2], args)
            elif op[0] == "energy":
                energies.append(float(np.sum(dev.energy_terms())))
            elif op[0] == "planes":
                _, f, x0, n = op
                x0 = x0 % nplanes
                n = min(n, nplanes - x0)
                dev.ctx.upload_planes(f, x0, np.ascontiguousarray(
                    getattr(fresh, "PQUV"[f])[x0 * plane:(x0 + n) * plane]))
            else:
                dev.upload(fresh)
        outs.append((dev.to_host(), energies))
        dev.close()
    assert_bitwise(outs[0][0], outs[1][0])
    np.testing.assert_allclose(outs[0][1], outs[1][1], rtol=1e-12, atol=1e-300)


@SETTINGS
@given(N=st.sampled_from([64, 96, 128]), slabs=st.sampled_from([2, 4]),
       planes=st.integers(1, 12), steps=st.integers(1, 7), stride=st.integers(1, 4),
       seed=st.integers(0, 2**31), tau=st.floats(1e-3, 0.05),
       poison=st.one_of(st.none(), st.integers(0, 127)))
def test_slab_pipeline_equals_one_slab(N, slabs, planes, steps, stride, seed, tau, poison):
    """The pipelined integrate on several slabs (face exchanges between the
    passes, pinned host arrays) against one slab's pipeline: same fields,
    same records to summation order, same first bad step."""
    if (N // slabs) // planes < 4:
        planes = max(1, (N // slabs) // 4)       # the pipeline needs >= 4 chunks per slab
    g = kgs.GridSpec(3, -6.0, 6.0, N)
    p = kgs.PhysParams(1.0, 0.8, 1.1, 0.9)
    s0 = _state(g, seed)
    if poison is not None:
        s0.Q[(poison % N) * N * N + 7] = np.inf
    outs = []
    for ex in (None, kgs.CudaExecutor((0,), slabs_per_device=slabs)):
        ctx = get_context(g, ex)
        ctx.set_param("pipeline_planes", planes)
        s = kgs.FieldState.pinned(g)
        for f in "PQUV":
            getattr(s, f)[:] = getattr(s0, f)
        try:
            tr = kgs.integrate(s, g, p, kgs.checkerboard_schedule(g), ex, tau, steps * tau,
                               record_stride=stride)
            outs.append((s.copy(), tr.energy, None))
        except FloatingPointError as e:
            outs.append((s.copy(), None, str(e)))
        ctx.set_param("pipeline_planes", 0)
    (a, ea, xa), (b, eb, xb) = outs
    assert xa == xb
    for f in "PQUV":
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
    assert a.t == b.t
    if ea is not None:
        np.testing.assert_allclose(ea, eb, rtol=1e-12, atol=1e-300)
