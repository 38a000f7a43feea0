"""GPU parity: the sm_100a path through the public API / C ABI against the
reference's golden vectors and the oracle.  Bar: fields bitwise identical
(np.array_equal) -- the reference arithmetic is reproduced exactly -- and
energies within the stated tolerance (the device reduction order differs
from numpy's pairwise sums; SURVEY.md App.B measured ~1e-15 relative).
"""
from __future__ import annotations

import hashlib

import numpy as np
import pytest

import oracle
import paper_2502_09537_b200 as kgs
from conftest import assert_bitwise, needs_experimental, run_names, sweep_names

pytestmark = pytest.mark.gpu

E_RTOL = 1e-13   # device energy vs reference energy (reduction order only)


@pytest.fixture(autouse=True, scope="module")
def _fresh_contexts():
    yield
    kgs.clear_contexts()


def _integrate(c, executor=None, state=None):
    s = c.state(0) if state is None else state
    tr = kgs.integrate(s, c.grid, c.params, kgs.checkerboard_schedule(c.grid),
                       executor, c.meta["tau"], c.meta["T"],
                       record_stride=c.meta["record_stride"])
    return s, tr


@pytest.mark.parametrize("name", run_names())
def test_integrate_bitwise_vs_reference(golden, name):
    c = golden.case(name)
    s, tr = _integrate(c)
    assert_bitwise(s, c.state(1))
    assert s.t == c.meta["t_final"]
    assert tr.steps == [int(v) for v in c.trace("steps")]
    assert tr.times == [float(v) for v in c.trace("times")]
    np.testing.assert_allclose(tr.energy, c.trace("energy"), rtol=E_RTOL, atol=0)
    np.testing.assert_allclose(tr.mass, c.trace("mass"), rtol=E_RTOL, atol=0)
    # energy conserved to the reference's round-off level
    assert tr.max_rel_error() <= max(10 * c.meta["max_rel_error"], 1e-13)


@pytest.mark.parametrize("name", sweep_names())
def test_single_sweeps_bitwise(golden, name):
    c = golden.case(name)
    s = c.state(0)
    coeffs = kgs.precompute_coefficients(c.params, c.meta["tau"], c.grid)
    step = kgs.step_adjoint if c.meta["kind"] == "adjoint" else kgs.step_base
    step(s, kgs.checkerboard_schedule(c.grid), coeffs, kgs.SerialExecutor(), c.grid)
    assert_bitwise(s, c.state(1))
    assert s.t == c.meta["t_final"]


@pytest.mark.parametrize("slabs", [2, 4])
@pytest.mark.parametrize("name", ["d2_rand_N32", "d3_rand_N8", "d3_rand_N12", "d3_ellip_N16",
                                  "d2_fourpeak_N64", "d3_rand_N4"])
def test_virtual_slabs_bitwise(golden, name, slabs):
    """Decomposition invariance: the multi-slab halo path
    gives the same bits as the reference for any slab count."""
    c = golden.case(name)
    if c.grid.N % slabs or c.grid.N // slabs < 2:
        pytest.skip("slab count does not divide N")
    s, tr = _integrate(c, kgs.CudaExecutor((0,), slabs_per_device=slabs))
    assert_bitwise(s, c.state(1))
    np.testing.assert_allclose(tr.energy, c.trace("energy"), rtol=E_RTOL, atol=0)


def test_step_dpavf2_api_matches_oracle(golden):
    c = golden.case("d3_rand_N8")
    coeffs = kgs.precompute_coefficients(c.params, c.meta["tau"] / 2.0, c.grid)
    s = c.state(0)
    ref = c.state(0)
    for _ in range(3):
        kgs.step_dpavf2(s, kgs.checkerboard_schedule(c.grid), coeffs, None, c.grid)
    oracle.numpy_step_dpavf2(ref, c.kernel_args, c.grid, 3)
    assert_bitwise(s, ref)


def test_device_state_roundtrip_and_resident_stepping(golden):
    c = golden.case("d3_rand_N12")
    dev = kgs.DeviceFieldState.from_host(c.state(0), c.grid)
    assert_bitwise(dev.to_host(), c.state(0))
    tr = kgs.integrate(dev, c.grid, c.params, kgs.checkerboard_schedule(c.grid), None,
                       c.meta["tau"], c.meta["T"], record_stride=c.meta["record_stride"])
    assert_bitwise(dev.to_host(), c.state(1))
    assert dev.t == c.meta["t_final"]
    np.testing.assert_allclose(tr.energy, c.trace("energy"), rtol=E_RTOL)
    dev.close()


def test_energy_and_mass_on_device(golden):
    c = golden.case("golden_seed42")
    s = c.state(0)
    e = kgs.discrete_energy(s, kgs.PhysParams(), c.grid)
    assert e == pytest.approx(66.88429062581992, rel=1e-14)
    assert kgs.mass(s, c.grid) == pytest.approx(c.meta["mass"], rel=1e-14)
    dev = kgs.DeviceFieldState.from_host(s, c.grid)
    terms = dev.energy_terms()
    np.testing.assert_allclose(terms, oracle.energy_terms(s, c.grid), rtol=1e-14)
    assert dev.is_finite()
    dev.close()


@pytest.mark.parametrize("name", ["d2_gauss_N16", "d3_rand_N8"])
def test_nonfinite_detection_names_the_step(golden, name):
    """integrate raises FloatingPointError "after step n" and leaves the host
    state exactly where the reference leaves it (integrator.py:169-171)."""
    c = golden.case(name)
    s0 = c.state(0)
    s0.U[3] = 1e308                     # overflows within a few steps
    s0.V[3] = 1e308
    ref = s0.copy()
    bad_ref = None
    for n in range(1, 50):
        oracle.numpy_step_dpavf2(ref, c.kernel_args, c.grid)
        if not ref.is_finite():
            bad_ref = n
            break
    assert bad_ref is not None
    s = s0.copy()
    with pytest.raises(FloatingPointError, match=f"after step {bad_ref} "):
        kgs.integrate(s, c.grid, c.params, kgs.checkerboard_schedule(c.grid), None,
                      c.meta["tau"], 100 * c.meta["tau"], record_stride=1)
    assert_bitwise(s, ref, equal_nan=True)


@pytest.mark.parametrize("slabs", [1, 2])
def test_nonfinite_on_a_device_state_rewinds_to_the_bad_step(golden, slabs):
    """integrate() on a DeviceFieldState: the device copy of the chunk start
    (KGS_STEP_BACKUP) is restored and replayed, so fields AND t are those
    after the first bad step, like a host state's."""
    c = golden.case("d3_rand_N8")
    s0 = c.state(0)
    s0.U[3] = 1e308
    s0.V[3] = 1e308
    ref = s0.copy()
    bad_ref = None
    for n in range(1, 50):
        oracle.numpy_step_dpavf2(ref, c.kernel_args, c.grid)
        if not ref.is_finite():
            bad_ref = n
            break
    ex = None if slabs == 1 else kgs.CudaExecutor((0,), slabs_per_device=slabs)
    dev = kgs.DeviceFieldState.from_host(s0, c.grid, ex)
    with pytest.raises(FloatingPointError, match=f"after step {bad_ref} "):
        kgs.integrate(dev, c.grid, c.params, kgs.checkerboard_schedule(c.grid), ex,
                      c.meta["tau"], 100 * c.meta["tau"], record_stride=7)
    t_ref = 0.0
    for _ in range(bad_ref):
        t_ref += c.meta["tau"] / 2
        t_ref += c.meta["tau"] / 2
    assert dev.t == t_ref
    assert_bitwise(dev.to_host(), ref, equal_nan=True)
    assert not dev.ctx.restore_backup()        # consumed
    dev.close()


def test_is_finite_flag(golden):
    c = golden.case("d3_rand_N4")
    s = c.state(0)
    dev = kgs.DeviceFieldState.from_host(s, c.grid)
    assert dev.is_finite()
    s.Q[17] = np.nan
    dev.upload(s)
    assert not dev.is_finite()
    dev.close()


def test_odd_n_rejected_by_device_context():
    with pytest.raises(ValueError, match="even N"):
        kgs.DeviceFieldState(kgs.GridSpec(2, -1.0, 1.0, 9))


# ---- full-size and large-grid properties --------------------------------
@pytest.mark.parametrize("d,N,scenario,steps", [
    (3, 64, "ellipsoids3d", 6), (2, 1024, "fourpeak2d", 4), (3, 128, "ellipsoids3d", 3)])
def test_large_grid_bitwise_vs_c_oracle(d, N, scenario, steps):
    sc = kgs.get_scenario(scenario)
    g = sc.default_grid(N)
    s = sc.state(g)
    ref = s.copy()
    tau = 0.01
    kgs.integrate(s, g, sc.params, kgs.checkerboard_schedule(g), None, tau, steps * tau,
                  record_stride=steps)
    orc = oracle.CheckerboardOracle(d, N)
    orc.step_dpavf2(ref, oracle.kernel_args(sc.params, tau / 2.0, g), steps,
                    workers=oracle.CheckerboardOracle.max_threads())
    assert_bitwise(s, ref)


def test_256cubed_decomposition_invariance_and_energy():
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(256)
    sch = kgs.checkerboard_schedule(g)
    outs = []
    for ex in (None, kgs.CudaExecutor((0,), slabs_per_device=4)):
        dev = kgs.DeviceFieldState.from_preset("ellipsoids3d", g, ex)
        tr = kgs.integrate(dev, g, sc.params, sch, None, 0.01, 0.2, record_stride=5)
        assert tr.max_rel_error() < 1e-12
        outs.append(dev.to_host())
        dev.close()
    assert_bitwise(outs[0], outs[1])


def test_device_presets_match_host_presets():
    for name, N in (("ellipsoids3d", 32), ("fourpeak2d", 64), ("gaussian2d", 64),
                    ("soliton1d", 1024)):
        sc = kgs.get_scenario(name)
        g = sc.default_grid(N)
        host = sc.state(g)
        dev = kgs.DeviceFieldState.from_preset(name, g).to_host()
        for f in "PQUV":
            np.testing.assert_allclose(getattr(dev, f), getattr(host, f), rtol=1e-13,
                                       atol=1e-15, err_msg=f"{name}.{f}")


def test_soliton_config1_matches_reference_error(golden):
    """BASELINE config 1: 1-D soliton, N=1024, tau=1e-3, T=1 -- same fields as
    the reference path, and the same error vs the exact solution."""
    c = golden.case("d1_soliton_N1024")
    s, tr = _integrate(c)
    assert_bitwise(s, c.state(1))
    exact = kgs.soliton1d_exact(c.grid, 1.0)
    h = c.grid.h
    err_u = np.sqrt(h * np.sum((s.U - exact.U)**2))
    assert err_u < 5e-3                       # reference: 2.21e-3 (SURVEY App.B)
    assert tr.max_rel_error() < 1e-11


def test_1024cubed_full_size_smoke():
    """The benchmark size fits and conserves energy over a few steps."""
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(1024)
    dev = kgs.DeviceFieldState.from_preset("ellipsoids3d", g)
    tr = kgs.integrate(dev, g, sc.params, kgs.checkerboard_schedule(g), None, 0.01, 0.03,
                       record_stride=1)
    assert dev.is_finite()
    assert tr.max_rel_error() < 1e-11
    dev.close()


def test_1024cubed_decomposition_invariance():
    """At the benchmark size: one slab (x wraps in the kernel) and 8 virtual
    slabs (fused halo stores between them) give the same bits.  After 3
    steps (7 passes) a decomposition error could only reach 7 planes from a
    slab boundary, so the planes within 8 of every boundary are compared."""
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(1024)
    args = kgs.precompute_coefficients(sc.params, 0.005, g).kernel_args()
    digests = []
    for ex in (None, kgs.CudaExecutor((0,), slabs_per_device=8)):
        dev = kgs.DeviceFieldState.from_preset("ellipsoids3d", g, ex)
        dev.ctx.step_dpavf2(args, 3, 0, 0)
        h = hashlib.sha256()
        buf = np.empty(16 * g.N * g.N)
        for f in range(4):
            for b in range(0, g.N, g.N // 8):          # slab boundaries (incl. the wrap)
                for x0 in ((b - 8) % g.N, b):
                    dev.ctx.download_planes(f, x0, buf[: 8 * g.N * g.N])
                    h.update(buf[: 8 * g.N * g.N].tobytes())
        digests.append(h.hexdigest())
        dev.close()
    assert digests[0] == digests[1]


def test_shared_reciprocal_division():
    """The kernels' shared-reciprocal quotient is bit-identical to IEEE `/`."""
    import ctypes
    from paper_2502_09537_b200 import _lib
    bad = ctypes.c_int64(-1)
    _lib.check(_lib.load().kgs_selftest_division(0, 1 << 26, 12345, ctypes.byref(bad)))
    assert bad.value == 0


_EXP = needs_experimental


_DEFAULT_VARIANTS = [(1, 0), (1, 1), (1, 2), (1, 3), (1, 128), (0, 8), (0, 1), (4, 0), (4, 3),
                     (4, 1), (4, 64)]
_EXP_VARIANTS = [(2, 5), (3, 0), (5, 0), (5, 1), (5, 7), (6, 0), (6, 2), (7, 0), (7, 5), (8, 0),
                 (8, 2), (9, 0), (9, 3), (10, 0), (10, 6), (11, 0), (11, 1), (12, 0), (12, 4),
                 (13, 0), (14, 3), (13, 16), (15, 0), (15, 1), (15, 5)]


@pytest.mark.parametrize("variant,xc", _DEFAULT_VARIANTS + [pytest.param(*v, marks=_EXP)
                                                            for v in _EXP_VARIANTS])
def test_march_kernel_matches_simple_kernel(variant, xc):
    """3-D marching (TMA ring) kernel == simple per-point kernel, bitwise, for
    every tile variant and several work-unit sizes (incl. a non-divisor)."""
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(256 if variant == 10 else 128)   # 8 x 128 tiles need 256 slots
    s0 = sc.state(g)
    args = kgs.precompute_coefficients(sc.params, 0.005, g).kernel_args()
    outs = []
    for planes in (-1, xc):
        dev = kgs.DeviceFieldState.from_host(s0, g)
        dev.ctx.set_tuning(march_planes=planes, march_variant=variant)
        terms, _ = dev.ctx.step_dpavf2(args, 5, 0, 5)
        outs.append((dev.to_host(), terms))
        dev.close()
    assert_bitwise(outs[0][0], outs[1][0])
    np.testing.assert_allclose(outs[0][1], outs[1][1], rtol=1e-13)


@pytest.mark.parametrize("xc", [0, 1, 5])
def test_march_own_tile_store_modes_are_bitwise(xc):
    """The march pass's own-tile write -- per-thread stores (tma_store 0), one
    TMA bulk store (1), bulk store with L2 evict-first (2, the default) --
    gives identical fields and records, incl. one-plane work units (every
    plane is a unit start: all three other-colour planes are waited for)."""
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(128)
    s0 = sc.state(g)
    args = kgs.precompute_coefficients(sc.params, 0.005, g).kernel_args()
    outs = []
    for mode in (0, 1, 2):
        dev = kgs.DeviceFieldState.from_host(s0, g)
        dev.ctx.set_tuning(march_planes=xc)
        dev.ctx.set_param("tma_store", mode)
        terms, bad = dev.ctx.step_dpavf2(args, 4, 0, 2)
        outs.append((dev.to_host(), terms, bad))
        dev.close()
    for st, terms, bad in outs[1:]:
        assert bad == outs[0][2] == 0
        assert_bitwise(st, outs[0][0])
        assert np.array_equal(terms, outs[0][1])


def test_step_at_a_time_with_deferred_tail_is_bitwise(golden):
    """Resident step_dpavf2 calls defer the last red adjoint into the next
    call's head; any later access (energy, download, sweep, coefficient
    change) sees exactly the reference state."""
    c = golden.case("d3_rand_N8")
    coeffs = kgs.precompute_coefficients(c.params, c.meta["tau"] / 2.0, c.grid)
    sch = kgs.checkerboard_schedule(c.grid)
    dev = kgs.DeviceFieldState.from_host(c.state(0), c.grid)
    ref = c.state(0)
    for k in range(1, 8):
        kgs.step_dpavf2(dev, sch, coeffs, None, c.grid)
        oracle.numpy_step_dpavf2(ref, c.kernel_args, c.grid)
        if k in (3, 7):
            assert_bitwise(dev.to_host(), ref)
            e = kgs.discrete_energy(dev, c.params, c.grid)
            assert e == pytest.approx(oracle.discrete_energy(ref, c.params, c.grid), rel=1e-13)
    # different coefficients after a deferred step: flush, then a fresh head
    other = kgs.precompute_coefficients(c.params, c.meta["tau"], c.grid)
    kgs.step_dpavf2(dev, sch, other, None, c.grid)
    oracle.numpy_step_dpavf2(ref, oracle.kernel_args(c.params, c.meta["tau"], c.grid), c.grid)
    assert_bitwise(dev.to_host(), ref)
    # a single sweep after a deferred step
    kgs.step_dpavf2(dev, sch, coeffs, None, c.grid)
    kgs.step_base(dev, sch, coeffs, None, c.grid)
    oracle.numpy_step_dpavf2(ref, c.kernel_args, c.grid)
    for colour in (1, 0):
        oracle.numpy_half_sweep(ref, c.kernel_args, c.grid, colour, False)
    assert_bitwise(dev.to_host(), ref)
    dev.close()


@pytest.mark.parametrize("N,steps,stride,slabs,planes", [
    (128, 7, 3, 1, 0), (256, 4, 4, 1, 0), (128, 1, 1, 1, 0), (64, 3, 1, 1, 0),
    (192, 3, 3, 1, 50), (128, 5, 5, 2, 0), (128, 4, 2, 4, 7), (64, 2, 1, 8, 0)])
@needs_experimental
@pytest.mark.parametrize("form", [1, 2])
def test_fused_step_matches_two_pass_and_oracle(N, steps, stride, slabs, planes, form):
    """One fused march per step (K3 on the tile + ring, K4 one plane behind,
    ping-pong buffer sets) gives the same bits as two colour passes, energy
    records equal to summation order, and (N <= 128) the same bits as the C
    oracle of the reference algorithm -- for one slab (x wraps in the
    kernel) and for several slabs (K4 boundary planes after the black face
    exchange), with chunk sizes that do not divide the slab."""
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(N)
    s0 = sc.state(g) if N <= 128 else None
    args = kgs.precompute_coefficients(sc.params, 0.005, g).kernel_args()
    ex = None if slabs == 1 else kgs.CudaExecutor((0,), slabs_per_device=slabs)
    outs = []
    for fused in (0, form):
        dev = (kgs.DeviceFieldState.from_host(s0, g, ex) if s0 is not None
               else kgs.DeviceFieldState.from_preset("ellipsoids3d", g, ex))
        dev.ctx.set_param("fused_step", fused)
        if planes:
            dev.ctx.set_param("fused_planes", planes)
        terms, bad = dev.ctx.step_dpavf2(args, steps, 0, stride)
        assert bad == 0
        outs.append((dev.to_host(), terms))
        dev.close()
    assert_bitwise(outs[0][0], outs[1][0])
    np.testing.assert_allclose(outs[0][1], outs[1][1], rtol=1e-13)
    if s0 is not None:
        ref = s0.copy()
        oracle.CheckerboardOracle(3, N).step_dpavf2(
            ref, args, steps, workers=oracle.CheckerboardOracle.max_threads())
        assert_bitwise(outs[1][0], ref)


@needs_experimental
@pytest.mark.parametrize("slabs", [1, 2])
def test_fused_step_deferred_tail_and_nonfinite(slabs):
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(128)
    s0 = sc.state(g)
    coeffs = kgs.precompute_coefficients(sc.params, 0.005, g)
    sch = kgs.checkerboard_schedule(g)
    ex = None if slabs == 1 else kgs.CudaExecutor((0,), slabs_per_device=slabs)
    dev = kgs.DeviceFieldState.from_host(s0, g, ex)
    ref = s0.copy()
    for _ in range(3):
        kgs.step_dpavf2(dev, sch, coeffs, ex, g)
    dev.ctx.step_dpavf2(coeffs.kernel_args(), 4, 3, 0)
    oracle.CheckerboardOracle(3, 128).step_dpavf2(ref, coeffs.kernel_args(), 7, workers=8)
    assert_bitwise(dev.to_host(), ref)
    bad = s0.copy()
    bad.U[12345] = np.inf
    dev.upload(bad)
    _, first_bad = dev.ctx.step_dpavf2(coeffs.kernel_args(), 3, 0, 0)
    assert first_bad == 1
    late = s0.copy()
    dev.upload(late)
    dev.ctx.step_dpavf2(coeffs.kernel_args(), 2, 0, 0)
    st = dev.to_host()
    st.P[777] = np.nan          # a red or black point of a middle plane
    dev.upload(st)
    _, first_bad = dev.ctx.step_dpavf2(coeffs.kernel_args(), 3, 2, 0)
    assert first_bad == 3
    dev.close()


@pytest.mark.parametrize("name", run_names())
def test_resident_kernel_matches_passes_and_reference(golden, name):
    """Small grids run a whole call in ONE launch with the state in shared
    memory; the fields are bitwise the per-pass path's (and the reference's),
    records equal to reduction order, for every golden run (records every
    step, a deferred tail, and a mid-call non-finite value)."""
    c = golden.case(name)
    args = c.kernel_args
    n = c.meta["n_steps"]
    outs = []
    for resident in (0, 1):
        dev = kgs.DeviceFieldState.from_host(c.state(0), c.grid)
        dev.ctx.set_param("resident", resident)
        terms, bad = dev.ctx.step_dpavf2(args, n, 0, 1)
        assert bad == 0
        dev.ctx.step_dpavf2(args, 2, n, 0, defer_tail=True)
        dev.ctx.step_dpavf2(args, 1, n + 2, 1)
        outs.append((dev.to_host(), terms))
        st = outs[-1][0].copy()
        st.V[st.V.size // 3] = np.nan
        dev.upload(st)
        _, first_bad = dev.ctx.step_dpavf2(args, 3, 10, 0)
        assert first_bad == 11
        dev.close()
    assert_bitwise(outs[0][0], outs[1][0])
    np.testing.assert_allclose(outs[0][1], outs[1][1], rtol=1e-13, atol=1e-300)
    ref = c.state(0)
    for _ in range(n + 3):
        oracle.numpy_step_dpavf2(ref, args, c.grid)
    assert_bitwise(outs[1][0], ref)


@pytest.mark.parametrize("scenario,N,steps,stride", [
    ("soliton1d", 1024, 37, 1), ("soliton1d", 1024, 16, 1), ("fourpeak2d", 64, 29, 3),
    ("ellipsoids3d", 16, 9, 1)])
def test_resident_record_batches(scenario, N, steps, stride):
    """The resident kernel stores its records in batches of 8 (per-warp sums,
    one block sum per batch): full and partial batches, strides > 1 -- the
    records equal the per-pass path's to reduction order and the fields
    stay bitwise."""
    sc = kgs.get_scenario(scenario)
    g = sc.default_grid(N)
    args = kgs.precompute_coefficients(sc.params, 0.005, g).kernel_args()
    outs = []
    for resident in (0, 1):
        dev = kgs.DeviceFieldState.from_preset(scenario, g)
        dev.ctx.set_param("resident", resident)
        terms, bad = dev.ctx.step_dpavf2(args, steps, 0, stride)
        assert bad == 0
        outs.append((dev.to_host(), np.asarray(terms)))
        dev.close()
    assert outs[1][1].shape == (steps // stride, 8)
    assert_bitwise(outs[0][0], outs[1][0])
    np.testing.assert_allclose(outs[1][1], outs[0][1], rtol=1e-13, atol=1e-300)


def test_oversized_grid_fails_cleanly_and_device_stays_usable():
    """2048^3 (275 GB) does not fit one B200: MemoryError naming the
    allocation, nothing leaked -- a normal context works right after."""
    g = kgs.GridSpec(3, -10.0, 10.0, 2048)
    with pytest.raises(MemoryError, match="cudaMalloc"):
        kgs.DeviceFieldState(g)
    sc = kgs.get_scenario("ellipsoids3d")
    g2 = sc.default_grid(64)
    dev = kgs.DeviceFieldState.from_preset("ellipsoids3d", g2)
    assert dev.is_finite()
    dev.close()


@pytest.mark.parametrize("N,slabs", [(64, 2), (128, 4), (96, 8), (16, 2)])
def test_fused_halo_stores_match_copy_exchange(N, slabs):
    """Single-process slabs exchange faces by storing them from the boundary
    launches straight into the neighbours' ghost planes (knob mirror_halo);
    the result is bitwise the copy-based exchange's and the oracle's, with
    records, single sweeps and step-at-a-time (deferred tail) calls mixed."""
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(N)
    s0 = sc.state(g)
    coeffs = kgs.precompute_coefficients(sc.params, 0.005, g)
    args = coeffs.kernel_args()
    sch = kgs.checkerboard_schedule(g)
    ex = kgs.CudaExecutor((0,), slabs_per_device=slabs)
    outs = []
    for mirror in (0, 1):
        dev = kgs.DeviceFieldState.from_host(s0, g, ex)
        dev.ctx.set_param("mirror_halo", mirror)
        terms, bad = dev.ctx.step_dpavf2(args, 4, 0, 2)
        assert bad == 0
        kgs.step_dpavf2(dev, sch, coeffs, ex, g)
        kgs.step_dpavf2(dev, sch, coeffs, ex, g)
        kgs.step_base(dev, sch, coeffs, ex, g)
        kgs.step_adjoint(dev, sch, coeffs, ex, g)
        outs.append((dev.to_host(), terms, kgs.discrete_energy(dev, sc.params, g)))
        dev.close()
    assert_bitwise(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])
    assert outs[0][2] == outs[1][2]
    ref = s0.copy()
    orc = oracle.CheckerboardOracle(3, N)
    orc.step_dpavf2(ref, args, 7, workers=oracle.CheckerboardOracle.max_threads())
    assert_bitwise(outs[1][0], ref)


@pytest.mark.parametrize("offset", [0.0, 40.0])
def test_record_forms_match_the_oracle(offset):
    """Both gradient-term forms of the record passes (knob record_form: 2 =
    sums of squares of the loaded neighbours, the default; 1 = differences
    to the pre-update value, cancellation-free) give the oracle's exactly
    summed energy terms; the fields do not depend on the form.  With a
    large constant offset on U the sum-of-squares form loses accuracy in
    proportion to (offset / neighbour difference)^2 -- the differences form
    does not."""
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(64)
    s0 = sc.state(g)
    s0.U += offset
    args = kgs.precompute_coefficients(sc.params, 0.005, g).kernel_args()
    ref = s0.copy()
    oracle.CheckerboardOracle(3, 64).step_dpavf2(
        ref, oracle.kernel_args(sc.params, 0.005, g), 3,
        workers=oracle.CheckerboardOracle.max_threads())
    want = oracle.energy_terms(ref, g)
    outs = {}
    for form in (2, 1):
        dev = kgs.DeviceFieldState.from_host(s0, g)
        dev.ctx.set_param("record_form", form)
        terms, bad = dev.ctx.step_dpavf2(args, 3, 0, 3)
        assert bad == 0
        outs[form] = (dev.to_host(), np.asarray(terms[-1]))
        dev.close()
    assert_bitwise(outs[1][0], outs[2][0])
    assert_bitwise(outs[1][0], ref)
    np.testing.assert_allclose(outs[1][1], want, rtol=1e-12, atol=1e-300)
    rel_u = abs(outs[2][1][2] - want[2]) / want[2]          # gradient sum of U
    assert rel_u < (1e-12 if offset == 0.0 else 1e-6), rel_u
    np.testing.assert_allclose(np.delete(outs[2][1], 2), np.delete(want, 2),
                               rtol=1e-12, atol=1e-300)


def test_record_form_knob_rejects_other_values():
    g = kgs.GridSpec(3, -1.0, 1.0, 16)
    dev = kgs.DeviceFieldState(g)
    with pytest.raises(ValueError, match="record_form"):
        dev.ctx.set_param("record_form", 0)
    dev.close()
