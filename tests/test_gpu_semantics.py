"""Device analogues of the reference's point-kernel and integrate semantics
tests (dpavf tests/test_integrator.py): exact special cases of the update
formulas, sweep-level round trips and the integrate() bookkeeping, on the
GPU path (single-colour sweeps keep the other colour frozen, which is the
per-point tests' setting)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2502_09537_b200 as kgs
from conftest import assert_bitwise

pytestmark = pytest.mark.gpu
RED, BLACK, BASE, ADJ = 1, 0, 0, 1


def _dev(state, g):
    return kgs.DeviceFieldState.from_host(state, g)


@pytest.mark.parametrize("d,N", [(2, 8), (3, 8), (3, 64)])
def test_psi_unchanged_when_decoupled(d, N):
    """kappa1 = gamma = 0: the Psi solve is the identity -- P, Q bitwise
    unchanged by base and adjoint sweeps (tests/test_integrator.py:53-61)."""
    g = kgs.GridSpec(d, 0.0, 4.0, N)
    s = kgs.seeded_random_state(g, 1, 0.5) if g.M <= 4096 else \
        kgs.get_scenario("ellipsoids3d").state(g)
    c = kgs.precompute_coefficients(kgs.PhysParams(0.0, 1.0, 1.0, 0.0), 0.3, g)
    dev = _dev(s, g)
    sch = kgs.checkerboard_schedule(g)
    kgs.step_base(dev, sch, c, None, g)
    kgs.step_adjoint(dev, sch, c, None, g)
    out = dev.to_host()
    dev.close()
    assert np.array_equal(out.P, s.P) and np.array_equal(out.Q, s.Q)
    assert not np.array_equal(out.U, s.U)


def test_oscillator_half_period_exact():
    """kappa2 = gamma = 0, mu = 1, tau = 2: (U, V) = (1, 0) -> (0, -1)
    exactly (tests/test_integrator.py:63-71), every point at once."""
    g = kgs.GridSpec(1, 0.0, 4.0, 4)
    c = kgs.precompute_coefficients(kgs.PhysParams(1.0, 0.0, 1.0, 0.0), 2.0, g)
    s = kgs.FieldState.zeros(g)
    s.U[:] = 1.0
    dev = _dev(s, g)
    kgs.step_base(dev, kgs.checkerboard_schedule(g), c, None, g)
    out = dev.to_host()
    dev.close()
    assert np.all(out.U == 0.0) and np.all(out.V == -1.0)


def test_zero_is_a_fixed_point():
    g = kgs.GridSpec(3, 0.0, 1.0, 8)
    s = kgs.FieldState.zeros(g)
    dev = _dev(s, g)
    dev.ctx.step_dpavf2(kgs.precompute_coefficients(kgs.PhysParams(), 0.05, g).kernel_args(), 5)
    out = dev.to_host()
    dev.close()
    for f in "PQUV":
        assert not np.any(getattr(out, f))


@pytest.mark.parametrize("colour", [RED, BLACK])
def test_gamma_zero_base_equals_adjoint(colour):
    """gamma = 0 decouples Psi and (U, V), so base and adjoint updates of a
    colour agree bitwise (tests/test_integrator.py:82-90)."""
    g = kgs.GridSpec(2, 0.0, 1.0, 16)
    c = kgs.precompute_coefficients(kgs.PhysParams(1.0, 1.0, 1.0, 0.0), 0.2, g).kernel_args()
    s = kgs.seeded_random_state(g, 8, 0.4)
    outs = []
    for kind in (BASE, ADJ):
        dev = _dev(s, g)
        dev.ctx.sweep(colour, kind, c)
        outs.append(dev.to_host())
        dev.close()
    assert_bitwise(outs[0], outs[1])


@pytest.mark.parametrize("colour", [RED, BLACK])
def test_adjoint_then_negative_base_restores_a_colour(colour):
    """adjoint(tau) then base(-tau) with the other colour frozen restores the
    swept colour to 1e-13 (tests/test_integrator.py:92-103)."""
    g = kgs.GridSpec(2, 0.0, 1.0, 16)
    p = kgs.PhysParams(0.9, 1.1, 1.2, 0.7)
    s = kgs.seeded_random_state(g, 4, 0.5)
    dev = _dev(s, g)
    dev.ctx.sweep(colour, ADJ, kgs.precompute_coefficients(p, 0.05, g).kernel_args())
    dev.ctx.sweep(colour, BASE, kgs.precompute_coefficients(p, -0.05, g).kernel_args())
    out = dev.to_host()
    dev.close()
    for f in "PQUV":
        np.testing.assert_allclose(getattr(out, f), getattr(s, f), rtol=1e-13, atol=1e-13)


class TestIntegrateBookkeeping:
    """tests/test_integrator.py:125-234 on the device path."""

    def _setup(self):
        g = kgs.GridSpec(2, -1.0, 1.0, 8)
        p = kgs.PhysParams(0.8, 1.2, 1.1, 0.9)
        return g, p, kgs.seeded_random_state(g, 3, 0.5), kgs.checkerboard_schedule(g)

    def test_t_advances(self):
        g, p, s, sch = self._setup()
        c = kgs.precompute_coefficients(p, 0.25, g)
        kgs.step_base(s, sch, c, None, g)
        assert s.t == pytest.approx(0.25)
        kgs.step_adjoint(s, sch, c, None, g)
        assert s.t == pytest.approx(0.5)

    def test_T_zero_single_record(self):
        g, p, s, sch = self._setup()
        before = s.copy()
        tr = kgs.integrate(s, g, p, sch, None, 0.1, 0.0)
        assert tr.steps == [0] and tr.rel_error == [0.0]
        assert_bitwise(s, before)

    def test_trace_length_stride_and_mass(self):
        g, p, s, sch = self._setup()
        tr = kgs.integrate(s, g, p, sch, None, 0.05, 1.0, record_stride=3)
        assert len(tr.steps) == 20 // 3 + 1 and tr.steps[1] == 3
        assert len(tr.mass) == len(tr.steps)
        assert tr.mass[0] == pytest.approx(kgs.mass(self._setup()[2], g), rel=1e-14)

    def test_snapshot_callback_cadence(self):
        g, p, s, sch = self._setup()
        seen = []
        kgs.integrate(s, g, p, sch, None, 0.1, 1.0, snapshot_stride=4,
                      snapshot_writer=lambda st, n: seen.append((n, st.t)))
        assert [n for n, _ in seen] == [4, 8]
        assert seen[0][1] == pytest.approx(0.4)

    def test_energy_trace_machine_precision(self):
        g, p, s, sch = self._setup()
        tr = kgs.integrate(s, g, p, sch, None, 0.05, 2.0)
        assert tr.max_rel_error() <= 1e-12 and tr.rel_error[0] == 0.0


def test_closed_cached_context_is_replaced():
    """A temporary device state shares the cached context of its grid;
    closing it must not poison later host-state calls on that grid."""
    from paper_2502_09537_b200.device import as_device_state
    g = kgs.GridSpec(2, 0.0, 4.0, 16)
    s = kgs.seeded_random_state(g, 3, 0.5)
    e0 = kgs.discrete_energy(s, kgs.PhysParams(), g)
    dev, temporary = as_device_state(s, g)
    assert temporary
    dev.close()                       # closes the cached context
    assert kgs.discrete_energy(s, kgs.PhysParams(), g) == e0


@pytest.mark.parametrize("d,N,march", [(1, 4096, False), (2, 96, False), (3, 32, False),
                                       (3, 64, True)])
def test_programmatic_dependent_launch_is_bitwise_neutral(d, N, march):
    """The colour passes (per-point and marching) and the record reductions
    launched as programmatic dependents of the previous kernel (knob "pdl",
    default on) give the plain stream-ordered result bit for bit, records
    included."""
    g = kgs.GridSpec(d, -4.0, 4.0, N)
    s = kgs.seeded_random_state(g, 5, 0.5)
    a = kgs.precompute_coefficients(kgs.PhysParams(), 0.01, g).kernel_args()
    res = []
    for pdl in (0, 1):
        dev = _dev(s, g)
        dev.ctx.set_param("resident", 0)
        if not march:
            dev.ctx.set_param("march_planes", -1)     # per-point kernel for every d
        dev.ctx.set_param("pdl", pdl)
        terms, bad = dev.ctx.step_dpavf2(a, 7, 0, 2)
        res.append((dev.to_host(), terms, bad))
        dev.close()
    (s0, t0, b0), (s1, t1, b1) = res
    assert b0 == b1 == 0 and np.array_equal(t0, t1)
    assert_bitwise(s1, s0)
