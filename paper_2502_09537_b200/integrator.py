"""Time integrators: base and adjoint sweeps, DP-AVF2, and the run loop.

Same names, signatures and semantics as the reference ``dpavf.integrator``
(dpavf/integrator.py), with the sweeps executed by the sm_100a colour-pass
kernels of ``libkgs_b200.so``:

* ``precompute_coefficients`` is the reference's host arithmetic verbatim
  (integrator.py:48-64) -- the 11 kernel scalars must be bit-identical;
* ``step_base`` = red then black base half-sweeps; ``step_adjoint`` = black
  then red adjoint half-sweeps; ``step_dpavf2`` = base then adjoint at tau/2
  (integrator.py:107-129, ordering.py:139-149);
* ``integrate`` (integrator.py:147-182) runs the fused stepping loop on the
  device (2 colour passes per step, energy/mass/finiteness fused into them)
  and fills the same ``EnergyTrace``.

State arguments may be a host ``FieldState`` (uploaded, stepped, copied
back in place) or a :class:`~paper_2502_09537_b200.device.DeviceFieldState`
(stepped in place on the GPU).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .device import DeviceFieldState, as_device_state, get_context
from .grid import FieldState, GridSpec, PhysParams, energy_from_terms
from .ordering import colour_order, is_reversed, require_checkerboard

KIND_BASE, KIND_ADJOINT = 0, 1


@dataclass(frozen=True)
class StepCoefficients:
    """Precomputed pointwise solve constants for step size tau
    (reference integrator.py:22-45)."""

    tau: float
    alpha: float      # Psi center weight  tau*kappa1*d / (2 h^2)
    beta: float       # Psi neighbor weight  tau*kappa1 / (2 h^2)
    gcoef: float      # Psi coupling weight  tau*gamma / 2
    c_uv: float       # tau*kappa2*d/h^2 + tau*mu^2/2
    uv_nbr: float     # tau*kappa2 / h^2
    gU: float         # tau*gamma
    uv_inv: tuple     # ((i00, i01), (i10, i11))

    def kernel_args(self) -> tuple:
        (i00, i01), (i10, i11) = self.uv_inv
        return (self.alpha, self.beta, self.gcoef, self.c_uv, self.uv_nbr,
                self.gU, self.tau / 2.0, i00, i01, i10, i11)


def precompute_coefficients(params: PhysParams, tau: float,
                            grid: GridSpec) -> StepCoefficients:
    """Host arithmetic identical to reference integrator.py:48-64."""
    if tau == 0.0 or not math.isfinite(tau):
        raise ValueError(f"step size must be nonzero and finite, got tau={tau}")
    h2 = grid.h**2
    d = grid.d
    alpha = tau * params.kappa1 * d / (2.0 * h2)
    beta = tau * params.kappa1 / (2.0 * h2)
    gcoef = tau * params.gamma / 2.0
    c_uv = tau * params.kappa2 * d / h2 + tau * params.mu**2 / 2.0
    det = 1.0 + (tau / 2.0) * c_uv
    if det == 0.0:
        raise ValueError(f"singular U-V system: 1 + (tau/2)*c_uv = 0 at tau={tau}")
    uv_inv = ((1.0 / det, (tau / 2.0) / det),
              (-c_uv / det, 1.0 / det))
    return StepCoefficients(tau, alpha, beta, gcoef, c_uv,
                            tau * params.kappa2 / h2, tau * params.gamma, uv_inv)


def _colours(schedule, grid: GridSpec, adjoint: bool) -> tuple[int, int]:
    """Colour order of one sweep: the schedule's own (ours, or the
    reference's UpdateSchedule incl. reverse_schedule'd ones), reversed for
    the adjoint (integrator.py:115-121)."""
    order = colour_order(schedule, grid)
    return tuple(reversed(order)) if adjoint else order


def _sweep(state, schedule, coeffs: StepCoefficients, executor, grid: GridSpec,
           kind: int) -> None:
    require_checkerboard(schedule, grid)
    dev, temp = as_device_state(state, grid, executor)
    args = coeffs.kernel_args()
    for colour in _colours(schedule, grid, kind == KIND_ADJOINT):
        dev.ctx.sweep(colour, kind, args)
    if temp:
        dev.ctx.download(state)
    state.t += coeffs.tau


def step_base(state, schedule, coeffs: StepCoefficients, executor,
              grid: GridSpec) -> None:
    """One base sweep over all points (red, then black); advances state.t by
    coeffs.tau (reference integrator.py:107-112)."""
    _sweep(state, schedule, coeffs, executor, grid, KIND_BASE)


def step_adjoint(state, schedule, coeffs: StepCoefficients, executor,
                 grid: GridSpec) -> None:
    """One adjoint sweep along the reversed schedule (black, then red);
    advances t by coeffs.tau (reference integrator.py:115-121)."""
    _sweep(state, schedule, coeffs, executor, grid, KIND_ADJOINT)


def step_dpavf2(state, schedule, coeffs_half: StepCoefficients, executor,
                grid: GridSpec) -> None:
    """Symmetric composition: base then adjoint, each at tau/2
    (reference integrator.py:124-129), as one fused device call."""
    require_checkerboard(schedule, grid)
    if is_reversed(schedule, grid):
        # a reversed schedule swaps the colour order of both halves
        step_base(state, schedule, coeffs_half, executor, grid)
        step_adjoint(state, schedule, coeffs_half, executor, grid)
        return
    dev, temp = as_device_state(state, grid, executor)
    # resident states defer the last red adjoint into the next call's head
    # (2 passes per step instead of 3; bitwise neutral, see kgs_b200.h)
    dev.ctx.step_dpavf2(coeffs_half.kernel_args(), 1, defer_tail=not temp)
    if temp:
        dev.ctx.download(state)
    state.t += coeffs_half.tau
    state.t += coeffs_half.tau


@dataclass
class EnergyTrace:
    """Per-record energy bookkeeping along an integration
    (reference integrator.py:132-144)."""

    steps: list
    times: list
    energy: list
    rel_error: list
    mass: list
    re_is_absolute: bool = False  # set when |E0| underflows the RE ratio

    def max_rel_error(self) -> float:
        return max(self.rel_error)


def _pipeline_ok(host, sizes) -> bool:
    """The one-call path hands the host arrays to C as raw pointers: they must
    be contiguous, writable float64 of one of `sizes` (the whole grid, or a
    rank's own slab) -- else the checked path runs."""
    for f in "PQUV":
        a = getattr(host, f)
        if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.ndim == 1
                and a.size in sizes and a.flags["C_CONTIGUOUS"] and a.flags["WRITEABLE"]):
            return False
    return True


def _one_call_ok(ctx, host, grid: GridSpec) -> bool:
    """The host arrays suit kgs_integrate_host; the ranks of a torchrun job
    agree on it (the call's halo exchanges are collective)."""
    ok = _pipeline_ok(host, (grid.M, ctx.points) if ctx.dist else (grid.M,))
    if ctx.dist and ctx.plan.world_size > 1:
        from .device import _torch_allgather
        ok = all(_torch_allgather(ok))
    return ok


def _append_records(trace, terms, k0, k1, record_stride, t, e0, absolute, params, grid,
                    advance_t) -> float:
    """Append the records of steps k0..k1 (every record_stride-th) from the
    device term sums; returns t after step k1."""
    rec = iter(terms)
    for k in range(k0, k1 + 1):
        t = advance_t(t, 1)
        if k % record_stride == 0:
            e, m = energy_from_terms(next(rec), params, grid)
            re = abs(e - e0) if absolute else abs(e - e0) / abs(e0)
            trace.steps.append(k)
            trace.times.append(t)
            trace.energy.append(e)
            trace.rel_error.append(re)
            trace.mass.append(m)
    return t


def _integrate_stepwise(state, grid, params, schedule, executor, tau, n_steps, record_stride,
                        snapshot_stride, snapshot_writer) -> EnergyTrace:
    """The reference loop (integrator.py:159-182) one step_dpavf2 call at a
    time -- for schedules the fused loop does not cover (a reversed
    checkerboard: black sweeps first in both halves)."""
    coeffs_half = precompute_coefficients(params, tau / 2.0, grid)
    dev, temp = as_device_state(state, grid, executor)
    e0, m0 = energy_from_terms(dev.energy_terms(), params, grid)
    absolute = abs(e0) < 1e-300
    trace = EnergyTrace([0], [state.t], [e0], [0.0], [m0], re_is_absolute=absolute)
    for n in range(1, n_steps + 1):
        step_dpavf2(dev, schedule, coeffs_half, executor, grid)
        state.t = dev.t
        if not dev.is_finite():
            if temp:
                dev.ctx.download(state)
            raise FloatingPointError(
                f"non-finite field values detected after step {n} (t={state.t})")
        if n % record_stride == 0:
            e, m = energy_from_terms(dev.energy_terms(), params, grid)
            trace.steps.append(n)
            trace.times.append(state.t)
            trace.energy.append(e)
            trace.rel_error.append(abs(e - e0) if absolute else abs(e - e0) / abs(e0))
            trace.mass.append(m)
        if snapshot_stride and snapshot_writer and n % snapshot_stride == 0:
            if temp:
                dev.ctx.download(state)
            snapshot_writer(state, n)
    if temp:
        dev.ctx.download(state)
    return trace


def integrate(state, grid: GridSpec, params: PhysParams,
              schedule, executor, tau: float, T: float,
              record_stride: int = 1, snapshot_stride: int = 0,
              snapshot_writer=None) -> EnergyTrace:
    """Run ceil(T/tau) composed steps on the GPU, recording energy and mass.

    Reference integrator.py:147-182.  The relative energy error is
    |E_n - E_0| / |E_0|; when E_0 underflows the quotient the absolute drift
    is recorded instead and flagged.  Non-finite values raise
    FloatingPointError naming the first bad step; for a host state the
    state is left exactly as the reference leaves it (after that step).
    """
    if tau <= 0 or T < 0:
        raise ValueError(f"need tau > 0 and T >= 0, got tau={tau}, T={T}")
    if record_stride < 1:
        raise ValueError("record_stride must be >= 1")
    require_checkerboard(schedule, grid)
    n_steps = int(math.ceil(T / tau - 1e-12)) if T > 0 else 0
    if is_reversed(schedule, grid):
        return _integrate_stepwise(state, grid, params, schedule, executor, tau, n_steps,
                                   record_stride, snapshot_stride, snapshot_writer)
    coeffs_half = precompute_coefficients(params, tau / 2.0, grid)
    args = coeffs_half.kernel_args()

    host = None if isinstance(state, DeviceFieldState) else state
    snap = snapshot_stride if (snapshot_stride and snapshot_writer) else 0

    def advance_t(t: float, k: int) -> float:
        for _ in range(k):       # t += tau/2 twice per step, like the reference
            t += coeffs_half.tau
            t += coeffs_half.tau
        return t

    ctx = get_context(grid, executor) if host is not None and not snap and n_steps > 0 else None
    if ctx is not None and _one_call_ok(ctx, host, grid):
        # one call: upload | steps | download overlapped (kgs_integrate_host;
        # several slabs or ranks run the pipeline side by side with face
        # exchanges; every rank of a torchrun job makes this same call)
        t_start = state.t
        terms0, terms, bad = ctx.integrate_host(host, args, n_steps, record_stride)
        e0, m0 = energy_from_terms(terms0, params, grid)
        absolute = abs(e0) < 1e-300
        trace = EnergyTrace([0], [t_start], [e0], [0.0], [m0], re_is_absolute=absolute)
        if bad:
            state.t = advance_t(t_start, bad)
            raise FloatingPointError(
                f"non-finite field values detected after step {bad} (t={state.t})")
        state.t = _append_records(trace, terms, 1, n_steps, record_stride, t_start, e0,
                                  absolute, params, grid, advance_t)
        return trace

    dev, _ = as_device_state(state, grid, executor)

    e0, m0 = energy_from_terms(dev.energy_terms(), params, grid)
    absolute = abs(e0) < 1e-300
    trace = EnergyTrace([0], [state.t], [e0], [0.0], [m0], re_is_absolute=absolute)

    # chunk boundaries: snapshot steps (the host state is synced there)
    n = 0
    while n < n_steps:
        n1 = n_steps if not snap else min(n_steps, (n // snap + 1) * snap)
        t_start = state.t
        # a device-resident state keeps a device copy of the chunk start so
        # a non-finite step can be replayed exactly (host states are re-uploaded)
        terms, bad = dev.ctx.step_dpavf2(args, n1 - n, n, record_stride,
                                         backup=host is None)
        if bad:
            if host is not None:
                # restore the step-n host state and replay exactly to `bad`
                dev.ctx.upload(host)
                dev.ctx.step_dpavf2(args, bad - n, n, 0)
                dev.ctx.download(host)
                state.t = advance_t(t_start, bad - n)
            elif dev.ctx.restore_backup():
                dev.ctx.step_dpavf2(args, bad - n, n, 0)
                state.t = advance_t(t_start, bad - n)
            else:   # no memory for the copy: fields and t both after step n1
                state.t = advance_t(t_start, n1 - n)
                raise FloatingPointError(
                    f"non-finite field values detected after step {bad} (t="
                    f"{advance_t(t_start, bad - n)}); the device state could not be "
                    f"rewound and is left after step {n1} (t={state.t})")
            raise FloatingPointError(
                f"non-finite field values detected after step {bad} (t={state.t})")
        state.t = _append_records(trace, terms, n + 1, n1, record_stride, t_start, e0,
                                  absolute, params, grid, advance_t)
        n = n1
        if snap and n % snap == 0:
            if host is not None:
                dev.ctx.download(host)
                snapshot_writer(host, n)
            else:
                snapshot_writer(state, n)
    if host is not None:
        dev.ctx.download(host)
    return trace
