"""TEST INFRASTRUCTURE ONLY -- the parity oracle for the checkerboard DP-AVF2
path.  Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg; the product package never imports
it.

Two restatements of the reference algorithm (/root/reference/pkg/src/dpavf):

* ``CheckerboardOracle`` -- ctypes over ``kgs_oracle.c``: the reference's
  own structure (neighbour table, colour lanes, phased threads, per-point
  arithmetic of dpavf/kernels.py:23-94), compiled with -ffp-contract=off.
  Fast enough for 256^3 and used as the CPU baseline ("port").
* numpy functions below: a vectorised colour-phase step (SURVEY.md App.B
  showed it bitwise equal to the reference) and the energy/mass diagnostics
  written with the reference's own numpy reductions (dpavf/grid.py:152-187),
  so energies match the reference to the last bit.

Pinned against the reference: tests/golden/kgs_golden.npz was produced by
running the reference itself (tests/golden/make_golden.py); the CPU test
suite checks both restatements against it bit for bit.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "libkgs_oracle.so"
SRC = HERE / "kgs_oracle.c"
CFLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def build(force: bool = False) -> Path:
    """gcc the C restatement (seconds)."""
    if force or not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        tmp = LIB.with_suffix(".so.tmp")
        subprocess.run(["gcc", *CFLAGS, "-o", str(tmp), str(SRC)], check=True)
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(LIB))
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        L.orc_neighbor_table.argtypes = [ctypes.c_int, I64, P]
        L.orc_colour_lists.argtypes = [ctypes.c_int, I64, P, P]
        L.orc_colour_lists.restype = I64
        L.orc_phase.argtypes = [P, P, P, P, P, ctypes.c_int, P, I64, ctypes.c_int, P, ctypes.c_int]
        L.orc_step_dpavf2.argtypes = [P, P, P, P, P, ctypes.c_int, P, I64, P, I64, P, I64,
                                      ctypes.c_int]
        L.orc_max_threads.restype = ctypes.c_int
        L.orc_free_sweep.argtypes = [ctypes.c_int, I64, P, P, P, P, ctypes.c_int, P]
        L.orc_free_step_dpavf2.argtypes = [ctypes.c_int, I64, P, P, P, P, P, I64]
        L.orc_energy_row_terms.argtypes = [ctypes.c_int, I64, P, P, P, P, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class CheckerboardOracle:
    """Reference-structured CPU stepper for one grid (d, N)."""

    def __init__(self, d: int, N: int):
        if N % 2:
            raise ValueError("checkerboard needs even N")
        self.d, self.N = d, N
        self.M = N**d
        self.nn = 2 * d
        L = lib()
        self.nbrs = np.empty((self.M, self.nn), dtype=np.int64)
        L.orc_neighbor_table(d, N, _p(self.nbrs))
        red = np.empty(self.M, dtype=np.int64)
        black = np.empty(self.M, dtype=np.int64)
        nr = L.orc_colour_lists(d, N, _p(red), _p(black))
        self.red = red[:nr].copy()
        self.black = black[:self.M - nr].copy()

    @staticmethod
    def max_threads() -> int:
        return int(lib().orc_max_threads())

    def _fields(self, state):
        f = [state.P, state.Q, state.U, state.V]
        for a in f:
            assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"] and a.shape == (self.M,)
        return f

    def sweep(self, state, kernel_args, adjoint: bool, workers: int = 1) -> None:
        """step_base (red, black) or step_adjoint (black, red), in place."""
        c = np.asarray(kernel_args, dtype=np.float64)
        f = self._fields(state)
        order = (self.black, self.red) if adjoint else (self.red, self.black)
        for idx in order:
            lib().orc_phase(*map(_p, f), _p(self.nbrs), self.nn, _p(idx), idx.shape[0],
                            int(adjoint), _p(c), workers)

    def step_dpavf2(self, state, kernel_args, nsteps: int = 1, workers: int = 1) -> None:
        c = np.asarray(kernel_args, dtype=np.float64)
        f = self._fields(state)
        lib().orc_step_dpavf2(*map(_p, f), _p(self.nbrs), self.nn, _p(self.red),
                              self.red.shape[0], _p(self.black), self.black.shape[0],
                              _p(c), nsteps, workers)


class TableFreeOracle:
    """The same restatement without the (M, 2d) neighbour table or index
    lists: periodic neighbours computed from coordinates, rows in parallel
    (kgs_oracle.c, ``orc_free_*``).  For grids whose table does not fit in
    host memory -- the 1024^3 headline config (tests/test_gpu_headline.py).
    Pinned to the golden vectors like ``CheckerboardOracle``."""

    def __init__(self, d: int, N: int):
        if N % 2:
            raise ValueError("checkerboard needs even N")
        self.d, self.N, self.M = d, N, N**d

    def _fields(self, state):
        f = [state.P, state.Q, state.U, state.V]
        for a in f:
            assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"] and a.shape == (self.M,)
        return f

    def sweep(self, state, kernel_args, adjoint: bool) -> None:
        c = np.asarray(kernel_args, dtype=np.float64)
        lib().orc_free_sweep(self.d, self.N, *map(_p, self._fields(state)), int(adjoint), _p(c))

    def step_dpavf2(self, state, kernel_args, nsteps: int = 1) -> None:
        c = np.asarray(kernel_args, dtype=np.float64)
        lib().orc_free_step_dpavf2(self.d, self.N, *map(_p, self._fields(state)), _p(c), nsteps)

    def energy_terms(self, state) -> np.ndarray:
        """The 8 unscaled sums (as ``energy_terms`` below): per-row partials
        in C, rows summed exactly."""
        import math
        rows = (self.N**(self.d - 1)) if self.d > 1 else 1
        part = np.empty((rows, 8))
        lib().orc_energy_row_terms(self.d, self.N, *map(_p, self._fields(state)), _p(part))
        return np.array([math.fsum(part[:, k]) for k in range(8)])


# ---------------------------------------------------------------------------
# numpy restatement
# ---------------------------------------------------------------------------
def kernel_args(params, tau: float, grid) -> tuple:
    """precompute_coefficients(params, tau, grid).kernel_args()
    (dpavf/integrator.py:42-64)."""
    h2 = grid.h**2
    d = grid.d
    alpha = tau * params.kappa1 * d / (2.0 * h2)
    beta = tau * params.kappa1 / (2.0 * h2)
    gcoef = tau * params.gamma / 2.0
    c_uv = tau * params.kappa2 * d / h2 + tau * params.mu**2 / 2.0
    det = 1.0 + (tau / 2.0) * c_uv
    uv_nbr = tau * params.kappa2 / h2
    gU = tau * params.gamma
    return (alpha, beta, gcoef, c_uv, uv_nbr, gU, tau / 2.0,
            1.0 / det, (tau / 2.0) / det, -c_uv / det, 1.0 / det)


def _nbr_sum(f: np.ndarray, shape) -> np.ndarray:
    """0.0 + f[-x] + f[+x] + f[-y] + ... in canonical order (kernels.py:35-42)."""
    g = f.reshape(shape)
    s = np.zeros(shape)
    for ax in range(len(shape)):
        s = s + np.roll(g, 1, axis=ax)
        s = s + np.roll(g, -1, axis=ax)
    return s.ravel()


def colour_mask(grid, colour: int) -> np.ndarray:
    return (np.indices(grid.shape).sum(axis=0).ravel() % 2) == colour


def numpy_half_sweep(state, kernel_args, grid, colour: int, adjoint: bool) -> None:
    """Update every point of one colour from the current arrays (its
    neighbours all have the other colour), in place."""
    alpha, beta, gcoef, c_uv, uv_nbr, gU, half_tau, i00, i01, i10, i11 = kernel_args
    P, Q, U, V = state.P, state.Q, state.U, state.V
    SP, SQ, SU = (_nbr_sum(a, grid.shape) for a in (P, Q, U))
    m = colour_mask(grid, colour)
    Pi, Qi, Ui, Vi = P[m], Q[m], U[m], V[m]
    SP, SQ, SU = SP[m], SQ[m], SU[m]
    if not adjoint:
        cr = gcoef * Ui - alpha
        rr = -cr * Pi - Qi - beta * SP
        ri = Pi - cr * Qi - beta * SQ
        den = cr * cr + 1.0
        Pn = (rr * cr + ri) / den
        Qn = (ri * cr - rr) / den
        r1 = Ui + half_tau * Vi
        r2 = Vi - c_uv * Ui + uv_nbr * SU + gU * (Pn * Pn + Qn * Qn)
        Un = i00 * r1 + i01 * r2
        Vn = i10 * r1 + i11 * r2
    else:
        r1 = Ui + half_tau * Vi
        r2 = Vi - c_uv * Ui + uv_nbr * SU + gU * (Pi * Pi + Qi * Qi)
        Un = i00 * r1 + i01 * r2
        Vn = i10 * r1 + i11 * r2
        cr = gcoef * Un - alpha
        rr = -cr * Pi - Qi - beta * SP
        ri = Pi - cr * Qi - beta * SQ
        den = cr * cr + 1.0
        Pn = (rr * cr + ri) / den
        Qn = (ri * cr - rr) / den
    P[m], Q[m], U[m], V[m] = Pn, Qn, Un, Vn


def numpy_step_dpavf2(state, kernel_args, grid, nsteps: int = 1) -> None:
    for _ in range(nsteps):
        numpy_half_sweep(state, kernel_args, grid, 1, False)
        numpy_half_sweep(state, kernel_args, grid, 0, False)
        numpy_half_sweep(state, kernel_args, grid, 0, True)
        numpy_half_sweep(state, kernel_args, grid, 1, True)


def _grad_sq_sum(field: np.ndarray, grid) -> float:
    """dpavf/grid.py:152-163."""
    f = field.reshape(grid.shape)
    total = 0.0
    for ax in range(grid.d):
        diff = (np.roll(f, -1, axis=ax) - f) / grid.h
        total += float(np.sum(diff * diff))
    return total


def discrete_energy(state, params, grid) -> float:
    """dpavf/grid.py:166-181."""
    quad = (params.kappa1 * _grad_sq_sum(state.P, grid)
            + params.kappa1 * _grad_sq_sum(state.Q, grid)
            + params.kappa2 * _grad_sq_sum(state.U, grid)
            + float(np.dot(state.V, state.V))
            + params.mu**2 * float(np.dot(state.U, state.U)))
    coupling = float(np.dot(state.P * state.P + state.Q * state.Q, state.U))
    return grid.h**grid.d * (0.5 * quad - params.gamma * coupling)


def mass(state, grid) -> float:
    """dpavf/grid.py:184-187."""
    return grid.h**grid.d * float(np.dot(state.P, state.P) + np.dot(state.Q, state.Q))


def energy_terms(state, grid) -> np.ndarray:
    """The 8 unscaled sums the device returns (include/kgs_b200.h), exact
    (math.fsum), for checking the device reduction."""
    import math
    out = np.zeros(8)
    for q, f in enumerate((state.P, state.Q, state.U)):
        g = f.reshape(grid.shape)
        tot = []
        for ax in range(grid.d):
            dlt = (np.roll(g, -1, axis=ax) - g).ravel()
            tot.append(dlt * dlt)
        out[q] = math.fsum(np.concatenate(tot))
    P, Q, U, V = state.P, state.Q, state.U, state.V
    out[3] = math.fsum(V * V)
    out[4] = math.fsum(U * U)
    out[5] = math.fsum((P * P + Q * Q) * U)
    out[6] = math.fsum(P * P)
    out[7] = math.fsum(Q * Q)
    return out
