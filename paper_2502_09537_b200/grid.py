"""Periodic grid geometry, field storage and the energy/mass diagnostics.

Mirrors ``dpavf.grid`` (reference ``dpavf/grid.py``) for the checkerboard
path: ``GridSpec`` (grid.py:16-64), ``PhysParams`` (:67-79), ``FieldState``
(:82-103), ``discrete_energy`` (:166-169), ``raw_energy`` (:172-181) and
``mass`` (:184-187), with the same names, argument meaning and errors.

Fields are stored flat with the reference linearisation
``i = x*N**(d-1) + y*N**(d-2) + z`` (first axis slowest).  The diagnostics
run on the GPU: a host ``FieldState`` is uploaded to a cached device
context, a :class:`~paper_2502_09537_b200.device.DeviceFieldState` is
reduced in place.  There is no numpy fallback.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class GridSpec:
    """Uniform periodic Cartesian grid, same endpoints and N per axis."""

    d: int
    a: float
    b: float
    N: int

    def __post_init__(self):
        if self.d not in (1, 2, 3):
            raise ValueError(f"dimension must be 1, 2 or 3, got {self.d}")
        if not self.b > self.a:
            raise ValueError(f"need b > a, got a={self.a}, b={self.b}")
        if self.N < 2:
            raise ValueError(f"need N >= 2, got N={self.N}")

    @property
    def h(self) -> float:
        return (self.b - self.a) / self.N

    @property
    def M(self) -> int:
        return self.N**self.d

    @property
    def shape(self) -> tuple[int, ...]:
        return (self.N,) * self.d

    def axis_coords(self) -> np.ndarray:
        """Node coordinates along one axis: a + j*h for j = 0..N-1."""
        return self.a + self.h * np.arange(self.N)

    def meshgrid(self) -> tuple[np.ndarray, ...]:
        """d coordinate arrays of shape ``self.shape`` ('ij' indexing)."""
        x = self.axis_coords()
        return np.meshgrid(*([x] * self.d), indexing="ij")


@dataclass(frozen=True)
class PhysParams:
    """Physical constants of the coupled nucleon/meson system."""

    kappa1: float = 1.0
    kappa2: float = 1.0
    mu: float = 1.0
    gamma: float = 1.0

    def __post_init__(self):
        for name in ("kappa1", "kappa2", "mu", "gamma"):
            if not np.isfinite(getattr(self, name)):
                raise ValueError(f"{name} must be finite")


@dataclass
class FieldState:
    """The four real scalar fields (Psi = P + iQ, meson U, velocity V) on the
    host, exactly as the reference's FieldState (grid.py:82-103)."""

    P: np.ndarray
    Q: np.ndarray
    U: np.ndarray
    V: np.ndarray
    t: float = 0.0

    @classmethod
    def zeros(cls, grid: GridSpec) -> "FieldState":
        M = grid.M
        return cls(np.zeros(M), np.zeros(M), np.zeros(M), np.zeros(M), 0.0)

    @classmethod
    def pinned(cls, grid: GridSpec, zero: bool = True) -> "FieldState":
        """State whose arrays live in page-locked host memory (fast,
        asynchronous host<->device copies; used for end-to-end timing);
        zero-filled unless ``zero=False`` (the caller fills every value)."""
        from .device import pinned_empty
        f = [pinned_empty(grid.M) for _ in range(4)]
        if zero:
            for a in f:
                a.fill(0.0)
        return cls(*f, 0.0)

    def copy(self) -> "FieldState":
        return FieldState(self.P.copy(), self.Q.copy(), self.U.copy(),
                          self.V.copy(), self.t)

    def is_finite(self) -> bool:
        # A property of the host container itself (no stepping involved).
        return bool(np.isfinite(self.P).all() and np.isfinite(self.Q).all()
                    and np.isfinite(self.U).all() and np.isfinite(self.V).all())


def neighbor_indices(grid: GridSpec, i: int) -> list[int]:
    """The 2d periodic axis neighbors of linear index i, canonical order
    (-x, +x, -y, +y, -z, +z) truncated to d (reference grid.py:106-123)."""
    if not 0 <= i < grid.M:
        raise IndexError(f"linear index {i} out of range for M={grid.M}")
    N = grid.N
    coords = np.unravel_index(i, grid.shape)
    strides = [N**(grid.d - 1 - ax) for ax in range(grid.d)]
    out = []
    for ax in range(grid.d):
        for step in (-1, 1):
            c = (int(coords[ax]) + step) % N
            out.append(i + (c - int(coords[ax])) * strides[ax])
    return out


def energy_from_terms(terms, params: PhysParams, grid: GridSpec) -> tuple[float, float]:
    """Combine the 8 device term sums (include/kgs_b200.h, kgs_energy_terms)
    into (discrete_energy, mass), following raw_energy / mass
    (reference grid.py:166-187)."""
    t = [float(v) for v in terms]
    h2 = grid.h**2
    quad = (params.kappa1 * (t[0] / h2) + params.kappa1 * (t[1] / h2)
            + params.kappa2 * (t[2] / h2) + t[3] + params.mu**2 * t[4])
    raw = 0.5 * quad - params.gamma * t[5]
    hd = grid.h**grid.d
    return hd * raw, hd * (t[6] + t[7])


def _device_terms(state, grid: GridSpec):
    from .device import as_device_state
    dev, _owned = as_device_state(state, grid)
    return dev.energy_terms()


def discrete_energy(state, params: PhysParams, grid: GridSpec) -> float:
    """Scaled discrete energy h^d * E_raw, computed on the GPU by a
    deterministic tree reduction (reference grid.py:166-169)."""
    return energy_from_terms(_device_terms(state, grid), params, grid)[0]


def raw_energy(state, params: PhysParams, grid: GridSpec) -> float:
    """Unscaled energy (reference grid.py:172-181)."""
    return discrete_energy(state, params, grid) / grid.h**grid.d


def mass(state, grid: GridSpec) -> float:
    """Discrete mass ||Psi||_h^2 (reference grid.py:184-187)."""
    return energy_from_terms(_device_terms(state, grid), PhysParams(), grid)[1]
