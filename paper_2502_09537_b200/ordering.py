"""Update schedules -- the checkerboard descriptor.

The reference materialises every schedule as index arrays: ``rank`` (M
int64), red/black index lanes and ``np.indices`` (d*M int64) in
``checkerboard_schedule`` (dpavf/ordering.py:114-136), i.e. ~50 GB at 1024^3.
On the device only the colour convention matters, so here a schedule is a
small descriptor:

* red = index-sum parity 1, swept first by the base sweep; black = parity 0
  (ordering.py:125-128);
* ``reverse_schedule`` flips the phase order (adjoint: black then red,
  ordering.py:139-149);
* odd N is rejected with the reference's message (ordering.py:120-122).

``rank``, ``phases`` and ``serial_order()`` are still available, computed
lazily on the host for small grids, so code that inspects a schedule keeps
working.  Only the checkerboard strategy runs on the device; every other
strategy of the reference (lexicographic, seeded-random, block-split) is
inherently serial or CPU-specific and is out of scope.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .grid import GridSpec

STRATEGIES = ("checkerboard",)
RED, BLACK = 1, 0


@dataclass
class Phase:
    parallel: bool
    lanes: list  # list of int64 index arrays, each in execution order


@dataclass
class UpdateSchedule:
    """Checkerboard schedule descriptor (cf. reference ordering.py:29-47)."""

    strategy: str
    grid: GridSpec
    workers: int = 1
    reversed: bool = False
    seed: int | None = None
    validated: bool = True
    _rev: "UpdateSchedule | None" = field(default=None, repr=False)

    @property
    def M(self) -> int:
        return self.grid.M

    @property
    def colour_order(self) -> tuple[int, int]:
        """Colours in sweep order: (red, black) or, reversed, (black, red)."""
        return (BLACK, RED) if self.reversed else (RED, BLACK)

    # -- lazily materialised host views (small grids only) -----------------
    def _colour_indices(self) -> tuple[np.ndarray, np.ndarray]:
        parity = np.indices(self.grid.shape).sum(axis=0).ravel() % 2
        red = np.nonzero(parity == 1)[0].astype(np.int64)
        black = np.nonzero(parity == 0)[0].astype(np.int64)
        return red, black

    @property
    def phases(self) -> list:
        red, black = self._colour_indices()
        stripe = lambda idx: [l for l in np.array_split(idx, self.workers) if l.size]
        ph = [Phase(True, stripe(red)), Phase(True, stripe(black))]
        if self.reversed:
            ph = [Phase(p.parallel, [l[::-1].copy() for l in reversed(p.lanes)])
                  for p in reversed(ph)]
        return ph

    def serial_order(self) -> np.ndarray:
        red, black = self._colour_indices()
        order = np.concatenate([red, black])
        return order[::-1].copy() if self.reversed else order

    @property
    def rank(self) -> np.ndarray:
        order = self.serial_order()
        rank = np.empty(order.shape[0], dtype=np.int64)
        rank[order] = np.arange(order.shape[0], dtype=np.int64)
        return rank


def checkerboard_schedule(grid: GridSpec, workers: int = 1) -> UpdateSchedule:
    """Two parallel phases: odd-parity ("red") points, then the rest."""
    if grid.N % 2 != 0:
        raise ValueError(
            f"checkerboard needs even N for a consistent periodic 2-coloring, got N={grid.N}")
    if workers < 1:
        raise ValueError("workers must be >= 1")
    return UpdateSchedule("checkerboard", grid, workers=workers)


def reverse_schedule(s: UpdateSchedule) -> UpdateSchedule:
    """Mirror the sweep: black phase first, then red (ordering.py:139-149)."""
    if s._rev is not None:
        return s._rev
    rev = UpdateSchedule(s.strategy, s.grid, workers=s.workers,
                         reversed=not s.reversed, seed=s.seed, validated=s.validated)
    rev._rev = s
    s._rev = rev
    return rev


def validate_schedule(s, grid: GridSpec) -> str | None:
    """None if ``s`` is a checkerboard schedule for ``grid`` (even N), else a
    report.  Accepts the reference's UpdateSchedule objects too (their
    strategy/rank are checked; the phase plan is the reference's own)."""
    strategy = getattr(s, "strategy", None)
    if strategy != "checkerboard":
        return (f"strategy {strategy!r} is not supported on the device; only the "
                "checkerboard schedule runs on the B200")
    if grid.N % 2 != 0:
        return f"checkerboard needs even N, got N={grid.N}"
    if isinstance(s, UpdateSchedule):
        if s.grid != grid:
            return f"schedule is for {s.grid}, grid is {grid}"
        return None
    rank = getattr(s, "rank", None)
    if rank is not None and rank.shape[0] != grid.M:
        return f"rank has {rank.shape[0]} entries, grid has {grid.M} points"
    return None


def colour_order(s, grid: GridSpec) -> tuple[int, int]:
    """The colours of a checkerboard schedule in sweep order.  Ours carry it
    (``reversed``); for the reference's UpdateSchedule objects it is read off
    the schedule itself -- the colour of the first point of its first phase
    (ordering.py:130-146: red first, or black first after
    ``reverse_schedule``), else of the point with rank 0."""
    if isinstance(s, UpdateSchedule):
        return s.colour_order
    first = None
    phases = getattr(s, "phases", None)
    if phases:
        for lane in phases[0].lanes:
            if len(lane):
                first = int(lane[0])
                break
    if first is None:
        rank = getattr(s, "rank", None)
        if rank is not None and len(rank):
            first = int(np.argmin(rank))
    if first is None:
        return (RED, BLACK)
    parity = int(sum(np.unravel_index(first, grid.shape))) % 2
    return (RED, BLACK) if parity == RED else (BLACK, RED)


def is_reversed(s, grid: GridSpec) -> bool:
    """True for a schedule that sweeps black before red (reverse_schedule)."""
    return colour_order(s, grid)[0] == BLACK


def require_checkerboard(s, grid: GridSpec) -> None:
    report = validate_schedule(s, grid)
    if report is not None:
        raise ValueError(f"invalid schedule: {report}")
