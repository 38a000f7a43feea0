"""Device contexts and the device-resident field state.

A :class:`DeviceContext` owns one ``kgs_ctx`` (include/kgs_b200.h): the
colour-split P, Q, U, V planes of one or more slabs in HBM.  A
:class:`DeviceFieldState` is the device-resident counterpart of the
reference ``FieldState`` (dpavf/grid.py:82-103): it keeps the state on the
GPU across calls, which is how long runs and benchmarks avoid host copies.

Host ``FieldState`` objects passed to the drop-in API are uploaded to a
cached context and copied back after the call (copy semantics, the caller's
arrays are updated in place like the reference's in-place sweeps).
"""
from __future__ import annotations

import ctypes
import os
from collections import OrderedDict

import numpy as np

from . import _lib
from .executor import DistributedExecutor, resolve
from .grid import FieldState, GridSpec, energy_from_terms, PhysParams

PRESETS = {"ellipsoids3d": 0, "fourpeak2d": 1, "gaussian2d": 2, "soliton1d": 3}


def slab_range(planes: int, rank: int, world: int) -> tuple[int, int]:
    """(first plane, plane count) of slab ``rank`` of ``world`` along axis 0.
    Equal slabs; the C library rejects N % world != 0 (KGS_EINVAL)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    if planes % world:
        raise ValueError(f"N={planes} not divisible by {world} ranks")
    per = planes // world
    return rank * per, per


def combine_rank_terms(per_rank_terms) -> np.ndarray:
    """Deterministic cross-rank sum of the 8 energy terms: rank order."""
    out = np.zeros(_lib.NTERMS)
    for t in per_rank_terms:
        out = out + np.asarray(t, dtype=np.float64)
    return out


def make_nccl_id(rank: int, broadcast) -> bytes:
    """Rank 0 creates the ncclUniqueId; ``broadcast(obj_or_None) -> obj``
    distributes it (torch.distributed.broadcast_object_list in practice)."""
    if rank == 0:
        buf = ctypes.create_string_buffer(128)
        _lib.check(_lib.load().kgs_nccl_unique_id(buf))
        nid = buf.raw
    else:
        nid = None
    return broadcast(nid)


def _torch_broadcast(obj):
    import torch.distributed as dist
    lst = [obj]
    dist.broadcast_object_list(lst, src=0)
    return lst[0]


def _torch_allgather(obj):
    import torch.distributed as dist
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


class DeviceContext:
    """One kgs_ctx (device buffers for a grid under an executor plan)."""

    def __init__(self, grid: GridSpec, executor=None):
        lib = _lib.load()
        self.grid = grid
        self.plan = resolve(executor)
        self.dist = isinstance(self.plan, DistributedExecutor)
        ptr = ctypes.c_void_p()
        if self.dist:
            p = self.plan
            if p.world_size > 1:
                nid = make_nccl_id(p.rank, _torch_broadcast)
            elif os.environ.get("KGS_SELF_EXCHANGE") == "1":
                # test hook: one rank exchanging its faces with itself over
                # NCCL -- the multi-rank code path on one GPU (kgs_b200.h)
                nid = make_nccl_id(0, lambda obj: obj)
            else:
                nid = None
            rc = lib.kgs_create_dist(grid.d, grid.N, grid.a, grid.b, p.rank,
                                     p.world_size, p.device, nid, ctypes.byref(ptr))
        else:
            devs = self.plan.slab_devices()
            arr = (ctypes.c_int * len(devs))(*devs)
            rc = lib.kgs_create(grid.d, grid.N, grid.a, grid.b, len(devs), arr,
                                ctypes.byref(ptr))
        _lib.check(rc)
        self.ptr = ptr
        x0, nx, pts = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _lib.check(lib.kgs_local_range(ptr, ctypes.byref(x0), ctypes.byref(nx),
                                       ctypes.byref(pts)), ptr)
        self.x0, self.nx, self.points = x0.value, nx.value, pts.value
        self.plane = grid.N**(grid.d - 1) if grid.d > 1 else grid.N
        self.offset = self.x0 * self.plane if grid.d > 1 else 0

    # -- lifetime ----------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "ptr", None) is not None and self.ptr.value:
            _lib.load().kgs_destroy(self.ptr)
            self.ptr = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- helpers -----------------------------------------------------------
    def check(self, rc: int) -> None:
        _lib.check(rc, self.ptr)

    def local(self, a: np.ndarray) -> np.ndarray:
        """This context's planes of a host field: a whole-grid array is
        sliced; a distributed rank may also pass just its own slab."""
        if a.shape == (self.grid.M,):
            return a[self.offset:self.offset + self.points]
        if self.dist and a.shape == (self.points,):
            return a
        raise ValueError(f"field has shape {a.shape}, grid needs ({self.grid.M},)")

    def upload_planes(self, field: int, x_begin: int, data: np.ndarray) -> None:
        """Planes [x_begin, x_begin + n) of one field (0 P .. 3 V), natural layout."""
        a = np.ascontiguousarray(data, dtype=np.float64)
        n = a.size // self.plane
        if n * self.plane != a.size:
            raise ValueError("data is not a whole number of planes")
        self.check(_lib.load().kgs_upload_planes(self.ptr, field, x_begin, n, _lib.dptr(a)))

    def download_planes(self, field: int, x_begin: int, out: np.ndarray) -> None:
        n = out.size // self.plane
        if n * self.plane != out.size or not out.flags["C_CONTIGUOUS"]:
            raise ValueError("out must be a contiguous whole number of planes")
        self.check(_lib.load().kgs_download_planes(self.ptr, field, x_begin, n,
                                                   _lib.dptr(out)))

    def upload(self, s: FieldState) -> None:
        f = [np.ascontiguousarray(self.local(np.asarray(a, dtype=np.float64)))
             for a in (s.P, s.Q, s.U, s.V)]
        self.check(_lib.load().kgs_upload(self.ptr, *[_lib.dptr(a) for a in f]))

    def download(self, s: FieldState) -> None:
        lib = _lib.load()
        views = [self.local(a) for a in (s.P, s.Q, s.U, s.V)]
        if all(v.flags["C_CONTIGUOUS"] and v.dtype == np.float64 and v.flags["WRITEABLE"]
               for v in views):
            self.check(lib.kgs_download(self.ptr, *[_lib.dptr(v) for v in views]))
        else:
            tmp = [np.empty(self.points) for _ in range(4)]
            self.check(lib.kgs_download(self.ptr, *[_lib.dptr(v) for v in tmp]))
            for v, t in zip(views, tmp):
                v[...] = t

    def energy_terms(self) -> np.ndarray:
        out = np.zeros(_lib.NTERMS)
        self.check(_lib.load().kgs_energy_terms(self.ptr, _lib.dptr(out)))
        if self.dist and self.plan.world_size > 1:
            out = combine_rank_terms(_torch_allgather(out))
        return out

    def all_finite(self) -> bool:
        ok = ctypes.c_int()
        self.check(_lib.load().kgs_all_finite(self.ptr, ctypes.byref(ok)))
        flag = bool(ok.value)
        if self.dist and self.plan.world_size > 1:
            flag = all(_torch_allgather(flag))
        return flag

    def sweep(self, colour: int, kind: int, kernel_args) -> None:
        c = _lib.coeffs_struct(kernel_args)
        self.check(_lib.load().kgs_sweep(self.ptr, colour, kind, ctypes.byref(c)))

    def integrate_host(self, state, kernel_args, nsteps: int, record_stride: int = 0):
        """One call for a whole host-state integration (kgs_integrate_host):
        upload, nsteps DP-AVF2 steps and download overlapped in a pipeline;
        the host arrays are updated in place.  Returns (terms0, terms[nrec, 8],
        bad_step); on a non-finite step the state is the one after `bad_step`."""
        lib = _lib.load()
        c = _lib.coeffs_struct(kernel_args)
        nrec = nsteps // record_stride if record_stride > 0 else 0
        terms0 = np.zeros(_lib.NTERMS)
        terms = np.zeros((max(nrec, 1), _lib.NTERMS))
        bad = ctypes.c_int64(0)
        # this context's planes (a rank: its slab of a whole-grid array, or its own slab)
        views = [self.local(getattr(state, f)) for f in "PQUV"]
        rc = lib.kgs_integrate_host(self.ptr, *(_lib.dptr(v) for v in views),
                                    ctypes.byref(c), nsteps, 0, record_stride,
                                    _lib.dptr(terms0), _lib.dptr(terms), ctypes.byref(bad), 0)
        if rc not in (_lib.KGS_OK, _lib.KGS_ENONFINITE):
            self.check(rc)
        terms = terms[:nrec]
        if self.dist and self.plan.world_size > 1:   # per-rank sums, added in rank order
            gathered = _torch_allgather((terms0, terms))
            terms0 = combine_rank_terms([t0 for t0, _ in gathered])
            terms = sum((np.asarray(t) for _, t in gathered[1:]), np.asarray(gathered[0][1]))
        # the library makes the ranks agree on the first bad step
        return terms0, terms, (bad.value if rc == _lib.KGS_ENONFINITE else 0)

    def step_dpavf2(self, kernel_args, nsteps: int, step_offset: int = 0,
                    record_stride: int = 0, defer_tail: bool = False, backup: bool = False):
        """Run nsteps fused DP-AVF2 steps; returns (terms[nrec, 8], bad_step).
        defer_tail: leave the last red adjoint pending (see kgs_b200.h);
        backup: keep a device copy of the starting state for
        restore_backup()."""
        lib = _lib.load()
        c = _lib.coeffs_struct(kernel_args)
        if record_stride > 0:
            nrec = (step_offset + nsteps) // record_stride - step_offset // record_stride
        else:
            nrec = 0
        terms = np.zeros((max(nrec, 1), _lib.NTERMS))
        bad = ctypes.c_int64(0)
        rc = lib.kgs_step_dpavf2(self.ptr, ctypes.byref(c), nsteps, step_offset,
                                 record_stride, _lib.dptr(terms), ctypes.byref(bad),
                                 (_lib.KGS_STEP_DEFER_TAIL if defer_tail else 0)
                                 | (_lib.KGS_STEP_BACKUP if backup else 0))
        if rc not in (_lib.KGS_OK, _lib.KGS_ENONFINITE):
            self.check(rc)
        bad_step = bad.value if rc == _lib.KGS_ENONFINITE else 0
        terms = terms[:nrec]
        if self.dist and self.plan.world_size > 1:
            gathered = _torch_allgather((terms, bad_step))
            terms = sum((np.asarray(t) for t, _ in gathered[1:]), np.asarray(gathered[0][0]))
            bads = [b for _, b in gathered if b]
            bad_step = min(bads) if bads else 0
        return terms, bad_step

    def restore_backup(self) -> bool:
        """Back to the state saved by the last step_dpavf2(..., backup=True);
        False if there is none (no memory for it, or the state changed)."""
        return _lib.load().kgs_restore_backup(self.ptr) == _lib.KGS_OK

    def fill_preset(self, name: str) -> None:
        if name not in PRESETS:
            raise ValueError(f"unknown device preset {name!r}; known: {', '.join(PRESETS)}")
        self.check(_lib.load().kgs_fill_preset(self.ptr, PRESETS[name]))

    def launch_count(self) -> int:
        return int(_lib.load().kgs_launch_count(self.ptr))

    def last_step_ms(self) -> float:
        return float(_lib.load().kgs_last_step_ms(self.ptr))

    def set_tuning(self, rows_per_tile: int = 4, band_rows: int = 64,
                   blocks_per_sm: int = 0, march_planes: int = 0,
                   march_variant: int = -1) -> None:
        self.check(_lib.load().kgs_set_tuning(self.ptr, rows_per_tile, band_rows,
                                              blocks_per_sm, march_planes, march_variant))

    def set_param(self, name: str, value: int) -> None:
        self.check(_lib.load().kgs_set_param(self.ptr, name.encode(), int(value)))

    def pass_timing(self, enable: bool) -> None:
        self.check(_lib.load().kgs_pass_timing(self.ptr, int(enable)))

    def pass_stats(self) -> tuple[int, float, int]:
        """(timed fused-pass launches, total ms, points updated per launch)."""
        n, ms, pts = ctypes.c_int64(), ctypes.c_double(), ctypes.c_int64()
        self.check(_lib.load().kgs_pass_stats(self.ptr, ctypes.byref(n), ctypes.byref(ms),
                                              ctypes.byref(pts)))
        return n.value, ms.value, pts.value


_CTX_CACHE: "OrderedDict[tuple, DeviceContext]" = OrderedDict()
_CTX_CACHE_MAX = 2


def get_context(grid: GridSpec, executor=None) -> DeviceContext:
    """Cached DeviceContext for (grid, executor plan)."""
    plan = resolve(executor)
    key = (grid.d, grid.a, grid.b, grid.N) + plan.key()
    ctx = _CTX_CACHE.get(key)
    if ctx is not None and ctx.ptr.value:
        _CTX_CACHE.move_to_end(key)
        return ctx
    if ctx is not None:   # closed by its user (DeviceFieldState.close): replace it
        del _CTX_CACHE[key]
    while len(_CTX_CACHE) >= _CTX_CACHE_MAX:
        _, old = _CTX_CACHE.popitem(last=False)
        old.close()
    ctx = DeviceContext(grid, plan)
    _CTX_CACHE[key] = ctx
    return ctx


def clear_contexts() -> None:
    while _CTX_CACHE:
        _, c = _CTX_CACHE.popitem()
        c.close()


class DeviceFieldState:
    """Device-resident P, Q, U, V (+ host-side time t).

    Accepted everywhere a FieldState is (step_*, integrate, discrete_energy,
    mass); operations run in place on the GPU without host copies."""

    def __init__(self, grid: GridSpec, executor=None, *, context: DeviceContext | None = None,
                 t: float = 0.0):
        self.grid = grid
        self.ctx = context if context is not None else DeviceContext(grid, executor)
        self.t = float(t)

    @classmethod
    def from_host(cls, state: FieldState, grid: GridSpec, executor=None) -> "DeviceFieldState":
        d = cls(grid, executor, t=state.t)
        d.ctx.upload(state)
        return d

    @classmethod
    def from_preset(cls, name: str, grid: GridSpec, executor=None) -> "DeviceFieldState":
        d = cls(grid, executor)
        d.ctx.fill_preset(name)
        return d

    def upload(self, state: FieldState) -> None:
        self.ctx.upload(state)
        self.t = state.t

    def download(self, into: FieldState | None = None) -> FieldState:
        s = into if into is not None else FieldState.zeros(self.grid)
        self.ctx.download(s)
        s.t = self.t
        return s

    def to_host(self) -> FieldState:
        return self.download()

    def energy_terms(self) -> np.ndarray:
        return self.ctx.energy_terms()

    def energy_mass(self, params: PhysParams) -> tuple[float, float]:
        return energy_from_terms(self.energy_terms(), params, self.grid)

    def is_finite(self) -> bool:
        return self.ctx.all_finite()

    def close(self) -> None:
        self.ctx.close()


def as_device_state(state, grid: GridSpec, executor=None):
    """(DeviceFieldState, is_temporary).  Host states are uploaded into a
    cached context; the caller downloads back when it mutated the state."""
    if isinstance(state, DeviceFieldState):
        if state.grid != grid:
            raise ValueError(f"state is on grid {state.grid}, got {grid}")
        return state, False
    ctx = get_context(grid, executor)
    ctx.upload(state)
    return DeviceFieldState(grid, context=ctx, t=state.t), True


class _PinnedBlock:
    """Owner of one cudaHostAlloc block; freed when the last array view dies."""

    def __init__(self, nbytes: int):
        p = ctypes.c_void_p()
        _lib.check(_lib.load().kgs_host_alloc(nbytes, ctypes.byref(p)))
        self.ptr = p

    def __del__(self):
        try:
            if self.ptr.value:
                _lib.load().kgs_host_free(self.ptr)
        except Exception:
            pass


def pinned_empty(n: int) -> np.ndarray:
    """float64[n] in page-locked host memory (cudaHostAlloc via the C ABI)."""
    block = _PinnedBlock(8 * n)
    buf = (ctypes.c_double * n).from_address(block.ptr.value)
    buf._owner = block          # keep the block alive as long as the buffer
    return np.ctypeslib.as_array(buf)
