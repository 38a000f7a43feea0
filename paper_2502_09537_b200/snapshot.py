"""KGS1 snapshots (the reference's bit-exact binary format,
dpavf/snapshot.py:1-64) written straight from device memory.

Layout (little-endian): b"KGS1", u32 version 1, u32 d, u32 N, f64 a, b, t,
then P, Q, U, V as N^d float64 each in the reference linearisation.

For a :class:`DeviceFieldState` the fields are streamed plane-chunk by
plane-chunk (kgs_download_planes) so a 2048^3 state (275 GB) never exists on
the host; in a distributed run rank 0 writes the header and sizes the file,
then every rank writes its own slab at its offset (pwrite), no gathering.
Host FieldStates are written exactly as the reference does.
"""
from __future__ import annotations

import os
import struct

import numpy as np

from .grid import FieldState, GridSpec

MAGIC = b"KGS1"
VERSION = 1
_HEADER = struct.Struct("<4sIIIddd")
CHUNK_BYTES = 256 << 20


def snapshot_size(grid: GridSpec) -> int:
    return _HEADER.size + 4 * 8 * grid.M


def _header(grid: GridSpec, t: float) -> bytes:
    return _HEADER.pack(MAGIC, VERSION, grid.d, grid.N, grid.a, grid.b, t)


def write_snapshot(state, grid: GridSpec, path) -> None:
    """Reference write_snapshot(state, grid, path) (snapshot.py:30-38); state
    may be a host FieldState or a DeviceFieldState."""
    from .device import DeviceFieldState
    try:
        if not isinstance(state, DeviceFieldState):
            with open(path, "wb") as fh:
                fh.write(_header(grid, state.t))
                for field in (state.P, state.Q, state.U, state.V):
                    fh.write(np.ascontiguousarray(field, dtype="<f8").tobytes())
            return
        _write_device(state, grid, path)
    except OSError as exc:
        raise OSError(f"snapshot write failed for {path}: {exc}") from exc


def _write_device(state, grid: GridSpec, path) -> None:
    ctx = state.ctx
    dist = ctx.dist and ctx.plan.world_size > 1
    if dist:
        import torch.distributed as tdist
    if not dist or ctx.plan.rank == 0:
        with open(path, "wb") as fh:
            fh.write(_header(grid, state.t))
            fh.truncate(snapshot_size(grid))
    if dist:
        tdist.barrier()
    plane = ctx.plane
    nx = ctx.nx if grid.d > 1 else 1
    x0 = ctx.x0 if grid.d > 1 else 0
    per = max(1, CHUNK_BYTES // (8 * plane))
    buf = np.empty(min(per, nx) * plane)
    fd = os.open(path, os.O_WRONLY)
    try:
        for f in range(4):
            for xs in range(x0, x0 + nx, per):
                n = min(per, x0 + nx - xs)
                view = buf[:n * plane]
                ctx.download_planes(f, xs, view)
                off = _HEADER.size + 8 * (f * grid.M + xs * plane)
                data = view.astype("<f8", copy=False).tobytes()
                written = 0
                while written < len(data):
                    written += os.pwrite(fd, data[written:], off + written)
    finally:
        os.close(fd)
    if dist:
        tdist.barrier()


def read_snapshot(path) -> tuple[FieldState, GridSpec]:
    """Reference read_snapshot (snapshot.py:41-64): host FieldState + grid."""
    try:
        with open(path, "rb") as fh:
            raw = fh.read()
    except OSError as exc:
        raise OSError(f"snapshot read failed for {path}: {exc}") from exc
    grid, t = _parse_header(raw, path, len(raw))
    fields = []
    off = _HEADER.size
    for _ in range(4):
        fields.append(np.frombuffer(raw, dtype="<f8", count=grid.M, offset=off).astype(np.float64))
        off += 8 * grid.M
    return FieldState(*fields, t=t), grid


def _parse_header(raw: bytes, path, size: int):
    if len(raw) < _HEADER.size:
        raise ValueError(f"snapshot {path} truncated: {len(raw)} bytes")
    magic, version, d, N, a, b, t = _HEADER.unpack_from(raw)
    if magic != MAGIC:
        raise ValueError(f"snapshot {path} has bad magic {magic!r}")
    if version != VERSION:
        raise ValueError(f"snapshot {path} has unsupported version {version}")
    grid = GridSpec(d, a, b, N)
    if size != snapshot_size(grid):
        raise ValueError(f"snapshot {path} has {size} bytes, expected {snapshot_size(grid)}")
    return grid, t


def read_snapshot_device(path, executor=None):
    """Stream a KGS1 file into a new DeviceFieldState (this rank's slab only
    in a distributed run) without materialising it on the host."""
    from .device import DeviceFieldState
    try:
        size = os.path.getsize(path)
        with open(path, "rb") as fh:
            grid, t = _parse_header(fh.read(_HEADER.size), path, size)
            dev = DeviceFieldState(grid, executor, t=t)
            ctx = dev.ctx
            plane, nx = ctx.plane, (ctx.nx if grid.d > 1 else 1)
            x0 = ctx.x0 if grid.d > 1 else 0
            per = max(1, CHUNK_BYTES // (8 * plane))
            for f in range(4):
                for xs in range(x0, x0 + nx, per):
                    n = min(per, x0 + nx - xs)
                    fh.seek(_HEADER.size + 8 * (f * grid.M + xs * plane))
                    data = np.frombuffer(fh.read(8 * n * plane), dtype="<f8")
                    ctx.upload_planes(f, xs, data.astype(np.float64))
    except OSError as exc:
        raise OSError(f"snapshot read failed for {path}: {exc}") from exc
    return dev
