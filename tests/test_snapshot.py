"""KGS1 snapshots: the reference's format (dpavf/snapshot.py; tests mirror
reference tests/test_cli.py:87-118), and the device streaming writer/reader
(bytes identical to the host writer, incl. multi-slab contexts)."""
from __future__ import annotations

import os

import numpy as np
import pytest

import paper_2502_09537_b200 as kgs
from conftest import assert_bitwise


def test_roundtrip_bitwise(tmp_path):
    g = kgs.GridSpec(2, -10.0, 10.0, 8)
    s = kgs.seeded_random_state(g, 4, 0.5)
    s.t = 1.25
    path = tmp_path / "snap.bin"
    kgs.write_snapshot(s, g, path)
    s2, g2 = kgs.read_snapshot(path)
    assert g2 == g and s2.t == 1.25
    assert_bitwise(s, s2)


def test_size_formula(tmp_path):
    g = kgs.GridSpec(2, -10.0, 10.0, 128)
    path = tmp_path / "snap.bin"
    kgs.write_snapshot(kgs.FieldState.zeros(g), g, path)
    assert os.path.getsize(path) == 524_328
    assert kgs.snapshot_size(g) == 4 + 4 * 3 + 8 * 3 + 4 * 128**2 * 8


def test_header_layout(tmp_path):
    g = kgs.GridSpec(3, -1.5, 2.5, 4)
    s = kgs.seeded_random_state(g, 1, 0.5)
    s.t = 0.75
    path = tmp_path / "h.bin"
    kgs.write_snapshot(s, g, path)
    raw = path.read_bytes()
    import struct
    assert struct.unpack_from("<4sIIIddd", raw) == (b"KGS1", 1, 3, 4, -1.5, 2.5, 0.75)
    assert np.array_equal(np.frombuffer(raw, "<f8", g.M, 40), s.P)


def test_bad_magic(tmp_path):
    path = tmp_path / "bad.bin"
    path.write_bytes(b"XXXX" + b"\x00" * 100)
    with pytest.raises(ValueError, match="magic"):
        kgs.read_snapshot(path)


def test_truncated(tmp_path):
    g = kgs.GridSpec(1, 0.0, 1.0, 8)
    path = tmp_path / "t.bin"
    kgs.write_snapshot(kgs.FieldState.zeros(g), g, path)
    path.write_bytes(path.read_bytes()[:-8])
    with pytest.raises(ValueError, match="bytes"):
        kgs.read_snapshot(path)


@pytest.mark.gpu
@pytest.mark.parametrize("d,N,slabs", [(3, 16, 1), (3, 16, 4), (2, 32, 2), (1, 64, 1)])
def test_device_snapshot_bytes_equal_host(tmp_path, d, N, slabs):
    g = kgs.GridSpec(d, -2.0, 2.0, N)
    s = kgs.seeded_random_state(g, 17, 0.5)
    s.t = 0.5
    ex = kgs.CudaExecutor((0,), slabs_per_device=slabs)
    dev = kgs.DeviceFieldState.from_host(s, g, ex)
    kgs.write_snapshot(dev, g, tmp_path / "dev.bin")
    kgs.write_snapshot(s, g, tmp_path / "host.bin")
    assert (tmp_path / "dev.bin").read_bytes() == (tmp_path / "host.bin").read_bytes()
    back = kgs.read_snapshot_device(tmp_path / "dev.bin", ex)
    assert back.t == 0.5
    assert_bitwise(back.to_host(), s)
    dev.close()
    back.close()


@pytest.mark.gpu
def test_integrate_snapshot_writer_matches_reference_states(golden, tmp_path):
    """snapshot_writer sees the state after step n (integrator.py:180-181)."""
    import oracle
    c = golden.case("d3_rand_N8")
    s = c.state(0)
    ref = c.state(0)
    written = []

    def writer(state, n):
        p = tmp_path / f"snapshot_{n:06d}.bin"
        kgs.write_snapshot(state, c.grid, p)
        written.append((n, p))

    kgs.integrate(s, c.grid, c.params, kgs.checkerboard_schedule(c.grid), None,
                  c.meta["tau"], c.meta["T"], record_stride=5, snapshot_stride=7,
                  snapshot_writer=writer)
    assert [n for n, _ in written] == [7, 14]
    done = 0
    for n, p in written:
        oracle.numpy_step_dpavf2(ref, c.kernel_args, c.grid, n - done)
        done = n
        snap, _ = kgs.read_snapshot(p)
        assert_bitwise(snap, ref)
    assert_bitwise(s, c.state(1))
