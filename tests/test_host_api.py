"""CPU: the C-ABI library loads and exports every declared symbol, the
host-side API validates arguments like the reference, and device entry
points fail loudly (no CPU fallback) when no GPU is present."""
from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2502_09537_b200 as kgs
from paper_2502_09537_b200 import _lib
from paper_2502_09537_b200.device import combine_rank_terms, slab_range
from paper_2502_09537_b200.ordering import BLACK, RED

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "kgs_b200.h"


def _have_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def declared_functions() -> list[str]:
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(kgs_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert sorted(_lib.EXPORTED) == declared_functions()


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.kgs_abi_version() == 102
    assert lib.kgs_build_flags() == 0   # the default library: no experimental code, no asserts


def test_library_is_sm100a():
    out = Path(_lib.LIB_PATH)
    data = out.read_bytes()
    assert b"sm_100a" in data or b"sm_100" in data


def test_create_rejects_bad_geometry_before_touching_a_device():
    lib = _lib.load()
    ptr = ctypes.c_void_p()
    dev = (ctypes.c_int * 1)(0)
    rc = lib.kgs_create(2, 7, -1.0, 1.0, 1, dev, ctypes.byref(ptr))
    assert rc == _lib.KGS_EINVAL
    assert b"even N" in lib.kgs_last_error(None)
    rc = lib.kgs_create(4, 8, -1.0, 1.0, 1, dev, ctypes.byref(ptr))
    assert rc == _lib.KGS_EINVAL
    rc = lib.kgs_create(2, 8, -1.0, 1.0, 3, (ctypes.c_int * 3)(0, 0, 0), ctypes.byref(ptr))
    assert rc == _lib.KGS_EINVAL
    assert not ptr.value


def test_null_arguments_are_rejected_without_touching_a_device():
    """Every entry point taking a context returns KGS_EINVAL for NULL
    arguments (no crash, no CUDA call), like the reference's ValueErrors."""
    lib = _lib.load()
    E = _lib.KGS_EINVAL
    buf = (ctypes.c_double * 8)()
    i64 = ctypes.c_int64()
    assert lib.kgs_upload(None, buf, buf, buf, buf) == E
    assert lib.kgs_download(None, buf, buf, buf, buf) == E
    assert lib.kgs_upload_planes(None, 0, 0, 1, buf) == E
    assert lib.kgs_download_planes(None, 0, 0, 1, buf) == E
    assert lib.kgs_sweep(None, 0, 0, None) == E
    assert lib.kgs_step_dpavf2(None, None, 1, 0, 0, None, ctypes.byref(i64), 0) == E
    assert lib.kgs_integrate_host(None, buf, buf, buf, buf, None, 1, 0, 0, buf, buf,
                                  ctypes.byref(i64), 0) == E
    assert lib.kgs_energy_terms(None, buf) == E
    assert lib.kgs_energy_mass(None, 1.0, 1.0, 1.0, 1.0, buf, buf) == E
    assert lib.kgs_all_finite(None, ctypes.byref(ctypes.c_int())) == E
    assert lib.kgs_fill_preset(None, 0) == E
    assert lib.kgs_local_range(None, None, None, None) == E
    assert lib.kgs_set_param(None, b"pipeline", 1) == E
    assert lib.kgs_set_tuning(None, 4, 0, 0, 0, -1) == E
    assert lib.kgs_set_promotion(None, 0, 0) == E
    assert lib.kgs_pass_timing(None, 1) == E
    assert lib.kgs_pass_stats(None, None, None, None) == E
    assert lib.kgs_upload_planes(None, 0, 0, 1, buf) == E
    assert b"NULL" in lib.kgs_last_error(None)
    assert lib.kgs_debug_pass(None, 0, 1, buf) == E
    assert lib.kgs_destroy(None) == _lib.KGS_OK
    assert lib.kgs_launch_count(None) == 0
    # the plan query validates its output buffer too
    assert lib.kgs_pipeline_plan(64, 8, 2, 0, None, 10) == -1
    assert lib.kgs_pipeline_plan(64, 8, 2, 0, None, 0) > 0


@pytest.mark.skipif(_have_gpu(), reason="checks the no-GPU failure path")
def test_device_entry_points_fail_loudly_without_gpu():
    g = kgs.GridSpec(2, -1.0, 1.0, 8)
    s = kgs.FieldState.zeros(g)
    with pytest.raises(_lib.KgsError):
        kgs.discrete_energy(s, kgs.PhysParams(), g)
    with pytest.raises(_lib.KgsError):
        kgs.integrate(s, g, kgs.PhysParams(), kgs.checkerboard_schedule(g),
                      kgs.SerialExecutor(), 0.1, 0.3)


# ---- reference-compatible validation --------------------------------------
def test_gridspec_validation():
    with pytest.raises(ValueError, match="dimension"):
        kgs.GridSpec(4, 0.0, 1.0, 8)
    with pytest.raises(ValueError, match="b > a"):
        kgs.GridSpec(2, 1.0, 1.0, 8)
    with pytest.raises(ValueError, match="N >= 2"):
        kgs.GridSpec(2, 0.0, 1.0, 1)
    g = kgs.GridSpec(3, -10.0, 10.0, 16)
    assert g.h == 20.0 / 16 and g.M == 16**3 and g.shape == (16, 16, 16)


def test_physparams_validation():
    with pytest.raises(ValueError, match="gamma"):
        kgs.PhysParams(gamma=float("nan"))


def test_coefficients_errors_and_hand_inverse():
    g = kgs.GridSpec(1, 0.0, 4.0, 4)
    with pytest.raises(ValueError, match="tau"):
        kgs.precompute_coefficients(kgs.PhysParams(), 0.0, g)
    with pytest.raises(ValueError, match="tau"):
        kgs.precompute_coefficients(kgs.PhysParams(), float("inf"), g)
    c = kgs.precompute_coefficients(kgs.PhysParams(1.0, 0.0, 1.0, 1.0), 2.0, g)
    (i00, i01), (i10, i11) = c.uv_inv
    assert (i00, i01, i10, i11) == pytest.approx((0.5, 0.5, -0.5, 0.5))


def test_coefficients_inverse_identity_and_kappa1_zero():
    """uv_inv inverts [[1, -tau/2], [c_uv, 1]]; kappa1 = 0 zeroes alpha, beta
    (reference tests/test_integrator.py:34-44)."""
    g = kgs.GridSpec(3, -1.0, 1.0, 6)
    c = kgs.precompute_coefficients(kgs.PhysParams(0.3, 1.7, 0.9, 1.1), 0.05, g)
    m = np.array([[1.0, -c.tau / 2], [c.c_uv, 1.0]])
    assert np.allclose(np.array(c.uv_inv) @ m, np.eye(2), atol=1e-14)
    c0 = kgs.precompute_coefficients(kgs.PhysParams(kappa1=0.0), 0.1, kgs.GridSpec(2, 0.0, 1.0, 8))
    assert c0.alpha == 0.0 and c0.beta == 0.0


def test_checkerboard_schedule_conventions():
    g = kgs.GridSpec(2, 0.0, 1.0, 4)
    with pytest.raises(ValueError, match="even N"):
        kgs.checkerboard_schedule(kgs.GridSpec(2, 0.0, 1.0, 5))
    with pytest.raises(ValueError, match="workers"):
        kgs.checkerboard_schedule(g, workers=0)
    s = kgs.checkerboard_schedule(g, workers=2)
    assert s.strategy == "checkerboard" and s.validated
    assert s.colour_order == (RED, BLACK)
    parity = np.indices(g.shape).sum(axis=0).ravel() % 2
    order = s.serial_order()
    assert np.all(parity[order[: g.M // 2]] == 1)        # red first
    assert np.array_equal(np.sort(s.rank), np.arange(g.M))
    assert [len(p.lanes) for p in s.phases] == [2, 2]
    r = kgs.reverse_schedule(s)
    assert r.colour_order == (BLACK, RED)
    assert kgs.reverse_schedule(r) is s
    assert np.array_equal(r.serial_order(), order[::-1])
    assert kgs.validate_schedule(s, g) is None


def test_non_checkerboard_schedules_refused():
    class Fake:
        strategy = "lexicographic-forward"
    g = kgs.GridSpec(2, 0.0, 1.0, 4)
    assert "not supported" in kgs.validate_schedule(Fake(), g)
    with pytest.raises(ValueError, match="invalid schedule"):
        kgs.integrate(kgs.FieldState.zeros(g), g, kgs.PhysParams(), Fake(), None, 0.1, 0.2)


def test_executor_config_modes():
    assert isinstance(kgs.ExecutorConfig("serial").build(), kgs.SerialExecutor)
    assert kgs.ExecutorConfig("phased", 4).build().workers == 4
    ex = kgs.ExecutorConfig("cuda", 2).build()
    assert isinstance(ex, kgs.CudaExecutor) and ex.nslabs == 2
    # one slab per GPU when the library sees enough devices, else virtual slabs
    assert ex.devices == ((0, 1) if _lib.device_count() >= 2 else (0,))
    with pytest.raises(ValueError):
        kgs.ExecutorConfig("gpu", 1)        # reference tests/test_executor.py:23-27
    with pytest.raises(ValueError):
        kgs.ExecutorConfig("serial", 0)
    v = kgs.CudaExecutor((0,), slabs_per_device=4)
    assert v.nslabs == 4 and v.slab_devices() == (0, 0, 0, 0)


def test_integrate_argument_validation():
    g = kgs.GridSpec(2, 0.0, 1.0, 4)
    s = kgs.FieldState.zeros(g)
    sch = kgs.checkerboard_schedule(g)
    with pytest.raises(ValueError, match="tau > 0"):
        kgs.integrate(s, g, kgs.PhysParams(), sch, None, 0.0, 1.0)
    with pytest.raises(ValueError, match="tau > 0"):
        kgs.integrate(s, g, kgs.PhysParams(), sch, None, 0.1, -1.0)
    with pytest.raises(ValueError, match="record_stride"):
        kgs.integrate(s, g, kgs.PhysParams(), sch, None, 0.1, 1.0, record_stride=0)


def test_slab_partition_and_rank_sum():
    cover = []
    for r in range(4):
        x0, nx = slab_range(16, r, 4)
        cover.extend(range(x0, x0 + nx))
    assert cover == list(range(16))
    with pytest.raises(ValueError):
        slab_range(10, 0, 4)
    t = combine_rank_terms([np.full(8, 1.0), np.full(8, 2.0)])
    assert np.array_equal(t, np.full(8, 3.0))


def test_energy_from_terms_formula():
    from paper_2502_09537_b200.grid import energy_from_terms
    g = kgs.GridSpec(2, 0.0, 2.0, 4)        # h = 0.5
    p = kgs.PhysParams(2.0, 3.0, 0.5, 0.25)
    t = [1.0, 2.0, 3.0, 4.0, 5.0, 6.0, 7.0, 8.0]
    e, m = energy_from_terms(t, p, g)
    quad = 2.0 * 4.0 + 2.0 * 8.0 + 3.0 * 12.0 + 4.0 + 0.25 * 5.0
    assert e == pytest.approx(0.25 * (0.5 * quad - 0.25 * 6.0))
    assert m == pytest.approx(0.25 * 15.0)


class TestExecutorRun:
    """executor.run(schedule, lane_fn) keeps the reference's host semantics
    (dpavf/executor.py:39-71) for code that drives its own lane functions."""

    def _grid(self):
        return kgs.GridSpec(2, -1.0, 1.0, 8)

    def test_serial_runs_the_serial_order_once(self):
        g = self._grid()
        sch = kgs.checkerboard_schedule(g, 3)
        seen = []
        kgs.SerialExecutor().run(sch, lambda lane: seen.append(np.array(lane)))
        assert len(seen) == 1
        assert np.array_equal(seen[0], sch.serial_order())
        parity = np.indices(g.shape).sum(axis=0).ravel() % 2
        n_red = int(parity.sum())
        assert (parity[seen[0][:n_red]] == 1).all() and (parity[seen[0][n_red:]] == 0).all()

    def test_phased_barrier_and_coverage(self):
        import threading
        g = self._grid()
        sch = kgs.checkerboard_schedule(g, 4)
        parity = np.indices(g.shape).sum(axis=0).ravel() % 2
        log, lock = [], threading.Lock()

        def lane_fn(lane):
            with lock:
                log.append((int(parity[lane[0]]), np.array(lane)))

        with kgs.PhasedExecutor(4) as ex:
            ex.run(sch, lane_fn)
        colours = [c for c, _ in log]
        assert colours == sorted(colours, reverse=True)      # every red lane before any black
        allidx = np.sort(np.concatenate([l for _, l in log]))
        assert np.array_equal(allidx, np.arange(g.M))          # each point exactly once
        rev = kgs.reverse_schedule(sch)
        log.clear()
        with kgs.PhasedExecutor(2) as ex:
            ex.run(rev, lane_fn)
        assert [c for c, _ in log] == sorted(c for c, _ in log)  # black first when reversed

    def test_phased_reraises_lane_errors_and_checks_validation(self):
        g = self._grid()
        sch = kgs.checkerboard_schedule(g, 4)

        def boom(lane):
            raise RuntimeError("lane failed")

        with kgs.PhasedExecutor(4) as ex:
            with pytest.raises(RuntimeError, match="lane failed"):
                ex.run(sch, boom)
        unvalidated = kgs.checkerboard_schedule(g, 2)
        unvalidated.validated = False
        with pytest.raises(ValueError, match="validation"):
            kgs.PhasedExecutor(2).run(unvalidated, lambda lane: None)

    def test_device_only_executors_reject_host_lanes(self):
        g = self._grid()
        with pytest.raises(TypeError):
            kgs.CudaExecutor((0,)).run(kgs.checkerboard_schedule(g), lambda lane: None)


def test_cuda_executor_config_uses_virtual_slabs_beyond_the_gpu_count(monkeypatch):
    from paper_2502_09537_b200 import executor as exm
    monkeypatch.setattr(exm, "_device_count", lambda: 1)
    ex = kgs.ExecutorConfig("cuda", 4).build()
    assert ex.devices == (0,) and ex.slabs_per_device == 4 and ex.nslabs == 4
    monkeypatch.setattr(exm, "_device_count", lambda: 8)
    ex = kgs.ExecutorConfig("cuda", 4).build()
    assert ex.devices == (0, 1, 2, 3) and ex.slabs_per_device == 1
    monkeypatch.setattr(exm, "_device_count", lambda: 0)   # no driver: never phantom devices
    ex = kgs.ExecutorConfig("cuda", 2).build()
    assert ex.devices == (0,) and ex.slabs_per_device == 2


def test_device_count_comes_from_the_library():
    n = _lib.device_count()
    assert n >= 0
    from paper_2502_09537_b200 import executor as exm
    assert exm._device_count() == n


def test_one_call_path_only_takes_whole_grid_writable_float64():
    """integrate() hands host arrays to kgs_integrate_host as raw pointers;
    anything else must take the shape-checked path (sizes: the whole grid, or
    for a torchrun rank also its own slab)."""
    from paper_2502_09537_b200.integrator import _pipeline_ok
    g = kgs.GridSpec(2, 0.0, 1.0, 8)
    s = kgs.FieldState.zeros(g)
    assert _pipeline_ok(s, (g.M,))
    assert not _pipeline_ok(s, (kgs.GridSpec(2, 0.0, 1.0, 16).M,))   # too small for the grid
    assert _pipeline_ok(s, (4 * g.M, g.M))                           # a rank's own slab
    bad = kgs.FieldState.zeros(g)
    bad.U = np.zeros(2 * g.M)[::2]                                   # strided view
    assert not _pipeline_ok(bad, (g.M,))
    ro = kgs.FieldState.zeros(g)
    ro.V.flags.writeable = False
    assert not _pipeline_ok(ro, (g.M,))
    f32 = kgs.FieldState.zeros(g)
    f32.P = np.zeros(g.M, dtype=np.float32)
    assert not _pipeline_ok(f32, (g.M,))
    two_d = kgs.FieldState.zeros(g)
    two_d.Q = np.zeros((g.N, g.N))
    assert not _pipeline_ok(two_d, (g.M,))


@pytest.mark.parametrize("name,N,block", [("ellipsoids3d", 48, 1000), ("ellipsoids3d", 64, 1 << 22),
                                          ("ellipsoids3d", 30, 7 * 900),
                                          ("fourpeak2d", 256, 3000), ("gaussian2d", 128, 128 * 5)])
def test_build_preset_blocks_bitwise(name, N, block):
    """The block-parallel host build (bench.py, the 1024^3 parity test) is
    bitwise the whole-grid preset, i.e. the reference's scenarios.py:40-89."""
    from paper_2502_09537_b200.scenarios import build_preset
    sc = kgs.get_scenario(name)
    g = sc.default_grid(N)
    whole = sc.state(g)
    blocks = build_preset(name, g, block_points=block, workers=4)
    for f in "PQUV":
        assert np.array_equal(getattr(whole, f), getattr(blocks, f)), f


def test_build_preset_slab_is_the_whole_grid_slice():
    from paper_2502_09537_b200.scenarios import build_preset
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(32)
    whole = sc.state(g)
    for lo, hi in ((0, 8), (8, 16), (24, 32), (5, 13)):
        slab = build_preset("ellipsoids3d", g, planes=(lo, hi), block_points=3000)
        for f in "PQUV":
            assert np.array_equal(getattr(slab, f), getattr(whole, f)[lo * 1024:hi * 1024])
    with pytest.raises(ValueError):
        build_preset("ellipsoids3d", g, planes=(0, 33))


def test_colour_order_of_foreign_schedules():
    """The reference's UpdateSchedule objects carry their colour order in
    their phases (ordering.py:130-146); reverse_schedule'd ones sweep black
    first and must run black first here too."""
    from types import SimpleNamespace as NS
    from paper_2502_09537_b200.ordering import colour_order, is_reversed
    g = kgs.GridSpec(3, -1.0, 1.0, 4)
    par = np.indices(g.shape).sum(axis=0).ravel() % 2
    red, black = np.nonzero(par == 1)[0], np.nonzero(par == 0)[0]
    fwd = NS(strategy="checkerboard", phases=[NS(lanes=[red[:5], red[5:]]), NS(lanes=[black])])
    rev = NS(strategy="checkerboard", phases=[NS(lanes=[black[::-1]]),
                                              NS(lanes=[red[5:][::-1], red[:5][::-1]])])
    assert colour_order(fwd, g) == (RED, BLACK) and not is_reversed(fwd, g)
    assert colour_order(rev, g) == (BLACK, RED) and is_reversed(rev, g)
    rank = np.empty(g.M, dtype=np.int64)
    rank[np.concatenate([black, red])] = np.arange(g.M)
    assert colour_order(NS(strategy="checkerboard", rank=rank), g) == (BLACK, RED)
    ours = kgs.checkerboard_schedule(g)
    assert colour_order(ours, g) == (RED, BLACK)
    assert colour_order(kgs.reverse_schedule(ours), g) == (BLACK, RED)
