"""ctypes binding of the C ABI in include/kgs_b200.h (libkgs_b200.so).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_2502_09537_b200.build``).  There is no CPU fallback: if the
library is missing or no B200 is visible, every device entry point raises.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

LIB_NAME = "libkgs_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

KGS_OK = 0
KGS_EINVAL = -1
KGS_ECUDA = -2
KGS_ENCCL = -3
KGS_ENONFINITE = -4
KGS_ENOMEM = -5
NTERMS = 8
KGS_STEP_DEFER_TAIL = 1
KGS_STEP_BACKUP = 8

# Every symbol include/kgs_b200.h declares (checked by the CPU test suite).
EXPORTED = (
    "kgs_create", "kgs_create_dist", "kgs_nccl_unique_id", "kgs_destroy",
    "kgs_local_range", "kgs_upload", "kgs_download", "kgs_sweep",
    "kgs_step_dpavf2", "kgs_integrate_host", "kgs_pipeline_plan", "kgs_step_program", "kgs_restore_backup", "kgs_energy_terms",
    "kgs_energy_mass",
    "kgs_all_finite", "kgs_last_error", "kgs_launch_count",
    "kgs_last_step_ms", "kgs_fill_preset", "kgs_abi_version", "kgs_build_flags", "kgs_device_count",
    "kgs_pass_timing", "kgs_pass_stats", "kgs_host_alloc", "kgs_host_free",
    "kgs_set_tuning", "kgs_selftest_division", "kgs_debug_pass",
    "kgs_set_promotion", "kgs_set_param", "kgs_upload_planes", "kgs_download_planes",
)


class KgsCoeffs(ctypes.Structure):
    """kgs_coeffs: StepCoefficients.kernel_args() order (integrator.py:42-45)."""

    _fields_ = [(n, ctypes.c_double) for n in (
        "alpha", "beta", "gcoef", "c_uv", "uv_nbr", "gU", "half_tau",
        "i00", "i01", "i10", "i11")]


class KgsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"kgs error {code}: {msg}")
        self.code = code
        self.msg = msg


_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double
_DP = ctypes.POINTER(ctypes.c_double)


def load() -> ctypes.CDLL:
    """Load libkgs_b200.so (once).  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("KGS_B200_LIB", str(LIB_PATH))
    if not os.path.exists(path):
        raise ImportError(
            f"{path} not found: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    lib = ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
    sig = {
        "kgs_create": (ctypes.c_int, [ctypes.c_int, _I64, _D, _D, ctypes.c_int,
                                      ctypes.POINTER(ctypes.c_int), ctypes.POINTER(_P)]),
        "kgs_create_dist": (ctypes.c_int, [ctypes.c_int, _I64, _D, _D, ctypes.c_int,
                                           ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                                           ctypes.POINTER(_P)]),
        "kgs_nccl_unique_id": (ctypes.c_int, [ctypes.c_char_p]),
        "kgs_destroy": (ctypes.c_int, [_P]),
        "kgs_local_range": (ctypes.c_int, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64),
                                           ctypes.POINTER(_I64)]),
        "kgs_upload": (ctypes.c_int, [_P, _DP, _DP, _DP, _DP]),
        "kgs_download": (ctypes.c_int, [_P, _DP, _DP, _DP, _DP]),
        "kgs_sweep": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int,
                                     ctypes.POINTER(KgsCoeffs)]),
        "kgs_step_dpavf2": (ctypes.c_int, [_P, ctypes.POINTER(KgsCoeffs), _I64, _I64, _I64,
                                           _DP, ctypes.POINTER(_I64), ctypes.c_int]),
        "kgs_integrate_host": (ctypes.c_int, [_P, _DP, _DP, _DP, _DP, ctypes.POINTER(KgsCoeffs),
                                              _I64, _I64, _I64, _DP, _DP,
                                              ctypes.POINTER(_I64), ctypes.c_int]),
        "kgs_pipeline_plan": (_I64, [_I64, _I64, _I64, ctypes.c_int, ctypes.POINTER(_I64), _I64]),
        "kgs_restore_backup": (ctypes.c_int, [_P]),
        "kgs_step_program": (_I64, [_I64, ctypes.c_int, _I64, _I64, _I64, ctypes.c_int,
                                    ctypes.POINTER(_I64), _I64]),
        "kgs_energy_terms": (ctypes.c_int, [_P, _DP]),
        "kgs_energy_mass": (ctypes.c_int, [_P, _D, _D, _D, _D, _DP, _DP]),
        "kgs_all_finite": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int)]),
        "kgs_last_error": (ctypes.c_char_p, [_P]),
        "kgs_launch_count": (_I64, [_P]),
        "kgs_last_step_ms": (_D, [_P]),
        "kgs_fill_preset": (ctypes.c_int, [_P, ctypes.c_int]),
        "kgs_abi_version": (ctypes.c_int, []),
        "kgs_build_flags": (ctypes.c_int, []),
        "kgs_device_count": (ctypes.c_int, []),
        "kgs_pass_timing": (ctypes.c_int, [_P, ctypes.c_int]),
        "kgs_pass_stats": (ctypes.c_int, [_P, ctypes.POINTER(_I64), _DP, ctypes.POINTER(_I64)]),
        "kgs_host_alloc": (ctypes.c_int, [_I64, ctypes.POINTER(_P)]),
        "kgs_host_free": (ctypes.c_int, [_P]),
        "kgs_set_tuning": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_int]),
        "kgs_selftest_division": (ctypes.c_int, [ctypes.c_int, _I64, ctypes.c_uint64,
                                                 ctypes.POINTER(_I64)]),
        "kgs_debug_pass": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, _DP]),
        "kgs_set_promotion": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int]),
        "kgs_set_param": (ctypes.c_int, [_P, ctypes.c_char_p, ctypes.c_int]),
        "kgs_upload_planes": (ctypes.c_int, [_P, ctypes.c_int, _I64, _I64, _DP]),
        "kgs_download_planes": (ctypes.c_int, [_P, ctypes.c_int, _I64, _I64, _DP]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, ctx=None) -> None:
    if rc == KGS_OK:
        return
    msg = load().kgs_last_error(ctx).decode(errors="replace")
    if rc == KGS_EINVAL:
        raise ValueError(msg)
    if rc == KGS_ENONFINITE:
        raise FloatingPointError(msg)
    if rc == KGS_ENOMEM:
        raise MemoryError(msg)
    raise KgsError(rc, msg)


def dptr(a: np.ndarray):
    """double* of a C-contiguous float64 array (no copy)."""
    if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"]:
        raise TypeError("field arrays must be C-contiguous float64")
    return a.ctypes.data_as(_DP)


def coeffs_struct(kernel_args) -> KgsCoeffs:
    vals = tuple(float(v) for v in kernel_args)
    if len(vals) != 11:
        raise ValueError("expected the 11 kernel_args() scalars")
    return KgsCoeffs(*vals)


# kgs_step_program row kinds (include/kgs_b200.h)
PG_LAUNCH, PG_WAIT_XCH, PG_XCH, PG_RECORD, PG_DEFER, PG_PASS_BEGIN, PG_PASS_END = range(1, 8)
KGS_PROGRAM_HEAD_FUSED = 2


def step_program(nx: int, split: bool, nsteps: int, step_offset: int = 0,
                 record_stride: int = 0, defer_tail: bool = False,
                 head_fused: bool = False):
    """The pass program kgs_step_dpavf2 runs on every slab / rank (pure host
    logic in the C library; no device needed): an int64 array of rows
    (kind, col, op1, op2, diag, check, step, xa, xb)."""
    import numpy as np
    lib = load()
    flags = (KGS_STEP_DEFER_TAIL if defer_tail else 0) | (KGS_PROGRAM_HEAD_FUSED if head_fused
                                                          else 0)
    n = lib.kgs_step_program(nx, int(split), nsteps, step_offset, record_stride, flags, None, 0)
    if n < 0:
        raise ValueError("kgs_step_program: bad arguments")
    out = np.zeros((max(n, 1), 9), dtype=np.int64)
    lib.kgs_step_program(nx, int(split), nsteps, step_offset, record_stride, flags,
                         out.ctypes.data_as(ctypes.POINTER(_I64)), n)
    return out[:n]


def device_count() -> int:
    """CUDA devices the library sees (0 without a driver)."""
    return max(0, int(load().kgs_device_count()))
