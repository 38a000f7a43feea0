"""Shared fixtures: golden vectors produced by the reference itself
(tests/golden/make_golden.py) and helpers to rebuild grids/params/states."""
from __future__ import annotations

import json
import sys
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from paper_2502_09537_b200 import FieldState, GridSpec, PhysParams  # noqa: E402

GOLDEN = ROOT / "tests" / "golden" / "kgs_golden.npz"


def experimental_build() -> bool:
    """The loaded library was built with -DKGS_EXPERIMENTAL (build.py
    --experimental, selected with KGS_B200_LIB): the slower fused one-march
    step, march variants 4..6 and kgs_debug_pass are only there."""
    try:
        from paper_2502_09537_b200 import _lib
        return bool(_lib.load().kgs_build_flags() & 1)
    except Exception:
        return False


needs_experimental = pytest.mark.skipif(
    not experimental_build(), reason="experimental kernels: needs libkgs_b200_exp.so "
                                     "(KGS_B200_LIB, build.py --experimental)")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")


@dataclass
class Case:
    name: str
    meta: dict
    arrays: dict

    @property
    def grid(self) -> GridSpec:
        m = self.meta
        return GridSpec(m["d"], m["a"], m["b"], m["N"])

    @property
    def params(self) -> PhysParams:
        return PhysParams(*self.meta["params"])

    def state(self, which: int) -> FieldState:
        a = self.arrays
        return FieldState(*(np.array(a[f"{f}{which}"], dtype=np.float64) for f in "PQUV"), 0.0)

    @property
    def kernel_args(self) -> tuple:
        return tuple(float(v) for v in self.arrays["kernel_args"])

    def trace(self, key: str) -> np.ndarray:
        return self.arrays["trace_" + key]


class Golden:
    def __init__(self, path: Path = GOLDEN):
        z = np.load(path)
        self.meta = json.loads(bytes(z["__meta__"]).decode())
        self._arrays: dict[str, dict] = {}
        for key in z.files:
            if key == "__meta__":
                continue
            name, field = key.split("/", 1)
            self._arrays.setdefault(name, {})[field] = z[key]

    def case(self, name: str) -> Case:
        return Case(name, self.meta[name], self._arrays.get(name, {}))

    def names(self, kind: str | tuple) -> list[str]:
        kinds = (kind,) if isinstance(kind, str) else kind
        return [n for n, m in self.meta.items() if m["kind"] in kinds]


_GOLDEN = Golden()


@pytest.fixture(scope="session")
def golden() -> Golden:
    return _GOLDEN


def run_names():
    return _GOLDEN.names("integrate")


def sweep_names():
    return _GOLDEN.names(("base", "adjoint"))


def assert_bitwise(a: FieldState, b: FieldState, equal_nan: bool = False):
    for f in "PQUV":
        x, y = getattr(a, f), getattr(b, f)
        assert np.array_equal(x, y, equal_nan=equal_nan), (
            f"field {f}: max |diff| = {np.nanmax(np.abs(x - y))}")
