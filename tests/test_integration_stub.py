"""The reference-side ctypes binding shown in INTEGRATION.md (what a
maintainer would add as dpavf/b200.py) is real code: it parses, binds only
entry points include/kgs_b200.h declares, and -- on a GPU, imported as a
module of a stand-in `dpavf` package -- reproduces the reference's golden
integration bitwise."""
from __future__ import annotations

import ast
import re
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2502_09537_b200 as kgs
from conftest import assert_bitwise

ROOT = Path(__file__).resolve().parent.parent


def stub_source() -> str:
    text = (ROOT / "INTEGRATION.md").read_text()
    m = re.search(r"```python\n(# dpavf/b200\.py.*?)```", text, re.S)
    assert m, "INTEGRATION.md lost its dpavf/b200.py block"
    return m.group(1)


def test_stub_parses_and_binds_declared_symbols():
    src = stub_source()
    ast.parse(src)
    used = set(re.findall(r"_lib\.(kgs_\w+)", src))
    header = (ROOT / "include" / "kgs_b200.h").read_text()
    declared = set(re.findall(r"\b(kgs_\w+)\s*\(", header))
    assert used and used <= declared, used - declared


@pytest.fixture
def stub(tmp_path, monkeypatch):
    pkg = tmp_path / "dpavf_stub"
    pkg.mkdir()
    (pkg / "__init__.py").write_text("")
    (pkg / "integrator.py").write_text(
        "from paper_2502_09537_b200.integrator import EnergyTrace, precompute_coefficients\n")
    (pkg / "b200.py").write_text(stub_source())
    from paper_2502_09537_b200 import _lib
    # the same file the package loaded (two copies in one process would
    # interpose each other's symbols)
    monkeypatch.setenv("KGS_B200_LIB", _lib.load()._name)
    monkeypatch.syspath_prepend(str(tmp_path))
    import importlib
    mod = importlib.import_module("dpavf_stub.b200")
    yield mod
    for name in ("dpavf_stub.b200", "dpavf_stub.integrator", "dpavf_stub"):
        sys.modules.pop(name, None)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["d3_rand_N12", "d2_fourpeak_N64", "d1_rand_N64"])
def test_stub_reproduces_reference_golden_run(golden, stub, name):
    c = golden.case(name)
    s = c.state(0)
    tr = stub.integrate_b200(s, c.grid, c.params, c.meta["tau"], c.meta["T"],
                             record_stride=c.meta["record_stride"])
    assert_bitwise(s, c.state(1))
    assert s.t == c.meta["t_final"]
    np.testing.assert_allclose(tr.energy, c.trace("energy"), rtol=1e-13, atol=0)
    ours = c.state(0)
    tr2 = kgs.integrate(ours, c.grid, c.params, kgs.checkerboard_schedule(c.grid),
                        kgs.SerialExecutor(), c.meta["tau"], c.meta["T"],
                        record_stride=c.meta["record_stride"])
    assert tr.energy == tr2.energy and tr.steps == tr2.steps and tr.times == tr2.times


@pytest.mark.gpu
def test_stub_nonfinite_matches_package(stub):
    g = kgs.GridSpec(2, -1.0, 1.0, 16)
    p = kgs.PhysParams(1.1, 0.9, 1.2, 0.8)
    s = kgs.seeded_random_state(g, 5, 0.5)
    s.U[7] = np.inf
    a, b = s.copy(), s.copy()
    with pytest.raises(FloatingPointError, match="after step 1"):
        stub.integrate_b200(a, g, p, 0.05, 0.5)
    with pytest.raises(FloatingPointError, match="after step 1"):
        kgs.integrate(b, g, p, kgs.checkerboard_schedule(g), kgs.SerialExecutor(), 0.05, 0.5)
    for f in "PQUV":
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
    assert a.t == b.t
