"""CPU: pin the oracle (and the package's host-side objects) to the golden
vectors the reference itself produced (tests/golden/make_golden.py).

Mirrors the reference's own parity pins: bitwise
checkerboard results (tests/test_oracle.py:60-105), the golden energy
(tests/test_scenarios.py:137-143), SplitMix64 known answers
(tests/test_prng.py:17-21) and the coefficient arithmetic
(tests/test_integrator.py:18-54).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from conftest import assert_bitwise, run_names, sweep_names
from paper_2502_09537_b200 import (GridSpec, PhysParams, get_scenario,
                                   precompute_coefficients, seeded_random_state)
from paper_2502_09537_b200.prng import SplitMix64, uniform_array
from paper_2502_09537_b200.scenarios import preset_soliton1d

GOLDEN_ENERGY_SEED42 = 66.88429062581992  # reference tests/test_scenarios.py:164


# ---- coefficients --------------------------------------------------------
@pytest.mark.parametrize("name", run_names() + sweep_names())
def test_kernel_args_bitwise(golden, name):
    c = golden.case(name)
    tau = c.meta["tau"] / 2.0 if c.meta["kind"] == "integrate" else c.meta["tau"]
    ours = precompute_coefficients(c.params, tau, c.grid).kernel_args()
    assert ours == c.kernel_args
    assert oracle.kernel_args(c.params, tau, c.grid) == c.kernel_args


# ---- oracle restatements vs the reference ----------------------------------
@pytest.mark.parametrize("name", run_names())
def test_numpy_oracle_integrate_bitwise(golden, name):
    c = golden.case(name)
    g, p = c.grid, c.params
    s = c.state(0)
    stride = c.meta["record_stride"]
    energies = []
    for n in range(1, c.meta["n_steps"] + 1):
        oracle.numpy_step_dpavf2(s, c.kernel_args, g)
        if n % stride == 0:
            energies.append(oracle.discrete_energy(s, p, g))
    assert_bitwise(s, c.state(1))
    ref_e = c.trace("energy")[1:]
    assert len(energies) == len(ref_e)
    np.testing.assert_allclose(energies, ref_e, rtol=1e-15, atol=0)


@pytest.mark.parametrize("workers", [1, 4])
@pytest.mark.parametrize("name", run_names())
def test_c_oracle_integrate_bitwise(golden, name, workers):
    c = golden.case(name)
    orc = oracle.CheckerboardOracle(c.grid.d, c.grid.N)
    s = c.state(0)
    orc.step_dpavf2(s, c.kernel_args, c.meta["n_steps"], workers=workers)
    assert_bitwise(s, c.state(1))


@pytest.mark.parametrize("name", sweep_names())
def test_oracle_single_sweeps_bitwise(golden, name):
    c = golden.case(name)
    adj = c.meta["kind"] == "adjoint"
    s = c.state(0)
    oracle.CheckerboardOracle(c.grid.d, c.grid.N).sweep(s, c.kernel_args, adj, workers=3)
    assert_bitwise(s, c.state(1))
    s = c.state(0)
    for colour in ((0, 1) if adj else (1, 0)):
        oracle.numpy_half_sweep(s, c.kernel_args, c.grid, colour, adj)
    assert_bitwise(s, c.state(1))


def test_golden_energy_constant(golden):
    c = golden.case("golden_seed42")
    s = c.state(0)
    e = oracle.discrete_energy(s, PhysParams(), c.grid)
    assert e == pytest.approx(GOLDEN_ENERGY_SEED42, rel=1e-14)
    assert e == c.meta["energy"]
    assert oracle.mass(s, c.grid) == c.meta["mass"]


def test_energy_terms_exact_vs_numpy(golden):
    """The exact-sum term oracle reproduces the reference energy formula."""
    from paper_2502_09537_b200.grid import energy_from_terms
    for name in ("golden_seed42", "d3_rand_N8", "d2_gauss_N16"):
        c = golden.case(name)
        s = c.state(0)
        e, m = energy_from_terms(oracle.energy_terms(s, c.grid), c.params, c.grid)
        assert e == pytest.approx(oracle.discrete_energy(s, c.params, c.grid), rel=1e-14)
        assert m == pytest.approx(oracle.mass(s, c.grid), rel=1e-14)


# ---- host-side objects of the package ------------------------------------
def test_splitmix_known_answers():
    rng = SplitMix64(0)
    assert rng.next_u64() == 0xE220A8397B1DCDAF
    assert rng.next_u64() == 0x6E789E6AA1B965F4


def test_uniform_array_matches_scalar_stream():
    rng = SplitMix64(12345)
    expect = np.array([-0.3 + 0.7 * rng.next_unit() for _ in range(1000)])
    got = uniform_array(1000, 12345, -0.3, 0.4)
    assert np.array_equal(got, expect)


@pytest.mark.parametrize("name", [n for n in run_names() + sweep_names()])
def test_seeded_random_state_bitwise(golden, name):
    c = golden.case(name)
    if c.meta.get("seed") is None:
        pytest.skip("not a seeded case")
    seed, amp = c.meta["seed"]
    assert_bitwise(seeded_random_state(c.grid, seed, amp), c.state(0))


@pytest.mark.parametrize("sc", ["gaussian2d", "fourpeak2d", "ellipsoids3d"])
def test_presets_bitwise(golden, sc):
    c = golden.case(f"preset_{sc}")
    spec = get_scenario(sc)
    assert_bitwise(spec.state(spec.default_grid(c.meta["N"])), c.state(0))


def test_soliton_ic_bitwise(golden):
    c = golden.case("d1_soliton_N1024")
    assert_bitwise(preset_soliton1d(c.grid), c.state(0))
    assert get_scenario("soliton1d").default_grid(1024) == c.grid


def test_c_oracle_tables_match_reference_conventions():
    """Neighbour table columns (-x,+x,-y,+y,-z,+z) and red = parity 1
    (reference grid.py:54-64, ordering.py:125-128)."""
    g = GridSpec(3, 0.0, 1.0, 4)
    orc = oracle.CheckerboardOracle(3, 4)
    idx = np.arange(g.M).reshape(g.shape)
    cols = []
    for ax in range(3):
        cols.append(np.roll(idx, 1, axis=ax).ravel())
        cols.append(np.roll(idx, -1, axis=ax).ravel())
    assert np.array_equal(orc.nbrs, np.stack(cols, axis=1))
    parity = np.indices(g.shape).sum(axis=0).ravel() % 2
    assert np.array_equal(orc.red, np.nonzero(parity == 1)[0])
    assert np.array_equal(orc.black, np.nonzero(parity == 0)[0])


# ---- the table-free restatement (checker for the 1024^3 headline config) --
@pytest.mark.parametrize("name", run_names())
def test_table_free_oracle_integrate_bitwise(golden, name):
    c = golden.case(name)
    s = c.state(0)
    oracle.TableFreeOracle(c.grid.d, c.grid.N).step_dpavf2(s, c.kernel_args, c.meta["n_steps"])
    assert_bitwise(s, c.state(1))


@pytest.mark.parametrize("name", sweep_names())
def test_table_free_oracle_single_sweeps_bitwise(golden, name):
    c = golden.case(name)
    s = c.state(0)
    oracle.TableFreeOracle(c.grid.d, c.grid.N).sweep(s, c.kernel_args,
                                                     c.meta["kind"] == "adjoint")
    assert_bitwise(s, c.state(1))


@pytest.mark.parametrize("d,N", [(3, 24), (2, 64), (1, 128), (3, 2)])
def test_table_free_oracle_matches_table_oracle(d, N):
    """Beyond the golden sizes: random state, 3 steps, both C restatements."""
    g = GridSpec(d, -3.0, 3.0, N)
    a = seeded_random_state(g, 77, 0.5)
    b = a.copy()
    args = oracle.kernel_args(PhysParams(-0.4, 0.1, 0.1, 0.2), 0.005, g)
    oracle.TableFreeOracle(d, N).step_dpavf2(a, args, 3)
    oracle.CheckerboardOracle(d, N).step_dpavf2(b, args, 3, workers=2)
    assert_bitwise(a, b)


@pytest.mark.parametrize("d,N", [(3, 16), (2, 64), (1, 256), (3, 2)])
def test_table_free_energy_terms(d, N):
    g = GridSpec(d, -3.0, 3.0, N)
    s = seeded_random_state(g, 11, 0.5)
    np.testing.assert_allclose(oracle.TableFreeOracle(d, N).energy_terms(s),
                               oracle.energy_terms(s, g), rtol=1e-13, atol=0)
