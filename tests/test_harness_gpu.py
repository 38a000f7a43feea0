"""Harness drivers on the device (reference tests/test_harness.py, the
checkerboard cases; other update orders are rejected with the reason)."""
from __future__ import annotations

import math

import pytest

import paper_2502_09537_b200 as kgs
from paper_2502_09537_b200.harness import (make_schedule, run_bench, run_convergence,
                                           run_energy_experiment)
from paper_2502_09537_b200.scenarios import ScenarioSpec, preset_gaussian2d


def _small_scenario():
    return ScenarioSpec("gaussian2d", 2, -10.0, 10.0, kgs.PhysParams(1.0, 1.0, 1.0, 1.0),
                        preset_gaussian2d)


def test_make_schedule_strategies():
    g = kgs.GridSpec(2, 0.0, 1.0, 8)
    assert make_schedule("checkerboard", g, seed=1, workers=2).strategy == "checkerboard"
    for strat in ("lexicographic-forward", "lexicographic-reverse", "seeded-random",
                  "block-split"):
        with pytest.raises(ValueError, match="does not run on the device"):
            make_schedule(strat, g)
    with pytest.raises(ValueError, match="unknown schedule strategy"):
        make_schedule("zigzag", g)


def test_energy_experiment_rejects_random_orders():
    with pytest.raises(ValueError, match="does not run on the device"):
        run_energy_experiment(_small_scenario(), 16, 0.1, 0.5, seeds=[1, 2, 3])


def test_convergence_too_few_levels():
    with pytest.raises(ValueError):
        run_convergence(_small_scenario(), 16, 0.05, 0.1, levels=1)


def test_bench_repetitions_floor():
    with pytest.raises(ValueError):
        run_bench(2, [16], [1], repetitions=2)


@pytest.mark.gpu
class TestOnDevice:
    def test_single_trace(self):
        tr = run_energy_experiment(_small_scenario(), 32, 0.1, 1.0)
        assert tr.rel_error[0] == 0.0 and tr.max_rel_error() <= 1e-12
        assert len(tr.steps) == 11

    def test_phased_checkerboard_is_the_same_run(self):
        a = run_energy_experiment(_small_scenario(), 32, 0.1, 0.5, workers=2, phased=True)
        b = run_energy_experiment(_small_scenario(), 32, 0.1, 0.5)
        assert a.max_rel_error() <= 1e-12 and a.energy == b.energy

    def test_mass_recorded(self):
        tr = run_energy_experiment(_small_scenario(), 16, 0.1, 0.5)
        assert len(tr.mass) == len(tr.steps) and all(m > 0 for m in tr.mass)

    def test_self_only_convergence(self):
        rep = run_convergence(_small_scenario(), 16, 0.05, 0.25, levels=3,
                              compute_reference=False)
        assert rep.order_u_ref == [] and len(rep.order_u_self) == 1
        assert math.isnan(rep.levels[-1].err_u_self)

    def test_bench_report_shape_and_speedup(self):
        rep = run_bench(2, [16, 32], [1], strategy="checkerboard", steps=1, repetitions=3)
        assert len(rep.rows) == 2 and all(r.seconds_per_step > 0 for r in rep.rows)
        assert (16, 32) in rep.scaling_ratios
        rep = run_bench(2, [16], [1, 2], strategy="checkerboard", steps=1, repetitions=3)
        base = [r for r in rep.rows if r.workers == 1][0]
        assert base.speedup == pytest.approx(1.0)
