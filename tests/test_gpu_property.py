"""Randomised parity (hypothesis): any even N, dimension, slab count, physical
parameters, step size, step count and record stride -- the device path is
bitwise the oracle's restatement of the reference (oracle/, pinned to the
reference's golden vectors), and every energy record matches the oracle's
discrete energy.  Covers the small-grid resident kernel and the per-pass
kernels (knob `resident`), single and multi-slab decompositions."""
from __future__ import annotations

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle
import paper_2502_09537_b200 as kgs
from conftest import assert_bitwise
from paper_2502_09537_b200.grid import energy_from_terms

pytestmark = pytest.mark.gpu


@st.composite
def cases(draw):
    d = draw(st.integers(1, 3))
    nmax = {1: 128, 2: 24, 3: 12}[d]
    N = 2 * draw(st.integers(1, nmax // 2))
    # slabs split axis 0 into planes; a 1-D grid is a single plane
    slabs = draw(st.sampled_from([s for s in (1, 2, 4)
                                  if s == 1 or (d > 1 and N % s == 0 and N // s >= 2)]))
    params = kgs.PhysParams(draw(st.floats(0.2, 2.0)), draw(st.floats(0.2, 2.0)),
                            draw(st.floats(0.0, 2.0)), draw(st.floats(-1.0, 1.0)))
    a = draw(st.floats(-12.0, -0.5))
    b = a + draw(st.floats(1.0, 24.0))
    tau = draw(st.floats(1e-3, 0.1))
    steps = draw(st.integers(1, 6))
    stride = draw(st.integers(0, 3))
    resident = draw(st.booleans())
    seed = draw(st.integers(0, 2**31))
    return d, N, slabs, params, a, b, tau, steps, stride, resident, seed


@settings(max_examples=200, deadline=None, suppress_health_check=list(HealthCheck))
@given(cases())
def test_random_cases_bitwise_vs_oracle(case):
    d, N, slabs, params, a, b, tau, steps, stride, resident, seed = case
    g = kgs.GridSpec(d, a, b, N)
    s0 = kgs.seeded_random_state(g, seed, 0.5)
    args = kgs.precompute_coefficients(params, tau / 2.0, g).kernel_args()
    ex = None if slabs == 1 else kgs.CudaExecutor((0,), slabs_per_device=slabs)
    dev = kgs.DeviceFieldState.from_host(s0, g, ex)
    dev.ctx.set_param("resident", int(resident))
    terms, bad = dev.ctx.step_dpavf2(args, steps, 0, stride)
    got = dev.to_host()
    dev.close()
    assert bad == 0
    ref = s0.copy()
    energies = []
    for n in range(1, steps + 1):
        oracle.numpy_step_dpavf2(ref, args, g, 1)
        if stride and n % stride == 0:
            energies.append(oracle.discrete_energy(ref, params, g))
    assert_bitwise(got, ref)
    assert len(terms) == len(energies)
    h2, hd = g.h ** 2, g.h ** g.d
    for t, e in zip(terms, energies):
        e_dev, _ = energy_from_terms(t, params, g)
        # E = h^d (quad/2 - gamma * coupling) can cancel almost completely for
        # random parameters; summation-order rounding scales with the terms
        scale = hd * (0.5 * (params.kappa1 * (t[0] + t[1]) / h2 + params.kappa2 * t[2] / h2
                             + t[3] + params.mu ** 2 * t[4]) + abs(params.gamma * t[5]))
        assert abs(e_dev - e) <= 1e-12 * scale + 1e-300, (e_dev, e, scale)
