"""The multi-rank (torchrun) code path on ONE GPU: a 1-rank dist context
that exchanges its faces with itself over NCCL (KGS_SELF_EXCHANGE=1,
include/kgs_b200.h kgs_create_dist) instead of wrapping them in the kernel.
Everything a rank of an N-GPU job runs executes here on real hardware --
ghost planes, the interior/boundary split of every pass, ncclSend/ncclRecv
on the comm stream, the event waits of the pass program -- and the fields
must stay bitwise the reference's: a missing or late exchange leaves stale
ghost planes, which changes the bits after the first pass.  (Reference
analogue: worker-count determinism, dpavf tests/test_executor.py:83-99.)
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2502_09537_b200 as kgs
from conftest import assert_bitwise

pytestmark = pytest.mark.gpu

E_RTOL = 1e-13


@pytest.fixture(autouse=True)
def _self_exchange(monkeypatch):
    kgs.clear_contexts()
    monkeypatch.setenv("KGS_SELF_EXCHANGE", "1")
    yield
    kgs.clear_contexts()


def _rank0():
    return kgs.DistributedExecutor(rank=0, world_size=1, device=0)


@pytest.mark.parametrize("name", ["d3_rand_N8", "d3_ellip_N16", "d3_rand_N12",
                                  "d2_fourpeak_N64", "d2_rand_N32"])
def test_self_exchange_integrate_bitwise_vs_reference(golden, name):
    c = golden.case(name)
    s = c.state(0)
    tr = kgs.integrate(s, c.grid, c.params, kgs.checkerboard_schedule(c.grid), _rank0(),
                       c.meta["tau"], c.meta["T"], record_stride=c.meta["record_stride"])
    assert_bitwise(s, c.state(1))
    np.testing.assert_allclose(tr.energy, c.trace("energy"), rtol=E_RTOL, atol=0)
    np.testing.assert_allclose(tr.mass, c.trace("mass"), rtol=E_RTOL, atol=0)


@pytest.mark.parametrize("N", [64, 128])
def test_self_exchange_march_path_matches_single_gpu(N):
    """The marching kernel at 64^3 / 128^3 with a record every step: the
    self-exchanging rank and the ordinary wrapped single slab give the same
    bits (and the same records)."""
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(N)
    args = kgs.precompute_coefficients(sc.params, 0.005, g).kernel_args()
    host = kgs.seeded_random_state(g, 11, 0.1)
    out = {}
    for key, ex in (("self", _rank0()), ("wrap", kgs.SerialExecutor())):
        dev = kgs.DeviceFieldState.from_host(host, g, ex)
        try:
            terms, bad = dev.ctx.step_dpavf2(args, 6, 0, 1)
            assert bad == 0
            out[key] = (dev.to_host(), terms)
        finally:
            dev.close()
        kgs.clear_contexts()
    assert_bitwise(out["self"][0], out["wrap"][0])
    np.testing.assert_allclose(out["self"][1], out["wrap"][1], rtol=1e-13, atol=0)


CHILD = """
import sys
sys.path.insert(0, %r)
import paper_2502_09537_b200 as kgs
sc = kgs.get_scenario("ellipsoids3d")
g = sc.default_grid(16)
s = kgs.seeded_random_state(g, 5, 0.1)
ex = kgs.DistributedExecutor(rank=0, world_size=1, device=0)
kgs.step_dpavf2(s, kgs.checkerboard_schedule(g), kgs.precompute_coefficients(sc.params, 0.01, g), ex, g)
import numpy as np
print("stepped", all(bool(np.isfinite(getattr(s, f)).all()) for f in "PQUV"))
"""


def test_self_exchange_initialises_nccl():
    """The hook really goes through NCCL: NCCL_DEBUG=INFO shows a 1-rank
    communicator being created by the library."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parent.parent)
    env = dict(os.environ, KGS_SELF_EXCHANGE="1", NCCL_DEBUG="INFO")
    out = subprocess.run([sys.executable, "-c", CHILD % root], env=env, capture_output=True,
                         text=True, timeout=300)
    text = out.stdout + out.stderr
    assert out.returncode == 0, text[-2000:]
    assert "stepped True" in text
    assert "Init COMPLETE" in text and "nranks 1" in text, text[-2000:]
