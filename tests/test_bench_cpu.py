"""CPU: bench.py's launch logic -- ``--gpus N`` without a launcher drives N
devices from one process (never silently fewer), the weak-scaling grid
sizes, and the reference arm's command-line contract."""
from __future__ import annotations

import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2502_09537_b200 as kgs  # noqa: E402


@pytest.fixture
def devices(monkeypatch):
    import torch

    def set_count(n):
        monkeypatch.setattr(torch.cuda, "device_count", lambda: n)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "LOCAL_WORLD_SIZE"):
        monkeypatch.delenv(k, raising=False)
    return set_count


def test_gpus_n_builds_an_n_device_single_process_plan(devices):
    devices(8)
    for n in (1, 2, 4, 8):
        L = bench.Launch(n)
        ex = L.executor()
        assert isinstance(ex, kgs.CudaExecutor)
        assert L.n_gpus == n and ex.devices == tuple(range(n)) and ex.slabs_per_device == 1
        assert ex.nslabs == n                      # one slab per GPU, n_gpus == GPUs used
    assert bench.Launch(2).mode == "single-process+peer-stores"


def test_gpus_n_fails_loudly_with_fewer_devices(devices):
    devices(1)
    with pytest.raises(SystemExit, match="only 1 CUDA devices"):
        bench.Launch(2)
    devices(0)
    with pytest.raises(SystemExit):
        bench.Launch(1)


def test_weak_scaling_grid_sizes():
    assert bench.weak_n(1024, 1) == 1024
    assert bench.weak_n(1024, 8) == 2048            # BASELINE configs[4]: 2048^3 on 8 GPUs
    for g in (2, 4, 8):
        n = bench.weak_n(1024, g)
        assert n % 128 == 0 and n % g == 0
        assert abs(n**3 / g / 1024**3 - 1) < 0.1    # ~1024^3 points per GPU


def test_bench_without_gpus_exits_nonzero():
    """No silent CPU fallback: on this GPU-less box the default run fails."""
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "1", "--warmup", "3",
                        "--no-e2e", "--no-cpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "CUDA devices visible" in (r.stderr + r.stdout)


def _agree_worker(rank, world, port, q):
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        q.put((rank, bench.all_ranks(rank != 1, world), bench.all_ranks(True, world)))
    finally:
        dist.destroy_process_group()


def test_collective_decisions_agree_over_ranks():
    """bench.all_ranks: a decision that gates collective work (host memory
    for the e2e inputs) holds on every rank or on none."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_agree_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(3))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [False] * 3 and [r[2] for r in res] == [True] * 3
