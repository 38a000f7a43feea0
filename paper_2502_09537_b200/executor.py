"""Executors: which GPUs a sweep runs on.

The reference executors (``dpavf/executor.py:17-93``) decide which host
thread calls a lane function over an index array, with a futures barrier
between the red and black phases.  On the B200 the colour phase is one
kernel launch and the barrier is stream order, so an executor here only
names the devices and the slab decomposition along axis 0:

* ``SerialExecutor`` / ``PhasedExecutor(workers)`` -- accepted for
  drop-in compatibility; both run on one GPU (``cuda:0``).  ``workers`` is
  kept as an attribute and has no effect on the result (bitwise identical
  for every worker count, like the reference, ``executor.py:1-8``).  Their
  ``run(schedule, lane_fn)`` keeps the reference's host semantics for code
  that drives its own lane functions (``executor.py:39-71``): the serial
  order on the calling thread, or phase by phase over a thread pool with a
  full barrier; the device sweeps never go through it.
* ``CudaExecutor(devices, slabs_per_device=1)`` -- single process driving
  one or more GPUs; the grid is split into ``len(devices)*slabs_per_device``
  slabs with face halos copied between them (several slabs on one device
  are "virtual slabs": the decomposition-invariance test on one GPU).
* ``DistributedExecutor()`` -- one process per GPU under torchrun; this
  rank owns one slab and halos travel over NCCL (see device.py).

``ExecutorConfig(mode, workers)`` accepts "serial", "phased" and "cuda"
(``workers`` = GPU count for "cuda"); any other mode is rejected exactly
as the reference does (``executor.py:22-26``).
"""
from __future__ import annotations

from dataclasses import dataclass

MODES = ("serial", "phased", "cuda")


@dataclass(frozen=True)
class ExecutorConfig:
    mode: str = "serial"   # "serial" | "phased" | "cuda"
    workers: int = 1

    def __post_init__(self):
        if self.mode not in MODES:
            raise ValueError(f"unknown executor mode {self.mode!r}")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")

    def build(self):
        if self.mode == "serial":
            return SerialExecutor()
        if self.mode == "phased":
            return PhasedExecutor(self.workers)
        # one slab per GPU; with fewer GPUs than workers, virtual slabs on
        # cuda:0 (same results bitwise: decomposition invariance)
        if self.workers <= _device_count():
            return CudaExecutor(tuple(range(self.workers)))
        return CudaExecutor((0,), slabs_per_device=self.workers)


def _device_count() -> int:
    """CUDA devices visible to the library (kgs_device_count, i.e.
    cudaGetDeviceCount); 0 without a driver or library."""
    try:
        from . import _lib
        return _lib.device_count()
    except Exception:
        return 0


class _DeviceExecutor:
    devices: tuple = (0,)
    slabs_per_device: int = 1

    @property
    def nslabs(self) -> int:
        return len(self.devices) * self.slabs_per_device

    def slab_devices(self) -> tuple:
        return tuple(d for d in self.devices for _ in range(self.slabs_per_device))

    def key(self) -> tuple:
        return ("local", self.slab_devices())

    def run(self, schedule, lane_fn) -> None:
        raise TypeError(
            "device executors do not run host lane functions; use step_base/"
            "step_adjoint/step_dpavf2/integrate from paper_2502_09537_b200")

    def close(self) -> None:
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class SerialExecutor(_DeviceExecutor):
    """One GPU (cuda:0); the drop-in for dpavf.executor.SerialExecutor."""

    workers = 1

    def run(self, schedule, lane_fn) -> None:
        """Host lane function over the whole serial order (executor.py:39-40)."""
        lane_fn(schedule.serial_order())


class PhasedExecutor(_DeviceExecutor):
    """One GPU (cuda:0); the drop-in for dpavf.executor.PhasedExecutor."""

    def __init__(self, workers: int):
        if workers < 1:
            raise ValueError("workers must be >= 1")
        self.workers = workers
        self._pool = None

    def run(self, schedule, lane_fn) -> None:
        """Host lane functions phase by phase, lanes of a parallel phase on a
        thread pool, full barrier between phases; lane errors re-raised
        (executor.py:60-71)."""
        if not getattr(schedule, "validated", True):
            raise ValueError(
                "schedule has not passed validation; run validate_schedule first")
        for phase in schedule.phases:
            if phase.parallel and self.workers > 1 and len(phase.lanes) > 1:
                if self._pool is None:
                    from concurrent.futures import ThreadPoolExecutor
                    self._pool = ThreadPoolExecutor(max_workers=self.workers)
                futures = [self._pool.submit(lane_fn, lane) for lane in phase.lanes]
                for f in futures:
                    f.result()
            else:
                for lane in phase.lanes:
                    lane_fn(lane)

    def close(self) -> None:
        if self._pool is not None:
            self._pool.shutdown(wait=True)
            self._pool = None


class CudaExecutor(_DeviceExecutor):
    """Single process over ``devices`` with ``slabs_per_device`` slabs each."""

    def __init__(self, devices=(0,), slabs_per_device: int = 1):
        devices = tuple(int(d) for d in devices)
        if not devices:
            raise ValueError("need at least one device")
        if slabs_per_device < 1:
            raise ValueError("slabs_per_device must be >= 1")
        self.devices = devices
        self.slabs_per_device = int(slabs_per_device)
        self.workers = self.nslabs


class DistributedExecutor(_DeviceExecutor):
    """One rank of a torchrun job: slab ``rank`` of ``world_size`` on
    ``cuda:local_rank``; halos over NCCL.  torch.distributed must be
    initialised (any backend) before the first use."""

    def __init__(self, rank: int | None = None, world_size: int | None = None,
                 device: int | None = None):
        import os
        if rank is None or world_size is None:
            import torch.distributed as dist
            rank = dist.get_rank() if rank is None else rank
            world_size = dist.get_world_size() if world_size is None else world_size
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", rank))
        self.rank, self.world_size, self.device = int(rank), int(world_size), int(device)
        self.devices = (self.device,)
        self.workers = self.world_size

    def key(self) -> tuple:
        return ("dist", self.rank, self.world_size, self.device)


def resolve(executor) -> _DeviceExecutor:
    """Map any executor (ours, the reference's, or None) to a device plan."""
    if isinstance(executor, _DeviceExecutor):
        return executor
    if executor is None or hasattr(executor, "run"):
        # reference SerialExecutor / PhasedExecutor or a duck-typed stand-in
        return SerialExecutor()
    raise TypeError(f"not an executor: {executor!r}")
