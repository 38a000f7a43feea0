"""Long-run energy conservation at scale -- BASELINE config 5: 3-D
ellipsoids3d, tau = 0.01, >= 1000 DP-AVF2 steps recording every 10, 2048^3
on 8 GPUs (one slab per GPU), state resident on the devices.

    python tools/long_run.py [--N 1024] [--steps 1000] [--stride 10] [--gpus 1]
    torchrun --nproc-per-node 8 tools/long_run.py --N 2048 --steps 1000 --stride 10

Launch modes as bench.py (bench.Launch): without a launcher, --gpus N drives
N GPUs from one process (fused halo stores over NVLink); under torchrun one
rank per GPU with NCCL halos.  The initial state is the preset evaluated on
the devices (kgs_fill_preset -- at 2048^3 the 275 GB state does not fit in
host memory).  Rank 0 prints one JSON line: energy / mass traces, the
maximum relative energy error, the step rate.
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402  (launch logic)
import paper_2502_09537_b200 as kgs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--stride", type=int, default=10)
    ap.add_argument("--gpus", type=int, default=1)
    a = ap.parse_args()
    import torch
    L = bench.Launch(a.gpus)
    ex = L.executor()
    sc = kgs.get_scenario("ellipsoids3d")
    g = sc.default_grid(a.N)
    dev = kgs.DeviceFieldState.from_preset("ellipsoids3d", g, ex)
    sch = kgs.checkerboard_schedule(g)
    bench.barrier(L.world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr = kgs.integrate(dev, g, sc.params, sch, ex, 0.01, a.steps * 0.01, record_stride=a.stride)
    torch.cuda.synchronize()
    wall = bench.max_over_ranks(time.perf_counter() - t0, L.world)
    finite = dev.is_finite()
    dev.close()
    if L.rank == 0:
        print(json.dumps({
            "config": "BASELINE configs[4]" if (a.N == 2048 and L.n_gpus == 8) else "long run",
            "N": a.N, "n_gpus": L.n_gpus, "mode": L.mode, "steps": a.steps, "tau": 0.01,
            "T": a.steps * 0.01, "record_stride": a.stride, "wall_s": wall,
            "point_updates_per_s": 2.0 * g.M * a.steps / wall,
            "E0": tr.energy[0], "E_final": tr.energy[-1], "max_rel_error": tr.max_rel_error(),
            "rel_error_trace": [float(f"{r:.3e}") for r in tr.rel_error],
            "mass0": tr.mass[0], "mass_final": tr.mass[-1], "finite": finite}), flush=True)


if __name__ == "__main__":
    main()
