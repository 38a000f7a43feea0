"""Benchmark: 3-D KGS checkerboard DP-AVF2 point-updates/s on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--N 1024] [--scaling strong|weak]

Workload (BASELINE.json configs[3], the metric's named config): 3-D
ellipsoids3d on a 1024^3 fp64 periodic grid, tau = 0.01.  A "step" is one
DP-AVF2 time step = 2 * N^3 point-updates.  Inputs are
generated on the device (synthetic, the reference's ellipsoids3d formulas);
the 32 GiB state is far larger than the 126 MB L2, so no flush is needed.

ours:       value = all ranks' point-updates / max-over-ranks device time of K
            fused steps (CUDA events on the library's stream); e2e = the same
            metric through the public API integrate() on a pinned host
            FieldState (upload, K steps, download inside the timed region).
reference:  the reference's CPU algorithm (oracle/ port: neighbour table,
            colour lanes, phased threads) on all host cores, on a bounded
            256^3 sample of the same scenario; rank 0 only.
Multi-GPU (torchrun): slab decomposition along axis 0, NCCL halos; strong
scaling at 1024^3 by default (--scaling weak: N = 1024 * cbrt(G) when G is
a cube, else strong).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "3D KGS grid-point updates/s at 1/2/4/8 B200; % of HBM roofline vs CPU ref"
UNIT = "point-updates/s"
BYTES_PER_UPDATE = 64          # P,Q,U,V read+write once per update
DESIGN_BYTES_PER_UPDATE = 44   # colour-split fused passes
DIAG_STEPS = 5                # steps of the record-every-step run (diagnostics price)
TAU = 0.01
SCENARIO = "ellipsoids3d"


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback"}


def ncu_traffic() -> dict | None:
    """dram bytes per fused-pass launch from the committed ncu summary."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text())
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
                self.lines = [l for l in out.splitlines() if l.strip()]
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            parts = [x.strip() for x in l.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(gpus: int):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def grid_n(args, world: int) -> int:
    if args.scaling == "weak":
        c = round(world ** (1 / 3))
        if c ** 3 == world:
            return args.N * c
    return args.N


# --------------------------------------------------------------------------
def cpu_baseline(steps: int, warmup: int, N: int = 256) -> dict:
    """Reference CPU algorithm (oracle port) on all host threads, bounded
    sample: N^3 ellipsoids3d, `steps` DP-AVF2 steps after `warmup`."""
    import oracle
    import paper_2502_09537_b200 as kgs
    sc = kgs.get_scenario(SCENARIO)
    g = sc.default_grid(N)
    s = sc.state(g)
    orc = oracle.CheckerboardOracle(3, N)
    threads = oracle.CheckerboardOracle.max_threads()
    args = oracle.kernel_args(sc.params, TAU / 2.0, g)
    orc.step_dpavf2(s, args, max(warmup, 1), workers=threads)
    t0 = time.perf_counter()
    orc.step_dpavf2(s, args, steps, workers=threads)
    dt = time.perf_counter() - t0
    return {"value": 2.0 * g.M * steps / dt, "unit": UNIT, "cores": threads,
            "kind": "port",
            "sample": f"{N}^3 {SCENARIO}, {steps} DP-AVF2 steps after {max(warmup, 1)} warm-up, "
                      f"PhasedExecutor-style {threads} threads (oracle/kgs_oracle.c)",
            "seconds": dt}


def run_reference(args):
    rank, world, _ = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), 0
    if rank != 0:
        return
    N = grid_n(args, world)
    steps = max(1, min(args.steps, 40))
    cb = cpu_baseline(steps, args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT,
        "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * cb["seconds"] / steps,
        "higher_is_better": True,
        "scaling": "weak" if (args.scaling == "weak" and round(world ** (1 / 3)) ** 3 == world)
                   else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"3D KGS {SCENARIO} N={N}^3 fp64, tau={TAU}, checkerboard DP-AVF2",
                   "sample": cb["sample"]},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
def run_ours(args):
    import torch
    import paper_2502_09537_b200 as kgs

    rank, world, local = dist_setup(args.gpus)
    N = grid_n(args, world)
    sc = kgs.get_scenario(SCENARIO)
    g = sc.default_grid(N)
    ex = kgs.DistributedExecutor(rank, world, local) if world > 1 else kgs.CudaExecutor((local,))
    sch = kgs.checkerboard_schedule(g)
    coeffs = kgs.precompute_coefficients(sc.params, TAU / 2.0, g)
    kargs = coeffs.kernel_args()
    K, W = args.steps, args.warmup

    dev = kgs.DeviceFieldState.from_preset(SCENARIO, g, ex)
    ctx = dev.ctx
    points_local = ctx.points
    # warm-up (untimed)
    ctx.step_dpavf2(kargs, W, 0, 0)
    barrier(world)
    torch.cuda.synchronize()
    l0 = ctx.launch_count()
    ctx.pass_timing(True)
    with ClockSampler(local) as clk:
        barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        terms, bad = ctx.step_dpavf2(kargs, K, W, K)     # one record at the end
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        barrier(world)
    ms_dev = ctx.last_step_ms()
    launches = ctx.launch_count() - l0
    n_pass, pass_ms, pass_pts = ctx.pass_stats()
    ctx.pass_timing(False)
    if bad:
        raise FloatingPointError(f"non-finite state at step {bad}")
    ms = max_over_ranks(ms_dev, world)
    updates = 2.0 * g.M * K                      # whole job, all ranks
    value = updates / (ms / 1e3)

    # roofline of the dominant kernel (fused colour pass), live
    avg_pass_ms = pass_ms / max(n_pass, 1)
    upd_per_launch = 2 * pass_pts                # each point of the colour updated twice
    pk = peaks()
    achieved = BYTES_PER_UPDATE * upd_per_launch / (avg_pass_ms / 1e3) / 1e9
    nc = ncu_traffic()
    traffic = None
    if nc and nc.get("N") == N and nc.get("world") == world:
        traffic = nc.get("dram_bytes_per_launch")
    roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / pk["hbm_gbs"], "traffic": traffic,
            "peak_source": pk["source"],
            "kernel": "march_pass (fused K3/K4 colour pass, TMA ring)",
            "algorithmic_bytes_per_update": BYTES_PER_UPDATE,
            "avg_launch_ms": avg_pass_ms, "launches_timed": n_pass,
            "design_bytes_per_update": DESIGN_BYTES_PER_UPDATE,
            "design_frac": DESIGN_BYTES_PER_UPDATE * upd_per_launch / (avg_pass_ms / 1e3) / 1e9
            / pk["hbm_gbs"]}
    if traffic:
        # what the kernel actually moves: ncu DRAM bytes per launch / live launch time
        roof["dram_achieved"] = traffic / (avg_pass_ms / 1e3) / 1e9
        roof["dram_frac"] = roof["dram_achieved"] / pk["hbm_gbs"]
        roof["dram_bytes_per_update"] = traffic / upd_per_launch

    # energy sanity (the timed run recorded step W+K)
    e = kgs.grid.energy_from_terms(terms[0], sc.params, g)[0] if len(terms) else None

    # price of the diagnostics (SURVEY.md §7 timed runs): a few more steps with
    # an energy/mass record after EVERY step, the reference's record_stride=1
    R = DIAG_STEPS
    barrier(world)
    terms_r, bad_r = ctx.step_dpavf2(kargs, R, W + K, 1)
    ms_r = max_over_ranks(ctx.last_step_ms(), world)
    if bad_r:
        raise FloatingPointError(f"non-finite state at step {bad_r}")
    em = [kgs.grid.energy_from_terms(t, sc.params, g) for t in [terms[-1], *terms_r]]
    diag = {"record_stride": 1, "steps": R, "ms_per_step": ms_r / R,
            "value": 2.0 * g.M * R / (ms_r / 1e3), "unit": UNIT,
            "cost_vs_unrecorded": (ms_r / R) / (ms / K),
            "max_rel_energy_change": max(abs(E - em[0][0]) / abs(em[0][0]) for E, _ in em),
            "max_rel_mass_change": max(abs(m - em[0][1]) / abs(em[0][1]) for _, m in em),
            "note": "energy is the scheme's invariant (round-off drift); mass is not conserved "
                    "by DP-AVF2 and drifts at the reference's own rate (grows with N)"}

    # e2e through the public API: integrate() on a pinned host state
    e2e = None
    if not args.no_e2e:
        if world == 1:
            host = kgs.FieldState.pinned(g)
        else:   # each rank holds only its own slab on the host (32 GiB / world)
            from paper_2502_09537_b200.device import pinned_empty
            host = kgs.FieldState(*(pinned_empty(points_local) for _ in range(4)), 0.0)
        dev.download(host)
        dev.close()
        del dev
        # untimed warm-up call (W steps): creates the cached context and its
        # pipeline buffers, as the device timing's warm-up steps do
        kgs.integrate(host, g, sc.params, sch, ex, TAU, W * TAU, record_stride=W)
        barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        kgs.integrate(host, g, sc.params, sch, ex, TAU, K * TAU, record_stride=K)
        torch.cuda.synchronize()
        e2e_wall = max_over_ranks(time.perf_counter() - t0, world)
        state_bytes = 4 * 8 * g.M // world
        e2e = {"value": updates / e2e_wall, "unit": UNIT,
               "h2d_bytes_per_step": state_bytes // K, "d2h_bytes_per_step": state_bytes // K,
               "wall_s": e2e_wall, "steps_per_call": K,
               "note": "integrate(host pinned FieldState): upload + K steps + download in one "
                       "call (pipelined: chunks stream in, passes follow as a wavefront, "
                       "finished chunks stream out); one untimed warm-up call first"}
        kgs.clear_contexts()
    else:
        dev.close()

    if rank != 0:
        return
    cb = None
    if world == 1 and not args.no_cpu:
        cb = cpu_baseline(min(K, 10), 1)
        cb = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": ms / K, "higher_is_better": True,
        # weak: per-GPU work fixed (N = 1024 * cbrt(G) for cube G, incl. G = 1)
        "scaling": "weak" if (args.scaling == "weak" and round(world ** (1 / 3)) ** 3 == world)
                   else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"3D KGS {SCENARIO} N={N}^3 fp64, tau={TAU}, checkerboard DP-AVF2",
                   "grid_points": g.M, "updates_per_step": 2 * g.M,
                   "parallelism": f"slab{world}", "l2": "inputs (32 GiB state) >> L2 (126 MB)",
                   "record_stride": K},
        "roofline": roof, "cpu_baseline": cb, "e2e": e2e, "gpu_launches": launches,
        "diagnostics": diag,
        "clocks": clk.summary(), "wall_s": wall, "energy_final": e,
        "pct_hbm_roofline": 100.0 * roof["frac"],
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--N", type=int, default=1024)
    ap.add_argument("--scaling", choices=("strong", "weak"), default="strong")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
