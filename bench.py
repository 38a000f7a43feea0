"""Benchmark: 3-D KGS checkerboard DP-AVF2 point-updates/s on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--N 1024] [--scaling strong|weak]

Workload (BASELINE.json configs[3], the metric's named config): 3-D
ellipsoids3d on a 1024^3 fp64 periodic grid, tau = 0.01.  A "step" is one
DP-AVF2 time step = 2 * N^3 point-updates.  Inputs are the
reference's own preset (scenarios.py:69-89) built on the host block-parallel
(bitwise the reference's numpy build) and uploaded; the 32 GiB state is far
larger than the 126 MB L2, so no flush is needed.
tests/test_gpu_headline.py checks this exact workload and call pattern bit
for bit against the table-free C restatement of the reference.

ours:       value = all GPUs' point-updates / max-over-ranks device time of K
            fused steps (CUDA events on the library's streams); e2e = the
            same metric through the public API integrate() on the page-locked
            host FieldState (upload, K steps, download inside the timed
            region); cpu_baseline = the reference itself (dpavf from
            baseline/_ref, numba, all host cores) on a 256^3 sample, the C
            port beside it.
reference:  the unmodified reference (baseline/_ref: dpavf.step_dpavf2,
            checkerboard_schedule, PhasedExecutor over all host cores, as its
            run_bench) on a bounded 512^3 sample; rank 0 only.
GPUs:       --gpus N without a launcher drives GPUs 0..N-1 from one process
            (one slab per GPU, halos stored into the neighbours' ghost
            planes over NVLink); under torchrun one rank per GPU with NCCL
            halos.  Strong scaling at 1024^3 by default; --scaling weak keeps
            ~1024^3 points per GPU (2048^3 on 8 GPUs).
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


class Launch:
    """Who this process is and which GPUs it drives.

    torchrun (WORLD_SIZE > 1): one rank per GPU, slab ``rank`` on
    ``cuda:LOCAL_RANK``, NCCL halos (DistributedExecutor).  Plain
    ``python bench.py --gpus N`` (no launcher): ONE process drives GPUs
    0..N-1, one slab each, halos stored straight into the neighbours' ghost
    planes over NVLink (CudaExecutor).  Either way fewer
    visible devices than requested is an error, never a silent fallback."""

    def __init__(self, gpus: int):
        import torch
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        ndev = torch.cuda.device_count()
        # torchrun with ONE rank and KGS_SELF_EXCHANGE=1: the rank exchanges
        # its faces with itself over NCCL -- the multi-rank path on one GPU
        self.selfx = (self.world == 1 and "WORLD_SIZE" in os.environ
                      and os.environ.get("KGS_SELF_EXCHANGE") == "1")
        self.dist = self.world > 1 or self.selfx
        if self.dist:
            if self.local >= ndev:
                raise SystemExit(f"bench.py: rank {self.rank} needs cuda:{self.local}, "
                                 f"only {ndev} devices visible")
            os.environ.setdefault("NCCL_DEBUG", "WARN")
            import torch.distributed as dist
            torch.cuda.set_device(self.local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.devices = (self.local,)
            self.n_gpus = self.world
            self.mode = "torchrun+nccl" + (" (1 rank, faces sent to itself)" if self.selfx else "")
        else:
            if gpus > ndev:
                raise SystemExit(f"bench.py --gpus {gpus}: only {ndev} CUDA devices visible")
            self.devices = tuple(range(max(gpus, 1)))
            self.n_gpus = len(self.devices)
            self.mode = "single-process" + ("+peer-stores" if self.n_gpus > 1 else "")
        self.host_ranks = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))

    def executor(self):
        import paper_2502_09537_b200 as kgs
        if self.dist:
            return kgs.DistributedExecutor(self.rank, self.world, self.local)
        return kgs.CudaExecutor(self.devices)

    def describe(self) -> list:
        """The GPUs actually used (all ranks), for the JSON line."""
        import torch
        mine = []
        for d in self.devices:
            pr = torch.cuda.get_device_properties(d)
            mine.append({"rank": self.rank, "device": d, "name": pr.name,
                         "pci_bus_id": getattr(pr, "pci_bus_id", None),
                         "uuid": str(getattr(pr, "uuid", ""))})
        if self.world > 1:
            import torch.distributed as dist
            out = [None] * self.world
            dist.all_gather_object(out, mine)
            mine = [x for r in out for x in r]
        return mine


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


def all_ranks(flag: bool, world: int) -> bool:
    """A decision every rank takes together (what follows is collective):
    true only if it holds on every rank -- e.g. host memory, which the
    ranks of one node check while the others are allocating."""
    if world == 1:
        return flag
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([1 if flag else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(t.item())


def weak_n(base: int, gpus: int) -> int:
    """Grid edge with ~base^3 points per GPU: base * cbrt(G) rounded to a
    multiple of 128 (the march kernel's tile) that G divides -- exact for
    cube G (8 GPUs: 2048^3, BASELINE configs[4])."""
    target = base * gpus ** (1.0 / 3.0)
    n = max(128, int(round(target / 128.0)) * 128)
    while n % gpus:
        n += 128
    return n


def grid_n(args, gpus: int) -> int:
    return weak_n(args.N, gpus) if args.scaling == "weak" else args.N


# --------------------------------------------------------------------------
REF_SITE = ROOT / "baseline" / "_ref"


def reference_cpu(steps: int, warmup: int, N: int) -> dict:
    """The reference's own CPU path, unmodified: ``dpavf`` installed into
    baseline/_ref, ``step_dpavf2`` with the checkerboard
    schedule and a ``PhasedExecutor`` over all host cores, timed exactly as
    its ``run_bench`` does (dpavf/harness.py:183-224: state, schedule and
    JIT warm-up untimed), on the bench's scenario at N^3."""
    if not (REF_SITE / "dpavf").is_dir():
        raise FileNotFoundError(f"reference not installed in {REF_SITE}")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/kgs_numba_cache")
    if str(REF_SITE) not in sys.path:
        sys.path.insert(0, str(REF_SITE))
    import dpavf
    from dpavf.harness import make_schedule
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    sc = dpavf.get_scenario(SCENARIO)
    g = sc.default_grid(N)
    st = sc.state(g)
    sched = make_schedule("checkerboard", g, workers=threads)
    coeffs = dpavf.precompute_coefficients(sc.params, TAU / 2.0, g)
    ex = dpavf.PhasedExecutor(threads) if threads > 1 else dpavf.SerialExecutor()
    setup = time.perf_counter() - t0
    try:
        for _ in range(max(warmup, 1)):
            dpavf.step_dpavf2(st, sched, coeffs, ex, g)
        t0 = time.perf_counter()
        for _ in range(steps):
            dpavf.step_dpavf2(st, sched, coeffs, ex, g)
        dt = time.perf_counter() - t0
    finally:
        ex.close()
    return {"value": 2.0 * g.M * steps / dt, "unit": UNIT, "cores": threads,
            "kind": "reference",
            "sample": f"{N}^3 {SCENARIO}, {steps} DP-AVF2 steps after {max(warmup, 1)} warm-up "
                      f"(incl. numba JIT), dpavf.step_dpavf2 + checkerboard_schedule + "
                      f"PhasedExecutor({threads}) from baseline/_ref (unmodified reference)",
            "seconds": dt, "setup_s": setup, "N": N,
            "numba": __import__("numba").__version__}


def port_cpu(steps: int, warmup: int, N: int = 256) -> dict:
    """The C restatement of the same algorithm (oracle/, "port"), all host
    threads -- reported beside the reference as a cross-check."""
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


def cpu_baseline(steps: int = 3, warmup: int = 1, N: int = 256) -> dict:
    """cpu_baseline for our arm's line: the reference itself on a bounded
    sample (port as a secondary field; the port alone if the reference
    cannot run here)."""
    port = port_cpu(steps, warmup, N)
    keys = ("value", "unit", "cores", "kind", "sample")
    try:
        ref = reference_cpu(steps, warmup, N)
    except Exception as e:  # noqa: BLE001 - reported, not hidden
        out = {k: port[k] for k in keys}
        out["reference_error"] = f"{type(e).__name__}: {e}"
        return out
    out = {k: ref[k] for k in keys}
    out["port"] = {k: port[k] for k in keys}
    return out


def run_reference(args):
    """--impl reference: the reference's CPU path on the host cores (rank 0
    only under torchrun; other ranks exit without work)."""
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    n_gpus = world if world > 1 else max(args.gpus, 1)
    N = grid_n(args, n_gpus)
    # bounded sample of the workload: 512^3 (1/8 of the 1024^3 grid; time is
    # linear in N^d), capped so the run ends in minutes
    ns = min(N, args.ref_N)
    steps = max(1, min(args.steps, 20))
    warm = max(1, min(args.warmup, 2))
    cb = reference_cpu(steps, warm, ns)
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT,
        "n_gpus": n_gpus, "steps": steps, "warmup": warm,
        "ms_per_step": 1e3 * cb["seconds"] / steps,
        "higher_is_better": True,
        "scaling": "weak" if args.scaling == "weak" else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"3D KGS {SCENARIO} N={N}^3 fp64, tau={TAU}, checkerboard DP-AVF2",
                   "sample": cb["sample"], "sample_N": ns},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "setup_s": cb["setup_s"], "numba": cb["numba"],
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
def host_preset(g, L: "Launch", pinned: bool):
    """The reference's ellipsoids3d preset (scenarios.py:69-89) on this
    process's planes, built block-parallel on the host (bitwise the
    reference's numpy build), in page-locked memory when ``pinned``."""
    import paper_2502_09537_b200 as kgs
    from paper_2502_09537_b200.device import pinned_empty, slab_range
    from paper_2502_09537_b200.scenarios import build_preset
    if L.world > 1:
        x0, nx = slab_range(g.N, L.rank, L.world)
        planes, n = (x0, x0 + nx), nx * g.N * g.N
    else:
        planes, n = None, g.M
    alloc = pinned_empty if pinned else np.empty
    out = kgs.FieldState(*(alloc(n) for _ in range(4)), 0.0)
    # the local ranks of one host share its cores
    workers = max(1, (os.cpu_count() or 1) // max(L.host_ranks, 1))
    return build_preset(SCENARIO, g, out=out, planes=planes, workers=workers)


def host_memory_ok(nbytes: int, L: "Launch") -> bool:
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        return True
    return nbytes * max(L.host_ranks, 1) * 1.15 < avail


def run_ours(args):
    import torch
    import paper_2502_09537_b200 as kgs

    L = Launch(args.gpus)
    world = L.world
    N = grid_n(args, L.n_gpus)
    sc = kgs.get_scenario(SCENARIO)
    g = sc.default_grid(N)
    ex = L.executor()
    sch = kgs.checkerboard_schedule(g)
    coeffs = kgs.precompute_coefficients(sc.params, TAU / 2.0, g)
    kargs = coeffs.kernel_args()
    K, W = args.steps, args.warmup

    # inputs: the reference's host preset, uploaded (bitwise scenarios.py);
    # kept on the host (page-locked) as the e2e input
    local_bytes = 32 * g.M // max(world, 1)
    t_in = time.perf_counter()
    host = None
    if all_ranks(host_memory_ok(local_bytes, L), world):
        host = host_preset(g, L, pinned=not args.no_e2e)
        dev = kgs.DeviceFieldState.from_host(host, g, ex)
        inputs = "host preset (block-parallel numpy, bitwise reference scenarios.py:69-89)"
    else:   # too little host memory for a host copy: same formulas on the device
        dev = kgs.DeviceFieldState.from_preset(SCENARIO, g, ex)
        inputs = "device preset (kgs_fill_preset; host memory too small for a host copy)"
    t_in = time.perf_counter() - t_in
    ctx = dev.ctx
    # warm-up (untimed)
    ctx.step_dpavf2(kargs, W, 0, 0)
    barrier(world)
    torch.cuda.synchronize()
    l0 = ctx.launch_count()
    ctx.pass_timing(True)
    with ClockSampler(L.devices[0]) as clk:
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
    if nc and nc.get("N") == N and nc.get("world") == L.n_gpus:
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
    # Interleaved blocks of B steps, recording every step or not at all, so
    # clock / power drift over the run hits both alike; cost = ratio of the
    # median block times (same step count, same head/tail share).
    B, pairs = 10, 4
    off = W + K
    rec_ms, plain_ms, recs = [], [], [terms[-1]]
    for _ in range(pairs):
        for rec in (True, False):
            barrier(world)
            t_b, bad_b = ctx.step_dpavf2(kargs, B, off, 1 if rec else 0)
            off += B
            if bad_b:
                raise FloatingPointError(f"non-finite state at step {bad_b}")
            (rec_ms if rec else plain_ms).append(max_over_ranks(ctx.last_step_ms(), world) / B)
            if rec:
                recs.extend(t_b)
    em = [kgs.grid.energy_from_terms(t, sc.params, g) for t in recs]
    ms_rec, ms_plain = float(np.median(rec_ms)), float(np.median(plain_ms))
    diag = {"record_stride": 1, "steps": B * pairs, "ms_per_step": ms_rec,
            "value": 2.0 * g.M / (ms_rec / 1e3), "unit": UNIT,
            "ms_per_step_unrecorded": ms_plain,
            "cost_vs_unrecorded": ms_rec / ms_plain,
            "blocks": f"{pairs} interleaved pairs of {B}-step calls (recorded / unrecorded)",
            "max_rel_energy_change": max(abs(E - em[0][0]) / abs(em[0][0]) for E, _ in em),
            "max_rel_mass_change": max(abs(m - em[0][1]) / abs(em[0][1]) for _, m in em),
            "note": "energy is the scheme's invariant (round-off drift); mass is not conserved "
                    "by DP-AVF2 and drifts at the reference's own rate (grows with N)"}
    dev.close()
    del dev

    # e2e through the public API: integrate() on the host state
    e2e = None
    if not args.no_e2e and host is not None:
        # untimed warm-up call (W steps): creates the cached context and its
        # pipeline buffers, as the device timing's warm-up steps do
        kgs.integrate(host, g, sc.params, sch, ex, TAU, W * TAU, record_stride=W)
        barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        kgs.integrate(host, g, sc.params, sch, ex, TAU, K * TAU, record_stride=K)
        torch.cuda.synchronize()
        e2e_wall = max_over_ranks(time.perf_counter() - t0, world)
        e2e = {"value": updates / e2e_wall, "unit": UNIT,
               "h2d_bytes_per_step": local_bytes * world // K,
               "d2h_bytes_per_step": local_bytes * world // K,
               "wall_s": e2e_wall, "steps_per_call": K,
               "note": "integrate(host page-locked FieldState): upload + K steps + download in "
                       "one call (pipelined on one slab: chunks stream in, passes follow as a "
                       "wavefront, finished chunks stream out); one untimed warm-up call first"}
        # the same call on ordinary (pageable) numpy arrays -- what a dpavf
        # user passes (grid.py:82-103): page-locked just in time inside the call
        if all_ranks(host_memory_ok(2 * local_bytes, L), world):
            plain = kgs.FieldState(*(np.array(getattr(host, f)) for f in "PQUV"), host.t)
            # untimed warm-up call: allocates the page-locked staging slots
            kgs.integrate(plain, g, sc.params, sch, ex, TAU, W * TAU, record_stride=W)
            barrier(world)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            kgs.integrate(plain, g, sc.params, sch, ex, TAU, K * TAU, record_stride=K)
            torch.cuda.synchronize()
            pw = max_over_ranks(time.perf_counter() - t0, world)
            e2e["pageable"] = {"value": updates / pw, "unit": UNIT, "wall_s": pw,
                               "vs_pinned": e2e_wall / pw,
                               "note": "integrate() on pageable numpy arrays (the reference's "
                                       "FieldState), staged through page-locked slots by host "
                                       "threads inside the call; one untimed warm-up call first"}
            del plain
        kgs.clear_contexts()
    gpus_used = L.describe()
    barrier(world)

    if L.rank != 0:
        return
    cb = None
    if not args.no_cpu:
        # after every GPU timing (rank 0 alone; no other rank is still working)
        cb = cpu_baseline(3, 1, 256)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": L.n_gpus, "steps": K,
        "warmup": W, "ms_per_step": ms / K, "higher_is_better": True,
        "scaling": "weak" if args.scaling == "weak" else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"3D KGS {SCENARIO} N={N}^3 fp64, tau={TAU}, checkerboard DP-AVF2",
                   "grid_points": g.M, "updates_per_step": 2 * g.M,
                   "points_per_gpu": g.M // L.n_gpus,
                   "parallelism": f"slab{L.n_gpus} ({L.mode})",
                   "l2": "inputs (32 GiB state) >> L2 (126 MB)",
                   "record_stride": K, "inputs": inputs, "input_build_s": t_in},
        "gpus": gpus_used,
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
    ap.add_argument("--ref-N", type=int, default=512,
                    help="--impl reference: grid edge of the bounded CPU sample")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
