"""CPU, multi-process (gloo): the N>1 host logic of the slab decomposition.

The device path splits the grid into slabs along axis 0; before every colour
pass each rank receives the other colour's freshly updated face planes from
ranks rank-1 / rank+1 (periodic) -- NCCL send/recv in
paper_2502_09537_b200/csrc/kgs_host.cu:exchange(), with the send/recv order
rule that keeps 2-rank rings (where both neighbours are the same peer)
matched.  Energy terms are summed in rank order after an all-gather.

These tests run that protocol with gloo processes on the CPU: each rank
steps its slab with the numpy colour-phase restatement (oracle/), exchanges
faces with the same order rule through torch.distributed, and the result
must be bitwise equal to the single-process oracle; the cross-rank energy
terms must match the whole-grid terms.  The rank-0 ncclUniqueId broadcast
of DeviceContext (device.make_nccl_id) is exercised for real.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2502_09537_b200 import GridSpec, PhysParams, seeded_random_state
from paper_2502_09537_b200.device import (_torch_allgather, _torch_broadcast,
                                          combine_rank_terms, make_nccl_id, slab_range)

PARAMS = PhysParams(1.1, 0.9, 1.2, 0.8)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def exchange_faces(slab: dict, rank: int, world: int) -> None:
    """Fill ghost planes 0 and -1 of every field from the neighbours, with the
    order rule of kgs_host.cu:exchange(): sends [to dn: first plane, to up:
    last plane], recvs [from up: ghost after, from dn: ghost before]."""
    up, dn = (rank + 1) % world, (rank - 1) % world
    for f in "PQUV":
        a = slab[f]
        first = np.ascontiguousarray(a[1])
        last = np.ascontiguousarray(a[-2])
        import torch
        t_first, t_last = torch.from_numpy(first), torch.from_numpy(last)
        r_after, r_before = torch.empty_like(t_first), torch.empty_like(t_first)
        ops = [dist.P2POp(dist.isend, t_first, dn), dist.P2POp(dist.isend, t_last, up),
               dist.P2POp(dist.irecv, r_after, up), dist.P2POp(dist.irecv, r_before, dn)]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        a[-1] = r_after.numpy()
        a[0] = r_before.numpy()


def slab_half_sweep(slab: dict, args, grid: GridSpec, x0: int, colour: int,
                    adjoint: bool) -> None:
    """numpy_half_sweep on a slab with ghost planes (x neighbours from the
    ghosts, y and z periodic) -- the same arithmetic as oracle/."""
    alpha, beta, gcoef, c_uv, uv_nbr, gU, half_tau, i00, i01, i10, i11 = args
    nx = slab["P"].shape[0] - 2
    inner = (slice(1, nx + 1),)

    def nsum(a):
        s = np.zeros(a[1:-1].shape)
        s = s + a[:-2]                                  # -x
        s = s + a[2:]                                   # +x
        for ax in (1, 2):
            s = s + np.roll(a[1:-1], 1, axis=ax)
            s = s + np.roll(a[1:-1], -1, axis=ax)
        return s

    SP, SQ, SU = (nsum(slab[f]) for f in "PQU")
    idx = np.indices((nx, grid.N, grid.N))
    m = ((idx[0] + x0 + idx[1] + idx[2]) % 2) == colour
    P, Q, U, V = (slab[f][inner][m] for f in "PQUV")
    SP, SQ, SU = SP[m], SQ[m], SU[m]
    if not adjoint:
        cr = gcoef * U - alpha
        rr = -cr * P - Q - beta * SP
        ri = P - cr * Q - beta * SQ
        den = cr * cr + 1.0
        Pn = (rr * cr + ri) / den
        Qn = (ri * cr - rr) / den
        r1 = U + half_tau * V
        r2 = V - c_uv * U + uv_nbr * SU + gU * (Pn * Pn + Qn * Qn)
        Un, Vn = i00 * r1 + i01 * r2, i10 * r1 + i11 * r2
    else:
        r1 = U + half_tau * V
        r2 = V - c_uv * U + uv_nbr * SU + gU * (P * P + Q * Q)
        Un, Vn = i00 * r1 + i01 * r2, i10 * r1 + i11 * r2
        cr = gcoef * Un - alpha
        rr = -cr * P - Q - beta * SP
        ri = P - cr * Q - beta * SQ
        den = cr * cr + 1.0
        Pn = (rr * cr + ri) / den
        Qn = (ri * cr - rr) / den
    for f, v in zip("PQUV", (Pn, Qn, Un, Vn)):
        view = slab[f][inner]
        view[m] = v


def slab_terms(slab: dict, grid: GridSpec) -> np.ndarray:
    """This rank's 8 energy/mass term sums; forward x-edges of the last
    plane use the ghost plane after it (each edge counted exactly once)."""
    import math
    t = np.zeros(8)
    for q, f in enumerate("PQU"):
        a = slab[f]
        parts = [(a[2:] - a[1:-1]).ravel()]
        for ax in (1, 2):
            d = np.roll(a[1:-1], -1, axis=ax) - a[1:-1]
            parts.append(d.ravel())
        t[q] = math.fsum(np.concatenate(parts) ** 2)
    P, Q, U, V = (slab[f][1:-1].ravel() for f in "PQUV")
    t[3] = math.fsum(V * V)
    t[4] = math.fsum(U * U)
    t[5] = math.fsum((P * P + Q * Q) * U)
    t[6] = math.fsum(P * P)
    t[7] = math.fsum(Q * Q)
    return t


def _worker(rank: int, world: int, port: int, N: int, steps: int, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nid = make_nccl_id(rank, _torch_broadcast)       # real kgs_nccl_unique_id on rank 0
        ids = _torch_allgather(nid)
        grid = GridSpec(3, -1.0, 1.0, N)
        s = seeded_random_state(grid, 42, 0.5)
        x0, nx = slab_range(N, rank, world)
        slab = {}
        for f in "PQUV":
            a = getattr(s, f).reshape(grid.shape)
            slab[f] = np.concatenate([a[(x0 - 1) % N][None], a[x0:x0 + nx],
                                      a[(x0 + nx) % N][None]]).copy()
        args = oracle.kernel_args(PARAMS, 0.02, grid)
        for _ in range(steps):
            for colour, adj in ((1, False), (0, False), (0, True), (1, True)):
                slab_half_sweep(slab, args, grid, x0, colour, adj)
                exchange_faces(slab, rank, world)
        terms = combine_rank_terms(_torch_allgather(slab_terms(slab, grid)))
        out.put((rank, x0, {f: slab[f][1:-1].copy() for f in "PQUV"}, terms,
                 len(set(ids)), len(nid)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,N", [(2, 8), (4, 8), (2, 6)])
def test_slab_halo_protocol_bitwise(world, N):
    steps = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, N, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    grid = GridSpec(3, -1.0, 1.0, N)
    ref = seeded_random_state(grid, 42, 0.5)
    oracle.numpy_step_dpavf2(ref, oracle.kernel_args(PARAMS, 0.02, grid), grid, steps)
    full = {f: getattr(ref, f).reshape(grid.shape) for f in "PQUV"}
    for rank, x0, fields, terms, n_ids, id_len in results:
        assert n_ids == 1 and id_len == 128           # one ncclUniqueId, everywhere
        for f in "PQUV":
            assert np.array_equal(fields[f], full[f][x0:x0 + fields[f].shape[0]]), (rank, f)
        np.testing.assert_allclose(terms, oracle.energy_terms(ref, grid), rtol=1e-13)
