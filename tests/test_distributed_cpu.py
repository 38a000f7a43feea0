"""CPU, multi-process (gloo): the N>1 schedule of the C++ library replayed.

A multi-GPU run (torchrun, one rank per GPU) splits the grid into slabs along
axis 0.  What every rank does, in order, is the pass program of
kgs_step_dpavf2 (csrc/kgs_program.cuh): colour-pass launches over plane
ranges (interior first, boundary planes after the halo wait), halo
exchanges of one colour's faces (P, Q, U of planes 0 and nx-1 into the
neighbours' ghost planes -- NCCL send/recv on the device), waits for them,
energy records and the deferred tail.  The library exports that exact list
(``kgs_step_program``, the same function the device executor runs), so
these tests fetch it from the C library and EXECUTE it in gloo worlds of 2
and 4 ranks: launches with the numpy restatement of the per-point
arithmetic (oracle/), exchanges with real send/recv of only that colour's
face values (the other colour's ghosts stay stale, V ghosts are NaN), energy
partials reduced at the records and summed in rank order.

Two timings of every exchange are replayed -- data taken and delivered when
the exchange starts ("eager") and when the program first waits for it
("lazy") -- so a launch placed between an exchange and its wait that read
the ghosts or wrote the faces would change the result.  Both must equal the
single-process oracle bit for bit (fields) and to summation order (records).
A mutated program (one wait removed) must fail, which shows the replay is
sensitive to the schedule.  The rank-0 ncclUniqueId broadcast of
DeviceContext (device.make_nccl_id) is exercised for real.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2502_09537_b200 import GridSpec, PhysParams, _lib, seeded_random_state
from paper_2502_09537_b200.device import (_torch_allgather, _torch_broadcast,
                                          combine_rank_terms, make_nccl_id, slab_range)

PARAMS = PhysParams(1.1, 0.9, 1.2, 0.8)
OP_NONE, OP_BASE, OP_ADJ = 0, 1, 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


# ---- the per-point arithmetic (oracle.numpy_half_sweep, kernels.py:43-94) ----
def _apply(op, P, Q, U, V, SP, SQ, SU, a):
    alpha, beta, gcoef, c_uv, uv_nbr, gU, half_tau, i00, i01, i10, i11 = a

    def psi(P, Q, Uc):
        cr = gcoef * Uc - alpha
        rr = -cr * P - Q - beta * SP
        ri = P - cr * Q - beta * SQ
        den = cr * cr + 1.0
        return (rr * cr + ri) / den, (ri * cr - rr) / den

    def uv(U, V, Pm, Qm):
        r1 = U + half_tau * V
        r2 = V - c_uv * U + uv_nbr * SU + gU * (Pm * Pm + Qm * Qm)
        return i00 * r1 + i01 * r2, i10 * r1 + i11 * r2

    if op == OP_BASE:
        P, Q = psi(P, Q, U)
        U, V = uv(U, V, P, Q)
    elif op == OP_ADJ:
        U, V = uv(U, V, P, Q)
        P, Q = psi(P, Q, U)
    return P, Q, U, V


class SlabReplay:
    """One rank's slab (natural layout, ghost planes at index 0 and nx+1)
    executing kgs_step_program rows."""

    def __init__(self, grid, state, rank, world, args, lazy):
        self.g, self.rank, self.world, self.args, self.lazy = grid, rank, world, args, lazy
        N = grid.N
        self.x0, self.nx = slab_range(N, rank, world)
        self.f = {}
        for name in "PQUV":
            a = getattr(state, name).reshape(grid.shape)
            s = np.full((self.nx + 2, N, N), np.nan)
            s[1:-1] = a[self.x0:self.x0 + self.nx]
            self.f[name] = s
        idx = np.indices((self.nx + 2, N, N))
        self.parity = (idx[0] - 1 + self.x0 + idx[1] + idx[2]) % 2   # global parity per slot
        self.pending = []          # exchanges started, not yet delivered (lazy)
        self.acc = {0: np.zeros(8), 1: np.zeros(8)}
        self.records = []
        self.deferred = False
        # ghosts as after an upload: both colours exchanged (V never: NaN)
        for col in (0, 1):
            self._exchange(col)

    # -- exchange: only colour `col` values of P, Q, U travel ------------------
    def _exchange(self, col):
        up, dn = (self.rank + 1) % self.world, (self.rank - 1) % self.world
        first = torch.from_numpy(np.stack([self.f[n][1] for n in "PQU"]).copy())
        last = torch.from_numpy(np.stack([self.f[n][self.nx] for n in "PQU"]).copy())
        from_up, from_dn = torch.empty_like(first), torch.empty_like(first)
        ops = [dist.P2POp(dist.isend, first, dn, tag=1), dist.P2POp(dist.isend, last, up, tag=2),
               dist.P2POp(dist.irecv, from_up, up, tag=1),
               dist.P2POp(dist.irecv, from_dn, dn, tag=2)]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        for gi, data in ((self.nx + 1, from_up.numpy()), (0, from_dn.numpy())):
            m = self.parity[gi] == col
            for k, n in enumerate("PQU"):
                self.f[n][gi][m] = data[k][m]

    # -- one launch: colour `col` over local planes [xa, xb) -------------------
    def _launch(self, col, op1, op2, diag, xa, xb):
        a, N = self.args, self.g.N
        sl = slice(xa + 1, xb + 1)

        def nsum(arr):     # canonical order -x, +x, -y, +y, -z, +z, seeded 0.0
            s = np.zeros((xb - xa, N, N))
            s = s + arr[xa:xb]
            s = s + arr[xa + 2:xb + 2]
            for ax in (1, 2):
                s = s + np.roll(arr[sl], 1, axis=ax)
                s = s + np.roll(arr[sl], -1, axis=ax)
            return s

        m = self.parity[sl] == col
        SP, SQ, SU = (nsum(self.f[n])[m] for n in "PQU")
        P, Q, U, V = (self.f[n][sl][m] for n in "PQUV")
        after = 1 if op1 == OP_ADJ else (2 if op2 == OP_ADJ else 0)
        P, Q, U, V = _apply(op1, P, Q, U, V, SP, SQ, SU, a)
        if diag and after == 1:
            self._measure(col, sl, m, P, Q, U, V)
        P, Q, U, V = _apply(op2, P, Q, U, V, SP, SQ, SU, a)
        if diag and after == 2:
            self._measure(col, sl, m, P, Q, U, V)
        for n, v in zip("PQUV", (P, Q, U, V)):
            view = self.f[n][sl]
            view[m] = v

    def _measure(self, col, sl, m, P, Q, U, V):
        """The fused record terms (DIAG): self terms of the colour's points;
        red points also add their 2d incident edges (each edge joins one red
        and one black point, so every edge is counted once)."""
        t = self.acc[col]
        pq = P * P + Q * Q
        t[3] += np.sum(V * V)
        t[4] += np.sum(U * U)
        t[5] += np.sum(pq * U)
        t[6] += np.sum(P * P)
        t[7] += np.sum(Q * Q)
        if col == 1:
            lo, hi = sl.start, sl.stop
            for q, (n, own) in enumerate(zip("PQU", (P, Q, U))):
                arr = self.f[n]
                nbs = [arr[lo - 1:hi - 1], arr[lo + 1:hi + 1]]
                for ax in (1, 2):
                    nbs += [np.roll(arr[sl], 1, axis=ax), np.roll(arr[sl], -1, axis=ax)]
                for nb in nbs:
                    t[q] += np.sum((nb[m] - own) ** 2)

    def run(self, program):
        for kind, col, op1, op2, diag, check, step, xa, xb in program.tolist():
            if kind == _lib.PG_PASS_BEGIN:
                if diag:
                    self.acc[col] = np.zeros(8)
            elif kind == _lib.PG_LAUNCH:
                self._launch(col, op1, op2, diag, xa, xb)
            elif kind == _lib.PG_XCH:
                if self.lazy:
                    self.pending.append(col)
                else:
                    self._exchange(col)
            elif kind == _lib.PG_WAIT_XCH:
                for c in self.pending:
                    self._exchange(c)
                self.pending = []
            elif kind == _lib.PG_RECORD:
                assert step == len(self.records)
                self.records.append(self.acc[1] + (self.acc[0] if xa else 0.0))
            elif kind == _lib.PG_DEFER:
                self.deferred = True
            elif kind == _lib.PG_PASS_END:
                pass
            else:
                raise AssertionError(f"unknown program row kind {kind}")
        assert not self.pending, "program ended with an exchange nobody waited for"


def _worker(rank, world, port, N, calls, lazy, mutate, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nid = make_nccl_id(rank, _torch_broadcast)       # real kgs_nccl_unique_id on rank 0
        ids = _torch_allgather(nid)
        grid = GridSpec(3, -1.0, 1.0, N)
        s = seeded_random_state(grid, 42, 0.5)
        args = oracle.kernel_args(PARAMS, 0.02, grid)
        rep = SlabReplay(grid, s, rank, world, args, lazy)
        offset, head_fused = 0, False
        for nsteps, stride, defer in calls:
            prog = _lib.step_program(rep.nx, True, nsteps, offset, stride, defer_tail=defer,
                                     head_fused=head_fused)
            if mutate:   # drop the first wait of every pass
                keep, seen = [], False
                for row in prog:
                    if row[0] == _lib.PG_PASS_BEGIN:
                        seen = False
                    if row[0] == _lib.PG_WAIT_XCH and not seen:
                        seen = True
                        continue
                    keep.append(row)
                prog = np.array(keep)
            rep.records = []
            rep.run(prog)
            head_fused, rep.deferred = rep.deferred, False
            offset += nsteps
        recs = [combine_rank_terms(_torch_allgather(r)) for r in rep.records]
        out.put((rank, rep.x0, {n: rep.f[n][1:-1].copy() for n in "PQUV"}, recs,
                 len(set(ids)), len(nid)))
    finally:
        dist.destroy_process_group()


def _run_world(world, N, calls, lazy, mutate=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, N, calls, lazy, mutate, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(results, key=lambda r: r[0])


def _reference(N, total_steps, record_steps):
    grid = GridSpec(3, -1.0, 1.0, N)
    ref = seeded_random_state(grid, 42, 0.5)
    args = oracle.kernel_args(PARAMS, 0.02, grid)
    terms = {}
    for n in range(1, total_steps + 1):
        oracle.numpy_step_dpavf2(ref, args, grid, 1)
        if n in record_steps:
            terms[n] = oracle.energy_terms(ref, grid)
    return grid, ref, terms


# (nsteps, record_stride, defer_tail) per call; a deferred tail is fused
# into the next call's head (KGS_PROGRAM_HEAD_FUSED), as on the device
CASES = [
    (2, 8, [(3, 1, False)]),                            # nx = 4, a record every step
    (4, 8, [(2, 2, True), (2, 2, False)]),              # nx = 2: no interior launch
    (2, 6, [(1, 0, True), (3, 3, True), (1, 1, False)]),
    (4, 12, [(3, 3, False)]),
]


@pytest.mark.parametrize("lazy", [False, True], ids=["eager", "lazy"])
@pytest.mark.parametrize("world,N,calls", CASES)
def test_step_program_replayed_over_gloo_is_bitwise(world, N, calls, lazy):
    results = _run_world(world, N, calls, lazy)
    total = sum(n for n, _, _ in calls)
    # record steps of each call (the deferred tail of a call records nothing:
    # a deferring call never ends on a record step, see kgs_step_program)
    rec_steps, off = [], 0
    for n, stride, _ in calls:
        rec_steps += [off + i for i in range(1, n + 1) if stride and (off + i) % stride == 0]
        off += n
    grid, ref, terms = _reference(N, total, set(rec_steps))
    full = {f: getattr(ref, f).reshape(grid.shape) for f in "PQUV"}
    last_recs = None
    for rank, x0, fields, recs, n_ids, id_len in results:
        assert n_ids == 1 and id_len == 128           # one ncclUniqueId, everywhere
        for f in "PQUV":
            assert np.array_equal(fields[f], full[f][x0:x0 + fields[f].shape[0]]), (rank, f)
        last_recs = recs
    # the records of the LAST call, summed over ranks in rank order
    last_n, last_stride, _ = calls[-1]
    off = total - last_n
    want = [terms[off + i] for i in range(1, last_n + 1)
            if last_stride and (off + i) % last_stride == 0]
    assert len(last_recs) == len(want)
    for got, w in zip(last_recs, want):
        np.testing.assert_allclose(got, w, rtol=1e-12, atol=1e-300)


def test_replay_detects_a_missing_wait():
    """Sanity of the replay itself: without the wait before the boundary
    planes, a lazily delivered exchange arrives too late and the fields are
    no longer the oracle's."""
    world, N, calls = 2, 8, [(2, 0, False)]
    results = _run_world(world, N, calls, lazy=True, mutate=True)
    grid, ref, _ = _reference(N, 2, set())
    full = {f: getattr(ref, f).reshape(grid.shape) for f in "PQUV"}
    same = all(np.array_equal(fields[f], full[f][x0:x0 + fields[f].shape[0]])
               for _, x0, fields, _, _, _ in results for f in "PQUV")
    assert not same


def test_step_program_structure():
    """The exported program's invariants (no ranks needed): every pass is
    bracketed, boundary planes follow the wait, each colour pass is followed
    by the exchange of its colour, records carry consecutive slots."""
    prog = _lib.step_program(6, True, 4, 0, 2)
    kinds = prog[:, 0].tolist()
    assert kinds.count(_lib.PG_PASS_BEGIN) == kinds.count(_lib.PG_PASS_END) == 1 + 2 * 4
    rec = prog[prog[:, 0] == _lib.PG_RECORD]
    assert rec[:, 6].tolist() == [0, 1]
    i = 0
    while i < len(prog):
        if prog[i, 0] == _lib.PG_PASS_BEGIN:
            body = prog[i + 1:i + 5]
            assert body[:, 0].tolist() == [_lib.PG_LAUNCH, _lib.PG_WAIT_XCH, _lib.PG_LAUNCH,
                                           _lib.PG_LAUNCH]
            assert body[0, 7:].tolist() == [1, 5] and body[2, 7:].tolist() == [0, 1]
            assert body[3, 7:].tolist() == [5, 6]
            assert prog[i + 5, 0] == _lib.PG_PASS_END
            assert prog[i + 6, 0] == _lib.PG_XCH and prog[i + 6, 1] == prog[i, 1]
            i += 7
        else:
            i += 1
    # one slab: a single whole-slab launch per pass, no waits inside passes
    one = _lib.step_program(6, False, 2, 0, 0)
    launches = one[one[:, 0] == _lib.PG_LAUNCH]
    assert (launches[:, 7] == 0).all() and (launches[:, 8] == 6).all()
    # a deferred tail leaves the red adjoint out; the next call fuses it
    d = _lib.step_program(6, False, 2, 0, 0, defer_tail=True)
    assert d[-2, 0] == _lib.PG_DEFER
    h = _lib.step_program(6, False, 1, 2, 0, head_fused=True)
    assert h[1, 1:4].tolist() == [1, OP_ADJ, OP_BASE]


# ---- the pipelined integrate (kgs_integrate_host) on several ranks --------
# Every rank runs the split pipeline plan (kgs_pipeline_plan(..., split=1),
# the list the device executor issues): chunks arrive in folded order, passes
# cover plane ranges as a wavefront, faces are exchanged after each writing
# pass has covered both boundary planes, a launch touching a boundary plane
# first takes delivery of pending exchanges (the device: the compute stream
# waits for the exchange event), and FINAL blocks are copied out at once --
# they must already hold the end state.

PIPE_ARRIVE, PIPE_PASS, PIPE_FINAL, PIPE_XCH = 0, 1, 2, 3


def pipeline_events(nx, C, nsteps):
    import ctypes
    lib = _lib.load()
    n = lib.kgs_pipeline_plan(nx, C, nsteps, 1, None, 0)
    buf = (ctypes.c_int64 * (4 * n))()
    assert lib.kgs_pipeline_plan(nx, C, nsteps, 1, buf, n) == n
    return [tuple(buf[4 * i:4 * i + 4]) for i in range(n)]


def pipeline_passes(nsteps):
    """(colour, op1, op2) of every pass, as integrate_pipelined builds them."""
    p = [(0, OP_NONE, OP_NONE), (1, OP_NONE, OP_NONE), (1, OP_BASE, OP_NONE)]
    for i in range(1, nsteps + 1):
        p += [(0, OP_BASE, OP_ADJ), (1, OP_ADJ, OP_BASE if i < nsteps else OP_NONE)]
    return p


class PipeReplay(SlabReplay):
    """One rank executing the split pipeline plan: nothing has arrived at
    the start (local planes and ghosts NaN)."""

    def __init__(self, grid, state, rank, world, args, lazy):
        super().__init__(grid, state, rank, world, args, lazy)
        self.host = {n: self.f[n][1:-1].copy() for n in "PQUV"}
        for n in "PQUV":
            self.f[n][:] = np.nan
        self.finals = {}

    def run_plan(self, events, passes):
        for kind, idx, a, b in events:
            if kind == PIPE_ARRIVE:
                for n in "PQUV":
                    self.f[n][a + 1:b + 1] = self.host[n][a:b]
            elif kind == PIPE_XCH:
                cols = (0, 1) if idx < 0 else (passes[idx][0],)
                for c in cols:
                    if self.lazy:
                        self.pending.append(c)
                    else:
                        self._exchange(c)
            elif kind == PIPE_PASS:
                if self.pending and (a == 0 or b == self.nx):
                    for c in self.pending:
                        self._exchange(c)
                    self.pending = []
                col, op1, op2 = passes[idx]
                self._launch(col, op1, op2, False, a, b)
            elif kind == PIPE_FINAL:
                self.finals[(a, b)] = {n: self.f[n][a + 1:b + 1].copy() for n in "PQUV"}
            else:
                raise AssertionError(f"unknown pipeline event {kind}")
        for c in self.pending:   # the last exchanges (ghosts for later calls)
            self._exchange(c)
        self.pending = []


def _pipe_worker(rank, world, port, N, C, nsteps, lazy, out, drop_xch=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        grid = GridSpec(3, -1.0, 1.0, N)
        s = seeded_random_state(grid, 42, 0.5)
        args = oracle.kernel_args(PARAMS, 0.02, grid)
        rep = PipeReplay(grid, s, rank, world, args, lazy)
        events = pipeline_events(rep.nx, C, nsteps)
        if drop_xch:   # mutation: the faces of the first K3 never travel
            events = [e for e in events if not (e[0] == PIPE_XCH and e[1] == 3)]
        rep.run_plan(events, pipeline_passes(nsteps))
        out.put((rank, rep.x0, {n: rep.f[n][1:-1].copy() for n in "PQUV"}, rep.finals))
    finally:
        dist.destroy_process_group()


def _run_pipe_world(world, N, C, nsteps, lazy, drop_xch=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pipe_worker,
                         args=(r, world, port, N, C, nsteps, lazy, q, drop_xch))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return results


@pytest.mark.parametrize("lazy", [False, True], ids=["eager", "lazy"])
@pytest.mark.parametrize("world,N,C,nsteps", [
    (2, 16, 2, 2), (2, 16, 3, 3), (4, 16, 1, 2), (2, 12, 1, 1), (4, 24, 2, 3)])
def test_pipeline_plan_replayed_over_gloo_is_bitwise(world, N, C, nsteps, lazy):
    results = _run_pipe_world(world, N, C, nsteps, lazy)
    grid, ref, _ = _reference(N, nsteps, set())
    full = {f: getattr(ref, f).reshape(grid.shape) for f in "PQUV"}
    for rank, x0, fields, finals in results:
        nx = fields["P"].shape[0]
        assert sorted(finals) == [(a, min(a + C, nx)) for a in range(0, nx, C)]
        for f in "PQUV":
            assert np.array_equal(fields[f], full[f][x0:x0 + nx]), (rank, f)
            for (a, b), blk in finals.items():   # copied back = the end state
                assert np.array_equal(blk[f], full[f][x0 + a:x0 + b]), (rank, f, a)


def test_pipeline_replay_detects_a_missing_exchange():
    """Sanity of the replay: without one pass's face exchange the ghosts
    hold stale faces and the fields are no longer the oracle's."""
    results = _run_pipe_world(2, 16, 2, 2, lazy=False, drop_xch=True)
    grid, ref, _ = _reference(16, 2, set())
    full = {f: getattr(ref, f).reshape(grid.shape) for f in "PQUV"}
    same = all(np.array_equal(fields[f], full[f][x0:x0 + fields[f].shape[0]])
               for _, x0, fields, _ in results for f in "PQUV")
    assert not same
