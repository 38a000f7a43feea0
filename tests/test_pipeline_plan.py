"""The schedule of the pipelined host integration (kgs_pipeline_plan -- the
exact event list kgs_integrate_host executes) checked on the CPU against the
true data dependencies of every pass, for many grid / chunk / step counts:
chunks of planes arrive around plane 0; each pass may only touch a plane
once what it reads is written (RAW) and what it overwrites has been read by
every earlier reader (WAR); every plane is covered once per pass; a block is
copied back exactly once, only when every pass is done on it.  With
split = 1 (several slabs / ranks, each running the plan on its own planes)
the plan also carries face exchanges, and reads of the ghost planes -1 and
N must see the exchanged faces of exactly the pass that wrote them last."""
from __future__ import annotations

import ctypes

import pytest

from paper_2502_09537_b200 import _lib

ARRIVE, PASS, FINAL, XCH = 0, 1, 2, 3


def plan(N, C, nsteps, split=0):
    lib = _lib.load()
    n = lib.kgs_pipeline_plan(N, C, nsteps, split, None, 0)
    assert n > 0
    buf = (ctypes.c_int64 * (4 * n))()
    assert lib.kgs_pipeline_plan(N, C, nsteps, split, buf, n) == n
    return [tuple(buf[4 * i: 4 * i + 4]) for i in range(n)]


def check(N, C, nsteps):
    J = 3 + 2 * nsteps
    arrived, done = set(), [set() for _ in range(J)]
    finals, nb = set(), (N + C - 1) // C
    nbr = lambda x: ((x - 1) % N, x, (x + 1) % N)   # noqa: E731
    events = plan(N, C, nsteps)
    assert all(k != XCH for k, *_ in events)
    for kind, idx, a, b in events:
        assert 0 <= a < b <= N
        if kind == ARRIVE:
            arrived.update(range(a, b))
            continue
        if kind == FINAL:
            assert idx not in finals and (a, b) == (idx * C, min(N, idx * C + C))
            finals.add(idx)
            for x in range(a, b):
                assert all(x in d for d in done), (N, C, nsteps, "early final", x)
            continue
        j = idx
        for x in range(a, b):
            assert x not in done[j], (N, C, nsteps, "twice", j, x)
            if j == 0:          # black self energy terms: reads black(x)
                ok = x in arrived
            elif j == 1:        # red energy terms: red(x), black(x-1..x+1)
                ok = all(p in arrived for p in nbr(x))
            elif j == 2:        # head (red base): reads black(x+-1); overwrites red(x),
                ok = (all(p in arrived for p in nbr(x))        # which pass 1 read at x
                      and x in done[1])
            else:               # K3/K4: other colour (pass j-1) at x-1..x+1, own (j-2) at x;
                ok = (all(p in done[j - 1] for p in nbr(x))  # WAR: pass j-1 read own(x)
                      and x in done[j - 2])                   # at its outputs x-1..x+1
                if j == 3:      # black: also read by pass 0 at x and pass 1 at x-1..x+1
                    ok = ok and x in done[0] and all(p in done[1] for p in nbr(x))
            assert ok, (N, C, nsteps, "dependency", j, x)
            done[j].add(x)
    assert arrived == set(range(N))
    assert all(len(d) == N for d in done), (N, C, nsteps, "coverage")
    assert finals == set(range(nb))


def colour(j):
    """Colour a pass writes / reads itself: 0 black energy, 1 red energy,
    2 head (red), then K3 black / K4 red."""
    return 0 if j == 0 else 1 if j in (1, 2) else (0 if j % 2 else 1)


def check_split(N, C, nsteps):
    """Every slab runs the same plan, so a slab's ghost plane -1 holds what
    its lower neighbour -- in the same state -- had at local plane N-1 when
    the exchange ran (and ghost N its upper neighbour's plane 0)."""
    J = 3 + 2 * nsteps
    arrived, done = set(), [set() for _ in range(J)]
    finals, nb = set(), (N + C - 1) // C
    ghost = [None, None]            # version held by each colour's ghost planes
    covered = lambda j: {0, N - 1} <= done[j]   # noqa: E731
    n_xch = 0
    for kind, idx, a, b in plan(N, C, nsteps, 1):
        if kind == XCH:
            n_xch += 1
            if idx == -1:           # arrived state: both boundary blocks in
                assert {0, N - 1} <= arrived, (N, C, nsteps, "early arrival exchange")
                ghost = ["A", "A"]
            else:
                c = colour(idx)
                assert idx >= 2 and covered(idx), (N, C, nsteps, "early exchange", idx)
                # WAR: the previous ghost version's readers are done with the boundary
                assert covered(idx - 1), (N, C, nsteps, "ghost overwritten early", idx)
                ghost[c] = idx
            continue
        assert 0 <= a < b <= N
        if kind == ARRIVE:
            arrived.update(range(a, b))
            continue
        if kind == FINAL:
            assert idx not in finals and (a, b) == (idx * C, min(N, idx * C + C))
            finals.add(idx)
            for x in range(a, b):
                assert all(x in d for d in done), (N, C, nsteps, "early final", x)
            continue
        j = idx
        other = 1 - colour(j)
        need = "A" if j in (1, 2) else j - 1    # version of the other colour read
        src = arrived if j in (1, 2) else (done[j - 1] if j >= 3 else None)
        for x in range(a, b):
            assert x not in done[j], (N, C, nsteps, "twice", j, x)
            if j == 0:
                ok = x in arrived
            else:
                ok = True
                for p in (x - 1, x, x + 1):
                    if 0 <= p < N:
                        ok = ok and p in src
                    else:           # ghost plane: the exchanged face of `need`
                        ok = ok and ghost[other] == need
                if j == 1:
                    ok = ok and x in arrived
                elif j == 2:
                    ok = ok and x in arrived and x in done[1]
                else:
                    ok = ok and x in done[j - 2]
                    if j == 3:
                        ok = ok and x in done[0] and all(
                            p in done[1] for p in (x - 1, x, x + 1) if 0 <= p < N)
            assert ok, (N, C, nsteps, "dependency", j, x)
            done[j].add(x)
    assert arrived == set(range(N))
    assert all(len(d) == N for d in done), (N, C, nsteps, "coverage")
    assert finals == set(range(nb))
    assert n_xch == 1 + (J - 2), (N, C, nsteps, "one exchange per writing pass")


@pytest.mark.parametrize("N", [4, 8, 64, 128, 130, 256])
@pytest.mark.parametrize("C", [1, 3, 5, 8, 32])
@pytest.mark.parametrize("nsteps", [0, 1, 2, 7])
def test_pipeline_plan_respects_every_dependency(N, C, nsteps):
    check(N, C, nsteps)


def test_pipeline_plan_headline_shape():
    """1024 planes, 32-plane chunks, 40 steps (the bench's e2e call)."""
    check(1024, 32, 40)


@pytest.mark.parametrize("N", [4, 8, 64, 128, 130, 256])
@pytest.mark.parametrize("C", [1, 3, 5, 8, 32])
@pytest.mark.parametrize("nsteps", [0, 1, 2, 7])
def test_split_plan_exchanges_every_face_in_time(N, C, nsteps):
    check_split(N, C, nsteps)


def test_split_plan_headline_shape():
    """1024^3 on 2 slabs: 512 planes each, 32-plane chunks, 40 steps."""
    check_split(512, 32, 40)


def test_pipeline_plan_rejects_bad_arguments():
    assert _lib.load().kgs_pipeline_plan(0, 32, 1, 0, None, 0) == -1
    assert _lib.load().kgs_pipeline_plan(64, 0, 1, 1, None, 0) == -1


from hypothesis import given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402


@settings(max_examples=300, deadline=None)
@given(N=st.integers(2, 300), C=st.integers(1, 80), nsteps=st.integers(0, 30))
def test_pipeline_plan_random_shapes(N, C, nsteps):
    check(N, C, nsteps)
    check_split(N, C, nsteps)
