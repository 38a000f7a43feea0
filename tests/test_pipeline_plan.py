"""The schedule of the pipelined host integration (kgs_pipeline_plan -- the
exact event list kgs_integrate_host executes) checked on the CPU against the
true data dependencies of every pass, for many grid / chunk / step counts:
chunks of planes arrive around plane 0; each pass may only touch a plane
once what it reads is written (RAW) and what it overwrites has been read by
every earlier reader (WAR); every plane is covered once per pass; a block is
copied back exactly once, only when every pass is done on it."""
from __future__ import annotations

import ctypes

import pytest

from paper_2502_09537_b200 import _lib

ARRIVE, PASS, FINAL = 0, 1, 2


def plan(N, C, nsteps):
    lib = _lib.load()
    n = lib.kgs_pipeline_plan(N, C, nsteps, None, 0)
    assert n > 0
    buf = (ctypes.c_int64 * (4 * n))()
    assert lib.kgs_pipeline_plan(N, C, nsteps, buf, n) == n
    return [tuple(buf[4 * i: 4 * i + 4]) for i in range(n)]


def check(N, C, nsteps):
    J = 3 + 2 * nsteps
    arrived, done = set(), [set() for _ in range(J)]
    finals, nb = set(), (N + C - 1) // C
    nbr = lambda x: ((x - 1) % N, x, (x + 1) % N)   # noqa: E731
    for kind, idx, a, b in plan(N, C, nsteps):
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


@pytest.mark.parametrize("N", [4, 8, 64, 128, 130, 256])
@pytest.mark.parametrize("C", [1, 3, 5, 8, 32])
@pytest.mark.parametrize("nsteps", [0, 1, 2, 7])
def test_pipeline_plan_respects_every_dependency(N, C, nsteps):
    check(N, C, nsteps)


def test_pipeline_plan_headline_shape():
    """1024 planes, 32-plane chunks, 40 steps (the bench's e2e call)."""
    check(1024, 32, 40)


def test_pipeline_plan_rejects_bad_arguments():
    assert _lib.load().kgs_pipeline_plan(0, 32, 1, None, 0) == -1
    assert _lib.load().kgs_pipeline_plan(64, 0, 1, None, 0) == -1


from hypothesis import given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402


@settings(max_examples=300, deadline=None)
@given(N=st.integers(2, 300), C=st.integers(1, 80), nsteps=st.integers(0, 30))
def test_pipeline_plan_random_shapes(N, C, nsteps):
    check(N, C, nsteps)
