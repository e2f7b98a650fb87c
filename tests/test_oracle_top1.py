"""Pins for the oracle's diff-top-1-proofs semiring (P:290,
P:617-628 §3.5; reading "top-1-proof"): one proof (a set of input
facts, cap 300) per tuple, p = Π over the SET in fp64 ascending ids rounded
once, ⊗ = union (dropped on an exclusion-group conflict), ⊕ = the more
likely proof.  Each test checks the oracle against a brute force, a closed
property or a hand-checked case — never against itself.  CPU only."""
from __future__ import annotations

import itertools

import numpy as np
import pytest

import oracle
import workloads as W
from tests import refs

SR = 5


def _dict(rel):
    return {(int(s),) + tuple(int(v) for v in c): float(t)
            for s, c, t in zip(rel.sample_ids, rel.cols, rel.tags)}


def _proof(rel, i):
    a, b = rel.grad_offsets[i], rel.grad_offsets[i + 1]
    return rel.grad_fact_ids[a:b].tolist(), rel.grad_values[a:b].tolist()


def _setp(ids, p):
    q = 1.0
    for f in sorted(ids):
        q *= float(p[f])
    return float(np.float32(q))


@pytest.mark.parametrize("seed", range(10))
def test_linear_tc_equals_best_simple_path(oracle_lib, seed):
    """Linear TC: the top-1 proof of path(x, y) is the most likely simple path
    (any walk's fact set contains a simple path's), by brute force."""
    rng = np.random.default_rng(1500 + seed)
    n = int(rng.integers(3, 8))
    w = W.random_digraph_workload(n, 0.35, 1500 + seed, SR, self_loops=bool(seed % 3 == 0))
    src, dst, p, _ = refs.edge_lists(w)
    rel = oracle.run_workload(w).relations["path"]
    got = _dict(rel)
    adj = refs.make_adj(n, src, dst)
    for x in range(n):
        for y in range(n):
            paths = refs.simple_paths(n, adj, x, y)
            if not paths:
                assert (0, x, y) not in got
                continue
            assert got[(0, x, y)] == max(_setp(pp, p) for pp in paths), (x, y)
    for i in range(len(rel)):  # the proof is a path whose set product is the tag
        ids, g = _proof(rel, i)
        assert _setp(ids, p) == float(rel.tags[i])
        for f, gv in zip(ids, g):
            exp = 1.0
            for h in ids:
                if h != f:
                    exp *= float(p[h])
            assert gv == float(np.float32(exp))


NONLINEAR = """
type edge(x: i32, y: i32)
rel path(x, y) :- edge(x, y) or (path(x, z) and path(z, y)).
output path
"""


@pytest.mark.parametrize("seed", range(6))
def test_nonlinear_tc_matches_linear(oracle_lib, seed):
    """path = path ∘ path under top-1: the same tags as the linear program
    (both reach the best simple path), proofs valid under unit."""
    rng = np.random.default_rng(1600 + seed)
    n = int(rng.integers(3, 9))
    w = W.random_digraph_workload(n, 0.3, 1600 + seed, SR)
    lin = _dict(oracle.run_workload(w).relations["path"])
    nl = oracle.run(NONLINEAR, SR, 1, w.facts, outputs=["path"]).relations["path"]
    assert _dict(nl) == lin
    src, dst, p, _ = refs.edge_lists(w)
    for i in range(len(nl)):
        ids, _ = _proof(nl, i)
        x, y = int(nl.cols[i][0]), int(nl.cols[i][1])
        # the proof's edges connect x to y
        reach = refs.floyd_warshall(n, src[ids], dst[ids], p[ids], "bool")
        assert reach[x, y]


def test_set_semantics_reused_fact(oracle_lib):
    """two(x) :- edge(x, y), edge(x, z): y = z uses ONE fact, so the proof is
    {best edge} with p = max p_e (max-mult would square it)."""
    prog = """
type edge(x: i32, y: i32)
rel two(x) :- edge(x, y), edge(x, z).
output two
"""
    f = W.Facts([np.array([0, 0, 1], np.int32), np.array([1, 2, 2], np.int32)], np.zeros(3, np.int32),
                np.array([0.5, 0.75, 0.25], np.float32))
    r = oracle.run(prog, SR, 1, {"edge": f}).relations["two"]
    assert _dict(r) == {(0, 0): 0.75, (0, 1): 0.25}
    assert _proof(r, 0) == ([1], [1.0])
    r3 = oracle.run(prog, 3, 1, {"edge": f}).relations["two"]
    assert _dict(r3)[(0, 0)] == 0.75 * 0.75


def test_exclusion_group_conflict(oracle_lib):
    """0 -> 1 -> 3 (0.9, 0.9) beats 0 -> 2 -> 3 (0.6, 0.6), but edges 0->1 and
    1->3 are mutually exclusive: path(0, 3)'s proof is the other path."""
    src = np.array([0, 1, 0, 2], np.int32)
    dst = np.array([1, 3, 2, 3], np.int32)
    p = np.array([0.9, 0.9, 0.6, 0.6], np.float32)
    f = {"edge": W.Facts([src, dst], np.zeros(4, np.int32), p)}
    free = _dict(oracle.run(W.PATH_PROGRAM, SR, 1, f).relations["path"])
    assert free[(0, 0, 3)] == _setp([0, 1], p)
    r = oracle.run(W.PATH_PROGRAM, SR, 1, f, groups={"edge": np.array([7, 7, -1, -1], np.int32)}).relations["path"]
    got = _dict(r)
    assert got[(0, 0, 3)] == _setp([2, 3], p)
    i = [tuple(c) for c in r.cols.tolist()].index((0, 3))
    assert _proof(r, i)[0] == [2, 3]
    # the conflicting facts are fine on their own
    assert got[(0, 0, 1)] == float(np.float32(0.9)) and got[(0, 1, 3)] == float(np.float32(0.9))


def test_conflicts_never_in_proofs_bruteforce(oracle_lib):
    """Random groups: no proof holds two facts of one group, and every tuple's
    tag is at most the best conflict-free simple path (brute force); tuples
    without any conflict-free path are absent."""
    rng = np.random.default_rng(1700)
    for trial in range(6):
        n = 6
        w = W.random_digraph_workload(n, 0.4, 1700 + trial, SR)
        src, dst, p, _ = refs.edge_lists(w)
        grp = rng.integers(-1, 3, size=src.shape[0]).astype(np.int32)
        rel = oracle.run(w.program, SR, 1, w.facts, groups={"edge": grp}).relations["path"]
        got = _dict(rel)
        adj = refs.make_adj(n, src, dst)
        for i in range(len(rel)):
            ids, _ = _proof(rel, i)
            g = [int(grp[f]) for f in ids if grp[f] >= 0]
            assert len(g) == len(set(g))
        for x, y in itertools.product(range(n), range(n)):
            ok = [pp for pp in refs.simple_paths(n, adj, x, y)
                  if len([grp[e] for e in pp if grp[e] >= 0]) == len({grp[e] for e in pp if grp[e] >= 0})]
            if (0, x, y) in got:
                assert ok and got[(0, x, y)] <= max(_setp(pp, p) for pp in ok)


def test_proof_cap(oracle_lib):
    """proofs are capped at 300 facts."""
    for n, fail in ((301, False), (302, True)):
        src = np.arange(n - 1, dtype=np.int32)
        f = {"edge": W.Facts([src, src + 1], np.zeros(n - 1, np.int32), np.full(n - 1, 0.999, np.float32))}
        if fail:
            with pytest.raises(oracle.OracleError) as e:
                oracle.run(W.PATH_PROGRAM, SR, 1, f)
            assert "300" in str(e.value)
        else:
            r = oracle.run(W.PATH_PROGRAM, SR, 1, f).relations["path"]
            assert int(np.max(np.diff(r.grad_offsets))) == 300


def test_c1_golden_and_pathfinder(oracle_lib):
    """C1 (a DAG: no fact can repeat on a path) equals the golden max-mult
    column; a reduced Pathfinder batch has valid, conflict-free proofs whose
    set products are the tags."""
    from tests.test_oracle_pins import _load_golden
    E, R, T, G = _load_golden()
    rel = oracle.run_workload(W.c1_workload(SR)).relations["path"]
    for i, c in enumerate(rel.cols):
        assert float(rel.tags[i]) == T[(int(c[0]), int(c[1]))][2]
    w = W.c2_workload(semiring=SR, n=5, batch=2)
    res = oracle.run_workload(w, outputs=["endpoints_connected"])
    ec = res.relations["endpoints_connected"]
    pall = np.concatenate([w.facts["edge"].probs, w.facts["is_endpoint"].probs])
    for i in range(len(ec)):
        ids, _ = _proof(ec, i)
        assert _setp(ids, pall) == float(ec.tags[i])
