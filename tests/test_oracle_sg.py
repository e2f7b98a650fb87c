"""Pins for the oracle on Same Generation (Table 2, P:802-803;
SURVEY §8(f) NEXT-3), the non-linear-looking two-rule program

    sg(x, y) :- edge(p, x), edge(p, y), x != y.
    sg(x, y) :- edge(a, x), sg(a, b), edge(b, y).

Expected tuple sets come from the plain definition written here as boolean
matrix algebra, independent of the oracle's semi-naive evaluator:
    SG_1 = offdiag(Eᵀ E),   SG_{k+1} = Eᵀ SG_k E,   SG = ∪_k SG_k
(a dropped `x != y`, a transposed edge atom or a missing recursive variant
changes the set).  CPU only."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workloads as W
from workloads import gen as G


def sg_reference(n, src, dst):
    E = np.zeros((n, n), np.int64)
    E[src, dst] = 1
    S = (E.T @ E) > 0
    np.fill_diagonal(S, False)
    total = S.copy()
    frontier = S
    while True:
        nxt = (E.T @ frontier.astype(np.int64) @ E) > 0
        new = nxt & ~total
        if not new.any():
            return total
        total |= new
        frontier = new


def _oracle_set(w):
    r = oracle.run_workload(w, outputs=["sg"]).relations["sg"]
    return {(int(a), int(b)) for a, b in r.cols}


@pytest.mark.parametrize("seed", range(5))
def test_sg_dag_matches_matrix_definition(oracle_lib, seed):
    n = 12 + 7 * seed
    w = G.sg_workload(nodes=n, out_degree=2 + seed % 2, seed=seed)
    e = w.facts["edge"]
    ref = sg_reference(n, e.cols[0], e.cols[1])
    assert _oracle_set(w) == {(int(a), int(b)) for a, b in zip(*np.nonzero(ref))}


@pytest.mark.parametrize("seed", range(4))
def test_sg_cyclic_digraph_matches_matrix_definition(oracle_lib, seed):
    """Cycles and self-loops: still the least fixpoint of the matrix recursion."""
    w = W.random_digraph_workload(14 + seed, 0.18, 300 + seed, G.UNIT, batch=1, self_loops=seed % 2 == 1,
                                  program=G.SG_PROGRAM)
    e = w.facts["edge"]
    ref = sg_reference(14 + seed, e.cols[0], e.cols[1])
    assert _oracle_set(w) == {(int(a), int(b)) for a, b in zip(*np.nonzero(ref))}


def test_sg_hand_example(oracle_lib):
    """A tree: root 0 -> {1, 2}, 1 -> {3, 4}, 2 -> {5}.  Rule 1 gives the
    sibling pairs (1,2), (2,1), (3,4), (4,3); rule 2 lifts sg(1,2) / sg(2,1)
    to the cousins (3,5), (4,5), (5,3), (5,4).  No (x, x): in a tree every
    node has one parent, so rule 2 would need sg(a, a), which never exists."""
    f = W.Facts([np.array([0, 0, 1, 1, 2], np.int32), np.array([1, 2, 3, 4, 5], np.int32)],
                np.zeros(5, np.int32), None)
    w = W.Workload("sg", G.SG_PROGRAM, G.UNIT, 1, {"edge": f})
    assert _oracle_set(w) == {(1, 2), (2, 1), (3, 4), (4, 3), (3, 5), (5, 3), (4, 5), (5, 4)}
