"""Pin for add-mult on CYCLIC inputs (formerly "parity
unpinned").  CPU only.

On a digraph with cycles, add-mult-prob sums over infinitely many derivations
(Fig. 7 add-mult: ⊕ = +, ⊗ = ×).  With spectral radius ρ(A) < 1 the
sum over walks of length ≥ 1 is the Neumann series Σ_{k≥1} A^k = (I−A)^{-1} − I,
a closed form independent of the evaluator.  Semi-naive evaluation in fp32
(reading 1: stop when no tag's fp32 bits change) adds the walks of length k in
round k and stops once every increment is absorbed: its result is that series
truncated at fp32 resolution.  Bound used here: with every row sum of A ≤ 0.5
(so ρ ≤ 0.5) the neglected tail after an absorbed increment δ < 2^-24·t is
≤ δ·ρ/(1−ρ) ≤ 2^-24·t, and each of the K ≤ ~60 rounds rounds the tag once
(≤ 2^-24·t each), so |oracle − closed form| ≤ ~62·2^-24·t < 4e-6·t; the test
uses 1e-5 relative.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workloads as W
from tests import refs


@pytest.fixture(scope="module")
def oracle_lib():
    oracle.build()


def _cyclic(n, p_edge, seed, rowsum=0.5, self_loops=True):
    rng = np.random.default_rng(seed)
    m = rng.random((n, n)) < p_edge
    if not self_loops:
        np.fill_diagonal(m, False)
    # a Hamiltonian cycle guarantees cycles through every node
    perm = rng.permutation(n)
    m[perm, np.roll(perm, -1)] = True
    a, b = np.nonzero(m)
    p = rng.uniform(0.05, 1.0, size=a.shape[0])
    rs = np.zeros(n)
    np.add.at(rs, a, p)
    p = p * (rowsum / rs[a])  # every row sum == rowsum
    f = W.Facts([a.astype(np.int32), b.astype(np.int32)], np.zeros(a.shape[0], np.int32), p.astype(np.float32))
    return W.Workload("cyclic", W.PATH_PROGRAM, 2, 1, {"edge": f})


@pytest.mark.parametrize("seed", range(8))
def test_addmult_cyclic_neumann_closed_form(oracle_lib, seed):
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(2, 24))
    w = _cyclic(n, float(rng.uniform(0.05, 0.4)), 900 + seed, self_loops=bool(seed % 2))
    src, dst, p, _ = refs.edge_lists(w)
    A = np.zeros((n, n))
    np.add.at(A, (src, dst), p.astype(np.float64))
    assert np.max(np.abs(np.linalg.eigvals(A))) <= 0.5 + 1e-6  # fp32 rounding of the tags
    K = refs.addmult_closed_form(n, src, dst, p)
    B = refs.floyd_warshall(n, src, dst, p, "bool")
    res = oracle.run_workload(w)
    rel = res.relations["path"]
    got = {(int(c[0]), int(c[1])): float(t) for c, t in zip(rel.cols, rel.tags)}
    assert set(got) == {(int(a), int(b)) for a, b in zip(*np.nonzero(B))}
    for (a, b), t in got.items():
        assert abs(t - K[a, b]) <= 1e-5 * K[a, b], (a, b, t, K[a, b])
    assert int(res.rounds.sum()) < 200


def test_addmult_single_cycle_geometric(oracle_lib):
    """One directed k-cycle with edge weight q: path(x, x) = q^k / (1 − q^k)
    (the geometric series of going round 1, 2, ... times)."""
    k, q = 5, 0.75
    a = np.arange(k, dtype=np.int32)
    f = W.Facts([a, (a + 1) % k], np.zeros(k, np.int32), np.full(k, q, np.float32))
    w = W.Workload("cycle", W.PATH_PROGRAM, 2, 1, {"edge": f})
    rel = oracle.run_workload(w).relations["path"]
    got = {(int(c[0]), int(c[1])): float(t) for c, t in zip(rel.cols, rel.tags)}
    assert len(got) == k * k
    r = q ** k
    for (x, y), t in got.items():
        d = (y - x) % k or k  # shortest walk length x -> y (k for x == y)
        exact = q ** d / (1.0 - r)
        assert abs(t - exact) <= 1e-5 * exact, (x, y, t, exact)


@pytest.mark.parametrize("seed", range(4))
def test_diff_addmult_cyclic_gradient_closed_form(oracle_lib, seed):
    """diff-add-mult on cyclic inputs: p bit-identical to add-mult, and
    ∂path(x, y)/∂p_(i,j) = M[x, i]·M[j, y] with M = (I − A)^{-1} (the
    derivative of the Neumann series; zero-entries = unreachable).  The
    gradient's tail after the fp32 stop is at most K times p's (walk length
    K multiplies each term): Σ_f q_f·∂p/∂q_f = Σ_walks length·weight, so an
    entry's truncation error is bounded by q_f·|Δg_f| ≤ K·2^-24·p(x, y), not
    by its own size (a far edge's small gradient converges later).  Checked:
    q_f·|g_f − M[x,i]M[j,y]| ≤ 1e-5·p(x, y)."""
    rng = np.random.default_rng(950 + seed)
    n = int(rng.integers(3, 16))
    w = _cyclic(n, float(rng.uniform(0.05, 0.3)), 950 + seed, self_loops=bool(seed % 2))
    w = W.Workload(w.name, w.program, 6, 1, w.facts)
    res = oracle.run_workload(w, outputs=["path"])
    base = oracle.run(w.program, 2, 1, w.facts, outputs=["path"]).relations["path"]
    rel = res.relations["path"]
    assert np.array_equal(base.tags.view(np.uint32), rel.tags.view(np.uint32))
    src, dst, p, fid = refs.edge_lists(w)
    A = np.zeros((n, n))
    np.add.at(A, (src, dst), p.astype(np.float64))
    M = np.linalg.inv(np.eye(n) - A)
    worst = 0.0
    for i, (c, t) in enumerate(zip(rel.cols, rel.tags)):
        x, y = int(c[0]), int(c[1])
        a, b = rel.grad_offsets[i], rel.grad_offsets[i + 1]
        g = dict(zip(rel.grad_fact_ids[a:b].tolist(), rel.grad_values[a:b].tolist()))
        want = {int(f): M[x, s] * M[d, y] for s, d, f in zip(src, dst, fid) if M[x, s] != 0 and M[d, y] != 0}
        assert set(g) == set(want), (x, y)
        for f, v in want.items():
            worst = max(worst, float(p[list(fid).index(f)]) * abs(g[f] - v) / float(t))
    assert worst <= 1e-5, worst
