"""Pins for the oracle's diff-add-mult-prob (§3.5; P:619 dual-number
tags; reading "diff-add-mult").  The expected gradients come from
the plain definitions, written here independently of the oracle:

* C1 (dyadic, exact): ∂/∂p_e Σ_paths Π p = Σ_{paths through e} Π_{other edges} p,
  by exact-rational path enumeration — equal bit for bit;
* random DAGs: with N = (I − A)^{-1}, path(x, y) = N − I and
  ∂path(x, y)/∂A_ij = N[x, i] · N[j, y] (fp64), within 1e-5 relative, and the
  support is exactly the edges on some x → y path;
* CLUTRR-shaped kinship: central finite differences of the interval DP;
* duplicate input facts: ⊕-merged by +, so each duplicate gets the same entry;
* the p part equals add-mult bit for bit.
A dropped product-rule term, a gradient taken w.r.t. the wrong factor, or a
missing Δ/NEW gradient in a variant fails one of these.  CPU only."""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workloads as W
from tests import refs

DADD = oracle.DIFF_ADD_MULT_PROB


def _rows(rel):
    out = {}
    for i in range(len(rel)):
        k = (int(rel.sample_ids[i]),) + tuple(int(v) for v in rel.cols[i])
        a, b = rel.grad_offsets[i], rel.grad_offsets[i + 1]
        out[k] = (float(rel.tags[i]), dict(zip(rel.grad_fact_ids[a:b].tolist(), rel.grad_values[a:b].tolist())))
    return out


def test_c1_exact(oracle_lib):
    w = W.c1_workload(DADD)
    rows = _rows(oracle.run_workload(w, outputs=["path"]).relations["path"])
    e = w.facts["edge"]
    edges = [(int(s), int(d), float(q)) for s, d, q in zip(e.cols[0], e.cols[1], e.probs)]
    ref = refs.exact_c1_bruteforce(edges)
    assert len(rows) == 14
    for (x, y), (am, _, _, paths, ps) in ref.items():
        p, g = rows[(0, x, y)]
        assert p == float(am)
        want = {}
        for path, q in zip(paths, ps):
            for k, eid in enumerate(path):
                want[eid] = want.get(eid, Fraction(0)) + math.prod(q[:k] + q[k + 1:])
        assert set(g) == set(want), (x, y)
        for f, v in want.items():
            assert g[f] == float(v), (x, y, f)
    # the worked example's headline: path(0,5) = 13/32, d/dp(e6: 3->5) = p(0,3) = 5/8
    assert rows[(0, 0, 5)][0] == 13 / 32 and rows[(0, 0, 5)][1][6] == 0.625


@pytest.mark.parametrize("seed", range(5))
def test_random_dag_closed_form(oracle_lib, seed):
    n = 10 + 4 * seed
    w = W.random_dag_workload(n, 0.25, 300 + seed, DADD, batch=2)
    res = oracle.run_workload(w, outputs=["path"])
    rows = _rows(res.relations["path"])
    base = oracle.run(w.program, oracle.ADD_MULT_PROB, w.batch_size, w.facts, outputs=["path"]).relations["path"]
    assert np.array_equal(base.tags.view(np.uint32), res.relations["path"].tags.view(np.uint32))
    for s in range(2):
        src, dst, p, fid = refs.edge_lists(w, s)
        A = np.zeros((n, n))
        A[src, dst] = p.astype(np.float64)
        N = np.linalg.inv(np.eye(n) - A)
        reach = (N != 0)
        for x in range(n):
            for y in range(n):
                if (s, x, y) not in rows:
                    continue
                _, g = rows[(s, x, y)]
                want = {int(f): N[x, i] * N[j, y] for i, j, f in zip(src, dst, fid) if reach[x, i] and reach[j, y]}
                assert set(g) == set(want), (s, x, y)
                for f, v in want.items():
                    assert abs(g[f] - v) <= 1e-5 * abs(v) + 1e-12, (s, x, y, f, g[f], v)


def test_duplicates_share_the_gradient(oracle_lib):
    f = W.Facts([np.array([0, 0, 1], np.int32), np.array([1, 1, 2], np.int32)], np.zeros(3, np.int32),
                np.array([0.25, 0.5, 0.5], np.float32))
    w = W.Workload("dup", W.PATH_PROGRAM, DADD, 1, {"edge": f})
    rows = _rows(oracle.run_workload(w, outputs=["path"]).relations["path"])
    assert rows[(0, 0, 1)] == (0.75, {0: 1.0, 1: 1.0})
    assert rows[(0, 0, 2)] == (0.375, {0: 0.5, 1: 0.5, 2: 0.75})


def test_kinship_finite_differences(oracle_lib):
    w = W.c3_workload(semiring=DADD, batch=1, entities=7, rtypes=4, skips=3, ncomp=8)
    w.program = w.program + "output kinship\n"
    rows = _rows(oracle.run_workload(w, outputs=["kinship"]).relations["kinship"])
    fct, cmp_ = w.facts["fact"], w.facts["composition"]
    comp = {(int(a), int(b)): int(c) for a, b, c in zip(*cmp_.cols)}
    keys = [(int(r), int(a), int(c)) for r, a, c in zip(*fct.cols)]
    base = {k: float(q) for k, q in zip(keys, fct.probs)}
    checked = 0
    for fi, k in enumerate(keys):
        h = 1e-6
        up, dn = dict(base), dict(base)
        up[k] += h
        dn[k] -= h
        d = (refs.kinship_interval_dp(7, 4, up, comp) - refs.kinship_interval_dp(7, 4, dn, comp)) / (2 * h)
        for (r, a, c) in zip(*np.nonzero(d)):
            if abs(d[r, a, c]) < 1e-9:
                continue
            _, g = rows[(0, int(r), int(a), int(c))]
            assert abs(g.get(fi, 0.0) - d[r, a, c]) <= 1e-4 * abs(d[r, a, c]) + 1e-7, (fi, r, a, c)
            checked += 1
    assert checked > 50
