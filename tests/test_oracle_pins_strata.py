"""Pins for the oracle's second stratum and its atom forms.

Fig. 3c:

    rel endpoints_connected() :- is_endpoint(x), is_endpoint(y), path(x, y), x != y.

Each test computes the expected value from the plain definition, written here
independently of the oracle: the closure `path` by Floyd–Warshall / Dijkstra /
the add-mult closed form (tests/refs.py), then the arity-0 head as the ⊕ over
every (x, y) with x != y of ep(x) ⊗ ep(y) ⊗ path(x, y) — ⊗ left-deep in body
order, ⊕ = max / + / or.  A dropped or inverted `!=`,
a wrong ⊗ order, a missing arity-0 ⊕ or a mis-bound constant / repeated
variable fails one of these.  CPU only.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle
import workloads as W
from workloads import gen as G
from tests import refs

F32 = np.float32


def _dict(rel):
    return {(int(s),) + tuple(int(v) for v in c): float(t)
            for s, c, t in zip(rel.sample_ids, rel.cols, rel.tags)}


def _grad(rel, i):
    a, b = rel.grad_offsets[i], rel.grad_offsets[i + 1]
    return dict(zip(rel.grad_fact_ids[a:b].tolist(), rel.grad_values[a:b].tolist()))


def _sample_arrays(w, s):
    e, ep = w.facts["edge"], w.facts["is_endpoint"]
    me, mp = e.sample_ids == s, ep.sample_ids == s
    src, dst, p = e.cols[0][me].astype(np.int64), e.cols[1][me].astype(np.int64), e.probs[me]
    cells, q = ep.cols[0][mp].astype(np.int64), ep.probs[mp]
    epv = np.zeros(int(cells.max()) + 1, np.float32)
    epv[cells] = q
    return src, dst, p, epv


# ---------------------------------------------------------------------------
# max-min: Floyd–Warshall is bit-exact (min/max are exact in fp32)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n", [3, 4, 5, 6, 7, 8])
def test_endpoints_connected_maxmin_floyd_warshall(oracle_lib, n):
    w = W.grid_workload(n, 3, 900 + n, 1)
    got = _dict(oracle.run_workload(w, outputs=["endpoints_connected", "path"]).relations["endpoints_connected"])
    assert set(got) == {(s,) for s in range(3)}
    for s in range(3):
        src, dst, p, epv = _sample_arrays(w, s)
        A = refs.floyd_warshall(n * n, src, dst, p, "maxmin")
        reach = refs.floyd_warshall(n * n, src, dst, p, "bool")
        exp = None
        for x in range(n * n):
            for y in range(n * n):
                if x != y and reach[x, y]:
                    v = min(min(float(epv[x]), float(epv[y])), A[x, y])
                    exp = v if exp is None else max(exp, v)
        assert got[(s,)] == exp, (n, s, got[(s,)], exp)


# ---------------------------------------------------------------------------
# max-mult, dyadic tags: integer shortest paths give the exact maximum product
# ---------------------------------------------------------------------------
def _int_dijkstra(nn, src, dst, k, x):
    """min over paths x -> y (length >= 1) of Σ k(e), integer weights."""
    import heapq
    adj = [[] for _ in range(nn)]
    for a, b, c in zip(src, dst, k):
        adj[int(a)].append((int(b), int(c)))
    best = [math.inf] * nn
    h = []
    for b, c in adj[x]:
        if c < best[b]:
            best[b] = c
            heapq.heappush(h, (c, b))
    while h:
        c, u = heapq.heappop(h)
        if c > best[u]:
            continue
        for v, cw in adj[u]:
            if c + cw < best[v]:
                best[v] = c + cw
                heapq.heappush(h, (c + cw, v))
    return best


@pytest.mark.parametrize("n", [3, 4, 5, 6, 8])
def test_endpoints_connected_maxmul_dyadic_exact(oracle_lib, n):
    """p(e) = 2^-k(e), ep(c) = 2^-j(c): every product is exact in fp32, so the
    maximum product is 2^-(min Σk) by integer Dijkstra — a bit-exact pin of the
    value, of `x != y` and of the arity-0 ⊕ = max."""
    rng = np.random.default_rng(950 + n)
    src, dst, _ = G.lattice(n)
    nn = n * n
    k = rng.integers(0, 3, size=src.shape[0])
    j = rng.integers(0, 5, size=nn)
    facts = {"edge": W.Facts([src.astype(np.int32), dst.astype(np.int32)], np.zeros(src.shape[0], np.int32),
                             (2.0 ** -k).astype(np.float32)),
             "is_endpoint": W.Facts([np.arange(nn, dtype=np.int32)], np.zeros(nn, np.int32),
                                    (2.0 ** -j).astype(np.float32))}
    res = oracle.run(W.PATHFINDER_PROGRAM, 3, 1, facts, outputs=["endpoints_connected"])
    ec = res.relations["endpoints_connected"]
    best_exp = None
    for x in range(nn):
        d = _int_dijkstra(nn, src, dst, k, x)
        for y in range(nn):
            if y != x and d[y] < math.inf:
                e = int(j[x] + j[y] + d[y])
                best_exp = e if best_exp is None else min(best_exp, e)
    assert len(ec) == 1
    assert float(ec.tags[0]) == 2.0 ** -best_exp
    # the proof (gradient support) uses two distinct endpoint facts (x != y)
    g = _grad(ec, 0)
    ep_ids = [f for f in g if f >= src.shape[0]]
    assert len(ep_ids) == 2 and ep_ids[0] != ep_ids[1]
    cells = [f - src.shape[0] for f in ep_ids]
    edges = [f for f in g if f < src.shape[0]]
    assert sum(int(k[e]) for e in edges) + sum(int(j[c]) for c in cells) == best_exp


# ---------------------------------------------------------------------------
# max-mult, random tags: Dijkstra on -log p (fp64) within the rounding bound
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n", [3, 5, 8, 12])
def test_endpoints_connected_maxmul_dijkstra(oracle_lib, n):
    batch = 2
    w = W.grid_workload(n, batch, 970 + n, 3)
    res = oracle.run_workload(w, outputs=["endpoints_connected"])
    got = _dict(res.relations["endpoints_connected"])
    for s in range(batch):
        src, dst, p, epv = _sample_arrays(w, s)
        exp = 0.0
        for x in range(n * n):
            best = refs.dijkstra_maxmul(n * n, src, dst, p, x)
            for y in range(n * n):
                if y != x:
                    exp = max(exp, float(epv[x]) * float(epv[y]) * best[y])
        # one rounding per ⊗ along a proof of <= n*n hops
        assert abs(got[(s,)] - exp) <= (n * n + 2) * 2.0 ** -24 * exp, (s, got[(s,)], exp)


# ---------------------------------------------------------------------------
# add-mult on a DAG: the arity-0 ⊕ is the sum over x != y (closed form)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(5))
def test_endpoints_connected_addmult_closed_form(oracle_lib, seed):
    n = 9
    w = W.random_dag_workload(n, 0.35, 990 + seed, 2, program=W.PATHFINDER_PROGRAM)
    rng = np.random.default_rng(990 + seed)
    epv = rng.uniform(0.1, 1.0, n).astype(np.float32)
    w.facts["is_endpoint"] = W.Facts([np.arange(n, dtype=np.int32)], np.zeros(n, np.int32), epv)
    src, dst, p, _ = refs.edge_lists(w)
    P = refs.addmult_closed_form(n, src, dst, p)
    exp = sum(float(epv[x]) * float(epv[y]) * P[x, y] for x in range(n) for y in range(n) if x != y)
    got = _dict(oracle.run_workload(w, outputs=["endpoints_connected"]).relations["endpoints_connected"])
    if exp == 0.0:
        assert got == {}
    else:
        assert abs(got[(0,)] - exp) <= 1e-5 * exp


# ---------------------------------------------------------------------------
# the filter itself: x == y candidates never count
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("sr", [0, 1, 2, 3])
def test_endpoints_connected_filter_excludes_cycles(oracle_lib, sr):
    # one endpoint on a 2-cycle: path(0,0) exists but x != y has no candidate
    e = W.Facts([np.array([0, 1], np.int32), np.array([1, 0], np.int32)], np.zeros(2, np.int32),
                np.array([0.5, 0.5], np.float32))
    one = {"edge": e, "is_endpoint": W.Facts([np.array([0], np.int32)], np.zeros(1, np.int32),
                                              np.array([1.0], np.float32))}
    r = oracle.run(W.PATHFINDER_PROGRAM, sr, 1, one, outputs=["endpoints_connected", "path"])
    assert (0, 0, 0) in _dict(r.relations["path"])
    assert len(r.relations["endpoints_connected"]) == 0
    # two endpoints: the self-cycle 0->0 (0.9·0.9) beats 0->1 (0.5) but is filtered
    e = W.Facts([np.array([0, 0, 2], np.int32), np.array([1, 2, 0], np.int32)], np.zeros(3, np.int32),
                np.array([0.5, 0.9, 0.9], np.float32))
    two = {"edge": e, "is_endpoint": W.Facts([np.array([0, 1], np.int32)], np.zeros(2, np.int32),
                                              np.array([1.0, 1.0], np.float32))}
    r = oracle.run(W.PATHFINDER_PROGRAM, sr, 1, two, outputs=["endpoints_connected"])
    got = _dict(r.relations["endpoints_connected"])
    # only (x, y) = (0, 1) survives the filter (1 has no out-edge)
    # add-mult sums every walk 0 -> 1: 0.5 · Σ_k 0.81^k (truncated by fp32
    # absorption, so within 1e-5 of the geometric series)
    exp = {0: 1.0, 1: 0.5, 2: 0.5 / (1.0 - 0.9 * 0.9), 3: 0.5}[sr]
    assert set(got) == {(0,)}
    if sr == 2:
        assert abs(got[(0,)] - exp) <= 1e-5 * exp
    else:
        assert got[(0,)] == exp


# ---------------------------------------------------------------------------
# constants, ==, repeated variables (plain definitions over the edge list)
# ---------------------------------------------------------------------------
FORMS = """
type edge(x: i32, y: i32)
rel loop(x) :- edge(x, x).
rel from3(y) :- edge(3, y).
rel back(x, z) :- edge(x, z), edge(z, y), x == y.
rel two(x) :- edge(x, y), edge(y, x), x != y.
rel tagged(x, 7) :- edge(x, 5).
output loop
"""


def _brute_forms(src, dst, p, sr):
    def times(a, b):
        return float(min(F32(a), F32(b))) if sr == 1 else float(F32(a) * F32(b))

    def plus(acc, v):
        if sr == 2:
            return acc + v  # fp64 accumulate, rounded once below
        return max(acc, v)

    edges = list(zip(src.tolist(), dst.tolist(), [float(x) for x in p]))
    out = {"loop": {}, "from3": {}, "back": {}, "two": {}, "tagged": {}}

    def add(rel, key, v):
        out[rel][key] = plus(out[rel].get(key, 0.0), v)
    for a, b, q in edges:
        if a == b:
            add("loop", (a,), q)
        if a == 3:
            add("from3", (b,), q)
        if b == 5:
            add("tagged", (a, 7), q)
    for a, b, q in edges:
        for c, d, r in edges:
            if b == c and d == a:
                add("back", (a, b), times(q, r))
                if a != b:
                    add("two", (a,), times(q, r))
    for rel in out:
        out[rel] = {k: float(F32(v)) for k, v in out[rel].items()}
    return out


@pytest.mark.parametrize("sr", [1, 2, 3])
@pytest.mark.parametrize("seed", range(4))
def test_constants_eq_repeated_vars(oracle_lib, sr, seed):
    w = W.random_digraph_workload(9, 0.3, 1100 + seed, sr, self_loops=True, program=FORMS)
    src, dst, p, _ = refs.edge_lists(w)
    exp = _brute_forms(src, dst, p, sr)
    res = oracle.run_workload(w, outputs=list(exp))
    for rel, e in exp.items():
        got = {k[1:]: v for k, v in _dict(res.relations[rel]).items()}
        assert set(got) == set(e), rel
        for k, v in e.items():
            if sr == 2:
                assert abs(got[k] - v) <= 2.0 ** -23 * abs(v), (rel, k)
            else:
                assert got[k] == v, (rel, k, got[k], v)


# ---------------------------------------------------------------------------
# diff-max-min-prob (NEXT-4; §3.5): tags = max-min, one-hot gradient
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(6))
def test_diff_maxmin_tags_equal_floyd_warshall(oracle_lib, seed):
    """The tag is the bottleneck value (Floyd–Warshall max-min, exact); the
    gradient is one-hot on an input fact whose p equals the tag."""
    n = 14
    w = W.random_digraph_workload(n, 0.2, 1200 + seed, 4, self_loops=bool(seed % 2))
    src, dst, p, _ = refs.edge_lists(w)
    A = refs.floyd_warshall(n, src, dst, p, "maxmin")
    reach = refs.floyd_warshall(n, src, dst, p, "bool")
    rel = oracle.run_workload(w).relations["path"]
    got = _dict(rel)
    assert set(got) == {(0, int(a), int(b)) for a, b in zip(*np.nonzero(reach))}
    for i, (s, a, b) in enumerate(zip(rel.sample_ids, rel.cols[:, 0], rel.cols[:, 1])):
        assert float(rel.tags[i]) == A[a, b]
        g = _grad(rel, i)
        assert list(g.values()) == [1.0]
        (f,) = g
        assert float(p[f]) == float(rel.tags[i])


@pytest.mark.parametrize("seed", range(4))
def test_diff_maxmin_forward_differences(oracle_lib, seed):
    """Distinct probabilities: raising the gradient's fact by h raises the tag
    by h; raising any other fact leaves it unchanged (forward differences)."""
    rng = np.random.default_rng(1300 + seed)
    w = W.random_dag_workload(8, 0.45, 1300 + seed, 4)
    f = w.facts["edge"]
    f.probs = rng.permutation(np.linspace(0.2, 0.9, f.n)).astype(np.float32)
    base = oracle.run_workload(w).relations["path"]
    keys = [tuple(int(v) for v in c) for c in base.cols]
    h = np.float32(2.0 ** -12)
    for fid in range(f.n):
        plus = f.probs.copy()
        plus[fid] += h
        tp = _dict(oracle.run(w.program, 4, 1, {"edge": W.Facts(f.cols, f.sample_ids, plus)}).relations["path"])
        for i, k in enumerate(keys):
            d = tp[(0,) + k] - float(base.tags[i])
            exp = float(h) if _grad(base, i).get(fid) == 1.0 else 0.0
            assert d == pytest.approx(exp, abs=1e-7), (k, fid, d)


def test_diff_maxmin_c1_golden(oracle_lib):
    """C1 worked example: diff-max-min tags are the max-min column of the
    golden table; the gradient names the bottleneck edge of the witnessed path."""
    from tests.test_oracle_pins import _load_golden
    E, R, T, G = _load_golden()
    rel = oracle.run_workload(W.c1_workload(4)).relations["path"]
    for i, c in enumerate(rel.cols):
        k = (int(c[0]), int(c[1]))
        assert float(rel.tags[i]) == T[k][1]
        (fid,) = _grad(rel, i)
        assert E[fid][2] == T[k][1]
