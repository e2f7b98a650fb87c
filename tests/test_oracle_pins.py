"""Pins for the oracle (SURVEY §8(c) "What pins each part").  Each test checks
the oracle against something other than itself: a value printed in a cited
source, a textbook algorithm, a closed form, brute force, or a law.  CPU only.
"""
from __future__ import annotations

import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workloads as W
from tests import refs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
SR_NAMES = {0: "unit", 1: "max_min", 2: "add_mult", 3: "max_mult"}


def _dict(rel):
    return {(int(s),) + tuple(int(v) for v in c): float(t)
            for s, c, t in zip(rel.sample_ids, rel.cols, rel.tags)}


def _grad(rel, i):
    a, b = rel.grad_offsets[i], rel.grad_offsets[i + 1]
    return dict(zip(rel.grad_fact_ids[a:b].tolist(), rel.grad_values[a:b].tolist()))


def _load_golden():
    E, R, T, G = [], None, {}, {}
    with open(os.path.join(GOLDEN, "c1_worked_example.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            k, *v = line.split()
            if k == "E":
                E.append((int(v[1]), int(v[2]), float(v[3])))
            elif k == "R":
                R = dict(zip([0, 1, 2, 3], [int(v[0]), int(v[1]), int(v[2]), int(v[3])]))
            elif k == "T":
                T[(int(v[0]), int(v[1]))] = (float(v[2]), float(v[3]), float(v[4]),
                                             sorted(int(x) for x in v[5].split(",")))
            elif k == "G":
                G[(int(v[0]), int(v[1]))] = {int(a): float(b) for a, b in (x.split(":") for x in v[2:])}
    return E, R, T, G


# ---------------------------------------------------------------------------
# Worked example (cited fixture) and its brute-force re-derivation
# ---------------------------------------------------------------------------
def test_c1_golden_bruteforce():
    """The golden table equals exact-rational enumeration of every DAG path."""
    E, R, T, G = _load_golden()
    assert E == W.C1_EDGES
    bf = refs.exact_c1_bruteforce(E)
    assert set(bf) == set(T)
    for k, (am, mm, mx, paths, ps) in bf.items():
        g_am, g_mm, g_mx, proof = T[k]
        assert Fraction(g_am) == am and Fraction(g_mm) == mm and Fraction(g_mx) == mx, k
        # the golden proof is one of the argmax paths
        best = [sorted(p) for p, q in zip(paths, ps) if math.prod(q) == mx]
        assert proof in best, k


@pytest.mark.parametrize("sr", [0, 1, 2, 3])
def test_c1_golden_oracle(oracle_lib, sr):
    E, R, T, G = _load_golden()
    res = oracle.run_workload(W.c1_workload(sr))
    got = _dict(res.relations["path"])
    assert set(got) == {(0,) + k for k in T}
    assert int(res.rounds[0]) == R[sr]
    col = {1: 1, 2: 0, 3: 2}.get(sr)
    for k, v in T.items():
        if col is not None:
            assert got[(0,) + k] == v[col], (k, got[(0,) + k], v[col])
    if sr == 3:
        rel = res.relations["path"]
        keys = [tuple(int(v) for v in c) for c in rel.cols]
        for i, k in enumerate(keys):
            assert sorted(_grad(rel, i)) == T[k][3], k
        assert _grad(rel, keys.index((0, 5))) == G[(0, 5)]


def test_spec_examples(oracle_lib):
    """SPEC.md:75 (TC of chain 1→2→3) and SPEC.md:76 (max-min path(1,3)=0.8)."""
    f = W.Facts([np.array([1, 2], np.int32), np.array([2, 3], np.int32)], np.zeros(2, np.int32),
                np.array([1, 1], np.float32))
    r = oracle.run(W.PATH_PROGRAM, 0, 1, {"edge": f})
    assert sorted(_dict(r.relations["path"])) == [(0, 1, 2), (0, 1, 3), (0, 2, 3)]
    assert int(r.rounds[0]) == 3  # reached in 3 iterations (incl. the empty one)
    f = W.Facts([np.array([1, 2, 1], np.int32), np.array([2, 3, 3], np.int32)], np.zeros(3, np.int32),
                np.array([0.9, 0.5, 0.8], np.float32))
    r = oracle.run(W.PATH_PROGRAM, 1, 1, {"edge": f})
    assert _dict(r.relations["path"])[(0, 1, 3)] == np.float32(0.8)


def test_paper_edge_example(oracle_lib):
    """the fact 0.97::edge(0,1) yields path(0,1) with tag 0.97 (max-min)."""
    f = W.Facts([np.array([0], np.int32), np.array([1], np.int32)], np.zeros(1, np.int32),
                np.array([0.97], np.float32))
    for sr in (1, 2, 3):
        r = oracle.run(W.PATH_PROGRAM, sr, 1, {"edge": f})
        assert _dict(r.relations["path"]) == {(0, 0, 1): float(np.float32(0.97))}


# ---------------------------------------------------------------------------
# Floyd–Warshall
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(12))
def test_floyd_warshall_bool_maxmin(oracle_lib, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 30))
    w = W.random_digraph_workload(n, float(rng.uniform(0.03, 0.3)), seed, 1,
                                  self_loops=bool(seed % 2))
    src, dst, p, _ = refs.edge_lists(w)
    A = refs.floyd_warshall(n, src, dst, p, "bool")
    M = refs.floyd_warshall(n, src, dst, p, "maxmin")
    for sr in (0, 1):
        got = _dict(oracle.run_workload(W.Workload("g", w.program, sr, 1, w.facts)).relations["path"])
        assert set(got) == {(0, int(a), int(b)) for a, b in zip(*np.nonzero(A))}
        if sr == 1:
            for (s, a, b), t in got.items():
                assert t == np.float32(M[a, b])


@pytest.mark.parametrize("seed", range(8))
def test_floyd_warshall_maxmul(oracle_lib, seed):
    """(max,×): bit-exact on powers of two, within 1e-6 on random fp32."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(2, 25))
    w = W.random_digraph_workload(n, 0.15, 100 + seed, 3)
    f = w.facts["edge"]
    if seed % 2 == 0:
        f.probs = (0.5 ** rng.integers(0, 4, size=f.n)).astype(np.float32)
    src, dst, p, _ = refs.edge_lists(w)
    M = refs.floyd_warshall(n, src, dst, p, "maxmul")
    got = _dict(oracle.run_workload(w, want_grads=False).relations["path"])
    assert set(got) == {(0, int(a), int(b)) for a, b in zip(*np.nonzero(refs.floyd_warshall(n, src, dst, p, "bool")))}
    for (s, a, b), t in got.items():
        if seed % 2 == 0:
            assert t == M[a, b]
        else:
            assert abs(t - M[a, b]) <= 1e-6 * M[a, b] + 1e-30


# ---------------------------------------------------------------------------
# Closed forms
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(10))
def test_addmult_closed_form_dag(oracle_lib, seed):
    rng = np.random.default_rng(200 + seed)
    n = int(rng.integers(2, 22))
    w = W.random_dag_workload(n, float(rng.uniform(0.1, 0.5)), 200 + seed, 2)
    src, dst, p, _ = refs.edge_lists(w)
    K = refs.addmult_closed_form(n, src, dst, p)
    B = refs.floyd_warshall(n, src, dst, p, "bool")
    got = _dict(oracle.run_workload(w).relations["path"])
    assert set(got) == {(0, int(a), int(b)) for a, b in zip(*np.nonzero(B))}
    for (s, a, b), t in got.items():
        assert abs(t - K[a, b]) <= 1e-5 * abs(K[a, b]), (a, b, t, K[a, b])


@pytest.mark.parametrize("seed", range(4))
def test_kinship_interval_dp(oracle_lib, seed):
    """CLUTRR-shaped program (C3) vs the interval DP closed form."""
    E, R = 9, 5
    w = W.c3_workload(batch=3, entities=E, rtypes=R, skips=6, ncomp=12, seed=300 + seed)
    res = oracle.run_workload(w)
    comp_f = w.facts["composition"]
    comp = {(int(a), int(b)): int(c) for a, b, c in zip(*comp_f.cols)}
    ff = w.facts["fact"]
    kin = _dict(res.relations["kinship"])
    ans = _dict(res.relations["answer"])
    for s in range(3):
        m = ff.sample_ids == s
        facts = {}
        for r, a, c, q in zip(ff.cols[0][m], ff.cols[1][m], ff.cols[2][m], ff.probs[m]):
            facts[(int(r), int(a), int(c))] = facts.get((int(r), int(a), int(c)), 0.0) + float(q)
        K = refs.kinship_interval_dp(E, R, facts, comp)
        nz = {(s, r, a, c) for r, a, c in zip(*np.nonzero(K > 0))}
        mine = {k for k in kin if k[0] == s}
        # tuple set: derivable tuples (K>0 since all facts have p>0 and comp tags are 1)
        assert mine == {(s, int(r), int(a), int(c)) for (_, r, a, c) in nz}
        for (_, r, a, c) in mine:
            assert abs(kin[(s, r, a, c)] - K[r, a, c]) <= 1e-5 * K[r, a, c]
        for r in range(R):
            if K[r, 0, E - 1] > 0:
                assert abs(ans[(s, r)] - K[r, 0, E - 1]) <= 1e-5 * K[r, 0, E - 1]


@pytest.mark.parametrize("n", [3, 4, 5, 6])
def test_grid_unit_closed_forms(oracle_lib, n):
    """Full lattice under unit: n^4 tuples, 2(n-1)+1 rounds, n^2|E|+|E| candidates."""
    src, dst, _ = W.gen.lattice(n)
    f = W.Facts([src.astype(np.int32), dst.astype(np.int32)], np.zeros(src.shape[0], np.int32), None)
    r = oracle.run(W.PATH_PROGRAM, 0, 1, {"edge": f})
    E = src.shape[0]
    assert E == 4 * n * (n - 1)
    assert len(r.relations["path"]) == n ** 4
    assert int(r.rounds[0]) == 2 * (n - 1) + 1
    assert int(r.candidates[0]) == n * n * E + E


# ---------------------------------------------------------------------------
# Brute force on tiny inputs
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(12))
def test_bruteforce_simple_paths(oracle_lib, seed):
    """Idempotent semirings: tag(x,y) = best over simple paths (cycles for x=y);
    max-mult gradient = ∂/∂p of the unique argmax path (distinct p)."""
    rng = np.random.default_rng(400 + seed)
    n = int(rng.integers(2, 7))
    w = W.random_digraph_workload(n, 0.45, 400 + seed, 3)
    src, dst, p, _ = refs.edge_lists(w)
    adj = refs.make_adj(n, src, dst)
    for sr in (0, 1, 3):
        ww = W.Workload("g", w.program, sr, 1, w.facts)
        res = oracle.run_workload(ww)
        rel = res.relations["path"]
        got = _dict(rel)
        exp = {}
        for x in range(n):
            for y in range(n):
                paths = refs.simple_paths(n, adj, x, y)
                if paths:
                    exp[(0, x, y)] = paths
        assert set(got) == set(exp)
        for i, (k, t) in enumerate(sorted(got.items())):
            paths = exp[k]
            if sr == 1:
                assert t == max(min(float(p[e]) for e in q) for q in paths)
            if sr == 3:
                prods = [math.prod(float(p[e]) for e in q) for q in paths]
                best = max(prods)
                assert abs(t - best) <= 1e-6 * best
                arg = [q for q, v in zip(paths, prods) if v == best]
                if len(arg) == 1 and len(set(prods)) == len(prods):
                    g = _grad(rel, i)
                    q = arg[0]
                    assert sorted(g) == sorted(set(int(e) for e in q))
                    for e in q:
                        other = math.prod(float(p[f]) for f in q if f != e)
                        assert abs(g[int(e)] - other) <= 1e-5 * other + 1e-30


@pytest.mark.parametrize("seed", range(8))
def test_bruteforce_addmult_derivations(oracle_lib, seed):
    """add-mult on a DAG = Σ over derivation trees = Σ over paths of Π p (the
    left-linear TC rule has exactly one derivation tree per path)."""
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(2, 8))
    w = W.random_dag_workload(n, 0.5, 500 + seed, 2)
    src, dst, p, _ = refs.edge_lists(w)
    adj = refs.make_adj(n, src, dst)
    got = _dict(oracle.run_workload(w).relations["path"])
    for x in range(n):
        for y in range(n):
            paths = refs.all_paths_dag(n, adj, x, y)
            if not paths:
                assert (0, x, y) not in got
                continue
            s = sum(math.prod(float(p[e]) for e in q) for q in paths)
            assert abs(got[(0, x, y)] - s) <= 1e-5 * s


# ---------------------------------------------------------------------------
# Textbook special cases
# ---------------------------------------------------------------------------
def test_reach_equals_bfs(oracle_lib):
    """Unit reachability per source = BFS (C4 shape, reduced graph)."""
    w = W.c4_workload(batch=6, nodes=2000, edges=12000, seed=41)
    res = oracle.run_workload(w)
    reach = res.relations["reach"]
    src = w.facts["edge"].cols[0].astype(np.int64)
    dst = w.facts["edge"].cols[1].astype(np.int64)
    sources = w.facts["source"].cols[0]
    for s in range(6):
        mine = np.sort(reach.cols[reach.sample_ids == s][:, 0])
        exp = refs.bfs_reach(2000, src, dst, int(sources[s]))
        assert np.array_equal(mine, exp)


@pytest.mark.parametrize("seed", range(4))
def test_maxmul_equals_dijkstra(oracle_lib, seed):
    n = 40
    w = W.random_digraph_workload(n, 0.08, 600 + seed, 3)
    src, dst, p, _ = refs.edge_lists(w)
    got = _dict(oracle.run_workload(w, want_grads=False).relations["path"])
    for x in range(n):
        best = refs.dijkstra_maxmul(n, src, dst, p, x)
        for y in range(n):
            if (0, x, y) in got:
                assert abs(got[(0, x, y)] - best[y]) <= 1e-6 * best[y] + 1e-37
            else:
                assert best[y] == 0.0


def test_maxmin_undirected_bottleneck(oracle_lib):
    """Max-min on a symmetric instance = bottleneck path on a maximum spanning tree."""
    rng = np.random.default_rng(7)
    n = 25
    pairs = [(a, b) for a in range(n) for b in range(a + 1, n) if rng.random() < 0.2]
    pr = rng.uniform(0.05, 1.0, size=len(pairs)).astype(np.float32)
    src = np.array([a for a, b in pairs] + [b for a, b in pairs], np.int32)
    dst = np.array([b for a, b in pairs] + [a for a, b in pairs], np.int32)
    p = np.concatenate([pr, pr])
    got = _dict(oracle.run(W.PATH_PROGRAM, 1, 1, {"edge": W.Facts([src, dst], np.zeros(len(src), np.int32), p)}).relations["path"])
    # Kruskal maximum spanning forest
    parent = list(range(n))

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a
    tree = [[] for _ in range(n)]
    for i in np.argsort(-pr, kind="stable"):
        a, b = pairs[i]
        ra, rb = find(a), find(b)
        if ra != rb:
            parent[ra] = rb
            tree[a].append((b, pr[i]))
            tree[b].append((a, pr[i]))
    for x in range(n):
        # bottleneck to every node in x's tree component
        bott = {x: np.float32(np.inf)}
        st = [x]
        while st:
            u = st.pop()
            for v, q in tree[u]:
                if v not in bott:
                    bott[v] = min(bott[u], q)
                    st.append(v)
        for y, b in bott.items():
            if y == x:
                if tree[x]:  # cycle x->nb->x: best incident edge
                    assert got[(0, x, x)] == max(q for _, q in tree[x])
                continue
            assert got[(0, x, y)] == b


# ---------------------------------------------------------------------------
# Semiring laws and naive ≡ semi-naive
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("sr", [1, 2, 3])
def test_semiring_laws(oracle_lib, sr):
    rng = np.random.default_rng(sr)
    v = rng.uniform(0, 1, size=(300, 3)).astype(np.float32)
    op, ot = oracle.oplus, oracle.otimes
    for a, b, c in v:
        a, b, c = float(a), float(b), float(c)
        assert op(sr, a, b) == op(sr, b, a)
        assert op(sr, a, 0.0) == np.float32(a)
        assert ot(sr, a, 1.0) == np.float32(a) and ot(sr, 1.0, a) == np.float32(a)
        assert ot(sr, a, 0.0) == 0.0
        l, r = ot(sr, ot(sr, a, b), c), ot(sr, a, ot(sr, b, c))
        if sr == 1:
            assert l == r
            assert op(sr, op(sr, a, b), c) == op(sr, a, op(sr, b, c))
            assert ot(sr, a, op(sr, b, c)) == op(sr, ot(sr, a, b), ot(sr, a, c))
        elif sr == 3:
            assert abs(l - r) <= 2e-7 * abs(l)
            assert op(sr, op(sr, a, b), c) == op(sr, a, op(sr, b, c))
            assert ot(sr, a, op(sr, b, c)) == op(sr, ot(sr, a, b), ot(sr, a, c))  # × monotone
        else:
            assert abs(l - r) <= 2e-7 * abs(l)
            x, y = op(sr, op(sr, a, b), c), op(sr, a, op(sr, b, c))
            assert abs(x - y) <= 2e-7 * abs(x)
            d1, d2 = ot(sr, a, op(sr, b, c)), op(sr, ot(sr, a, b), ot(sr, a, c))
            assert abs(d1 - d2) <= 4e-7 * abs(d1) + 1e-38


@pytest.mark.parametrize("seed", range(6))
def test_naive_kleene_equals_seminaive(oracle_lib, seed):
    rng = np.random.default_rng(700 + seed)
    n = int(rng.integers(3, 15))
    dag = W.random_dag_workload(n, 0.4, 700 + seed, 2)
    cyc = W.random_digraph_workload(n, 0.2, 700 + seed, 1)
    for w, kind in ((dag, "addmul"), (cyc, "maxmin"), (cyc, "bool")):
        src, dst, p, _ = refs.edge_lists(w)
        Ph, P = refs.kleene_naive_tc(n, src, dst, p, kind)
        sr = {"addmul": 2, "maxmin": 1, "bool": 0}[kind]
        got = _dict(oracle.run_workload(W.Workload("g", w.program, sr, 1, w.facts)).relations["path"])
        assert set(got) == {(0, int(a), int(b)) for a, b in zip(*np.nonzero(Ph))}
        for (s, a, b), t in got.items():
            if kind == "maxmin":
                assert t == P[a, b]
            elif kind == "addmul":
                assert abs(t - P[a, b]) <= 1e-5 * P[a, b]


# ---------------------------------------------------------------------------
# Gradients: finite differences and proof validity
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(4))
def test_gradient_finite_differences(oracle_lib, seed):
    rng = np.random.default_rng(800 + seed)
    n = 7
    w = W.random_dag_workload(n, 0.45, 800 + seed, 3)
    f = w.facts["edge"]
    f.probs = rng.permutation(np.linspace(0.3, 0.95, f.n)).astype(np.float32)  # distinct
    base = oracle.run_workload(w).relations["path"]
    keys = [tuple(int(v) for v in c) for c in base.cols]
    h = 1e-3
    for fid in range(f.n):
        plus = f.probs.copy(); plus[fid] += h
        minus = f.probs.copy(); minus[fid] -= h
        tp = _dict(oracle.run(w.program, 3, 1, {"edge": W.Facts(f.cols, f.sample_ids, plus)}).relations["path"])
        tm = _dict(oracle.run(w.program, 3, 1, {"edge": W.Facts(f.cols, f.sample_ids, minus)}).relations["path"])
        for i, k in enumerate(keys):
            fd = (tp[(0,) + k] - tm[(0,) + k]) / (float(np.float32(plus[fid])) - float(np.float32(minus[fid])))
            g = _grad(base, i).get(fid, 0.0)
            assert abs(fd - g) <= 1e-3 * max(abs(g), 1e-2), (k, fid, fd, g)


def test_proof_validity(oracle_lib):
    """The proof (gradient support) re-derives its tuple under unit."""
    w = W.c2_workload(samples=[0], n=6, batch=1)
    res = oracle.run_workload(w, outputs=["endpoints_connected"])
    ec = res.relations["endpoints_connected"]
    allf = {}
    fid = 0
    for rel, f in w.facts.items():
        for i in range(f.n):
            allf[fid] = (rel, i)
            fid += 1
    for i in range(len(ec)):
        proof = sorted(_grad(ec, i))
        sub = {}
        for rel, f in w.facts.items():
            idx = [allf[q][1] for q in proof if allf[q][0] == rel]
            sub[rel] = W.Facts([c[idx] for c in f.cols], f.sample_ids[idx], None)
        r = oracle.run(w.program, 0, 1, sub, outputs=["endpoints_connected"])
        assert len(r.relations["endpoints_connected"]) == 1


# ---------------------------------------------------------------------------
# Batching ≡ independent runs; sample subsets; errors
# ---------------------------------------------------------------------------
def test_batching_equals_independent(oracle_lib):
    w = W.c2_workload(semiring=3, n=6, batch=3)
    full = oracle.run_workload(w, outputs=["path", "endpoints_connected"])
    for s in range(3):
        one = W.c2_workload(semiring=3, n=6, batch=3, samples=[s])
        r1 = oracle.run_workload(one, outputs=["path", "endpoints_connected"])
        for rel in ("path", "endpoints_connected"):
            a = {k: v for k, v in _dict(full.relations[rel]).items() if k[0] == s}
            assert a == _dict(r1.relations[rel])
        part = oracle.run_workload(w, samples=[s], outputs=["path"])
        assert _dict(part.relations["path"]) == {k: v for k, v in _dict(full.relations["path"]).items() if k[0] == s}


def test_duplicate_facts_merged(oracle_lib):
    """Reading 16: duplicate input tuples are ⊕-merged; max-mult keeps larger p, then smaller id."""
    cols = [np.array([0, 0, 1], np.int32), np.array([1, 1, 2], np.int32)]
    for sr, exp in ((1, 0.75), (2, 1.25), (3, 0.75)):
        f = W.Facts(cols, np.zeros(3, np.int32), np.array([0.5, 0.75, 0.5], np.float32))
        r = oracle.run(W.PATH_PROGRAM, sr, 1, {"edge": f}).relations["path"]
        d = _dict(r)
        assert d[(0, 0, 1)] == exp
        if sr == 3:
            assert _grad(r, 0) == {1: 1.0}


@pytest.mark.parametrize("text,frag", [
    ("rel r(x) :- s(y).", "unknown relation"),
    ("type s(a: i32)\nrel r(x) :- s(y).", "unbound head variable"),
    ("type s(a: i32)\nrel r(x) :- s(x, y).", "arity"),
    ("type s(a: i32)\nrel r(x) :- s(x) $", "2:18"),
    ("type s(a: i32)\nrel r(x) :- s(x) and", "expected"),
])
def test_parse_errors(oracle_lib, text, frag):
    with pytest.raises(oracle.OracleError) as e:
        oracle.run(text, 0, 1, {})
    assert frag in str(e.value)


def test_range_errors(oracle_lib):
    f = W.Facts([np.array([0], np.int32), np.array([1], np.int32)], np.zeros(1, np.int32), np.array([1.5], np.float32))
    with pytest.raises(oracle.OracleError):
        oracle.run(W.PATH_PROGRAM, 1, 1, {"edge": f})
    f = W.Facts([np.array([0], np.int32), np.array([1], np.int32)], np.array([3], np.int32), None)
    with pytest.raises(oracle.OracleError):
        oracle.run(W.PATH_PROGRAM, 1, 2, {"edge": f})


def test_iteration_cap(oracle_lib):
    w = W.c1_workload(2)
    with pytest.raises(oracle.OracleError) as e:
        oracle.run_workload(w, max_iters=2)
    assert e.value.code == 7


def test_empty_and_self_loop(oracle_lib):
    f = W.Facts([np.zeros(0, np.int32), np.zeros(0, np.int32)], np.zeros(0, np.int32), np.zeros(0, np.float32))
    r = oracle.run(W.PATH_PROGRAM, 1, 1, {"edge": f})
    assert len(r.relations["path"]) == 0 and int(r.rounds[0]) == 1
    f = W.Facts([np.array([3], np.int32), np.array([3], np.int32)], np.zeros(1, np.int32), np.array([0.5], np.float32))
    r = oracle.run(W.PATH_PROGRAM, 3, 1, {"edge": f})
    assert _dict(r.relations["path"]) == {(0, 3, 3): 0.5}
