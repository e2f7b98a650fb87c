"""Independent reference computations that pin the oracle (SURVEY §8(c)
"What pins each part").  Textbook algorithms written directly in numpy /
Python; none of them shares code with the oracle or the CUDA path."""
from __future__ import annotations

import heapq
import itertools
import math
from fractions import Fraction

import numpy as np


def edge_lists(w, sample=0):
    f = w.facts["edge"]
    m = np.ones(f.n, dtype=bool) if f.sample_ids is None else (f.sample_ids == sample)
    return (f.cols[0][m].astype(np.int64), f.cols[1][m].astype(np.int64),
            (f.probs[m] if f.probs is not None else np.ones(m.sum(), np.float32)),
            np.nonzero(m)[0])


def floyd_warshall(n, src, dst, p, kind):
    """Closure over paths of length >= 1 (no reflexive init).
    kind: 'bool' | 'maxmin' | 'maxmul'.  Values in fp32 ops for maxmin,
    float64 for maxmul (caller compares with a tolerance unless inputs are
    powers of two)."""
    if kind == "bool":
        A = np.zeros((n, n), dtype=bool)
        A[src, dst] = True
        for k in range(n):
            A = A | (A[:, k:k + 1] & A[k:k + 1, :])
        return A
    A = np.zeros((n, n), dtype=np.float64)
    for s, d, q in zip(src, dst, p):  # duplicate edges: ⊕ = max
        A[s, d] = max(A[s, d], float(q))
    for k in range(n):
        if kind == "maxmin":
            A = np.maximum(A, np.minimum(A[:, k:k + 1], A[k:k + 1, :]))
        else:
            A = np.maximum(A, A[:, k:k + 1] * A[k:k + 1, :])
    return A


def addmult_closed_form(n, src, dst, p):
    """Σ_{k≥1} A^k = (I−A)^{-1} − I for a DAG (A nilpotent), fp64."""
    A = np.zeros((n, n), dtype=np.float64)
    for s, d, q in zip(src, dst, p):
        A[s, d] += float(q)
    return np.linalg.inv(np.eye(n) - A) - np.eye(n)


def simple_paths(n, adj, x, y):
    """All simple paths x -> y of length >= 1 as lists of edge indices.  For
    x == y: simple cycles through x.  adj[u] = list of (v, edge_index)."""
    out = []

    def rec(u, seen, path):
        for v, e in adj[u]:
            if v == y:
                out.append(path + [e])
            if v not in seen and v != y:
                rec(v, seen | {v}, path + [e])

    rec(x, {x}, [])
    return out


def all_paths_dag(n, adj, x, y):
    out = []

    def rec(u, path):
        for v, e in adj[u]:
            if v == y:
                out.append(path + [e])
            rec(v, path + [e])

    rec(x, [])
    return out


def make_adj(n, src, dst):
    adj = [[] for _ in range(n)]
    for i, (s, d) in enumerate(zip(src, dst)):
        adj[int(s)].append((int(d), i))
    return adj


def bfs_reach(nodes, src, dst, source):
    """Nodes reachable from `source` by a path of length >= 1."""
    order = np.argsort(src, kind="stable")
    s_sorted = src[order]
    d_sorted = dst[order]
    start = np.searchsorted(s_sorted, np.arange(nodes + 1))
    seen = np.zeros(nodes, dtype=bool)
    frontier = [int(source)]
    first = True
    while frontier:
        nxt = []
        for u in frontier:
            for v in d_sorted[start[u]:start[u + 1]]:
                if not seen[v]:
                    seen[v] = True
                    nxt.append(int(v))
        frontier = nxt
        first = False
    return np.nonzero(seen)[0]


def dijkstra_maxmul(n, src, dst, p, x):
    """max over paths (length >= 1) of Π p, via Dijkstra on -log p (fp64)."""
    w = {}
    for s, d, q in zip(src, dst, p):
        s, d, q = int(s), int(d), float(q)
        if q > 0:
            w[(s, d)] = min(w.get((s, d), math.inf), -math.log(q))
    adj = [[] for _ in range(n)]
    for (s, d), c in w.items():
        adj[s].append((d, c))
    best = np.full(n, math.inf)
    h = []
    for d, c in adj[x]:  # length >= 1: start from x's out-edges
        if c < best[d]:
            best[d] = c
            heapq.heappush(h, (c, d))
    while h:
        c, u = heapq.heappop(h)
        if c > best[u]:
            continue
        for v, cw in adj[u]:
            if c + cw < best[v]:
                best[v] = c + cw
                heapq.heappush(h, (c + cw, v))
    return np.exp(-best)  # inf -> 0 (unreachable or product 0)


def kleene_naive_tc(n, src, dst, p, kind, max_rounds=10_000):
    """Naive Kleene iteration of path = edge ∪ path∘edge on full relations
    (S:608): P_{t+1} = E ⊕ (P_t ⊗ E) until P stops changing.  add-mult on a
    DAG gives the height-bounded derivation sum, which converges."""
    E = np.zeros((n, n), dtype=np.float64)
    has = np.zeros((n, n), dtype=bool)
    for s, d, q in zip(src, dst, p):
        has[s, d] = True
        if kind == "addmul":
            E[s, d] += float(q)
        else:
            E[s, d] = max(E[s, d], float(q))
    P = np.zeros_like(E)
    Ph = np.zeros_like(has)
    for _ in range(max_rounds):
        if kind == "addmul":
            N = E + P @ E
        elif kind == "maxmin":
            N = np.maximum(E, np.max(np.minimum(P[:, :, None], E[None, :, :]), axis=1))
        else:  # bool
            N = np.zeros_like(E)
        Nh = has | ((Ph.astype(np.int64) @ has.astype(np.int64)) > 0)
        if np.array_equal(N, P) and np.array_equal(Nh, Ph):
            break
        P, Ph = N, Nh
    return Ph, P


def kinship_interval_dp(E, R, facts, comp):
    """Closed form for the CLUTRR-shaped program on forward-pair inputs (a DAG
    over entity order): K(r,a,c) = fact(r,a,c) + Σ_b Σ_{comp(r1,r2)=r}
    K(r1,a,b)·K(r2,b,c), computed by increasing span c-a, in fp64.
    facts: dict (r,a,c) -> p; comp: dict (r1,r2) -> r3."""
    K = np.zeros((R, E, E), dtype=np.float64)
    for (r, a, c), q in facts.items():
        K[r, a, c] += q
    by_r3 = {}
    for (r1, r2), r3 in comp.items():
        by_r3.setdefault(r3, []).append((r1, r2))
    for span in range(2, E):
        for a in range(0, E - span):
            c = a + span
            for b in range(a + 1, c):
                for r3, pairs in by_r3.items():
                    s = 0.0
                    for r1, r2 in pairs:
                        s += K[r1, a, b] * K[r2, b, c]
                    K[r3, a, c] += s
    return K


def exact_c1_bruteforce(edges):
    """C1 by enumerating every path of the DAG in exact rationals:
    add-mult = Σ_paths Π p; max-min = max_paths min p; max-mult = max Π p."""
    n = 1 + max(max(s, d) for s, d, _ in edges)
    adj = [[] for _ in range(n)]
    for i, (s, d, q) in enumerate(edges):
        adj[s].append((d, i))
    res = {}
    for x in range(n):
        for y in range(n):
            paths = all_paths_dag(n, adj, x, y)
            if not paths:
                continue
            ps = [[Fraction(edges[e][2]).limit_denominator(1 << 20) for e in path] for path in paths]
            am = sum(math.prod(q) for q in ps)
            mm = max(min(q) for q in ps)
            mx = max(math.prod(q) for q in ps)
            res[(x, y)] = (am, mm, mx, paths, ps)
    return res
