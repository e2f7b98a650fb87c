"""Seeded input generators for the five BASELINE.json configs.

Every generator returns a `Workload`: program text (the Datalog subset of
Fig. 3c), batch size and the input facts as columnar int32
arrays plus fp32 probabilities.  Probabilities are drawn in fp64 and rounded to
fp32.  Sample i of a batched config draws from
`SeedSequence(seed).spawn(batch)[i]`, so any single sample can be regenerated
alone (sampled parity at full size).

No method arithmetic lives here: no joins, no semiring ops, no fixpoint.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

# ---------------------------------------------------------------------------
# Programs (Fig. 3c; CLUTRR-style kinship cf. P:782-786;
# TC-shaped reachability cf. P:799-800).
# ---------------------------------------------------------------------------
PATH_PROGRAM = """
type edge(x: i32, y: i32)
rel path(x, y) :- edge(x, y) or (path(x, z) and edge(z, y)).
output path
"""

PATHFINDER_PROGRAM = """
type Cell = u32
type edge(x: Cell, y: Cell)
type is_endpoint(x: Cell)
rel path(x, y) :- edge(x, y) or (path(x, z) and edge(z, y)).
rel endpoints_connected() :- is_endpoint(x), is_endpoint(y), path(x, y), x != y.
output endpoints_connected
"""

KINSHIP_PROGRAM = """
type fact(r: i32, x: i32, y: i32)
shared type composition(r1: i32, r2: i32, r3: i32)
type query(x: i32, y: i32)
rel kinship(r, x, y) :- fact(r, x, y).
rel kinship(r3, x, z) :- kinship(r1, x, y), kinship(r2, y, z), composition(r1, r2, r3).
rel answer(r) :- query(x, z), kinship(r, x, z).
output answer
"""

REACH_PROGRAM = """
shared type edge(x: i32, y: i32)
type source(x: i32)
rel reach(y) :- source(x), edge(x, y).
rel reach(y) :- reach(x), edge(x, y).
output reach
"""

# Same Generation (Table 2: "which nodes in a directed graph
# are the same distance from a common ancestor"; 2 rules, unit).  One graph =
# one sample (batch 1); the key-partitioned multi-GPU mode (SURVEY §8(f)
# NEXT-3) splits its tuples across ranks instead of its samples.
SG_PROGRAM = """
type edge(x: i32, y: i32)
rel sg(x, y) :- edge(p, x), edge(p, y), x != y.
rel sg(x, y) :- edge(a, x), sg(a, b), edge(b, y).
output sg
"""

PROGRAMS = {
    "path": PATH_PROGRAM,
    "pathfinder": PATHFINDER_PROGRAM,
    "kinship": KINSHIP_PROGRAM,
    "reach": REACH_PROGRAM,
    "sg": SG_PROGRAM,
}

UNIT, MAX_MIN_PROB, ADD_MULT_PROB, DIFF_MAX_MULT_PROB, DIFF_MAX_MIN_PROB, DIFF_TOP1_PROOFS, DIFF_ADD_MULT_PROB = 0, 1, 2, 3, 4, 5, 6


@dataclass
class Facts:
    """Columnar facts for one input relation.

    cols: list of int32 arrays (one per column, equal length n)
    sample_ids: int32 array of length n, or None for a shared relation
    probs: float32 array of length n, or None (= 1.0)
    """
    cols: List[np.ndarray]
    sample_ids: Optional[np.ndarray]
    probs: Optional[np.ndarray]

    @property
    def n(self) -> int:
        if self.cols:
            return int(self.cols[0].shape[0])
        if self.sample_ids is not None:
            return int(self.sample_ids.shape[0])
        return 0 if self.probs is None else int(self.probs.shape[0])


@dataclass
class Workload:
    name: str
    program: str
    semiring: int
    batch_size: int
    facts: Dict[str, Facts]
    meta: dict = field(default_factory=dict)

    def n_facts(self) -> int:
        return sum(f.n for f in self.facts.values())


def _f32(x) -> np.ndarray:
    return np.asarray(x, dtype=np.float64).astype(np.float32)


def _i32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int64).astype(np.int32))


def _concat(parts: Sequence[Facts], batched: bool = True) -> Facts:
    arity = len(parts[0].cols)
    cols = [_i32(np.concatenate([p.cols[c] for p in parts])) for c in range(arity)]
    sids = _i32(np.concatenate([p.sample_ids for p in parts])) if batched else None
    probs = _f32(np.concatenate([p.probs for p in parts]))
    return Facts(cols, sids, probs)


# ---------------------------------------------------------------------------
# C1: 6-node dyadic DAG (SURVEY §8(c) worked example).
# ---------------------------------------------------------------------------
C1_EDGES = [  # (src, dst, p) — e0..e7
    (0, 1, 0.5), (0, 2, 0.25), (1, 2, 0.5), (1, 3, 0.75),
    (2, 3, 0.5), (2, 4, 0.75), (3, 5, 0.5), (4, 5, 0.25),
]


def c1_workload(semiring: int = ADD_MULT_PROB) -> Workload:
    src = _i32([e[0] for e in C1_EDGES])
    dst = _i32([e[1] for e in C1_EDGES])
    p = _f32([e[2] for e in C1_EDGES])
    facts = {"edge": Facts([src, dst], _i32(np.zeros(len(src))), p)}
    return Workload("C1", PATH_PROGRAM, semiring, 1, facts)


# ---------------------------------------------------------------------------
# C2 / C5: Pathfinder-shaped lattice G_{n,n}.
# ---------------------------------------------------------------------------
_DIRS = ((0, 1), (0, -1), (1, 0), (-1, 0))  # right, left, down, up
_OPP = (1, 0, 3, 2)


def lattice(n: int):
    """Directed lattice edges of G_{n,n}: both directions of every grid edge.

    Returns (src, dst, eid) where eid[cell, d] is the edge index of
    cell -> neighbour(d), or -1 off-grid.  |E| = 4 n (n-1).
    """
    eid = -np.ones((n * n, 4), dtype=np.int64)
    src, dst = [], []
    for r in range(n):
        for c in range(n):
            a = r * n + c
            for d, (dr, dc) in enumerate(_DIRS):
                rr, cc = r + dr, c + dc
                if 0 <= rr < n and 0 <= cc < n:
                    eid[a, d] = len(src)
                    src.append(a)
                    dst.append(rr * n + cc)
    return np.asarray(src, dtype=np.int64), np.asarray(dst, dtype=np.int64), eid


_LATTICE_CACHE: dict = {}


def _lattice_cached(n):
    if n not in _LATTICE_CACHE:
        _LATTICE_CACHE[n] = lattice(n)
    return _LATTICE_CACHE[n]


def pathfinder_sample(rng: np.random.Generator, n: int):
    """One Pathfinder-shaped sample (SURVEY §8.0 C2 value distribution).

    Background edges p~U(0.01,0.3); 2-4 random lattice walks of length 3n with
    p~U(0.85,0.99) on both directions; two endpoint cells p~U(0.9,0.99), all
    other cells U(0,0.05).  Positive (50%): endpoints at both ends of curve 0;
    negative: start of curve 0 and end of curve 1.
    """
    src, dst, eid = _lattice_cached(n)
    p = rng.uniform(0.01, 0.3, size=src.shape[0])
    ncurves = int(rng.integers(2, 5))
    ends = []
    for _ in range(ncurves):
        a = int(rng.integers(n * n))
        start, prev = a, -1
        for _step in range(3 * n):
            ds = [d for d in range(4) if eid[a, d] >= 0 and dst[eid[a, d]] != prev]
            d = ds[int(rng.integers(len(ds)))]
            e = eid[a, d]
            b = int(dst[e])
            p[e] = rng.uniform(0.85, 0.99)
            p[eid[b, _OPP[d]]] = rng.uniform(0.85, 0.99)
            prev, a = a, b
        ends.append((start, a))
    positive = bool(rng.random() < 0.5)
    e1 = ends[0][0]
    e2 = ends[0][1] if positive else ends[1][1]
    if e2 == e1:
        e2 = ends[1][0] if ends[1][0] != e1 else (e1 + 1) % (n * n)
    ep = rng.uniform(0.0, 0.05, size=n * n)
    ep[e1] = rng.uniform(0.9, 0.99)
    ep[e2] = rng.uniform(0.9, 0.99)
    return (src, dst, _f32(p)), (np.arange(n * n), _f32(ep)), positive


def grid_workload(n: int, batch: int, seed: int, semiring: int,
                  samples: Optional[Sequence[int]] = None, name: str = "grid",
                  program: str = PATHFINDER_PROGRAM) -> Workload:
    """Batch of Pathfinder grids. `samples` selects a subset of sample indices
    (their facts keep their global sample ids; the batch size stays `batch`)."""
    seqs = np.random.SeedSequence(seed).spawn(batch)
    idx = range(batch) if samples is None else samples
    edges, eps, labels = [], [], {}
    for i in idx:
        rng = np.random.default_rng(seqs[i])
        (s, d, p), (cells, ep), pos = pathfinder_sample(rng, n)
        edges.append(Facts([s, d], np.full(s.shape[0], i), p))
        eps.append(Facts([cells], np.full(cells.shape[0], i), ep))
        labels[int(i)] = pos
    facts = {"edge": _concat(edges)}
    if "is_endpoint" in program:
        facts["is_endpoint"] = _concat(eps)
    return Workload(name, program, semiring, batch, facts,
                    meta={"n": n, "seed": seed, "labels": labels,
                          "samples": list(idx)})


def c2_workload(semiring: int = DIFF_MAX_MULT_PROB, samples=None, n: int = 32,
                batch: int = 64) -> Workload:
    return grid_workload(n, batch, 2, semiring, samples, "C2")


def c5_workload(semiring: int = DIFF_MAX_MULT_PROB, samples=None, n: int = 64,
                batch: int = 4096) -> Workload:
    return grid_workload(n, batch, 5, semiring, samples, "C5")


# ---------------------------------------------------------------------------
# C3: CLUTRR-shaped kinship.
# ---------------------------------------------------------------------------
def c3_workload(semiring: int = ADD_MULT_PROB, samples=None, batch: int = 256,
                entities: int = 20, rtypes: int = 20, skips: int = 10,
                ncomp: int = 200, seed: int = 3) -> Workload:
    root = np.random.SeedSequence(seed)
    comp_seq, sample_seq = root.spawn(2)
    crng = np.random.default_rng(comp_seq)
    keys = crng.choice(rtypes * rtypes, size=min(ncomp, rtypes * rtypes), replace=False)
    keys.sort()
    r3 = crng.integers(0, rtypes, size=keys.shape[0])
    comp = Facts([_i32(keys // rtypes), _i32(keys % rtypes), _i32(r3)], None,
                 _f32(np.ones(keys.shape[0])))
    seqs = sample_seq.spawn(batch)
    idx = range(batch) if samples is None else samples
    fparts, qparts = [], []
    for i in idx:
        rng = np.random.default_rng(seqs[i])
        pairs = [(k, k + 1) for k in range(entities - 1)]
        cand = [(a, b) for a in range(entities) for b in range(a + 2, entities)]
        pick = rng.choice(len(cand), size=min(skips, len(cand)), replace=False)
        pairs += [cand[j] for j in sorted(pick)]
        rs, xs, ys, ps = [], [], [], []
        for (a, b) in pairs:
            logits = rng.normal(0.0, 2.0, size=rtypes)
            w = np.exp(logits - logits.max())
            w = w / w.sum()
            for r in range(rtypes):
                rs.append(r); xs.append(a); ys.append(b); ps.append(w[r])
        fparts.append(Facts([_i32(rs), _i32(xs), _i32(ys)], np.full(len(rs), i), _f32(ps)))
        qparts.append(Facts([_i32([0]), _i32([entities - 1])], np.full(1, i), _f32([1.0])))
    facts = {"fact": _concat(fparts), "composition": comp, "query": _concat(qparts)}
    return Workload("C3", KINSHIP_PROGRAM, semiring, batch, facts,
                    meta={"samples": list(idx)})


# ---------------------------------------------------------------------------
# C4: power-law reachability.
# ---------------------------------------------------------------------------
_C4_EDGE_CACHE: dict = {}


def chung_lu_edges(nodes: int, edges: int, gamma: float, seed: int):
    """Directed Chung-Lu graph: endpoints drawn independently with weight
    w_i ∝ (i+1)^(-1/(γ-1)) over a shuffled id space; self-loops and duplicate
    edges rejected until `edges` distinct edges exist."""
    key = (nodes, edges, gamma, seed)
    if key in _C4_EDGE_CACHE:
        return _C4_EDGE_CACHE[key]
    rng = np.random.default_rng(np.random.SeedSequence(seed).spawn(1)[0])
    w = (np.arange(nodes, dtype=np.float64) + 1.0) ** (-1.0 / (gamma - 1.0))
    w /= w.sum()
    perm = rng.permutation(nodes)
    seen = np.empty(0, dtype=np.int64)
    order = np.empty(0, dtype=np.int64)
    while seen.shape[0] < edges:
        need = edges - seen.shape[0]
        m = int(need * 1.3) + 1024
        u = perm[rng.choice(nodes, size=m, p=w)]
        v = perm[rng.choice(nodes, size=m, p=w)]
        ok = u != v
        k = (u[ok].astype(np.int64) * nodes + v[ok])
        allk = np.concatenate([order, k])
        _, first = np.unique(allk, return_index=True)
        first.sort()
        order = allk[first][:edges]
        seen = order
    src = order // nodes
    dst = order % nodes
    _C4_EDGE_CACHE[key] = (src, dst)
    return src, dst


def c4_workload(semiring: int = UNIT, samples=None, batch: int = 1024,
                nodes: int = 100_000, edges: int = 1_000_000, gamma: float = 2.1,
                seed: int = 4) -> Workload:
    src, dst = chung_lu_edges(nodes, edges, gamma, seed)
    outdeg = np.bincount(src, minlength=nodes)
    cands = np.nonzero(outdeg > 0)[0]
    srng = np.random.default_rng(np.random.SeedSequence(seed).spawn(2)[1])
    sources = cands[srng.integers(0, cands.shape[0], size=batch)]
    idx = np.arange(batch) if samples is None else np.asarray(list(samples), dtype=np.int64)
    facts = {
        "edge": Facts([_i32(src), _i32(dst)], None, _f32(np.ones(src.shape[0]))),
        "source": Facts([_i32(sources[idx])], _i32(idx), _f32(np.ones(idx.shape[0]))),
    }
    return Workload("C4", REACH_PROGRAM, semiring, batch, facts,
                    meta={"samples": [int(i) for i in idx], "nodes": nodes,
                          "max_outdeg": int(outdeg.max())})


# ---------------------------------------------------------------------------
# Small random graphs for oracle pins and parity cases.
# ---------------------------------------------------------------------------
def random_digraph_workload(nodes: int, p_edge: float, seed: int, semiring: int,
                            batch: int = 1, dyadic: bool = False,
                            self_loops: bool = False, program: str = PATH_PROGRAM) -> Workload:
    rng = np.random.default_rng(seed)
    parts = []
    for s in range(batch):
        m = rng.random((nodes, nodes)) < p_edge
        if not self_loops:
            np.fill_diagonal(m, False)
        a, b = np.nonzero(m)
        if dyadic:
            p = rng.integers(1, 9, size=a.shape[0]) / 8.0
        else:
            p = rng.uniform(0.05, 1.0, size=a.shape[0])
        parts.append(Facts([_i32(a), _i32(b)], np.full(a.shape[0], s), _f32(p)))
    if sum(p.n for p in parts) == 0:
        facts = {"edge": Facts([_i32([]), _i32([])], _i32([]), _f32([]))}
    else:
        facts = {"edge": _concat([p for p in parts if p.n] or parts)}
    return Workload(f"digraph{nodes}", program, semiring, batch, facts)


def random_dag_workload(nodes: int, p_edge: float, seed: int, semiring: int,
                        batch: int = 1, program: str = PATH_PROGRAM) -> Workload:
    """Edges only from lower to higher node id (a DAG; finitely many derivations)."""
    rng = np.random.default_rng(seed)
    parts = []
    for s in range(batch):
        m = np.triu(rng.random((nodes, nodes)) < p_edge, k=1)
        a, b = np.nonzero(m)
        p = rng.uniform(0.05, 1.0, size=a.shape[0])
        parts.append(Facts([_i32(a), _i32(b)], np.full(a.shape[0], s), _f32(p)))
    facts = {"edge": _concat(parts)}
    return Workload(f"dag{nodes}", program, semiring, batch, facts)


# ---------------------------------------------------------------------------
# Same Generation over a synthetic SNAP-shaped graph.
# ---------------------------------------------------------------------------
def sg_workload(nodes: int = 16384, out_degree: int = 3, seed: int = 6, semiring: int = UNIT,
                tree_levels: int = 0) -> Workload:
    """A directed graph of `nodes` nodes in which node i draws `out_degree`
    distinct successors uniformly among the nodes after it (a DAG, like a
    citation / hierarchy graph, so same-generation pairs stay finite in
    number per level).  Unit tags; one sample."""
    rng = np.random.default_rng(seed)
    src, dst = [], []
    for i in range(nodes - 1):
        k = min(out_degree, nodes - 1 - i)
        succ = i + 1 + rng.choice(nodes - 1 - i, size=k, replace=False)
        src.append(np.full(k, i))
        dst.append(np.sort(succ))
    src = np.concatenate(src)
    dst = np.concatenate(dst)
    facts = {"edge": Facts([_i32(src), _i32(dst)], np.zeros(src.shape[0], np.int32),
                           _f32(np.ones(src.shape[0])))}
    return Workload("SG", SG_PROGRAM, semiring, 1, facts, meta={"nodes": nodes, "edges": int(src.shape[0])})


def workload_by_name(name: str, semiring: Optional[int] = None, **kw) -> Workload:
    name = name.upper()
    if name == "C1":
        return c1_workload(ADD_MULT_PROB if semiring is None else semiring)
    if name == "C2":
        return c2_workload(DIFF_MAX_MULT_PROB if semiring is None else semiring, **kw)
    if name == "C3":
        return c3_workload(ADD_MULT_PROB if semiring is None else semiring, **kw)
    if name == "C4":
        return c4_workload(UNIT if semiring is None else semiring, **kw)
    if name == "C5":
        return c5_workload(DIFF_MAX_MULT_PROB if semiring is None else semiring, **kw)
    raise ValueError(name)
