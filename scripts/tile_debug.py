"""Tile-path (k_tile.cu) parity probes on small programs: which rule shapes
differ from the oracle (prints per case: tuples, tags differing, rounds)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import workloads as W  # noqa: E402
from paper_2503_21937_b200 import Engine  # noqa: E402

PROGS = {
    "tc": W.PATH_PROGRAM,
    "nonlinear": """
type edge(x: i32, y: i32)
rel path(x, y) :- edge(x, y) or (path(x, z) and path(z, y)).
output path
""",
    "twohop": """
type edge(x: i32, y: i32)
rel path(x, y) :- edge(x, y).
rel path(x, w) :- path(x, y), edge(y, z), edge(z, w).
output path
""",
}


def cmp(name, w, rel, sr):
    eng = Engine(w.program, sr, batch_size=w.batch_size)
    eng.push_facts(w.facts)
    st = eng.run()
    o = eng.output(rel)
    res = oracle.run(w.program, sr, w.batch_size, w.facts, outputs=[rel])
    r = res.relations[rel]
    g = {(int(s),) + tuple(int(c[i]) for c in o.cols): float(p) for i, (s, p) in enumerate(zip(o.sample_ids, o.probs if o.probs is not None else np.zeros(o.n, np.float32)))}
    q = {(int(s),) + tuple(int(v) for v in c): float(t) for s, c, t in zip(r.sample_ids, r.cols, r.tags)}
    diff = [k for k in q if k in g and np.float32(g[k]).view(np.uint32) != np.float32(q[k]).view(np.uint32)]
    print(f"{name:12s} sr={sr} tiles={st['tile_strata']} gpu={len(g)} oracle={len(q)} "
          f"missing={len(set(q) - set(g))} extra={len(set(g) - set(q))} tagdiff={len(diff)} "
          f"rounds gpu={st['rounds_total']} oracle={int(res.rounds.sum())} cands={st['candidates']}", flush=True)
    for k in diff[:3]:
        print("   ", k, g[k], q[k])


for sr in (0, 1, 2):
    for name, prog in PROGS.items():
        mk = W.random_dag_workload if sr == 2 else W.random_digraph_workload
        w = mk(14, 0.2, 5, sr, batch=2, program=prog)
        cmp(name, w, "path", sr)
    w = W.c3_workload(semiring=sr, batch=2, entities=6, rtypes=3, skips=3, ncomp=5)
    cmp("c3small", w, "kinship", sr)
    w = W.c3_workload(semiring=sr, batch=6, entities=10, rtypes=6, skips=5, ncomp=20)
    cmp("c3reduced", w, "kinship", sr)
