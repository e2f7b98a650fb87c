"""Timing / parity probe of diff-top-1-proofs at Pathfinder scale."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
from paper_2503_21937_b200 import Engine

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 64
w = W.c2_workload(semiring=5, n=n, batch=batch)
for rep in range(3):
    e = Engine(w.program, 5, batch_size=batch)
    e.push_facts(w.facts)
    t = time.perf_counter()
    st = e.run()
    dt = time.perf_counter() - t
    print(f"n={n} batch={batch} rep={rep}: {dt*1e3:.1f} ms, rounds {st['rounds_total']}, tuples {st['tuples_derived']}, "
          f"cands {st['candidates']}", flush=True)
    e.close()
if len(sys.argv) > 3:
    import oracle
    from tests.gpu_util import assert_parity
    e = Engine(w.program, 5, batch_size=batch)
    e.push_facts(w.facts)
    e.run()
    samples = [0, batch - 1]
    res = oracle.run(w.program, 5, batch, w.facts, outputs=["path", "endpoints_connected"], samples=samples)
    assert_parity(e, res, "path", 5, samples=samples)
    assert_parity(e, res, "endpoints_connected", 5, samples=samples)
    print("parity ok on samples", samples)
