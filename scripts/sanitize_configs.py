"""Small C1-C3 (and C4/C5-shaped) runs for compute-sanitizer:
every semiring, every store path, with outputs and gradients read back."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2503_21937_b200 import Engine  # noqa: E402

cases = [(W.c1_workload(sr), ["path"]) for sr in (0, 1, 2, 3, 4)]
cases += [(W.c2_workload(semiring=sr, n=8, batch=4), ["path", "endpoints_connected"]) for sr in (1, 3, 4)]
cases += [(W.c3_workload(batch=4, entities=10, rtypes=6, skips=5, ncomp=20), ["kinship", "answer"])]
# full per-sample C3 size: compacted composition rounds, split items, certified rounding (add-mult),
# and the same rounds under max-min and unit
cases += [(W.c3_workload(semiring=sr, batch=2, samples=[0, 1]), ["kinship", "answer"]) for sr in (2, 1, 0)]
cases += [(W.c4_workload(batch=4, nodes=3000, edges=20000, seed=44), ["reach"])]
cases += [(W.c5_workload(n=10, batch=4), ["endpoints_connected"])]
for w, outs in cases:
    e = Engine(w.program, w.semiring, batch_size=w.batch_size)
    e.push_facts(w.facts)
    st = e.run()
    for o in outs:
        r = e.output(o)
        print(w.name, w.semiring, o, r.n, st["rounds_total"], flush=True)
    e.close()
print("sanitize cases done")
