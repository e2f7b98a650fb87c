"""One C2 fixpoint (diff-max-mult + max-min) for ncu launch lists / captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from paper_2503_21937_b200 import Engine, DIFF_MAX_MULT_PROB, MAX_MIN_PROB

srs = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["3"])]
w = W.c2_workload(semiring=3)
for sr in srs:
    e = Engine(w.program, sr, batch_size=64)
    e.push_facts(w.facts)
    s = e.run()
    print(sr, {k: (round(v, 3) if isinstance(v, float) else v) for k, v in s.items()}, flush=True)
    e.close()
