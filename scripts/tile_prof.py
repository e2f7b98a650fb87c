"""C3-shaped batch through the tile path (for ncu captures of tile_fixpoint_k)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
from paper_2503_21937_b200 import Engine
b = int(sys.argv[1]) if len(sys.argv) > 1 else 32
w = W.c3_workload(batch=b, samples=list(range(b)))
e = Engine(w.program, 2, batch_size=b)
e.push_facts(w.facts)
s = e.run()
print(s["ms_total"], s["candidates"], s["rounds_total"], s["tile_strata"])
