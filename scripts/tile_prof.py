"""C3-shaped batch through the tile path, repeated in one process (the first
run includes the NVRTC compile of the plan): ms per run, candidates, rounds."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time
import workloads as W
from paper_2503_21937_b200 import Engine
b = int(sys.argv[1]) if len(sys.argv) > 1 else 32
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = W.c3_workload(batch=b, samples=list(range(b)))
e = Engine(w.program, 2, batch_size=b)
for _ in range(reps):
    t = time.time()
    e.push_facts(w.facts)
    s = e.run()
    print(f"ms_total {s['ms_total']:.2f} wall {1000 * (time.time() - t):.1f} cands {s['candidates']} rounds {s['rounds_total']} "
          f"tiles {s['tile_strata']}", flush=True)
