"""C3 (first 8 samples of the batch, full per-sample size) through the tile
path with LOBSTER_TILE_TRACE=1: per round candidates, |Δ'|, the U phase and
the longest single head item in cycles / 16 (stderr)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["LOBSTER_TILE_TRACE"] = "1"
import workloads as W
from paper_2503_21937_b200 import Engine
w = W.c3_workload(batch=8, samples=list(range(8)))
e = Engine(w.program, 2, batch_size=8)
e.push_facts(w.facts)
print(e.run())
