"""One fixpoint per semiring of a bench.py config (default C3), for ncu launch
lists / captures and LOBSTER_LOG=1 traces.  usage: profile_cfg.py C3 [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2503_21937_b200 import Engine

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = bench.CONFIGS[name]
w = bench._rank_batch(cfg["make"], cfg["per_gpu"], 0)
for sr in cfg["semirings"]:
    e = Engine(w.program, sr, batch_size=cfg["per_gpu"])
    for _ in range(reps):
        e.push_facts(w.facts)
        s = e.run()
    print(name, sr, {k: (round(v, 3) if isinstance(v, float) else v) for k, v in s.items()}, flush=True)
    e.close()
