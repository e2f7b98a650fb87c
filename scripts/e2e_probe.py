"""Time the parts of one end-to-end step (host facts -> run -> host outputs) of a
bench config: push, run, output_get(host), for diagnosing e2e vs device time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2503_21937_b200 import Engine

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = bench.CONFIGS[name]
w = bench._rank_batch(cfg["make"], cfg["per_gpu"], 0)
sr = cfg["semirings"][0]
e = Engine(w.program, sr, batch_size=cfg["per_gpu"])
hf = {r: type(f)([torch.as_tensor(c).pin_memory() for c in f.cols],
                 None if f.sample_ids is None else torch.as_tensor(f.sample_ids).pin_memory(),
                 torch.as_tensor(f.probs).pin_memory()) for r, f in w.facts.items()}
for it in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    e.push_facts(hf); torch.cuda.synchronize(); t1 = time.perf_counter()
    e.run(); torch.cuda.synchronize(); t2 = time.perf_counter()
    o = e.output(cfg["out"], device=False, copy=False); t3 = time.perf_counter()
    o2 = e.output(cfg["out"], device=False, copy=False); t4 = time.perf_counter()
    print(f"{name} it{it}: push {1e3*(t1-t0):.2f} run {1e3*(t2-t1):.2f} output {1e3*(t3-t2):.2f} (again {1e3*(t4-t3):.3f}) ms, n={o.n}", flush=True)
