"""Time the parts of one bench step (device-resident facts) of a config:
push, run, output(device), backward — host wall with a sync after each."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import workloads as W
from paper_2503_21937_b200 import DIFF_MAX_MULT_PROB, Engine

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = bench.CONFIGS[name]
w = bench._rank_batch(cfg["make"], cfg["per_gpu"], 0)
dev = torch.device("cuda", 0)
df = {r: W.Facts([torch.as_tensor(c).to(dev) for c in f.cols],
                 None if f.sample_ids is None else torch.as_tensor(f.sample_ids).to(dev),
                 torch.as_tensor(f.probs).to(dev)) for r, f in w.facts.items()}
engines = {sr: Engine(w.program, sr, batch_size=cfg["per_gpu"]) for sr in cfg["semirings"]}
g = torch.zeros(w.n_facts(), dtype=torch.float32, device=dev)
for it in range(5):
    tt = {}
    for sr, e in engines.items():
        torch.cuda.synchronize(); t0 = time.perf_counter()
        e.push_facts(df); torch.cuda.synchronize(); t1 = time.perf_counter()
        e.run(); torch.cuda.synchronize(); t2 = time.perf_counter()
        tt[f"push{sr}"] = 1e3 * (t1 - t0); tt[f"run{sr}"] = 1e3 * (t2 - t1)
    if DIFF_MAX_MULT_PROB in engines:
        e = engines[DIFF_MAX_MULT_PROB]
        torch.cuda.synchronize(); t0 = time.perf_counter()
        o = e.output(cfg["out"], device=True); torch.cuda.synchronize(); t1 = time.perf_counter()
        g.zero_(); e.backward(cfg["out"], torch.ones(o.n, dtype=torch.float32, device=dev), g)
        torch.cuda.synchronize(); t2 = time.perf_counter()
        tt["output"] = 1e3 * (t1 - t0); tt["backward"] = 1e3 * (t2 - t1)
    print(name, {k: round(v, 3) for k, v in tt.items()}, flush=True)
