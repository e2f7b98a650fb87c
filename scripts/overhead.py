"""Where does a C2 step's time go?  Host-timed push / run / output per semiring."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from paper_2503_21937_b200 import Engine, MAX_MIN_PROB, DIFF_MAX_MULT_PROB
w = W.c2_workload(semiring=3)
dev = torch.device("cuda", 0)
dfacts = {r: W.Facts([torch.as_tensor(c).to(dev) for c in f.cols], torch.as_tensor(f.sample_ids).to(dev),
                     torch.as_tensor(f.probs).to(dev)) for r, f in w.facts.items()}
engs = {sr: Engine(w.program, sr, batch_size=64) for sr in (MAX_MIN_PROB, DIFF_MAX_MULT_PROB)}
for it in range(4):
    for sr, e in engs.items():
        torch.cuda.synchronize(); t0 = time.perf_counter()
        e.push_facts(dfacts)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        s = e.run()
        torch.cuda.synchronize(); t2 = time.perf_counter()
        ph = s["ms_join"] + s["ms_merge"] + s["ms_grad"] + s["ms_sort"] + s["ms_reduce"]
        if it == 3:
            print(f"sr={sr} push {1e3*(t1-t0):.2f} ms  run(host) {1e3*(t2-t1):.2f} ms  run(events) {s['ms_total']:.2f}  "
                  f"phases {ph:.2f}  rounds {s['rounds_total']} fj {s['ms_fused_join']:.2f} merge {s['ms_merge']:.2f}")
