"""Does running the two C2 fixpoints (max-min, diff-max-mult) on two streams from two
host threads overlap usefully?  Device time of sequential vs concurrent steps."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import workloads as W
from paper_2503_21937_b200 import Engine

cfg = bench.CONFIGS["C2"]
w = bench._rank_batch(cfg["make"], cfg["per_gpu"], 0)
dev = torch.device("cuda", 0)
df = {r: W.Facts([torch.as_tensor(c).to(dev) for c in f.cols],
                 None if f.sample_ids is None else torch.as_tensor(f.sample_ids).to(dev),
                 torch.as_tensor(f.probs).to(dev)) for r, f in w.facts.items()}
streams = {sr: torch.cuda.Stream() for sr in cfg["semirings"]}
eng_seq = {sr: Engine(w.program, sr, batch_size=cfg["per_gpu"]) for sr in cfg["semirings"]}
eng_con = {sr: Engine(w.program, sr, batch_size=cfg["per_gpu"], stream=streams[sr].cuda_stream)
           for sr in cfg["semirings"]}


def seq():
    for sr, e in eng_seq.items():
        e.push_facts(df); e.run()


def con():
    e0 = torch.cuda.Event()
    e0.record()
    def one(sr):
        with torch.cuda.stream(streams[sr]):
            streams[sr].wait_event(e0)
            eng_con[sr].push_facts(df); eng_con[sr].run()
    ts = [threading.Thread(target=one, args=(sr,)) for sr in eng_con]
    for t in ts: t.start()
    for t in ts: t.join()
    for s in streams.values():
        torch.cuda.current_stream().wait_stream(s)


for name, fn in (("seq", seq), ("con", con), ("seq", seq), ("con", con)):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): fn()
    b.record(); torch.cuda.synchronize()
    print(name, round(a.elapsed_time(b) / 5, 2), "ms per step", flush=True)
