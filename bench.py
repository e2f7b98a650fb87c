#!/usr/bin/env python
"""Benchmark: derived tuples/s of the semi-naive fixpoint.

Default workload = config C2 (BASELINE.json configs[1]: Pathfinder-shaped 32x32
grids, batch 64 per GPU, max-min-prob and diff-max-mult-prob with input-fact
gradients).  `--config C1|C3|C4|C5` measures the other BASELINE configs the
same way (C5 = the 512-sample per-GPU shard of the 4096 batch).

One step = one pass of the whole hot path over one
batch: ingest (facts already in HBM) -> fixpoint under each of the config's
semirings -> (diff-max-mult) witness walk + gradients -> dense dL/dp
contraction; with N > 1 ranks also the NCCL all-gather of per-sample output
records and the all-reduce of the input-fact gradient.  Weak scaling: every
rank owns its own samples.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl lobster|reference]

Prints one JSON line (rank 0).  See DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from workloads import gen as G  # noqa: E402

METRIC = "derived tuples/s"
UNIT = "tuples/s"


def _rank_batch(make, per_gpu, rank):
    """This rank's samples with their GLOBAL ids [per_gpu*rank, per_gpu*(rank+1))
    (the shard the library assigns to `rank` of a per_gpu*world batch)."""
    samples = list(range(per_gpu * rank, per_gpu * (rank + 1)))
    w = make(per_gpu * (rank + 1), samples)
    lo = per_gpu * rank
    for f in w.facts.values():  # generators without a sample selector (C1) start at 0
        if f.sample_ids is not None and f.n and int(np.min(f.sample_ids)) < lo:
            f.sample_ids = (np.asarray(f.sample_ids) + lo).astype(np.int32)
    return w


CONFIGS = {
    "C2": dict(per_gpu=64, semirings=[G.MAX_MIN_PROB, G.DIFF_MAX_MULT_PROB], out="endpoints_connected",
               make=lambda b, s: G.grid_workload(32, b, 2, G.DIFF_MAX_MULT_PROB, samples=s, name="C2"),
               desc="C2: Pathfinder-shaped 32x32 lattice connectivity (Fig. 3c program), batch 64 per GPU, "
                    "max-min-prob + diff-max-mult-prob with input-fact gradients"),
    "C2P": dict(per_gpu=64, semirings=[G.DIFF_TOP1_PROOFS], out="endpoints_connected",
                make=lambda b, s: G.grid_workload(32, b, 2, G.DIFF_TOP1_PROOFS, samples=s, name="C2P"),
                desc="C2 under the paper's own Pathfinder provenance (P:290): diff-top-1-proofs, proofs of "
                     "<= 300 facts with input-fact gradients, 32x32 lattice, batch 64 per GPU"),
    "C1": dict(per_gpu=1, semirings=[G.ADD_MULT_PROB], out="path",
               make=lambda b, s: G.c1_workload(G.ADD_MULT_PROB),
               desc="C1: transitive closure over the 6-node dyadic DAG, add-mult-prob (latency-bound)"),
    "C3": dict(per_gpu=256, semirings=[G.ADD_MULT_PROB], out="answer",
               make=lambda b, s: G.c3_workload(G.ADD_MULT_PROB, samples=s, batch=b),
               desc="C3: CLUTRR-shaped kinship composition, 20 entities x 20 relation types, batch 256 per GPU, "
                    "add-mult-prob"),
    "C4": dict(per_gpu=1024, semirings=[G.UNIT], out="reach",
               make=lambda b, s: G.c4_workload(G.UNIT, samples=s, batch=b),
               desc="C4: unit reachability over a shared 100k-node / 1M-edge Chung-Lu graph, 1024 sources per GPU"),
    # one graph split by key across the ranks: strong scaling
    "SG": dict(per_gpu=1, semirings=[G.UNIT], out="sg", partition=True,
               make=lambda b, s: G.sg_workload(nodes=16384, out_degree=3, seed=6),
               cpu_make=lambda: G.sg_workload(nodes=2048, out_degree=3, seed=6),
               desc="Same Generation (P:756, P:802-803) over a fe-sphere-sized synthetic DAG (16384 nodes, "
                    "49149 edges), unit; N > 1: key-partitioned across the ranks (NCCL all-to-all per round)"),
    "C5": dict(per_gpu=512, semirings=[G.DIFF_MAX_MULT_PROB], out="endpoints_connected",
               make=lambda b, s: G.grid_workload(64, b, 5, G.DIFF_MAX_MULT_PROB, samples=s, name="C5"),
               desc="C5: 64x64 lattice connectivity, 512 samples per GPU (the 8-GPU shard of the 4096 batch), "
                    "diff-max-mult-prob with input-fact gradients"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="lobster", choices=["lobster", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--serial", action="store_true",
                    help="run the config's semiring fixpoints one after another instead of on two streams")
    return ap.parse_args()


def spawn_ranks(n):
    """`--gpus N` without a torchrun environment: launch N ranks of this script
    (one per GPU) through torch.distributed.run on 127.0.0.1 and wait."""
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: NVML every
    10 ms (pynvml), else nvidia-smi (~5 per second)."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(device))
            self._sample_nvml()  # the first queries are slow (~0.1 s): take them before the timed region
            self.rows.clear()
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv, h = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        flags = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                 nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        self.rows.append([str(self.device), str(sm), str(mx), "", ""] +
                         ["Active" if bits & f else "Not Active" for f in flags])

    def _loop(self):
        while not self._stop.is_set():
            try:
                if self._nvml is not None:
                    self._sample_nvml()
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                self._nvml = None
            self._stop.wait(0.01 if self._nvml is not None else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._loop, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = self.NAMES
        reasons = set()
        for r in self.rows:
            for k, nm in enumerate(names):
                if len(r) > 5 + k and r[5 + k].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows),
                "source": "nvml (10 ms)" if self._nvml is not None else "nvidia-smi"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


# ------------------------------------------------------------ cpu baseline
def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(cfg_name: str, threads: int, sr_indices=None, nsamples: int = 0):
    """The oracle, as it stands, on a bounded sample of the config's workload:
    `nsamples` samples (default one per thread, at most the per-GPU batch)
    under each listed semiring of the config, samples in parallel on
    `threads` host threads.  Returns (tuples, seconds, description)."""
    import oracle
    cfg = CONFIGS[cfg_name]
    srs = [cfg["semirings"][i] for i in (sr_indices if sr_indices is not None else range(len(cfg["semirings"])))]
    n = nsamples or max(1, min(threads, cfg["per_gpu"]))
    if cfg_name == "C4":
        n = min(n, 8)
    # the config's semirings run concurrently (the oracle's ctypes calls release
    # the GIL), the threads split between them, so that the sample stays at
    # roughly one oracle sample's wall time (~30 s on C2) instead of one per semiring
    per = max(1, threads // len(srs)) if len(srs) > 1 and n > 1 else threads
    n = max(1, min(n, per)) if per < threads else n
    w = cfg["cpu_make"]() if "cpu_make" in cfg else cfg["make"](cfg["per_gpu"], list(range(n)))
    if cfg_name == "C1":
        n = 1
    reps = 200 if cfg_name == "C1" else 1  # C1 is one 14-tuple problem: repeat it
    counts = [0] * len(srs)

    def one(k):
        for _ in range(reps):
            res = oracle.run(w.program, srs[k], w.batch_size, w.facts, samples=list(range(n)), threads=per)
            counts[k] += sum(len(r) for r in res.relations.values())

    t = time.perf_counter()
    if len(srs) > 1 and per < threads:
        import threading
        ths = [threading.Thread(target=one, args=(k,)) for k in range(len(srs))]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
    else:
        for k in range(len(srs)):
            one(k)
    dt = time.perf_counter() - t
    tuples = sum(counts)
    names = {0: "unit", 1: "max-min-prob", 2: "add-mult-prob", 3: "diff-max-mult-prob", 4: "diff-max-min-prob",
             5: "diff-top-1-proofs"}
    what = (f"{n} of the {cfg['per_gpu']} {cfg_name} samples" if "cpu_make" not in cfg else
            f"the {cfg_name} program on a {w.meta.get('nodes')}-node graph of the same generator")
    how = (f" concurrently, {per} thread(s) each" if len(srs) > 1 and per < threads else f" on {threads} thread(s)")
    return tuples, dt, (f"{what} under {' + '.join(names[x] for x in srs)}" + how
                        + (f", repeated {reps}x" if reps > 1 else ""))


def run_reference(args):
    """--impl reference: the oracle (CPU), as it stands, on a bounded sample of
    the config per step; rank 0 only (other ranks exit without work)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    cores = os.cpu_count() or 1
    threads = max(1, min(cores, cfg["per_gpu"]))
    nsr = len(cfg["semirings"])
    for i in range(args.warmup):  # warm-up: load and exercise the oracle library (C1-sized, ms)
        cpu_baseline("C1", 1, [-1], 1)
    tot_t, tot_tuples, desc = 0.0, 0, ""
    if "cpu_make" not in cfg and args.config != "C1" and (args.steps + nsr - 1) // nsr <= cfg["per_gpu"]:
        # the K steps' units — step i = sample i // S under semiring i % S — run
        # concurrently on the host cores (the config's semirings side by side,
        # the cores split between them): one oracle sample takes ~26 s on C2,
        # so K sequential steps took K x that (round 1: 571 s for K = 20)
        import threading
        import oracle
        per = max(1, cores // nsr)
        units = {k: [i // nsr for i in range(args.steps) if i % nsr == k] for k in range(nsr)}
        alls = sorted({x for u in units.values() for x in u})
        w = cfg["make"](cfg["per_gpu"], alls)
        counts = [0] * nsr

        def one(k):
            if units[k]:
                res = oracle.run(w.program, cfg["semirings"][k], w.batch_size, w.facts, samples=units[k], threads=per)
                counts[k] = sum(len(r) for r in res.relations.values())

        t0 = time.perf_counter()
        ths = [threading.Thread(target=one, args=(k,)) for k in range(nsr)]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        tot_t = time.perf_counter() - t0
        tot_tuples = sum(counts)
        threads = per * nsr
        names = {0: "unit", 1: "max-min-prob", 2: "add-mult-prob", 3: "diff-max-mult-prob", 4: "diff-max-min-prob",
                 5: "diff-top-1-proofs"}
        desc = (f"{args.steps} steps = {args.steps} (sample, semiring) units of the {args.config} batch (step i: "
                f"sample i // {nsr} under {' / '.join(names[x] for x in cfg['semirings'])} by i % {nsr}), run "
                f"concurrently, {per} thread(s) per semiring, {tot_t:.1f} s wall")
    else:
        for i in range(args.steps):
            tuples, dt, desc = cpu_baseline(args.config, threads, [i % nsr])
            tot_t += dt
            tot_tuples += tuples
        desc += "; semirings alternate by step"
    v = tot_tuples / tot_t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {"workload": cfg["desc"], "global_batch": cfg["per_gpu"]},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "cpu_model": cpu_model(), "sample": desc},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- lobster
def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    from paper_2503_21937_b200 import DIFF_MAX_MIN_PROB, DIFF_MAX_MULT_PROB, DIFF_TOP1_PROOFS, Engine, Group, _lib
    from paper_2503_21937_b200 import dist as D

    cfg = CONFIGS[args.config]
    per_gpu = cfg["per_gpu"]
    ws, rank, local = dist_env()
    # LOBSTER_BENCH_BACKEND=gloo + LOBSTER_BENCH_ONE_DEVICE=1: every rank on cuda:0 with
    # gloo collectives — exercises the multi-rank path on a one-GPU box (not a measurement)
    if os.environ.get("LOBSTER_BENCH_ONE_DEVICE"):
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    backend = os.environ.get("LOBSTER_BENCH_BACKEND", "nccl")
    if ws > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", init_method="env://", device_id=dev)
        else:
            dist.init_process_group(backend, init_method="env://")
    L = _lib.load()
    part = bool(cfg.get("partition"))  # key-partitioned: every rank holds the whole input
    gbatch = per_gpu if part else per_gpu * ws
    lo = 0 if part else per_gpu * rank  # == dist.shard(gbatch, rank, ws)[0]

    w = cfg["make"](per_gpu, None) if part else _rank_batch(cfg["make"], per_gpu, rank)
    # device-resident inputs (value) and pinned host inputs (e2e)
    dfacts, hfacts, h2d = {}, {}, 0
    for rel, f in w.facts.items():
        cols_d = [torch.as_tensor(c).to(dev) for c in f.cols]
        cols_h = [torch.as_tensor(c).pin_memory() for c in f.cols]
        s_d = None if f.sample_ids is None else torch.as_tensor(f.sample_ids).to(dev)
        s_h = None if f.sample_ids is None else torch.as_tensor(f.sample_ids).pin_memory()
        p_d = torch.as_tensor(f.probs).to(dev)
        p_h = torch.as_tensor(f.probs).pin_memory()
        dfacts[rel] = W.Facts(cols_d, s_d, p_d)
        hfacts[rel] = W.Facts(cols_h, s_h, p_h)
        h2d += sum(c.numel() * 4 for c in cols_h) + (0 if s_h is None else s_h.numel() * 4) + p_h.numel() * 4
    h2d *= len(cfg["semirings"])  # pushed once per semiring

    # independent fixpoints (one per semiring) overlap on their own streams,
    # each driven by its own host thread (the ctypes calls release the GIL)
    overlap = len(cfg["semirings"]) > 1 and not args.serial
    streams = {sr: (torch.cuda.Stream(device=dev) if overlap else torch.cuda.current_stream(dev))
               for sr in cfg["semirings"]}
    engines = {sr: Engine(w.program, sr, batch_size=gbatch, device=local, rank=0 if part else rank,
                          world_size=1 if part else ws, stream=streams[sr].cuda_stream if overlap else None)
               for sr in cfg["semirings"]}
    group = None
    if part and ws > 1:  # NCCL group of the ranks; the id travels over torch.distributed
        uid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(Group.nccl_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        group = Group.nccl(bytes(uid.cpu().numpy().tobytes()), rank, ws, local)
        for e in engines.values():
            e.partition(group, rank)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    nfacts = w.n_facts()
    rel = cfg["out"]
    arity0 = rel in ("endpoints_connected",)
    grad_local = torch.zeros(nfacts, dtype=torch.float32, device=dev)
    layout = D.fact_layout(w.facts, device=dev) if ws > 1 else None
    grad_global = torch.zeros(layout.total if layout else nfacts, dtype=torch.float32, device=dev)

    def run_one(sr, facts, host_out, box):
        try:
            _run_one(sr, facts, host_out, box)
        except BaseException as e:  # surfaced by step() on the main thread
            box[("error", sr)] = e

    def _run_one(sr, facts, host_out, box):
        eng = engines[sr]
        with torch.cuda.stream(streams[sr]):
            eng.push_facts(facts)
            st = eng.run()
            d2h = 0
            if sr in (DIFF_MAX_MULT_PROB, DIFF_MAX_MIN_PROB, DIFF_TOP1_PROOFS):
                out_dev = eng.output(rel, device=True)
                grad_local.zero_()
                eng.backward(rel, torch.ones(out_dev.n, dtype=torch.float32, device=dev), grad_local)
                if ws > 1:
                    box["rec"] = D.arity0_records(out_dev.sample_ids, out_dev.probs, lo, per_gpu, device=dev)
            if host_out:  # e2e: results back to the host through the C ABI
                o = eng.output(rel, device=False, copy=False)  # pinned host views (valid until next run)
                d2h += o.n * 4 * (1 + o.arity) + o.sample_offsets.nbytes
                if o.probs is not None:
                    d2h += o.probs.nbytes
                if o.grad_values is not None:
                    d2h += o.grad_offsets.nbytes + o.grad_fact_ids.nbytes + o.grad_values.nbytes
            box[sr] = (st, d2h)

    def step(facts, host_out=False):
        box = {}
        main = torch.cuda.current_stream(dev)
        if overlap:
            ev = torch.cuda.Event()
            ev.record(main)
            for s_ in streams.values():
                s_.wait_event(ev)
            ths = [threading.Thread(target=run_one, args=(sr, facts, host_out, box)) for sr in engines]
            for t in ths:
                t.start()
            for t in ths:
                t.join()
            for sr in engines:
                if ("error", sr) in box:
                    raise box[("error", sr)]
                main.wait_stream(streams[sr])
        else:
            for sr in engines:
                _run_one(sr, facts, host_out, box)
        if ws > 1 and not part:  # the exchange after the fixpoint
            if any(x in engines for x in (DIFF_MAX_MULT_PROB, DIFF_MAX_MIN_PROB, DIFF_TOP1_PROOFS)):
                grad_global.zero_()
                D.scatter_grad(grad_local, layout, grad_global)
                D.all_reduce_grad(grad_global)
            rec = box.get("rec")
            if rec is None or not arity0:  # variable-size outputs: per-sample row counts
                o = engines[list(engines)[-1]].output(rel, device=True)
                rec = torch.diff(o.sample_offsets).float()
            D.records_global(D.all_gather_records(rec), gbatch, ws) if arity0 else D.all_gather_records(rec)
        return [box[sr][0] for sr in engines], sum(box[sr][1] for sr in engines)

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up: the device path and (outside the timed region) the e2e path's
    # pinned output buffers, allocated on first use
    for _ in range(max(args.warmup, 0)):
        step(dfacts)
    if not args.no_e2e:
        step(hfacts, True)
    barrier()

    def timed(facts, host_out):
        total_ms, stats_all, d2h = 0.0, [], 0
        l0 = L.lobster_kernel_launches()
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            st, d2h = step(facts, host_out)
            e1.record()
            barrier()
            total_ms += e0.elapsed_time(e1)
            stats_all.append(st)
        launches = L.lobster_kernel_launches() - l0
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        per_rank = [total_ms]
        if ws > 1:
            allt = [torch.zeros_like(t) for _ in range(ws)]
            dist.all_gather(allt, t)
            per_rank = [float(x.item()) for x in allt]
        return max(per_rank), stats_all, d2h, launches, per_rank

    with ClockSampler(local) as clk:
        total_ms, stats_all, _, launches, per_rank = timed(dfacts, False)
    e2e_ms, e2e_d2h = None, 0
    if not args.no_e2e:
        e2e_ms, _, e2e_d2h, _, _ = timed(hfacts, True)
    # Roofline pass: the dominant kernel's live CUDA-event time is taken with the
    # fixpoints serialised (overlapping streams would charge one fixpoint's
    # kernels to the other's events); same steps, same inputs, after the timed region.
    rf_stats = stats_all
    if overlap:
        was = overlap
        overlap = False
        rf_stats = []
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            rf_stats.append(step(dfacts)[0])
        barrier()
        overlap = was

    tuples_step = sum(s["tuples_derived"] for s in stats_all[-1])
    cands_step = sum(s["candidates"] for s in stats_all[-1])
    if part and ws > 1:  # each rank holds its owned tuples: the job's total is their sum
        tt = torch.tensor([tuples_step, cands_step], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(tt)
        tuples_step, cands_step = int(tt[0].item()), int(tt[1].item())
    mult = 1 if part else ws  # weak scaling: every rank did per-GPU work of the same size
    ms_step = total_ms / args.steps
    value = tuples_step * mult / (ms_step / 1000.0)
    ph = {k: sum(s[k] for s in rf_stats[-1]) for k in ("ms_join", "ms_sort", "ms_reduce", "ms_merge", "ms_grad")}
    peak, peak_src = peaks()
    # Dominant kernel: the fused row-centric join + direct ⊕ (join_rows_direct_k).
    # SURVEY §8(d) algorithmic bytes per launch = |Δ|·r_Δ (probe read) + 2·|C|·r_C
    # (candidate write + re-read for dedup), r = packed key (4 B) + tag bytes;
    # the engine times every 4th fused launch with CUDA events on its stream
    # (an event pair per launch costs ~8% of the step); bytes and time below
    # are those of exactly the timed launches.
    fj_l = sum(s["fj_timed_launches"] for st in rf_stats for s in st)
    fj_all = sum(s["fj_launches"] for st in rf_stats for s in st)
    fj_ms = sum(s["ms_fused_join"] for st in rf_stats for s in st)
    fj_b = sum(s["fj_timed_probe_rows"] * s["fj_row_bytes"] + 2 * s["fj_timed_candidates"] * s["fj_row_bytes"]
               for st in rf_stats for s in st)
    tr = ncu_traffic() if args.config == "C2" else {}
    if fj_l and fj_ms > 0:
        achieved = fj_b / fj_l / (fj_ms / fj_l / 1000.0) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": tr.get("dram_bytes_per_launch"),
                    "kernel": "join_rows_rec32_k / join_rows_direct_k (fused count-free join + ⊗ + direct ⊕ into the "
                              "dense store; the 32-bit fast path takes every C2 launch)",
                    "launches_per_step": fj_all / len(rf_stats), "timed_launches_per_step": fj_l / len(rf_stats),
                    "timing": "CUDA events on the engine stream around every 4th launch (systematic sample); "
                              "bytes and time are those of the timed launches" +
                              ("; taken over K serialised steps after the overlapped timed region" if overlap else ""),
                    "avg_launch_us": 1000.0 * fj_ms / fj_l,
                    "alg_bytes_per_launch": fj_b / fj_l,
                    "alg_bytes_def": "SURVEY §8(d): |Δ|·r + 2·|C|·r per launch, r = 4 B key + tag (8 B max-mult)",
                    "traffic_source": tr.get("source"), "peak_source": peak_src}
    else:
        bytes_alg = sum(s["bytes_algorithmic"] for s in rf_stats[-1])
        t_alg = max(1e-9, sum(ph[k] for k in ("ms_join", "ms_sort", "ms_reduce", "ms_merge")) / 1000.0)
        achieved = bytes_alg / t_alg / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": None, "kernel": "fixpoint phases (SURVEY §8(d) B_alg / summed phase time)",
                    "peak_source": peak_src}
        # the same phases under SURVEY §8(d)'s per-candidate model (|Δ|·r + 2|C|·r): what a
        # candidate-materialising join would have to move; the bit-sliced (C4) and tile (C1, C3)
        # kernels process many candidates per word / in shared memory, so this can exceed 1
        b8 = sum(s["tuples_derived"] * s["fj_row_bytes"] + 2 * s["candidates"] * s["fj_row_bytes"]
                 for s in rf_stats[-1])
        roofline["per_candidate_model"] = {"achieved": b8 / t_alg / 1e9, "frac": b8 / t_alg / 1e9 / peak,
                                           "def": "(Σ tuples·r + 2·candidates·r) / summed phase time, "
                                                  "r = 4 B key + tag bytes"}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if part else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg["desc"], "name": args.config, "global_batch": gbatch,
                       "parallelism": (f"key-partitioned x{ws} (tuples owned by key hash; candidate all-to-all "
                                       f"and Σ|Δ'| all-reduce every round over NCCL)" if part else
                                       f"dp{ws} (batch sharded, global sample ids; no collective inside the fixpoint)"),
                       "semiring_fixpoints": "overlapped on two streams" if overlap else "serial",
                       "l2": "flushed between timed steps (256 MiB write)"},
            "samples_per_s": gbatch / (ms_step / 1000.0),
            "candidates_per_s": cands_step * mult / (ms_step / 1000.0),
            "tuples_per_step": tuples_step * mult, "rounds_per_step": sum(s["rounds_total"] for s in stats_all[-1]),
            "per_rank_ms_per_step": [t_ / args.steps for t_ in per_rank],
            "phases_ms": ph, "gpu_launches": launches, "roofline": roofline}
    if e2e_ms is not None:
        line["e2e"] = {"value": tuples_step * mult / (e2e_ms / args.steps / 1000.0), "unit": UNIT,
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": e2e_d2h,
                       "ms_per_step": e2e_ms / args.steps}
    line["clocks"] = clk.summary()
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and args.config != "C5":
        cores = os.cpu_count() or 1
        tuples, dt, desc = cpu_baseline(args.config, cores)
        t1, d1, desc1 = cpu_baseline(args.config, 1, [0], 1)
        line["cpu_baseline"] = {"value": tuples / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
                                "cpu_model": cpu_model(), "sample": f"{desc}, {dt:.1f} s wall",
                                "single_thread": {"value": t1 / d1, "unit": UNIT, "sample": f"{desc1}, {d1:.1f} s"}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    for e in engines.values():
        e.close()
    if group is not None:
        group.close()
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
