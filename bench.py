#!/usr/bin/env python
"""Benchmark: derived tuples/s of the semi-naive fixpoint on config C2
(BASELINE.json configs[1]: Pathfinder-shaped 32x32 grids, batch 64 per GPU,
max-min-prob and diff-max-mult-prob with input-fact gradients).

One step = one pass of the whole hot path over one
batch: ingest (facts already in HBM) -> fixpoint under max-min-prob -> fixpoint
under diff-max-mult-prob -> witness walk + gradients -> dense dL/dp contraction;
with N > 1 ranks also all-gather of per-sample outputs and all-reduce of the
input-fact gradient (NCCL).  Weak scaling: every rank owns 64 samples.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl lobster|reference]

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

BATCH_PER_GPU = 64
GRID_N = 32
METRIC = "derived tuples/s"
UNIT = "tuples/s"
WORKLOAD = ("C2: Pathfinder-shaped 32x32 lattice connectivity (Fig. 3c program), batch 64 per GPU, "
            "max-min-prob + diff-max-mult-prob with input-fact gradients")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="lobster", choices=["lobster", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _loop(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

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
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, nm in enumerate(names):
                if len(r) > 5 + k and r[5 + k].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ------------------------------------------------------------------ workload
def make_batch(rank: int):
    """This rank's 64 samples (global ids 64*rank ...); pushed with local ids."""
    samples = list(range(BATCH_PER_GPU * rank, BATCH_PER_GPU * (rank + 1)))
    w = W.grid_workload(GRID_N, BATCH_PER_GPU * (rank + 1), 2, W.gen.DIFF_MAX_MULT_PROB, samples=samples, name="C2")
    for f in w.facts.values():
        if f.sample_ids is not None:
            f.sample_ids = (f.sample_ids - BATCH_PER_GPU * rank).astype(np.int32)
    w.batch_size = BATCH_PER_GPU
    return w


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
def cpu_baseline(threads: int, semiring: int, nsamples: int):
    import oracle
    w = W.grid_workload(GRID_N, BATCH_PER_GPU, 2, semiring, samples=list(range(nsamples)), name="C2")
    t = time.perf_counter()
    res = oracle.run(w.program, semiring, w.batch_size, w.facts, outputs=["path", "endpoints_connected"],
                     samples=list(range(nsamples)), threads=threads)
    dt = time.perf_counter() - t
    tuples = sum(len(r) for r in res.relations.values())
    return tuples, dt


def run_reference(args):
    """--impl reference: the oracle (CPU), as it stands, on a bounded sample of
    C2 per step; rank 0 only."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    nsamp = max(1, min(cores, BATCH_PER_GPU))
    sr_cycle = [W.gen.MAX_MIN_PROB, W.gen.DIFF_MAX_MULT_PROB]
    for i in range(args.warmup):
        cpu_baseline(nsamp, sr_cycle[i % 2], 1)  # warm-up on one sample
    tot_t, tot_tuples = 0.0, 0
    for i in range(args.steps):
        tuples, dt = cpu_baseline(nsamp, sr_cycle[i % 2], nsamp)
        tot_t += dt
        tot_tuples += tuples
    v = tot_tuples / tot_t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {"workload": WORKLOAD, "global_batch": BATCH_PER_GPU},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": nsamp, "kind": "oracle",
                             "sample": f"{nsamp} of the 64 C2 samples per step (one per thread), semiring "
                                       f"alternating max-min / diff-max-mult by step"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- lobster
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    from paper_2503_21937_b200 import DIFF_MAX_MULT_PROB, MAX_MIN_PROB, Engine, _lib

    ws, rank, local = dist_env()
    if ws > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    L = _lib.load()

    w = make_batch(rank)
    # device-resident inputs (value) and pinned host inputs (e2e)
    dfacts, hfacts, h2d = {}, {}, 0
    for rel, f in w.facts.items():
        cols_d = [torch.as_tensor(c).to(dev) for c in f.cols]
        cols_h = [torch.as_tensor(c).pin_memory() for c in f.cols]
        s_d = torch.as_tensor(f.sample_ids).to(dev)
        s_h = torch.as_tensor(f.sample_ids).pin_memory()
        p_d = torch.as_tensor(f.probs).to(dev)
        p_h = torch.as_tensor(f.probs).pin_memory()
        dfacts[rel] = W.Facts(cols_d, s_d, p_d)
        hfacts[rel] = W.Facts(cols_h, s_h, p_h)
        h2d += sum(c.numel() * 4 for c in cols_h) + s_h.numel() * 4 + p_h.numel() * 4
    h2d *= 2  # pushed once per semiring

    engines = {sr: Engine(w.program, sr, batch_size=BATCH_PER_GPU, device=local)
               for sr in (MAX_MIN_PROB, DIFF_MAX_MULT_PROB)}
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    nfacts = w.n_facts()
    grad_dense = torch.zeros(nfacts * ws, dtype=torch.float32, device=dev)

    def step(facts, host_out=False):
        stats, d2h = [], 0
        grad_dense.zero_()
        for sr, eng in engines.items():
            eng.push_facts(facts)
            stats.append(eng.run())
        em = engines[DIFF_MAX_MULT_PROB]
        out_dev = em.output("endpoints_connected", device=True)
        up = torch.ones(out_dev.n, dtype=torch.float32, device=dev)
        g = grad_dense[rank * nfacts:(rank + 1) * nfacts]
        em.backward("endpoints_connected", up, g)
        rec = torch.zeros(2 * BATCH_PER_GPU, dtype=torch.float32, device=dev)  # per-sample (present, p)
        if out_dev.n:
            rec[2 * out_dev.sample_ids.long()] = 1.0
            rec[2 * out_dev.sample_ids.long() + 1] = out_dev.probs
        if ws > 1:
            allrec = torch.empty(ws * rec.numel(), dtype=rec.dtype, device=dev)
            dist.all_gather_into_tensor(allrec, rec)
            dist.all_reduce(grad_dense)
        if host_out:  # e2e: results back to the host through the C ABI
            for sr, eng in engines.items():
                o = eng.output("endpoints_connected", device=False)
                d2h += o.n * 8 + o.sample_offsets.nbytes
                if o.probs is not None:
                    d2h += o.probs.nbytes
                if o.grad_values is not None:
                    d2h += o.grad_offsets.nbytes + o.grad_fact_ids.nbytes + o.grad_values.nbytes
        return stats, d2h

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step(dfacts)
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
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), stats_all, d2h, launches

    with ClockSampler(local) as clk:
        total_ms, stats_all, _, launches = timed(dfacts, False)
    e2e_ms, e2e_d2h = None, 0
    if not args.no_e2e:
        e2e_ms, _, e2e_d2h, _ = timed(hfacts, True)

    tuples_step = sum(s["tuples_derived"] for s in stats_all[-1])
    cands_step = sum(s["candidates"] for s in stats_all[-1])
    ms_step = total_ms / args.steps
    value = tuples_step * ws / (ms_step / 1000.0)
    # phase breakdown (engine CUDA events, summed over both semirings, last step)
    ph = {k: sum(s[k] for s in stats_all[-1]) for k in ("ms_join", "ms_sort", "ms_reduce", "ms_merge", "ms_grad")}
    peak, peak_src = peaks()
    # Dominant kernel: the fused row-centric join + direct ⊕ (join_rows_direct_k).
    # SURVEY §8(d) algorithmic bytes per launch = |Δ|·r_Δ (probe read) + 2·|C|·r_C
    # (candidate write + re-read for dedup), r = packed key (4 B) + tag bytes;
    # duration = the engine's CUDA events around each launch, on its stream,
    # summed over the timed steps (averaged per launch).
    last = stats_all  # every timed step
    fj_l = sum(s["fj_launches"] for st in last for s in st)
    fj_ms = sum(s["ms_fused_join"] for st in last for s in st)
    fj_b = sum(s["fj_probe_rows"] * s["fj_row_bytes"] + 2 * s["fj_candidates"] * s["fj_row_bytes"]
               for st in last for s in st)
    tr = ncu_traffic()
    if fj_l and fj_ms > 0:
        achieved = fj_b / fj_l / (fj_ms / fj_l / 1000.0) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": tr.get("dram_bytes_per_launch"),
                    "kernel": "join_rows_direct_k (fused count-free join + ⊗ + direct ⊕ into the dense store)",
                    "launches_per_step": fj_l / len(last), "avg_launch_us": 1000.0 * fj_ms / fj_l,
                    "alg_bytes_per_launch": fj_b / fj_l,
                    "alg_bytes_def": "SURVEY §8(d): |Δ|·r + 2·|C|·r per launch, r = 4 B key + tag (8 B max-mult)",
                    "traffic_source": tr.get("source"), "peak_source": peak_src}
    else:
        bytes_alg = sum(s["bytes_algorithmic"] for s in stats_all[-1])
        t_alg = sum(ph[k] for k in ("ms_join", "ms_sort", "ms_reduce", "ms_merge")) / 1000.0
        achieved = bytes_alg / t_alg / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": None, "kernel": "fixpoint phases (no fused join launched)", "peak_source": peak_src}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "global_batch": BATCH_PER_GPU * ws, "grid": f"{GRID_N}x{GRID_N}",
                       "parallelism": f"dp{ws} (batch sharded, no collective inside the fixpoint)",
                       "l2": "flushed between timed steps (256 MiB write)"},
            "samples_per_s": BATCH_PER_GPU * ws / (ms_step / 1000.0),
            "candidates_per_s": cands_step * ws / (ms_step / 1000.0),
            "tuples_per_step": tuples_step * ws, "rounds_per_step": sum(s["rounds_total"] for s in stats_all[-1]),
            "phases_ms": ph, "gpu_launches": launches, "roofline": roofline}
    if e2e_ms is not None:
        line["e2e"] = {"value": tuples_step * ws / (e2e_ms / args.steps / 1000.0), "unit": UNIT,
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": e2e_d2h,
                       "ms_per_step": e2e_ms / args.steps}
    line["clocks"] = clk.summary()
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        ns = max(1, min(cores, 16))
        tuples, dt = cpu_baseline(ns, W.gen.DIFF_MAX_MULT_PROB, ns)
        line["cpu_baseline"] = {"value": tuples / dt, "unit": UNIT, "cores": ns, "kind": "oracle",
                                "sample": f"{ns} of the 64 C2 samples under diff-max-mult-prob "
                                          f"(one sample per thread), {dt:.1f} s wall"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    for e in engines.values():
        e.close()
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
