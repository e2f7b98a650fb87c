"""Batch sharding through the CUDA engine.

* The full C5 batch (4096 x 64x64 grids) as its 8 rank shards,
  run one after another on one GPU with lobster_options.rank / world_size:
  every sample completes, and shard outputs (global sample ids; gradients
  mapped to global fact ids by dist.layout_from_counts) equal one engine over
  the whole batch bit for bit ("1 GPU ≡ k GPUs").
* Global sample ids across the ABI; out-of-shard pushes fail with RANGE.
* `dist.run_sharded` over NCCL with 2 ranks (skipped on a 1-GPU box).
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_21937_b200 import build
    build()
    oracle.build()


def _counts(shards):
    return np.array([[f.n for f in lf.values()] for lf in shards])


def test_c5_full_batch_as_eight_sequential_shards():
    from paper_2503_21937_b200 import DIFF_MAX_MULT_PROB, Engine
    from paper_2503_21937_b200 import dist as D
    w = W.c5_workload()
    B, world = w.batch_size, 8
    shards = [D.local_facts(w.facts, *D.shard(B, r, world)) for r in range(world)]
    counts = _counts(shards)
    shared = [f.sample_ids is None for f in w.facts.values()]
    rec = np.zeros((B, 2), np.float32)
    proofs = {}
    for r in range(world):
        lo, hi = D.shard(B, r, world)
        eng = Engine(w.program, DIFF_MAX_MULT_PROB, batch_size=B, rank=r, world_size=world)
        eng.push_facts(shards[r])
        eng.run()
        o = eng.output("endpoints_connected")
        assert o.n == hi - lo, f"rank {r}: {o.n} of {hi - lo} samples produced an output"
        assert o.sample_ids.min() == lo and o.sample_ids.max() == hi - 1
        assert o.sample_offsets.shape[0] == hi - lo + 1
        rec[o.sample_ids] = np.stack([np.ones(o.n, np.float32), o.probs], 1)
        lay = D.layout_from_counts(counts, shared, r)
        gids = lay.to_global(o.grad_fact_ids)
        for i, s in enumerate(o.sample_ids.tolist()):
            a, b = o.grad_offsets[i], o.grad_offsets[i + 1]
            proofs[s] = (gids[a:b].copy(), o.grad_values[a:b].copy())
        eng.close()
    assert np.all(rec[:, 0] == 1.0)
    # one engine over the whole batch (micro-batched automatically)
    full = Engine(w.program, DIFF_MAX_MULT_PROB, batch_size=B)
    full.push_facts(w.facts)
    full.run()
    f = full.output("endpoints_connected")
    assert np.array_equal(f.sample_ids, np.arange(B))
    assert np.array_equal(f.probs.view(np.uint32), rec[:, 1].view(np.uint32))
    for i in range(B):
        a, b = f.grad_offsets[i], f.grad_offsets[i + 1]
        gf, gv = proofs[i]
        assert np.array_equal(gf, f.grad_fact_ids[a:b]), i
        assert np.array_equal(gv.view(np.uint32), f.grad_values[a:b].view(np.uint32)), i
    full.close()


def test_global_sample_ids_and_range():
    from paper_2503_21937_b200 import DIFF_MAX_MULT_PROB, Engine, LobsterError
    from paper_2503_21937_b200 import dist as D
    w = W.c2_workload(semiring=3, n=6, batch=7)
    ref = oracle.run(w.program, 3, 7, w.facts, outputs=["endpoints_connected"]).relations["endpoints_connected"]
    for r in range(3):
        lo, hi = D.shard(7, r, 3)
        eng = Engine(w.program, DIFF_MAX_MULT_PROB, batch_size=7, rank=r, world_size=3)
        eng.push_facts(D.local_facts(w.facts, lo, hi))
        eng.run()
        o = eng.output("endpoints_connected")
        m = (ref.sample_ids >= lo) & (ref.sample_ids < hi)
        assert np.array_equal(o.sample_ids, ref.sample_ids[m])
        assert np.array_equal(o.probs.view(np.uint32), ref.tags[m].view(np.uint32))
        od = eng.output("endpoints_connected", device=True)
        assert od.sample_ids.cpu().numpy().tolist() == o.sample_ids.tolist()
        eng.close()
    eng = Engine(w.program, DIFF_MAX_MULT_PROB, batch_size=7, rank=1, world_size=3)
    bad = D.local_facts(w.facts, 0, 1)  # sample 0 belongs to rank 0
    with pytest.raises(LobsterError) as e:
        eng.push_facts(bad)
    assert "RANGE" in str(e.value)
    eng.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _nccl_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        from paper_2503_21937_b200 import DIFF_MAX_MULT_PROB, Engine
        from paper_2503_21937_b200 import dist as D
        w = W.c2_workload(semiring=3, n=8, batch=6)
        lo, hi = D.shard(6, rank, world)
        eng = Engine(w.program, DIFF_MAX_MULT_PROB, batch_size=6, device=rank, rank=rank, world_size=world)
        dev = torch.device("cuda", rank)
        res = D.run_sharded(eng, "endpoints_connected", D.local_facts(w.facts, lo, hi), 6, device=dev)
        if rank == 0:
            q.put((res.records.cpu().numpy(), res.grad.cpu().numpy()))
        eng.close()
    finally:
        dist.destroy_process_group()


def test_run_sharded_nccl_two_ranks():
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    rec, grad = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = W.c2_workload(semiring=3, n=8, batch=6)
    full = oracle.run(w.program, 3, 6, w.facts, outputs=["endpoints_connected"]).relations["endpoints_connected"]
    exp = np.zeros((6, 2), np.float32)
    for s, p in zip(full.sample_ids, full.tags):
        exp[s] = (1.0, p)
    assert np.array_equal(rec, exp)
    g = np.zeros(w.n_facts(), np.float64)
    for i in range(len(full)):
        for k in range(full.grad_offsets[i], full.grad_offsets[i + 1]):
            g[int(full.grad_fact_ids[k])] += float(full.grad_values[k])
    assert np.allclose(grad, g, rtol=1e-6, atol=0)
