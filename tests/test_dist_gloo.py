"""Multi-rank host logic of the batch-sharded path on CPU with
the gloo backend, world_size 2: sharding with global sample ids, the
per-sample record all-gather in global order, the global fact-id layout
(shared relations on one range) and the gradient all-reduce.  The per-rank
fixpoint is computed by the oracle here (no GPU in CI); the sharded result
must equal a single-process run over the whole batch, slot for slot.  The
same host logic over the CUDA engine is covered on one GPU by
tests/test_gpu_shards.py (sequential shards) and on >= 2 GPUs by its NCCL
test."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _workload(kind, batch):
    import workloads as W
    if kind == "c2":
        return W.c2_workload(semiring=3, n=6, batch=batch), "endpoints_connected"
    # kinship with the SHARED composition relation, under diff-max-mult: its
    # facts collect gradient from every rank's samples
    return W.c3_workload(semiring=3, batch=batch, entities=8, rtypes=5, skips=3, ncomp=12), "answer"


def _dense_grad(rel, nfacts):
    g = np.zeros(nfacts, np.float64)
    for i in range(len(rel)):
        for k in range(rel.grad_offsets[i], rel.grad_offsets[i + 1]):
            g[int(rel.grad_fact_ids[k])] += float(rel.grad_values[k])
    return g


def _worker(rank, world, port, kind, batch, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2503_21937_b200 import dist as D
        w, out = _workload(kind, batch)
        lo, hi = D.shard(batch, rank, world)
        lf = D.local_facts(w.facts, lo, hi)       # global sample ids
        # the per-rank fixpoint (the engine's job on a GPU) is the oracle here;
        # it sees this rank's facts only, pushed in the same relation order
        res = oracle.run(w.program, 3, batch, lf, outputs=[out], samples=list(range(lo, hi)))
        ec = res.relations[out]
        rec = D.arity0_records(ec.sample_ids, ec.tags, lo, D.max_shard(batch, world))
        allrec = D.records_global(D.all_gather_records(rec), batch, world)
        lay = D.fact_layout(lf)
        assert lay.nlocal == sum(f.n for f in lf.values())
        local = torch.as_tensor(_dense_grad(ec, lay.nlocal), dtype=torch.float32)
        grad = D.scatter_grad(local, lay, torch.zeros(lay.total, dtype=torch.float32))
        D.all_reduce_grad(grad)
        if rank == 0:
            q.put((allrec.numpy(), grad.numpy(), lay.total))
    finally:
        dist.destroy_process_group()


def _run_world(kind, batch, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, batch, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return got


@pytest.mark.parametrize("batch", [4, 5])
def test_sharded_equals_single_process(batch, oracle_lib):
    """Records in global sample order and the gradient over GLOBAL fact ids
    equal a single process over the whole batch, slot for slot."""
    import oracle
    allrec, grad, total = _run_world("c2", batch)
    w, out = _workload("c2", batch)
    full = oracle.run(w.program, 3, batch, w.facts, outputs=[out]).relations[out]
    exp = np.zeros((batch, 2), np.float32)
    for s, p in zip(full.sample_ids, full.tags):
        exp[s] = (1.0, p)
    assert np.array_equal(allrec, exp)
    assert total == w.n_facts()
    g_full = _dense_grad(full, w.n_facts())
    # every batched fact is written by exactly one rank: exact
    assert np.array_equal(grad, g_full.astype(np.float32))


def test_shared_relation_gradients_sum_across_ranks(oracle_lib):
    """C3-shaped kinship (shared `composition`) under diff-max-mult: a shared
    fact's global slot holds the sum over every rank's samples."""
    import oracle
    batch = 6
    allrec, grad, total = _run_world("kinship", batch)
    w, out = _workload("kinship", batch)
    assert total == w.n_facts()
    full = oracle.run(w.program, 3, batch, w.facts, outputs=[out]).relations[out]
    g_full = _dense_grad(full, w.n_facts())
    names = list(w.facts)
    ncomp_lo = sum(w.facts[r].n for r in names[:names.index("composition")])
    ncomp = w.facts["composition"].n
    assert np.any(g_full[ncomp_lo:ncomp_lo + ncomp] != 0.0)
    assert np.allclose(grad, g_full, rtol=1e-5, atol=1e-30)


def test_layout_from_counts():
    from paper_2503_21937_b200.dist import layout_from_counts
    # relations: a (batched), s (shared), b (batched); 3 ranks
    counts = np.array([[3, 2, 1], [4, 2, 0], [1, 2, 5]])
    shared = [False, True, False]
    totals = 3 + 4 + 1 + 2 + 1 + 0 + 5
    lays = [layout_from_counts(counts, shared, r) for r in range(3)]
    assert all(l.total == totals for l in lays)
    assert lays[0].segments == [(0, 0, 3), (3, 8, 2), (5, 10, 1)]
    assert lays[1].segments == [(0, 3, 4), (4, 8, 2), (6, 11, 0)]
    assert lays[2].segments == [(0, 7, 1), (1, 8, 2), (3, 11, 5)]
    assert lays[1].to_global(np.array([5, 0, 3])).tolist() == [9, 3, 6]
    # every global id is covered exactly once by batched segments, shared once per rank
    hits = np.zeros(totals, int)
    for l in lays:
        for ls, gs, n in l.segments:
            hits[gs:gs + n] += 1
    assert hits[8:10].tolist() == [3, 3] and np.all(np.delete(hits, [8, 9]) == 1)
    with pytest.raises(ValueError):
        layout_from_counts(np.array([[1, 2], [1, 3]]), [False, True], 0)


def test_shard_ranges_cover_batch():
    from paper_2503_21937_b200.dist import shard
    for batch in (1, 7, 64, 4096):
        for world in (1, 2, 3, 8):
            rs = [shard(batch, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == batch
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1
