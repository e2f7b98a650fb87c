"""Multi-rank host logic of the batch-sharded path on CPU with
the gloo backend, world_size 2: sharding, per-sample record all-gather,
global fact offsets and the gradient all-reduce.  The per-rank fixpoint is
computed by the oracle here (no GPU in CI); the sharded result must equal a
single-process run over the whole batch."""
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


def _fact_index(facts):
    """(relation, row) of every fact in push order = fact id order."""
    out = []
    for rel, f in facts.items():
        out += [(rel, i) for i in range(f.n)]
    return out


def _worker(rank, world, port, batch, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import workloads as W
        from paper_2503_21937_b200 import dist as D
        w = W.c2_workload(semiring=3, n=6, batch=batch)
        lo, hi = D.shard(batch, rank, world)
        lf = D.local_facts(w.facts, lo, hi)
        res = oracle.run(w.program, 3, hi - lo, lf, outputs=["endpoints_connected"])
        ec = res.relations["endpoints_connected"]
        rec = D.arity0_records(ec.sample_ids, ec.tags, D.max_shard(batch, world))
        allrec = D.all_gather_records(rec)
        nf = sum(f.n for f in lf.values())
        off, total = D.fact_offsets(nf)
        grad = torch.zeros(total, dtype=torch.float32)
        for i in range(len(ec)):
            for k in range(ec.grad_offsets[i], ec.grad_offsets[i + 1]):
                grad[off + int(ec.grad_fact_ids[k])] += float(ec.grad_values[k])
        D.all_reduce_grad(grad)
        # map this rank's local fact ids to full-batch fact ids
        local_to_full = []
        for rel, f in w.facts.items():
            sid = np.asarray(f.sample_ids)
            base = sum(g.n for r2, g in w.facts.items() if list(w.facts).index(r2) < list(w.facts).index(rel))
            idx = np.nonzero((sid >= lo) & (sid < hi))[0] + base
            local_to_full += idx.tolist()
        maps = [None] * world
        dist.all_gather_object(maps, (off, local_to_full))
        if rank == 0:
            q.put((allrec.numpy(), grad.numpy(), maps))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch", [4, 5])
def test_sharded_equals_single_process(batch, oracle_lib):
    import oracle
    import workloads as W
    from paper_2503_21937_b200 import dist as D
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, batch, q)) for r in range(2)]
    for p in procs:
        p.start()
    allrec, grad, maps = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = W.c2_workload(semiring=3, n=6, batch=batch)
    full = oracle.run(w.program, 3, batch, w.facts, outputs=["endpoints_connected"]).relations["endpoints_connected"]
    # records: rank r's local samples occupy global slots [lo_r, hi_r) in rank order
    exp = np.zeros(2 * batch, np.float32)
    for s, p in zip(full.sample_ids, full.tags):
        exp[2 * s] = 1.0
        exp[2 * s + 1] = p
    got = np.zeros(2 * batch, np.float32)
    pos = 0
    for r in range(2):
        lo, hi = D.shard(batch, r, 2)
        n = hi - lo
        got[2 * lo:2 * hi] = allrec[pos:pos + 2 * n]
        pos += 2 * (D.shard(batch, 0, 2)[1] - D.shard(batch, 0, 2)[0])  # gathered slices are rank-0 sized
    assert np.array_equal(got, exp)
    # gradient: permute the sharded fact-id space back to the full run's
    nfull = w.n_facts()
    g_full = np.zeros(nfull, np.float64)
    for i in range(len(full)):
        for k in range(full.grad_offsets[i], full.grad_offsets[i + 1]):
            g_full[int(full.grad_fact_ids[k])] += float(full.grad_values[k])
    g_shard = np.zeros(nfull, np.float64)
    for off, l2f in maps:
        for j, fid in enumerate(l2f):
            g_shard[fid] = grad[off + j]
    assert np.allclose(g_shard, g_full, rtol=1e-6, atol=0)


def test_shard_ranges_cover_batch():
    from paper_2503_21937_b200.dist import shard
    for batch in (1, 7, 64, 4096):
        for world in (1, 2, 3, 8):
            rs = [shard(batch, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == batch
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1
