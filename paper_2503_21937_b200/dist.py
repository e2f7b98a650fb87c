"""Multi-GPU batch sharding.

A training batch is a set of independent program instances (PAPER.md:681,
689-690 §4.3), so the batch shards across ranks with no communication inside
the fixpoint: rank r owns global samples [lo_r, hi_r) and runs its own engine.
After the fixpoint two collectives run on the ranks' NCCL process group (gloo
in CPU tests):

  * all-gather of fixed-size per-sample output records (arity-0 outputs such as
    endpoints_connected(): (present, p) per sample);
  * all-reduce (sum, fp32) of the dense input-fact gradient over global fact
    ids; every rank fills only its own facts' slots, so per-sample facts are
    exact (x + 0 + ... + 0) and only shared facts see NCCL's summation order.

Host-side logic only; the fixpoint itself runs in liblobster.so.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Optional, Tuple

import numpy as np


def shard(batch: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous global sample range [lo, hi) of `rank` (balanced to +-1)."""
    base, extra = divmod(batch, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def max_shard(batch: int, world: int) -> int:
    """Records are padded to the largest shard so the all-gather is uniform."""
    return -(-batch // world)


def local_facts(facts: Dict[str, object], lo: int, hi: int) -> Dict[str, object]:
    """Facts of samples [lo, hi) with sample ids rebased to [0, hi - lo);
    shared relations (sample_ids None) are replicated unchanged."""
    out = {}
    for rel, f in facts.items():
        if f.sample_ids is None:
            out[rel] = f
            continue
        sid = np.asarray(f.sample_ids)
        m = (sid >= lo) & (sid < hi)
        cls = type(f)
        out[rel] = cls([np.asarray(c)[m] for c in f.cols], (sid[m] - lo).astype(np.int32),
                       None if f.probs is None else np.asarray(f.probs)[m])
    return out


def arity0_records(sample_ids, probs, nlocal: int, torch_mod=None, device=None):
    """(present, p) per local sample for an arity-0 output relation -> [2*nlocal] fp32."""
    import torch
    rec = torch.zeros(2 * nlocal, dtype=torch.float32, device=device)
    if len(sample_ids):
        s = torch.as_tensor(np.asarray(sample_ids) if not isinstance(sample_ids, torch.Tensor) else sample_ids,
                            device=device).long()
        rec[2 * s] = 1.0
        if probs is not None:
            rec[2 * s + 1] = torch.as_tensor(probs, device=device).float()
    return rec


def all_gather_records(rec, group=None):
    """All-gather equal-size per-rank record tensors -> [world * rec.numel()]."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out = torch.empty(world * rec.numel(), dtype=rec.dtype, device=rec.device)
    if rec.device.type == "cuda":
        dist.all_gather_into_tensor(out, rec.contiguous(), group=group)
    else:  # gloo
        parts = [torch.empty_like(rec) for _ in range(world)]
        dist.all_gather(parts, rec.contiguous(), group=group)
        out.copy_(torch.cat(parts))
    return out


def fact_offsets(nfacts_local: int, group=None, device=None) -> Tuple[int, int]:
    """(offset of this rank's facts in the global fact-id space, total facts)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.tensor([nfacts_local], dtype=torch.int64, device=device)
    allt = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(allt, t, group=group)
    counts = [int(x.item()) for x in allt]
    r = dist.get_rank(group)
    return sum(counts[:r]), sum(counts)


def all_reduce_grad(grad, group=None):
    """Sum the dense input-fact gradient across ranks (in place)."""
    import torch.distributed as dist
    dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)
    return grad


@dataclass
class ShardResult:
    records: object          # [batch * 2] (present, p) per global sample
    grad: Optional[object]   # dense dL/dp over global fact ids


def run_sharded(engine, relation: str, facts_local: Dict[str, object], nlocal: int, upstream=None,
                group=None, device=None) -> ShardResult:
    """Push this rank's facts, run the fixpoint, gather per-sample records of an
    arity-0 output relation and all-reduce its input-fact gradient."""
    import torch
    engine.push_facts(facts_local)
    engine.run()
    out = engine.output(relation, device=True)
    rec = arity0_records(out.sample_ids, out.probs, nlocal, device=device)  # nlocal: max_shard() for uneven shards
    allrec = all_gather_records(rec, group)
    grad = None
    if out.grad_offsets is not None:
        off, total = fact_offsets(engine.num_facts, group, device)
        grad = torch.zeros(total, dtype=torch.float32, device=device)
        up = upstream if upstream is not None else torch.ones(out.n, dtype=torch.float32, device=device)
        engine.backward(relation, up, grad[off:off + engine.num_facts])
        all_reduce_grad(grad, group)
    return ShardResult(allrec, grad)
