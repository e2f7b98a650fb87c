"""Multi-GPU batch sharding.

A training batch is a set of independent program instances (PAPER.md:681,
689-690 §4.3), so the batch shards across ranks with no communication inside
the fixpoint: rank r owns the global samples [lo_r, hi_r) (the same split the
library applies when `lobster_options.world_size > 1`) and runs its own
engine on them.  Sample ids stay GLOBAL across the ABI.  After the fixpoint
two collectives run on the ranks' process group (NCCL on GPUs, gloo in the
CPU tests):

  * all-gather of fixed-size per-sample output records (arity-0 outputs such
    as endpoints_connected(): (present, p) per sample), reassembled in global
    sample order;
  * all-reduce (sum, fp32) of the dense input-fact gradient over GLOBAL fact
    ids — the ids a single process pushing the whole batch in the same
    relation order would assign: relation by relation, each batched
    relation's rows rank after rank.  A `shared` relation (no sample column)
    is pushed identically on every rank and maps onto ONE global range, so
    its facts receive the genuine sum of every rank's contribution; every
    other slot is written by exactly one rank (x + 0 + ... + 0 = x, exact).

Host-side logic only; the fixpoint itself runs in liblobster.so.
"""
from __future__ import annotations

from dataclasses import dataclass, field
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
    """Facts of samples [lo, hi), keeping their GLOBAL sample ids; shared
    relations (sample_ids None) are replicated unchanged."""
    out = {}
    for rel, f in facts.items():
        if f.sample_ids is None:
            out[rel] = f
            continue
        sid = np.asarray(f.sample_ids)
        m = (sid >= lo) & (sid < hi)
        cls = type(f)
        out[rel] = cls([np.asarray(c)[m] for c in f.cols], sid[m].astype(np.int32),
                       None if f.probs is None else np.asarray(f.probs)[m])
    return out


# ------------------------------------------------------------- fact-id layout
@dataclass
class FactLayout:
    """Where this rank's local fact ids land in the global fact-id space."""
    segments: List[Tuple[int, int, int]] = field(default_factory=list)  # (local start, global start, n)
    total: int = 0          # global number of facts
    nlocal: int = 0

    def to_global(self, local_ids: np.ndarray) -> np.ndarray:
        """Map local fact ids (any order) to global ids."""
        ids = np.asarray(local_ids, np.int64)
        out = np.empty_like(ids)
        for ls, gs, n in self.segments:
            m = (ids >= ls) & (ids < ls + n)
            out[m] = ids[m] - ls + gs
        return out


def _counts_matrix(local_counts: List[int], group=None, device=None) -> np.ndarray:
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if dist.get_backend(group) != "nccl":
        device = "cpu"
    t = torch.tensor(local_counts, dtype=torch.int64, device=device)
    allt = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(allt, t, group=group)
    return np.stack([x.cpu().numpy() for x in allt])


def layout_from_counts(counts: np.ndarray, shared: List[bool], rank: int) -> FactLayout:
    """counts[r, k] = facts of relation k (push order) on rank r."""
    lay = FactLayout()
    lstart = gbase = 0
    for k, sh in enumerate(shared):
        n = int(counts[rank, k])
        if sh:
            if not np.all(counts[:, k] == counts[0, k]):
                raise ValueError(f"shared relation {k} was pushed with different sizes on different ranks")
            gstart, total_k = gbase, int(counts[0, k])
        else:
            gstart, total_k = gbase + int(counts[:rank, k].sum()), int(counts[:, k].sum())
        lay.segments.append((lstart, gstart, n))
        lstart += n
        gbase += total_k
    lay.total, lay.nlocal = gbase, lstart
    return lay


def fact_layout(facts_local: Dict[str, object], group=None, device=None) -> FactLayout:
    """Global fact-id layout of facts pushed in dict order on every rank."""
    import torch.distributed as dist
    names = list(facts_local)
    counts = _counts_matrix([int(facts_local[r].n) for r in names], group, device)
    return layout_from_counts(counts, [facts_local[r].sample_ids is None for r in names], dist.get_rank(group))


def scatter_grad(local_grad, layout: FactLayout, global_grad):
    """global_grad[global ids] += local_grad (contiguous segment copies)."""
    for ls, gs, n in layout.segments:
        if n:
            global_grad[gs:gs + n] += local_grad[ls:ls + n]
    return global_grad


# ------------------------------------------------------------------- records
def arity0_records(sample_ids, probs, lo: int, nmax: int, device=None):
    """(present, p) per local sample of an arity-0 output relation: [2 * nmax]
    fp32, slot i = global sample lo + i (padded to the largest shard)."""
    import torch
    rec = torch.zeros(2 * nmax, dtype=torch.float32, device=device)
    if len(sample_ids):
        s = torch.as_tensor(np.asarray(sample_ids) if not isinstance(sample_ids, torch.Tensor) else sample_ids,
                            device=device).long() - lo
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
    if rec.device.type == "cuda" and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, rec.contiguous(), group=group)
    else:  # gloo (host-staged)
        parts = [torch.empty_like(rec, device="cpu") for _ in range(world)]
        dist.all_gather(parts, rec.contiguous().cpu(), group=group)
        out.copy_(torch.cat(parts).to(out.device))
    return out


def records_global(gathered, batch: int, world: int):
    """Gathered padded per-rank records -> [batch, 2] in global sample order."""
    nmax = max_shard(batch, world)
    g = gathered.view(world, nmax, 2)
    parts = []
    for r in range(world):
        lo, hi = shard(batch, r, world)
        parts.append(g[r, :hi - lo])
    import torch
    return torch.cat(parts)


def all_reduce_grad(grad, group=None):
    """Sum the dense input-fact gradient across ranks (in place)."""
    import torch.distributed as dist
    if grad.device.type == "cuda" and dist.get_backend(group) != "nccl":  # gloo: host-staged
        h = grad.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
        grad.copy_(h)
        return grad
    dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)
    return grad


@dataclass
class ShardResult:
    records: object          # [batch, 2] (present, p) per global sample
    grad: Optional[object]   # dense dL/dp over global fact ids
    layout: Optional[FactLayout] = None


def run_sharded(engine, relation: str, facts_local: Dict[str, object], batch: int, upstream=None,
                group=None, device=None, layout: Optional[FactLayout] = None) -> ShardResult:
    """Push this rank's facts (global sample ids) into `engine` (created with
    batch_size=batch, rank, world_size), run the fixpoint, gather the
    per-sample records of an arity-0 output relation in global order and
    all-reduce its input-fact gradient over global fact ids."""
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    lo, hi = shard(batch, rank, world)
    engine.push_facts(facts_local)
    engine.run()
    out = engine.output(relation, device=True)
    rec = arity0_records(out.sample_ids, out.probs, lo, max_shard(batch, world), device=device)
    allrec = records_global(all_gather_records(rec, group), batch, world)
    grad = None
    if out.grad_offsets is not None:
        lay = layout or fact_layout(facts_local, group, device)
        local = torch.zeros(engine.num_facts, dtype=torch.float32, device=device)
        up = upstream if upstream is not None else torch.ones(out.n, dtype=torch.float32, device=device)
        engine.backward(relation, up, local)
        grad = scatter_grad(local, lay, torch.zeros(lay.total, dtype=torch.float32, device=device))
        all_reduce_grad(grad, group)
        layout = lay
    return ShardResult(allrec, grad, layout)
