"""Key-partitioned evaluation of ONE database across ranks (SURVEY §8(f)
NEXT-3; include/lobster.h lobster_partition) against the oracle.

W engines of this process form a local group (one host thread and one CUDA
stream each; on a 1-GPU box they share the device, which exercises the same
owner hashing, candidate all-to-all, global Σ|Δ'| and stratum-end gather as W
GPUs).  The union of the ranks' outputs must equal the oracle's relation: tuple
sets bit-exact, unit / max-min tags bit-exact, add-mult within 1e-5; the ranks'
parts are disjoint and every rank runs the oracle's number of rounds.  A W=1
NCCL group runs the NCCL transport end to end (self send / receive)."""
from __future__ import annotations

import threading

import numpy as np
import pytest

import oracle
import workloads as W
from workloads import gen as G
from tests.gpu_util import REL_TOL

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_21937_b200 import build
    build()
    oracle.build()


def run_partitioned(w, world, rels, sr=None, group=None):
    import torch
    from paper_2503_21937_b200 import Engine, Group
    sr = w.semiring if sr is None else sr
    g = group or Group.local(world)
    streams = [torch.cuda.Stream() for _ in range(world)]
    engines = [Engine(w.program, sr, batch_size=w.batch_size, stream=streams[r].cuda_stream) for r in range(world)]
    for r, e in enumerate(engines):
        e.partition(g, r)
    out = [None] * world
    errs = []

    def work(r):
        try:
            engines[r].push_facts(w.facts)
            st = engines[r].run()
            out[r] = (st, {rel: engines[r].output(rel) for rel in rels})
        except BaseException as ex:  # noqa: BLE001
            errs.append(ex)

    ths = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if errs:
        raise errs[0]
    return engines, g, out


def union_matches(out, res, rel, sr):
    keys, tags = [], []
    for st, o in out:
        x = o[rel]
        m = np.empty((x.n, 1 + x.arity), np.int64)
        m[:, 0] = x.sample_ids
        for c in range(x.arity):
            m[:, 1 + c] = x.cols[c]
        keys.append(m)
        if sr != 0:
            tags.append(x.probs)
    K = np.concatenate(keys)
    order = np.lexsort(K.T[::-1])
    K = K[order]
    r = res.relations[rel]
    O = np.empty((len(r), 1 + r.cols.shape[1]), np.int64)
    O[:, 0] = r.sample_ids
    O[:, 1:] = r.cols
    assert K.shape == O.shape and np.array_equal(K, O), f"{rel}: tuple sets differ ({K.shape[0]} vs {O.shape[0]})"
    assert np.unique(K, axis=0).shape[0] == K.shape[0], "ranks' parts overlap"
    if sr != 0:
        P = np.concatenate(tags)[order]
        if REL_TOL[sr] == 0.0:
            assert np.array_equal(P.view(np.uint32), r.tags.view(np.uint32))
        else:
            err = np.abs(P.astype(np.float64) - r.tags) / np.maximum(np.abs(r.tags.astype(np.float64)), 1e-30)
            assert float(err.max(initial=0.0)) <= REL_TOL[sr]


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_same_generation(world):
    w = G.sg_workload(nodes=400, out_degree=2, seed=11)
    res = oracle.run_workload(w, outputs=["sg"])
    engines, g, out = run_partitioned(w, world, ["sg"])
    union_matches(out, res, "sg", 0)
    assert {st["rounds_total"] for st, _ in out} == {int(res.rounds.sum())}
    if world > 1:
        assert all(o["sg"].n > 0 for _, o in out), "a rank owns nothing"


@pytest.mark.parametrize("sr", [0, 1, 2])
@pytest.mark.parametrize("world", [2, 3])
def test_tc_batched_semirings(sr, world):
    mk = W.random_dag_workload if sr == 2 else W.random_digraph_workload
    w = mk(40, 0.08, 21 + world, sr, batch=3)
    res = oracle.run_workload(w, outputs=["path"])
    engines, g, out = run_partitioned(w, world, ["path"])
    union_matches(out, res, "path", sr)


TWO_STRATA_PROGRAM = """
type edge(x: i32, y: i32)
rel path(x, y) :- edge(x, y) or (path(x, z) and edge(z, y)).
rel hop2(x, w) :- path(x, y), edge(y, z), edge(z, w), x != w.
output hop2
"""


@pytest.mark.parametrize("sr", [0, 1])
def test_later_stratum_sees_gathered_relation(sr):
    """`path` is read by the next stratum: it is gathered whole onto every rank
    at its stratum's end (each rank then holds all of it), `hop2` stays split."""
    w = W.random_digraph_workload(30, 0.1, 77, sr, batch=2, program=TWO_STRATA_PROGRAM)
    res = oracle.run_workload(w, outputs=["hop2", "path"])
    engines, g, out = run_partitioned(w, 3, ["hop2", "path"])
    union_matches(out, res, "hop2", sr)
    for _, o in out:  # the gathered relation: complete on every rank
        union_matches([(None, o)], res, "path", sr)


def test_nccl_group_world1():
    from paper_2503_21937_b200 import Group
    g = Group.nccl(Group.nccl_id(), 0, 1, 0)
    w = G.sg_workload(nodes=300, out_degree=2, seed=12)
    res = oracle.run_workload(w, outputs=["sg"])
    engines, _, out = run_partitioned(w, 1, ["sg"], group=g)
    union_matches(out, res, "sg", 0)


def test_partition_errors():
    from paper_2503_21937_b200 import Engine, Group, LobsterError, _lib
    g = Group.local(2)
    e = Engine(W.PATH_PROGRAM, 3, batch_size=1)
    with pytest.raises(LobsterError) as ex:
        e.partition(g, 0)
    assert ex.value.status == _lib.E_INVALID_ARG
    e = Engine("type edge(x: i32, y: i32)\nrel path(x, y) :- edge(x, y) or (path(x, z) and path(z, y)).", 0)
    with pytest.raises(LobsterError) as ex:
        e.partition(g, 1)
    assert ex.value.status == _lib.E_SCHEMA
    e = Engine(W.PATH_PROGRAM, 0)
    with pytest.raises(LobsterError) as ex:
        e.partition(g, 2)
    assert ex.value.status == _lib.E_INVALID_ARG
