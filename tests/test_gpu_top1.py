"""GPU parity for diff-top-1-proofs:
tags bit-exact with the oracle, proofs (the gradient's fact ids) identical,
gradients within 1e-6; exclusion-group conflicts, the 300-fact cap and the
linear-recursion restriction of the GPU path."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workloads as W
from tests.gpu_util import assert_parity, engine_run, run_both

pytestmark = pytest.mark.gpu
SR = 5


@pytest.fixture(scope="module", autouse=True)
def _built():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_21937_b200 import build
    build()
    oracle.build()


def test_c1():
    eng, stats, res = run_both(W.c1_workload(SR))
    assert assert_parity(eng, res, "path", SR) == 14
    assert stats["rounds_total"] == int(res.rounds.sum())


@pytest.mark.parametrize("seed", range(6))
def test_random_digraphs(seed):
    rng = np.random.default_rng(80 + seed)
    n = int(rng.integers(3, 30))
    w = W.random_digraph_workload(n, float(rng.uniform(0.05, 0.3)), 80 + seed, SR, batch=3,
                                  self_loops=bool(seed % 2), dyadic=seed % 3 == 0)
    eng, stats, res = run_both(w)
    assert_parity(eng, res, "path", SR)
    assert stats["rounds_total"] == int(res.rounds.sum())


@pytest.mark.parametrize("n,batch", [(6, 4), (12, 3)])
def test_pathfinder_reduced(n, batch):
    w = W.c2_workload(semiring=SR, n=n, batch=batch)
    eng, stats, res = run_both(w, outputs=["path", "endpoints_connected"])
    assert_parity(eng, res, "path", SR)
    assert_parity(eng, res, "endpoints_connected", SR)


def test_set_semantics_and_groups():
    prog = """
type edge(x: i32, y: i32)
rel two(x) :- edge(x, y), edge(x, z).
output two
"""
    f = W.Facts([np.array([0, 0, 1], np.int32), np.array([1, 2, 2], np.int32)], np.zeros(3, np.int32),
                np.array([0.5, 0.75, 0.25], np.float32))
    eng, _, res = run_both(W.Workload("two", prog, SR, 1, {"edge": f}), outputs=["two"])
    assert_parity(eng, res, "two", SR)
    # conflict: 0->1->3 (exclusive pair) loses to 0->2->3
    src = np.array([0, 1, 0, 2, 3], np.int32)
    dst = np.array([1, 3, 2, 3, 4], np.int32)
    p = np.array([0.9, 0.9, 0.6, 0.6, 0.5], np.float32)
    facts = {"edge": W.Facts([src, dst], np.zeros(5, np.int32), p)}
    groups = np.array([7, 7, -1, -1, -1], np.int32)
    from paper_2503_21937_b200 import Engine
    e = Engine(W.PATH_PROGRAM, SR, batch_size=1)
    first = e.push_facts(facts)
    e.facts_groups(first["edge"], groups)
    e.run()
    ref = oracle.run(W.PATH_PROGRAM, SR, 1, facts, outputs=["path"], groups={"edge": groups})
    assert_parity(e, ref, "path", SR)
    got = {tuple(c): float(q) for c, q in zip(e.output("path").cols.T.tolist(), e.output("path").probs)}
    assert got[(0, 3)] == float(np.float32(np.float64(p[2]) * np.float64(p[3])))


def test_random_groups_batched():
    rng = np.random.default_rng(90)
    w = W.random_digraph_workload(12, 0.25, 90, SR, batch=4)
    grp = rng.integers(-1, 6, size=w.facts["edge"].n).astype(np.int32)
    from paper_2503_21937_b200 import Engine
    e = Engine(w.program, SR, batch_size=4)
    first = e.push_facts(w.facts)
    e.facts_groups(first["edge"], grp)
    e.run()
    ref = oracle.run(w.program, SR, 4, w.facts, outputs=["path"], groups={"edge": grp})
    assert_parity(e, ref, "path", SR)


def test_cap_and_linear_only():
    from paper_2503_21937_b200 import Engine, LobsterError
    n = 302
    src = np.arange(n - 1, dtype=np.int32)
    f = {"edge": W.Facts([src, src + 1], np.zeros(n - 1, np.int32), np.full(n - 1, 0.999, np.float32))}
    e = Engine(W.PATH_PROGRAM, SR, batch_size=1)
    e.push_facts(f)
    with pytest.raises(LobsterError) as ex:
        e.run()
    assert "RANGE" in str(ex.value) and "300" in str(ex.value)
    nl = """
type edge(x: i32, y: i32)
rel path(x, y) :- edge(x, y) or (path(x, z) and path(z, y)).
"""
    e = Engine(nl, SR, batch_size=1)
    e.push_facts({"edge": W.Facts([src[:5], src[:5] + 1], np.zeros(5, np.int32), None)})
    with pytest.raises(LobsterError) as ex:
        e.run()
    assert "SCHEMA" in str(ex.value)


def test_chain_300_proof():
    n = 301
    src = np.arange(n - 1, dtype=np.int32)
    rng = np.random.default_rng(91)
    f = {"edge": W.Facts([src, src + 1], np.zeros(n - 1, np.int32), rng.uniform(0.95, 1.0, n - 1).astype(np.float32))}
    eng, stats, res = run_both(W.Workload("chain", W.PATH_PROGRAM, SR, 1, f), outputs=["path"])
    assert assert_parity(eng, res, "path", SR) == n * (n - 1) // 2


def test_c2_full_size_sampled():
    """Full C2 batch (64 x 32x32, the paper's Pathfinder provenance)
    under diff-top-1-proofs; the oracle recomputes samples 0 and 63."""
    w = W.c2_workload(semiring=SR)
    eng, stats, _ = engine_run(w)
    samples = [0, 63]
    res = oracle.run(w.program, SR, w.batch_size, w.facts, outputs=["path", "endpoints_connected"], samples=samples)
    assert_parity(eng, res, "path", SR, samples=samples)
    assert_parity(eng, res, "endpoints_connected", SR, samples=samples)
    assert stats["tuples_derived"] == 64 * 32 ** 4 + 64
