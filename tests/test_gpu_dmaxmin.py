"""GPU parity for diff-max-min-prob (§3.5): tags
bit-exact with the oracle (= max-min), witnesses under the same tie rules as
diff-max-mult, one-hot gradients on the same fact."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workloads as W
from tests.gpu_util import assert_parity, engine_run, run_both

pytestmark = pytest.mark.gpu
SR = 4


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


@pytest.mark.parametrize("seed", range(5))
def test_random_digraphs(seed):
    rng = np.random.default_rng(40 + seed)
    n = int(rng.integers(3, 40))
    w = W.random_digraph_workload(n, float(rng.uniform(0.03, 0.25)), 40 + seed, SR, batch=3,
                                  self_loops=bool(seed % 2), dyadic=seed % 2 == 0)
    eng, stats, res = run_both(w)
    assert_parity(eng, res, "path", SR)
    assert stats["rounds_total"] == int(res.rounds.sum())


def test_c2_reduced_both_strata():
    w = W.c2_workload(semiring=SR, n=8, batch=5)
    eng, stats, res = run_both(w, outputs=["path", "endpoints_connected"])
    assert_parity(eng, res, "path", SR, check_grads=False)
    assert_parity(eng, res, "endpoints_connected", SR)


def test_c2_full_size_sampled():
    w = W.c2_workload(semiring=SR)
    samples = [1, 42]
    eng, stats, _ = engine_run(w)
    res = oracle.run(w.program, SR, w.batch_size, w.facts, outputs=["endpoints_connected"], samples=samples)
    assert_parity(eng, res, "endpoints_connected", SR, samples=samples)


def test_kinship_nonlinear():
    w = W.c3_workload(semiring=SR, batch=4, entities=12, rtypes=8, skips=6, ncomp=30)
    eng, stats, res = run_both(w, outputs=["kinship", "answer"])
    assert_parity(eng, res, "kinship", SR)
    assert_parity(eng, res, "answer", SR)


def test_tags_equal_max_min_and_backward():
    import torch
    w = W.c2_workload(semiring=SR, n=6, batch=3)
    e4, _, _ = engine_run(w)
    e1, _, _ = engine_run(w, semiring=1)
    a, b = e4.output("endpoints_connected"), e1.output("endpoints_connected")
    assert np.array_equal(a.probs.view(np.uint32), b.probs.view(np.uint32))
    assert np.all(a.grad_values == 1.0) and np.array_equal(a.grad_offsets, np.arange(a.n + 1))
    up = torch.arange(1, a.n + 1, dtype=torch.float32, device="cuda")
    g = torch.zeros(e4.num_facts, dtype=torch.float32, device="cuda")
    e4.backward("endpoints_connected", up, g)
    exp = np.zeros(e4.num_facts, np.float32)
    for i in range(a.n):
        exp[a.grad_fact_ids[i]] += float(i + 1)
    assert np.array_equal(g.cpu().numpy(), exp)
