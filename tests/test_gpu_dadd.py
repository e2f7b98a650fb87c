"""diff-add-mult-prob on the GPU (the adjoint program, include/lobster.h;
DESIGN.md reading "diff-add-mult") against the oracle's dual-number forward
mode (tests/test_oracle_dadd.py pins it to closed forms).  Tuple sets
bit-exact, p within 1e-5 (add-mult), per-row gradient fact-id sets exact and
values within 1e-5 of the row's largest entry.  On dyadic C1 both sides are
exact, so the gradients must match bit for bit."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workloads as W
from tests.gpu_util import assert_parity, engine_run

pytestmark = pytest.mark.gpu
DADD = 6


@pytest.fixture(scope="module", autouse=True)
def _built():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_21937_b200 import build
    build()
    oracle.build()


def _grad_rows(o, n):
    goff = np.asarray(o.grad_offsets, np.int64)
    return [(np.asarray(o.grad_fact_ids)[goff[i]:goff[i + 1]], np.asarray(o.grad_values)[goff[i]:goff[i + 1]])
            for i in range(n)]


def check(w, rel, exact=False, samples=None):
    eng, stats, _ = engine_run(w, DADD)
    res = oracle.run(w.program, DADD, w.batch_size, w.facts, outputs=[rel], samples=samples)
    assert_parity(eng, res, rel, 2, samples=samples, check_grads=False)
    o = eng.output(rel)
    r = res.relations[rel]
    assert o.grad_offsets is not None
    sel = np.arange(o.n) if samples is None else np.nonzero(np.isin(o.sample_ids, samples))[0]
    gr = _grad_rows(o, o.n)
    goff = np.asarray(r.grad_offsets, np.int64)
    for j, i in enumerate(sel):
        gf, gv = gr[i]
        of = np.asarray(r.grad_fact_ids)[goff[j]:goff[j + 1]]
        ovals = np.asarray(r.grad_values)[goff[j]:goff[j + 1]]
        assert np.array_equal(gf, of), (rel, i, gf[:8], of[:8])
        if exact:
            assert np.array_equal(gv.view(np.uint32), ovals.view(np.uint32)), (rel, i)
        else:
            scale = max(float(np.abs(ovals).max(initial=0.0)), 1e-30)
            assert float(np.abs(gv.astype(np.float64) - ovals).max(initial=0.0)) <= 1e-5 * scale, (rel, i)
    return eng, stats, res


def test_c1_exact():
    check(W.c1_workload(DADD), "path", exact=True)


@pytest.mark.parametrize("seed", range(4))
def test_random_dags(seed):
    check(W.random_dag_workload(16 + 6 * seed, 0.2, 400 + seed, DADD, batch=3), "path")


def test_c3_reduced_answer():
    w = W.c3_workload(semiring=DADD, batch=5, entities=9, rtypes=5, skips=4, ncomp=12)
    check(w, "answer")


def test_two_strata_filters_constants():
    prog = """
    type edge(x: i32, y: i32)
    type lab(x: i32, l: i32)
    rel path(x, y) :- edge(x, y) or (path(x, z) and edge(z, y)).
    rel hop(x, w) :- path(x, y), edge(y, w), lab(w, 2), x != w.
    rel root(y) :- path(0, y).
    output hop
    output root
    """
    rng = np.random.default_rng(9)
    w = W.random_dag_workload(14, 0.25, 31, DADD, batch=2, program=prog)
    n = 14
    lab = W.Facts([np.tile(np.arange(n, dtype=np.int32), 2), rng.integers(0, 3, 2 * n).astype(np.int32)],
                  np.repeat(np.arange(2, dtype=np.int32), n), rng.uniform(0.2, 1.0, 2 * n).astype(np.float32))
    w.facts["lab"] = lab
    check(w, "hop")
    check(w, "root")


def test_backward_dense():
    import torch
    w = W.random_dag_workload(20, 0.2, 77, DADD, batch=2)
    eng, _, _ = engine_run(w, DADD)
    o = eng.output("path")
    up = torch.rand(o.n, device="cuda")
    g = torch.zeros(eng.num_facts, device="cuda")
    eng.backward("path", up, g)
    ref = np.zeros(eng.num_facts, np.float64)
    u = up.cpu().numpy()
    for i, (gf, gv) in enumerate(_grad_rows(o, o.n)):
        np.add.at(ref, gf, np.float32(u[i]) * gv.astype(np.float64))
    assert np.allclose(g.cpu().numpy(), ref, rtol=1e-5, atol=1e-6)
