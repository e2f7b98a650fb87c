"""GPU parity for the bit-sliced multi-source frontier (k_slice.cu; VERDICT r1
item 4): unit reachability through shared relations, every sample a bit of a
node's words.  Tuple sets bit-exact with the oracle, round counts equal, and
equal to the per-sample bitmap path (LOBSTER_NO_SLICE=1)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workloads as W
from tests.gpu_util import assert_parity, engine_run, run_both

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_21937_b200 import build
    build()
    oracle.build()


REVERSE = """
shared type edge(x: i32, y: i32)
type source(x: i32)
rel reach(y) :- source(x), edge(x, y).
rel reach(y) :- edge(y, x), reach(x).
output reach
"""

TWO_GRAPHS = """
shared type edge(x: i32, y: i32)
shared type link(x: i32, y: i32)
type source(x: i32)
rel reach(x) :- source(x).
rel reach(y) :- reach(x), edge(x, y).
rel reach(y) :- reach(x), link(x, y).
output reach
"""


@pytest.mark.parametrize("batch", [1, 31, 33, 100])
def test_batches_not_multiple_of_32(batch):
    w = W.c4_workload(batch=batch, nodes=3000, edges=20000, seed=60 + batch)
    eng, stats, res = run_both(w, outputs=["reach"])
    assert_parity(eng, res, "reach", 0)
    assert stats["rounds_total"] == int(res.rounds.sum())


def test_reverse_column_and_two_graphs():
    base = W.c4_workload(batch=40, nodes=2000, edges=9000, seed=71)
    w = W.Workload("rev", REVERSE, 0, 40, base.facts)
    eng, stats, res = run_both(w, outputs=["reach"])
    assert_parity(eng, res, "reach", 0)
    assert stats["rounds_total"] == int(res.rounds.sum())
    rng = np.random.default_rng(72)
    link = W.Facts([rng.integers(0, 2000, 3000).astype(np.int32), rng.integers(0, 2000, 3000).astype(np.int32)],
                   None, None)
    facts = {"edge": base.facts["edge"], "link": link, "source": base.facts["source"]}
    w2 = W.Workload("two", TWO_GRAPHS, 0, 40, facts)
    eng, stats, res = run_both(w2, outputs=["reach"])
    assert_parity(eng, res, "reach", 0)
    assert stats["rounds_total"] == int(res.rounds.sum())


def test_tiny_domain():
    """Node domain below 32 (bit fields narrower than a word)."""
    src = np.array([0, 1, 2, 3, 4, 5, 2], np.int32)
    dst = np.array([1, 2, 3, 4, 5, 0, 6], np.int32)
    facts = {"edge": W.Facts([src, dst], None, None),
             "source": W.Facts([np.array([0, 3, 6, 2, 5], np.int32)], np.arange(5, dtype=np.int32), None)}
    w = W.Workload("tiny", W.REACH_PROGRAM, 0, 5, facts)
    eng, stats, res = run_both(w, outputs=["reach"])
    assert_parity(eng, res, "reach", 0)
    assert stats["rounds_total"] == int(res.rounds.sum())


def test_equals_bitmap_path(monkeypatch):
    w = W.c4_workload(batch=64, nodes=20000, edges=150000, seed=73)
    a, sa, _ = engine_run(w)
    oa = a.output("reach")
    monkeypatch.setenv("LOBSTER_NO_SLICE", "1")
    b, sb, _ = engine_run(w)
    ob = b.output("reach")
    assert np.array_equal(oa.sample_ids, ob.sample_ids) and np.array_equal(oa.cols, ob.cols)
    assert sa["rounds_total"] == sb["rounds_total"]
    assert sa["candidates"] == sb["candidates"]


def test_iteration_cap():
    from paper_2503_21937_b200 import LobsterError
    w = W.c4_workload(batch=8, nodes=3000, edges=20000, seed=74)
    from paper_2503_21937_b200 import Engine
    e = Engine(w.program, 0, batch_size=8, max_iters=3)
    e.push_facts(w.facts)
    with pytest.raises(LobsterError) as ex:
        e.run()
    assert "ITER_CAP" in str(ex.value)
    r = oracle.run(w.program, 0, 8, w.facts, outputs=["reach"], max_iters=10_000)
    assert int(r.rounds.sum()) > 3
