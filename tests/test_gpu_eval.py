"""GPU parity of integer expressions (§5.2 eval; include/lobster.h
grammar) against the oracle (tests/test_oracle_eval.py pins it): arithmetic
head columns and expression comparisons run as bytecode in the projection
kernel over the rule's __eval body relation; <, <=, >, >= on variables run
natively in every join, lookup, fused and tile kernel.  Tuple sets bit-exact,
tags by the semiring's tolerance, diff-max-mult proofs through the __eval
relation exact."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workloads as W
from tests.gpu_util import assert_parity, engine_run

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_21937_b200 import build
    build()
    oracle.build()


def facts(cols, probs=None, sids=None):
    cols = [np.asarray(c, np.int32) for c in cols]
    n = cols[0].shape[0]
    return W.Facts(cols, np.zeros(n, np.int32) if sids is None else np.asarray(sids, np.int32),
                   None if probs is None else np.asarray(probs, np.float32))


def both(prog, sr, batch, fs, rels, rounds=True):
    w = W.Workload("t", prog, sr, batch, fs)
    eng, stats, _ = engine_run(w)
    res = oracle.run(prog, sr, batch, fs, outputs=rels)
    for r in rels:
        assert_parity(eng, res, r, sr)
    if rounds:
        assert stats["rounds_total"] == int(res.rounds.sum())
    return eng, stats, res


ARITH = """
type a(x: i32)
type b(y: i32)
rel r(x + y, x * y) :- a(x), b(y), x < y.
rel s(x - y * 2 + -x, x) :- a(x), b(y), x * 2 >= y + 1, x != 5.
rel q(x / y, x % y) :- a(x), b(y).
output r
output q
"""


@pytest.mark.parametrize("sr", [0, 1, 2, 3])
def test_arithmetic_heads_and_filters(sr):
    A = [-7, -3, 0, 2, 3, 5, 9]
    B = [-4, -1, 0, 2, 3, 7]
    rng = np.random.default_rng(sr)
    S = 3
    fa = facts([np.tile(A, S)], rng.uniform(0.1, 1.0, len(A) * S), np.repeat(np.arange(S), len(A)))
    fb = facts([np.tile(B, S)], rng.uniform(0.1, 1.0, len(B) * S), np.repeat(np.arange(S), len(B)))
    both(ARITH, sr, S, {"a": fa, "b": fb}, ["r", "s", "q"])


@pytest.mark.parametrize("sr", [0, 1])
def test_comparisons_constants_strata(sr):
    prog = """
    type e(x: i32, y: i32)
    rel nxt(x, y) :- e(x, y), x + 1 == y.
    rel neg(y) :- e(-2, y).
    rel big(z) :- nxt(z, w), z > 2, w <= 6.
    rel two(x, y) :- e(x, y), (x - y) % 3 == 0.
    """
    E = [(-2, 4), (-2, -1), (0, 1), (1, 2), (3, 4), (4, 5), (5, 6), (6, 7), (7, 1), (2, 8)]
    p = np.linspace(0.1, 1.0, len(E))
    both(prog, sr, 1, {"e": facts(list(zip(*E)), p)}, ["nxt", "neg", "big", "two"])


def test_wrap_and_recursion_upstream():
    prog = """
    type a(x: i32)
    type e(x: i32, y: i32)
    rel o(x * 1000000, 0 - x) :- a(x).
    rel p(x, y) :- e(x, y) or (p(x, z) and e(z, y)).
    rel d(x, y - x) :- p(x, y), y > x.
    """
    A = [3, 2147, 4000, -5000]
    E = [(0, 1), (1, 2), (2, 3), (3, 1)]
    both(prog, 0, 1, {"a": facts([A]), "e": facts(list(zip(*E)))}, ["o", "d"])


@pytest.mark.parametrize("tile", [True, False])
@pytest.mark.parametrize("sr", [0, 1, 2, 3])
def test_relational_filters_in_recursive_rules(sr, tile, monkeypatch):
    """`<` inside recursion: native comparisons in the tile, fused and join kernels."""
    if not tile:
        monkeypatch.setenv("LOBSTER_NO_TILE", "1")
    prog = """
    type edge(x: i32, y: i32)
    rel up(x, y) :- edge(x, y), x < y.
    rel up(x, y) :- up(x, z), edge(z, y), z < y, y <= 30.
    output up
    """
    mk = W.random_dag_workload if sr == 2 else W.random_digraph_workload
    w = mk(36, 0.12, 5 + sr, sr, batch=3, program=prog)
    eng, stats, res = both(prog, sr, 3, w.facts, ["up"])
    assert (stats["tile_strata"] > 0) == (tile and sr != 3)


def test_recursive_arithmetic_is_refused():
    from paper_2503_21937_b200 import Engine, LobsterError, _lib
    with pytest.raises(LobsterError) as e:
        Engine("type e(x: i32, y: i32)\nrel d(y, n + 1) :- d(x, n), e(x, y).\nrel d(x, 0) :- e(x, y).", 0)
    assert e.value.status == _lib.E_PARSE
