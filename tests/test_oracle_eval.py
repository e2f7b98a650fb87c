"""Pins for the oracle's expression evaluation (§5.2 "Project
expressions that contain arithmetic or comparison of tuple elements";
DESIGN.md reading "eval"): integer head expressions and comparisons,
int32 two's-complement + - * and unary -, / and % truncating toward zero, a
division / remainder by zero failing the candidate.  Every expected relation is
written out here in plain Python over the input facts (no oracle code), so a
wrong precedence, a flipped relational operator, floor instead of truncating
division or a missing wrap fails a test.  CPU only."""
from __future__ import annotations

import itertools

import numpy as np
import pytest

import oracle
import workloads as W


def i32(v):
    return ((int(v) + 2 ** 31) % 2 ** 32) - 2 ** 31


def cdiv(x, y):
    q = abs(x) // abs(y)
    return q if (x >= 0) == (y >= 0) else -q


def cmod(x, y):
    return x - y * cdiv(x, y)


def facts(cols, probs=None, shared=False):
    cols = [np.asarray(c, np.int32) for c in cols]
    n = cols[0].shape[0]
    return W.Facts(cols, None if shared else np.zeros(n, np.int32),
                   None if probs is None else np.asarray(probs, np.float32))


def rel_dict(res, name):
    r = res.relations[name]
    return {tuple(int(v) for v in c): float(t) for c, t in zip(r.cols, r.tags)}


def test_arithmetic_heads_and_relational_filters(oracle_lib):
    prog = """
    type a(x: i32)
    type b(y: i32)
    rel r(x + y, x * y) :- a(x), b(y), x < y.
    rel s(x - y * 2 + -x, x) :- a(x), b(y), x * 2 >= y + 1, x != 5.
    rel q(x / y, x % y) :- a(x), b(y).
    """
    A = [-7, -3, 0, 2, 3, 5, 9]
    B = [-4, -1, 0, 2, 3, 7]
    pa = np.linspace(0.1, 0.9, len(A)).astype(np.float32)
    pb = np.linspace(0.2, 0.8, len(B)).astype(np.float32)
    w = W.Workload("t", prog, 2, 1, {"a": facts([A], pa), "b": facts([B], pb)})
    res = oracle.run_workload(w, outputs=["r", "s", "q"])
    r, s_, q = rel_dict(res, "r"), rel_dict(res, "s"), rel_dict(res, "q")
    er, es, eq = {}, {}, {}
    for (x, px), (y, py) in itertools.product(zip(A, pa), zip(B, pb)):
        t = float(np.float32(px) * np.float32(py))
        if x < y:
            k = (i32(x + y), i32(x * y))
            er[k] = er.get(k, 0.0) + t
        if 2 * x >= y + 1 and x != 5:
            k = (i32(x - y * 2 + (-x)), x)
            es[k] = es.get(k, 0.0) + t
        if y != 0:
            k = (cdiv(x, y), cmod(x, y))
            eq[k] = eq.get(k, 0.0) + t
    for got, want in ((r, er), (s_, es), (q, eq)):
        assert set(got) == set(want)
        for k, v in want.items():
            assert abs(got[k] - v) <= 1e-6 * abs(v)


def test_expression_comparisons_constants_and_strata(oracle_lib):
    prog = """
    type e(x: i32, y: i32)
    rel nxt(x, y) :- e(x, y), x + 1 == y.
    rel neg(y) :- e(-2, y).
    rel big(z) :- nxt(z, w), z > 2, w <= 6.
    rel two(x, y) :- e(x, y), (x - y) % 3 == 0.
    """
    E = [(-2, 4), (-2, -1), (0, 1), (1, 2), (3, 4), (4, 5), (5, 6), (6, 7), (7, 1), (2, 8)]
    w = W.Workload("t", prog, 0, 1, {"e": facts(list(zip(*E)))})
    res = oracle.run_workload(w, outputs=["nxt", "neg", "big", "two"])
    assert set(rel_dict(res, "nxt")) == {(x, y) for x, y in E if x + 1 == y}
    assert set(rel_dict(res, "neg")) == {(y,) for x, y in E if x == -2}
    assert set(rel_dict(res, "big")) == {(x,) for x, y in E if x + 1 == y and x > 2 and y <= 6}
    assert set(rel_dict(res, "two")) == {(x, y) for x, y in E if cmod(x - y, 3) == 0}


def test_int32_wrap_and_recursion_through_an_expression_free_rule(oracle_lib):
    prog = """
    type a(x: i32)
    type e(x: i32, y: i32)
    rel o(x * 1000000, 0 - x) :- a(x).
    rel p(x, y) :- e(x, y) or (p(x, z) and e(z, y)).
    rel d(x, y - x) :- p(x, y), y > x.
    """
    A = [3, 2147, 4000, -5000]
    E = [(0, 1), (1, 2), (2, 3), (3, 1)]
    w = W.Workload("t", prog, 0, 1, {"a": facts([A]), "e": facts(list(zip(*E)))})
    res = oracle.run_workload(w, outputs=["o", "d"])
    assert set(rel_dict(res, "o")) == {(i32(x * 1000000), -x) for x in A}
    reach = {(x, y) for x, y in E}
    while True:
        more = {(x, y) for (x, z) in reach for (z2, y) in E if z == z2} | reach
        if more == reach:
            break
        reach = more
    assert set(rel_dict(res, "d")) == {(x, y - x) for x, y in reach if y > x}


def test_max_mult_witness_through_an_expression_head(oracle_lib):
    """diff-max-mult: the walk binds a variable used only inside a head
    expression from the witness (it is a non-head variable)."""
    prog = """
    type a(x: i32)
    rel r(x / 2) :- a(x).
    output r
    """
    A, P = [4, 5, 6, 7], [0.5, 0.75, 0.25, 0.125]
    w = W.Workload("t", prog, 3, 1, {"a": facts([A], P)})
    r = oracle.run_workload(w, outputs=["r"]).relations["r"]
    got = {int(c[0]): (float(t), r.grad_fact_ids[r.grad_offsets[i]:r.grad_offsets[i + 1]].tolist())
           for i, (c, t) in enumerate(zip(r.cols, r.tags))}
    assert got == {2: (0.75, [1]), 3: (0.25, [2])}
