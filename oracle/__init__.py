"""ctypes wrapper around the C++ oracle (oracle/oracle.cpp).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs may import this package.  The product
package `paper_2503_21937_b200` never imports it; the two share no code.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field
from typing import Dict, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "oracle.cpp")
LIB = os.path.join(HERE, "liboracle.so")

UNIT, MAX_MIN_PROB, ADD_MULT_PROB, DIFF_MAX_MULT_PROB, DIFF_MAX_MIN_PROB, DIFF_TOP1_PROOFS, DIFF_ADD_MULT_PROB = 0, 1, 2, 3, 4, 5, 6


def build(force: bool = False) -> str:
    """Compile the oracle with g++ -O2, no fast-math, no FP contraction."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-pthread",
               "-ffp-contract=off", "-fno-fast-math", SRC, "-o", LIB + ".tmp"]
        subprocess.check_call(cmd)
        os.replace(LIB + ".tmp", LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        vp, cp, i64p, i32p, f32p = (ctypes.c_void_p, ctypes.c_char_p,
                                    ctypes.POINTER(ctypes.c_int64),
                                    ctypes.POINTER(ctypes.c_int32),
                                    ctypes.POINTER(ctypes.c_float))
        L.orc_create.restype = vp
        L.orc_create.argtypes = [cp, ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.c_int]
        L.orc_destroy.argtypes = [vp]
        L.orc_last_error.restype = cp
        L.orc_last_error.argtypes = [vp]
        L.orc_set_max_iters.argtypes = [vp, ctypes.c_int]
        L.orc_rel_arity.argtypes = [vp, cp]
        L.orc_num_strata.argtypes = [vp]
        L.orc_push.argtypes = [vp, cp, ctypes.c_int64, i32p, i32p, f32p, i64p]
        L.orc_run.argtypes = [vp, ctypes.c_int, i32p, ctypes.c_int]
        L.orc_set_groups.argtypes = [vp, ctypes.c_int64, ctypes.c_int64, i32p]
        L.orc_result_size.restype = ctypes.c_int64
        L.orc_result_size.argtypes = [vp, cp]
        L.orc_result.argtypes = [vp, cp, i32p, i32p, f32p]
        L.orc_grad_size.restype = ctypes.c_int64
        L.orc_grad_size.argtypes = [vp, cp]
        L.orc_grad.argtypes = [vp, cp, i64p, i64p, f32p]
        L.orc_stats.argtypes = [vp, i32p, i64p]
        L.orc_stratum.argtypes = [vp, ctypes.c_int, ctypes.c_char_p, ctypes.c_int]
        L.orc_otimes.restype = ctypes.c_float
        L.orc_otimes.argtypes = [ctypes.c_int, ctypes.c_float, ctypes.c_float]
        L.orc_oplus.restype = ctypes.c_float
        L.orc_oplus.argtypes = [ctypes.c_int, ctypes.c_float, ctypes.c_float]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


def _ptr(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t)) if a is not None else None


@dataclass
class Relation:
    sample_ids: np.ndarray          # (n,) int32, sorted by (sample, cols)
    cols: np.ndarray                # (n, arity) int32
    tags: np.ndarray                # (n,) float32
    grad_offsets: Optional[np.ndarray] = None
    grad_fact_ids: Optional[np.ndarray] = None
    grad_values: Optional[np.ndarray] = None

    def __len__(self):
        return int(self.sample_ids.shape[0])


@dataclass
class Result:
    relations: Dict[str, Relation]
    strata: list
    rounds: np.ndarray
    candidates: np.ndarray
    first_fact_ids: Dict[str, int] = field(default_factory=dict)


def otimes(sr: int, a: float, b: float) -> float:
    return lib().orc_otimes(sr, a, b)


def oplus(sr: int, a: float, b: float) -> float:
    return lib().orc_oplus(sr, a, b)


def run(program: str, semiring: int, batch: int, facts: dict, outputs: Sequence[str] = (),
        samples: Optional[Sequence[int]] = None, threads: int = 0,
        max_iters: Optional[int] = None, want_grads: bool = True,
        groups: Optional[Dict[str, np.ndarray]] = None) -> Result:
    """Evaluate `program` on `facts` (dict rel -> workloads.Facts-like object with
    .cols list, .sample_ids, .probs). Facts are pushed in dict order, so fact ids
    are dense in that order. `outputs`: IDB relations to read back
    (default: every IDB relation).  `groups`: rel -> int32 exclusion group per
    fact (top-1-proof conflicts; -1 = none)."""
    L = lib()
    err = ctypes.create_string_buffer(512)
    h = L.orc_create(program.encode(), semiring, batch, err, 512)
    if not h:
        raise OracleError(2, err.value.decode())
    try:
        if max_iters is not None:
            L.orc_set_max_iters(h, int(max_iters))
        first_ids = {}
        for rel, f in facts.items():
            ar = L.orc_rel_arity(h, rel.encode())
            n = f.n if hasattr(f, "n") else len(f.cols[0])
            if ar < 0:
                raise OracleError(3, f"unknown relation {rel}")
            cols = (np.stack([np.asarray(c, dtype=np.int32) for c in f.cols], axis=1)
                    if ar > 0 else np.zeros((n, 0), dtype=np.int32))
            cols = np.ascontiguousarray(cols, dtype=np.int32)
            sids = None if f.sample_ids is None else np.ascontiguousarray(f.sample_ids, dtype=np.int32)
            probs = None if f.probs is None else np.ascontiguousarray(f.probs, dtype=np.float32)
            first = ctypes.c_int64(0)
            rc = L.orc_push(h, rel.encode(), n, _ptr(cols, ctypes.c_int32), _ptr(sids, ctypes.c_int32),
                            _ptr(probs, ctypes.c_float), ctypes.byref(first))
            if rc:
                raise OracleError(rc, L.orc_last_error(h).decode())
            first_ids[rel] = first.value
            if groups and rel in groups and n:
                g = np.ascontiguousarray(groups[rel], dtype=np.int32)
                rc = L.orc_set_groups(h, first.value, n, _ptr(g, ctypes.c_int32))
                if rc:
                    raise OracleError(rc, L.orc_last_error(h).decode())
        s = np.asarray([] if samples is None else list(samples), dtype=np.int32)
        rc = L.orc_run(h, int(s.shape[0]), _ptr(s, ctypes.c_int32) if s.shape[0] else None, threads)
        if rc:
            raise OracleError(rc, L.orc_last_error(h).decode())
        ns = L.orc_num_strata(h)
        strata = []
        buf = ctypes.create_string_buffer(4096)
        for i in range(ns):
            L.orc_stratum(h, i, buf, 4096)
            strata.append(buf.value.decode().split(","))
        rounds = np.zeros(ns, dtype=np.int32)
        cands = np.zeros(ns, dtype=np.int64)
        L.orc_stats(h, _ptr(rounds, ctypes.c_int32), _ptr(cands, ctypes.c_int64))
        rels = {}
        names = list(outputs) if outputs else [r for st in strata for r in st]
        for rel in names:
            ar = L.orc_rel_arity(h, rel.encode())
            n = L.orc_result_size(h, rel.encode())
            sid = np.zeros(n, dtype=np.int32)
            cols = np.zeros((n, max(ar, 0)), dtype=np.int32)
            tags = np.zeros(n, dtype=np.float32)
            rc = L.orc_result(h, rel.encode(), _ptr(sid, ctypes.c_int32),
                              _ptr(cols, ctypes.c_int32) if ar > 0 else ctypes.cast(ctypes.create_string_buffer(4), ctypes.POINTER(ctypes.c_int32)),
                              _ptr(tags, ctypes.c_float))
            if rc:
                raise OracleError(rc, L.orc_last_error(h).decode())
            r = Relation(sid, cols, tags)
            if semiring in (DIFF_MAX_MULT_PROB, DIFF_MAX_MIN_PROB, DIFF_TOP1_PROOFS, DIFF_ADD_MULT_PROB) and want_grads:
                g = L.orc_grad_size(h, rel.encode())
                off = np.zeros(n + 1, dtype=np.int64)
                fid = np.zeros(max(g, 1), dtype=np.int64)
                val = np.zeros(max(g, 1), dtype=np.float32)
                rc = L.orc_grad(h, rel.encode(), _ptr(off, ctypes.c_int64), _ptr(fid, ctypes.c_int64),
                                _ptr(val, ctypes.c_float))
                if rc == 0:
                    r.grad_offsets, r.grad_fact_ids, r.grad_values = off, fid[:g], val[:g]
            rels[rel] = r
        return Result(rels, strata, rounds, cands, first_ids)
    finally:
        L.orc_destroy(h)


def run_workload(w, samples=None, threads: int = 0, outputs=(), **kw) -> Result:
    return run(w.program, w.semiring, w.batch_size, w.facts, outputs=outputs,
               samples=samples, threads=threads, **kw)
