"""Helpers for GPU-vs-oracle parity tests (compare element by element)."""
from __future__ import annotations

import numpy as np

import oracle

REL_TOL = {0: 0.0, 1: 0.0, 2: 1e-5, 3: 0.0}   # unit / max-min / max-mult bit-exact; add-mult 1e-5 (reading 9)
GRAD_TOL = 1e-6


def engine_run(w, semiring=None, stream=None, **kw):
    from paper_2503_21937_b200 import Engine
    sr = w.semiring if semiring is None else semiring
    eng = Engine(w.program, sr, batch_size=w.batch_size, stream=stream, **kw)
    first = eng.push_facts(w.facts)
    stats = eng.run()
    return eng, stats, first


def gpu_rel(eng, rel):
    o = eng.output(rel)
    keys = [tuple([int(s)] + [int(o.cols[c][i]) for c in range(o.arity)]) for i, s in enumerate(o.sample_ids)]
    return o, keys


def oracle_rel(res, rel):
    r = res.relations[rel]
    keys = [tuple([int(s)] + [int(v) for v in c]) for s, c in zip(r.sample_ids, r.cols)]
    return r, keys


def assert_parity(eng, res, rel, semiring, samples=None, check_grads=True):
    """Tuple sets bit-exact; tags within the semiring's tolerance; gradients
    (fact ids exact, values 1e-6 rel).  `samples`: restrict the GPU side to
    the oracle's sample subset."""
    o, gk = gpu_rel(eng, rel)
    r, ok = oracle_rel(res, rel)
    idx = np.arange(len(gk))
    if samples is not None:
        sset = set(int(s) for s in samples)
        idx = np.array([i for i, k in enumerate(gk) if k[0] in sset], dtype=np.int64)
        gk = [gk[i] for i in idx]
    assert gk == ok, f"{rel}: tuple sets differ (gpu {len(gk)} vs oracle {len(ok)}): " \
                     f"{sorted(set(gk) ^ set(ok))[:10]}"
    if semiring != 0:
        gp = o.probs[idx]
        tol = REL_TOL[semiring]
        if tol == 0.0:
            bad = np.nonzero(gp.view(np.uint32) != r.tags.view(np.uint32))[0]
            assert bad.size == 0, f"{rel}: {bad.size} tags differ, e.g. {[(gk[i], gp[i], r.tags[i]) for i in bad[:5]]}"
        else:
            err = np.abs(gp.astype(np.float64) - r.tags) / np.maximum(np.abs(r.tags.astype(np.float64)), 1e-30)
            assert float(err.max(initial=0.0)) <= tol, f"{rel}: max rel err {err.max()}"
    if semiring == 3 and check_grads and r.grad_offsets is not None:
        assert o.grad_offsets is not None, "GPU produced no gradients"
        for j, i in enumerate(idx):
            a, b = o.grad_offsets[i], o.grad_offsets[i + 1]
            c, d = r.grad_offsets[j], r.grad_offsets[j + 1]
            gf, gv = o.grad_fact_ids[a:b], o.grad_values[a:b]
            of, ov = r.grad_fact_ids[c:d], r.grad_values[c:d]
            assert np.array_equal(gf, of), f"{rel} {gk[j]}: proof differs {gf} vs {of}"
            e = np.abs(gv.astype(np.float64) - ov) / np.maximum(np.abs(ov.astype(np.float64)), 1e-30)
            assert float(e.max(initial=0.0)) <= GRAD_TOL, f"{rel} {gk[j]}: grad err {e.max()}"
    return len(gk)


def run_both(w, semiring=None, samples=None, outputs=(), threads=0):
    sr = w.semiring if semiring is None else semiring
    eng, stats, _ = engine_run(w, sr)
    res = oracle.run(w.program, sr, w.batch_size, w.facts, outputs=outputs, samples=samples, threads=threads)
    return eng, stats, res
