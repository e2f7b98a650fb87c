"""Helpers for GPU-vs-oracle parity tests (compare element by element)."""
from __future__ import annotations

import numpy as np

import oracle

REL_TOL = {0: 0.0, 1: 0.0, 2: 1e-5, 3: 0.0, 4: 0.0, 5: 0.0, 6: 1e-5}   # unit / max-min / max-mult / diff-max-min bit-exact; add-mult 1e-5
GRAD_TOL = 1e-6


def engine_run(w, semiring=None, stream=None, **kw):
    from paper_2503_21937_b200 import Engine
    sr = w.semiring if semiring is None else semiring
    eng = Engine(w.program, sr, batch_size=w.batch_size, stream=stream, **kw)
    first = eng.push_facts(w.facts)
    stats = eng.run()
    return eng, stats, first


def _key_matrix(sample_ids, cols, arity, n):
    """(n, 1 + arity) int64 matrix of (sample, c0, ...) rows."""
    m = np.empty((n, 1 + arity), np.int64)
    m[:, 0] = np.asarray(sample_ids, np.int64)[:n]
    for c in range(arity):
        m[:, 1 + c] = np.asarray(cols[c], np.int64)[:n]
    return m


def gpu_rel(eng, rel):
    o = eng.output(rel)
    keys = [tuple(k) for k in _key_matrix(o.sample_ids, o.cols, o.arity, o.n).tolist()]
    return o, keys


def oracle_rel(res, rel):
    r = res.relations[rel]
    keys = [tuple(k) for k in _key_matrix(r.sample_ids, r.cols.T, r.cols.shape[1], len(r)).tolist()]
    return r, keys


def assert_parity(eng, res, rel, semiring, samples=None, check_grads=True, exact=False):
    """Tuple sets bit-exact; tags within the semiring's tolerance; gradients
    (fact ids exact, values 1e-6 rel).  `samples`: restrict the GPU side to
    the oracle's sample subset.  Vectorised: full-size outputs (C2 `path`,
    67M rows) compare in seconds."""
    o = eng.output(rel)
    r = res.relations[rel]
    G = _key_matrix(o.sample_ids, o.cols, o.arity, o.n)
    O = _key_matrix(r.sample_ids, r.cols.T, r.cols.shape[1], len(r))
    idx = np.arange(G.shape[0])
    if samples is not None:
        idx = np.nonzero(np.isin(G[:, 0], np.asarray(list(samples), np.int64)))[0]
        G = G[idx]
    if G.shape != O.shape or not np.array_equal(G, O):
        gs = set(map(tuple, G.tolist()))
        os_ = set(map(tuple, O.tolist()))
        raise AssertionError(f"{rel}: tuple sets differ (gpu {G.shape[0]} vs oracle {O.shape[0]}): "
                             f"{sorted(gs ^ os_)[:10]}")
    gk = G
    if semiring != 0:
        gp = o.probs[idx]
        tol = 0.0 if exact else REL_TOL[semiring]
        if tol == 0.0:
            bad = np.nonzero(gp.view(np.uint32) != r.tags.view(np.uint32))[0]
            assert bad.size == 0, f"{rel}: {bad.size} tags differ, e.g. {[(gk[i].tolist(), gp[i], r.tags[i]) for i in bad[:5]]}"
        else:
            err = np.abs(gp.astype(np.float64) - r.tags) / np.maximum(np.abs(r.tags.astype(np.float64)), 1e-30)
            assert float(err.max(initial=0.0)) <= tol, f"{rel}: max rel err {err.max()}"
    if semiring in (3, 4, 5) and check_grads and r.grad_offsets is not None:
        assert o.grad_offsets is not None, "GPU produced no gradients"
        goff = np.asarray(o.grad_offsets, np.int64)
        glen = goff[idx + 1] - goff[idx]
        olen = np.diff(np.asarray(r.grad_offsets, np.int64))
        bad = np.nonzero(glen != olen)[0]
        assert bad.size == 0, f"{rel} {gk[bad[0]].tolist()}: proof sizes differ {glen[bad[0]]} vs {olen[bad[0]]}"
        # gather the selected rows' CSR segments in one pass
        sel = np.repeat(goff[idx] - np.concatenate([[0], np.cumsum(glen)[:-1]]), glen) + np.arange(int(glen.sum()))
        gf = np.asarray(o.grad_fact_ids)[sel]
        gv = np.asarray(o.grad_values)[sel].astype(np.float64)
        of = np.asarray(r.grad_fact_ids)[:sel.shape[0]]
        ov = np.asarray(r.grad_values)[:sel.shape[0]].astype(np.float64)
        if not np.array_equal(gf, of):
            j = int(np.searchsorted(np.cumsum(glen), int(np.nonzero(gf != of)[0][0]), side="right"))
            raise AssertionError(f"{rel} {gk[j].tolist()}: proof differs")
        e = np.abs(gv - ov) / np.maximum(np.abs(ov), 1e-30)
        assert float(e.max(initial=0.0)) <= GRAD_TOL, f"{rel}: grad err {e.max()}"
    return int(G.shape[0])


def run_both(w, semiring=None, samples=None, outputs=(), threads=0):
    sr = w.semiring if semiring is None else semiring
    eng, stats, _ = engine_run(w, sr)
    res = oracle.run(w.program, sr, w.batch_size, w.facts, outputs=outputs, samples=samples, threads=threads)
    return eng, stats, res
