"""CPU check of the rounding certificate the tile kernel's composition rounds
use (tile_device.cuh certify32): an fp64 sum of n fp32 terms
formed in ANY order, S_par, certifies fl32(S_seq) of the canonical sequential
sum when every value in S_par ± d, d = (2(n + k) + 4)·2^-53·Σ|t|·1.01, rounds
to one fp32 value.  Here the claim is checked directly: over many random term
sets (mixed magnitudes, exact ties, cancellation-free nonnegative terms as in
add-mult) and random summation orders, every certified result equals the
fp32 rounding of the sequential sum; and the certificate is not vacuous.
(k = 0: one thread's reordered walk; k = P: P partial sums combined.)"""
from __future__ import annotations

import numpy as np


def _certify(s, ab, n, k):
    d = (2.0 * (n + k) + 4.0) * 2.0 ** -53 * ab * 1.01
    lo, hi = np.float32(s - d), np.float32(s + d)
    return lo == hi, lo


def _seq(terms):
    acc = 0.0
    for t in terms:
        acc = acc + float(t)
    return acc


def test_certificate_never_accepts_a_wrong_rounding():
    rng = np.random.default_rng(2503)
    certified = 0
    trials = 4000
    for trial in range(trials):
        n = int(rng.integers(1, 200))
        kind = trial % 4
        if kind == 0:    # probabilities, products of three
            t = (rng.random(n) * rng.random(n) * rng.random(n)).astype(np.float32)
        elif kind == 1:  # wide dynamic range
            t = (rng.random(n) * 10.0 ** rng.integers(-30, 1, n)).astype(np.float32)
        elif kind == 2:  # dyadic terms: exact sums that can land on fp32 ties
            t = (rng.integers(1, 2 ** 10, n) * 2.0 ** rng.integers(-40, -20, n)).astype(np.float32)
        else:            # near-equal terms
            t = np.float32(0.1) + (rng.random(n) * 1e-6).astype(np.float32)
        want = np.float32(_seq(t))
        # one thread in another order (k = 0)
        perm = rng.permutation(n)
        s = _seq(t[perm])
        ab = _seq(np.abs(t[perm]))
        ok, got = _certify(s, ab, n, 0)
        if ok:
            certified += 1
            assert got == want, (trial, got, want)
        # P partial sums over a split, combined in part order (k = P)
        P = int(rng.integers(2, 9))
        parts = [t[perm[i::P]] for i in range(P)]
        ps = [_seq(p) for p in parts]
        s2 = _seq(np.array(ps))
        ab2 = _seq(np.array([_seq(np.abs(p)) for p in parts]))
        ok2, got2 = _certify(s2, ab2, n, P)
        if ok2:
            assert got2 == want, (trial, got2, want)
    assert certified > 0.9 * trials  # the certificate decides almost every head
