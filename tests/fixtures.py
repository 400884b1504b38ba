"""Seeded inputs for parity tests, built with the reference's own generators
(generators.cpp via oracle/_ref) following SURVEY.md Appendix C, so both sides see the
same host buffer."""
from __future__ import annotations

import numpy as np


def planted_plus_noise(ref, dims, ranks, seed, rho):
    """A = A0 + (rho |A0| / |E|) E with A0 = reconstruct(gen_planted_tt(seed)),
    E = gen_gaussian(seed + 1)."""
    a0 = ref.gen_planted_dense(dims, ranks, seed)
    if rho == 0.0:
        return a0
    e = ref.gen_gaussian(dims, seed + 1)
    return a0 + (rho * ref.frobenius_norm(a0) / ref.frobenius_norm(e)) * e


def shifted_hilbert(dims, shift=None):
    """A(i1..id) = 1 / (i1 + ... + id - shift), 1-based indices, first index fastest.
    The default shift d-1 puts the value 1 at the origin (BASELINE config 2: d=5, shift 4)."""
    if shift is None:
        shift = len(dims) - 1
    grids = np.meshgrid(*[np.arange(1, n + 1, dtype=np.float64) for n in dims], indexing="ij")
    s = sum(grids) - shift
    return (1.0 / s).ravel(order="F")


def cfg1(ref):
    return planted_plus_noise(ref, [20] * 4, [1, 5, 5, 5, 1], 1, 1e-8), [20] * 4, [1, 5, 5, 5, 1]
