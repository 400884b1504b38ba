"""Test helper: replay the reference sweeps (tt_decomp.cpp:156-339) cut by cut with the
reference's own factorisations (oracle/_ref ``ulv``/``urv``), to expose the per-cut
quantities the reference API does not return (|diag T11|, ranks, residual masses).
Only the cheap glue (reshape, leading-block carry product, kept-mass scan) is numpy.
"""
from __future__ import annotations

import math

import numpy as np


def kept_mass(t: np.ndarray, lower: bool) -> np.ndarray:
    """kept_mass_lower / kept_mass_upper (factor.cpp:479-499), same summation order."""
    p = t.shape[0]
    kept = np.zeros(p + 1)
    acc = 0.0
    for r in range(1, p + 1):
        s = 0.0
        for j in range(r):
            v = t[r - 1, j] if lower else t[j, r - 1]
            s += v * v
        acc += s
        kept[r] = acc
    return kept


def pick_rank(kept: np.ndarray, eps: float) -> int:
    p = kept.size - 1
    if eps == 0.0:
        return p
    target = kept[-1] - eps * eps
    for r in range(1, p):
        if kept[r] >= target:
            return r
    return p


def replay(ref, a: np.ndarray, dims, method: str, ranks=None, eps=None):
    """Returns a list (unfolding order) of dicts: rank, diag, m, n, step_error."""
    dims = [int(x) for x in dims]
    d = len(dims)
    n_tot = int(np.prod(dims))
    a = np.asarray(a, np.float64).reshape(-1)
    norm = ref.frobenius_norm(a)
    budgets = [eps * norm / math.sqrt(max(d - 1, 1))] * (d - 1) if ranks is None else None
    cuts = [None] * (d - 1)
    if method == "ulv":
        c = a.reshape((dims[0], n_tot // dims[0]), order="F")
        for k in range(1, d):
            m, n = c.shape
            p = min(m, n)
            u, t, v = ref.utv(c, lower=True, refine=1)
            kept = kept_mass(t, True)
            r = min(ranks[k], p) if ranks is not None else pick_rank(kept, budgets[k - 1])
            carry = t[:r, :r] @ v[:, :r].T
            cuts[k - 1] = dict(rank=r, diag=np.abs(np.diag(t)[:r]), m=m, n=n,
                               step_error=math.sqrt(max(0.0, kept[-1] - kept[r])))
            if k < d - 1:
                c = carry.reshape((r * dims[k], carry.shape[1] // dims[k]), order="F")
    else:
        c = a.reshape((n_tot // dims[-1], dims[-1]), order="F")
        for k in range(d, 1, -1):
            m, n = c.shape
            p = min(m, n)
            u, t, v = ref.utv(c, lower=False, refine=1)
            kept = kept_mass(t, False)
            r = min(ranks[k - 1], p) if ranks is not None else pick_rank(kept, budgets[k - 2])
            carry = u[:, :r] @ t[:r, :r]
            cuts[k - 2] = dict(rank=r, diag=np.abs(np.diag(t)[:r]), m=m, n=n,
                               step_error=math.sqrt(max(0.0, kept[-1] - kept[r])))
            if k > 2:
                c = carry.reshape((m // dims[k - 2], dims[k - 2] * r), order="F")
    return cuts
