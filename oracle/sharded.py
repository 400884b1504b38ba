"""TEST INFRASTRUCTURE ONLY: numpy restatement of the column-sharded first cut that
csrc/sweep.cu (decompose_sharded) and csrc/qrcp_wide.cu (WideQrcp with a ShardSpec) run
across GPUs, for the world-size > 1 tests on CPU over torch.distributed (gloo).

The protocol, per pass-1 step t (the greedy QRCP of factor.cpp:62-135 with its columns
split across ranks):
  1. every rank exports a record (kind, norm^2, global position, global column, column):
     its best unpivoted column by (norm desc, global position asc), kind 1; or, when it
     has none, the column at position t if it owns it, kind 2; else kind 0;
  2. the records are all-gathered and every rank picks the same winner (best kind-1
     record, else the kind-2 one), swaps positions t <-> winner in the replicated global
     permutation (factor.cpp:88-93), and builds the same dlarfg reflector (factor.cpp:24-38)
     from the winner's column;
  3. every rank applies it to its own columns and downdates their norms with the 1e-16
     recompute guard (factor.cpp:98-107).
Pass 2 needs R_B of B = R1[:s, :]^T only: each rank reduces its rows of B to a triangle,
the triangles are all-gathered, stacked in rank order and factored again.

Only tests/ import this module; the product path never does.
"""
from __future__ import annotations

import numpy as np


def shard_range(dims, method: str, nranks: int, rank: int):
    """(lo, hi, rows, cols) -- restates ttg::shard_range (csrc/sweep.cu)."""
    d = len(dims)
    total = int(np.prod(dims))
    first = dims[0] if method == "ulv" else dims[d - 1]
    count = total // first
    if count % nranks:
        raise ValueError(f"sharded dimension {count} is not divisible by {nranks} ranks")
    per = count // nranks
    lo, hi = per * rank, per * (rank + 1)
    return (lo, hi, first, per) if method == "ulv" else (lo, hi, per, first)


def _householder(x):
    """make_householder (factor.cpp:24-38): v (v[0] = 1), beta, and the new leading entry."""
    alpha = x[0]
    sigma = float(np.dot(x[1:], x[1:])) if x.size > 1 else 0.0
    v = np.zeros_like(x)
    v[0] = 1.0
    if x.size <= 1 or sigma == 0.0:
        return v, 0.0, alpha
    mu = np.sqrt(alpha * alpha + sigma)
    smu = np.copysign(mu, alpha)
    v0 = alpha + smu
    v[1:] = x[1:] / v0
    return v, (v0 * v0) / (smu * v0), -smu


def sharded_pass1(W_local: np.ndarray, off: int, N_global: int, steps: int, allgather):
    """Greedy QRCP of the k x N_global matrix whose columns [off, off + N_local) are
    W_local. allgather(x: 1-d float64) -> (G, x.size) array in rank order.

    Returns (piv, R_local, Q): piv[t] = global column of step t, R_local = rows 0..steps-1
    of R for the local columns (by original column), Q = the k x steps economy Q."""
    k, nl = W_local.shape
    A = np.array(W_local, dtype=np.float64, copy=True)
    nu = np.einsum("ij,ij->j", A, A)
    cref = nu.copy()
    pos = off + np.arange(nl)
    perm = np.arange(N_global)
    R = np.zeros((steps, nl))
    refl = []
    piv = []
    for t in range(steps):
        live = np.flatnonzero(pos >= t)
        rec = np.zeros(4 + k)
        if live.size:
            order = np.lexsort((pos[live], -nu[live]))  # norm desc, position asc
            j = live[order[0]]
            rec[:4] = (1.0, nu[j], pos[j], off + j)
            rec[4:] = A[:, j]
        else:
            ct = perm[t]
            if off <= ct < off + nl:
                rec[:4] = (2.0, 0.0, t, ct)
                rec[4:] = A[:, ct - off]
        recs = allgather(rec)
        ones = [g for g in range(recs.shape[0]) if recs[g, 0] == 1.0]
        if ones:
            w = min(ones, key=lambda g: (-recs[g, 1], recs[g, 2]))
        else:
            w = next(g for g in range(recs.shape[0]) if recs[g, 0] == 2.0)
        gpos, gcol = int(recs[w, 2]), int(recs[w, 3])
        col = recs[w, 4:]
        ct = perm[t]
        perm[t], perm[gpos] = gcol, ct
        if off <= gcol < off + nl:
            pos[gcol - off] = t
        if ct != gcol and off <= ct < off + nl:
            pos[ct - off] = gpos
        piv.append(gcol)
        v, beta, rtt = _householder(col[t:])
        refl.append((v, beta))
        # apply H_t to the local columns (rows t..), the pivot column gets (rtt, 0, ...)
        sub = A[t:, :]
        sub -= np.outer(v, beta * (v @ sub))
        if off <= gcol < off + nl:
            A[t, gcol - off] = rtt
            A[t + 1:, gcol - off] = 0.0
        R[t, :] = np.where(pos < t, 0.0, A[t, :])
        if off <= gcol < off + nl:
            R[t, gcol - off] = rtt
        # downdate the unpivoted norms with the recompute guard
        rest = np.flatnonzero(pos > t)
        nu[rest] = nu[rest] - A[t, rest] ** 2
        bad = rest[(nu[rest] < 1e-16 * cref[rest]) | (nu[rest] < 0.0)]
        for j in bad:
            nu[j] = float(np.dot(A[t + 1:, j], A[t + 1:, j]))
            cref[j] = nu[j]
    Q = np.eye(k)[:, :steps].copy()
    for t in range(steps - 1, -1, -1):
        v, beta = refl[t]
        Q[t:, :] -= np.outer(v, beta * (v @ Q[t:, :]))
    return np.array(piv, dtype=np.int64), R, Q


def sharded_rb(R_local: np.ndarray, allgather) -> np.ndarray:
    """R_B (s x s) of B = R1^T over all ranks: local triangle, all-gather, stack, refactor."""
    s = R_local.shape[0]
    B = R_local.T
    if B.shape[0] >= s:
        tri = np.linalg.qr(B, mode="r")
    else:
        tri = np.zeros((s, s))
        tri[:B.shape[0], :] = np.linalg.qr(B, mode="r")
    stack = allgather(tri.reshape(-1, order="F")).reshape(-1, s * s)
    tall = np.vstack([blk.reshape(s, s, order="F") for blk in stack])
    return np.linalg.qr(tall, mode="r")


def gather_carry_urv(mine: np.ndarray, allgather) -> np.ndarray:
    """Rank blocks (N_local x r, column-major) -> the N_global x r carry (row blocks)."""
    nl, r = mine.shape
    blocks = allgather(mine.reshape(-1, order="F")).reshape(-1, nl * r)
    return np.vstack([b.reshape(nl, r, order="F") for b in blocks])


def gather_carry_ulv(mine: np.ndarray, allgather) -> np.ndarray:
    """Rank blocks (r x N_local) -> the r x N_global carry (column blocks, no repack)."""
    r, nl = mine.shape
    flat = allgather(mine.reshape(-1, order="F")).reshape(-1)
    return flat.reshape(r, -1, order="F")


def kshard_gram_pass1(W_rows: np.ndarray, s: int, allgather):
    """Row-sharded tall pass 1 (csrc/sweep.cu GramPass1 with a comm): each rank holds a row
    block of the k x N matrix W; the ranks' Gram matrices are all-gathered and summed in
    rank order, then the pivoted Cholesky of G = W^T W picks pivots by (residual diagonal
    desc, position asc) -- the qr_col_pivot rule -- and builds R row by row.
    Returns (piv, R rows by original column (s x N), local rows of Q[:, :s])."""
    N = W_rows.shape[1]
    Gl = W_rows.T @ W_rows
    G = allgather(Gl.reshape(-1)).reshape(-1, N, N).sum(axis=0)
    D = np.diag(G).copy()
    pos = np.arange(N)
    perm = np.arange(N)
    R = np.zeros((s, N))
    piv = []
    for t in range(s):
        live = np.flatnonzero(pos >= t)
        order = np.lexsort((pos[live], -D[live]))
        jp = live[order[0]]
        pp, ct = pos[jp], perm[t]
        perm[t], perm[pp] = jp, ct
        pos[jp], pos[ct] = t, pp
        piv.append(jp)
        rtt = np.sqrt(max(D[jp], 0.0))
        for j in range(N):
            if j == jp:
                R[t, j] = rtt
            elif pos[j] < t:
                R[t, j] = 0.0
            else:
                a = G[jp, j] - R[:t, jp] @ R[:t, j]
                R[t, j] = a / rtt if rtt > 0 else 0.0
                D[j] -= R[t, j] ** 2
    piv = np.array(piv)
    R11 = R[:, piv]  # s x s upper triangular over positions
    Q = np.linalg.solve(R11.T, W_rows[:, piv].T).T  # q R11 = x
    return piv, R, Q
