"""Whole-step roofline of a TT-UTV sweep.

The work model counts exactly the loops of the reference's qr_col_pivot
(src/factor.cpp:62-135) for the cut shapes the sweep visits with the chosen ranks:

  QRCP(m, n), p = min(m, n): initial norms 2mn; per step s: 2(m-s) reflector,
      4(m-s)(n-s-1) apply_reflector, 2(n-s-1) norm downdate; Q formation
      sum_{s<p} 4(m-s)(p-s)
  ULV(c: m x n) = QRCP(m, n) + QRCP(n, p); URV(c) = QRCP(n, m) + QRCP(m, p)
      (factor.cpp:384-417, refine_passes = 1)
  carry: L2R 2 r^2 n, R2L 2 m r^2
  F_min: the same factorisation with pass 2's Q formation limited to the r kept columns,
      sum_{s<r} 4(N-s)(r-s), N the long side of the cut
  B_comp per cut = 8 (m n + |core| + |carry|) bytes

T_roof = sum over cuts of max(F_min / P_FP64, B_comp / BW_HBM); the step's roofline
fraction is T_roof / T_dev. The formulas are summed in closed form (no per-step loops).
"""
from __future__ import annotations


def _s1(n):  # sum_{s<n} s
    return n * (n - 1) // 2


def _s2(n):  # sum_{s<n} s^2
    return (n - 1) * n * (2 * n - 1) // 6


def _sum_prod(a, b, n):
    """sum_{s<n} (a - s)(b - s)."""
    return n * a * b - (a + b) * _s1(n) + _s2(n)


def qrcp_flops(m: int, n: int, q_cols: int | None = None) -> int:
    """Flops of qr_col_pivot(m x n) (Appendix B); q_cols limits Q formation to that many columns."""
    p = min(m, n)
    f = 2 * m * n
    f += 2 * (p * m - _s1(p))                     # reflectors
    f += 4 * _sum_prod(m, n - 1, p)               # apply_reflector
    f += 2 * (p * (n - 1) - _s1(p))               # norm downdate
    qc = p if q_cols is None else min(q_cols, p)
    f += 4 * _sum_prod(m, qc if q_cols is not None else p, qc)  # Q formation (columns j >= s)
    return f


def cut_shapes(dims, ranks, method):
    """(m, n, r) of each cut in visiting order for ULV-L2R (method 'ulv') or URV-R2L ('urv')."""
    d = len(dims)
    total = 1
    for x in dims:
        total *= x
    out = []
    if method == "ulv":
        m, n = dims[0], total // dims[0]
        for k in range(1, d):
            r = ranks[k]
            out.append((m, n, r))
            if k < d - 1:
                m, n = r * dims[k], n // dims[k]
    else:
        m, n = total // dims[-1], dims[-1]
        for k in range(d, 1, -1):
            r = ranks[k - 1]
            out.append((m, n, r))
            if k > 2:
                m, n = m // dims[k - 2], dims[k - 2] * r
    return out


def cut_work(m: int, n: int, r: int, method: str) -> dict:
    p = min(m, n)
    if method == "ulv":
        p1 = qrcp_flops(m, n)
        p2 = qrcp_flops(n, p)
        p2min = qrcp_flops(n, p, q_cols=r)
        carry = 2 * r * r * n
        core, carry_sz = m * r, r * n
    else:
        p1 = qrcp_flops(n, m)
        p2 = qrcp_flops(m, p)
        p2min = qrcp_flops(m, p, q_cols=r)
        carry = 2 * m * r * r
        core, carry_sz = r * n, m * r
    return {"m": m, "n": n, "r": r, "f_ref": p1 + p2 + carry, "f_min": p1 + p2min + carry,
            "b_comp": 8 * (m * n + core + carry_sz)}


def step_roofline(dims, runs, ranks_by_method: dict, p_fp64_tflops: float, bw_gbs: float) -> dict:
    """T_roof of one step (every (method, sweep) in `runs` once) with the chosen ranks."""
    cuts = []
    t_roof = 0.0
    f_min = f_ref = b_comp = 0
    for method, _sweep in runs:
        for (m, n, r) in cut_shapes(dims, ranks_by_method[method], method):
            w = cut_work(m, n, r, method)
            tf = w["f_min"] / (p_fp64_tflops * 1e12)
            tb = w["b_comp"] / (bw_gbs * 1e9)
            w.update(method=method, t_flop_ms=tf * 1e3, t_byte_ms=tb * 1e3,
                     bound="fp64" if tf >= tb else "hbm")
            cuts.append(w)
            t_roof += max(tf, tb)
            f_min += w["f_min"]
            f_ref += w["f_ref"]
            b_comp += w["b_comp"]
    return {"t_roof_ms": t_roof * 1e3, "f_min": f_min, "f_ref": f_ref, "b_comp": b_comp, "cuts": cuts}
