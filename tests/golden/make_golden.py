"""Regenerate tests/golden/*.npz from the UNMODIFIED reference library (oracle/_ref).

Run in the build container (where /root/reference exists and `make -C oracle ref` has been
run):  python tests/golden/make_golden.py
Inputs are produced by the reference's own seeded generators (generators.cpp), so the
fixtures only store seeds plus the reference's outputs.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import ref  # noqa: E402

OUT = Path(__file__).resolve().parent


def matrix(m, n, seed):
    return ref.gen_gaussian([m, n], seed).reshape((m, n), order="F")


QR_CASES = {
    "g30x20": lambda: matrix(30, 20, 1),
    "g20x30": lambda: matrix(20, 30, 2),
    "g7x1": lambda: matrix(7, 1, 3),
    "g1x7": lambda: matrix(1, 7, 4),
    "g12x12": lambda: matrix(12, 12, 5),
    # duplicated columns: exact pivot ties resolved to the lowest position
    "dup9x16": lambda: np.asfortranarray(np.repeat(matrix(9, 4, 6), 4, axis=1)),
    "zero5x3": lambda: np.zeros((5, 3), order="F"),
    "hilbert16x24": lambda: ref.gen_hilbert([16, 24]).reshape((16, 24), order="F"),
}

SWEEP_CASES = [
    # name, dims, planted ranks (None: hilbert), seed, rho, method, sweep, mode, arg, retain
    ("cfg1_urv_rank", [20] * 4, [1, 5, 5, 5, 1], 1, 1e-8, "urv", "r2l", "rank", [1, 5, 5, 5, 1], 0),
    ("cfg1_ulv_rank", [20] * 4, [1, 5, 5, 5, 1], 1, 1e-8, "ulv", "l2r", "rank", [1, 5, 5, 5, 1], 0),
    ("cfg1_svd_rank", [20] * 4, [1, 5, 5, 5, 1], 1, 1e-8, "svd", "l2r", "rank", [1, 5, 5, 5, 1], 0),
    ("cfg1_urv_tol", [20] * 4, [1, 5, 5, 5, 1], 1, 1e-8, "urv", "r2l", "tol", 1e-6, 0),
    ("cfg1_ulv_tol", [20] * 4, [1, 5, 5, 5, 1], 1, 1e-8, "ulv", "l2r", "tol", 1e-6, 0),
    ("o6_urv_rank", [6] * 6, [1, 4, 5, 5, 5, 4, 1], 3, 1e-4, "urv", "r2l", "rank", [1, 4, 5, 5, 5, 4, 1], 0),
    ("o6_ulv_rank", [6] * 6, [1, 4, 5, 5, 5, 4, 1], 3, 1e-4, "ulv", "l2r", "rank", [1, 4, 5, 5, 5, 4, 1], 0),
    ("hilb_urv_tol", [12] * 4, None, 0, 0.0, "urv", "r2l", "tol", 1e-6, 0),
    ("hilb_ulv_tol", [12] * 4, None, 0, 0.0, "ulv", "l2r", "tol", 1e-6, 0),
    ("alg4_l11", [6, 5, 7, 4], [1, 3, 4, 2, 1], 11, 1e-3, "ulv", "r2l", "rank", [1, 3, 4, 2, 1], 0),
    ("alg4_full", [6, 5, 7, 4], [1, 3, 4, 2, 1], 11, 1e-3, "ulv", "r2l", "rank", [1, 3, 4, 2, 1], 1),
    ("clamp_ulv", [4, 6, 1], [1, 1, 1, 1], 5, 0.0, "ulv", "l2r", "rank", [1, 9, 9, 1], 0),
]


def sweep_input(dims, ranks, seed, rho):
    if ranks is None:  # shifted Hilbert, value 1 at the origin
        return hilbert_shifted(dims)
    a0 = ref.gen_planted_dense(dims, ranks, seed)
    if rho == 0.0:
        return a0
    e = ref.gen_gaussian(dims, seed + 1)
    return a0 + (rho * ref.frobenius_norm(a0) / ref.frobenius_norm(e)) * e


def hilbert_shifted(dims):
    g = np.meshgrid(*[np.arange(1, n + 1, dtype=np.float64) for n in dims], indexing="ij")
    return (1.0 / (sum(g) - (len(dims) - 1))).ravel(order="F")


def main():
    qr = {}
    for name, fn in QR_CASES.items():
        a = fn()
        q, r, perm = ref.qr_col_pivot(a)
        qr[f"{name}/a"], qr[f"{name}/q"], qr[f"{name}/r"], qr[f"{name}/perm"] = a, q, r, perm
        for lower in (0, 1):
            for refine in (0, 1, 2):
                u, t, v = ref.utv(a, lower, refine)
                key = f"{name}/utv{lower}{refine}"
                qr[key + "/u"], qr[key + "/t"], qr[key + "/v"] = u, t, v
    np.savez_compressed(OUT / "factor.npz", **qr)

    sw = {}
    for name, dims, ranks, seed, rho, method, sweep, mode, arg, retain in SWEEP_CASES:
        a = sweep_input(dims, ranks, seed, rho)
        kw = dict(ranks=arg) if mode == "rank" else dict(eps=arg)
        res = ref.decompose(a, dims, method, sweep, retain=retain, **kw)
        sw[f"{name}/sum_a"] = np.array([a.sum(), ref.frobenius_norm(a)])
        sw[f"{name}/ranks"] = np.array(res.ranks_chosen)
        sw[f"{name}/step_errors"] = np.array(res.step_errors)
        sw[f"{name}/scalars"] = np.array([res.bound, res.bound_kind, res.input_norm, ref.rse(res, a, dims)])
        for k, c in enumerate(res.cores):
            sw[f"{name}/core{k}"] = c
        sw[f"{name}/warnings"] = np.array(res.warnings or [""])
    np.savez_compressed(OUT / "sweeps.npz", **sw)

    gen = {"gauss_1000_7": ref.gen_gaussian([1000], 7), "hilbert_5x6x7": ref.gen_hilbert([5, 6, 7]),
           "planted_4x5x6_123_42": np.concatenate([c.ravel(order="F") for c in
                                                  ref.gen_planted_cores([4, 5, 6], [1, 2, 3, 1], 42)])}
    np.savez_compressed(OUT / "generators.npz", **gen)
    print("wrote", sorted(p.name for p in OUT.glob("*.npz")))


if __name__ == "__main__":
    main()
