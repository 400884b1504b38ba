"""TEST INFRASTRUCTURE ONLY: ctypes access to liboracle.so, the plain-C restatement of the
reference path (oracle/ttutv_oracle.c). Used by tests/ to pin against the golden
fixtures and the reference library, and by bench.py's CPU leg when oracle/_ref is absent.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int64)
_lib = None


def available() -> bool:
    return LIB.exists()


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            raise ImportError(f"oracle port not built: {LIB} (make -C oracle oracle)")
        h = C.CDLL(str(LIB))
        h.orc_last_error.restype = C.c_char_p
        h.orc_gen_gaussian.argtypes = [C.c_int64, C.c_uint64, dp]
        h.orc_gen_hilbert.argtypes = [ip, C.c_int, C.c_double, dp]
        h.orc_gen_planted_cores.argtypes = [ip, C.c_int, ip, C.c_uint64, dp]
        h.orc_sum_squares.argtypes = [dp, C.c_int64]
        h.orc_sum_squares.restype = C.c_double
        h.orc_qr_col_pivot.argtypes = [dp, C.c_int64, C.c_int64, dp, dp, ip]
        h.orc_utv.argtypes = [dp, C.c_int64, C.c_int64, C.c_int, C.c_int, dp, dp, dp]
        h.orc_svd.argtypes = [dp, C.c_int64, C.c_int64, C.c_int, C.c_double, dp, dp, dp]
        h.orc_truncate.argtypes = [C.c_int, dp, dp, dp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_double, ip,
                                   dp, dp, dp, dp]
        h.orc_reconstruct.argtypes = [dp, ip, ip, C.c_int, dp]
        h.orc_rse.argtypes = [dp, dp, C.c_int64]
        h.orc_rse.restype = C.c_double
        h.orc_decompose.argtypes = [dp, ip, C.c_int, C.c_int, C.c_int, C.c_int, ip, C.c_double, dp, C.c_int, C.c_int,
                                    C.c_int, dp, C.c_int64, ip, dp, ip, dp, C.POINTER(C.c_int), dp]
        _lib = h
    return _lib


def _d(a):
    return a.ctypes.data_as(dp)


def _i(a):
    return a.ctypes.data_as(ip)


def _check(rc):
    if rc != 0:
        raise RuntimeError(f"[{rc}] {lib().orc_last_error().decode()}")


def gen_gaussian(count, seed):
    out = np.empty(int(count), np.float64)
    lib().orc_gen_gaussian(int(count), int(seed), _d(out))
    return out


def gen_hilbert(dims, shift=0.0):
    dims = np.ascontiguousarray(dims, np.int64)
    out = np.empty(int(np.prod(dims)), np.float64)
    lib().orc_gen_hilbert(_i(dims), dims.size, float(shift), _d(out))
    return out


def gen_planted_cores(dims, ranks, seed):
    dims = np.ascontiguousarray(dims, np.int64)
    ranks = np.ascontiguousarray(ranks, np.int64)
    tot = int(sum(ranks[k] * dims[k] * ranks[k + 1] for k in range(dims.size)))
    out = np.empty(tot, np.float64)
    lib().orc_gen_planted_cores(_i(dims), dims.size, _i(ranks), int(seed), _d(out))
    return out


def reconstruct_flat(cores_flat, dims, ranks):
    dims = np.ascontiguousarray(dims, np.int64)
    ranks = np.ascontiguousarray(ranks, np.int64)
    out = np.empty(int(np.prod(dims)), np.float64)
    _check(lib().orc_reconstruct(_d(np.ascontiguousarray(cores_flat, np.float64)), _i(dims), _i(ranks), dims.size,
                                 _d(out)))
    return out


def sum_squares(a):
    a = np.ascontiguousarray(a, np.float64).reshape(-1)
    return lib().orc_sum_squares(_d(a), a.size)


def qr_col_pivot(a):
    a = np.asfortranarray(a, np.float64)
    m, n = a.shape
    p = min(m, n)
    q = np.zeros((m, p), order="F")
    r = np.zeros((p, n), order="F")
    perm = np.zeros(n, np.int64)
    _check(lib().orc_qr_col_pivot(_d(a), m, n, _d(q), _d(r), _i(perm)))
    return q, r, perm


def utv(a, lower, refine=1):
    a = np.asfortranarray(a, np.float64)
    m, n = a.shape
    p = min(m, n)
    u = np.zeros((m, p), order="F")
    t = np.zeros((p, p), order="F")
    v = np.zeros((n, p), order="F")
    _check(lib().orc_utv(_d(a), m, n, int(lower), int(refine), _d(u), _d(t), _d(v)))
    return u, t, v


def svd(a, max_sweeps=60, pair_tol=1e-14):
    a = np.asfortranarray(a, np.float64)
    m, n = a.shape
    p = min(m, n)
    u = np.zeros((m, p), order="F")
    s = np.zeros(p)
    v = np.zeros((n, p), order="F")
    _check(lib().orc_svd(_d(a), m, n, int(max_sweeps), float(pair_tol), _d(u), _d(s), _d(v)))
    return u, s, v


def truncate(kind, u, t, v, rank=0, eps=0.0):
    u = np.asfortranarray(u, np.float64)
    v = np.asfortranarray(v, np.float64)
    t = np.asfortranarray(t, np.float64)
    m, p = u.shape
    n = v.shape[0]
    u1 = np.zeros((m, p), order="F")
    v1 = np.zeros((n, p), order="F")
    t11 = np.zeros((p, p), order="F")
    r = C.c_int64()
    res = C.c_double()
    _check(lib().orc_truncate(int(kind), _d(u), _d(t), _d(v), m, n, p, int(rank), float(eps), C.byref(r), C.byref(res),
                              _d(u1), _d(t11), _d(v1)))
    rr = r.value
    return rr, res.value, u1.reshape(-1, order="F")[: m * rr].reshape((m, rr), order="F"), \
        t11.reshape(-1, order="F")[: rr * rr].reshape((rr, rr), order="F"), \
        v1.reshape(-1, order="F")[: n * rr].reshape((n, rr), order="F")


def decompose(a, dims, method="urv", sweep="r2l", ranks=None, eps=0.0, weights=(), refine=1, retain=0):
    a = np.ascontiguousarray(a, np.float64).reshape(-1)
    dims = np.ascontiguousarray(dims, np.int64)
    d = dims.size
    r = np.ascontiguousarray(ranks if ranks is not None else [1] * (d + 1), np.int64)
    w = np.ascontiguousarray(list(weights) or [0.0], np.float64)
    cap = 8 * a.size + 4096
    cores = np.zeros(cap)
    cd = np.zeros(3 * d, np.int64)
    se = np.zeros(max(d - 1, 1))
    rc = np.zeros(d + 1, np.int64)
    b, ni = C.c_double(), C.c_double()
    bk = C.c_int()
    m = {"svd": 0, "ulv": 1, "urv": 2}[method]
    s = {"l2r": 0, "r2l": 1}[sweep]
    _check(lib().orc_decompose(_d(a), _i(dims), d, m, s, int(ranks is not None), _i(r), float(eps), _d(w), len(weights),
                               int(refine), int(retain), _d(cores), cap, _i(cd), _d(se), _i(rc), C.byref(b),
                               C.byref(bk), C.byref(ni)))
    out, off = [], 0
    for k in range(d):
        shp = tuple(int(x) for x in cd[3 * k:3 * k + 3])
        sz = shp[0] * shp[1] * shp[2]
        out.append(cores[off:off + sz].reshape(shp, order="F"))
        off += sz
    return dict(cores=out, step_errors=se[: d - 1].tolist(), ranks_chosen=rc.tolist(), bound=b.value,
                bound_kind=bk.value, input_norm=ni.value)
