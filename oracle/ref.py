"""TEST INFRASTRUCTURE ONLY: ctypes access to the UNMODIFIED reference library.

``oracle/_ref/libttutv_ref.so`` is compiled from /root/reference/proj/src by
``oracle/Makefile`` (target ``ref``) together with ``oracle/ref_shim.cpp``. It is the
checker for the device engine (tests/, __graft_entry__.smoke()) and the CPU arm of
bench.py; it is never used by the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_ref" / "libttutv_ref.so"

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int64)

_lib = None


def available() -> bool:
    return LIB.exists()


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            raise ImportError(f"reference oracle not built: {LIB} (make -C oracle ref)")
        h = C.CDLL(str(LIB), mode=os.RTLD_LOCAL)
        h.ref_last_error.restype = C.c_char_p
        h.ref_decompose.argtypes = [dp, ip, C.c_int, C.c_int, C.c_int, C.c_int, ip, C.c_double, dp, C.c_int, C.c_int,
                                    C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        h.ref_result_free.argtypes = [C.c_void_p]
        h.ref_result_order.argtypes = [C.c_void_p]
        h.ref_result_core_dims.argtypes = [C.c_void_p, C.c_int, ip]
        h.ref_result_core_copy.argtypes = [C.c_void_p, C.c_int, dp]
        h.ref_result_report.argtypes = [C.c_void_p, dp, ip, dp, C.POINTER(C.c_int), dp, dp]
        h.ref_result_warning.argtypes = [C.c_void_p, C.c_int]
        h.ref_result_warning.restype = C.c_char_p
        h.ref_result_rse.argtypes = [C.c_void_p, dp, ip, C.c_int, C.c_int64, dp]
        h.ref_result_reconstruct.argtypes = [C.c_void_p, C.c_int64, dp]
        h.ref_qr_col_pivot.argtypes = [dp, C.c_int64, C.c_int64, dp, dp, ip]
        h.ref_utv.argtypes = [dp, C.c_int64, C.c_int64, C.c_int, C.c_int, dp, dp, dp]
        h.ref_svd.argtypes = [dp, C.c_int64, C.c_int64, dp, dp, dp]
        h.ref_truncate.argtypes = [C.c_int, dp, dp, dp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_double, ip,
                                   dp, dp, dp, dp]
        h.ref_gen_gaussian.argtypes = [ip, C.c_int, C.c_uint64, dp]
        h.ref_gen_hilbert.argtypes = [ip, C.c_int, dp]
        h.ref_gen_planted_dense.argtypes = [ip, C.c_int, ip, C.c_uint64, C.c_int64, dp]
        h.ref_gen_planted_cores.argtypes = [ip, C.c_int, ip, C.c_uint64, dp]
        h.ref_frobenius_norm.argtypes = [dp, C.c_int64]
        h.ref_frobenius_norm.restype = C.c_double
        h.ref_set_parallel.argtypes = [C.c_int]
        h.ref_sweep_trace.argtypes = [dp, ip, C.c_int, C.c_int, C.c_int, ip, C.c_double, C.POINTER(C.c_void_p)]
        h.ref_trace_result.argtypes = [C.c_void_p]
        h.ref_trace_result.restype = C.c_void_p
        h.ref_trace_free.argtypes = [C.c_void_p]
        h.ref_trace_cut.argtypes = [C.c_void_p, C.c_int, ip, ip, dp]
        h.ref_trace_cut.restype = C.c_int64
        h.ref_trace_cut_copy.argtypes = [C.c_void_p, C.c_int, dp, dp]
        h.ref_read_tensor.argtypes = [C.c_char_p, ip, C.POINTER(C.c_int), ip, dp]
        h.ref_write_tensor.argtypes = [C.c_char_p, dp, ip, C.c_int]
        h.ref_write_tt.argtypes = [C.c_char_p, C.c_int, ip, ip, dp]
        _lib = h
    return _lib


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(st):
    if st != 0:
        raise RefError(st, lib().ref_last_error().decode())


def _d(a):
    return a.ctypes.data_as(dp)


def _i(a):
    return a.ctypes.data_as(ip)


@dataclass
class RefResult:
    cores: list
    step_errors: list
    ranks_chosen: list
    bound: float
    bound_kind: int
    input_norm: float
    wall_time_ms: float
    warnings: list
    handle: object = None


class _Handle:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        if self.h:
            lib().ref_result_free(self.h)


def decompose(a, dims, method="urv", sweep="r2l", ranks=None, eps=0.0, weights=(), refine=1, retain=0,
              debug=False) -> RefResult:
    a = np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1))
    dims = np.ascontiguousarray(np.asarray(dims, np.int64))
    d = dims.size
    m = {"svd": 0, "ulv": 1, "urv": 2}[method]
    s = {"l2r": 0, "r2l": 1}[sweep]
    r = np.ascontiguousarray(np.asarray(ranks if ranks is not None else [1] * (d + 1), np.int64))
    w = np.ascontiguousarray(np.asarray(list(weights) or [0.0], np.float64))
    h = C.c_void_p()
    _check(lib().ref_decompose(_d(a), _i(dims), d, m, s, int(ranks is not None), _i(r), float(eps), _d(w),
                               len(weights), int(refine), int(retain), int(debug), C.byref(h)))
    hh = _Handle(h)
    order = lib().ref_result_order(h)
    cores = []
    for k in range(order):
        cd = np.zeros(3, np.int64)
        lib().ref_result_core_dims(h, k, _i(cd))
        buf = np.empty(int(np.prod(cd)), np.float64)
        lib().ref_result_core_copy(h, k, _d(buf))
        cores.append(buf.reshape(tuple(cd), order="F"))
    se = np.zeros(max(order - 1, 1), np.float64)
    rc = np.zeros(order + 1, np.int64)
    b, ni, wt = C.c_double(), C.c_double(), C.c_double()
    bk = C.c_int()
    nw = lib().ref_result_report(h, _d(se), _i(rc), C.byref(b), C.byref(bk), C.byref(ni), C.byref(wt))
    warns = [lib().ref_result_warning(h, i).decode() for i in range(nw)]
    return RefResult(cores, se[: max(order - 1, 0)].tolist(), rc.tolist(), b.value, bk.value, ni.value, wt.value,
                     warns, hh)


class _TraceHandle:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        if self.h:
            lib().ref_trace_free(self.h)


def _result_from(h, owner) -> RefResult:
    order = lib().ref_result_order(h)
    cores = []
    for k in range(order):
        cd = np.zeros(3, np.int64)
        lib().ref_result_core_dims(h, k, _i(cd))
        buf = np.empty(int(np.prod(cd)), np.float64)
        lib().ref_result_core_copy(h, k, _d(buf))
        cores.append(buf.reshape(tuple(cd), order="F"))
    se = np.zeros(max(order - 1, 1), np.float64)
    rc = np.zeros(order + 1, np.int64)
    b, ni, wt = C.c_double(), C.c_double(), C.c_double()
    bk = C.c_int()
    nw = lib().ref_result_report(h, _d(se), _i(rc), C.byref(b), C.byref(bk), C.byref(ni), C.byref(wt))
    warns = [lib().ref_result_warning(h, i).decode() for i in range(nw)]
    return RefResult(cores, se[: max(order - 1, 0)].tolist(), rc.tolist(), b.value, bk.value, ni.value, wt.value,
                     warns, owner)


def sweep_trace(a, dims, method="urv", ranks=None, eps=0.0):
    """ULV-L2R / URV-R2L through the reference's public calls (ref_shim.cpp ref_sweep_trace),
    returning (RefResult, cuts) with per cut (unfolding order) m, n, |diag T| (all p), the
    kept-mass vector and the directly computed discarded norm (-1 when skipped)."""
    a = np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1))
    dims = np.ascontiguousarray(np.asarray(dims, np.int64))
    d = dims.size
    r = np.ascontiguousarray(np.asarray(ranks if ranks is not None else [1] * (d + 1), np.int64))
    h = C.c_void_p()
    _check(lib().ref_sweep_trace(_d(a), _i(dims), d, {"ulv": 1, "urv": 2}[method], int(ranks is not None), _i(r),
                                 float(eps), C.byref(h)))
    owner = _TraceHandle(h)
    res = _result_from(lib().ref_trace_result(h), owner)
    cuts = []
    for k in range(d - 1):
        m, n, direct = C.c_int64(), C.c_int64(), C.c_double()
        p = lib().ref_trace_cut(h, k, C.byref(m), C.byref(n), C.byref(direct))
        dg = np.empty(p, np.float64)
        kp = np.empty(p + 1, np.float64)
        lib().ref_trace_cut_copy(h, k, _d(dg), _d(kp))
        cuts.append(dict(m=m.value, n=n.value, diag=dg, kept=kp, direct=direct.value,
                         rank=res.ranks_chosen[k + 1], step_error=res.step_errors[k]))
    return res, cuts


def rse(res: RefResult, a, dims, cap=10**10) -> float:
    a = np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1))
    dims = np.ascontiguousarray(np.asarray(dims, np.int64))
    out = C.c_double()
    _check(lib().ref_result_rse(res.handle.h, _d(a), _i(dims), dims.size, int(cap), C.byref(out)))
    return out.value


def qr_col_pivot(a):
    a = np.asfortranarray(a, dtype=np.float64)
    m, n = a.shape
    p = min(m, n)
    q = np.zeros((m, p), order="F")
    r = np.zeros((p, n), order="F")
    perm = np.zeros(n, np.int64)
    _check(lib().ref_qr_col_pivot(_d(a), m, n, _d(q), _d(r), _i(perm)))
    return q, r, perm


def utv(a, lower, refine=1):
    a = np.asfortranarray(a, dtype=np.float64)
    m, n = a.shape
    p = min(m, n)
    u = np.zeros((m, p), order="F")
    t = np.zeros((p, p), order="F")
    v = np.zeros((n, p), order="F")
    _check(lib().ref_utv(_d(a), m, n, int(lower), int(refine), _d(u), _d(t), _d(v)))
    return u, t, v


def gen_gaussian(dims, seed):
    dims = np.ascontiguousarray(np.asarray(dims, np.int64))
    out = np.empty(int(np.prod(dims)), np.float64)
    _check(lib().ref_gen_gaussian(_i(dims), dims.size, int(seed), _d(out)))
    return out


def gen_hilbert(dims):
    dims = np.ascontiguousarray(np.asarray(dims, np.int64))
    out = np.empty(int(np.prod(dims)), np.float64)
    _check(lib().ref_gen_hilbert(_i(dims), dims.size, _d(out)))
    return out


def gen_planted_dense(dims, ranks, seed, cap=10**10):
    dims = np.ascontiguousarray(np.asarray(dims, np.int64))
    ranks = np.ascontiguousarray(np.asarray(ranks, np.int64))
    out = np.empty(int(np.prod(dims)), np.float64)
    _check(lib().ref_gen_planted_dense(_i(dims), dims.size, _i(ranks), int(seed), int(cap), _d(out)))
    return out


def gen_planted_cores(dims, ranks, seed):
    dims = [int(x) for x in dims]
    ranks = [int(x) for x in ranks]
    tot = sum(ranks[k] * dims[k] * ranks[k + 1] for k in range(len(dims)))
    out = np.empty(tot, np.float64)
    dd = np.ascontiguousarray(np.asarray(dims, np.int64))
    rr = np.ascontiguousarray(np.asarray(ranks, np.int64))
    _check(lib().ref_gen_planted_cores(_i(dd), dd.size, _i(rr), int(seed), _d(out)))
    cores, off = [], 0
    for k in range(len(dims)):
        n = ranks[k] * dims[k] * ranks[k + 1]
        cores.append(out[off:off + n].reshape((ranks[k], dims[k], ranks[k + 1]), order="F"))
        off += n
    return cores


def frobenius_norm(a) -> float:
    a = np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1))
    return lib().ref_frobenius_norm(_d(a), a.size)


def set_parallel(enabled: bool):
    lib().ref_set_parallel(int(enabled))


def read_tensor(path):
    """The reference's read_tensor: (dims, flat payload) or raises RefError; a ParseError
    (code 3) carries `.offset`."""
    off = np.zeros(1, np.int64)
    order = C.c_int()
    dims = np.zeros(255, np.int64)
    st = lib().ref_read_tensor(str(path).encode(), _i(off), C.byref(order), _i(dims), None)
    if st != 0:
        e = RefError(st, lib().ref_last_error().decode())
        e.message, e.offset = lib().ref_last_error().decode(), int(off[0])
        raise e
    d = dims[: order.value].copy()
    out = np.zeros(int(np.prod(d)), np.float64)
    _check(lib().ref_read_tensor(str(path).encode(), _i(off), C.byref(order), _i(dims), _d(out)))
    return d.tolist(), out


def write_tensor(path, a, dims):
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    dims = np.asarray(dims, dtype=np.int64)
    _check(lib().ref_write_tensor(str(path).encode(), _d(a), _i(dims), dims.size))


def write_tt(path, cores):
    """write_tt of cores given as (r_{k-1}, I_k, r_k) arrays in storage (Fortran) order."""
    ranks = np.array([c.shape[0] for c in cores] + [cores[-1].shape[2]], np.int64)
    dims = np.array([c.shape[1] for c in cores], np.int64)
    flat = np.concatenate([np.asarray(c, np.float64).reshape(-1, order="F") for c in cores])
    _check(lib().ref_write_tt(str(path).encode(), len(cores), _i(ranks), _i(dims), _d(flat)))
