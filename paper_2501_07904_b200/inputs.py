"""Seeded synthetic inputs for bench.py and the tests (harness code, not the product path).

The paper's datasets are not available; BASELINE.json's configs are built from their
recipes with the reference's own generator algorithms, restated in
``hostgen/inputs.cpp`` (``lib/libttutv_inputs.so``): splitmix64 + Box-Muller normals
(generators.cpp:13-48), gen_planted_tt -> reconstruct (generators.cpp:62-79, tt.cpp:52-73),
the 4096-blocked norm (kernels.cpp:84-102). The buffers are bitwise those the reference's
generators give (tests/test_inputs_cpu.py), so the committed full-size golden fixtures
(tests/golden/full_cfg*.npz, produced by the reference on its own generators) apply to the
bench's inputs as well.

  cfg1  20^4 planted TT (1,5,5,5,1), cores Rng(1), + 1e-8 relative noise Rng(2)
  cfg2  32^5 A = 1/(i1+..+i5-4), 1-based (deterministic)
  cfg3  24^6 planted TT ranks 20, cores Rng(3), + 1e-4 relative noise Rng(4)
  cfg4  256^3 MRI-like volume (64 blobs Rng(4), 1% noise Rng(40)) as 4^12, Bernoulli(0.5)
        mask Rng(41)
  cfg5  1024^3 planted TT (1,128,128,1), cores Rng(5), + 1e-6 relative noise Rng(6)
Tensors are flat float64 buffers in the reference's storage order (first index fastest).
"""
from __future__ import annotations

import ctypes as C
import math
from pathlib import Path

import numpy as np

CONFIGS = {
    1: dict(dims=[20] * 4, ranks=[1, 5, 5, 5, 1], rho=1e-8, seed=1, mode="rank"),
    2: dict(dims=[32] * 5, eps=1e-8, mode="tol"),
    3: dict(dims=[24] * 6, ranks=[1, 20, 20, 20, 20, 20, 1], rho=1e-4, seed=3, mode="rank"),
    4: dict(dims=[4] * 12, eps=1e-3, mode="tol", iters=20, blob_seed=4, noise_seed=40, mask_seed=41),
    5: dict(dims=[1024] * 3, ranks=[1, 128, 128, 1], rho=1e-6, seed=5, mode="rank"),
}

_LIB = Path(__file__).resolve().parent / "lib" / "libttutv_inputs.so"
_lib = None
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int64)


def lib():
    global _lib
    if _lib is None:
        if not _LIB.exists():
            from .build import build_inputs
            build_inputs()
        h = C.CDLL(str(_LIB))
        h.tig_u64.argtypes = [C.c_uint64, C.c_int64, C.POINTER(C.c_uint64)]
        h.tig_gaussian.argtypes = [C.c_uint64, C.c_int64, _dp]
        h.tig_uniform.argtypes = [C.c_uint64, C.c_int64, _dp]
        h.tig_sum_squares.argtypes = [_dp, C.c_int64]
        h.tig_sum_squares.restype = C.c_double
        h.tig_planted_cores.argtypes = [_ip, C.c_int, _ip, C.c_uint64, _dp]
        h.tig_contract.argtypes = [_dp, _ip, C.c_int, _ip, _dp, _dp]
        h.tig_add_scaled.argtypes = [_dp, _dp, C.c_double, C.c_int64]
        h.tig_scale.argtypes = [_dp, C.c_double, C.c_int64]
        h.tig_blobs.argtypes = [C.c_int64, C.c_int, C.c_uint64, _dp]
        h.tig_bernoulli_mask.argtypes = [C.c_uint64, C.c_double, C.c_int64, _dp]
        h.tig_bernoulli_mask.restype = C.c_int64
        _lib = h
    return _lib


def _d(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _i64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, np.int64))


def gaussian(n: int, seed: int) -> np.ndarray:
    """gen_gaussian(shape, seed) flattened (generators.cpp:81-86)."""
    out = np.empty(int(n), np.float64)
    lib().tig_gaussian(int(seed), int(n), _d(out))
    return out


def u64(n: int, seed: int) -> np.ndarray:
    out = np.empty(int(n), np.uint64)
    lib().tig_u64(int(seed), int(n), out.ctypes.data_as(C.POINTER(C.c_uint64)))
    return out


def frobenius_norm(a: np.ndarray) -> float:
    """frobenius_norm (tensor_ops.cpp:95-97): sqrt of the 4096-blocked sum of squares."""
    a = np.ascontiguousarray(a, np.float64).reshape(-1)
    return math.sqrt(lib().tig_sum_squares(_d(a), a.size))


def planted_cores(dims, ranks, seed) -> list:
    """gen_planted_tt(shape, ranks, seed) cores, each (r_{k-1}, I_k, r_k) Fortran-ordered."""
    dims, ranks = _i64(dims), _i64(ranks)
    sizes = [int(ranks[k] * dims[k] * ranks[k + 1]) for k in range(dims.size)]
    flat = np.empty(sum(sizes), np.float64)
    lib().tig_planted_cores(dims.ctypes.data_as(_ip), dims.size, ranks.ctypes.data_as(_ip), int(seed), _d(flat))
    out, off = [], 0
    for k, s in enumerate(sizes):
        out.append(flat[off:off + s].reshape((int(ranks[k]), int(dims[k]), int(ranks[k + 1])), order="F"))
        off += s
    return out


def planted(dims, ranks, seed, rho) -> np.ndarray:
    """A = A0 + (rho |A0| / |E|) E with A0 = reconstruct(gen_planted_tt(seed)) and
    E = gen_gaussian(seed + 1) (tests/fixtures.planted_plus_noise)."""
    dims, ranks = _i64(dims), _i64(ranks)
    n = int(np.prod(dims))
    sizes = [int(ranks[k] * dims[k] * ranks[k + 1]) for k in range(dims.size)]
    cores = np.empty(sum(sizes), np.float64)
    lib().tig_planted_cores(dims.ctypes.data_as(_ip), dims.size, ranks.ctypes.data_as(_ip), int(seed), _d(cores))
    a = np.empty(n, np.float64)
    work = np.empty(n, np.float64)
    lib().tig_contract(_d(cores), dims.ctypes.data_as(_ip), dims.size, ranks.ctypes.data_as(_ip), _d(a), _d(work))
    if rho > 0.0:
        e = work  # the contraction's scratch holds the noise
        lib().tig_gaussian(int(seed) + 1, n, _d(e))
        s = rho * frobenius_norm(a) / frobenius_norm(e)
        lib().tig_add_scaled(_d(a), _d(e), s, n)
    del work
    return a


def hilbert_shifted(dims) -> np.ndarray:
    """A(i1..id) = 1/(i1+...+id-(d-1)) with 1-based indices (value 1 at the origin)."""
    d = len(dims)
    s = np.zeros(1, np.int64)
    for n in reversed(dims):  # first index fastest
        s = (s[:, None] + np.arange(1, n + 1, dtype=np.int64)[None, :]).reshape(-1)
    return 1.0 / (s - (d - 1)).astype(np.float64)


def mri_like(n=256, nblobs=64, blob_seed=4, noise_seed=40, noise=0.01) -> np.ndarray:
    """Config 4 volume: 64 Gaussian blobs (hostgen tig_blobs) plus
    gen_gaussian(n^3, noise_seed) scaled to `noise` |V|; the flat buffer is the 4^12 tensor."""
    v = np.empty(n ** 3, np.float64)
    lib().tig_blobs(n, nblobs, int(blob_seed), _d(v))
    e = gaussian(n ** 3, noise_seed)
    s = noise * frobenius_norm(v) / frobenius_norm(e)
    lib().tig_add_scaled(_d(v), _d(e), s, v.size)
    return v


def bernoulli_mask(count: int, seed=41, p=0.5) -> np.ndarray:
    """1.0 where Rng(seed).uniform() < p, per entry in storage order."""
    out = np.empty(int(count), np.float64)
    lib().tig_bernoulli_mask(int(seed), float(p), int(count), _d(out))
    return out


def build_host(cfg: int) -> np.ndarray:
    c = CONFIGS[cfg]
    if cfg == 4:
        return mri_like(blob_seed=c["blob_seed"], noise_seed=c["noise_seed"])
    if cfg == 2:
        return hilbert_shifted(c["dims"])
    return planted(c["dims"], c["ranks"], c["seed"], c["rho"])


def build(cfg: int, device):
    """The config's tensor as a flat float64 torch tensor on `device` (built on the host)."""
    import torch
    a = build_host(cfg)
    t = torch.from_numpy(a)
    return t.to(device) if str(device) != "cpu" else t
