"""Seeded synthetic inputs for bench.py (harness code, not the product path).

The paper's datasets are not available; BASELINE.json's configs are built from their
recipes directly in HBM with torch as plumbing:
  cfg1  20^4 planted TT (1,5,5,5,1) + 1e-8 relative Gaussian noise
  cfg2  32^5 A = 1/(i1+..+i5-4), 1-based (deterministic)
  cfg3  24^6 planted TT ranks 20 + 1e-4 relative noise
  cfg5  1024^3 planted TT (1,128,128,1) + 1e-6 relative noise
Tensors are flat float64 buffers in the reference's storage order (first index fastest).
"""
from __future__ import annotations

import math

import torch

CONFIGS = {
    1: dict(dims=[20] * 4, ranks=[1, 5, 5, 5, 1], rho=1e-8, seed=1, mode="rank"),
    2: dict(dims=[32] * 5, eps=1e-8, mode="tol"),
    3: dict(dims=[24] * 6, ranks=[1, 20, 20, 20, 20, 20, 1], rho=1e-4, seed=3, mode="rank"),
    4: dict(dims=[4] * 12, eps=1e-3, mode="tol", iters=20),
    5: dict(dims=[1024] * 3, ranks=[1, 128, 128, 1], rho=1e-6, seed=5, mode="rank"),
}


def hilbert_shifted(dims, device) -> torch.Tensor:
    """A(i1..id) = 1/(i1+...+id-(d-1)) with 1-based indices (value 1 at the origin)."""
    n = math.prod(dims)
    idx = torch.arange(n, device=device, dtype=torch.int64)
    s = torch.zeros(n, device=device, dtype=torch.float64)
    for d in dims:
        s += (idx % d).to(torch.float64)
        idx = idx // d
    # 0-based digit sum + d = 1-based sum; subtract d-1
    return 1.0 / (s + 1.0)


def planted(dims, ranks, seed, rho, device) -> torch.Tensor:
    """Dense contraction of random N(0,1) TT cores plus rho-relative Gaussian noise.

    Core k, shape (r_{k-1}, I_k, r_k) first-index-fastest, is generated as the C-order
    matrix G^T of shape (I_k r_k, r_{k-1}); the chain B^T <- G^T B^T reproduces
    reconstruct() (tt.cpp:52-73) in transposed storage."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    bt = None
    for k, n in enumerate(dims):
        gt = torch.randn(n * ranks[k + 1], ranks[k], generator=g, device=device, dtype=torch.float64)
        if bt is None:
            # core 1 is (1, I1, r1): its memory is col-major I1 x r1 = C-order (r1, I1)
            bt = gt.reshape(ranks[1], n)
        else:
            bt = (gt @ bt).reshape(ranks[k + 1], -1)
    a = bt.reshape(-1).contiguous()
    if rho > 0:
        e = torch.randn(a.numel(), generator=g, device=device, dtype=torch.float64)
        a.add_(e, alpha=float(rho * a.norm() / e.norm()))
        del e
    return a


def mri_like(device, seed=4, nblobs=64, n=256, noise=0.01):
    """Config 4: sum of `nblobs` axis-aligned anisotropic Gaussian
    blobs on an n^3 grid (centres U[0,n), widths sigma U[4,32], amplitudes U[0.2,1]) plus
    Gaussian noise at `noise` relative Frobenius level. Returns the flat volume (first
    index fastest: x + n*y + n^2*z), i.e. the 4^12 tensor by pure reinterpretation."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    u = lambda *s: torch.rand(*s, generator=g, device=device, dtype=torch.float64)
    c = u(nblobs, 3) * n
    w = 4.0 + 28.0 * u(nblobs, 3)
    amp = 0.2 + 0.8 * u(nblobs)
    ax = torch.arange(n, device=device, dtype=torch.float64)
    f = [torch.exp(-0.5 * ((ax[None, :] - c[:, a, None]) / w[:, a, None]) ** 2) for a in range(3)]
    v = torch.einsum("b,bx,by,bz->zyx", amp, f[0], f[1], f[2]).reshape(-1).contiguous()
    e = torch.randn(v.numel(), generator=g, device=device, dtype=torch.float64)
    v.add_(e, alpha=float(noise * v.norm() / e.norm()))
    return v


def bernoulli_mask(count: int, device, seed=41, p=0.5) -> torch.Tensor:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return (torch.rand(count, generator=g, device=device, dtype=torch.float64) < p).to(torch.float64)


def build(cfg: int, device) -> torch.Tensor:
    if cfg == 4:
        return mri_like(device)
    c = CONFIGS[cfg]
    if cfg == 2:
        return hilbert_shifted(c["dims"], device)
    return planted(c["dims"], c["ranks"], c["seed"], c["rho"], device)
