"""The engine's FP64 tensor-core GEMM (ttg_gemm_device: DMMA m8n8k4 tiles, the 128 x 128
cp.async-pipelined kernel for aligned operands, split-K for long reductions) against an fp64
torch reference of the same product (cuBLAS, test-only)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(ta, tb, m, n, k, lda_pad=0, alpha=1.0, beta=0.0):
    import torch
    from paper_2501_07904_b200._native import lib, check
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n * 3 + k)
    ar, ac = (k, m) if ta else (m, k)
    br, bc = (n, k) if tb else (k, n)
    lda, ldb = ar + lda_pad, br + lda_pad
    A = torch.randn(ac, lda, generator=g, device="cuda", dtype=torch.float64)  # column-major ar x ac, ld lda
    B = torch.randn(bc, ldb, generator=g, device="cuda", dtype=torch.float64)
    Cm = torch.randn(n, m, generator=g, device="cuda", dtype=torch.float64)
    Aop = A[:, :ar].T if not ta else A[:, :ar]        # op(A) as m x k
    Bop = B[:, :br].T if not tb else B[:, :br]        # op(B) as k x n
    want = alpha * (Aop @ Bop) + beta * Cm.T
    torch.cuda.synchronize()
    check(lib().ttg_gemm_device(int(ta), int(tb), m, n, k, alpha, A.data_ptr(), lda, B.data_ptr(), ldb, beta,
                                Cm.data_ptr(), m))
    check(lib().ttg_synchronize())
    got = Cm.T
    err = (got - want).abs().max().item()
    scale = (Aop.abs() @ Bop.abs()).max().item() * abs(alpha) + abs(beta) * 4
    return err, scale


@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("m,n,k", [(128, 128, 64), (300, 200, 96), (257, 130, 33), (1024, 96, 5000),
                                   (96, 96, 20000), (512, 384, 512)])
def test_gemm_matches_fp64_reference(ta, tb, m, n, k):
    err, scale = _run(ta, tb, m, n, k)
    assert err <= 1e-14 * scale * max(1.0, k ** 0.5), (err, scale)


@pytest.mark.parametrize("pad", [0, 1, 2])
def test_gemm_alpha_beta_and_ld(pad):
    err, scale = _run(False, True, 260, 190, 300, lda_pad=pad, alpha=-0.5, beta=2.0)
    assert err <= 1e-13 * scale, (err, scale)
