"""FP64 GEMM throughput of the engine's DMMA kernel (ttg_gemm_device) against cuBLAS DGEMM
(torch.matmul float64, measurement only) on the shapes the TT-UTV path uses. Prints JSON."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2501_07904_b200._native import lib, check  # noqa: E402


def time_it(fn, reps=5):
    s = torch.cuda.ExternalStream(lib().ttg_stream())
    fn()
    check(lib().ttg_synchronize())
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return best


def cublas(m, n, k, ta, tb):
    a = torch.randn(k if ta else m, m if ta else k, dtype=torch.float64, device="cuda")
    b = torch.randn(n if tb else k, k if tb else n, dtype=torch.float64, device="cuda")
    A = a.T if ta else a
    B = b.T if tb else b
    torch.matmul(A, B)
    torch.cuda.synchronize()
    best = None
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(A, B)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return best


rows = []
for name, (m, n, k, ta, tb) in {
    "square 8192^3": (8192, 8192, 8192, 0, 0),
    "config-5 cut-2 Gram c c^T (1024 x 1024, K 131072)": (1024, 1024, 131072, 0, 1),
    "config-4 reconstruct step (4096 x 4096, K 4079)": (4096, 4096, 4079, 0, 0),
    "Gram W^T W (1024 x 1024, K 131072, col W)": (1024, 1024, 131072, 1, 0),
}.items():
    A = torch.randn((k if ta else m) * (m if ta else k), dtype=torch.float64, device="cuda")
    B = torch.randn((n if tb else k) * (k if tb else n), dtype=torch.float64, device="cuda")
    Cm = torch.empty(m * n, dtype=torch.float64, device="cuda")
    lda, ldb = (k if ta else m), (n if tb else k)
    ms = time_it(lambda: check(lib().ttg_gemm_device(ta, tb, m, n, k, 1.0, A.data_ptr(), lda, B.data_ptr(), ldb,
                                                     0.0, Cm.data_ptr(), m)))
    cb = cublas(m, n, k, ta, tb)
    f = 2.0 * m * n * k
    rows.append({"shape": name, "m": m, "n": n, "k": k, "ta": ta, "tb": tb, "engine_ms": ms,
                 "engine_tflops": f / ms / 1e9, "cublas_ms": cb, "cublas_tflops": f / cb / 1e9,
                 "engine_vs_cublas": cb / ms})
    del A, B, Cm
    torch.cuda.empty_cache()
print(json.dumps({"gemm": rows}, indent=1))
