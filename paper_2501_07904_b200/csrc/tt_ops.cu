// Train contraction on device: reconstruct (tt.cpp:52-73) as a left-to-right chain of
// DMMA GEMMs, and the residual |A - reconstruct|_F^2 used by verify_bound / rse
// (tt_decomp.cpp:445-462, tensor_ops.cpp:101-111).
#include "sweep.hpp"

namespace ttg {

void reconstruct(const std::vector<const double*>& cores, const std::vector<int64_t>& dims,
                 const std::vector<int64_t>& ranks, double* out) {
    const size_t d = dims.size();
    if (d == 1) {
        TTG_CUDA(cudaMemcpyAsync(out, cores[0], sizeof(double) * dims[0], cudaMemcpyDeviceToDevice, stream()));
        return;
    }
    // B holds (I_1...I_{k}) x r_k, column-major.
    DevBuf<double> cur, nxt;
    const double* b = cores[0];
    int64_t left = dims[0];
    for (size_t k = 1; k < d; ++k) {
        const int64_t rk0 = ranks[k], rk1 = ranks[k + 1], ik = dims[k];
        double* dst;
        if (k == d - 1) {
            dst = out;
        } else {
            nxt.alloc((size_t)(left * ik * rk1));
            dst = nxt.get();
        }
        // (left x r_{k-1}) * (r_{k-1} x I_k r_k) -> left x (I_k r_k) == (left I_k) x r_k
        gemm(false, false, left, ik * rk1, rk0, b, left, cores[k], rk0, dst, left);
        left *= ik;
        if (k != d - 1) {
            cur = std::move(nxt);
            b = cur.get();
        }
    }
}

double residual_squared(const TTResult& r, const double* a) {
    int64_t total = 1;
    for (int64_t v : r.dims) total *= v;
    std::vector<const double*> cores;
    std::vector<int64_t> ranks{1};
    for (size_t k = 0; k < r.cores.size(); ++k) {
        cores.push_back(r.cores[k].get());
        ranks.push_back(r.core_dims[k][2]);
    }
    DevBuf<double> hat((size_t)total);
    reconstruct(cores, r.dims, ranks, hat.get());
    return diff_squares(hat.get(), a, total);
}

}  // namespace ttg
