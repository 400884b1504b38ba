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

namespace {
constexpr int64_t kChunk = 4096;

// One pass: y <- mask ? observed : y, with the completion trace sums of the reconstruction
// X (the incoming y) per 4096-entry chunk (combined in chunk order on the host side).
__global__ void __launch_bounds__(256) k_completion_reset(double* y, const double* __restrict__ obs,
                                                          const double* __restrict__ mask,
                                                          const double* __restrict__ truth, int64_t n,
                                                          double* part) {
    __shared__ double sd[8];
    const int64_t nchunk = cdiv(n, kChunk);
    for (int64_t b = blockIdx.x; b < nchunk; b += gridDim.x) {
        const int64_t lo = b * kChunk, hi = min(n, lo + kChunk);
        double so = 0.0, sm = 0.0, sf = 0.0, st = 0.0, mx = -INFINITY;
        for (int64_t i = lo + threadIdx.x; i < hi; i += 256) {
            const double x = y[i];
            const bool on = mask[i] != 0.0;
            if (on) {
                const double d = x - obs[i];
                so = fma(d, d, so);
                sm = fma(obs[i], obs[i], sm);
                y[i] = obs[i];
            }
            if (truth) {
                const double d = x - truth[i];
                sf = fma(d, d, sf);
                st = fma(truth[i], truth[i], st);
                mx = fmax(mx, truth[i]);
            }
        }
        so = block_sum(so, sd);
        sm = block_sum(sm, sd);
        sf = block_sum(sf, sd);
        st = block_sum(st, sd);
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        __shared__ double smx[8];
        __syncthreads();
        if ((threadIdx.x & 31) == 0) smx[threadIdx.x >> 5] = mx;
        __syncthreads();
        if (threadIdx.x == 0) {
            double m = smx[0];
            for (int w = 1; w < 8; ++w) m = fmax(m, smx[w]);
            part[5 * b + 0] = so;
            part[5 * b + 1] = sm;
            part[5 * b + 2] = sf;
            part[5 * b + 3] = st;
            part[5 * b + 4] = m;
        }
    }
}
}  // namespace

void completion_reset(double* y, const double* observed, const double* mask, const double* truth, int64_t n,
                      double stats[5]) {
    const int64_t nchunk = cdiv(n, kChunk);
    DevBuf<double> part((size_t)(5 * nchunk));
    const int grid = (int)std::min<int64_t>(nchunk, (int64_t)sm_count() * 8);
    TTG_LAUNCH(k_completion_reset, grid, 256, 0, stream(), y, observed, mask, truth, n, part.get());
    std::vector<double> h = part.to_host((size_t)(5 * nchunk));
    for (int k = 0; k < 4; ++k) stats[k] = 0.0;
    stats[4] = truth ? -INFINITY : 0.0;
    for (int64_t b = 0; b < nchunk; ++b) {
        for (int k = 0; k < 4; ++k) stats[k] += h[(size_t)(5 * b + k)];
        if (truth) stats[4] = std::max(stats[4], h[(size_t)(5 * b + 4)]);
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
