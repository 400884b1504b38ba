// Tensor algebra of tensor_ops.hpp / tt.hpp beyond the sweeps, on the device:
// mode_product (tensor_ops.cpp:49-80), kron (:82-93), psnr (:113-126), reverse_indices
// (:128-143), reverse_tt (tt.cpp:108-123). mode_product and kron compute every output with the
// reference's own operation order (sequential sum over the contracted index, products and sums
// rounded separately, no FMA), so their results are bitwise the reference's.
#include "sweep.hpp"

namespace ttg {
namespace {

// out(i, jn, r) = sum_j m(jn, j) x(i, j, r); x is left x mid x right, m is new_mid x mid.
__global__ void k_mode_product(const double* __restrict__ x, int64_t left, int64_t mid, int64_t right,
                               const double* __restrict__ m, int64_t new_mid, double* __restrict__ out) {
    const int64_t total = left * new_mid * right;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % left, jn = (e / left) % new_mid, r = e / (left * new_mid);
        const double* src = x + r * left * mid + i;
        double sum = 0.0;
        for (int64_t j = 0; j < mid; ++j) sum = __dadd_rn(sum, __dmul_rn(m[jn + j * new_mid], src[j * left]));
        out[e] = sum;
    }
}

// out(ia * br + ib, ja * bc + jb) = a(ia, ja) * b(ib, jb), column-major
__global__ void k_kron(const double* __restrict__ a, int64_t ar, int64_t ac, const double* __restrict__ b,
                       int64_t br, int64_t bc, double* __restrict__ out) {
    const int64_t rows = ar * br, total = rows * ac * bc;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % rows, j = e / rows;
        const int64_t ia = i / br, ib = i % br, ja = j / bc, jb = j % bc;
        out[e] = __dmul_rn(a[ia + ja * ar], b[ib + jb * br]);
    }
}

// per-block maxima (psnr's max over the truth)
__global__ void __launch_bounds__(256) k_block_max(const double* __restrict__ x, int64_t n, double* part) {
    double mx = -INFINITY;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        mx = fmax(mx, x[i]);
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    __shared__ double sm[8];
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) mx = fmax(mx, sm[w]);
        part[blockIdx.x] = mx;
    }
}

struct DimsR {
    int d;
    int64_t n[32];
};

// B(i_d, ..., i_1) = A(i_1, ..., i_d)
__global__ void k_reverse(const double* __restrict__ A, DimsR dims, int64_t total, double* __restrict__ B) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        int64_t rest = e, src = 0;
        for (int k = 0; k < dims.d; ++k) {  // B's mode k is A's mode d-1-k
            const int ka = dims.d - 1 - k;
            int64_t stride = 1;
            for (int q = 0; q < ka; ++q) stride *= dims.n[q];
            const int64_t nk = dims.n[ka];
            src += (rest % nk) * stride;
            rest /= nk;
        }
        B[e] = A[src];
    }
}

// out(b, i, a) = in(a, i, b) for a core (rl, mid, rr)
__global__ void k_flip_core(const double* __restrict__ in, int64_t rl, int64_t mid, int64_t rr, double* __restrict__ out) {
    const int64_t total = rl * mid * rr;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = e % rl, i = (e / rl) % mid, b = e / (rl * mid);
        out[b + i * rr + a * rr * mid] = in[e];
    }
}

int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), (int64_t)sm_count() * 16)); }

}  // namespace

void mode_product_dev(const double* x, int64_t left, int64_t mid, int64_t right, const double* m, int64_t new_mid,
                      double* out) {
    const int64_t total = left * new_mid * right;
    if (total == 0) return;
    TTG_LAUNCH(k_mode_product, grid_for(total), 256, 0, stream(), x, left, mid, right, m, new_mid, out);
}

void kron_dev(const double* a, int64_t ar, int64_t ac, const double* b, int64_t br, int64_t bc, double* out) {
    const int64_t total = ar * br * ac * bc;
    if (total == 0) return;
    TTG_LAUNCH(k_kron, grid_for(total), 256, 0, stream(), a, ar, ac, b, br, bc, out);
}

double max_value_dev(const double* x, int64_t n) {
    const int g = grid_for(n);
    DevBuf<double> part((size_t)g);
    TTG_LAUNCH(k_block_max, g, 256, 0, stream(), x, n, part.get());
    const std::vector<double> h = part.to_host((size_t)g);
    double mx = -INFINITY;
    for (double v : h) mx = std::max(mx, v);
    return mx;
}

void reverse_indices_dev(const double* a, const std::vector<int64_t>& dims, double* out) {
    if (dims.size() > 32) argument_error("reverse_indices supports order <= 32");
    DimsR dd{(int)dims.size(), {}};
    int64_t total = 1;
    for (size_t k = 0; k < dims.size(); ++k) {
        dd.n[k] = dims[k];
        total *= dims[k];
    }
    if (total == 0) return;
    TTG_LAUNCH(k_reverse, grid_for(total), 256, 0, stream(), a, dd, total, out);
}

void flip_core_dev(const double* in, int64_t rl, int64_t mid, int64_t rr, double* out) {
    const int64_t total = rl * mid * rr;
    if (total == 0) return;
    TTG_LAUNCH(k_flip_core, grid_for(total), 256, 0, stream(), in, rl, mid, rr, out);
}

}  // namespace ttg
