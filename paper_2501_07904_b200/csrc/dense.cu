// Dense device helpers: FP64 tensor-core GEMM (mma.sync m8n8k4 f64 -> SASS DMMA; sm_100a
// has no tcgen05 kind for f64), tiled transpose and deterministic reductions.
#include <cmath>
#include <cstdlib>

#include "engine.hpp"

namespace ttg {
namespace {

// ---------------------------------------------------------------------------
// GEMM: C = alpha op(A) op(B) + beta C, column-major. CTA tile 64x64, K step 16,
// 4 warps each owning a 32x32 sub-tile = 4x4 DMMA 8x8x4 fragments. Operand tiles are
// staged in shared memory with a two-stage register prefetch.
// ---------------------------------------------------------------------------
constexpr int BM = 64, BN = 64, BK = 16;


// Split-K: blockIdx.y selects the K chunk [y kc, (y+1) kc); chunk y writes its partial
// product to C + y * cstride (beta must be 0 then). kc = k, cstride = 0 for a plain GEMM.
template <bool TA, bool TB>
__global__ void __launch_bounds__(128) k_gemm(int64_t m, int64_t n, int64_t k, const double* __restrict__ A,
                                              int64_t lda, const double* __restrict__ B, int64_t ldb, double* C,
                                              int64_t ldc, double alpha, double beta, int64_t kc, int64_t cstride) {
    {
        const int64_t kb = (int64_t)blockIdx.y * kc;
        k = min(kc, k - kb);
        A += TA ? kb : kb * lda;
        B += TB ? kb * ldb : kb;
        C += (int64_t)blockIdx.y * cstride;
    }
    __shared__ double As[BK][BM + 1];
    __shared__ double Bs[BK][BN + 1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t tm = cdiv(m, BM);
    const int64_t m0 = ((int64_t)blockIdx.x % tm) * BM, n0 = ((int64_t)blockIdx.x / tm) * BN;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    // Each thread loads 8 elements of each tile per stage (64*16 / 128).
    double ra[8], rb[8];
    auto load = [&](int64_t k0) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int idx = tid + e * 128;
            // A tile element (row r in [0,64), kk in [0,16))
            int r, kk;
            if (!TA) { r = idx & 63; kk = idx >> 6; } else { kk = idx & 15; r = idx >> 4; }
            const int64_t gi = m0 + r, gk = k0 + kk;
            ra[e] = (gi < m && gk < k) ? (TA ? A[gk + gi * lda] : A[gi + gk * lda]) : 0.0;
            int c, kb;
            if (!TB) { kb = idx & 15; c = idx >> 4; } else { c = idx & 63; kb = idx >> 6; }
            const int64_t gj = n0 + c, gk2 = k0 + kb;
            rb[e] = (gj < n && gk2 < k) ? (TB ? B[gj + gk2 * ldb] : B[gk2 + gj * ldb]) : 0.0;
        }
    };
    auto store = [&]() {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int idx = tid + e * 128;
            int r, kk;
            if (!TA) { r = idx & 63; kk = idx >> 6; } else { kk = idx & 15; r = idx >> 4; }
            As[kk][r] = ra[e];
            int c, kb;
            if (!TB) { kb = idx & 15; c = idx >> 4; } else { c = idx & 63; kb = idx >> 6; }
            Bs[kb][c] = rb[e];
        }
    };
    load(0);
    for (int64_t k0 = 0; k0 < k; k0 += BK) {
        __syncthreads();
        store();
        __syncthreads();
        if (k0 + BK < k) load(k0 + BK);
#pragma unroll
        for (int ks = 0; ks < BK; ks += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = As[ks + (lane & 3)][wm + i * 8 + (lane >> 2)];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = Bs[ks + (lane & 3)][wn + j * 8 + (lane >> 2)];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t gi = m0 + wm + i * 8 + (lane >> 2);
                const int64_t gj = n0 + wn + j * 8 + 2 * (lane & 3) + h;
                if (gi < m && gj < n) {
                    double* cp = C + gi + gj * ldc;
                    *cp = beta == 0.0 ? alpha * acc[i][j][h] : fma(alpha, acc[i][j][h], beta * *cp);
                }
            }
}

// ---------------------------------------------------------------------------
// Large GEMM: CTA tile 128 x 128, K step 16, 8 warps (2 x 4) each owning a 64 x 32 sub-tile
// = 8 x 4 DMMA 8x8x4 fragments (64 accumulators per thread). Operand tiles move global ->
// shared with 16-byte cp.async (LDGSTS) through a 4-stage ring, so the next three K steps are
// in flight while the DMMAs of the current one run. Shared layouts are chosen per operand so
// that the 16-byte copies land contiguously and the fragment loads are conflict-free:
//   A (!TA, m contiguous): As[k][m], row stride 132;  A (TA, k contiguous): As[m][k], stride 20
//   B (TB,  n contiguous): Bs[k][n], row stride 132;  B (!TB, k contiguous): Bs[n][k], stride 20
// (strides = 4 mod 16 doubles: the 16 lanes of a half-warp hit 16 distinct bank pairs).
// Requires 16-byte aligned A, B and even lda, ldb (the dispatcher checks); edges zero-fill.
// Split-K over blockIdx.y like k_gemm (kc, cstride).
// ---------------------------------------------------------------------------
constexpr int G2M = 128, G2N = 128, G2K = 16, G2STAGES = 4;
constexpr int G2WIDE = 132, G2NARROW = 20;
constexpr int G2TILE = G2M * G2NARROW > G2K * G2WIDE ? G2M * G2NARROW : G2K * G2WIDE;  // doubles per operand tile

__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, int bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
// elements (0..2) of a 16-byte chunk that lie inside the matrix, `left` = extent - index
__device__ __forceinline__ int g2cnt(int64_t left) { return left <= 0 ? 0 : left >= 2 ? 2 : 1; }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <bool TA, bool TB>
__global__ void __launch_bounds__(256, 1) k_gemm128(int64_t m, int64_t n, int64_t k, const double* __restrict__ A,
                                                    int64_t lda, const double* __restrict__ B, int64_t ldb, double* C,
                                                    int64_t ldc, double alpha, double beta, int64_t kc,
                                                    int64_t cstride, int sym) {
    {
        const int64_t kb = (int64_t)blockIdx.y * kc;
        k = min(kc, k - kb);
        A += TA ? kb : kb * lda;
        B += TB ? kb * ldb : kb;
        C += (int64_t)blockIdx.y * cstride;
    }
    extern __shared__ double g2s[];  // G2STAGES x (A tile, B tile)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t tm = cdiv(m, G2M);
    int64_t m0 = ((int64_t)blockIdx.x % tm) * G2M, n0 = ((int64_t)blockIdx.x / tm) * G2N;
    if (sym) {  // symmetric product: only the tiles on and above the diagonal (tile row <= col)
        const int64_t idx = blockIdx.x;
        int64_t tn = (int64_t)((sqrt(8.0 * (double)idx + 1.0) - 1.0) * 0.5);
        while ((tn + 1) * (tn + 2) / 2 <= idx) ++tn;
        while (tn * (tn + 1) / 2 > idx) --tn;
        m0 = (idx - tn * (tn + 1) / 2) * G2M;
        n0 = tn * G2N;
    }
    const int wm = (warp & 1) * 64, wn = (warp >> 1) * 32;

    auto load_stage = [&](int stage, int64_t k0) {
        double* As = g2s + (size_t)stage * 2 * G2TILE;
        double* Bs = As + G2TILE;
#pragma unroll
        for (int e = 0; e < 4; ++e) {  // 1024 16-byte chunks per operand tile
            const int c = tid + e * 256;
            if (!TA) {
                const int kk = c >> 6, mm = (c & 63) * 2;
                const int64_t gi = m0 + mm, gk = k0 + kk;
                const int bytes = gk < k ? g2cnt(m - gi) * 8 : 0;
                cp_async16(As + kk * G2WIDE + mm, bytes ? A + gi + gk * lda : A, bytes);
            } else {
                const int mm = c >> 3, kk = (c & 7) * 2;
                const int64_t gi = m0 + mm, gk = k0 + kk;
                const int bytes = gi < m ? g2cnt(k - gk) * 8 : 0;
                cp_async16(As + mm * G2NARROW + kk, bytes ? A + gk + gi * lda : A, bytes);
            }
            if (TB) {
                const int kk = c >> 6, nn = (c & 63) * 2;
                const int64_t gj = n0 + nn, gk = k0 + kk;
                const int bytes = gk < k ? g2cnt(n - gj) * 8 : 0;
                cp_async16(Bs + kk * G2WIDE + nn, bytes ? B + gj + gk * ldb : B, bytes);
            } else {
                const int nn = c >> 3, kk = (c & 7) * 2;
                const int64_t gj = n0 + nn, gk = k0 + kk;
                const int bytes = gj < n ? g2cnt(k - gk) * 8 : 0;
                cp_async16(Bs + nn * G2NARROW + kk, bytes ? B + gk + gj * ldb : B, bytes);
            }
        }
    };

    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const int64_t nk = cdiv(k, G2K);
#pragma unroll
    for (int s = 0; s < G2STAGES - 1; ++s) {
        if (s < nk) load_stage(s, (int64_t)s * G2K);
        cp_async_commit();
    }
    const int fr = lane >> 2, fk = lane & 3;
    for (int64_t kt = 0; kt < nk; ++kt) {
        cp_async_wait<G2STAGES - 2>();
        __syncthreads();
        {  // refill the stage consumed G2STAGES - 1 steps ago
            const int64_t nxt = kt + G2STAGES - 1;
            if (nxt < nk) load_stage((int)(nxt % G2STAGES), nxt * G2K);
            cp_async_commit();
        }
        const double* As = g2s + (size_t)(kt % G2STAGES) * 2 * G2TILE;
        const double* Bs = As + G2TILE;
#pragma unroll
        for (int ks = 0; ks < G2K; ks += 4) {
            double af[8], bf[4];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int r = wm + i * 8 + fr;
                af[i] = TA ? As[r * G2NARROW + ks + fk] : As[(ks + fk) * G2WIDE + r];
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int cidx = wn + j * 8 + fr;
                bf[j] = TB ? Bs[(ks + fk) * G2WIDE + cidx] : Bs[cidx * G2NARROW + ks + fk];
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
        }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t gi = m0 + wm + i * 8 + fr;
                const int64_t gj = n0 + wn + j * 8 + 2 * fk + h;
                if (gi < m && gj < n) {
                    double* cp = C + gi + gj * ldc;
                    *cp = beta == 0.0 ? alpha * acc[i][j][h] : fma(alpha, acc[i][j][h], beta * *cp);
                }
            }
}

__global__ void k_transpose(const double* __restrict__ A, int64_t m, int64_t n, int64_t lda, double* B,
                            int64_t ldb) {
    __shared__ double tile[32][33];
    const int64_t i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t i = i0 + threadIdx.x, j = j0 + r;
        if (i < m && j < n) tile[r][threadIdx.x] = A[i + j * lda];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t j = j0 + threadIdx.x, i = i0 + r;
        if (i < m && j < n) B[j + i * ldb] = tile[threadIdx.x][r];
    }
}

// Blocked sum of squares: partial per 4096-element block (the reference's kReduceBlock,
// kernels.cpp:16), one block per CTA iteration.
constexpr int64_t kBlock = 4096;

template <bool DIFF>
__global__ void __launch_bounds__(256) k_sq_part(const double* __restrict__ x, const double* __restrict__ y,
                                                 int64_t n, double* part) {
    __shared__ double sd[8];
    const int64_t nb = cdiv(n, kBlock);
    for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
        const int64_t lo = b * kBlock, hi = min(n, lo + kBlock);
        double s = 0.0;
        for (int64_t i = lo + threadIdx.x; i < hi; i += 256) {
            const double v = DIFF ? x[i] - y[i] : x[i];
            s = fma(v, v, s);
        }
        s = block_sum(s, sd);
        if (threadIdx.x == 0) part[b] = s;
    }
}

// Combine partials in block order with a fixed tree: 1 CTA.
__global__ void __launch_bounds__(1024) k_sum_parts(const double* part, int64_t nb, double* out) {
    __shared__ double sd[32];
    double s = 0.0;
    const int64_t chunk = cdiv(nb, 1024);
    const int64_t lo = threadIdx.x * chunk, hi = min(nb, lo + chunk);
    for (int64_t i = lo; i < hi; ++i) s += part[i];
    s = block_sum(s, sd);
    if (threadIdx.x == 0) *out = s;
}

double reduce_sq(const double* x, const double* y, int64_t n) {
    if (n == 0) return 0.0;
    const int64_t nb = cdiv(n, kBlock);
    DevBuf<double> part(nb), out(1);
    const int grid = (int)std::min<int64_t>(nb, (int64_t)sm_count() * 8);
    if (y) TTG_LAUNCH(k_sq_part<true>, grid, 256, 0, stream(), x, y, n, part.get());
    else TTG_LAUNCH(k_sq_part<false>, grid, 256, 0, stream(), x, y, n, part.get());
    TTG_LAUNCH(k_sum_parts, 1, 1024, 0, stream(), part.get(), nb, out.get());
    return out.to_host(1)[0];
}

// ---------------------------------------------------------------------------
// Gram matrix G = B^T B of a tall N x s block (s <= S <= 32, column t at B + t*ld) on the
// FP64 tensor cores. A warp takes 4 rows at a time: lane l loads x_c = B(row0 + l%4,
// 8c + l/4) for the S/8 column blocks -- in the m8n8k4 fragment layouts that one value is
// both the A fragment (B^T, 8x4 row-major) and the B fragment (B, 4x8 col-major) -- and
// issues (S/8)^2 DMMAs. Each warp writes its partial G; k_gram_sum adds the partials in
// warp order (deterministic).
// ---------------------------------------------------------------------------
template <int S>
__global__ void __launch_bounds__(256) k_gram_small(const double* __restrict__ B, int64_t N, int s, int64_t ld,
                                                    double* part) {
    constexpr int CB = S / 8;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * 8 + warp, nw = (int64_t)gridDim.x * 8;
    double acc[CB][CB][2];
#pragma unroll
    for (int a = 0; a < CB; ++a)
#pragma unroll
        for (int b = 0; b < CB; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    const int kr = lane & 3, mc = lane >> 2;
    // (four row groups per trip, 12 loads in flight per lane, measured slower: 561 vs 463 us on
    // config 3's 20 x 7,962,624 R1)
    int64_t r0 = gw * 4;
    for (; r0 < N; r0 += nw * 4) {
        const int64_t row = r0 + kr;
        double x[CB];
#pragma unroll
        for (int c = 0; c < CB; ++c) {
            const int col = 8 * c + mc;
            x[c] = (row < N && col < s) ? __ldg(B + row + (int64_t)col * ld) : 0.0;
        }
#pragma unroll
        for (int a = 0; a < CB; ++a)
#pragma unroll
            for (int b = 0; b < CB; ++b) dmma(acc[a][b], x[a], x[b]);
    }
    // the CTA's 8 warps add into one S x S tile in warp order, then one partial per CTA
    __shared__ double tile[S * S];
    for (int e = threadIdx.x; e < S * S; e += 256) tile[e] = 0.0;
    for (int w = 0; w < 8; ++w) {
        __syncthreads();
        if (warp == w) {
#pragma unroll
            for (int a = 0; a < CB; ++a)
#pragma unroll
                for (int b = 0; b < CB; ++b)
#pragma unroll
                    for (int h = 0; h < 2; ++h) tile[(8 * a + mc) + (8 * b + 2 * kr + h) * S] += acc[a][b][h];
        }
    }
    __syncthreads();
    double* out = part + (int64_t)blockIdx.x * (S * S);
    for (int e = threadIdx.x; e < S * S; e += 256) out[e] = tile[e];
}

// two-level fixed-order sum of the per-CTA Gram partials: block b of the grid sums parts
// [b*per, (b+1)*per) into mid[b]; the last CTA to finish (atomic ticket) adds mid[] in order
__global__ void k_gram_sum(const double* __restrict__ part, int64_t nparts, int S, int s, double* G, double* mid,
                           unsigned* ticket) {
    const int64_t per = cdiv(nparts, (int64_t)gridDim.x);
    const int64_t p0 = (int64_t)blockIdx.x * per, p1 = min(nparts, p0 + per);
    for (int e = threadIdx.x; e < s * s; e += blockDim.x) {
        const int j = e / s, i = e - j * s;
        double a = 0.0;
        for (int64_t p = p0; p < p1; ++p) a += part[p * S * S + i + j * S];
        mid[(int64_t)blockIdx.x * s * s + e] = a;
    }
    __threadfence();
    __syncthreads();
    __shared__ unsigned last;
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int e = threadIdx.x; e < s * s; e += blockDim.x) {
        double a = 0.0;
        for (unsigned b = 0; b < gridDim.x; ++b) a += mid[(int64_t)b * s * s + e];
        G[e] = a;
    }
    if (threadIdx.x == 0) *ticket = 0;
}

// C = sum_c part[c] (+ beta C), chunks in order.
__global__ void k_reduce_chunks(const double* __restrict__ part, int64_t ks, int64_t m, int64_t n, double* C,
                                int64_t ldc, double beta) {
    const int64_t mn = m * n;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < mn; e += (int64_t)gridDim.x * blockDim.x) {
        double a = 0.0;
        for (int64_t c = 0; c < ks; ++c) a += part[c * mn + e];
        const int64_t j = e / m, i = e - j * m;
        double* cp = C + i + j * ldc;
        *cp = beta == 0.0 ? a : fma(beta, *cp, a);
    }
}

}  // namespace

namespace {
// The pipelined 128 x 128 kernel for problems that fill its tiles; operands 16-byte aligned
// with even leading dimensions (cp.async). TTG_GEMM128=0 keeps every call on k_gemm.
bool gemm128_ok(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B, int64_t ldb) {
    static const bool off = [] {
        const char* e = std::getenv("TTG_GEMM128");
        return e && *e == '0';
    }();
    const auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    return !off && m >= 96 && n >= 96 && k >= 32 && al(A) && al(B) && lda % 2 == 0 && ldb % 2 == 0;
}

template <bool TA, bool TB>
void launch128(dim3 grid, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
               int64_t ldb, double* C, int64_t ldc, double al, double be, int64_t kc, int64_t cs, int sym = 0) {
    const size_t smem = sizeof(double) * (size_t)G2STAGES * 2 * G2TILE;
    allow_smem(k_gemm128<TA, TB>, smem);
    TTG_LAUNCH((k_gemm128<TA, TB>), grid, 256, smem, stream(), m, n, k, A, lda, B, ldb, C, ldc, al, be, kc, cs,
               sym);
}

// C(i, j) = C(j, i) for i > j (the lower triangle from the upper)
__global__ void k_mirror_lower(double* C, int64_t n, int64_t ldc) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = e / n, i = e - j * n;
        if (i > j) C[i + j * ldc] = C[j + i * ldc];
    }
}
}  // namespace

void gemm(bool ta, bool tb, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
          int64_t ldb, double* C, int64_t ldc, double alpha, double beta) {
    if (m <= 0 || n <= 0) return;
    if (k > 0 && gemm128_ok(m, n, k, A, lda, B, ldb)) {
        const int sms = sm_count();
        const int64_t tiles = cdiv(m, G2M) * cdiv(n, G2N);
        if (tiles > INT32_MAX) argument_error("gemm: problem too large for one launch");
        auto go = [&](dim3 grid, double* Cp, int64_t ldcp, double al, double be, int64_t kc, int64_t cs) {
            if (!ta && !tb) launch128<false, false>(grid, m, n, k, A, lda, B, ldb, Cp, ldcp, al, be, kc, cs);
            else if (ta && !tb) launch128<true, false>(grid, m, n, k, A, lda, B, ldb, Cp, ldcp, al, be, kc, cs);
            else if (!ta && tb) launch128<false, true>(grid, m, n, k, A, lda, B, ldb, Cp, ldcp, al, be, kc, cs);
            else launch128<true, true>(grid, m, n, k, A, lda, B, ldb, Cp, ldcp, al, be, kc, cs);
        };
        if (tiles < 2 * sms && k >= 4096) {
            // few output tiles and a long K (Gram matrices of tall blocks): split K so every SM
            // gets work, partials reduced in chunk order (deterministic)
            int64_t ks = std::min<int64_t>(cdiv(2 * sms, tiles), cdiv(k, 1024));
            const int64_t kc = cdiv(cdiv(k, ks), G2K) * G2K;
            ks = cdiv(k, kc);
            if (ks > 1) {
                DevBuf<double> part((size_t)(ks * m * n));
                go(dim3((unsigned)tiles, (unsigned)ks), part.get(), m, alpha, 0.0, kc, m * n);
                TTG_LAUNCH(k_reduce_chunks, (int)std::min<int64_t>(cdiv(m * n, 256), 8 * sms), 256, 0, stream(),
                           part.get(), ks, m, n, C, ldc, beta);
                return;
            }
        }
        go(dim3((unsigned)tiles), C, ldc, alpha, beta, k, 0);
        return;
    }
    const int64_t tiles = cdiv(m, BM) * cdiv(n, BN);
    if (tiles > INT32_MAX) argument_error("gemm: problem too large for one launch");
    auto launch = [&](dim3 grid, double* Cp, int64_t ldcp, double al, double be, int64_t kc, int64_t cs) {
        if (!ta && !tb) TTG_LAUNCH((k_gemm<false, false>), grid, 128, 0, stream(), m, n, k, A, lda, B, ldb, Cp, ldcp, al, be, kc, cs);
        else if (ta && !tb) TTG_LAUNCH((k_gemm<true, false>), grid, 128, 0, stream(), m, n, k, A, lda, B, ldb, Cp, ldcp, al, be, kc, cs);
        else if (!ta && tb) TTG_LAUNCH((k_gemm<false, true>), grid, 128, 0, stream(), m, n, k, A, lda, B, ldb, Cp, ldcp, al, be, kc, cs);
        else TTG_LAUNCH((k_gemm<true, true>), grid, 128, 0, stream(), m, n, k, A, lda, B, ldb, Cp, ldcp, al, be, kc, cs);
    };
    const int sms = sm_count();
    if (tiles < sms && k >= 8192) {
        // few output tiles, long K (Gram matrices of tall blocks): split K over the SMs,
        // partials reduced in chunk order (deterministic)
        int64_t ks = std::min<int64_t>(cdiv(2 * sms, tiles), cdiv(k, 2048));
        const int64_t kc = cdiv(cdiv(k, ks), BK) * BK;
        ks = cdiv(k, kc);
        DevBuf<double> part((size_t)(ks * m * n));
        launch(dim3((unsigned)tiles, (unsigned)ks), part.get(), m, alpha, 0.0, kc, m * n);
        TTG_LAUNCH(k_reduce_chunks, (int)std::min<int64_t>(cdiv(m * n, 256), 8 * sms), 256, 0, stream(), part.get(),
                   ks, m, n, C, ldc, beta);
        return;
    }
    launch(dim3((unsigned)tiles), C, ldc, alpha, beta, k, 0);
}

void syrk(bool ta, int64_t n, int64_t k, const double* A, int64_t lda, double* C, int64_t ldc) {
    // C = op(A) op(A)^T (op(A) n x k): the tiles on and above the diagonal on the DMMA kernel,
    // then the lower triangle mirrored (about half the flops of the full product)
    if (n <= 0) return;
    const double* B = A;
    if (k <= 0 || !gemm128_ok(n, n, k, A, lda, B, lda)) {
        gemm(ta, !ta, n, n, k, A, lda, A, lda, C, ldc);
        return;
    }
    const int sms = sm_count();
    const int64_t tn = cdiv(n, G2N), tiles = tn * (tn + 1) / 2;
    auto go = [&](dim3 grid, double* Cp, int64_t ldcp, int64_t kc, int64_t cs) {
        if (ta) launch128<true, false>(grid, n, n, k, A, lda, A, lda, Cp, ldcp, 1.0, 0.0, kc, cs, 1);
        else launch128<false, true>(grid, n, n, k, A, lda, A, lda, Cp, ldcp, 1.0, 0.0, kc, cs, 1);
    };
    int64_t ks = 1, kc = k;
    if (tiles < 2 * sms && k >= 4096) {
        ks = std::min<int64_t>(cdiv(2 * sms, tiles), cdiv(k, 1024));
        kc = cdiv(cdiv(k, ks), G2K) * G2K;
        ks = cdiv(k, kc);
    }
    if (ks > 1) {
        DevBuf<double> part((size_t)(ks * n * n));
        go(dim3((unsigned)tiles, (unsigned)ks), part.get(), n, kc, n * n);
        TTG_LAUNCH(k_reduce_chunks, (int)std::min<int64_t>(cdiv(n * n, 256), 8 * sms), 256, 0, stream(), part.get(),
                   ks, n, n, C, ldc, 0.0);
    } else {
        go(dim3((unsigned)tiles), C, ldc, k, 0);
    }
    TTG_LAUNCH(k_mirror_lower, (int)std::min<int64_t>(cdiv(n * n, 256), 8 * sms), 256, 0, stream(), C, n, ldc);
}

void gram_small(const double* B, int64_t N, int64_t s, int64_t ld, double* G) {
    const int S = s <= 8 ? 8 : s <= 16 ? 16 : s <= 24 ? 24 : 32;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(4 * sm_count(), cdiv(N, 4 * 8)));
    const int64_t nparts = blocks;
    DevBuf<double> part((size_t)(nparts * S * S));
    switch (S) {
        case 8: TTG_LAUNCH(k_gram_small<8>, blocks, 256, 0, stream(), B, N, (int)s, ld, part.get()); break;
        case 16: TTG_LAUNCH(k_gram_small<16>, blocks, 256, 0, stream(), B, N, (int)s, ld, part.get()); break;
        case 24: TTG_LAUNCH(k_gram_small<24>, blocks, 256, 0, stream(), B, N, (int)s, ld, part.get()); break;
        default: TTG_LAUNCH(k_gram_small<32>, blocks, 256, 0, stream(), B, N, (int)s, ld, part.get()); break;
    }
    const int g2 = (int)std::min<int64_t>(32, nparts);
    DevBuf<double> mid((size_t)g2 * s * s);
    DevBuf<unsigned> ticket(1);
    ticket.zero();
    TTG_LAUNCH(k_gram_sum, g2, 256, 0, stream(), part.get(), nparts, S, (int)s, G, mid.get(), ticket.get());
}

void transpose(const double* A, int64_t m, int64_t n, int64_t lda, double* B, int64_t ldb) {
    if (m <= 0 || n <= 0) return;
    dim3 grid((unsigned)cdiv(m, 32), (unsigned)cdiv(n, 32));
    TTG_LAUNCH(k_transpose, grid, dim3(32, 8), 0, stream(), A, m, n, lda, B, ldb);
}

double sum_squares(const double* x, int64_t n) { return reduce_sq(x, nullptr, n); }
double diff_squares(const double* x, const double* y, int64_t n) { return reduce_sq(x, y, n); }

}  // namespace ttg
