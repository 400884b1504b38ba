// Tall in-place Householder QR with column pivoting (pass 2 of the QLP and every tall
// factor-level QRCP). Mirrors qr_col_pivot (factor.cpp:62-135) step by step on an
// N x n column-major matrix: the long dimension is split over CTAs (partial sums combined
// in CTA order by a single finishing CTA, so the arithmetic is fixed), the n columns are
// addressed through a position -> physical-column map instead of swapping memory.
//
// Step t:
//   K1 dots    (row blocks)  redundant pivot argmax; partial sigma = sum_{i>t} x_i^2 and
//                            d_j = sum_{i>t} x_i c_j(i) for every active column j
//   K2 house   (1 CTA)       combine partials; dlarfg reflector (factor.cpp:24-38);
//                            row t of R; t_j = beta (c_j(t) + d_j / v0); norm downdate and
//                            guard flags (factor.cpp:98-107); position swap
//   K3 apply   (row blocks)  v_i = x_i / v0 stored in the pivot column; c_j(i) -= t_j v_i
//                            (factor.cpp:43-58, no contraction)
//   K4 guard   (row blocks + 1 CTA, only when flagged) recompute flagged norms from rows > t
#include <cooperative_groups.h>

#include <cmath>
#include <cstdlib>
#include <string>

#include "engine.hpp"

namespace ttg {
namespace {
namespace cg = cooperative_groups;

constexpr int kT = 256;
constexpr int kSub = 1024;  // rows staged per sub-block in K1/K4

struct TallView {
    double* B;
    int64_t N, n, ld;
    double* nu;
    double* cref;
    int64_t* colmap;  // position -> physical
    int64_t* pos;     // physical -> position
    double* part;     // nblk x (n + 1)
    double* tq;       // n (physical)
    double* R;        // p x n over positions, ld = p
    int64_t ldr;
    double* beta;
    double* v0;
    double* pnorm;
    int* flag;        // [0] any flagged, [1 + j] flagged(j)
    int64_t rpb;      // rows per block
};

// Redundant pivot choice over positions t..n-1: (nu desc, position asc).
__device__ int64_t pick_pivot(const TallView& s, int64_t t, int64_t* out_pos) {
    __shared__ double bnu[kT / 32];
    __shared__ int64_t bpos[kT / 32];
    double best = -1.0;
    int64_t bp = INT64_MAX;
    // unrolled so the colmap -> nu load pairs of several positions are in flight together
#pragma unroll 8
    for (int64_t q = t + threadIdx.x; q < s.n; q += kT) {
        const double v = s.nu[s.colmap[q]];
        if (v > best || (v == best && q < bp)) { best = v; bp = q; }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int64_t op = __shfl_xor_sync(0xffffffffu, bp, o);
        if (ov > best || (ov == best && op < bp)) { best = ov; bp = op; }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) { bnu[warp] = best; bpos[warp] = bp; }
    __syncthreads();
    __shared__ int64_t spiv;
    if (threadIdx.x == 0) {
        best = -1.0;
        bp = INT64_MAX;
        for (int w = 0; w < kT / 32; ++w)
            if (bnu[w] > best || (bnu[w] == best && bpos[w] < bp)) { best = bnu[w]; bp = bpos[w]; }
        bpos[0] = bp;
        spiv = s.colmap[bp];
    }
    __syncthreads();
    *out_pos = bpos[0];
    const int64_t piv = spiv;
    __syncthreads();
    return piv;
}

// Column norms of all n columns (partials per block, combined by k_norm_fin).
__global__ void __launch_bounds__(kT) k_norm_part(TallView s, int64_t row0) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t r0 = row0 + (int64_t)blockIdx.x * s.rpb;
    const int64_t r1 = min(s.N, r0 + s.rpb);
    for (int64_t j = warp; j < s.n; j += kT / 32) {
        const double* c = s.B + j * s.ld;
        double a = 0.0;
        for (int64_t i = r0 + lane; i < r1; i += 32) a = fma(c[i], c[i], a);
        a = warp_sum(a);
        if (lane == 0) s.part[(int64_t)blockIdx.x * (s.n + 1) + j] = a;
    }
}

__global__ void __launch_bounds__(kT) k_norm_fin(TallView s, int nblk) {
    for (int64_t j = threadIdx.x; j < s.n; j += kT) {
        double a = 0.0;
        for (int b = 0; b < nblk; ++b) a += s.part[(int64_t)b * (s.n + 1) + j];
        s.nu[j] = a;
        s.cref[j] = a;
        s.colmap[j] = j;
        s.pos[j] = j;
    }
    if (threadIdx.x == 0) s.flag[0] = 0;
}

__global__ void __launch_bounds__(kT) k_dots(TallView s, int64_t t) {
    extern __shared__ double x[];  // kSub
    __shared__ double acc[1024];   // per physical column partial (n <= 1023 here; larger n use global)
    int64_t pp;
    const int64_t piv = pick_pivot(s, t, &pp);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t r0 = max(t + 1, (int64_t)blockIdx.x * s.rpb);
    const int64_t r1 = min(s.N, (int64_t)(blockIdx.x + 1) * s.rpb);
    double* outp = s.part + (int64_t)blockIdx.x * (s.n + 1);
    const bool smem_acc = s.n < 1024;
    for (int64_t j = threadIdx.x; j <= s.n; j += kT) {
        if (smem_acc) acc[j < 1024 ? j : 0] = 0.0;
        else outp[j] = 0.0;
    }
    __syncthreads();
    double sig = 0.0;
    const double* xp = s.B + piv * s.ld;
    for (int64_t b0 = r0; b0 < r1; b0 += kSub) {
        const int64_t b1 = min(r1, b0 + kSub);
        __syncthreads();
        for (int64_t i = b0 + threadIdx.x; i < b1; i += kT) {
            const double v = xp[i];
            x[i - b0] = v;
            sig = fma(v, v, sig);
        }
        __syncthreads();
        for (int64_t q = t + warp; q < s.n; q += kT / 32) {
            const int64_t j = s.colmap[q];
            if (j == piv) continue;
            const double* c = s.B + j * s.ld;
            double a = 0.0;
            for (int64_t i = b0 + lane; i < b1; i += 32) a = fma(x[i - b0], c[i], a);
            a = warp_sum(a);
            if (lane == 0) {
                if (smem_acc) acc[j] += a;
                else outp[j] += a;
            }
        }
    }
    __shared__ double sd[kT / 32];
    sig = block_sum(sig, sd);
    __syncthreads();
    if (smem_acc)
        for (int64_t j = threadIdx.x; j < s.n; j += kT) outp[j] = acc[j];
    if (threadIdx.x == 0) outp[s.n] = sig;
}

__global__ void __launch_bounds__(kT) k_house(TallView s, int64_t t, int nblk) {
    int64_t pp;
    const int64_t piv = pick_pivot(s, t, &pp);
    __shared__ double sh[4];
    // sigma: combine partials in block order.
    double sg = 0.0;
    if (threadIdx.x == 0) {
        for (int b = 0; b < nblk; ++b) sg += s.part[(int64_t)b * (s.n + 1) + s.n];
        const double alpha = s.B[t + piv * s.ld];
        const int64_t len = s.N - t;
        double beta = 0.0, v0 = 1.0, rkk = alpha;
        if (len > 1 && sg != 0.0) {
            const double mu = __dsqrt_rn(__dadd_rn(__dmul_rn(alpha, alpha), sg));
            const double smu = copysign(mu, alpha);
            v0 = __dadd_rn(alpha, smu);
            beta = __ddiv_rn(__dmul_rn(v0, v0), __dmul_rn(smu, v0));
            rkk = -smu;
        }
        sh[0] = beta;
        sh[1] = v0;
        sh[2] = rkk;
        s.beta[t] = beta;
        s.v0[t] = v0;
        s.pnorm[t] = s.nu[piv];
        s.B[t + piv * s.ld] = rkk;
        // position swap (factor.cpp:88-93)
        const int64_t other = s.colmap[t];
        s.colmap[t] = piv;
        s.colmap[pp] = other;
        s.pos[piv] = t;
        s.pos[other] = pp;
        s.flag[0] = 0;
    }
    __syncthreads();
    const double beta = sh[0], v0 = sh[1];
    for (int64_t q = t + 1 + threadIdx.x; q < s.n; q += kT) {
        const int64_t j = s.colmap[q];
        double d = 0.0;
        for (int b = 0; b < nblk; ++b) d += s.part[(int64_t)b * (s.n + 1) + j];
        const double c0 = s.B[t + j * s.ld];
        double tj = 0.0, rt = c0;
        if (beta != 0.0) {
            tj = __dmul_rn(beta, __dadd_rn(c0, __ddiv_rn(d, v0)));
            rt = __dsub_rn(c0, tj);
        }
        s.tq[j] = tj;
        s.B[t + j * s.ld] = rt;
        const double nv = __dsub_rn(s.nu[j], __dmul_rn(rt, rt));
        s.nu[j] = nv;
        const int fl = (nv < __dmul_rn(1e-16, s.cref[j]) || nv < 0.0) ? 1 : 0;
        s.flag[1 + j] = fl;
        if (fl) atomicOr(&s.flag[0], 1);
    }
}

__global__ void __launch_bounds__(kT) k_apply(TallView s, int64_t t) {
    const double beta = s.beta[t];
    if (beta == 0.0) return;
    const double v0 = s.v0[t];
    const int64_t piv = s.colmap[t];
    const int64_t r0 = max(t + 1, (int64_t)blockIdx.x * s.rpb);
    const int64_t r1 = min(s.N, (int64_t)(blockIdx.x + 1) * s.rpb);
    double* xp = s.B + piv * s.ld;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += kT) {
        const double v = __ddiv_rn(xp[i], v0);
        xp[i] = v;
        for (int64_t q = t + 1; q < s.n; ++q) {
            const int64_t j = s.colmap[q];
            double* c = s.B + j * s.ld + i;
            *c = __dsub_rn(*c, __dmul_rn(s.tq[j], v));
        }
    }
}

__global__ void __launch_bounds__(kT) k_guard_part(TallView s, int64_t t) {
    if (s.flag[0] == 0) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t r0 = max(t + 1, (int64_t)blockIdx.x * s.rpb);
    const int64_t r1 = min(s.N, (int64_t)(blockIdx.x + 1) * s.rpb);
    for (int64_t q = t + 1 + warp; q < s.n; q += kT / 32) {
        const int64_t j = s.colmap[q];
        if (!s.flag[1 + j]) continue;
        const double* c = s.B + j * s.ld;
        double a = 0.0;
        for (int64_t i = r0 + lane; i < r1; i += 32) a = fma(c[i], c[i], a);
        a = warp_sum(a);
        if (lane == 0) s.part[(int64_t)blockIdx.x * (s.n + 1) + j] = a;
    }
}

__global__ void __launch_bounds__(kT) k_guard_fin(TallView s, int64_t t, int nblk) {
    if (s.flag[0] == 0) return;
    for (int64_t q = t + 1 + threadIdx.x; q < s.n; q += kT) {
        const int64_t j = s.colmap[q];
        if (!s.flag[1 + j]) continue;
        double a = 0.0;
        for (int b = 0; b < nblk; ++b) {
            // blocks entirely above row t+1 wrote nothing for this step: skip them
            const int64_t r1 = min(s.N, (int64_t)(b + 1) * s.rpb);
            if (r1 <= t + 1) continue;
            a += s.part[(int64_t)b * (s.n + 1) + j];
        }
        s.nu[j] = a;
        s.cref[j] = a;
    }
}

// Q formation: reflector t applied to columns [t, q) of Q (backward accumulation,
// factor.cpp:116-133). Partial dots per block, combine, apply.
__global__ void __launch_bounds__(kT) k_q_dots(TallView s, int64_t t, const double* Q, int64_t ldq, int64_t q) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t r0 = max(t + 1, (int64_t)blockIdx.x * s.rpb);
    const int64_t r1 = min(s.N, (int64_t)(blockIdx.x + 1) * s.rpb);
    const double* v = s.B + s.colmap[t] * s.ld;
    for (int64_t j = t + warp; j < q; j += kT / 32) {
        const double* c = Q + j * ldq;
        double a = 0.0;
        for (int64_t i = r0 + lane; i < r1; i += 32) a = fma(v[i], c[i], a);
        a = warp_sum(a);
        if (lane == 0) s.part[(int64_t)blockIdx.x * (s.n + 1) + (j - t)] = a;
    }
}

__global__ void __launch_bounds__(kT) k_q_fin(TallView s, int64_t t, const double* Q, int64_t ldq, int64_t q,
                                              int nblk) {
    const double beta = s.beta[t];
    for (int64_t j = t + threadIdx.x; j < q; j += kT) {
        double a = Q[t + j * ldq];
        for (int b = 0; b < nblk; ++b) {
            const int64_t r1 = min(s.N, (int64_t)(b + 1) * s.rpb);
            if (r1 <= t + 1) continue;
            a += s.part[(int64_t)b * (s.n + 1) + (j - t)];
        }
        s.tq[j - t] = __dmul_rn(a, beta);
    }
}

__global__ void __launch_bounds__(kT) k_q_apply(TallView s, int64_t t, double* Q, int64_t ldq, int64_t q) {
    const int64_t r0 = max(t, (int64_t)blockIdx.x * s.rpb);
    const int64_t r1 = min(s.N, (int64_t)(blockIdx.x + 1) * s.rpb);
    const double* v = s.B + s.colmap[t] * s.ld;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += kT) {
        const double vi = i == t ? 1.0 : v[i];
        for (int64_t j = t; j < q; ++j) {
            double* c = Q + i + j * ldq;
            *c = __dsub_rn(*c, __dmul_rn(s.tq[j - t], vi));
        }
    }
}

// R over final positions: R(t,q) = B(t, colmap[q]) for t <= q (rows < steps), else 0.
__global__ void k_extract_r(TallView s, int64_t steps, double* out, int64_t ldo) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= steps * s.n) return;
    const int64_t q = e / steps, t = e - q * steps;
    out[t + q * ldo] = t <= q ? s.B[t + s.colmap[q] * s.ld] : 0.0;
}

__global__ void k_eye(double* Q, int64_t N, int64_t q, int64_t ldq) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < N * q) {
        const int64_t j = e / N, i = e - j * N;
        Q[i + j * ldq] = i == j ? 1.0 : 0.0;
    }
}


// ---- column-parallel step (col mode: N <= kColRows) ------------------------------------
// For square and moderately tall matrices the row blocks above leave most SMs idle and
// loop over every column inside a CTA. Col mode keeps qr_col_pivot's per-column structure
// instead: one CTA per trailing column does the dot, the update (factor.cpp:43-58), the
// row-t value, the norm downdate and -- when the guard flags it -- the recompute of the
// norm from the column it just updated (factor.cpp:98-107), in one read and one write of
// the column. A single CTA picks the pivot and builds the reflector beforehand.
constexpr int64_t kColRows = 25600;  // column staged in shared memory (<= 200 KB)
constexpr int64_t kQBlock = 32;     // reflectors per compact-WY block in form_q

// pick_pivot for NT threads
template <int NT>
__device__ int64_t pick_pivot_nt(const TallView& s, int64_t t, int64_t* out_pos) {
    __shared__ double bnu[NT / 32];
    __shared__ int64_t bpos[NT / 32];
    __shared__ int64_t spiv;
    double best = -1.0;
    int64_t bp = INT64_MAX;
#pragma unroll 4
    for (int64_t q = t + threadIdx.x; q < s.n; q += NT) {
        const double v = s.nu[s.colmap[q]];
        if (v > best || (v == best && q < bp)) { best = v; bp = q; }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int64_t op = __shfl_xor_sync(0xffffffffu, bp, o);
        if (ov > best || (ov == best && op < bp)) { best = ov; bp = op; }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) { bnu[warp] = best; bpos[warp] = bp; }
    __syncthreads();
    if (warp == 0) {  // one warp folds the NT/32 warp results
        best = lane < NT / 32 ? bnu[lane] : -1.0;
        bp = lane < NT / 32 ? bpos[lane] : INT64_MAX;
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, best, o);
            const int64_t op = __shfl_xor_sync(0xffffffffu, bp, o);
            if (ov > best || (ov == best && op < bp)) { best = ov; bp = op; }
        }
        if (lane == 0) {
            bpos[0] = bp;
            spiv = s.colmap[bp];
        }
    }
    __syncthreads();
    *out_pos = bpos[0];
    return spiv;
}

// Step t's pivot and reflector (make_householder, factor.cpp:24-38): one CTA of 1024
// threads, so the pivot scan, the column mass and the normalisation are one batch of
// loads per thread for columns of up to 4096 rows.
constexpr int kHouseT = 1024;
__global__ void __launch_bounds__(kHouseT) k_col_house(TallView s, int64_t t) {
    int64_t pp;
    const int64_t piv = pick_pivot_nt<kHouseT>(s, t, &pp);
    __shared__ double sd[kHouseT / 32];
    __shared__ double sh[2];
    double* x = s.B + piv * s.ld;
    double sg = 0.0;
#pragma unroll 4
    for (int64_t i = t + 1 + threadIdx.x; i < s.N; i += kHouseT) sg = fma(x[i], x[i], sg);
    sg = block_sum(sg, sd);
    if (threadIdx.x == 0) {
        const double alpha = x[t];
        const int64_t len = s.N - t;
        double beta = 0.0, v0 = 1.0, rkk = alpha;
        if (len > 1 && sg != 0.0) {  // make_householder (factor.cpp:24-38)
            const double mu = __dsqrt_rn(__dadd_rn(__dmul_rn(alpha, alpha), sg));
            const double smu = copysign(mu, alpha);
            v0 = __dadd_rn(alpha, smu);
            beta = __ddiv_rn(__dmul_rn(v0, v0), __dmul_rn(smu, v0));
            rkk = -smu;
        }
        sh[0] = beta;
        sh[1] = v0;
        s.beta[t] = beta;
        s.v0[t] = v0;
        s.pnorm[t] = s.nu[piv];
        x[t] = rkk;
        const int64_t other = s.colmap[t];
        s.colmap[t] = piv;
        s.colmap[pp] = other;
        s.pos[piv] = t;
        s.pos[other] = pp;
    }
    __syncthreads();
    const double beta = sh[0], v0 = sh[1];
    if (beta != 0.0)
#pragma unroll 4
        for (int64_t i = t + 1 + threadIdx.x; i < s.N; i += kHouseT) x[i] = __ddiv_rn(x[i], v0);
}

__global__ void __launch_bounds__(kT) k_col_apply(TallView s, int64_t t) {
    extern __shared__ double cs[];  // rows t+1.. of this CTA's column
    __shared__ double sd[kT / 32];
    const int64_t j = s.colmap[t + 1 + blockIdx.x];
    const double beta = s.beta[t];
    const double* __restrict__ v = s.B + s.colmap[t] * s.ld;
    double* c = s.B + j * s.ld;
    double rt = c[t];
    double sq = 0.0;
    bool fl;
    if (beta != 0.0) {
        double d = 0.0;
#pragma unroll 4
        for (int64_t i = t + 1 + threadIdx.x; i < s.N; i += kT) {
            const double xi = c[i];
            cs[i - t - 1] = xi;
            d = fma(v[i], xi, d);
        }
        d = block_sum(d, sd);
        const double tj = __dmul_rn(beta, __dadd_rn(rt, d));
        rt = __dsub_rn(rt, tj);
#pragma unroll 4
        for (int64_t i = t + 1 + threadIdx.x; i < s.N; i += kT) {
            const double y = __dsub_rn(cs[i - t - 1], __dmul_rn(tj, v[i]));
            c[i] = y;
            sq = fma(y, y, sq);
        }
        sq = block_sum(sq, sd);
        const double nv = __dsub_rn(s.nu[j], __dmul_rn(rt, rt));
        fl = nv < __dmul_rn(1e-16, s.cref[j]) || nv < 0.0;
        if (threadIdx.x == 0) {
            c[t] = rt;
            s.nu[j] = fl ? sq : nv;
            if (fl) s.cref[j] = sq;
        }
    } else {  // H_t = I: the column is unchanged, only the norm downdate and the guard
        const double nv = __dsub_rn(s.nu[j], __dmul_rn(rt, rt));
        fl = nv < __dmul_rn(1e-16, s.cref[j]) || nv < 0.0;
        if (fl) {
            for (int64_t i = t + 1 + threadIdx.x; i < s.N; i += kT) sq = fma(c[i], c[i], sq);
            sq = block_sum(sq, sd);
        }
        if (threadIdx.x == 0) {
            s.nu[j] = fl ? sq : nv;
            if (fl) s.cref[j] = sq;
        }
    }
}

// Q formation in col mode: reflector t applied to columns [t, q) of Q, one CTA per column
// (the k_col_apply structure; factor.cpp:116-133 per column).
__global__ void __launch_bounds__(kT) k_q_col(TallView s, int64_t t, double* Q, int64_t ldq) {
    __shared__ double sd[kT / 32];
    const double beta = s.beta[t];
    const double* __restrict__ v = s.B + s.colmap[t] * s.ld;
    double* c = Q + (t + blockIdx.x) * ldq;
    double d = 0.0;
#pragma unroll 4
    for (int64_t i = t + 1 + threadIdx.x; i < s.N; i += kT) d = fma(v[i], c[i], d);
    d = block_sum(d, sd);
    const double tj = __dmul_rn(__dadd_rn(c[t], d), beta);
#pragma unroll 4
    for (int64_t i = t + 1 + threadIdx.x; i < s.N; i += kT) c[i] = __dsub_rn(c[i], __dmul_rn(tj, v[i]));
    if (threadIdx.x == 0) c[t] = __dsub_rn(c[t], tj);
}

// Short columns (N <= kWarpRows): a warp per column, the column held in registers (lane l
// owns rows t+1+l, t+1+l+32, ...), eight columns per CTA.
constexpr int64_t kWarpRows = 2048;

template <int R>  // rows per lane: R * 32 >= N - t - 1
__global__ void __launch_bounds__(kT) k_col_apply_warp(TallView s, int64_t t) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t q = t + 1 + (int64_t)blockIdx.x * (kT / 32) + warp;
    if (q >= s.n) return;
    const int64_t j = s.colmap[q];
    const double beta = s.beta[t];
    const double* __restrict__ v = s.B + s.colmap[t] * s.ld;
    double* c = s.B + j * s.ld;
    double rt = c[t];
    double x[R];
    double d = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = t + 1 + lane + 32 * r;
        x[r] = i < s.N ? c[i] : 0.0;
        if (i < s.N) d = fma(v[i], x[r], d);
    }
    double sq = 0.0;
    if (beta != 0.0) {
        d = warp_sum(d);
        const double tj = __dmul_rn(beta, __dadd_rn(rt, d));
        rt = __dsub_rn(rt, tj);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t i = t + 1 + lane + 32 * r;
            if (i < s.N) {
                const double y = __dsub_rn(x[r], __dmul_rn(tj, v[i]));
                c[i] = y;
                sq = fma(y, y, sq);
            }
        }
    } else {
#pragma unroll
        for (int r = 0; r < R; ++r) sq = fma(x[r], x[r], sq);
    }
    sq = warp_sum(sq);
    if (lane == 0) {
        const double nv = __dsub_rn(s.nu[j], __dmul_rn(rt, rt));
        const bool fl = nv < __dmul_rn(1e-16, s.cref[j]) || nv < 0.0;
        if (beta != 0.0) c[t] = rt;
        s.nu[j] = fl ? sq : nv;
        if (fl) s.cref[j] = sq;
    }
}

// Col-mode initial norms: a warp per column over all rows (sequential lane partials + tree).
__global__ void __launch_bounds__(kT) k_col_norms(TallView s) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t j = (int64_t)blockIdx.x * (kT / 32) + warp;
    if (j >= s.n) return;
    const double* c = s.B + j * s.ld;
    double a = 0.0;
#pragma unroll 8
    for (int64_t i = lane; i < s.N; i += 32) a = fma(c[i], c[i], a);
    a = warp_sum(a);
    if (lane == 0) {
        s.nu[j] = a;
        s.cref[j] = a;
        s.colmap[j] = j;
        s.pos[j] = j;
    }
    if (j == 0 && lane == 0) s.flag[0] = 0;
}

// k_col_apply with the column in registers (thread r holds rows t+1+r, t+1+r+kT, ...):
// no shared memory, so several CTAs share an SM (R * kT >= N - t - 1).
template <int R, int NT = kT>
__global__ void __launch_bounds__(NT) k_col_apply_reg(TallView s, int64_t t) {
    __shared__ double sd[NT / 32];
    const int64_t j = s.colmap[t + 1 + blockIdx.x];
    const double beta = s.beta[t];
    const double* __restrict__ v = s.B + s.colmap[t] * s.ld;
    double* c = s.B + j * s.ld;
    double rt = c[t];
    double x[R], w[R];
    double d = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = t + 1 + threadIdx.x + (int64_t)NT * r;
        const bool in = i < s.N;
        x[r] = in ? c[i] : 0.0;
        w[r] = in ? v[i] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) d = fma(w[r], x[r], d);
    double sq = 0.0;
    if (beta != 0.0) {
        d = block_sum(d, sd);
        const double tj = __dmul_rn(beta, __dadd_rn(rt, d));
        rt = __dsub_rn(rt, tj);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t i = t + 1 + threadIdx.x + (int64_t)NT * r;
            if (i < s.N) {
                const double y = __dsub_rn(x[r], __dmul_rn(tj, w[r]));
                c[i] = y;
                sq = fma(y, y, sq);
            }
        }
    } else {
#pragma unroll
        for (int r = 0; r < R; ++r) sq = fma(x[r], x[r], sq);
    }
    sq = block_sum(sq, sd);
    if (threadIdx.x == 0) {
        const double nv = __dsub_rn(s.nu[j], __dmul_rn(rt, rt));
        const bool fl = nv < __dmul_rn(1e-16, s.cref[j]) || nv < 0.0;
        if (beta != 0.0) c[t] = rt;
        s.nu[j] = fl ? sq : nv;
        if (fl) s.cref[j] = sq;
    }
}

// Blocked Q formation (col mode): the reflectors of steps [b0, b0 + kb) as one compact-WY
// block H_b0 ... H_{b0+kb-1} = I - V T V^T (V gathered from the pivot columns, T by the
// forward column-wise recurrence from the Gram matrix V^T V), applied to Q[b0:, b0:q]
// with three DMMA GEMMs (W = V^T Q, W = T W, Q -= V W), blocks taken last to first.
__global__ void k_gather_v(TallView s, int64_t b0, int kb, double* V) {
    const int64_t rows = s.N - b0;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= rows * kb) return;
    const int64_t jj = e / rows, i = e - jj * rows;
    const int64_t r = b0 + i, j = b0 + jj;
    V[e] = r < j ? 0.0 : (r == j ? 1.0 : s.B[r + s.colmap[j] * s.ld]);
}

// T (kb x kb, upper): T(j, j) = beta_j, T(0:j, j) = -beta_j T(0:j, 0:j) G(0:j, j).
__global__ void k_larft(const double* __restrict__ G, const double* __restrict__ beta, int kb, double* T) {
    __shared__ double Ts[64 * 65];
    __shared__ double col[64];
    for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) Ts[(e % kb) + (e / kb) * 65] = 0.0;
    __syncthreads();
    for (int j = 0; j < kb; ++j) {
        const double bj = beta[j];
        if (threadIdx.x < j) {
            double a = 0.0;
            for (int l = threadIdx.x; l < j; ++l) a = fma(Ts[threadIdx.x + l * 65], G[l + j * kb], a);
            col[threadIdx.x] = -bj * a;
        }
        __syncthreads();
        if (threadIdx.x < j) Ts[threadIdx.x + j * 65] = col[threadIdx.x];
        if (threadIdx.x == 0) Ts[j + j * 65] = bj;
        __syncthreads();
    }
    for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) T[e] = Ts[(e % kb) + (e / kb) * 65];
}

// ---- persistent blocked steps (one cooperative launch per run) --------------------------
// Per-step application of H_t to every trailing column reads AND writes the whole trailing
// matrix once per step. A panel of kb steps (the dlaqps organisation) instead leaves the
// trailing columns untouched below the panel's rows and keeps the pending update in
// factored form, B <- B - V F^T (V: the panel's reflectors, F(j, l) = beta_l
// (H_{l-1}..H_0 b_j)^T v_l), so a step only READS the trailing matrix, and the whole update
// lands once per panel as FP64 tensor-core (DMMA) tiles. The grid stays resident for the run:
// two grid barriers per step, every per-column quantity (norm, position, the column's row of
// F) in the owning CTA's shared memory. Exact arithmetic gives factor.cpp's values; the
// rounding differs from its column-by-column order at the ulp level.
//  * physical column j belongs to CTA j mod G for the run (pivoting relabels positions, so a
//    pivot only leaves its owner's list);
//  * phase P (after barrier A): every CTA reads the G candidate records and picks the same
//    pivot (factor.cpp:85-87); CTA g brings rows slice g of the pivot column up to date,
//    x = b_p - V F(p, :)^T, and publishes its partial sigma, V^T x (and x(t) if it holds row
//    t); the owners update the position map (factor.cpp:88-93);
//  * phase G (after barrier B): every CTA combines the G partials in CTA order and rebuilds
//    the same reflector (make_householder, factor.cpp:24-38), stages v, and runs the
//    read-only GEMV, F(j, k), R(t, j), downdate and guard (factor.cpp:98-107) for its own
//    columns; publishes its best candidate;
//  * panel end: each CTA applies B(t1:, j) -= V F(j, :)^T to its own columns as DMMA tiles
//    (V from L2, F from shared memory) and stores the finished reflectors in their pivot
//    columns.
constexpr int kNb = 32;  // reflectors per panel

struct BlkView {
    double* B;
    int64_t N, n, ld;
    double* nu;
    double* cref;
    int64_t* colmap;
    int64_t* pos;
    double* beta;
    double* v0;
    double* pnorm;
    double* Vp;  // N x kNb, column l = reflector t0 + l (1 at its row, 0 above)
    double* F;   // n x kNb by physical column
};

constexpr int kPT = 512;  // threads per CTA

struct PersistArgs {
    BlkView s;
    double* part;    // [G][kNb + 2]: sigma, V^T x (kNb), x(t)
    Cand* pcand;     // [2][G]
    int64_t t0, t1;
    int nloc;        // owned-column capacity per CTA
};

__global__ void __launch_bounds__(kPT, 1) k_qrcp_persist(PersistArgs A) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double psm[];
    const BlkView& s = A.s;
    const int64_t N = s.N, n = s.n;
    const int G = gridDim.x, me = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = kPT / 32;
    const int nloc = A.nloc;
    // shared: vsm[N] | ofl[nloc * kNb] (F rows of owned columns) | onu | ocref [nloc] | ocol | opos (int64)
    double* vsm = psm;
    double* ofl = vsm + N;
    double* onu = ofl + (size_t)nloc * kNb;
    double* ocref = onu + nloc;
    int64_t* ocol = reinterpret_cast<int64_t*>(ocref + nloc);
    int64_t* opos = ocol + nloc;
    __shared__ int cnt_s;
    __shared__ Cand sc[NW];
    __shared__ double red[NW];
    __shared__ double fp[kNb];
    __shared__ double hsm[3 + kNb];
    __shared__ double vt[kNb];
    __shared__ double comb[kNb + 2];
    __shared__ Cand win_s;

    if (tid == 0) {
        int c = 0;
        for (int64_t j = me; j < n; j += G) {
            const int64_t q = s.pos[j];
            if (q >= A.t0) {
                ocol[c] = j;
                opos[c] = q;
                onu[c] = s.nu[j];
                ocref[c] = s.cref[j];
                ++c;
            }
        }
        cnt_s = c;
    }
    __syncthreads();
    int cnt = cnt_s;
    auto publish = [&](int64_t slot) {
        Cand b = cand_none();
        for (int l = tid; l < cnt; l += kPT) {
            const Cand c{onu[l], opos[l], ocol[l]};
            if (better(c, b)) b = c;
        }
        b = block_best(b, sc);
        if (tid == 0) A.pcand[slot * G + me] = b;
    };
    publish(A.t0 & 1);
    for (int64_t t0 = A.t0; t0 < A.t1; t0 += kNb) {
        const int kb = (int)min((int64_t)kNb, A.t1 - t0);
        // panel start: V's rows above each reflector read as zero
        for (int64_t e = (int64_t)me * kPT + tid; e < N * kb; e += (int64_t)G * kPT) s.Vp[e] = 0.0;
        grid.sync();
        for (int k = 0; k < kb; ++k) {
            const int64_t t = t0 + k;
            // ---- phase P ----
            if (warp == 0) {
                Cand b = cand_none();
                for (int g = lane; g < G; g += 32) {
                    const Cand* cp = A.pcand + (t & 1) * G + g;
                    const Cand c{__ldcg(&cp->nu), __ldcg(&cp->pos), __ldcg(&cp->col)};
                    if (better(c, b)) b = c;
                }
                b = warp_best(b);
                if (lane == 0) win_s = b;
            }
            __syncthreads();
            const Cand win = win_s;
            const int64_t piv = win.col, pp = win.pos;
            if (tid < k) fp[tid] = __ldcg(s.F + piv + (int64_t)tid * n);
            // bookkeeping (factor.cpp:88-93): the pivot leaves its owner's list; the column
            // at position t moves to pp
            if (tid == 0) {
                int c = cnt;
                for (int l = 0; l < c; ++l) {
                    if (ocol[l] == piv) {
                        s.colmap[t] = piv;
                        s.pos[piv] = t;
                        s.pnorm[t] = onu[l];
                        --c;
                        ocol[l] = ocol[c]; opos[l] = opos[c]; onu[l] = onu[c]; ocref[l] = ocref[c];
                        for (int q = 0; q < k; ++q) ofl[(size_t)l * kNb + q] = ofl[(size_t)c * kNb + q];
                        --l;
                        continue;
                    }
                    if (opos[l] == t && pp != t) {
                        opos[l] = pp;
                        s.colmap[pp] = ocol[l];
                        s.pos[ocol[l]] = pp;
                    }
                }
                cnt_s = c;
            }
            __syncthreads();
            cnt = cnt_s;
            {
                // rows slice `me` of [t, N): x = b_p - V F(p, :)^T and the partial sums
                const int64_t per = cdiv(N - t, G);
                const int64_t r0 = t + (int64_t)me * per, r1 = min(N, r0 + per);
                double* x = s.B + piv * s.ld;
                double* part = A.part + (size_t)me * (kNb + 2);
                for (int64_t i = r0 + tid; i < r1; i += kPT) {
                    double xi = __ldcg(x + i);
                    double vl[kNb];
#pragma unroll
                    for (int l = 0; l < kNb; ++l) vl[l] = l < k ? __ldcg(s.Vp + i + l * N) : 0.0;
#pragma unroll
                    for (int l = 0; l < kNb; ++l)
                        if (l < k) xi = fma(-vl[l], fp[l], xi);
                    __stcg(x + i, xi);
                    vsm[i - r0] = xi;  // scratch: this slice's x
                    if (i == t) part[kNb + 1] = xi;
                }
                __syncthreads();
                // sigma and V(t+1:, l)^T x over the slice: a warp per quantity, lanes over rows
                for (int q = warp; q <= k; q += NW) {
                    double a = 0.0;
                    for (int64_t i = max(r0, t + 1) + lane; i < r1; i += 32) {
                        const double xi = vsm[i - r0];
                        a = fma(q == 0 ? xi : __ldcg(s.Vp + i + (q - 1) * N), xi, a);
                    }
                    a = warp_sum(a);
                    if (lane == 0) part[q] = a;
                }
            }
            grid.sync();  // barrier B
            // ---- phase G ----
            for (int q = warp; q <= k; q += NW) {  // combine the G partials in CTA order
                double a = 0.0;
                for (int g = lane; g < G; g += 32) a += __ldcg(A.part + (size_t)g * (kNb + 2) + q);
                a = warp_sum(a);
                if (lane == 0) comb[q] = a;
            }
            if (tid < k) vt[tid] = __ldcg(s.Vp + t + (int64_t)tid * N);
            __syncthreads();
            if (tid == 0) {
                const double sg = comb[0], alpha = __ldcg(A.part + (kNb + 1));  // CTA 0 holds row t
                double beta = 0.0, v0 = 1.0, rkk = alpha;
                if (N - t > 1 && sg != 0.0) {  // make_householder (factor.cpp:24-38)
                    const double mu = __dsqrt_rn(__dadd_rn(__dmul_rn(alpha, alpha), sg));
                    const double smu = copysign(mu, alpha);
                    v0 = __dadd_rn(alpha, smu);
                    beta = __ddiv_rn(__dmul_rn(v0, v0), __dmul_rn(smu, v0));
                    rkk = -smu;
                }
                hsm[0] = beta;
                hsm[1] = v0;
                hsm[2] = rkk;
            }
            __syncthreads();
            const double beta = hsm[0], v0 = hsm[1];
            if (tid < k) hsm[3 + tid] = -beta * (vt[tid] + comb[1 + tid] / v0);
            {
                // v over rows t.. (v_t = 1); this CTA stores its rows slice of V's column k
                const double* x = s.B + piv * s.ld;
                const int64_t per = cdiv(N - t, G);
                const int64_t r0 = t + (int64_t)me * per, r1 = min(N, r0 + per);
                for (int64_t i = t + tid; i < N; i += kPT) {
                    const double v = i == t ? 1.0 : (beta != 0.0 ? __ddiv_rn(__ldcg(x + i), v0) : 0.0);
                    vsm[i - t] = v;
                    if (i >= r0 && i < r1) s.Vp[i + (int64_t)k * N] = v;
                }
            }
            if ((int)(piv % G) == me && tid == 0) {
                s.beta[t] = beta;
                s.v0[t] = v0;
                s.B[t + piv * s.ld] = hsm[2];
            }
            __syncthreads();
            // own trailing columns: GEMV, epilogue, downdate + guard
            for (int l = warp; l < cnt; l += NW) {
                const int64_t j = ocol[l];
                const double* c = s.B + j * s.ld;
                double a = 0.0;
                if (beta != 0.0) {
#pragma unroll 16
                    for (int64_t i = t + lane; i < N; i += 32) a = fma(vsm[i - t], __ldcg(c + i), a);
                    a = warp_sum(a);
                }
                double p1 = 0.0, p2 = 0.0;
                if (lane < k) {
                    const double fl = ofl[(size_t)l * kNb + lane];
                    p1 = fl * hsm[3 + lane];
                    p2 = vt[lane] * fl;
                }
                p1 = warp_sum(p1);
                p2 = warp_sum(p2);
                const double f = fma(beta, a, p1);
                const double rt = __dsub_rn(__dsub_rn(__ldcg(c + t), p2), f);
                double nv = __dsub_rn(onu[l], __dmul_rn(rt, rt));
                const bool flag = nv < __dmul_rn(1e-16, ocref[l]) || nv < 0.0;
                if (flag) {  // guard (factor.cpp:103-105): |b_j(t+1:) - V F(j, :)^T|^2
                    double q = 0.0;
                    for (int64_t i = t + 1 + lane; i < N; i += 32) {
                        double y = __ldcg(c + i);
                        for (int m = 0; m < k; ++m) y = fma(-__ldcg(s.Vp + i + (int64_t)m * N), ofl[(size_t)l * kNb + m], y);
                        y = fma(-vsm[i - t], f, y);
                        q = fma(y, y, q);
                    }
                    nv = warp_sum(q);
                }
                if (lane == 0) {
                    ofl[(size_t)l * kNb + k] = f;
                    s.F[j + (int64_t)k * n] = f;
                    s.B[t + j * s.ld] = rt;
                    onu[l] = nv;
                    if (flag) ocref[l] = nv;
                }
            }
            __syncthreads();
            publish((t + 1) & 1);
            grid.sync();  // barrier A
        }
        // ---- panel end: own trailing columns B(t1:, j) -= V(t1:, :kb) F(j, :kb)^T (DMMA) ----
        const int64_t t1 = t0 + kb;
        if (t1 < N && t1 < n) {
            const int ar = lane >> 2, ak = lane & 3;
            const int64_t nrt = cdiv(N - t1, 32), nct = cdiv(cnt, 8);
            for (int64_t u = warp; u < nrt * nct; u += NW) {
                const int64_t rt = u % nrt, ct = u / nrt;
                const int64_t row0 = t1 + rt * 32;
                const int cl = (int)(ct * 8 + ar);             // B fragment column (owned index)
                const bool cok = cl < cnt;
                double d[4][2];
                int64_t dj[2];
                bool dok[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int ce = (int)(ct * 8 + 2 * ak + e);
                    dok[e] = ce < cnt;
                    dj[e] = dok[e] ? ocol[ce] : 0;
                }
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const int64_t r = row0 + a * 8 + ar;
#pragma unroll
                    for (int e = 0; e < 2; ++e) d[a][e] = (r < N && dok[e]) ? -__ldcg(s.B + r + dj[e] * s.ld) : 0.0;
                }
                for (int kk = 0; kk < kb; kk += 4) {
                    const int kq = kk + ak;
                    const double bf = (cok && kq < kb) ? ofl[(size_t)cl * kNb + kq] : 0.0;
#pragma unroll
                    for (int a = 0; a < 4; ++a) {
                        const int64_t r = row0 + a * 8 + ar;
                        const double af = (r < N && kq < kb) ? __ldcg(s.Vp + r + (int64_t)kq * N) : 0.0;
                        dmma(d[a], af, bf);
                    }
                }
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const int64_t r = row0 + a * 8 + ar;
                    if (r >= N) continue;
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        if (dok[e]) __stcg(s.B + r + dj[e] * s.ld, -d[a][e]);
                }
            }
        }
        // the panel's reflectors into their pivot columns (owners), below the diagonal
        for (int u = 0; u < kb; ++u) {
            const int64_t t = t0 + u;
            const int64_t pj = __ldcg(s.colmap + t);
            if ((int)(pj % G) != me) continue;
            if (__ldcg(s.beta + t) == 0.0) continue;
            double* x = s.B + pj * s.ld;
            for (int64_t i = t + 1 + tid; i < N; i += kPT) x[i] = __ldcg(s.Vp + i + (int64_t)u * N);
        }
        grid.sync();
    }
    for (int l = tid; l < cnt; l += kPT) {
        s.nu[ocol[l]] = onu[l];
        s.cref[ocol[l]] = ocref[l];
    }
}

TallView view_of(double* B, int64_t N, int64_t n, int64_t ld, DevBuf<double>& nu, DevBuf<double>& cref,
                 DevBuf<int64_t>& colmap, DevBuf<int64_t>& pos, DevBuf<double>& part, DevBuf<double>& tq,
                 DevBuf<double>& R, int64_t ldr, DevBuf<double>& beta, DevBuf<double>& v0, DevBuf<double>& pn,
                 DevBuf<int>& flag, int64_t rpb) {
    return TallView{B, N, n, ld, nu.get(), cref.get(), colmap.get(), pos.get(), part.get(), tq.get(),
                    R.get(), ldr, beta.get(), v0.get(), pn.get(), flag.get(), rpb};
}

}  // namespace

TallQrcp::TallQrcp(double* B, int64_t N, int64_t n, int64_t ld) : B_(B), N_(N), n_(n), ld_(ld), p_(std::min(N, n)) {
    if (N <= 0 || n <= 0) argument_error("qr_col_pivot: empty matrix");
    // Rows per block: enough blocks to fill the GPU, at least 256 rows each.
    const int64_t target = (int64_t)sm_count() * 4;
    rows_per_blk_ = std::max<int64_t>(256, cdiv(N, target));
    rows_per_blk_ = cdiv(rows_per_blk_, 32) * 32;
    nblk_ = (int)cdiv(N, rows_per_blk_);
    // column-parallel steps unless the matrix is tall enough for the row blocks to fill the GPU
    col_mode_ = N <= kColRows && n >= 64;
    nu_.alloc(n); cref_.alloc(n); colmap_.alloc(n); pos_.alloc(n);
    part_.alloc((size_t)nblk_ * (n + 1)); tq_.alloc(std::max(n, p_));
    R_.alloc(p_ * n); R_.zero();
    beta_.alloc(p_); v0_.alloc(p_); pnorm_.alloc(p_); flag_.alloc(n + 1);
    TallView s = view_of(B_, N_, n_, ld_, nu_, cref_, colmap_, pos_, part_, tq_, R_, p_, beta_, v0_, pnorm_, flag_,
                         rows_per_blk_);
    if (col_mode_) {
        TTG_LAUNCH(k_col_norms, (int)cdiv(n, kT / 32), kT, 0, stream(), s);
        return;
    }
    TTG_LAUNCH(k_norm_part, nblk_, kT, 0, stream(), s, (int64_t)0);
    TTG_LAUNCH(k_norm_fin, 1, kT, 0, stream(), s, nblk_);
}

// Persistent blocked run (k_qrcp_persist); false when the shape does not suit it (fewer
// columns than CTAs, or the pivot column does not fit in shared memory).
bool TallQrcp::run_persist(int64_t steps) {
    const int G = sm_count();
    if (n_ < G || N_ > 16384) return false;
    const int64_t nloc = cdiv(n_, G);
    const size_t smem = sizeof(double) * (size_t)(N_ + nloc * kNb + 2 * nloc) + sizeof(int64_t) * 2 * (size_t)nloc;
    if (smem > 200 * 1024) return false;
    raise_smem_limit(reinterpret_cast<const void*>(k_qrcp_persist));
    int occ = 0;
    TTG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_qrcp_persist, kPT, smem));
    if (occ < 1) return false;
    if (!Vp_.get()) {
        Vp_.alloc((size_t)N_ * kNb);
        F_.alloc((size_t)n_ * kNb);
    }
    DevBuf<double> part((size_t)G * (kNb + 2));
    DevBuf<Cand> pc((size_t)2 * G);
    BlkView s{B_, N_, n_, ld_, nu_.get(), cref_.get(), colmap_.get(), pos_.get(), beta_.get(), v0_.get(),
              pnorm_.get(), Vp_.get(), F_.get()};
    PersistArgs A{s, part.get(), pc.get(), steps_, steps, (int)nloc};
    void* args[] = {&A};
    PhaseTimer pt("in-place persistent (blocked)");
    TTG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_qrcp_persist), dim3((unsigned)G), dim3(kPT),
                                         args, smem, stream()));
    count_launch();
    if (debug_sync()) check_sync("k_qrcp_persist", __FILE__, __LINE__);
    steps_ = std::max(steps_, steps);
    return true;
}

void TallQrcp::run(int64_t steps) {
    steps = std::min(steps, p_);
    // The persistent blocked engine (DMMA panel updates) measured faster than the per-step
    // kernels only on square matrices (config 4's 4096 x 4096 pass 2: 116 vs 131 ms) and
    // slower on every other config-4 shape (the per-step latency chain, not the trailing
    // traffic, bounds both). TTG_TALL_ENGINE=steps / persist forces one (A/B, tests).
    static const int engine = [] {
        const char* e = std::getenv("TTG_TALL_ENGINE");
        if (!e) return -1;
        return std::string(e) == "steps" ? 0 : 1;
    }();
    const bool persist = engine == 1 || (engine < 0 && N_ == n_ && n_ >= 2048);
    if (steps > steps_ && persist && run_persist(steps)) return;
    TallView s = view_of(B_, N_, n_, ld_, nu_, cref_, colmap_, pos_, part_, tq_, R_, p_, beta_, v0_, pnorm_, flag_,
                         rows_per_blk_);
    if (col_mode_) {
        allow_smem(k_col_apply, sizeof(double) * (size_t)N_);
        for (int64_t t = steps_; t < steps; ++t) {
            {
                PhaseTimer pt("col house");
                TTG_LAUNCH(k_col_house, 1, kHouseT, 0, stream(), s, t);
            }
            if (t + 1 >= n_) continue;
            PhaseTimer pt(N_ <= kWarpRows ? "col apply (warp)" : "col apply (cta)");
            const int64_t len = N_ - t - 1, nc = n_ - t - 1;
            if (N_ <= kWarpRows)
            {
                auto kern = len <= 16 * 32 ? k_col_apply_warp<16>
                            : len <= 32 * 32 ? k_col_apply_warp<32>
                                             : k_col_apply_warp<kWarpRows / 32>;
                TTG_LAUNCH(kern, (int)cdiv(nc, kT / 32), kT, 0, stream(), s, t);
            }
            else if (len <= 32 * 128)  // 128-thread CTAs: more columns resident per SM
                TTG_LAUNCH((k_col_apply_reg<32, 128>), (int)nc, 128, 0, stream(), s, t);
            else if (len <= 16 * kT)
                TTG_LAUNCH(k_col_apply_reg<16>, (int)nc, kT, 0, stream(), s, t);
            else if (len <= 32 * kT)
                TTG_LAUNCH(k_col_apply_reg<32>, (int)nc, kT, 0, stream(), s, t);
            else if (len <= 64 * kT)
                TTG_LAUNCH(k_col_apply_reg<64>, (int)nc, kT, 0, stream(), s, t);
            else
                TTG_LAUNCH(k_col_apply, (int)(n_ - t - 1), kT, sizeof(double) * (size_t)(N_ - t - 1), stream(), s,
                           t);
        }
        steps_ = std::max(steps_, steps);
        return;
    }
    for (int64_t t = steps_; t < steps; ++t) {
        TTG_LAUNCH(k_dots, nblk_, kT, sizeof(double) * kSub, stream(), s, t);
        TTG_LAUNCH(k_house, 1, kT, 0, stream(), s, t, nblk_);
        TTG_LAUNCH(k_apply, nblk_, kT, 0, stream(), s, t);
        TTG_LAUNCH(k_guard_part, nblk_, kT, 0, stream(), s, t);
        TTG_LAUNCH(k_guard_fin, 1, kT, 0, stream(), s, t, nblk_);
    }
    steps_ = std::max(steps_, steps);
}

namespace {
// out(t, colmap[q]) = R(t, q) = B(t, colmap[q]) for t <= q, else 0 (t < steps).
__global__ void k_r_by_column(const double* __restrict__ B, int64_t ld, int64_t n, const int64_t* __restrict__ colmap,
                              const int64_t* __restrict__ pos, int64_t steps, double* out, int64_t ldo) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= steps * n) return;
    const int64_t t = e / n, j = e - t * n;  // j = physical (original) column
    out[t * ldo + j] = pos[j] >= t ? B[t + j * ld] : 0.0;
}

// Partial sums of squares of rows >= s over the unpivoted columns (positions >= s).
__global__ void __launch_bounds__(256) k_tail_mass(const double* __restrict__ B, int64_t N, int64_t ld, int64_t n,
                                                   const int64_t* __restrict__ colmap, int64_t s, double* part) {
    __shared__ double sd[8];
    double a = 0.0;
    for (int64_t q = s + blockIdx.y; q < n; q += gridDim.y) {
        const double* c = B + colmap[q] * ld;
        for (int64_t i = s + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
            a = fma(c[i], c[i], a);
    }
    a = block_sum(a, sd);
    if (threadIdx.x == 0) part[blockIdx.y * gridDim.x + blockIdx.x] = a;
}
}  // namespace

void TallQrcp::r_rows_by_column(double* out, int64_t ldo) const {
    if (steps_ > 0)
        TTG_LAUNCH(k_r_by_column, (int)cdiv(steps_ * n_, 256), 256, 0, stream(), B_, ld_, n_, colmap_.get(), pos_.get(),
                   steps_, out, ldo);
}

double TallQrcp::trailing_mass_exact() const {
    if (steps_ >= std::min(N_, n_)) return 0.0;
    const dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(N_ - steps_, 256), 64)),
                    (unsigned)std::min<int64_t>(n_ - steps_, 64));
    DevBuf<double> part((size_t)grid.x * grid.y);
    TTG_LAUNCH(k_tail_mass, grid, 256, 0, stream(), B_, N_, ld_, n_, colmap_.get(), steps_, part.get());
    std::vector<double> h = part.to_host(part.size());
    double s = 0.0;
    for (double v : h) s += v;
    return s;
}

void TallQrcp::extract_r(double* out, int64_t ldo) const {
    TallView s{B_, N_, n_, ld_, nullptr, nullptr, colmap_.get(), nullptr, nullptr, nullptr, nullptr, 0,
               nullptr, nullptr, nullptr, nullptr, rows_per_blk_};
    if (steps_ > 0) TTG_LAUNCH(k_extract_r, (int)cdiv(steps_ * n_, 256), 256, 0, stream(), s, steps_, out, ldo);
}

void TallQrcp::form_q(double* Q, int64_t q, int64_t ldq) {
    TallView s = view_of(B_, N_, n_, ld_, nu_, cref_, colmap_, pos_, part_, tq_, R_, p_, beta_, v0_, pnorm_, flag_,
                         rows_per_blk_);
    TTG_LAUNCH(k_eye, (int)cdiv(N_ * q, 256), 256, 0, stream(), Q, N_, q, ldq);
    std::vector<double> hb = beta_.to_host(p_);
    const int64_t top = std::min(q, steps_);
    if (top >= 2 * kQBlock && q >= 2 * kQBlock) {
        const int64_t nbk = cdiv(top, kQBlock);
        DevBuf<double> V((size_t)(N_ * kQBlock)), G((size_t)(kQBlock * kQBlock)), T((size_t)(kQBlock * kQBlock)),
            W((size_t)(kQBlock * q)), W2((size_t)(kQBlock * q));
        for (int64_t bi = nbk - 1; bi >= 0; --bi) {
            const int64_t b0 = bi * kQBlock, kb = std::min<int64_t>(kQBlock, top - b0);
            const int64_t rows = N_ - b0, cols = q - b0;
            TTG_LAUNCH(k_gather_v, (int)cdiv(rows * kb, 256), 256, 0, stream(), s, b0, (int)kb, V.get());
            gemm(true, false, kb, kb, rows, V.get(), rows, V.get(), rows, G.get(), kb);
            TTG_LAUNCH(k_larft, 1, 64, 0, stream(), G.get(), beta_.get() + b0, (int)kb, T.get());
            double* Qb = Q + b0 + b0 * ldq;
            gemm(true, false, kb, cols, rows, V.get(), rows, Qb, ldq, W.get(), kb);
            gemm(false, false, kb, cols, kb, T.get(), kb, W.get(), kb, W2.get(), kb);
            gemm(false, false, rows, cols, kb, V.get(), rows, W2.get(), kb, Qb, ldq, -1.0, 1.0);
        }
        return;
    }
    for (int64_t t = top - 1; t >= 0; --t) {
        if (hb[(size_t)t] == 0.0) continue;
        if (col_mode_) {
            TTG_LAUNCH(k_q_col, (int)(q - t), kT, 0, stream(), s, t, Q, ldq);
            continue;
        }
        TTG_LAUNCH(k_q_dots, nblk_, kT, 0, stream(), s, t, Q, ldq, q);
        TTG_LAUNCH(k_q_fin, 1, kT, 0, stream(), s, t, Q, ldq, q, nblk_);
        TTG_LAUNCH(k_q_apply, nblk_, kT, 0, stream(), s, t, Q, ldq, q);
    }
}

}  // namespace ttg
