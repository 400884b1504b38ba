// Pass-1 engine: greedy column-pivoted Householder QR of a k x N matrix W (k moderate)
// without ever writing W. See engine.hpp for the contract.
//
// One pivot step t = four launches:
//   A  pick:     every CTA reduces the per-CTA pivot candidates of step t-1 (key: larger
//                norm, then lower position -- factor.cpp:85-87); CTA 0 applies the
//                position swap (factor.cpp:88-93). Then y = Q_t[:, t:]^T w_piv (warp per
//                output), i.e. the pivot column in reflected coordinates.
//   B  reflect:  dlarfg-convention reflector from y (factor.cpp:24-38, same formulas and
//                rounding), and the right update Q_{t+1} = Q_t H_t on row blocks of Q.
//                Column t of Q_{t+1} is q_t, the t-th economy-Q column.
//   C  stream:   R(t,j) = q_t^T w_j for every unpivoted column j (one HBM pass over W),
//                norm downdate nu_j -= R(t,j)^2 with the 1e-16 recompute guard
//                (factor.cpp:98-107), per-CTA pivot candidates and trailing mass.
//   D  guard:    (only when C flagged columns) recompute flagged norms from the projected
//                column, then recompute the candidates.
#include <cmath>

#include "engine.hpp"

namespace ttg {
namespace {

constexpr int kThreads = 256;

// ---- per-column streaming primitives -------------------------------------------------
// MODE 0: Row layout, one thread per column, sequential accumulation over rows.
// MODE 1: Col layout with k >= 64, one warp per column, lane-strided partials + shuffle tree.
// MODE 2: Col layout with k < 64 and ld == k, a 256-column tile staged flat through smem,
//         one thread per column, sequential accumulation.
// Within one problem every column uses the same arithmetic order, so identical columns
// produce bitwise identical results (Hilbert-type ties).

__device__ __forceinline__ double ld_w(const double* __restrict__ W, int64_t ld, int layout, int64_t i,
                                       int64_t j) {
    return layout == 0 ? W[i + j * ld] : W[i * ld + j];
}

// MODE 2 tile: columns [j0, j0+256) of a contiguous k x N (k < 64) matrix into smem as
// tile[i*(256+1) + c]; one warp per column segment (coalesced, no integer division).
__device__ __forceinline__ void load_tile_small_k(const double* __restrict__ W, int64_t k, int64_t N, int64_t j0,
                                                  double* tile) {
    // The tile is contiguous in memory (ld == k): flat coalesced loads, element e of the
    // tile is (row e % k, column e / k), tracked incrementally (no division per element).
    const int nc = (int)min((int64_t)kThreads, N - j0);
    const int kk = (int)k;
    const int total = nc * kk;
    const int dq = kThreads / kk, dr = kThreads - dq * kk;
    int c = threadIdx.x / kk, i = threadIdx.x - c * kk;
    const double* __restrict__ base = W + j0 * k;
    __syncthreads();
#pragma unroll 8
    for (int e = threadIdx.x; e < total; e += kThreads) {
        tile[i * (kThreads + 1) + c] = __ldg(base + e);
        c += dq;
        i += dr;
        if (i >= kk) {
            i -= kk;
            ++c;
        }
    }
    __syncthreads();
}

// Per-column epilogue shared by the init and stream kernels.
struct ColOut {
    Cand best;
    double mass;
};

// ---------------------------------------------------------------------------
// Init: nu_j = cref_j = |w_j|^2 (sequential, no contraction: sum_squares_serial),
// identity positions, candidates for step 0 and the initial mass.
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(kThreads) k_init(const double* __restrict__ W, int64_t k, int64_t N,
                                                   int64_t ld, double* nu, double* cref, int64_t* pos,
                                                   int64_t* perm, Cand* cand, double* mass) {
    __shared__ Cand sc[kThreads / 32];
    __shared__ double sd[kThreads / 32];
    extern __shared__ double tile[];
    Cand best = cand_none();
    double msum = 0.0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (MODE == 1) {
        const int64_t gw = (int64_t)blockIdx.x * (kThreads / 32) + warp;
        const int64_t nwarps = (int64_t)gridDim.x * (kThreads / 32);
        for (int64_t j = gw; j < N; j += nwarps) {
            const double* w = W + j * ld;
            double a = 0.0;
            for (int64_t i = lane; i < k; i += 32) a = __dadd_rn(a, __dmul_rn(w[i], w[i]));
            a = warp_sum(a);
            if (lane == 0) {
                nu[j] = a; cref[j] = a; pos[j] = j; perm[j] = j;
                Cand c{a, j, j};
                if (better(c, best)) best = c;
                msum += a;
            }
        }
    } else {
        for (int64_t j0 = (int64_t)blockIdx.x * kThreads; j0 < N; j0 += (int64_t)gridDim.x * kThreads) {
            const int64_t j = j0 + threadIdx.x;
            double a = 0.0;
            if (MODE == 2) {
                load_tile_small_k(W, k, N, j0, tile);
                if (j < N)
                    for (int64_t i = 0; i < k; ++i) {
                        const double v = tile[i * (kThreads + 1) + threadIdx.x];
                        a = __dadd_rn(a, __dmul_rn(v, v));
                    }
            } else if (j < N) {
                for (int64_t i = 0; i < k; ++i) {
                    const double v = W[i * ld + j];
                    a = __dadd_rn(a, __dmul_rn(v, v));
                }
            }
            if (j < N) {
                nu[j] = a; cref[j] = a; pos[j] = j; perm[j] = j;
                Cand c{a, j, j};
                if (better(c, best)) best = c;
                msum += a;
            }
        }
    }
    best = block_best(best, sc);
    msum = block_sum(msum, sd);
    if (threadIdx.x == 0) { cand[blockIdx.x] = best; mass[blockIdx.x] = msum; }
}

// ---------------------------------------------------------------------------
// A: pick the pivot of step t, apply the position swap, y = Q_t[:, t:]^T w_piv.
// grid.x = ceil((k - t) / 8) CTAs of 8 warps; one output per warp.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_pick(const double* __restrict__ W, int64_t k, int64_t N,
                                                   int64_t ld, int layout, int64_t t, const Cand* cand,
                                                   int ncand, int64_t* pos, int64_t* perm, int64_t* piv,
                                                   int* nflag, const double* __restrict__ Q, double* y) {
    __shared__ Cand sc[kThreads / 32];
    extern __shared__ double w[];  // k doubles
    Cand best = cand_none();
    for (int i = threadIdx.x; i < ncand; i += kThreads)
        if (better(cand[i], best)) best = cand[i];
    best = block_best(best, sc);
    // No comparable candidate (all remaining norms NaN): the reference's strict '>' scan
    // then keeps the column already at position t (factor.cpp:85-87).
    const bool none = best.col < 0;
    const int64_t jp = none ? perm[t] : best.col;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const int64_t pp = none ? t : best.pos;
        const int64_t ct = perm[t];
        perm[t] = jp;
        perm[pp] = ct;
        pos[jp] = t;
        pos[ct] = pp;
        piv[t] = jp;
        *nflag = 0;
    }
    for (int64_t i = threadIdx.x; i < k; i += kThreads) w[i] = ld_w(W, ld, layout, i, jp);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t out = t + (int64_t)blockIdx.x * (kThreads / 32) + warp;
    if (out < k) {
        const double* q = Q + out * k;
        double a = 0.0;
        for (int64_t l = lane; l < k; l += 32) a = fma(q[l], w[l], a);
        a = warp_sum(a);
        if (lane == 0) y[out] = a;
    }
}

// ---------------------------------------------------------------------------
// B: reflector of step t from y (every CTA recomputes it identically) and
// Q[:, t:] -= beta * (Q[:, t:] v) v^T on a block of 32 rows (256 threads = 32 rows x 8
// column groups). CTA 0 records R(t,t) and beta.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_reflect(int64_t k, int64_t t, const double* __restrict__ y,
                                                      double* Q, double* diag, double* betas) {
    __shared__ double sd[kThreads / 32];
    __shared__ double part[8][33];
    extern __shared__ double v[];  // k - t doubles
    const int64_t len = k - t;
    double s = 0.0;
    for (int64_t i = 1 + threadIdx.x; i < len; i += kThreads) s = fma(y[t + i], y[t + i], s);
    const double sigma = block_sum(s, sd);
    const double alpha = y[t];
    // make_householder (factor.cpp:24-38): beta = 0 for len <= 1 or sigma == 0.
    if (len <= 1 || sigma == 0.0) {
        if (blockIdx.x == 0 && threadIdx.x == 0) { diag[t] = alpha; betas[t] = 0.0; }
        return;
    }
    const double mu = __dsqrt_rn(__dadd_rn(__dmul_rn(alpha, alpha), sigma));
    const double smu = copysign(mu, alpha);
    const double v0 = __dadd_rn(alpha, smu);
    const double beta = __ddiv_rn(__dmul_rn(v0, v0), __dmul_rn(smu, v0));
    if (blockIdx.x == 0 && threadIdx.x == 0) { diag[t] = -smu; betas[t] = beta; }
    for (int64_t i = threadIdx.x; i < len; i += kThreads) v[i] = i == 0 ? 1.0 : __ddiv_rn(y[t + i], v0);
    __syncthreads();
    const int r = threadIdx.x & 31, g = threadIdx.x >> 5;
    const int64_t row = (int64_t)blockIdx.x * 32 + r;
    double u = 0.0;
    if (row < k)
        for (int64_t i = g; i < len; i += 8) u = fma(Q[row + (t + i) * k], v[i], u);
    part[g][r] = u;
    __syncthreads();
    if (g == 0) {
        double tot = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) tot += part[q][r];
        part[0][r] = tot * beta;
    }
    __syncthreads();
    const double bu = part[0][r];
    if (row < k)
        for (int64_t i = g; i < len; i += 8) {
            double* qp = Q + row + (t + i) * k;
            *qp = fma(-bu, v[i], *qp);
        }
}

// ---------------------------------------------------------------------------
// C: R(t,j) = q_t^T w_j, downdate, guard, candidates for step t+1, trailing mass.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void stream_epilogue(int64_t t, int64_t j, int64_t N, double r, double* R,
                                                double* nu, const double* cref, const int64_t* pos,
                                                int64_t* flags, int* nflag, Cand& best, double& mass) {
    R[t * N + j] = r;
    // factor.cpp:101-102: cnorm2 -= rkj*rkj; guard at 1e-16 * cref2 (no contraction).
    const double nv = __dsub_rn(nu[j], __dmul_rn(r, r));
    nu[j] = nv;
    if (nv < __dmul_rn(1e-16, cref[j]) || nv < 0.0) {
        const int slot = atomicAdd(nflag, 1);
        flags[slot] = j;
    } else {
        Cand c{nv, pos[j], j};
        if (better(c, best)) best = c;
        mass += nv;
    }
}

// MODE 3: Row layout with few columns (N too small to fill the GPU one thread per column,
// e.g. k = 640, N = 32768): a CTA owns 32 columns, its 8 warps split the k rows (each row
// read as a coalesced 256-byte segment), partials combined in warp order in smem.
__global__ void __launch_bounds__(kThreads) k_stream_splitk(const double* __restrict__ W, int64_t k, int64_t N,
                                                            int64_t ld, int64_t t, const double* __restrict__ Q,
                                                            const double* diag, const int64_t* piv, double* R,
                                                            double* nu, const double* cref, const int64_t* pos,
                                                            int64_t* flags, int* nflag, Cand* cand, double* mass) {
    __shared__ Cand sc[kThreads / 32];
    __shared__ double sd[kThreads / 32];
    __shared__ double part[kThreads / 32][33];
    extern __shared__ double q[];
    for (int64_t i = threadIdx.x; i < k; i += kThreads) q[i] = Q[i + t * k];
    __syncthreads();
    const int64_t jp = piv[t];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    Cand best = cand_none();
    double msum = 0.0;
    for (int64_t j0 = (int64_t)blockIdx.x * 32; j0 < N; j0 += (int64_t)gridDim.x * 32) {
        const int64_t j = j0 + lane;
        const bool active = j < N;
        double a = 0.0;
        if (active)
#pragma unroll 4
            for (int64_t i = warp; i < k; i += kThreads / 32) a = fma(q[i], W[i * ld + j], a);
        part[warp][lane] = a;
        __syncthreads();
        if (warp == 0) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < kThreads / 32; ++w) s += part[w][lane];
            const int64_t pj = active ? pos[j] : 0;
            const bool chosen = active && (pj < t || j == jp);
            if (chosen) R[t * N + j] = j == jp ? diag[t] : 0.0;
            bool fl = false;
            if (active && !chosen) {
                R[t * N + j] = s;
                const double nv = __dsub_rn(nu[j], __dmul_rn(s, s));
                nu[j] = nv;
                fl = nv < __dmul_rn(1e-16, cref[j]) || nv < 0.0;
                if (!fl) {
                    Cand c{nv, pj, j};
                    if (better(c, best)) best = c;
                    msum += nv;
                }
            }
            const unsigned m = __ballot_sync(0xffffffffu, fl);
            if (m) {
                const int leader = __ffs(m) - 1;
                int base = 0;
                if (lane == leader) base = atomicAdd(nflag, __popc(m));
                base = __shfl_sync(0xffffffffu, base, leader);
                if (fl) flags[base + __popc(m & ((1u << lane) - 1u))] = j;
            }
        }
        __syncthreads();
    }
    best = block_best(best, sc);
    msum = block_sum(msum, sd);
    if (threadIdx.x == 0) { cand[blockIdx.x] = best; mass[blockIdx.x] = msum; }
}

template <int MODE>
__global__ void __launch_bounds__(kThreads) k_stream(const double* __restrict__ W, int64_t k, int64_t N,
                                                     int64_t ld, int64_t t, const double* __restrict__ Q,
                                                     const double* diag, const int64_t* piv, double* R,
                                                     double* nu, const double* cref, const int64_t* pos,
                                                     int64_t* flags, int* nflag, Cand* cand, double* mass) {
    __shared__ Cand sc[kThreads / 32];
    __shared__ double sd[kThreads / 32];
    extern __shared__ double sm[];  // q (k doubles) then the MODE-2 tile
    double* q = sm;
    double* tile = sm + ((k + 1) & ~int64_t(1));
    for (int64_t i = threadIdx.x; i < k; i += kThreads) q[i] = Q[i + t * k];
    __syncthreads();
    const int64_t jp = piv[t];
    Cand best = cand_none();
    double msum = 0.0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (MODE == 1) {
        const int64_t gw = (int64_t)blockIdx.x * (kThreads / 32) + warp;
        const int64_t nwarps = (int64_t)gridDim.x * (kThreads / 32);
        for (int64_t j = gw; j < N; j += nwarps) {
            const int64_t pj = pos[j];
            if (pj < t || j == jp) {
                if (lane == 0) R[t * N + j] = j == jp ? diag[t] : 0.0;
                continue;
            }
            const double* w = W + j * ld;
            double a = 0.0;
            for (int64_t i = lane; i < k; i += 32) a = fma(q[i], w[i], a);
            a = warp_sum(a);
            if (lane == 0) stream_epilogue(t, j, N, a, R, nu, cref, pos, flags, nflag, best, msum);
        }
    } else {
        for (int64_t j0 = (int64_t)blockIdx.x * kThreads; j0 < N; j0 += (int64_t)gridDim.x * kThreads) {
            const int64_t j = j0 + threadIdx.x;
            if (MODE == 2) {
                load_tile_small_k(W, k, N, j0, tile);
            }
            // No early exits: every lane reaches the warp-aggregated flag append below.
            const bool active = j < N;
            const int64_t pj = active ? pos[j] : 0;
            const bool chosen = active && (pj < t || j == jp);
            if (chosen) R[t * N + j] = j == jp ? diag[t] : 0.0;
            const bool work = active && !chosen;
            bool fl = false;
            if (work) {
                double a = 0.0;
                if (MODE == 2) {
                    for (int64_t i = 0; i < k; ++i) a = fma(q[i], tile[i * (kThreads + 1) + threadIdx.x], a);
                } else {
#pragma unroll 8
                    for (int64_t i = 0; i < k; ++i) a = fma(q[i], W[i * ld + j], a);
                }
                R[t * N + j] = a;
                // factor.cpp:101-102: cnorm2 -= rkj*rkj; guard at 1e-16 * cref2 (no contraction).
                const double nv = __dsub_rn(nu[j], __dmul_rn(a, a));
                nu[j] = nv;
                fl = nv < __dmul_rn(1e-16, cref[j]) || nv < 0.0;
                if (!fl) {
                    Cand c{nv, pj, j};
                    if (better(c, best)) best = c;
                    msum += nv;
                }
            }
            // Hilbert-type ties flag thousands of columns per step: one atomic per warp.
            const unsigned m = __ballot_sync(0xffffffffu, fl);
            if (m) {
                const int leader = __ffs(m) - 1;
                int base = 0;
                if (lane == leader) base = atomicAdd(nflag, __popc(m));
                base = __shfl_sync(0xffffffffu, base, leader);
                if (fl) flags[base + __popc(m & ((1u << lane) - 1u))] = j;
            }
        }
    }
    best = block_best(best, sc);
    msum = block_sum(msum, sd);
    if (threadIdx.x == 0) { cand[blockIdx.x] = best; mass[blockIdx.x] = msum; }
}

// ---------------------------------------------------------------------------
// D1: guard recompute. For each flagged column j, the trailing norm after step t is
// |w_j - Q[:, :t+1] R(0:t, j)|^2 (= the sum of squares of rows t+1.. of the updated
// column, factor.cpp:103-105). One warp per flagged column.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_guard(const double* __restrict__ W, int64_t k, int64_t N,
                                                    int64_t ld, int layout, int64_t t,
                                                    const double* __restrict__ Q, const double* R,
                                                    const int64_t* flags, const int* nflag, double* nu,
                                                    double* cref) {
    const int nf = *nflag;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t f = (int64_t)blockIdx.x * (kThreads / 32) + warp; f < nf; f += (int64_t)gridDim.x * (kThreads / 32)) {
        const int64_t j = flags[f];
        double s = 0.0;
        for (int64_t i = lane; i < k; i += 32) {
            double x = ld_w(W, ld, layout, i, j);
            for (int64_t l = 0; l <= t; ++l) x = fma(-Q[i + l * k], R[l * N + j], x);
            s = fma(x, x, s);
        }
        s = warp_sum(s);
        if (lane == 0) { nu[j] = s; cref[j] = s; }
    }
}

// D1 for k <= 64: the trailing norm is |Q_{t+1}[:, t+1:]^T w_j|^2, the sum of squares of
// rows t+1.. of the reflected column -- exactly the quantity factor.cpp:103-105 sums.
// The k x (k-t-1) complement of the explicit Q sits in shared memory; one thread per
// flagged column keeps w_j in registers.
__global__ void __launch_bounds__(kThreads) k_guard_perp(const double* __restrict__ W, int64_t k, int64_t N,
                                                         int64_t ld, int layout, int64_t t,
                                                         const double* __restrict__ Q, const int64_t* flags,
                                                         const int* nflag, double* nu, double* cref) {
    __shared__ double qp[64 * 64];
    const int nf = *nflag;
    if (nf == 0) return;
    const int kk = (int)k, m = (int)(k - t - 1);
    for (int e = threadIdx.x; e < kk * m; e += kThreads) qp[e] = Q[(t + 1) * k + e];
    __syncthreads();
    for (int64_t f = (int64_t)blockIdx.x * kThreads + threadIdx.x; f < nf; f += (int64_t)gridDim.x * kThreads) {
        const int64_t j = flags[f];
        double w[64];
#pragma unroll
        for (int i = 0; i < 64; ++i) w[i] = i < kk ? ld_w(W, ld, layout, i, j) : 0.0;
        double s = 0.0;
        for (int c = 0; c < m; ++c) {
            const double* qc = qp + c * kk;
            double d = 0.0;
#pragma unroll
            for (int i = 0; i < 64; ++i)
                if (i < kk) d = fma(qc[i], w[i], d);
            s = fma(d, d, s);
        }
        nu[j] = s;
        cref[j] = s;
    }
}

// D2: candidates and trailing mass over all unpivoted columns (after a guard recompute).
__global__ void __launch_bounds__(kThreads) k_recand(int64_t N, int64_t t, const int* nflag, const double* nu,
                                                     const int64_t* pos, Cand* cand, double* mass) {
    if (*nflag == 0) return;
    __shared__ Cand sc[kThreads / 32];
    __shared__ double sd[kThreads / 32];
    Cand best = cand_none();
    double msum = 0.0;
    for (int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x; j < N; j += (int64_t)gridDim.x * kThreads) {
        const int64_t pj = pos[j];
        if (pj <= t) continue;
        Cand c{nu[j], pj, j};
        if (better(c, best)) best = c;
        msum += nu[j];
    }
    best = block_best(best, sc);
    msum = block_sum(msum, sd);
    if (threadIdx.x == 0) { cand[blockIdx.x] = best; mass[blockIdx.x] = msum; }
}

// Exact trailing norms from the residual Y = W - Q[:, :s] R(0:s, :) (already formed):
// nu_j = cref_j = |y_j|^2 for every unpivoted column, then candidates and trailing mass.
// Layout 0: Y is k x N col-major (ld k); layout 1: Y^T is N x k col-major (ld N).
__global__ void __launch_bounds__(kThreads) k_resnorm(const double* __restrict__ Y, int64_t k, int64_t N,
                                                      int layout, int64_t s, double* nu, double* cref,
                                                      const int64_t* pos, Cand* cand, double* mass) {
    __shared__ Cand sc[kThreads / 32];
    __shared__ double sd[kThreads / 32];
    Cand best = cand_none();
    double msum = 0.0;
    for (int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x; j < N; j += (int64_t)gridDim.x * kThreads) {
        const int64_t pj = pos[j];
        if (pj < s) continue;
        double a = 0.0;
        if (layout == 0)
            for (int64_t i = 0; i < k; ++i) a = fma(Y[i + j * k], Y[i + j * k], a);
        else
            for (int64_t i = 0; i < k; ++i) a = fma(Y[j + i * N], Y[j + i * N], a);
        nu[j] = a;
        cref[j] = a;
        Cand c{a, pj, j};
        if (better(c, best)) best = c;
        msum += a;
    }
    best = block_best(best, sc);
    msum = block_sum(msum, sd);
    if (threadIdx.x == 0) { cand[blockIdx.x] = best; mass[blockIdx.x] = msum; }
}

__global__ void k_identity(double* Q, int64_t k) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < k * k) Q[e] = (e % (k + 1) == 0) ? 1.0 : 0.0;
}

}  // namespace

WideQrcp::WideQrcp(const double* W, int64_t k, int64_t N, int64_t ld, Layout layout, int64_t cap_steps)
    : W_(W), k_(k), N_(N), ld_(ld), p_(std::min(k, N)), layout_(layout) {
    if (k <= 0 || N <= 0) argument_error("qr_col_pivot: empty matrix");
    if (layout == Layout::Col) mode_ = (k >= 64 || ld != k) ? 1 : 2;
    else mode_ = (k >= 64 && N < (int64_t)sm_count() * 4 * kThreads) ? 3 : 0;
    const int per_sm = 8;
    const int64_t want = mode_ == 1 ? cdiv(N, kThreads / 32) : mode_ == 3 ? cdiv(N, 32) : cdiv(N, kThreads);
    ncand_ = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count() * per_sm));
    nu_.alloc(N); cref_.alloc(N); pos_.alloc(N); perm_.alloc(N); flags_.alloc(N);
    cand_.alloc(ncand_); mass_.alloc(ncand_); nflag_.alloc(1); nflag_.zero();
    Q_.alloc(k * k); y_.alloc(k);
    diag_.alloc(p_); beta_.alloc(p_); piv_.alloc(p_);
    grow(std::max<int64_t>(1, std::min(p_, cap_steps)));
    TTG_LAUNCH(k_identity, cdiv(k * k, 256), 256, 0, stream(), Q_.get(), k);
    const size_t smem = mode_ == 2 ? sizeof(double) * k * (kThreads + 1) : 0;
    auto init = (mode_ == 0 || mode_ == 3) ? k_init<0> : mode_ == 1 ? k_init<1> : k_init<2>;
    allow_smem(init, smem);
    TTG_LAUNCH(init, ncand_, kThreads, smem, stream(), W_, k_, N_, ld_, nu_.get(), cref_.get(), pos_.get(),
               perm_.get(), cand_.get(), mass_.get());
}

void WideQrcp::grow(int64_t cap) {
    if (cap <= cap_) return;
    DevBuf<double> nr(cap * N_);
    if (steps_ > 0)
        TTG_CUDA(cudaMemcpyAsync(nr.get(), R_.get(), sizeof(double) * steps_ * N_, cudaMemcpyDeviceToDevice,
                                 stream()));
    R_ = std::move(nr);
    cap_ = cap;
}

double WideQrcp::trailing_mass() {
    std::vector<double> h = mass_.to_host(ncand_);
    double s = 0.0;
    for (double v : h) s += v;
    return s;
}

double WideQrcp::refresh_exact() {
    const int64_t s = steps_;
    if (s == 0) return trailing_mass();
    DevBuf<double> Y((size_t)(k_ * N_));
    if (layout_ == Layout::Col) {
        TTG_CUDA(cudaMemcpy2DAsync(Y.get(), sizeof(double) * k_, W_, sizeof(double) * ld_, sizeof(double) * k_, N_,
                                   cudaMemcpyDeviceToDevice, stream()));
        // Y (k x N) -= Q[:, :s] * C with C(t, j) = R[t*N + j], i.e. C = (N x s col-major)^T
        gemm(false, true, k_, N_, s, Q_.get(), k_, R_.get(), N_, Y.get(), k_, -1.0, 1.0);
    } else {
        TTG_CUDA(cudaMemcpy2DAsync(Y.get(), sizeof(double) * N_, W_, sizeof(double) * ld_, sizeof(double) * N_, k_,
                                   cudaMemcpyDeviceToDevice, stream()));
        // Y^T (N x k) -= C^T (N x s) * Q[:, :s]^T
        gemm(false, true, N_, k_, s, R_.get(), N_, Q_.get(), k_, Y.get(), N_, -1.0, 1.0);
    }
    TTG_LAUNCH(k_resnorm, ncand_, kThreads, 0, stream(), Y.get(), k_, N_, (int)layout_, s, nu_.get(), cref_.get(),
               pos_.get(), cand_.get(), mass_.get());
    return trailing_mass();
}

void WideQrcp::run_to(int64_t steps) {
    steps = std::min(steps, p_);
    if (steps > cap_) grow(std::min(p_, std::max(steps, 2 * cap_)));
    while (steps_ < steps) step();
}

void WideQrcp::step() {
    const int64_t t = steps_;
    const int64_t nout = k_ - t;
    allow_smem(k_pick, sizeof(double) * k_);
    allow_smem(k_reflect, sizeof(double) * nout);
    TTG_LAUNCH(k_pick, (int)cdiv(nout, kThreads / 32), kThreads, sizeof(double) * k_, stream(), W_, k_, N_,
               ld_, (int)layout_, t, cand_.get(), ncand_, pos_.get(), perm_.get(), piv_.get(), nflag_.get(),
               Q_.get(), y_.get());
    TTG_LAUNCH(k_reflect, (int)cdiv(k_, 32), kThreads, sizeof(double) * nout, stream(), k_, t, y_.get(),
               Q_.get(), diag_.get(), beta_.get());
    gemv_step(t);
    steps_ = t + 1;
}

void WideQrcp::gemv_step(int64_t t) {
    const size_t qbytes = sizeof(double) * ((k_ + 1) & ~int64_t(1));
    const size_t smem = qbytes + (mode_ == 2 ? sizeof(double) * k_ * (kThreads + 1) : 0);
    auto kern = mode_ == 0 ? k_stream<0> : mode_ == 1 ? k_stream<1> : mode_ == 2 ? k_stream<2> : k_stream_splitk;
    allow_smem(kern, smem);
    prof_begin();
    TTG_LAUNCH(kern, ncand_, kThreads, smem, stream(), W_, k_, N_, ld_, t, Q_.get(), diag_.get(), piv_.get(),
               R_.get(), nu_.get(), cref_.get(), pos_.get(), flags_.get(), nflag_.get(), cand_.get(), mass_.get());
    // Algorithmic bytes: the unpivoted columns of W read once, their norms read and
    // written once, and row t of R written.
    prof_end(8.0 * (double)(N_ - t) * (double)(k_ + 2) + 8.0 * (double)N_);
    if (k_ <= 64)
        TTG_LAUNCH(k_guard_perp, std::max(1, sm_count() * 2), kThreads, 0, stream(), W_, k_, N_, ld_, (int)layout_,
                   t, Q_.get(), flags_.get(), nflag_.get(), nu_.get(), cref_.get());
    else
        TTG_LAUNCH(k_guard, std::max(1, sm_count() * 2), kThreads, 0, stream(), W_, k_, N_, ld_, (int)layout_, t,
                   Q_.get(), R_.get(), flags_.get(), nflag_.get(), nu_.get(), cref_.get());
    TTG_LAUNCH(k_recand, ncand_, kThreads, 0, stream(), N_, t, nflag_.get(), nu_.get(), pos_.get(),
               cand_.get(), mass_.get());
}

}  // namespace ttg
