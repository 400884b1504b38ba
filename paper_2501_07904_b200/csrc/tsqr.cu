// Pass 2 without BLAS-2 traffic, and a one-CTA pivoted QR for small matrices.
//
// The pass-2 decisions (pivot order P2, |R2|, pivot norms, kept masses) depend on
// B = R1[:s,:]^T only through B^T B: QRCP(B) and QRCP(R_B) with B = Q_B R_B pick the
// same pivots and produce the same R up to row signs in exact arithmetic (column norms
// and their projections are invariant under Q_B^T). R_B comes from a Householder TSQR:
// every CTA factors a row block of B in shared memory, and the stacked triangles are
// factored again until one s x s triangle remains -- one HBM pass over B instead of the
// 2s passes of the in-place algorithm. B is read straight out of R1's row storage (the
// row order of B only changes rounding), so the gather is not needed either.
//
// k_small_qrcp is the reference's qr_col_pivot (factor.cpp:62-135) for a matrix that
// fits in shared memory: physical column swaps, dlarfg reflectors, sequential norms,
// the 1e-16 recompute guard -- one launch for the whole factorisation.
#include <cmath>

#include "engine.hpp"

namespace ttg {
namespace {

constexpr int kT = 256;

// Householder QR (no pivoting) of the rows x s block X (col-major, ld = rows) held in
// shared memory; leaves R in the upper triangle. Deterministic fixed-shape reductions.
__device__ void smem_householder(double* X, int rows, int s, int64_t ld, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int p = min(rows, s);
    for (int c = 0; c < p; ++c) {
        double* x = X + c * ld;
        double part = 0.0;
        for (int i = c + 1 + threadIdx.x; i < rows; i += blockDim.x) part = fma(x[i], x[i], part);
        const double sigma = block_sum(part, red);
        const double alpha = x[c];
        if (rows - c <= 1 || sigma == 0.0) {
            __syncthreads();
            continue;
        }
        const double mu = sqrt(fma(alpha, alpha, sigma));
        const double smu = copysign(mu, alpha);
        const double v0 = alpha + smu;
        const double beta = v0 / smu;
        __syncthreads();
        for (int i = c + 1 + threadIdx.x; i < rows; i += blockDim.x) x[i] /= v0;
        if (threadIdx.x == 0) x[c] = -smu;
        __syncthreads();
        for (int j = c + 1 + warp; j < s; j += nw) {
            double* y = X + j * ld;
            double t = 0.0;
            for (int i = c + 1 + lane; i < rows; i += 32) t = fma(x[i], y[i], t);
            t = warp_sum(t);
            t = beta * (y[c] + t);
            for (int i = c + 1 + lane; i < rows; i += 32) y[i] = fma(-t, x[i], y[i]);
            if (lane == 0) y[c] -= t;
        }
        __syncthreads();
    }
}

// Level 0: block b of B (rows [b*rb, min(N, (b+1)*rb)), all s columns; column t of B is
// at B + t*ld) -> its s x s triangle written at out + b*s (col-major, ld = ldo).
__global__ void __launch_bounds__(kT) k_tsqr_leaf(const double* __restrict__ B, int64_t N, int s, int64_t ld,
                                                  int rb, double* out, int64_t ldo) {
    extern __shared__ double X[];
    __shared__ double red[kT / 32];
    const int64_t r0 = (int64_t)blockIdx.x * rb;
    const int rows = (int)min((int64_t)rb, N - r0);
    for (int c = 0; c < s; ++c)
        for (int i = threadIdx.x; i < rows; i += kT) X[c * rows + i] = B[r0 + i + c * ld];
    __syncthreads();
    smem_householder(X, rows, s, rows, red);
    // upper triangle (rows < s padded with zeros)
    for (int e = threadIdx.x; e < s * s; e += kT) {
        const int c = e / s, i = e - c * s;
        out[(int64_t)blockIdx.x * s + i + c * ldo] = (i <= c && i < rows) ? X[c * rows + i] : 0.0;
    }
}

// Register-resident Householder QR of a ROWS x s block (s <= S <= 32) for the TSQR tree:
// thread `tid` holds rows i*256 + tid (i < RPT) of all S columns in registers, so a
// reflector step is two block reductions (the column mass, then the S column dots in one
// warp reduce-scatter) and a register update -- no shared-memory traffic over the data.
// Column c's reflector has v = 1 at row c (thread c, slot 0) and x/v0 below, the
// formulas of smem_householder. Columns padded past s are zero and stay zero.
template <int S, int RPT>
__global__ void __launch_bounds__(kT, 1) k_tsqr_reg(const double* __restrict__ B, int64_t N, int s, int64_t ld,
                                                    double* __restrict__ out, int64_t ldo) {
    constexpr int ROWS = kT * RPT, NW = kT / 32;
    __shared__ double part[NW][S];
    __shared__ double tau[S];
    __shared__ double red[NW];
    __shared__ double bc;
    __shared__ double Rs[S * S];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t r0 = (int64_t)blockIdx.x * ROWS;
    const int rows = (int)min((int64_t)ROWS, N - r0);
    double x[RPT][S];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const int row = i * kT + tid;
#pragma unroll
        for (int j = 0; j < S; ++j) x[i][j] = (row < rows && j < s) ? B[r0 + row + (int64_t)j * ld] : 0.0;
    }
    const int p = min(rows, s);
    double* orow = out + (int64_t)blockIdx.x * s;
    // Step c works on register column 0: after every step the columns shift left by one,
    // so all register indices are static and the loop stays rolled (small code).
#pragma unroll 1
    for (int c = 0; c < p; ++c) {
        // column mass below row c, and alpha = x(c, c)
        double sg = 0.0;
#pragma unroll
        for (int i = 0; i < RPT; ++i)
            if (i * kT + tid > c) sg = fma(x[i][0], x[i][0], sg);
        sg = warp_sum(sg);
        if (lane == 0) red[warp] = sg;
        if (tid == c) bc = x[0][0];
        __syncthreads();
        double sigma = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) sigma += red[w];
        const double alpha = bc;
        if (rows - c > 1 && sigma != 0.0) {
            const double mu = sqrt(fma(alpha, alpha, sigma));
            const double smu = copysign(mu, alpha);
            const double v0 = alpha + smu;
            const double beta = v0 / smu;
            double v[RPT];
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const int row = i * kT + tid;
                v[i] = row > c ? x[i][0] / v0 : (row == c ? 1.0 : 0.0);
            }
            // d_j = sum_rows v_i x_ij (register column j = matrix column c + j), reduce-
            // scattered so lane j holds the warp sum of column j
            // first reduce-scatter level fused with the dots, so only S/2 partials live
            constexpr int H = S / 2;
            double d[H];
            {
                const bool up = (lane & H) != 0;
#pragma unroll
                for (int j = 0; j < H; ++j) {
                    double lo = 0.0, hi = 0.0;
#pragma unroll
                    for (int i = 0; i < RPT; ++i) {
                        if (j > 0) lo = fma(v[i], x[i][j], lo);
                        hi = fma(v[i], x[i][j + H], hi);
                    }
                    if (S < 32) {
#pragma unroll
                        for (int off = 16; off >= S; off >>= 1) {
                            lo += __shfl_xor_sync(0xffffffffu, lo, off);
                            hi += __shfl_xor_sync(0xffffffffu, hi, off);
                        }
                    }
                    const double send = up ? lo : hi;
                    const double keep = up ? hi : lo;
                    d[j] = keep + __shfl_xor_sync(0xffffffffu, send, H);
                }
            }
#pragma unroll
            for (int h = H / 2; h >= 1; h >>= 1) {
                const bool up = (lane & h) != 0;
#pragma unroll
                for (int j = 0; j < h; ++j) {
                    const double send = up ? d[j] : d[j + h];
                    const double keep = up ? d[j + h] : d[j];
                    d[j] = keep + __shfl_xor_sync(0xffffffffu, send, h);
                }
            }
            if (lane < S) part[warp][lane] = d[0];
            __syncthreads();
            if (tid < S) {
                double w = 0.0;
#pragma unroll
                for (int q = 0; q < NW; ++q) w += part[q][tid];
                tau[tid] = beta * w;
            }
            __syncthreads();
#pragma unroll
            for (int j = 1; j < S; ++j) {
                const double tj = tau[j];
#pragma unroll
                for (int i = 0; i < RPT; ++i) x[i][j] = fma(-tj, v[i], x[i][j]);
            }
            if (tid == c) x[0][0] = -smu;
        } else {
            __syncthreads();
        }
        // row c of R is final: thread c parks it in shared memory
        if (tid == c) {
#pragma unroll
            for (int j = 0; j < S; ++j)
                if (c + j < S) Rs[(c + j) * S + c] = x[0][j];
        }
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
#pragma unroll
            for (int j = 0; j + 1 < S; ++j) x[i][j] = x[i][j + 1];
            x[i][S - 1] = 0.0;
        }
    }
    __syncthreads();
    // upper triangle out (rows >= p, i.e. blocks with fewer than s rows, are zero)
    for (int e = tid; e < s * s; e += kT) {
        const int j = e / s, i = e - j * s;
        orow[i + (int64_t)j * ldo] = (i <= j && i < p) ? Rs[j * S + i] : 0.0;
    }
}

// Leaf variant of k_tsqr_reg with the column loop fully unrolled (static register
// columns, no shifting, dead columns skipped at compile time). Its code is large, which
// costs instruction fetch on a lone CTA but pays off when every SM runs the same blocks
// (the leaf level); the rolled kernel serves the small upper levels.
template <int S, int RPT>
__global__ void __launch_bounds__(kT, 1) k_tsqr_unr(const double* __restrict__ B, int64_t N, int s, int64_t ld,
                                                    double* __restrict__ out, int64_t ldo) {
    // A CTA streams its share of the rows through the register block: the first chunk
    // fills all ROWS rows, every later chunk keeps the running triangle in rows 0..S-1
    // (threads 0..S-1, slot 0) and refills the other ROWS - S rows, so one triangle per
    // CTA (one per SM) leaves the leaf level instead of one per ROWS rows.
    constexpr int ROWS = kT * RPT, NW = kT / 32;
    __shared__ double part[NW][S];
    __shared__ double tau[S];
    __shared__ double red[NW];
    __shared__ double bc;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t per = (N + gridDim.x - 1) / gridDim.x;
    const int64_t g0 = (int64_t)blockIdx.x * per, g1 = min(N, g0 + per);
    double x[RPT][S];
    int p = 0;  // rows of the running triangle held in rows 0..p-1 of the block
    for (int64_t base = g0; base < g1 || (base == g0 && g0 >= g1);) {
        const int keep = p;  // rows 0..keep-1 hold R from the previous chunk
        const int64_t avail = max((int64_t)0, g1 - base);
        const int fresh = (int)min((int64_t)(ROWS - keep), avail);
        const int rows = keep + fresh;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int row = i * kT + tid;
            if (row < keep) {  // R row: zero below its diagonal
#pragma unroll
                for (int j = 0; j < S; ++j)
                    if (j < row) x[i][j] = 0.0;
            } else {
                const bool in = row < rows;
                const int64_t gr = base + (row - keep);
#pragma unroll
                for (int j = 0; j < S; ++j) x[i][j] = (in && j < s) ? B[gr + (int64_t)j * ld] : 0.0;
            }
        }
        base += fresh;
        p = min(rows, s);
#pragma unroll
        for (int c = 0; c < S; ++c) {
            if (c >= p) break;
            double sg = 0.0;
#pragma unroll
            for (int i = 0; i < RPT; ++i)
                if (i * kT + tid > c && i * kT + tid < rows) sg = fma(x[i][c], x[i][c], sg);
            sg = warp_sum(sg);
            if (lane == 0) red[warp] = sg;
            if (tid == c) bc = x[0][c];
            __syncthreads();
            double sigma = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) sigma += red[w];
            const double alpha = bc;
            if (rows - c <= 1 || sigma == 0.0) {
                __syncthreads();
                continue;
            }
            const double mu = sqrt(fma(alpha, alpha, sigma));
            const double smu = copysign(mu, alpha);
            const double v0 = alpha + smu;
            const double beta = v0 / smu;
            double v[RPT];
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const int row = i * kT + tid;
                v[i] = (row > c && row < rows) ? x[i][c] / v0 : (row == c ? 1.0 : 0.0);
            }
            double d[S];
#pragma unroll
            for (int j = 0; j < S; ++j) {
                double t = 0.0;
                if (j > c) {
#pragma unroll
                    for (int i = 0; i < RPT; ++i) t = fma(v[i], x[i][j], t);
                }
                d[j] = t;
            }
            if (S < 32) {
#pragma unroll
                for (int off = 16; off >= S; off >>= 1)
#pragma unroll
                    for (int j = 0; j < S; ++j) d[j] += __shfl_xor_sync(0xffffffffu, d[j], off);
            }
#pragma unroll
            for (int h = S / 2; h >= 1; h >>= 1) {
                const bool up = (lane & h) != 0;
#pragma unroll
                for (int j = 0; j < h; ++j) {
                    const double send = up ? d[j] : d[j + h];
                    const double keep2 = up ? d[j + h] : d[j];
                    d[j] = keep2 + __shfl_xor_sync(0xffffffffu, send, h);
                }
            }
            if (lane < S) part[warp][lane] = d[0];
            __syncthreads();
            if (tid < S) {
                double w = 0.0;
#pragma unroll
                for (int q = 0; q < NW; ++q) w += part[q][tid];
                tau[tid] = beta * w;
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < S; ++j) {
                if (j > c) {
                    const double tj = tau[j];
#pragma unroll
                    for (int i = 0; i < RPT; ++i) x[i][j] = fma(-tj, v[i], x[i][j]);
                }
            }
            if (tid == c) x[0][c] = -smu;
        }
        if (g0 >= g1) break;
    }
    if (tid < s) {
#pragma unroll
        for (int j = 0; j < S; ++j)
            if (j < s) out[(int64_t)blockIdx.x * s + tid + (int64_t)j * ldo] = (j >= tid && tid < p) ? x[0][j] : 0.0;
    }
}

// Levels >= 1: stack g consecutive s x s triangles (rows [b*g*s, ...)) and factor. When
// the stack does not fit in shared memory it is factored in place in the (scratch) input.
__global__ void __launch_bounds__(kT) k_tsqr_node(double* in, int64_t nrows, int s, int64_t ldi, int g,
                                                  int in_smem, double* out, int64_t ldo) {
    extern __shared__ double X[];
    __shared__ double red[kT / 32];
    const int64_t r0 = (int64_t)blockIdx.x * g * s;
    const int rows = (int)min((int64_t)g * s, nrows - r0);
    double* base;
    int64_t ld;
    if (in_smem) {
        for (int c = 0; c < s; ++c)
            for (int i = threadIdx.x; i < rows; i += kT) X[c * rows + i] = in[r0 + i + c * ldi];
        __syncthreads();
        base = X;
        ld = rows;
    } else {
        base = in + r0;
        ld = ldi;
    }
    smem_householder(base, rows, s, ld, red);
    __syncthreads();
    for (int e = threadIdx.x; e < s * s; e += kT) {
        const int c = e / s, i = e - c * s;
        out[(int64_t)blockIdx.x * s + i + c * ldo] = (i <= c && i < rows) ? base[c * ld + i] : 0.0;
    }
}

// Pairwise tree node for larger s: QR of two stacked upper triangles [T1; T2] with the
// structure kept. Step c reflects T1(c,c) against T2(0..c, c) only, and touches rows c of
// T1 and 0..c of T2 in the columns to the right, so T2 stays upper triangular and both
// live packed in shared memory (s(s+1) doubles; s = 160 -> 206 KB) with about a sixth of
// the flops of a dense 2s x s factorisation.
__global__ void __launch_bounds__(kT) k_tsqr_pair(const double* __restrict__ in, int64_t nrows, int s, int64_t ldi,
                                                  double* out, int64_t ldo) {
    extern __shared__ double sm[];
    const int tri = s * (s + 1) / 2;
    double* T1 = sm;
    double* T2 = sm + tri;
    __shared__ double red[kT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kT / 32;
    const int64_t r1 = (int64_t)blockIdx.x * 2 * s, r2 = r1 + s;
    const bool has2 = r2 < nrows;
    for (int e = threadIdx.x; e < tri; e += kT) {
        int c = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);  // column of packed index e
        while ((c + 1) * (c + 2) / 2 <= e) ++c;
        while (c * (c + 1) / 2 > e) --c;
        const int i = e - c * (c + 1) / 2;
        T1[e] = in[r1 + i + (int64_t)c * ldi];
        T2[e] = has2 ? in[r2 + i + (int64_t)c * ldi] : 0.0;
    }
    __syncthreads();
    if (has2)
        for (int c = 0; c < s; ++c) {
            double* x2 = T2 + c * (c + 1) / 2;  // T2(0..c, c)
            double part = 0.0;
            for (int i = threadIdx.x; i <= c; i += kT) part = fma(x2[i], x2[i], part);
            const double sigma = block_sum(part, red);
            double* d1 = T1 + c * (c + 1) / 2 + c;  // T1(c, c)
            const double alpha = *d1;
            if (sigma == 0.0) {
                __syncthreads();
                continue;
            }
            const double mu = sqrt(fma(alpha, alpha, sigma));
            const double smu = copysign(mu, alpha);
            const double v0 = alpha + smu;
            const double beta = v0 / smu;
            __syncthreads();
            for (int i = threadIdx.x; i <= c; i += kT) x2[i] /= v0;
            if (threadIdx.x == 0) *d1 = -smu;
            __syncthreads();
            for (int j = c + 1 + warp; j < s; j += nw) {
                double* y1 = T1 + j * (j + 1) / 2 + c;  // T1(c, j)
                double* y2 = T2 + j * (j + 1) / 2;      // T2(0..c, j)
                double w = 0.0;
                for (int i = lane; i <= c; i += 32) w = fma(x2[i], y2[i], w);
                w = warp_sum(w) + *y1;
                const double tau = beta * w;
                for (int i = lane; i <= c; i += 32) y2[i] = fma(-tau, x2[i], y2[i]);
                if (lane == 0) *y1 -= tau;
            }
            __syncthreads();
        }
    for (int e = threadIdx.x; e < s * s; e += kT) {
        const int c = e / s, i = e - c * s;
        out[(int64_t)blockIdx.x * s + i + (int64_t)c * ldo] = i <= c ? T1[c * (c + 1) / 2 + i] : 0.0;
    }
}

// ---------------------------------------------------------------------------
// One-CTA qr_col_pivot of an m x n matrix (col-major, ld = m) held in smem.
// Outputs: perm[n] (position -> source column), R over positions (p x n, ld = p),
// pnorm[p] (norm^2 of the pivot when chosen), optional Q (m x p, ld = m) formed by
// backward accumulation (factor.cpp:116-133).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(512) k_small_qrcp(const double* __restrict__ A, int m, int n, int64_t lda,
                                                    int64_t* perm_out, double* R, double* pnorm, double* Q,
                                                    int want_q) {
    extern __shared__ double sm[];
    double* X = sm;                       // m x n
    double* nu = X + (size_t)m * n;       // n
    double* cref = nu + n;                // n
    double* beta = cref + n;              // p
    double* tq = beta + min(m, n);        // n
    int* perm = (int*)(tq + n);           // n
    __shared__ double red[16];
    __shared__ int spiv;
    const int p = min(m, n);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int c = 0; c < n; ++c)
        for (int i = threadIdx.x; i < m; i += blockDim.x) X[c * m + i] = A[i + c * lda];
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        double a = 0.0;
        for (int i = 0; i < m; ++i) a = __dadd_rn(a, __dmul_rn(X[j * m + i], X[j * m + i]));
        nu[j] = a;
        cref[j] = a;
        perm[j] = j;
    }
    __syncthreads();
    for (int k = 0; k < p; ++k) {
        if (threadIdx.x == 0) {  // strict '>' scan from position k (factor.cpp:85-87)
            int piv = k;
            for (int j = k + 1; j < n; ++j)
                if (nu[j] > nu[piv]) piv = j;
            spiv = piv;
            pnorm[k] = nu[piv];
        }
        __syncthreads();
        const int piv = spiv;
        if (piv != k) {
            for (int i = threadIdx.x; i < m; i += blockDim.x) {
                const double t = X[k * m + i];
                X[k * m + i] = X[piv * m + i];
                X[piv * m + i] = t;
            }
            if (threadIdx.x == 0) {
                int ti = perm[k]; perm[k] = perm[piv]; perm[piv] = ti;
                double td = nu[k]; nu[k] = nu[piv]; nu[piv] = td;
                td = cref[k]; cref[k] = cref[piv]; cref[piv] = td;
            }
        }
        __syncthreads();
        // make_householder (factor.cpp:24-38)
        double* x = X + k * m;
        double part = 0.0;
        for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) part = fma(x[i], x[i], part);
        const double sigma = block_sum(part, red);
        const double alpha = x[k];
        double b = 0.0;
        if (m - k > 1 && sigma != 0.0) {
            const double mu = __dsqrt_rn(__dadd_rn(__dmul_rn(alpha, alpha), sigma));
            const double smu = copysign(mu, alpha);
            const double v0 = __dadd_rn(alpha, smu);
            b = __ddiv_rn(__dmul_rn(v0, v0), __dmul_rn(smu, v0));
            __syncthreads();
            for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) x[i] = __ddiv_rn(x[i], v0);
            if (threadIdx.x == 0) x[k] = -smu;
        }
        if (threadIdx.x == 0) beta[k] = b;
        __syncthreads();
        // apply_reflector to columns k+1..n-1 (factor.cpp:43-58)
        if (b != 0.0)
            for (int j = k + 1 + warp; j < n; j += nw) {
                double* y = X + j * m;
                double t = 0.0;
                for (int i = k + 1 + lane; i < m; i += 32) t = fma(x[i], y[i], t);
                t = warp_sum(t);
                t = __dmul_rn(__dadd_rn(y[k], t), b);
                for (int i = k + 1 + lane; i < m; i += 32) y[i] = __dsub_rn(y[i], __dmul_rn(t, x[i]));
                if (lane == 0) y[k] = __dsub_rn(y[k], t);
            }
        __syncthreads();
        // downdate + guard (factor.cpp:98-107), one warp per column
        for (int j = k + 1 + warp; j < n; j += nw) {
            double nv = 0.0;
            if (lane == 0) {
                const double rkj = X[j * m + k];
                nv = __dsub_rn(nu[j], __dmul_rn(rkj, rkj));
            }
            nv = __shfl_sync(0xffffffffu, nv, 0);
            if (nv < __dmul_rn(1e-16, cref[j]) || nv < 0.0) {
                double a = 0.0;
                for (int i = k + 1 + lane; i < m; i += 32) a = fma(X[j * m + i], X[j * m + i], a);
                a = warp_sum(a);
                nv = a;
                if (lane == 0) cref[j] = a;
            }
            if (lane == 0) nu[j] = nv;
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < p * n; e += blockDim.x) {
        const int c = e / p, i = e - c * p;
        R[i + (int64_t)c * p] = i <= c ? X[c * m + i] : 0.0;
    }
    for (int j = threadIdx.x; j < n; j += blockDim.x) perm_out[j] = perm[j];
    if (!want_q) return;
    // economy Q, backward accumulation; Q lives in global memory (m x p)
    for (int e = threadIdx.x; e < m * p; e += blockDim.x) {
        const int c = e / m, i = e - c * m;
        Q[i + (int64_t)c * m] = i == c ? 1.0 : 0.0;
    }
    __syncthreads();
    for (int k = p - 1; k >= 0; --k) {
        const double bk = beta[k];
        if (bk == 0.0) continue;
        const double* v = X + k * m;
        for (int j = k + warp; j < p; j += nw) {
            double* c = Q + (int64_t)j * m;
            double t = 0.0;
            for (int i = k + 1 + lane; i < m; i += 32) t = fma(v[i], c[i], t);
            t = warp_sum(t);
            t = __dmul_rn(__dadd_rn(c[k], t), bk);
            for (int i = k + 1 + lane; i < m; i += 32) c[i] = __dsub_rn(c[i], __dmul_rn(t, v[i]));
            if (lane == 0) c[k] = __dsub_rn(c[k], t);
        }
        __syncthreads();
    }
    (void)tq;
}

// k_small_qrcp for n <= 32 columns with one warp per column (1024 threads): the pivot is
// chosen by warp 0 (the strict '>' scan from position k as a warp argmax: first maximal
// position, a NaN at position k keeps k), the reflector by the warp owning column k, and
// each warp applies it to its own column and downdates that column's norm in the same
// pass -- three barriers per step instead of five, no idle threads. Per-column arithmetic
// is k_small_qrcp's (lanes over rows, warp tree), so R and the pivots are bitwise equal.
__global__ void __launch_bounds__(1024) k_small_qrcp32(const double* __restrict__ A, int m, int n, int64_t lda,
                                                      int64_t* perm_out, double* R, double* pnorm, double* Q,
                                                      int want_q) {
    extern __shared__ double sm[];
    double* X = sm;                  // m x n
    double* beta = X + (size_t)m * n; // p
    __shared__ double nu[32], cref[32];
    __shared__ int perm[32];
    __shared__ int spiv;
    __shared__ double sh[3];  // v0, beta, -smu of the step
    const int p = min(m, n);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int c = warp; c < n; c += 32)
        for (int i = lane; i < m; i += 32) X[c * m + i] = A[i + c * lda];
    __syncthreads();
    if (warp < n && lane == 0) {
        double a = 0.0;
        for (int i = 0; i < m; ++i) a = __dadd_rn(a, __dmul_rn(X[warp * m + i], X[warp * m + i]));
        nu[warp] = a;
        cref[warp] = a;
        perm[warp] = warp;
    }
    __syncthreads();
    for (int k = 0; k < p; ++k) {
        if (warp == 0) {  // strict '>' scan from position k (factor.cpp:85-87)
            const bool nan_k = isnan(nu[k]);
            double v = (lane >= k && lane < n && !isnan(nu[lane])) ? nu[lane] : -INFINITY;
            int idx = (lane >= k && lane < n) ? lane : 1 << 30;
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, v, o);
                const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
                if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
            }
            if (lane == 0) {
                // the scan keeps k unless a later value is strictly greater; -inf (all NaN) keeps k
                int piv = idx;
                if (nan_k || !(v > -INFINITY) || !(nu[piv] > nu[k])) piv = k;
                spiv = piv;
                pnorm[k] = nu[piv];
            }
        }
        __syncthreads();
        const int piv = spiv;
        if (piv != k) {  // swap columns k and piv (warp k does the data, lane 0 of warp 0 the state)
            if (warp == 0)
                for (int i = lane; i < m; i += 32) {
                    const double t = X[k * m + i];
                    X[k * m + i] = X[piv * m + i];
                    X[piv * m + i] = t;
                }
            if (threadIdx.x == 0) {
                int ti = perm[k]; perm[k] = perm[piv]; perm[piv] = ti;
                double td = nu[k]; nu[k] = nu[piv]; nu[piv] = td;
                td = cref[k]; cref[k] = cref[piv]; cref[piv] = td;
            }
            __syncthreads();
        }
        // make_householder (factor.cpp:24-38) by warp 0
        double* x = X + k * m;
        if (warp == 0) {
            double part = 0.0;
            for (int i = k + 1 + lane; i < m; i += 32) part = fma(x[i], x[i], part);
            const double sigma = warp_sum(part);
            const double alpha = x[k];
            double b = 0.0, v0 = 1.0, smu = 0.0;
            if (m - k > 1 && sigma != 0.0) {
                const double mu = __dsqrt_rn(__dadd_rn(__dmul_rn(alpha, alpha), sigma));
                smu = copysign(mu, alpha);
                v0 = __dadd_rn(alpha, smu);
                b = __ddiv_rn(__dmul_rn(v0, v0), __dmul_rn(smu, v0));
                for (int i = k + 1 + lane; i < m; i += 32) x[i] = __ddiv_rn(x[i], v0);
                __syncwarp();
                if (lane == 0) x[k] = -smu;
            }
            if (lane == 0) beta[k] = b;
        }
        __syncthreads();
        const double b = beta[k];
        // apply_reflector to column j = warp (factor.cpp:43-58), then its downdate + guard
        const int j = warp;
        if (j > k && j < n) {
            double* y = X + j * m;
            if (b != 0.0) {
                double t = 0.0;
                for (int i = k + 1 + lane; i < m; i += 32) t = fma(x[i], y[i], t);
                t = warp_sum(t);
                t = __dmul_rn(__dadd_rn(y[k], t), b);
                for (int i = k + 1 + lane; i < m; i += 32) y[i] = __dsub_rn(y[i], __dmul_rn(t, x[i]));
                __syncwarp();
                if (lane == 0) y[k] = __dsub_rn(y[k], t);
                __syncwarp();
            }
            double nv = 0.0;
            if (lane == 0) {
                const double rkj = y[k];
                nv = __dsub_rn(nu[j], __dmul_rn(rkj, rkj));
            }
            nv = __shfl_sync(0xffffffffu, nv, 0);
            if (nv < __dmul_rn(1e-16, cref[j]) || nv < 0.0) {
                double a = 0.0;
                for (int i = k + 1 + lane; i < m; i += 32) a = fma(y[i], y[i], a);
                a = warp_sum(a);
                nv = a;
                if (lane == 0) cref[j] = a;
            }
            if (lane == 0) nu[j] = nv;
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < p * n; e += blockDim.x) {
        const int c = e / p, i = e - c * p;
        R[i + (int64_t)c * p] = i <= c ? X[c * m + i] : 0.0;
    }
    for (int c = threadIdx.x; c < n; c += blockDim.x) perm_out[c] = perm[c];
    if (!want_q) return;
    for (int e = threadIdx.x; e < m * p; e += blockDim.x) {
        const int c = e / m, i = e - c * m;
        Q[i + (int64_t)c * m] = i == c ? 1.0 : 0.0;
    }
    __syncthreads();
    for (int k = p - 1; k >= 0; --k) {
        const double bk = beta[k];
        if (bk == 0.0) continue;
        const double* v = X + k * m;
        const int c0 = warp;
        if (c0 >= k && c0 < p) {
            double* c = Q + (int64_t)c0 * m;
            double t = 0.0;
            for (int i = k + 1 + lane; i < m; i += 32) t = fma(v[i], c[i], t);
            t = warp_sum(t);
            t = __dmul_rn(__dadd_rn(c[k], t), bk);
            for (int i = k + 1 + lane; i < m; i += 32) c[i] = __dsub_rn(c[i], __dmul_rn(t, v[i]));
            if (lane == 0) c[k] = __dsub_rn(c[k], t);
        }
        __syncthreads();
    }
}

}  // namespace

size_t small_qrcp_smem(int64_t m, int64_t n) {
    const int64_t p = std::min(m, n);
    return sizeof(double) * (size_t)(m * n + 3 * n + p) + sizeof(int) * (size_t)n + 64;
}

bool small_qrcp_fits(int64_t m, int64_t n) { return small_qrcp_smem(m, n) <= 220 * 1024; }

void small_qrcp(const double* A, int64_t m, int64_t n, int64_t lda, int64_t* perm, double* R, double* pnorm,
                double* Q) {
    if (n <= 32) {
        const size_t smem = sizeof(double) * (size_t)(m * n + std::min(m, n));
        allow_smem(k_small_qrcp32, smem);
        TTG_LAUNCH(k_small_qrcp32, 1, 1024, smem, stream(), A, (int)m, (int)n, lda, perm, R, pnorm, Q, Q ? 1 : 0);
        return;
    }
    const size_t smem = small_qrcp_smem(m, n);
    allow_smem(k_small_qrcp, smem);
    TTG_LAUNCH(k_small_qrcp, 1, 512, smem, stream(), A, (int)m, (int)n, lda, perm, R, pnorm, Q, Q ? 1 : 0);
}

bool tsqr_fits(int64_t s) { return s <= 160; }

namespace {
// In-place Cholesky G = R^T R of an s x s SPD matrix (col-major, ld s) in shared memory,
// one CTA; R written upper (zeros below). ok[0] = 1 when every pivot is positive and
// min_i R_ii >= min_ratio * max_i R_ii.
__global__ void __launch_bounds__(kT) k_cholesky(const double* __restrict__ G, int64_t s, double min_ratio, double* R,
                                                 int* ok) {
    extern __shared__ double A[];
    __shared__ int bad;
    for (int64_t e = threadIdx.x; e < s * s; e += kT) A[e] = G[e];
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    for (int64_t j = 0; j < s; ++j) {
        // A(j, j..) -= sum_{k<j} A(k, j) A(k, ..) is already applied (right-looking)
        if (threadIdx.x == 0) {
            const double d = A[j + j * s];
            if (!(d > 0.0)) bad = 1;
            A[j + j * s] = d > 0.0 ? sqrt(d) : 0.0;
        }
        __syncthreads();
        const double rjj = A[j + j * s];
        for (int64_t i = j + 1 + threadIdx.x; i < s; i += kT) A[j + i * s] = rjj > 0.0 ? A[j + i * s] / rjj : 0.0;
        __syncthreads();
        // trailing update A(a, b) -= R(j, a) R(j, b) for j < a <= b
        const int64_t m = s - j - 1;
        for (int64_t e = threadIdx.x; e < m * m; e += kT) {
            const int64_t b = j + 1 + e / m, a = j + 1 + e % m;
            if (a <= b) A[a + b * s] = fma(-A[j + a * s], A[j + b * s], A[a + b * s]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double mx = 0.0, mn = INFINITY;
        for (int64_t i = 0; i < s; ++i) {
            mx = fmax(mx, A[i + i * s]);
            mn = fmin(mn, A[i + i * s]);
        }
        ok[0] = (!bad && mn >= min_ratio * mx) ? 1 : 0;
    }
    for (int64_t e = threadIdx.x; e < s * s; e += kT) {
        const int64_t c = e / s, r = e - c * s;
        R[e] = r <= c ? A[e] : 0.0;
    }
}
}  // namespace

bool cholesky_r(const double* G, int64_t s, double min_ratio, double* R) {
    const size_t smem = sizeof(double) * (size_t)(s * s);
    if (smem > 200 * 1024) return false;
    DevBuf<int> ok(1);
    allow_smem(k_cholesky, smem);
    TTG_LAUNCH(k_cholesky, 1, kT, smem, stream(), G, s, min_ratio, R, ok.get());
    return ok.to_host(1)[0] == 1;
}

// Leaf level with the unrolled kernel <S, RL> when it spans at least a wave, then the
// rolled kernel <S, RU> up the tree.
template <int S, int RL, int RU>
void tsqr_reg_tree(const double* B, int64_t N, int64_t s, int64_t ld, double* Rout) {
    DevBuf<double> lvl;
    const double* in = B;
    int64_t rows = N, ldi = ld;
    bool leaf = true;
    while (true) {
        const bool unr = leaf && cdiv(rows, (int64_t)kT * RL) >= sm_count();
        // the unrolled leaf runs one CTA per SM, each streaming its share of the rows
        const int64_t nb = unr ? (int64_t)sm_count() : cdiv(rows, (int64_t)kT * RU);
        double* dst = Rout;
        DevBuf<double> nxt;
        if (nb > 1) {
            nxt = DevBuf<double>((size_t)(nb * s * s));
            dst = nxt.get();
        }
        if (unr)
            TTG_LAUNCH((k_tsqr_unr<S, RL>), (int)nb, kT, 0, stream(), in, rows, (int)s, ldi, dst, nb * s);
        else
            TTG_LAUNCH((k_tsqr_reg<S, RU>), (int)nb, kT, 0, stream(), in, rows, (int)s, ldi, dst, nb * s);
        leaf = false;
        if (nb == 1) break;
        lvl = std::move(nxt);
        in = lvl.get();
        rows = nb * s;
        ldi = rows;
    }
}

void tsqr_r(const double* B, int64_t N, int64_t s, int64_t ld, double* Rout) {
    if (s <= 8) return tsqr_reg_tree<8, 8, 4>(B, N, s, ld, Rout);
    if (s <= 16) return tsqr_reg_tree<16, 4, 2>(B, N, s, ld, Rout);
    if (s <= 32) return tsqr_reg_tree<32, 2, 1>(B, N, s, ld, Rout);
    // rows per leaf block: a multiple of s, >= 128, within ~200 KB of shared memory
    int rb = (int)std::max<int64_t>(s, 128);
    while ((int64_t)rb * 2 * s * 8 <= 160 * 1024 && rb < 1024) rb *= 2;
    const int64_t nb = cdiv(N, rb);
    DevBuf<double> lvl((size_t)(nb * s * s));
    const size_t smem0 = sizeof(double) * (size_t)rb * s;
    allow_smem(k_tsqr_leaf, smem0);
    TTG_LAUNCH(k_tsqr_leaf, (int)nb, kT, smem0, stream(), B, N, (int)s, ld, rb, lvl.get(), nb * s);
    int64_t rows = nb * s;
    const int g = (int)std::max<int64_t>(2, std::min<int64_t>(16, (160 * 1024) / (8 * s * s)));
    if (g * s * s * 8 > 160 * 1024) {  // large s: structured pairwise tree in packed smem
        const size_t smem = sizeof(double) * (size_t)(s * (s + 1));
        allow_smem(k_tsqr_pair, smem);
        while (rows > s) {
            const int64_t nt = rows / s, nbl = cdiv(nt, 2);
            DevBuf<double> nxt((size_t)(nbl * s * s));
            TTG_LAUNCH(k_tsqr_pair, (int)nbl, kT, smem, stream(), lvl.get(), rows, (int)s, rows, nxt.get(), nbl * s);
            lvl = std::move(nxt);
            rows = nbl * s;
        }
    }
    while (rows > s) {
        const int64_t nbl = cdiv(rows, (int64_t)g * s);
        DevBuf<double> nxt((size_t)(nbl * s * s));
        const size_t need = sizeof(double) * (size_t)g * s * s;
        const bool fits = need <= 200 * 1024;
        const size_t smem = fits ? need : 0;
        allow_smem(k_tsqr_node, smem);
        TTG_LAUNCH(k_tsqr_node, (int)nbl, kT, smem, stream(), lvl.get(), rows, (int)s, rows, g, fits ? 1 : 0,
                   nxt.get(), nbl * s);
        lvl = std::move(nxt);
        rows = nbl * s;
    }
    TTG_CUDA(cudaMemcpyAsync(Rout, lvl.get(), sizeof(double) * s * s, cudaMemcpyDeviceToDevice, stream()));
}

}  // namespace ttg
