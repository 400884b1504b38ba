// Sweep drivers: TT-ULV left-to-right (Alg. 1/2) and TT-URV right-to-left (Alg. 3 and its
// prescribed-accuracy analogue), reference tt_decomp.cpp:156-339.
//
// One cut on device (refine_passes = 1, the two-pass QLP of factor.cpp:376-430):
//   W = c (ULV) or c^T read in place (URV), k x N with k = r * I the short side.
//   pass 1  WideQrcp on W for s steps: pivots P1, explicit Q1[:, :s], R1 rows 0..s-1.
//   pass 2  TallQrcp on B = R1[:s, :]^T (N x s, rows in P1 position order): P2, R2.
//   kept masses from R2 columns (factor.cpp:479-499, same summation order), rank rule
//   (factor.cpp:512-520) or the fixed rank, residual sqrt(total - kept[r]).
//   core   ULV: U1 = Q1[:, P2[:r]]           URV: V1^T = Q1[:, P2[:r]]^T
//   carry  ULV: L11 V1^T = U1^T c = R1[P2[:r], :]   URV: U1 R11 = c V1 = R1[P2[:r], :]^T
// so neither the second orthogonal factor nor a carry GEMM is ever formed: the carry is a
// gather of R1 rows (exactly equal in exact arithmetic, since c = U T V^T with T triangular).
//
// Early exit: s starts at the requested rank (fixed) or grows until the pass-1 trailing
// mass T1(s) falls below the budget (tolerance). The result equals the full p-step QLP
// in exact arithmetic when every pass-2 pivot norm^2 of the kept steps is >= T1(s), the
// largest possible norm^2 of any R1 row not yet computed;
// otherwise s is extended and pass 2 is redone. s = p is exactly the reference schedule.
#include <algorithm>
#include <chrono>
#include <memory>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "sweep.hpp"
#include "utv.hpp"

namespace ttg {
namespace {

using Clock = std::chrono::steady_clock;

// TTG_CUT_TIMING=1: synchronise after every cut and print its wall time (diagnostics).
bool cut_timing() {
    static const bool on = [] {
        const char* e = std::getenv("TTG_CUT_TIMING");
        return e && *e == '1';
    }();
    return on;
}

// ---- small device kernels -----------------------------------------------------------

// B(i, c) = R1(c, perm[i]) for the first s rows of R1 (row c stored at R + c*N).
__global__ void k_gather_b(const double* __restrict__ R, const int64_t* __restrict__ perm, int64_t N, int64_t s,
                           double* B) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= N * s) return;
    const int64_t c = e / N, i = e - c * N;
    B[i + c * N] = R[c * N + perm[i]];
}

// out[e] = sum_p in[p * n + e] in rank order (deterministic cross-rank sum).
__global__ void k_sum_blocks(const double* __restrict__ in, int P, int64_t n, double* out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    double a = 0.0;
    for (int p = 0; p < P; ++p) a += in[(int64_t)p * n + e];
    out[e] = a;
}

// R2 over positions (s x s, col-major): R2(t, q) = R(t, piv[q]) for q >= t (row t of the
// wide engine's R at R + t*s), zero below the diagonal.
__global__ void k_r2_positions(const double* __restrict__ R, const int64_t* __restrict__ piv, int64_t s,
                               double* R2) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= s * s) return;
    const int64_t q = e / s, t = e - q * s;
    R2[e] = q >= t ? R[t * s + piv[q]] : 0.0;
}

__global__ void k_sq_diag(const double* __restrict__ d, int64_t s, double* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < s) out[i] = d[i] * d[i];
}

// kept[0] = 0, kept[c+1] = kept[c] + sum_{i<=c} R2(i,c)^2, sequential sums without
// contraction (kept_mass_upper / kept_mass_lower of factor.cpp:479-499).
__global__ void k_kept(const double* __restrict__ R2, int64_t s, int64_t ldr, double* colmass, double* kept) {
    for (int64_t c = threadIdx.x; c < s; c += blockDim.x) {
        double a = 0.0;
        for (int64_t i = 0; i <= c; ++i) {
            const double v = R2[i + c * ldr];
            a = __dadd_rn(a, __dmul_rn(v, v));
        }
        colmass[c] = a;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double acc = 0.0;
        kept[0] = 0.0;
        for (int64_t c = 0; c < s; ++c) {
            acc = __dadd_rn(acc, colmass[c]);
            kept[c + 1] = acc;
        }
    }
}

// out(:, q) = Q(:, sel[q]) (k x r), or transposed out(q, :) = Q(:, sel[q])^T (r x k).
__global__ void k_gather_qcols(const double* __restrict__ Q, int64_t k, const int64_t* __restrict__ sel, int64_t r,
                               bool transposed, double* out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= k * r) return;
    if (!transposed) {
        const int64_t q = e / k, i = e - q * k;
        out[i + q * k] = Q[i + sel[q] * k];
    } else {
        const int64_t i = e / r, q = e - i * r;
        out[q + i * r] = Q[i + sel[q] * k];
    }
}

// ULV carry: out(q, j) = R1(sel[q], j), r x N column-major (tiled through shared memory).
__global__ void k_carry_rows_t(const double* __restrict__ R, int64_t N, const int64_t* __restrict__ sel, int64_t r,
                               double* out) {
    __shared__ double tile[32][33];
    const int64_t j0 = (int64_t)blockIdx.x * 32, q0 = (int64_t)blockIdx.y * 32;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int64_t q = q0 + y, j = j0 + threadIdx.x;
        if (q < r && j < N) tile[y][threadIdx.x] = R[sel[q] * N + j];
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int64_t j = j0 + y, q = q0 + threadIdx.x;
        if (q < r && j < N) out[q + j * r] = tile[threadIdx.x][y];
    }
}

// URV carry: out(j, q) = R1(sel[q], j), N x r column-major.
__global__ void k_carry_rows(const double* __restrict__ R, int64_t N, const int64_t* __restrict__ sel, int64_t r,
                             double* out) {
    const int64_t q = blockIdx.y;
    const int64_t src = sel[q];
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x)
        out[j + q * N] = R[src * N + j];
}

// ---- mode resolution (tt_decomp.cpp:32-71) ---------------------------------------------
struct Resolved {
    bool fixed = false;
    std::vector<int64_t> ranks;
    std::vector<double> budgets;
};

Resolved resolve_mode(const SweepConfig& cfg, int64_t d, double norm_a, bool rss) {
    const int64_t cuts = d - 1;
    Resolved out;
    if (cfg.fixed_rank) {
        out.fixed = true;
        if ((int64_t)cfg.ranks.size() != d + 1)
            argument_error("rank chain has " + std::to_string(cfg.ranks.size()) + " entries, expected " +
                           std::to_string(d + 1));
        if (cfg.ranks.front() != 1 || cfg.ranks.back() != 1) argument_error("boundary ranks must both be 1");
        for (int64_t r : cfg.ranks)
            if (r < 1) argument_error("ranks must be >= 1");
        out.ranks = cfg.ranks;
        return out;
    }
    if (cfg.eps < 0.0) argument_error("tolerance must be >= 0");
    std::vector<double> w = cfg.weights;
    if (w.empty()) {
        const double c = (double)std::max<int64_t>(cuts, 1);
        w.assign((size_t)cuts, rss ? 1.0 / std::sqrt(c) : 1.0 / c);
    } else {
        if ((int64_t)w.size() != cuts)
            argument_error(std::to_string(w.size()) + " weights given, expected " + std::to_string(cuts));
        double total = 0.0;
        for (double x : w) {
            if (x < 0.0) argument_error("weights must be >= 0");
            total += rss ? x * x : x;
        }
        if (std::abs(total - 1.0) > 1e-12)
            argument_error(rss ? "squared weights must sum to 1" : "weights must sum to 1");
    }
    for (double x : w) out.budgets.push_back(x * cfg.eps * norm_a);
    return out;
}

// ---- one cut ------------------------------------------------------------------------------
struct CutOut {
    int64_t rank = 0, steps = 0, extensions = 0;
    double step_error = 0.0;    // the reference's sqrt(max(0, kept[p] - kept[r])) (factor.cpp:507-510)
    double direct_error = 0.0;  // the discarded mass computed directly (no cancellation)
    std::vector<double> kept;   // kept[0..s] of the rank rule, then kept[p] (the total) last
    std::vector<double> diag;
    DevBuf<int64_t> sel;  // P2[:rank] on device
};

struct CutRequest {
    bool fixed;
    int64_t rank;   // fixed mode (already clamped to p)
    double budget;  // tolerance mode
    int policy;
};

// Pass 1 of a cut behind one interface: the wide read-only engine (k moderate) or, when W
// is tall (k >> N, e.g. the last URV cut of config 5: W = 131072 x 1024), the in-place
// Householder engine on a column-major copy of W.
bool gram_r(const double* R1, int64_t N, int64_t s, Comm* comm, double* RB, double r1_ratio);

struct Pass1 {
    virtual ~Pass1() = default;
    virtual int64_t p() const = 0;
    virtual int64_t N() const = 0;
    virtual int64_t k() const = 0;
    virtual void run_to(int64_t s) = 0;
    virtual double trailing_mass() = 0;  // may carry downdating noise
    virtual double refresh_exact() = 0;  // exact trailing mass
    virtual const double* R() = 0;       // R1 rows 0..s-1 by original column, row t at R + t*N
    virtual const int64_t* perm() = 0;   // positions -> columns
    virtual const double* Q() = 0;       // economy Q columns 0..s-1, leading dimension k
    virtual bool sharded() const { return false; }
    // Sharded with each rank holding only its own columns of R1 (the column-sharded wide
    // engine); the Gram route's R1 is replicated on every rank.
    virtual Comm* partitioned_comm() { return nullptr; }
    // R_B (s x s, ld s) of B = R1[:s, :]^T over all columns (all ranks when sharded).
    virtual void r_factor(int64_t s, double* RB) {
        if (!gram_r(R(), N(), s, nullptr, RB, 0.0)) tsqr_r(R(), N(), s, N(), RB);
    }
};

// R_B from the Gram matrix B^T B = R1 R1^T (one DMMA GEMM over the s x N rows of R1, summed
// over the ranks in rank order when sharded) and its Cholesky factor. Only for s > 32 (the
// register TSQR is fast below) and only when the factor is well conditioned: the error of
// a Gram-based R is about eps * cond(B) relative to |T_00|, so min/max R_ii >= 1e-4 keeps
// it far inside the 1e-10 parity tolerance. Otherwise the caller falls back to TSQR.
bool gram_r(const double* R1, int64_t N, int64_t s, Comm* comm, double* RB, double r1_ratio) {
    constexpr double kMinRatio = 1e-4;
    if ((size_t)(s * s) * sizeof(double) > 200 * 1024) return false;
    // s <= 32: only when pass 1's own diagonal says R1 is well conditioned (the register
    // TSQR is the fallback and costs about as much as a rejected Gram attempt)
    if (s <= 32 && !(r1_ratio >= 1e-3)) return false;
    DevBuf<double> G((size_t)(s * s));
    if (s <= 32) gram_small(R1, N, s, N, G.get());
    else gemm(true, false, s, s, N, R1, N, R1, N, G.get(), s);
    if (comm && comm->size() > 1) {
        const int P = comm->size();
        DevBuf<double> all((size_t)(P * s * s));
        comm->allgather(G.get(), all.get(), sizeof(double) * (size_t)(s * s));
        TTG_LAUNCH(k_sum_blocks, (int)cdiv(s * s, 256), 256, 0, stream(), all.get(), P, s * s, G.get());
    }
    const bool ok = cholesky_r(G.get(), s, kMinRatio, RB);
    if (cut_timing()) {
        std::vector<double> r((size_t)(s * s));
        TTG_CUDA(cudaMemcpyAsync(r.data(), RB, sizeof(double) * s * s, cudaMemcpyDeviceToHost, stream()));
        sync();
        double mx = 0.0, mn = 1e300;
        for (int64_t i = 0; i < s; ++i) { mx = std::max(mx, r[(size_t)(i + i * s)]); mn = std::min(mn, r[(size_t)(i + i * s)]); }
        std::fprintf(stderr, "[ttg]   gram R_B (s=%lld): %s, min/max diag %.3e\n", (long long)s, ok ? "used" : "rejected", mn / mx);
    }
    return ok;
}

struct WidePass1 final : Pass1 {
    WideQrcp e;
    WidePass1(const double* W, int64_t k, int64_t N, int64_t ld, Layout l, int64_t cap,
              const ShardSpec* shard = nullptr, bool subspace = false)
        : e(W, k, N, ld, l, cap, shard, subspace) {}
    bool sharded() const override { return e.sharded(); }
    Comm* partitioned_comm() override { return e.sharded() ? e.comm() : nullptr; }
    // Sharded: every rank reduces its own rows of B to a triangle, the triangles are
    // all-gathered and stacked in rank order, and every rank factors the same stack.
    // |R1(s-1, s-1)| / |R1(0, 0)| from pass 1's diagonal (host sync of two values)
    double r1_ratio(int64_t s) {
        double d0 = 0.0, ds = 0.0;
        TTG_CUDA(cudaMemcpyAsync(&d0, e.diag(), sizeof(double), cudaMemcpyDeviceToHost, stream()));
        TTG_CUDA(cudaMemcpyAsync(&ds, e.diag() + (s - 1), sizeof(double), cudaMemcpyDeviceToHost, stream()));
        sync();
        return d0 != 0.0 ? std::abs(ds) / std::abs(d0) : 0.0;
    }
    void r_factor(int64_t s, double* RB) override {
        if (gram_r(e.R(), e.N(), s, e.comm(), RB, s <= 32 ? r1_ratio(s) : 1.0)) return;
        if (!e.sharded()) return tsqr_r(e.R(), e.N(), s, e.N(), RB);
        Comm& comm = *e.comm();
        const int G = comm.size();
        if (comm.has_p2p() && G > 1) {
            // binary TSQR tree over the ranks (log2 G point-to-point rounds): at round l, rank
            // g with g % 2l == 0 receives the triangle of rank g + l, stacks the two and
            // refactors; rank 0's final triangle is then broadcast (all-gather, block 0)
            DevBuf<double> mine((size_t)(s * s)), other((size_t)(s * s)), stack((size_t)(2 * s * s));
            tsqr_r(e.R(), e.N(), s, e.N(), mine.get());
            const int g = comm.rank();
            for (int l = 1; l < G; l <<= 1) {
                const bool recv = g % (2 * l) == 0 && g + l < G;
                const bool send = g % (2 * l) == l;
                comm.sendrecv(mine.get(), send ? g - l : -1, other.get(), recv ? g + l : -1,
                              sizeof(double) * (size_t)(s * s));
                if (recv) {
                    TTG_CUDA(cudaMemcpy2DAsync(stack.get(), sizeof(double) * 2 * s, mine.get(), sizeof(double) * s,
                                               sizeof(double) * s, s, cudaMemcpyDeviceToDevice, stream()));
                    TTG_CUDA(cudaMemcpy2DAsync(stack.get() + s, sizeof(double) * 2 * s, other.get(),
                                               sizeof(double) * s, sizeof(double) * s, s, cudaMemcpyDeviceToDevice,
                                               stream()));
                    tsqr_r(stack.get(), 2 * s, s, 2 * s, mine.get());
                }
            }
            DevBuf<double> all((size_t)(G * s * s));
            comm.allgather(mine.get(), all.get(), sizeof(double) * (size_t)(s * s));
            TTG_CUDA(cudaMemcpyAsync(RB, all.get(), sizeof(double) * (size_t)(s * s), cudaMemcpyDeviceToDevice,
                                     stream()));
            return;
        }
        DevBuf<double> mine((size_t)(s * s)), all((size_t)(G * s * s)), stack((size_t)(G * s * s));
        tsqr_r(e.R(), e.N(), s, e.N(), mine.get());
        comm.allgather(mine.get(), all.get(), sizeof(double) * (size_t)(s * s));
        for (int g = 0; g < G; ++g)
            TTG_CUDA(cudaMemcpy2DAsync(stack.get() + (int64_t)g * s, sizeof(double) * G * s, all.get() + (int64_t)g * s * s,
                                       sizeof(double) * s, sizeof(double) * s, s, cudaMemcpyDeviceToDevice, stream()));
        tsqr_r(stack.get(), G * s, s, G * s, RB);
    }
    int64_t p() const override { return e.p(); }
    int64_t N() const override { return e.N(); }
    int64_t k() const override { return e.k(); }
    void run_to(int64_t s) override { e.run_to(s); }
    double trailing_mass() override { return e.trailing_mass(); }
    double refresh_exact() override { return e.refresh_exact(); }
    const double* R() override { return e.R(); }
    const int64_t* perm() override { return e.perm(); }
    const double* Q() override { return e.Q(); }
};

struct TallPass1 final : Pass1 {
    DevBuf<double> B, rrows, qbuf;
    int64_t k_, N_, rs_ = -1, qs_ = -1;
    std::unique_ptr<TallQrcp> e;
    TallPass1(const double* W, int64_t k, int64_t N, int64_t ld, Layout l) : k_(k), N_(N) {
        B.alloc((size_t)(k * N));
        if (l == Layout::Col)
            TTG_CUDA(cudaMemcpy2DAsync(B.get(), sizeof(double) * k, W, sizeof(double) * ld, sizeof(double) * k, N,
                                       cudaMemcpyDeviceToDevice, stream()));
        else  // W(i,j) = W[i*ld + j]: the buffer is an N x k column-major matrix
            transpose(W, N, k, ld, B.get(), k);
        e = std::make_unique<TallQrcp>(B.get(), k, N, k);
    }
    int64_t p() const override { return e->p(); }
    int64_t N() const override { return N_; }
    int64_t k() const override { return k_; }
    void run_to(int64_t s) override { e->run(s); }
    double trailing_mass() override { return e->trailing_mass_exact(); }
    double refresh_exact() override { return e->trailing_mass_exact(); }
    const double* R() override {
        const int64_t s = e->steps();
        if (rs_ != s) {
            rrows.alloc((size_t)(s * N_));
            e->r_rows_by_column(rrows.get(), N_);
            rs_ = s;
        }
        return rrows.get();
    }
    const int64_t* perm() override { return e->perm(); }
    const double* Q() override {
        const int64_t s = e->steps();
        if (qs_ != s) {
            qbuf.alloc((size_t)(k_ * s));
            e->form_q(qbuf.get(), s, k_);
            qs_ = s;
        }
        return qbuf.get();
    }
};

// Narrow W (k <= 32) in tolerance mode: the bitwise engine (qrcp_exact.cu), so the R1 rows past
// the numerical rank -- pass 1's rounding residue, which decides an ulp-level rank -- are the
// reference's own.
struct ExactPass1 final : Pass1 {
    ExactQrcp e;
    int64_t k_, N_, rs_ = -1, qs_ = -1;
    DevBuf<double> rrows, qbuf;
    ExactPass1(const double* W, int64_t k, int64_t N, int64_t ld, Layout l) : e(W, k, N, ld, l), k_(k), N_(N) {}
    int64_t p() const override { return e.p(); }
    int64_t N() const override { return N_; }
    int64_t k() const override { return k_; }
    void run_to(int64_t s) override { e.run_to(s); }
    double trailing_mass() override { return e.trailing_mass_exact(); }
    double refresh_exact() override { return e.trailing_mass_exact(); }
    const double* R() override {
        const int64_t s = e.steps();
        if (rs_ != s) {
            rrows.alloc((size_t)(s * N_));
            e.r_rows(rrows.get(), s);
            rs_ = s;
        }
        return rrows.get();
    }
    const int64_t* perm() override { return e.perm(); }
    const double* Q() override {
        const int64_t s = e.steps();
        if (qs_ != s) {
            qbuf.alloc((size_t)(k_ * s));
            e.form_q(qbuf.get(), s);
            qs_ = s;
        }
        return qbuf.get();
    }
};

// Small W (fits one CTA's shared memory): the whole pass 1 is the reference's
// qr_col_pivot run step for step by one CTA (k_small_qrcp), one launch instead of a few
// launches per step; every prefix s of the full factorisation is what the early exit
// asks for, and the trailing mass of rows s.. is exact.
__global__ void k_scatter_rows(const double* __restrict__ Rpos, const int64_t* __restrict__ perm, int64_t p,
                               int64_t N, double* Rrow) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= p * N) return;
    const int64_t q = e / p, t = e - q * p;
    Rrow[t * N + perm[q]] = Rpos[t + q * p];
}

// ---- tall W (k >> N), fixed rank: pivoted Cholesky of the Gram matrix -------------------
// QRCP of W and pivoted Cholesky of G = W^T W choose the same pivots (the residual column
// norms are the residual diagonal of G) and the same R in exact arithmetic, so for a tall
// W the whole pass 1 runs on the N x N Gram matrix: one DMMA GEMM over W (split-K, summed
// over the ranks when W's rows are sharded), then O(N t) per step. The economy Q columns
// are Q[:, :s] = W[:, piv] R11^{-1} (a triangular solve per row). Gram-based factors carry
// eps * cond^2 errors, so the engine only keeps this result when R_ss / R_00 >= 1e-4
// (otherwise it falls back to the Householder engine): then every R entry is within about
// eps * cond |R_00| of the Householder one, far inside the 1e-10 parity contract.
__global__ void k_gc_init(const double* __restrict__ G, int64_t N, double* D, double* Dref, int64_t* pos,
                          int64_t* perm) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
        D[j] = G[j + j * N];
        Dref[j] = D[j];
        pos[j] = j;
        perm[j] = j;
    }
}

// One step of the pivoted Cholesky (one CTA of 1024 threads): pivot by (D desc, position
// asc) like qr_col_pivot (factor.cpp:85-93), row t of R, downdate of D.
__global__ void __launch_bounds__(1024) k_gc_step(const double* __restrict__ G, int64_t N, int64_t t, double* D,
                                                  int64_t* pos, int64_t* perm, int64_t* piv, double* R) {
    __shared__ Cand sc[32];
    extern __shared__ double rp[];  // R(0:t, piv) then the new row's pivot scalar
    Cand best = cand_none();
    for (int64_t j = threadIdx.x; j < N; j += blockDim.x) {
        const int64_t pj = pos[j];
        if (pj < t) continue;
        const Cand c{D[j], pj, j};
        if (better(c, best)) best = c;
    }
    {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        best = warp_best(best);
        if (lane == 0) sc[warp] = best;
        __syncthreads();
        Cand b = lane < nw ? sc[lane] : cand_none();
        best = warp_best(b);
    }
    const int64_t jp = best.col >= 0 ? best.col : perm[t];
    const int64_t pp = best.col >= 0 ? best.pos : t;
    const int64_t ct = perm[t];
    __syncthreads();
    if (threadIdx.x == 0) {
        perm[t] = jp;
        perm[pp] = ct;
        pos[jp] = t;
        pos[ct] = pp;
        piv[t] = jp;
    }
    for (int64_t l = threadIdx.x; l < t; l += blockDim.x) rp[l] = R[l * N + jp];
    __syncthreads();
    const double dj = D[jp];
    const double rtt = dj > 0.0 ? sqrt(dj) : 0.0;
    for (int64_t j = threadIdx.x; j < N; j += blockDim.x) {
        const int64_t pj = (j == jp) ? t : (j == ct ? pp : pos[j]);
        double r;
        if (j == jp) {
            r = rtt;
        } else if (pj < t) {
            r = 0.0;
        } else {
            double a = G[jp + j * N];
            for (int64_t l = 0; l < t; ++l) a = fma(-rp[l], R[l * N + j], a);
            r = rtt > 0.0 ? a / rtt : 0.0;
            D[j] = D[j] - r * r;
        }
        R[t * N + j] = r;
    }
}

// Rows of Q[:, :s] = W[:, piv[:s]] R11^{-1}: q R11 = x by forward substitution, one thread
// per row of W, R11 (s x s over positions) staged in shared memory.
__global__ void k_gc_q(const double* __restrict__ W, int64_t k, int64_t ld, int layout,
                       const double* __restrict__ R, int64_t N, const int64_t* __restrict__ piv, int64_t s,
                       double* Q) {
    extern __shared__ double r11[];  // r11[m + l*s] = R(m, piv_l)
    for (int64_t e = threadIdx.x; e < s * s; e += blockDim.x) {
        const int64_t l = e / s, m = e - l * s;
        r11[e] = m <= l ? R[m * N + piv[l]] : 0.0;
    }
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        for (int64_t l = 0; l < s; ++l) {
            const int64_t c = piv[l];
            double x = layout == 0 ? W[i + c * ld] : W[i * ld + c];
            for (int64_t m = 0; m < l; ++m) x = fma(-Q[i + m * k], r11[m + l * s], x);
            const double d = r11[l + l * s];
            Q[i + l * k] = d != 0.0 ? x / d : 0.0;
        }
    }
}

// R11^{-1} (s x s upper, col-major) with R11(m, l) = R(m, piv_l): column j solves R11 x = e_j
// by back substitution, one thread per column.
__global__ void k_gc_rinv(const double* __restrict__ R, int64_t N, const int64_t* __restrict__ piv, int64_t s,
                          double* Rinv) {
    extern __shared__ double r11[];  // r11[m + l s]
    for (int64_t e = threadIdx.x; e < s * s; e += blockDim.x) {
        const int64_t l = e / s, m = e - l * s;
        r11[e] = m <= l ? R[m * N + piv[l]] : 0.0;
    }
    __syncthreads();
    for (int64_t j = threadIdx.x; j < s; j += blockDim.x) {
        double* x = Rinv + j * s;
        for (int64_t i = s - 1; i >= 0; --i) {
            if (i > j) { x[i] = 0.0; continue; }
            double a = i == j ? 1.0 : 0.0;
            for (int64_t l = i + 1; l <= j; ++l) a = fma(-r11[i + l * s], x[l], a);
            const double d = r11[i + i * s];
            x[i] = d != 0.0 ? a / d : 0.0;
        }
    }
}

// X (k x s, col-major) = W[:, piv[0..s)]
__global__ void k_gc_gather(const double* __restrict__ W, int64_t k, int64_t ld, int layout,
                            const int64_t* __restrict__ piv, int64_t s, double* X) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < k * s; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t l = e / k, i = e - l * k;
        X[e] = layout == 0 ? W[i + piv[l] * ld] : W[i * ld + piv[l]];
    }
}

__global__ void k_masked_sum(const double* __restrict__ D, const int64_t* __restrict__ pos, int64_t N, int64_t s,
                             double* out) {
    __shared__ double red[32];
    double a = 0.0;
    for (int64_t j = threadIdx.x; j < N; j += blockDim.x)
        if (pos[j] >= s) a += fmax(D[j], 0.0);
    a = block_sum(a, red);
    if (threadIdx.x == 0) out[0] = a;
}

struct GramPass1 final : Pass1 {
    const double* W_;
    int64_t k_, N_, ld_, kg_;
    Layout l_;
    Comm* comm_;
    int64_t s_ = 0, qs_ = -1;
    DevBuf<double> G, D, Dref, Rb, Qb;
    DevBuf<int64_t> posb, permb, pivb;
    // W: k local rows (of kg in all) by N columns; comm non-null when the rows are sharded.
    GramPass1(const double* W, int64_t k, int64_t N, int64_t ld, Layout l, Comm* comm, int64_t cap)
        : W_(W), k_(k), N_(N), ld_(ld), kg_(k), l_(l), comm_(comm) {
        G.alloc((size_t)(N * N));
        // G = W^T W; Col: W is k x N (ld); Row: W^T is N x k column-major (ld)
        if (l == Layout::Col) syrk(true, N, k, W, ld, G.get(), N);
        else syrk(false, N, k, W, ld, G.get(), N);
        if (comm && comm->size() > 1) {
            const int P = comm->size();
            DevBuf<double> all((size_t)(P * N * N));
            comm->allgather(G.get(), all.get(), sizeof(double) * (size_t)(N * N));
            TTG_LAUNCH(k_sum_blocks, (int)cdiv(N * N, 256), 256, 0, stream(), all.get(), P, N * N, G.get());
            kg_ = (int64_t)llround(global_sum(*comm, (double)k));
        }
        D.alloc((size_t)N);
        Dref.alloc((size_t)N);
        posb.alloc((size_t)N);
        permb.alloc((size_t)N);
        pivb.alloc((size_t)std::min(cap, N));
        Rb.alloc((size_t)(std::min(cap, N) * N));
        TTG_LAUNCH(k_gc_init, (int)cdiv(N, 256), 256, 0, stream(), G.get(), N, D.get(), Dref.get(), posb.get(),
                   permb.get());
    }
    int64_t p() const override { return std::min(kg_, N_); }
    int64_t N() const override { return N_; }
    int64_t k() const override { return k_; }
    bool sharded() const override { return comm_ != nullptr && comm_->size() > 1; }
    void run_to(int64_t s) override {
        s = std::min(s, p());
        if ((size_t)(s * N_) > Rb.size()) {  // grow R rows and pivots
            DevBuf<double> nr((size_t)(s * N_));
            DevBuf<int64_t> np((size_t)s);
            if (s_ > 0) {
                TTG_CUDA(cudaMemcpyAsync(nr.get(), Rb.get(), sizeof(double) * s_ * N_, cudaMemcpyDeviceToDevice, stream()));
                TTG_CUDA(cudaMemcpyAsync(np.get(), pivb.get(), sizeof(int64_t) * s_, cudaMemcpyDeviceToDevice, stream()));
            }
            Rb = std::move(nr);
            pivb = std::move(np);
        }
        for (int64_t t = s_; t < s; ++t) {
            const size_t sm = sizeof(double) * (size_t)(t + 1);
            allow_smem(k_gc_step, sm);
            TTG_LAUNCH(k_gc_step, 1, 1024, sm, stream(), G.get(), N_, t, D.get(), posb.get(), permb.get(), pivb.get(),
                       Rb.get());
        }
        s_ = std::max(s_, s);
    }
    double trailing_mass() override {
        DevBuf<double> m(1);
        TTG_LAUNCH(k_masked_sum, 1, 1024, 0, stream(), D.get(), posb.get(), N_, s_, m.get());
        return m.to_host(1)[0];
    }
    double refresh_exact() override { return trailing_mass(); }
    const double* R() override { return Rb.get(); }
    const int64_t* perm() override { return permb.get(); }
    const double* Q() override {
        if (qs_ != s_) {
            Qb.alloc((size_t)(k_ * s_));
            const size_t sm = sizeof(double) * (size_t)(s_ * s_);
            // Q[:, :s] = W[:, piv] R11^{-1}: the triangular inverse (one CTA) and one DMMA GEMM
            // (config 5's 131072 x 128: 5 ms of per-row substitution before). R11 is well
            // conditioned here (cut_with keeps the route only for R_ss / R_00 >= 1e-4).
            DevBuf<double> Rinv((size_t)(s_ * s_)), X((size_t)(k_ * s_));
            allow_smem(k_gc_rinv, sm);
            TTG_LAUNCH(k_gc_rinv, 1, 128, sm, stream(), Rb.get(), N_, pivb.get(), s_, Rinv.get());
            TTG_LAUNCH(k_gc_gather, (int)std::min<int64_t>(cdiv(k_ * s_, 256), 16 * sm_count()), 256, 0, stream(), W_,
                       k_, ld_, (int)l_, pivb.get(), s_, X.get());
            gemm(false, false, k_, s_, s_, X.get(), k_, Rinv.get(), s_, Qb.get(), k_);
            qs_ = s_;
        }
        return Qb.get();
    }
    // R_ss / R_00 over the first s steps (host sync): the acceptance test of the Gram route.
    double diag_ratio() {
        if (s_ == 0) return 1.0;
        std::vector<int64_t> pv = pivb.to_host((size_t)s_);
        double r0 = 0.0, rs = 0.0;
        TTG_CUDA(cudaMemcpyAsync(&r0, Rb.get() + pv[0], sizeof(double), cudaMemcpyDeviceToHost, stream()));
        TTG_CUDA(cudaMemcpyAsync(&rs, Rb.get() + (s_ - 1) * N_ + pv[(size_t)(s_ - 1)], sizeof(double),
                                 cudaMemcpyDeviceToHost, stream()));
        sync();
        return r0 > 0.0 ? rs / r0 : 0.0;
    }
};

struct SmemPass1 final : Pass1 {
    int64_t k_, N_, p_;
    DevBuf<double> Wc, Rpos, Rrow, Qb, pn;
    DevBuf<int64_t> permb;
    std::vector<double> rowmass;  // |R row t|^2 over positions
    SmemPass1(const double* W, int64_t k, int64_t N, int64_t ld, Layout l) : k_(k), N_(N), p_(std::min(k, N)) {
        const double* A = W;
        int64_t lda = ld;
        if (l == Layout::Row) {  // W(i, j) = W[i*ld + j]: make the k x N column-major copy
            Wc.alloc((size_t)(k * N));
            transpose(W, N, k, ld, Wc.get(), k);
            A = Wc.get();
            lda = k;
        }
        Rpos.alloc((size_t)(p_ * N));
        Rrow.alloc((size_t)(p_ * N));
        Qb.alloc((size_t)(k * p_));
        pn.alloc((size_t)p_);
        permb.alloc((size_t)N);
        small_qrcp(A, k, N, lda, permb.get(), Rpos.get(), pn.get(), Qb.get());
        TTG_LAUNCH(k_scatter_rows, (int)cdiv(p_ * N, 256), 256, 0, stream(), Rpos.get(), permb.get(), p_, N,
                   Rrow.get());
        std::vector<double> h = Rpos.to_host((size_t)(p_ * N));
        rowmass.assign((size_t)p_, 0.0);
        for (int64_t q = 0; q < N; ++q)
            for (int64_t t = 0; t < p_; ++t) rowmass[(size_t)t] += h[(size_t)(t + q * p_)] * h[(size_t)(t + q * p_)];
    }
    int64_t p() const override { return p_; }
    int64_t N() const override { return N_; }
    int64_t k() const override { return k_; }
    void run_to(int64_t s) override { s_ = std::min(s, p_); }
    double trailing_mass() override {
        double m = 0.0;
        for (int64_t t = s_; t < p_; ++t) m += rowmass[(size_t)t];
        return m;
    }
    double refresh_exact() override { return trailing_mass(); }
    const double* R() override { return Rrow.get(); }
    const int64_t* perm() override { return permb.get(); }
    const double* Q() override { return Qb.get(); }

private:
    int64_t s_ = 0;
};

// Engine choice: the read-only WY engine costs O(k t) per step besides the stream over W,
// so it serves wide and tall W alike; TTG_TALL_INPLACE=1 selects the in-place engine for
// tall W instead (kept as a cross-check).
std::unique_ptr<Pass1> make_pass1(const double* W, int64_t k, int64_t N, int64_t ld, Layout l, int64_t cap,
                                  bool fixed = false, bool prev_near_full = false, int policy = 0) {
    // bitwise QLP: narrow W runs the reference's own arithmetic (its rounding residue decides
    // ulp-level ranks, config 2)
    if (policy == 2 && k <= 32) return std::make_unique<ExactPass1>(W, k, N, ld, l);
    static const bool inplace = [] {
        const char* e = std::getenv("TTG_TALL_INPLACE");
        return e && *e == '1';
    }();
    static const bool no_gram = [] {
        const char* e = std::getenv("TTG_NO_GRAM_PASS1");
        return e && *e == '1';
    }();
    // very tall W run to many steps (config 4's 16304 x 1024 cut in tolerance mode): the
    // compact-WY reflector costs O(k t) per step and dominates once t ~ N, the in-place
    // engine O(k N) (measured 1.34 s -> 0.43 s); short runs (N < 512) stay read-only
    if ((inplace && k > 2048 && k > N) || (!fixed && k > 2048 && k >= 8 * N && N >= 64))
        return std::make_unique<TallPass1>(W, k, N, ld, l);
    // square / wide near-full-rank cuts in tolerance mode (config 4's 4096 x 4096 and
    // 1024 x 16384; k >= 1024 keeps configs 2-3's short early-exit runs read-only): the in-place
    // engine's column-parallel steps (TallQrcp col mode) instead of O(k t) WY / O(k^2)
    // explicit-Q work per step
    static const int64_t inplace_mink = [] {  // experiment: TTG_INPLACE_MINK
        const char* e = std::getenv("TTG_INPLACE_MINK");
        return e ? (int64_t)std::atoll(e) : (int64_t)1024;
    }();
    if (!fixed && k >= inplace_mink && k <= 25600 && N >= 2048) return std::make_unique<TallPass1>(W, k, N, ld, l);
    // shorter unfoldings go in place too when the previous cut of the sweep kept >= 90% of
    // its p (a near-full-rank tensor: config 4's 256 x 65,536 cut 87 -> 54 ms); an early
    // exit (config 2's mid cuts) keeps the read-only engine
    if (!fixed && prev_near_full && k >= 256 && k <= 25600 && N >= 2048)
        return std::make_unique<TallPass1>(W, k, N, ld, l);
    // tall W, fixed rank: the pivoted Cholesky of W^T W (cut_with() checks its conditioning)
    if (fixed && !no_gram && k >= 8 * N && N <= 4096 && cap <= 160 && cap >= 1)
        return std::make_unique<GramPass1>(W, k, N, ld, l, nullptr, cap);
    const int64_t p = std::min(k, N);
    if (small_qrcp_fits(k, N) && (k * N <= 16384 || 2 * cap >= p)) return std::make_unique<SmemPass1>(W, k, N, ld, l);
    return std::make_unique<WidePass1>(W, k, N, ld, l, cap, nullptr, fixed);
}

// Pass-2 outputs on the host: pivot order, kept masses, pivot norms, |diag R2|.
struct Pass2 {
    std::vector<double> kept, colmass, pnorm, diag;
    DevBuf<int64_t> perm;  // positions -> R1 row (pass-1 step) index
};

Pass2 run_pass2(Pass1& e1, int64_t s, int policy = 0) {
    const int64_t N = e1.N();
    PhaseTimer pt("pass2 (incl. host sync)");
    Pass2 out;
    DevBuf<double> R2((size_t)s * s), colmass(s), kept(s + 1), pn(s);
    out.perm.alloc(s);
    if (policy == 2 && s == e1.p() && s <= 32 && dynamic_cast<ExactPass1*>(&e1)) {
        // bitwise: qr_col_pivot(transpose(R1)) as the reference runs it (factor.cpp:362-372),
        // B's rows in pass-1 position order
        DevBuf<double> B((size_t)N * s);
        TTG_LAUNCH(k_gather_b, (int)cdiv(N * s, 256), 256, 0, stream(), e1.R(), e1.perm(), N, s, B.get());
        exact_tall_qrcp(B.get(), N, s, R2.get(), out.perm.get(), pn.get());
    } else if (tsqr_fits(s) && small_qrcp_fits(s, s)) {
        // QRCP(R_B) with B = R1[:s,:]^T = Q_B R_B: same pivots and |R| as QRCP(B).
        DevBuf<double> RB((size_t)s * s);
        e1.r_factor(s, RB.get());
        small_qrcp(RB.get(), s, s, s, out.perm.get(), R2.get(), pn.get(), nullptr);
    } else {
        if (Comm* comm = e1.partitioned_comm()) {
            // Long sharded pass 1 (s beyond the TSQR / Gram sizes, e.g. a fixed rank above 160
            // or a tolerance cut that grew): all-gather the ranks' blocks of B = R1[:s, :]^T
            // (R1's rows are B's columns, N local rows each) and run the in-place QRCP on the
            // stacked B, replicated. Row order does not change QRCP's pivots or R.
            const int G = comm->size();
            DevBuf<double> all((size_t)G * N * s), Bs((size_t)G * N * s);
            comm->allgather(e1.R(), all.get(), sizeof(double) * (size_t)(N * s));
            for (int g = 0; g < G; ++g)
                TTG_CUDA(cudaMemcpy2DAsync(Bs.get() + (int64_t)g * N, sizeof(double) * (size_t)(G * N),
                                           all.get() + (int64_t)g * N * s, sizeof(double) * (size_t)N,
                                           sizeof(double) * (size_t)N, (size_t)s, cudaMemcpyDeviceToDevice, stream()));
            TallQrcp e2(Bs.get(), G * N, s, G * N);
            e2.run(s);
            e2.extract_r(R2.get(), s);
            TTG_CUDA(cudaMemcpyAsync(pn.get(), e2.pivot_norm2(), sizeof(double) * s, cudaMemcpyDeviceToDevice, stream()));
            TTG_CUDA(cudaMemcpyAsync(out.perm.get(), e2.perm(), sizeof(int64_t) * s, cudaMemcpyDeviceToDevice, stream()));
            goto kept;
        }
        static const bool wide_pass2 = [] {  // TTG_WIDE_PASS2=1: the read-only engine below
            const char* e = std::getenv("TTG_WIDE_PASS2");
            return e && *e == '1';
        }();
        if (wide_pass2 && N <= 8192) {
            // B = R1[:s, :]^T read in place (column c of B = row c of R1): the read-only engine,
            // which switches to an explicit Q for these long factorisations. The default is the
            // in-place engine below (column-parallel steps for N <= 25600): measured 28 -> 3 ms
            // at s = 256, 800 -> 150 ms at s = 4096 (config 4)
            WideQrcp e2(e1.R(), N, s, N, Layout::Col, s);
            e2.run_to(s);
            TTG_LAUNCH(k_r2_positions, (int)cdiv(s * s, 256), 256, 0, stream(), e2.R(), e2.piv(), s, R2.get());
            TTG_LAUNCH(k_sq_diag, (int)cdiv(s, 256), 256, 0, stream(), e2.diag(), s, pn.get());
            TTG_CUDA(cudaMemcpyAsync(out.perm.get(), e2.piv(), sizeof(int64_t) * s, cudaMemcpyDeviceToDevice,
                                     stream()));
            goto kept;
        }
        {
        DevBuf<double> B((size_t)N * s);
        TTG_LAUNCH(k_gather_b, (int)cdiv(N * s, 256), 256, 0, stream(), e1.R(), e1.perm(), N, s, B.get());
        TallQrcp e2(B.get(), N, s, N);
        e2.run(s);
        e2.extract_r(R2.get(), s);
        TTG_CUDA(cudaMemcpyAsync(pn.get(), e2.pivot_norm2(), sizeof(double) * s, cudaMemcpyDeviceToDevice, stream()));
        TTG_CUDA(cudaMemcpyAsync(out.perm.get(), e2.perm(), sizeof(int64_t) * s, cudaMemcpyDeviceToDevice, stream()));
        }
    }
kept:
    TTG_LAUNCH(k_kept, 1, 256, 0, stream(), R2.get(), s, s, colmass.get(), kept.get());
    out.kept.resize((size_t)s + 1);
    out.colmass.resize((size_t)s);
    out.pnorm.resize((size_t)s);
    out.diag.resize((size_t)s);
    kept.download(out.kept.data(), (size_t)s + 1);
    colmass.download(out.colmass.data(), (size_t)s);
    pn.download(out.pnorm.data(), (size_t)s);
    // only the diagonal of R2 goes to the host (a strided copy: s values, not s^2)
    TTG_CUDA(cudaMemcpy2DAsync(out.diag.data(), sizeof(double), R2.get(), sizeof(double) * (size_t)(s + 1),
                               sizeof(double), (size_t)s, cudaMemcpyDeviceToHost, stream()));
    sync();
    for (int64_t t = 0; t < s; ++t) out.diag[(size_t)t] = std::abs(out.diag[(size_t)t]);
    return out;
}

CutOut run_cut(Pass1& e1, const CutRequest& req) {
    const int64_t p = e1.p();
    int64_t s;
    if (req.policy >= 1) s = p;
    else if (req.fixed) s = req.rank;
    else s = std::min<int64_t>(p, 16);
    const double b2 = req.budget * req.budget;
    CutOut out;
    auto extend = [&] {
        s = std::min(p, std::max(2 * s, s + 8));
        ++out.extensions;
    };
    auto phase = [&](const char* what, Clock::time_point t0) {
        if (!cut_timing()) return;
        sync();
        std::fprintf(stderr, "[ttg]   %s (s=%lld): %.3f ms\n", what, (long long)s,
                     std::chrono::duration<double, std::milli>(Clock::now() - t0).count());
    };
    for (;;) {
        auto tp = Clock::now();
        e1.run_to(s);
        phase("pass 1", tp);
        tp = Clock::now();
        // Trailing mass of pass 1 = total mass of the R1 rows not yet computed. Tolerance
        // mode needs it exactly (the rank rule works at the budget^2 level, far below the
        // rounding noise of downdated norms), fixed rank only for the validity bound.
        double t1 = 0.0;
        bool exact = false;
        if (s < p) {
            if (!req.fixed) {
                PhaseTimer pt("refresh_exact");
                t1 = e1.refresh_exact();
                exact = true;
            } else {
                t1 = std::max(0.0, e1.trailing_mass());
            }
        }
        if (!req.fixed && s < p && t1 > b2) {  // no r <= s can meet the budget yet
            extend();
            continue;
        }
        phase("trailing mass", tp);
        tp = Clock::now();
        Pass2 p2 = run_pass2(e1, s, req.policy);
        phase("pass 2", tp);
        const std::vector<double>& hk = p2.kept;
        // total = kept[p] of the full factorisation = |R1[:s]|^2 + |R1[s:]|^2
        const double total = s == p ? hk[(size_t)s] : hk[(size_t)s] + t1;
        int64_t r;
        if (req.fixed) {
            r = req.rank;
        } else if (req.budget == 0.0) {  // pick_rank: eps == 0 keeps p
            if (s < p) { s = p; ++out.extensions; continue; }
            r = p;
        } else {  // pick_rank (factor.cpp:512-520) with the same target expression
            const double target = total - b2;
            r = -1;
            const int64_t hi = std::min(s, p - 1);
            for (int64_t c = 1; c <= hi; ++c)
                if (hk[(size_t)c] >= target) { r = c; break; }
            if (r < 0) {
                if (s == p) r = p;
                else { extend(); continue; }
            }
        }
        // Early-exit validity: every kept pass-2 pivot must dominate any unseen R1 row
        // (each has norm^2 <= t1), so the full factorisation picks the same pivots.
        if (s < p) {
            // The bound is exact (refreshed) or an over-estimate; the factor 4 absorbs the
            // rounding of the downdated pivot norms, which the 1e-16 guard keeps accurate.
            auto valid = [&](double bound) {
                const double slack = 4.0 * bound + 1e-300;
                for (int64_t t = 0; t < r; ++t)
                    if (!(p2.pnorm[(size_t)t] >= slack)) return false;
                return true;
            };
            bool ok = valid(t1);
            if (!ok && !exact) ok = valid(e1.refresh_exact());
            if (!ok) { extend(); continue; }
        }
        out.rank = r;
        out.steps = s;
        // Step error as the reference reports it: residual_from_mass (factor.cpp:507-510),
        // sqrt(max(0, kept[p] - kept[r])) with kept[p] the total above -- a subtraction that
        // cancels below ~1e-8 |A| (SURVEY finding 2; config 1 reports 0). The discarded mass
        // computed directly (discarded pass-2 columns plus the unseen R1 rows) is kept beside
        // it (report the reference value, log the direct one).
        double disc = t1;
        for (int64_t c = r; c < s; ++c) disc += p2.colmass[(size_t)c];
        out.direct_error = std::sqrt(std::max(0.0, disc));
        out.step_error = std::sqrt(std::max(0.0, total - hk[(size_t)r]));
        out.kept.assign(hk.begin(), hk.begin() + s + 1);
        out.kept.push_back(total);
        out.diag.assign(p2.diag.begin(), p2.diag.begin() + r);
        out.sel = std::move(p2.perm);
        return out;
    }
}

void check_refine(int refine) {
    if (refine < 0) argument_error("refine_passes must be >= 0");
    if (refine > 64) argument_error("refine_passes is unreasonably large");
}

int64_t product(const std::vector<int64_t>& v, size_t lo, size_t hi) {
    int64_t p = 1;
    for (size_t i = lo; i < hi; ++i) p *= v[i];
    return p;
}

void finish(TTResult& res, bool rss, Clock::time_point start) {
    double b = 0.0;
    for (double e : res.step_errors) b += rss ? e * e : e;
    res.bound = rss ? std::sqrt(b) : b;
    res.bound_kind = rss ? 0 : 1;
    sync();
    res.wall_ms = std::chrono::duration<double, std::milli>(Clock::now() - start).count();
}

// DecompConfig::debug_checks (tt_decomp.cpp:82-98): the carried matrix must equal the
// projection of the unfolding onto the kept factor, |carry - ref| <= 1e-10 |c|_F.
void debug_carry_check(const double* carry, const double* refm, int64_t count, const double* c, int64_t csize,
                       const char* where) {
    const double scale = std::sqrt(sum_squares(c, csize));
    const double dev = std::sqrt(diff_squares(carry, refm, count));
    if (dev > 1e-10 * scale) {
        char buf[256];
        std::snprintf(buf, sizeof buf, "%s: carried matrix deviates from the projected previous one by %.3e (allowed %.3e)",
                      where, dev, 1e-10 * scale);
        invariant_error(buf);
    }
}

void set_core(TTResult& res, size_t k, DevBuf<double>&& buf, int64_t r0, int64_t n, int64_t r1) {
    res.cores[k] = std::move(buf);
    res.core_dims[k] = {r0, n, r1};
}

// ---- general path: any method / sweep / refine_passes / retain -------------------------

// kept[j+1] = kept[j] + |L(:, j)|^2 over all p rows (column_mass, tt_decomp.cpp:102-109)
__global__ void k_colmass_full(const double* __restrict__ L, int64_t p, double* part, double* kept) {
    for (int64_t j = threadIdx.x; j < p; j += blockDim.x) {
        double a = 0.0;
        for (int64_t i = 0; i < p; ++i) a = __dadd_rn(a, __dmul_rn(L[i + j * p], L[i + j * p]));
        part[j] = a;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double acc = 0.0;
        kept[0] = 0.0;
        for (int64_t j = 0; j < p; ++j) {
            acc = __dadd_rn(acc, part[j]);
            kept[j + 1] = acc;
        }
    }
}

// B(i_d, ..., i_1) = A(i_1, ..., i_d) (reverse_indices, tensor_ops.cpp:128-143)
struct Dims64 {
    int d;
    int64_t n[32];
};
__global__ void k_reverse_indices(const double* __restrict__ A, Dims64 dims, int64_t total, double* B) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        // e indexes B, whose mode k is A's mode d-1-k; rebuild A's linear index
        int64_t rest = e, src = 0, stride_a[32];
        int64_t s = 1;
        for (int k = 0; k < dims.d; ++k) {
            stride_a[k] = s;
            s *= dims.n[k];
        }
        for (int k = 0; k < dims.d; ++k) {
            const int64_t nk = dims.n[dims.d - 1 - k];
            const int64_t ik = rest % nk;
            rest /= nk;
            src += ik * stride_a[dims.d - 1 - k];
        }
        B[e] = A[src];
    }
}

// out(b, i, a) = in(a, i, b): core of the reversed train (reverse_tt, tt.cpp:108-123)
__global__ void k_reverse_core(const double* __restrict__ in, int64_t rl, int64_t mid, int64_t rr, double* out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= rl * mid * rr) return;
    const int64_t a = e % rl, i = (e / rl) % mid, b = e / (rl * mid);
    out[b + i * rr + a * rr * mid] = in[e];
}

DevBuf<double> leading_block(const double* t, int64_t p, int64_t r) {
    DevBuf<double> o((size_t)(r * r));
    if (r > 0)
        TTG_CUDA(cudaMemcpy2DAsync(o.get(), sizeof(double) * r, t, sizeof(double) * p, sizeof(double) * r, r,
                                   cudaMemcpyDeviceToDevice, stream()));
    return o;
}

DevBuf<double> prefix(const double* x, int64_t count) {
    DevBuf<double> o((size_t)count);
    if (count > 0)
        TTG_CUDA(cudaMemcpyAsync(o.get(), x, sizeof(double) * count, cudaMemcpyDeviceToDevice, stream()));
    return o;
}

// One factorisation + truncation of a cut (factor level, any refine / method).
struct GenCut {
    int64_t r = 0;
    double res = 0.0;
    DevBuf<double> u1, t11, v1;  // m x r, r x r, n x r
    DMat fu, ft;                 // full U and T (kept for Alg. 4 full column)
};

GenCut general_cut(int method, const double* c, int64_t m, int64_t n, int refine, bool fixed, int64_t want,
                   double budget, bool keep_full) {
    GenCut g;
    const int64_t p = std::min(m, n);
    DMat u, t, v;
    int kind;
    DevBuf<double> sdev;
    if (method == 0) {
        DSvd f = svd(c, m, n, 60, 1e-14);
        kind = 0;
        sdev.alloc((size_t)p);
        sdev.upload(f.s.data(), (size_t)p);
        u = std::move(f.u);
        v = std::move(f.v);
    } else {
        DUtv f = utv(c, m, n, method == 1, refine);
        kind = method;
        u = std::move(f.u);
        t = std::move(f.t);
        v = std::move(f.v);
    }
    const double* tp = kind == 0 ? sdev.get() : t.get();
    const DTrunc tr = truncate_rank(kind, tp, p, fixed ? want : 0, budget);
    g.r = tr.rank;
    g.res = tr.residual;
    g.u1 = prefix(u.get(), m * g.r);
    g.v1 = prefix(v.get(), n * g.r);
    if (kind == 0) {
        std::vector<double> hs = sdev.to_host((size_t)p), d((size_t)(g.r * g.r), 0.0);
        for (int64_t i = 0; i < g.r; ++i) d[(size_t)(i + i * g.r)] = hs[(size_t)i];
        g.t11.alloc(d.size());
        g.t11.upload(d.data(), d.size());
    } else {
        g.t11 = leading_block(t.get(), p, g.r);
    }
    if (keep_full) {
        g.fu = std::move(u);
        g.ft = std::move(t);
    }
    return g;
}

void general_sweep(const double* a, const std::vector<int64_t>& dims, const SweepConfig& cfg, const Resolved& mode,
                   TTResult& res) {
    const int64_t d = (int64_t)dims.size();
    const int64_t total_n = product(dims, 0, dims.size());
    DevBuf<double> carry;
    if (cfg.sweep == 0) {  // sweep_l2r (tt_decomp.cpp:156-211) with svd or ulv
        const double* c = a;
        int64_t m = dims[0], n = total_n / dims[0], r_prev = 1;
        for (int64_t k = 1; k <= d - 1; ++k) {
            const int64_t p = std::min(m, n);
            int64_t want = 0;
            if (mode.fixed) {
                const int64_t req = mode.ranks[(size_t)k];
                want = std::min(req, p);
                if (want < req)
                    res.warnings.push_back("cut " + std::to_string(k) + ": requested rank " + std::to_string(req) +
                                           " clamped to " + std::to_string(want));
            }
            GenCut g = general_cut(cfg.method, c, m, n, cfg.refine, mode.fixed, want,
                                   mode.fixed ? 0.0 : mode.budgets[(size_t)(k - 1)], false);
            const int64_t r = g.r;
            res.step_errors[(size_t)(k - 1)] = g.res;
            res.ranks_chosen[(size_t)k] = r;
            res.cuts[(size_t)(k - 1)] = CutInfo{m, n, p, p, r, 0, {}};
            DevBuf<double> next((size_t)(r * n));
            gemm(false, true, r, n, r, g.t11.get(), r, g.v1.get(), n, next.get(), r);  // T11 V1^T (:192)
            if (cfg.debug) {
                DevBuf<double> refm((size_t)(r * n));
                gemm(true, false, r, n, m, g.u1.get(), m, c, m, refm.get(), r);
                debug_carry_check(next.get(), refm.get(), r * n, c, m * n, "left-to-right sweep");
            }
            set_core(res, (size_t)(k - 1), std::move(g.u1), r_prev, dims[(size_t)(k - 1)], r);
            r_prev = r;
            if (k < d - 1) {
                carry = std::move(next);
                c = carry.get();
                m = r * dims[(size_t)k];
                n = n / dims[(size_t)k];
            } else {
                set_core(res, (size_t)(d - 1), std::move(next), r, dims[(size_t)(d - 1)], 1);
            }
        }
        return;
    }
    // sweep_r2l (tt_decomp.cpp:216-339) with svd, urv or ulv (+ retain policy)
    const double* c = a;
    int64_t M = total_n / dims[(size_t)(d - 1)], n = dims[(size_t)(d - 1)], r_next = 1;
    const bool full_column = cfg.method == 1 && cfg.retain == 1;
    for (int64_t k = d; k >= 2; --k) {
        const int64_t p = std::min(M, n);
        int64_t want = 0;
        if (mode.fixed) {
            const int64_t req = mode.ranks[(size_t)(k - 1)];
            want = std::min(req, p);
            if (want < req)
                res.warnings.push_back("cut " + std::to_string(k - 1) + ": requested rank " + std::to_string(req) +
                                       " clamped to " + std::to_string(want));
        }
        const double budget = mode.fixed ? 0.0 : mode.budgets[(size_t)(k - 2)];
        int64_t r;
        double step_err;
        DevBuf<double> next, v1;
        if (full_column) {  // Alg. 4 keeping L(:, :r): carry = U L(:, :r) (:241-270)
            GenCut g = general_cut(1, c, M, n, cfg.refine, true, p, 0.0, true);
            DevBuf<double> part((size_t)p), kept((size_t)p + 1);
            TTG_LAUNCH(k_colmass_full, 1, 256, 0, stream(), g.ft.get(), p, part.get(), kept.get());
            const std::vector<double> hk = kept.to_host((size_t)p + 1);
            if (mode.fixed) {
                r = want;
            } else {
                r = p;
                if (budget > 0.0) {
                    const double target = hk[(size_t)p] - budget * budget;
                    for (int64_t cand = 1; cand < p; ++cand)
                        if (hk[(size_t)cand] >= target) { r = cand; break; }
                }
            }
            step_err = std::sqrt(std::max(0.0, hk[(size_t)p] - hk[(size_t)r]));
            next.alloc((size_t)(M * r));
            gemm(false, false, M, r, p, g.fu.get(), M, g.ft.get(), p, next.get(), M);
            v1 = prefix(g.v1.get(), n * r);
            if (cfg.debug) {
                DevBuf<double> refm((size_t)(M * r));
                gemm(false, false, M, r, n, c, M, v1.get(), n, refm.get(), M);
                debug_carry_check(next.get(), refm.get(), M * r, c, M * n, "right-to-left sweep (full column)");
            }
        } else {
            const bool coupling = cfg.debug && cfg.method == 1;  // ULV L11-only: L21 check
            GenCut g = general_cut(cfg.method, c, M, n, cfg.refine, mode.fixed, want, budget, coupling);
            r = g.r;
            step_err = g.res;
            next.alloc((size_t)(M * r));
            gemm(false, false, M, r, r, g.u1.get(), M, g.t11.get(), r, next.get(), M);  // U1 T11 (:302)
            v1 = std::move(g.v1);
            if (cfg.debug) {
                DevBuf<double> refm((size_t)(M * r));
                gemm(false, false, M, r, n, c, M, v1.get(), n, refm.get(), M);
                if (coupling) {
                    // the discarded coupling block is what the carry misses (tt_decomp.cpp:288-309)
                    DevBuf<double> part((size_t)p), kept((size_t)p + 1);
                    TTG_LAUNCH(k_colmass_full, 1, 256, 0, stream(), g.ft.get(), p, part.get(), kept.get());
                    const std::vector<double> ck = kept.to_host((size_t)p + 1);
                    const double l22 = ck[(size_t)p] - ck[(size_t)r];
                    const double l21 = std::sqrt(std::max(0.0, step_err * step_err - l22));
                    const double dev = std::sqrt(diff_squares(next.get(), refm.get(), M * r));
                    const double scale = std::sqrt(sum_squares(c, M * n));
                    if (std::abs(dev - l21) > 1e-10 * scale) {
                        char buf[256];
                        std::snprintf(buf, sizeof buf, "right-to-left sweep: carry deviation %.3e != coupling norm %.3e",
                                      dev, l21);
                        invariant_error(buf);
                    }
                } else {
                    debug_carry_check(next.get(), refm.get(), M * r, c, M * n, "right-to-left sweep");
                }
            }
        }
        res.step_errors[(size_t)(k - 2)] = step_err;
        res.ranks_chosen[(size_t)(k - 1)] = r;
        res.cuts[(size_t)(k - 2)] = CutInfo{M, n, p, p, r, 0, {}};
        DevBuf<double> core((size_t)(r * n));  // V1^T (core_from_left_unfolding, :77-80)
        transpose(v1.get(), n, r, n, core.get(), r);
        set_core(res, (size_t)(k - 1), std::move(core), r, dims[(size_t)(k - 1)], r_next);
        r_next = r;
        if (k > 2) {
            carry = std::move(next);
            c = carry.get();
            M = M / dims[(size_t)(k - 2)];
            n = dims[(size_t)(k - 2)] * r;
        } else {
            set_core(res, 0, std::move(next), 1, dims[0], r);
        }
    }
}

// ---- fast sweeps (refine_passes = 1), resumable at any cut ------------------------------

CutRequest make_request(TTResult& res, const Resolved& mode, const SweepConfig& cfg, int64_t cut, int64_t p) {
    CutRequest rq{mode.fixed, 0, 0.0, cfg.policy};
    if (mode.fixed) {
        const int64_t req = mode.ranks[(size_t)cut];
        rq.rank = std::min(req, p);
        if (rq.rank < req)
            res.warnings.push_back("cut " + std::to_string(cut) + ": requested rank " + std::to_string(req) +
                                   " clamped to " + std::to_string(rq.rank));
    } else {
        rq.budget = mode.budgets[(size_t)(cut - 1)];
    }
    return rq;
}

void print_cut(const char* what, int64_t cut, int64_t m, int64_t n, const CutOut& co, Clock::time_point t0) {
    if (!cut_timing()) return;
    sync();
    std::fprintf(stderr, "[ttg] %s cut %lld (%lld x %lld): %lld steps, %.3f ms\n", what, (long long)cut, (long long)m,
                 (long long)n, (long long)co.steps, std::chrono::duration<double, std::milli>(Clock::now() - t0).count());
}

// run_cut with the engine make_pass1 chose; a Gram-route result that is not well
// conditioned (R_ss / R_00 < 1e-4) is recomputed by the Householder engine.
CutOut cut_with(std::unique_ptr<Pass1>& e1, const CutRequest& rq, const double* W, int64_t k, int64_t N, int64_t ld,
                Layout l, int64_t cap) {
    CutOut co = run_cut(*e1, rq);
    if (auto* g = dynamic_cast<GramPass1*>(e1.get())) {
        const double ratio = g->diag_ratio();
        if (cut_timing())
            std::fprintf(stderr, "[ttg]   gram pass 1 (%lld x %lld, s=%lld): R_ss/R_00 = %.3e, %s\n", (long long)k,
                         (long long)N, (long long)co.steps, ratio, ratio >= 1e-4 ? "kept" : "redone");
        if (!(ratio >= 1e-4)) {
            e1 = std::make_unique<WidePass1>(W, k, N, ld, l, cap, nullptr, true);
            co = run_cut(*e1, rq);
        }
    }
    return co;
}

// TT-ULV left to right (tt_decomp.cpp:156-211) from cut k0 (1-based), c the m x n unfolding.
void ulv_cuts(TTResult& res, const double* c, int64_t m, int64_t n, int64_t k0, int64_t r_prev,
              const std::vector<int64_t>& dims, const Resolved& mode, const SweepConfig& cfg) {
    const int64_t d = (int64_t)dims.size();
    DevBuf<double> carry;  // current working matrix when not the input itself
    bool prev_near_full = false;
    for (int64_t k = k0; k <= d - 1; ++k) {
        const int64_t p = std::min(m, n);
        const CutRequest rq = make_request(res, mode, cfg, k, p);
        const auto tc0 = Clock::now();
        const int64_t cap = mode.fixed ? rq.rank : 32;
        auto e1 = make_pass1(c, m, n, m, Layout::Col, cap, mode.fixed, prev_near_full, cfg.policy);
        CutOut co = cut_with(e1, rq, c, m, n, m, Layout::Col, cap);
        print_cut("ulv", k, m, n, co, tc0);
        prev_near_full = co.rank * 10 >= p * 9;
        const int64_t r = co.rank;
        res.step_errors[(size_t)(k - 1)] = co.step_error;
        res.ranks_chosen[(size_t)k] = r;
        res.cuts[(size_t)(k - 1)] = CutInfo{m, n, p, co.steps, r, co.extensions, co.diag, co.direct_error, co.kept};
        DevBuf<double> core((size_t)(m * r));
        TTG_LAUNCH(k_gather_qcols, (int)cdiv(m * r, 256), 256, 0, stream(), e1->Q(), m, co.sel.get(), r, false,
                   core.get());
        set_core(res, (size_t)(k - 1), std::move(core), r_prev, dims[(size_t)(k - 1)], r);
        DevBuf<double> next((size_t)(r * n));
        dim3 g((unsigned)cdiv(n, 32), (unsigned)cdiv(r, 32));
        TTG_LAUNCH(k_carry_rows_t, g, dim3(32, 8), 0, stream(), e1->R(), n, co.sel.get(), r, next.get());
        if (cfg.debug) {  // carry = T11 V1^T against U1^T c (tt_decomp.cpp:193-196)
            DevBuf<double> refm((size_t)(r * n));
            gemm(true, false, r, n, m, res.cores[(size_t)(k - 1)].get(), m, c, m, refm.get(), r);
            debug_carry_check(next.get(), refm.get(), r * n, c, m * n, "left-to-right sweep");
        }
        r_prev = r;
        if (k < d - 1) {
            carry = std::move(next);
            c = carry.get();
            m = r * dims[(size_t)k];
            n = n / dims[(size_t)k];
        } else {
            set_core(res, (size_t)(d - 1), std::move(next), r, dims[(size_t)(d - 1)], 1);
        }
    }
}

// TT-URV right to left (tt_decomp.cpp:216-339) from cut index k0 (the core k0-1 is next),
// c the M x n unfolding.
void urv_cuts(TTResult& res, const double* c, int64_t M, int64_t n, int64_t k0, int64_t r_next,
              const std::vector<int64_t>& dims, const Resolved& mode, const SweepConfig& cfg) {
    DevBuf<double> carry;
    bool prev_near_full = false;
    for (int64_t k = k0; k >= 2; --k) {
        const int64_t p = std::min(M, n);
        const CutRequest rq = make_request(res, mode, cfg, k - 1, p);
        // W = c^T: k_W = n rows, N_W = M columns, W(i,j) = c[j + i*M].
        const auto tc0 = Clock::now();
        const int64_t cap = mode.fixed ? rq.rank : 32;
        auto e1 = make_pass1(c, n, M, M, Layout::Row, cap, mode.fixed, prev_near_full, cfg.policy);
        CutOut co = cut_with(e1, rq, c, n, M, M, Layout::Row, cap);
        print_cut("urv", k - 1, M, n, co, tc0);
        prev_near_full = co.rank * 10 >= p * 9;
        const int64_t r = co.rank;
        res.step_errors[(size_t)(k - 2)] = co.step_error;
        res.ranks_chosen[(size_t)(k - 1)] = r;
        res.cuts[(size_t)(k - 2)] = CutInfo{M, n, p, co.steps, r, co.extensions, co.diag, co.direct_error, co.kept};
        DevBuf<double> core((size_t)(n * r));
        TTG_LAUNCH(k_gather_qcols, (int)cdiv(n * r, 256), 256, 0, stream(), e1->Q(), n, co.sel.get(), r, true,
                   core.get());
        set_core(res, (size_t)(k - 1), std::move(core), r, dims[(size_t)(k - 1)], r_next);
        DevBuf<double> next((size_t)(M * r));
        dim3 g((unsigned)std::min<int64_t>(cdiv(M, 256), 4096), (unsigned)r);
        TTG_LAUNCH(k_carry_rows, g, 256, 0, stream(), e1->R(), M, co.sel.get(), r, next.get());
        if (cfg.debug) {  // carry = U1 T11 against c V1 (tt_decomp.cpp:310-317); the core is V1^T
            DevBuf<double> refm((size_t)(M * r));
            gemm(false, true, M, r, n, c, M, res.cores[(size_t)(k - 1)].get(), r, refm.get(), M);
            debug_carry_check(next.get(), refm.get(), M * r, c, M * n, "right-to-left sweep");
        }
        r_next = r;
        if (k > 2) {
            carry = std::move(next);
            c = carry.get();
            n = dims[(size_t)(k - 2)] * r;
            M = M / dims[(size_t)(k - 2)];
        } else {
            set_core(res, 0, std::move(next), 1, dims[0], r);
        }
    }
}

}  // namespace

TTResult decompose(const double* a, const std::vector<int64_t>& dims, const SweepConfig& cfg) {
    const auto start = Clock::now();
    const int64_t d = (int64_t)dims.size();
    if (d < 1) argument_error("train needs at least one core");
    for (size_t k = 0; k < dims.size(); ++k)
        if (dims[k] < 1)
            argument_error("shape dim " + std::to_string(k + 1) + " is " + std::to_string(dims[k]) + ", must be >= 1");
    const int64_t total_n = product(dims, 0, dims.size());
    // working set: the R1 rows / carry / exact-refresh residual of the first cut are each
    // at most about the input's size
    ensure_pool((size_t)(2.5 * 8.0 * (double)total_n) + ((size_t)256 << 20));
    if (cfg.method == 2 && cfg.sweep == 0) {
        // left_orthogonal_via_urv (tt_decomp.cpp:408-427): sweep the index-reversed tensor
        // right to left with the reversed rank chain / weights, then reverse the train.
        if (d > 32) argument_error("order above 32 is not supported by the device reversal");
        SweepConfig c2 = cfg;
        c2.sweep = 1;
        std::reverse(c2.ranks.begin(), c2.ranks.end());
        std::reverse(c2.weights.begin(), c2.weights.end());
        Dims64 dd{(int)d, {}};
        for (int64_t k = 0; k < d; ++k) dd.n[k] = dims[(size_t)k];
        DevBuf<double> rev((size_t)total_n);
        TTG_LAUNCH(k_reverse_indices, (int)std::min<int64_t>(cdiv(total_n, 256), (int64_t)sm_count() * 16), 256, 0,
                   stream(), a, dd, total_n, rev.get());
        TTResult r = decompose(rev.get(), std::vector<int64_t>(dims.rbegin(), dims.rend()), c2);
        TTResult out;
        out.dims = dims;
        out.cores.resize((size_t)d);
        out.core_dims.resize((size_t)d);
        for (int64_t k = 0; k < d; ++k) {
            const auto& cd = r.core_dims[(size_t)(d - 1 - k)];
            DevBuf<double> core((size_t)(cd[0] * cd[1] * cd[2]));
            TTG_LAUNCH(k_reverse_core, (int)cdiv(cd[0] * cd[1] * cd[2], 256), 256, 0, stream(),
                       r.cores[(size_t)(d - 1 - k)].get(), cd[0], cd[1], cd[2], core.get());
            set_core(out, (size_t)k, std::move(core), cd[2], cd[1], cd[0]);
        }
        out.step_errors.assign(r.step_errors.rbegin(), r.step_errors.rend());
        out.ranks_chosen.assign(r.ranks_chosen.rbegin(), r.ranks_chosen.rend());
        out.ranks_requested.assign(r.ranks_requested.rbegin(), r.ranks_requested.rend());
        out.cuts.assign(r.cuts.rbegin(), r.cuts.rend());
        out.bound = r.bound;
        out.bound_kind = r.bound_kind;
        out.input_norm = r.input_norm;
        out.warnings = r.warnings;
        out.warnings.push_back("left-orthogonal train built by sweeping the reversed tensor");
        sync();
        out.wall_ms = std::chrono::duration<double, std::milli>(Clock::now() - start).count();
        return out;
    }
    const bool plain = cfg.method == 1 && cfg.sweep == 1 && cfg.retain == 0;  // bound_kind_for
    const bool rss = !plain;

    TTResult res;
    res.dims = dims;
    res.cores.resize((size_t)d);
    res.core_dims.resize((size_t)d);
    const double norm_a = std::sqrt(sum_squares(a, total_n));
    const Resolved mode = resolve_mode(cfg, d, norm_a, rss);
    res.input_norm = norm_a;
    if (mode.fixed) res.ranks_requested = mode.ranks;

    if (norm_a == 0.0) {  // zero_input_result (tt_decomp.cpp:126-142)
        res.step_errors.assign((size_t)std::max<int64_t>(d - 1, 0), 0.0);
        res.ranks_chosen.assign((size_t)d + 1, 1);
        if (mode.fixed && *std::max_element(mode.ranks.begin(), mode.ranks.end()) > 1)
            res.warnings.push_back("input tensor is zero; all ranks clamped to 1");
        for (int64_t k = 0; k < d; ++k) {
            DevBuf<double> z((size_t)dims[(size_t)k]);
            z.zero();
            set_core(res, (size_t)k, std::move(z), 1, dims[(size_t)k], 1);
        }
        finish(res, rss, start);
        return res;
    }
    if (d == 1) {  // order_one_result
        res.ranks_chosen = {1, 1};
        DevBuf<double> c((size_t)total_n);
        TTG_CUDA(cudaMemcpyAsync(c.get(), a, sizeof(double) * total_n, cudaMemcpyDeviceToDevice, stream()));
        set_core(res, 0, std::move(c), 1, dims[0], 1);
        finish(res, rss, start);
        return res;
    }
    check_refine(cfg.refine);
    const bool fast = cfg.refine == 1 && ((cfg.method == 1 && cfg.sweep == 0) || (cfg.method == 2 && cfg.sweep == 1));

    res.step_errors.assign((size_t)(d - 1), 0.0);
    res.ranks_chosen.assign((size_t)d + 1, 1);
    res.cuts.resize((size_t)(d - 1));
    if (!fast) {
        general_sweep(a, dims, cfg, mode, res);
        finish(res, rss, start);
        return res;
    }

    if (cfg.method == 1) ulv_cuts(res, a, dims[0], total_n / dims[0], 1, 1, dims, mode, cfg);
    else urv_cuts(res, a, total_n / dims[(size_t)(d - 1)], dims[(size_t)(d - 1)], d, 1, dims, mode, cfg);
    finish(res, rss, start);
    return res;
}

}  // namespace ttg

namespace ttg {

ShardRange shard_range(const std::vector<int64_t>& dims, int method, int nranks, int rank) {
    const int64_t d = (int64_t)dims.size();
    if (d < 2) argument_error("sharded decomposition needs order >= 2");
    if (method != 1 && method != 2) argument_error("sharded decomposition supports ulv (l2r) and urv (r2l)");
    if (nranks < 1 || rank < 0 || rank >= nranks) argument_error("invalid rank / size");
    const int64_t total = product(dims, 0, dims.size());
    // ULV: the columns of c = A(i1; rest); URV: the rows of c = A(i1..i(d-1); id).
    const int64_t first = method == 1 ? dims[0] : dims[(size_t)(d - 1)];
    const int64_t count = total / first;
    if (count % nranks != 0)
        argument_error("sharded dimension " + std::to_string(count) + " is not divisible by " + std::to_string(nranks) +
                       " ranks");
    ShardRange r;
    const int64_t per = count / nranks;
    r.lo = per * rank;
    r.hi = r.lo + per;
    r.rows = method == 1 ? first : per;
    r.cols = method == 1 ? per : first;
    return r;
}

namespace {

// Global core (r2 x n', n' = i + I * q, I = dims[d-2]) from the ranks' transposed local
// cores (r2 x kl each, local row l = il + L q with il < L = I / G): rank g holds i in
// [g L, (g+1) L).
__global__ void k_core_from_shards(const double* __restrict__ parts, int G, int64_t r2, int64_t kl, int64_t L,
                                   int64_t I, double* out) {
    const int64_t total = (int64_t)G * kl * r2;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = e / (kl * r2), rem = e - g * kl * r2;
        const int64_t l = rem / r2, q2 = rem - l * r2;
        const int64_t il = l % L, q = l / L;
        const int64_t np = g * L + il + I * q;
        out[q2 + np * r2] = parts[e];
    }
}

}  // namespace

// Config 5's second URV cut without moving the carry: the previous cut's
// carry rows held by this rank are a row block of W' = c'^T (Row layout, ld M'), so pass 1
// runs as the pivoted Cholesky of the rank-summed Gram matrix (GramPass1 with the comm),
// pass 2 and the next carry are replicated, and only the core rows (k' x r, distributed)
// are all-gathered. Returns false (nothing done) when the cut does not qualify or the Gram
// route is not well conditioned; the caller then gathers the carry.
bool k_sharded_next(TTResult& res, const double* mine, int64_t Nl, int64_t Ng, int64_t r, Comm& comm,
                    const std::vector<int64_t>& dims, const Resolved& mode, const SweepConfig& cfg) {
    const int64_t d = (int64_t)dims.size();
    const int G = comm.size();
    const int64_t I = dims[(size_t)(d - 2)];
    const int64_t Mp = Ng / I;                 // M' = rows of c' = columns of W'
    if (Nl % Mp != 0) {  // each rank must hold whole i_{d-1} slices
        if (cut_timing()) std::fprintf(stderr, "[ttg]   k-sharded cut: %lld local rows not a multiple of %lld\n",
                                       (long long)Nl, (long long)Mp);
        return false;
    }
    const int64_t L = Nl / Mp, kl = L * r;     // local i_{d-1} range, local rows of W'
    const int64_t kg = I * r, p = std::min(kg, Mp);
    const CutRequest rq = make_request(res, mode, cfg, d - 2, p);
    if (!(kg >= 8 * Mp && Mp <= 4096 && rq.rank <= 160 && rq.rank >= 1)) {
        if (cut_timing())
            std::fprintf(stderr, "[ttg]   k-sharded cut not eligible (k' %lld, N' %lld, rank %lld)\n", (long long)kg,
                         (long long)Mp, (long long)rq.rank);
        return false;
    }
    const auto tc0 = Clock::now();
    GramPass1 gp(mine, kl, Mp, Mp, Layout::Row, &comm, rq.rank);
    CutOut co = run_cut(gp, rq);
    const double ratio = gp.diag_ratio();
    if (cut_timing())
        std::fprintf(stderr, "[ttg]   k-sharded gram pass 1 (%lld x %lld local rows %lld): R_ss/R_00 = %.3e\n",
                     (long long)kg, (long long)Mp, (long long)kl, ratio);
    if (!(ratio >= 1e-4)) return false;
    print_cut("urv(k-sharded)", d - 2, Mp, kg, co, tc0);
    const int64_t r2 = co.rank;
    res.step_errors[(size_t)(d - 3)] = co.step_error;
    res.ranks_chosen[(size_t)(d - 2)] = r2;
    res.cuts[(size_t)(d - 3)] = CutInfo{Mp, kg, p, co.steps, r2, co.extensions, co.diag, co.direct_error, co.kept};
    // core (r2 x I x r): local transposed core rows, all-gathered, scattered to n' order
    DevBuf<double> mineT((size_t)(kl * r2)), parts((size_t)(G * kl * r2)), core((size_t)(kg * r2));
    TTG_LAUNCH(k_gather_qcols, (int)cdiv(kl * r2, 256), 256, 0, stream(), gp.Q(), kl, co.sel.get(), r2, true,
               mineT.get());
    comm.allgather(mineT.get(), parts.get(), sizeof(double) * (size_t)(kl * r2));
    TTG_LAUNCH(k_core_from_shards, (int)std::min<int64_t>(cdiv(G * kl * r2, 256), 8 * sm_count()), 256, 0, stream(),
               parts.get(), G, r2, kl, L, I, core.get());
    set_core(res, (size_t)(d - 2), std::move(core), r2, I, r);
    // carry M' x r2 (replicated: R1 rows are replicated)
    DevBuf<double> next((size_t)(Mp * r2));
    dim3 g((unsigned)std::min<int64_t>(cdiv(Mp, 256), 4096), (unsigned)r2);
    TTG_LAUNCH(k_carry_rows, g, 256, 0, stream(), gp.R(), Mp, co.sel.get(), r2, next.get());
    if (d == 3) set_core(res, 0, std::move(next), 1, dims[0], r2);
    else urv_cuts(res, next.get(), Mp / dims[(size_t)(d - 3)], dims[(size_t)(d - 3)] * r2, d - 2, r2, dims, mode, cfg);
    return true;
}

TTResult decompose_sharded(const double* a_local, const std::vector<int64_t>& dims, const SweepConfig& cfg,
                           Comm& comm) {
    if (cfg.debug) argument_error("debug_checks is not supported by the column-sharded sweep");
    const auto start = Clock::now();
    const int64_t d = (int64_t)dims.size();
    for (size_t k = 0; k < dims.size(); ++k)
        if (dims[k] < 1)
            argument_error("shape dim " + std::to_string(k + 1) + " is " + std::to_string(dims[k]) + ", must be >= 1");
    const bool ulv = cfg.method == 1 && cfg.sweep == 0, urv = cfg.method == 2 && cfg.sweep == 1;
    if (!ulv && !urv) argument_error("sharded decomposition supports ulv (l2r) and urv (r2l)");
    check_refine(cfg.refine);
    if (cfg.refine != 1) argument_error("sharded decomposition supports refine_passes = 1");
    const int G = comm.size();
    const ShardRange sr = shard_range(dims, cfg.method, G, comm.rank());
    const int64_t local_n = sr.rows * sr.cols;
    ensure_pool((size_t)(4.5 * 8.0 * (double)local_n) + ((size_t)256 << 20));
    const bool rss = !(cfg.method == 1 && cfg.sweep == 1 && cfg.retain == 0);

    TTResult res;
    res.dims = dims;
    res.cores.resize((size_t)d);
    res.core_dims.resize((size_t)d);
    // |A|_F: local blocked sums, combined in rank order
    const double norm_a = std::sqrt(global_sum(comm, sum_squares(a_local, local_n)));
    if (cut_timing())
        std::fprintf(stderr, "[ttg] sharded norm: %.3f ms\n",
                     std::chrono::duration<double, std::milli>(Clock::now() - start).count());
    const Resolved mode = resolve_mode(cfg, d, norm_a, rss);
    res.input_norm = norm_a;
    if (mode.fixed) res.ranks_requested = mode.ranks;
    res.step_errors.assign((size_t)(d - 1), 0.0);
    res.ranks_chosen.assign((size_t)d + 1, 1);
    res.cuts.resize((size_t)(d - 1));
    if (norm_a == 0.0) {  // zero_input_result (tt_decomp.cpp:126-142)
        if (mode.fixed && *std::max_element(mode.ranks.begin(), mode.ranks.end()) > 1)
            res.warnings.push_back("input tensor is zero; all ranks clamped to 1");
        for (int64_t k = 0; k < d; ++k) {
            DevBuf<double> z((size_t)dims[(size_t)k]);
            z.zero();
            set_core(res, (size_t)k, std::move(z), 1, dims[(size_t)k], 1);
        }
        res.cuts.clear();
        finish(res, rss, start);
        return res;
    }

    // First cut, sharded: W = c (ULV, columns of c) or c^T (URV, rows of c).
    const int64_t cut = ulv ? 1 : d - 1;
    const int64_t kW = ulv ? dims[0] : dims[(size_t)(d - 1)];
    const int64_t Nl = sr.hi - sr.lo, Ng = Nl * G;
    const int64_t p = std::min(kW, Ng);
    const CutRequest rq = make_request(res, mode, cfg, cut, p);
    const auto tc0 = Clock::now();
    ShardSpec spec{&comm, sr.lo, Ng};
    WidePass1 e1(a_local, kW, Nl, ulv ? kW : Nl, ulv ? Layout::Col : Layout::Row, mode.fixed ? rq.rank : 32, &spec);
    CutOut co = run_cut(e1, rq);
    print_cut(ulv ? "ulv(sharded)" : "urv(sharded)", cut, ulv ? kW : Ng, ulv ? Ng : kW, co, tc0);
    const int64_t r = co.rank;
    res.step_errors[(size_t)(cut - 1)] = co.step_error;
    res.ranks_chosen[(size_t)cut] = r;
    res.cuts[(size_t)(cut - 1)] = ulv ? CutInfo{kW, Ng, p, co.steps, r, co.extensions, co.diag, co.direct_error, co.kept}
                                      : CutInfo{Ng, kW, p, co.steps, r, co.extensions, co.diag, co.direct_error, co.kept};
    // the core from the replicated Q; the local carry block, then the all-gathered carry
    DevBuf<double> core((size_t)(kW * r));
    TTG_LAUNCH(k_gather_qcols, (int)cdiv(kW * r, 256), 256, 0, stream(), e1.Q(), kW, co.sel.get(), r, !ulv,
               core.get());
    DevBuf<double> mine((size_t)(Nl * r)), all((size_t)(Ng * r));
    if (ulv) {
        set_core(res, 0, std::move(core), 1, dims[0], r);
        dim3 g((unsigned)cdiv(Nl, 32), (unsigned)cdiv(r, 32));
        TTG_LAUNCH(k_carry_rows_t, g, dim3(32, 8), 0, stream(), e1.R(), Nl, co.sel.get(), r, mine.get());
        // rank blocks of r x Nl are the column blocks of the r x Ng carry: no repack
        comm.allgather(mine.get(), all.get(), sizeof(double) * (size_t)(Nl * r));
        if (d == 2) set_core(res, 1, std::move(all), r, dims[1], 1);
        else ulv_cuts(res, all.get(), r * dims[1], Ng / dims[1], 2, r, dims, mode, cfg);
    } else {
        set_core(res, (size_t)(d - 1), std::move(core), r, dims[(size_t)(d - 1)], 1);
        dim3 g((unsigned)std::min<int64_t>(cdiv(Nl, 256), 4096), (unsigned)r);
        TTG_LAUNCH(k_carry_rows, g, 256, 0, stream(), e1.R(), Nl, co.sel.get(), r, mine.get());
        if (d >= 3 && mode.fixed && k_sharded_next(res, mine.get(), Nl, Ng, r, comm, dims, mode, cfg)) {
            finish(res, rss, start);
            return res;
        }
        DevBuf<double> gathered((size_t)(Ng * r));
        if (cut_timing()) {
            sync();
            std::fprintf(stderr, "[ttg] carry rows + allocs: %.3f ms since the cut began\n",
                         std::chrono::duration<double, std::milli>(Clock::now() - tc0).count());
        }
        comm.allgather(mine.get(), gathered.get(), sizeof(double) * (size_t)(Nl * r));
        if (cut_timing()) {
            sync();
            std::fprintf(stderr, "[ttg] carry allgather: %.3f ms since the cut began\n",
                         std::chrono::duration<double, std::milli>(Clock::now() - tc0).count());
        }
        // rank g's Nl x r block -> rows [g Nl, (g+1) Nl) of the Ng x r carry
        for (int q = 0; q < G; ++q)
            TTG_CUDA(cudaMemcpy2DAsync(all.get() + (int64_t)q * Nl, sizeof(double) * Ng,
                                       gathered.get() + (int64_t)q * Nl * r, sizeof(double) * Nl, sizeof(double) * Nl,
                                       r, cudaMemcpyDeviceToDevice, stream()));
        if (cut_timing()) {
            sync();
            std::fprintf(stderr, "[ttg] carry gather: %.3f ms since the cut began\n",
                         std::chrono::duration<double, std::milli>(Clock::now() - tc0).count());
        }
        if (d == 2) set_core(res, 0, std::move(all), 1, dims[0], r);
        else urv_cuts(res, all.get(), Ng / dims[(size_t)(d - 2)], dims[(size_t)(d - 2)] * r, d - 1, r, dims, mode, cfg);
    }
    finish(res, rss, start);
    return res;
}

}  // namespace ttg
