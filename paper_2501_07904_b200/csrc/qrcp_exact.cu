// Bitwise pass 1 for narrow W (k <= 32 rows): the reference's qr_col_pivot
// (src/factor.cpp:62-135) reproduced operation for operation, on a working copy of W.
//
// Why: at a prescribed accuracy below half an ulp of the kept mass (BASELINE config 2:
// eps_k^2 = 2.5e-17 |A|^2), the rank rule kept[r] >= kept[p] - eps^2 (factor.cpp:512-520)
// is decided by which of the noise-level rows of the triangular factor still move the
// rounded running sum. A noise row's mass is set by pass 1's own rounding residue (the rows
// of R1 past the numerical rank), and a row moves the sum iff its mass exceeds half an ulp of
// the running total -- independent of the total's last bits. So when R1 is bitwise the
// reference's, the pass-2 factor's noise-row masses agree with the reference's to ~1e-14
// relative and the chosen rank is the reference's (barring a mass within ~1e-14 of the
// threshold). The read-only WY engine computes the same R1 in exact arithmetic but with
// different rounding residue, hence other noise rows and another ulp-decided rank.
//
// Per column every operation is the reference's: sequential sums (sum_squares_serial and the
// reflector dot), products and sums rounded separately (no FMA: __dmul_rn / __dadd_rn), the
// dlarfg-convention reflector with its exact formulas, the downdate with the 1e-16 recompute
// guard from the updated trailing rows, and the position bookkeeping of the column swaps
// (ties go to the lowest position). The working copy is stored by rows (work[i * N + j]) so
// that a thread owning a column reads and writes coalesced.
#include <cmath>

#include "engine.hpp"

namespace ttg {
namespace {

constexpr int kEx = 32;  // largest k
constexpr int kExThreads = 256;

struct ExStep {  // the step record k_ex_pick leaves for k_ex_apply
    int64_t jp, ct, pp;
    double beta;
    double v[kEx];  // v[0] = 1 (implicit); v[1..len-1] the scaled reflector
};

__device__ __forceinline__ double dsq(double x) { return __dmul_rn(x, x); }

__global__ void __launch_bounds__(kExThreads) k_ex_init(const double* __restrict__ W, int64_t k, int64_t N,
                                                        int64_t ld, int layout, double* work, double* cn,
                                                        double* cr, int64_t* pos, int64_t* perm, Cand* cand) {
    __shared__ Cand sc[kExThreads / 32];
    Cand best = cand_none();
    for (int64_t j = (int64_t)blockIdx.x * kExThreads + threadIdx.x; j < N; j += (int64_t)gridDim.x * kExThreads) {
        double s = 0.0;
        for (int64_t i = 0; i < k; ++i) {
            const double x = layout == 0 ? W[i + j * ld] : W[i * ld + j];
            work[i * N + j] = x;
            s = __dadd_rn(s, dsq(x));  // sum_squares_serial (kernels.cpp:78-82)
        }
        cn[j] = s;
        cr[j] = s;
        pos[j] = j;
        perm[j] = j;
        const Cand c{s, j, j};
        if (better(c, best)) best = c;
    }
    best = block_best(best, sc);
    if (threadIdx.x == 0) cand[blockIdx.x] = best;
}

// One CTA: the pivot of step t (largest norm, lowest position: factor.cpp:85-87), the swap
// bookkeeping (:88-93), and make_householder on the pivot column (:24-38).
__global__ void __launch_bounds__(kExThreads) k_ex_pick(double* work, int64_t k, int64_t N, int64_t t,
                                                        const Cand* __restrict__ cand, int ncand, int64_t* pos,
                                                        int64_t* perm, double* betas, double* diag, ExStep* st) {
    __shared__ Cand sc[kExThreads / 32];
    Cand best = cand_none();
    for (int i = threadIdx.x; i < ncand; i += kExThreads)
        if (better(cand[i], best)) best = cand[i];
    best = block_best(best, sc);
    if (threadIdx.x != 0) return;
    const int64_t ct = perm[t];
    // no comparable candidate (NaN norms): the strict '>' scan keeps the column at position t
    const int64_t jp = best.col >= 0 ? best.col : ct;
    const int64_t pp = best.col >= 0 ? best.pos : t;
    perm[t] = jp;
    perm[pp] = ct;
    pos[jp] = t;
    pos[ct] = pp;
    const int64_t len = k - t;
    double x[kEx];
    for (int64_t i = 0; i < len; ++i) x[i] = work[(t + i) * N + jp];
    double beta = 0.0;
    if (len > 1) {
        double sigma = 0.0;
        for (int64_t i = 1; i < len; ++i) sigma = __dadd_rn(sigma, dsq(x[i]));
        const double alpha = x[0];
        if (sigma != 0.0) {
            const double mu = __dsqrt_rn(__dadd_rn(dsq(alpha), sigma));
            const double smu = copysign(mu, alpha);
            const double v0 = __dadd_rn(alpha, smu);
            beta = __ddiv_rn(dsq(v0), __dmul_rn(smu, v0));
            for (int64_t i = 1; i < len; ++i) x[i] = __ddiv_rn(x[i], v0);
            x[0] = -smu;
        }
    }
    for (int64_t i = 0; i < len; ++i) work[(t + i) * N + jp] = x[i];
    betas[t] = beta;
    diag[t] = x[0];
    st->jp = jp;
    st->ct = ct;
    st->pp = pp;
    st->beta = beta;
    st->v[0] = 1.0;
    for (int64_t i = 1; i < len; ++i) st->v[i] = x[i];
}

// apply_reflector (factor.cpp:43-58) to every column at a position > t, then the downdate and
// guard (:96-107), and the candidates of step t+1.
template <int KM>
__global__ void __launch_bounds__(kExThreads) k_ex_apply(double* work, int64_t k, int64_t N, int64_t t,
                                                         const ExStep* __restrict__ stp, const int64_t* pos,
                                                         double* cn, double* cr, Cand* cand) {
    __shared__ Cand sc[kExThreads / 32];
    __shared__ double v[KM];
    __shared__ double beta_s;
    __shared__ int64_t jps, cts, pps;
    if (threadIdx.x < KM) v[threadIdx.x] = threadIdx.x < k - t ? stp->v[threadIdx.x] : 0.0;
    if (threadIdx.x == 0) {
        beta_s = stp->beta;
        jps = stp->jp;
        cts = stp->ct;
        pps = stp->pp;
    }
    __syncthreads();
    const double beta = beta_s;
    const int64_t jp = jps, ct = cts, pp = pps;
    const int len = (int)(k - t);
    Cand best = cand_none();
    for (int64_t j = (int64_t)blockIdx.x * kExThreads + threadIdx.x; j < N; j += (int64_t)gridDim.x * kExThreads) {
        if (j == jp) continue;
        const int64_t pj = j == ct ? pp : pos[j];
        if (pj <= t) continue;
        double c[KM];
#pragma unroll
        for (int i = 0; i < KM; ++i) c[i] = i < len ? work[(t + i) * N + j] : 0.0;
        if (beta != 0.0) {
            double tt = c[0];
#pragma unroll
            for (int i = 1; i < KM; ++i)
                if (i < len) tt = __dadd_rn(tt, __dmul_rn(v[i], c[i]));
            tt = __dmul_rn(tt, beta);
            c[0] = __dsub_rn(c[0], tt);
#pragma unroll
            for (int i = 1; i < KM; ++i)
                if (i < len) c[i] = __dsub_rn(c[i], __dmul_rn(tt, v[i]));
#pragma unroll
            for (int i = 0; i < KM; ++i)
                if (i < len) work[(t + i) * N + j] = c[i];
        }
        double nv = __dsub_rn(cn[j], dsq(c[0]));
        double rv = cr[j];
        if (nv < __dmul_rn(1e-16, rv) || nv < 0.0) {
            double s = 0.0;
#pragma unroll
            for (int i = 1; i < KM; ++i)
                if (i < len) s = __dadd_rn(s, dsq(c[i]));
            nv = s;
            rv = s;
            cr[j] = rv;
        }
        cn[j] = nv;
        const Cand cd{nv, pj, j};
        if (better(cd, best)) best = cd;
    }
    best = block_best(best, sc);
    if (threadIdx.x == 0) cand[blockIdx.x] = best;
}

// R1 rows 0..s-1 by original column (row t at R + t N): work(t, j) for columns at positions
// >= t (the pivot of step t holds R(t, t)), 0 for columns pivoted before step t.
__global__ void k_ex_rrows(const double* __restrict__ work, int64_t N, int64_t s, const int64_t* __restrict__ pos,
                           double* R) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < s * N; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = e / N, j = e - t * N;
        R[e] = pos[j] >= t ? work[t * N + j] : 0.0;
    }
}

// Economy Q columns 0..s-1 (k x s, ld k) by the reference's backward accumulation
// (factor.cpp:116-133); column j only meets reflectors 0..j (the later ones leave e_j
// untouched bitwise).
__global__ void k_ex_q(const double* __restrict__ work, int64_t k, int64_t N, int64_t s,
                       const int64_t* __restrict__ perm, const double* __restrict__ betas, double* Q) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= s) return;
    double c[kEx];
    for (int64_t i = 0; i < k; ++i) c[i] = i == j ? 1.0 : 0.0;
    for (int64_t kk = j; kk >= 0; --kk) {
        const double b = betas[kk];
        if (b == 0.0) continue;
        const int64_t col = perm[kk];
        const int64_t len = k - kk;
        double tt = c[kk];
        for (int64_t i = 1; i < len; ++i) tt = __dadd_rn(tt, __dmul_rn(work[(kk + i) * N + col], c[kk + i]));
        tt = __dmul_rn(tt, b);
        c[kk] = __dsub_rn(c[kk], tt);
        for (int64_t i = 1; i < len; ++i) c[kk + i] = __dsub_rn(c[kk + i], __dmul_rn(tt, work[(kk + i) * N + col]));
    }
    for (int64_t i = 0; i < k; ++i) Q[i + j * k] = c[i];
}

// Exact trailing mass: rows s.. of the updated columns at positions >= s (per-CTA partials).
__global__ void __launch_bounds__(kExThreads) k_ex_mass(const double* __restrict__ work, int64_t k, int64_t N,
                                                        int64_t s, const int64_t* __restrict__ pos, double* part) {
    __shared__ double sd[kExThreads / 32];
    double a = 0.0;
    for (int64_t j = (int64_t)blockIdx.x * kExThreads + threadIdx.x; j < N; j += (int64_t)gridDim.x * kExThreads)
        if (pos[j] >= s)
            for (int64_t i = s; i < k; ++i) a = fma(work[i * N + j], work[i * N + j], a);
    a = block_sum(a, sd);
    if (threadIdx.x == 0) part[blockIdx.x] = a;
}

}  // namespace

ExactQrcp::ExactQrcp(const double* W, int64_t k, int64_t N, int64_t ld, Layout layout)
    : k_(k), N_(N), p_(std::min(k, N)) {
    if (k > kEx) argument_error("exact pass 1 supports at most 32 rows");
    grid_ = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(N, kExThreads), (int64_t)sm_count() * 8));
    work_.alloc((size_t)(k * N));
    cn_.alloc((size_t)N);
    cr_.alloc((size_t)N);
    pos_.alloc((size_t)N);
    perm_.alloc((size_t)N);
    cand_.alloc((size_t)(2 * grid_) * (sizeof(Cand) / sizeof(double)));
    betas_.alloc((size_t)p_);
    diag_.alloc((size_t)p_);
    step_.alloc(sizeof(ExStep) / sizeof(double) + 1);
    TTG_LAUNCH(k_ex_init, grid_, kExThreads, 0, stream(), W, k, N, ld, (int)layout, work_.get(), cn_.get(),
               cr_.get(), pos_.get(), perm_.get(), reinterpret_cast<Cand*>(cand_.get()));
}

void ExactQrcp::run_to(int64_t s) {
    s = std::min(s, p_);
    Cand* cand = reinterpret_cast<Cand*>(cand_.get());
    ExStep* st = reinterpret_cast<ExStep*>(step_.get());
    for (; steps_ < s; ++steps_) {
        const int64_t t = steps_;
        Cand* in = cand + (t & 1) * grid_;
        Cand* out = cand + ((t + 1) & 1) * grid_;
        TTG_LAUNCH(k_ex_pick, 1, kExThreads, 0, stream(), work_.get(), k_, N_, t, in, grid_, pos_.get(), perm_.get(),
                   betas_.get(), diag_.get(), st);
        prof_begin();
        if (k_ <= 16)
            TTG_LAUNCH(k_ex_apply<16>, grid_, kExThreads, 0, stream(), work_.get(), k_, N_, t, st, pos_.get(),
                       cn_.get(), cr_.get(), out);
        else
            TTG_LAUNCH(k_ex_apply<32>, grid_, kExThreads, 0, stream(), work_.get(), k_, N_, t, st, pos_.get(),
                       cn_.get(), cr_.get(), out);
        prof_end(8.0 * (double)(N_ - t) * (2.0 * (double)(k_ - t) + 3.0),
                 "k_ex_apply (bitwise qr_col_pivot step, k <= 32: reflector + downdate + guard)");
    }
}

double ExactQrcp::trailing_mass_exact() {
    DevBuf<double> part((size_t)grid_);
    TTG_LAUNCH(k_ex_mass, grid_, kExThreads, 0, stream(), work_.get(), k_, N_, steps_, pos_.get(), part.get());
    const std::vector<double> h = part.to_host((size_t)grid_);
    double s = 0.0;
    for (double v : h) s += v;
    return s;
}

void ExactQrcp::r_rows(double* R, int64_t s) const {
    TTG_LAUNCH(k_ex_rrows, (int)std::min<int64_t>(cdiv(s * N_, 256), (int64_t)sm_count() * 16), 256, 0, stream(),
               work_.get(), N_, s, pos_.get(), R);
}

void ExactQrcp::form_q(double* Q, int64_t s) const {
    TTG_LAUNCH(k_ex_q, (int)cdiv(s, 32), 32, 0, stream(), work_.get(), k_, N_, s, perm_.get(), betas_.get(), Q);
}

// ===========================================================================================
// Bitwise pass 2: the reference's qr_col_pivot of the tall B = R1^T (N x s, s <= 32; the
// reference's `middle` = transpose(R1) with rows in pass-1 position order, factor.cpp:349-359)
// reproduced operation for operation. Its sums run over all N rows in order (sum_squares_serial,
// make_householder's sigma, apply_reflector's dot), so they are sequential chains: one warp per
// chain streams its column(s) through shared memory with cp.async while lane 0 accumulates in
// order. Everything else (scaling by 1/v0, the axpy updates) is elementwise and parallel.
// It is the engine of the "bitwise" QLP policy (TTG_QLP_BITWISE), under which a cut whose rank
// is decided by rounding (BASELINE config 2) picks the reference's rank: that rank depends on the
// pass-2 pivot order among the noise-level rows, itself set by pass 2's rounding.
// ===========================================================================================
namespace {

constexpr int kChainTile = 512;   // elements per operand per stage
constexpr int kChainStages = 3;

struct ChainSpec {      // chain c: out[c] = init[c] + sum_{i < len} a_c[i] * b_c[i] (b = a: squares)
    int64_t col[kEx];   // physical column of operand a in `work` (ld N)
    int64_t bcol;       // physical column of operand b (dots) or -1 (sum of squares)
    int64_t r0, len;    // rows [r0, r0 + len)
    int n;              // number of chains
    double init[kEx];
    double out[kEx];
};

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}

// One warp per chain: all 32 lanes copy tiles of the operands into a shared-memory ring
// (cp.async, in flight while lane 0 works), lane 0 adds the products in row order.
__global__ void __launch_bounds__(32) k_chain(const double* __restrict__ work, int64_t N, ChainSpec* sp) {
    __shared__ __align__(16) double ta[kChainStages][kChainTile];
    __shared__ __align__(16) double tb[kChainStages][kChainTile];
    const int c = blockIdx.x;
    if (c >= sp->n) return;
    const int lane = threadIdx.x;
    const bool sq = sp->bcol < 0;
    const double* a = work + sp->col[c] * N + sp->r0;
    const double* b = sq ? a : work + sp->bcol * N + sp->r0;
    const int64_t len = sp->len;
    const int64_t ntile = (len + kChainTile - 1) / kChainTile;
    auto issue = [&](int64_t tile) {
        const int st = (int)(tile % kChainStages);
        const int64_t base = tile * kChainTile;
        for (int e = lane; e < kChainTile; e += 32) {
            const int64_t i = base + e;
            if (i < len) {
                cp_async8(&ta[st][e], a + i);
                if (!sq) cp_async8(&tb[st][e], b + i);
            }
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    for (int64_t tl = 0; tl < kChainStages - 1; ++tl) {
        if (tl < ntile) issue(tl);
        else asm volatile("cp.async.commit_group;\n" ::);
    }
    double s = sp->init[c];
    for (int64_t tile = 0; tile < ntile; ++tile) {
        asm volatile("cp.async.wait_group %0;\n" ::"n"(kChainStages - 2));
        __syncwarp();
        const int64_t nxt = tile + kChainStages - 1;
        if (nxt < ntile) issue(nxt);
        else asm volatile("cp.async.commit_group;\n" ::);
        if (lane == 0) {
            const int st = (int)(tile % kChainStages);
            const int64_t cnt = min((int64_t)kChainTile, len - tile * kChainTile);
            const double* x = ta[st];
            const double* y = sq ? ta[st] : tb[st];
#pragma unroll 8
            for (int64_t e = 0; e < cnt; ++e) s = __dadd_rn(s, __dmul_rn(x[e], y[e]));
        }
        __syncwarp();
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
    if (lane == 0) sp->out[c] = s;
}

struct TallState {          // bookkeeping of the bitwise tall QRCP (device)
    int64_t colmap[kEx];    // position -> physical column of work
    int64_t perm[kEx];      // position -> original column (the reference's perm)
    double cn[kEx], cr[kEx];  // cnorm2 / cref2 by position
    double beta[kEx], v0, smu;
    int64_t jp;             // physical pivot column of the current step
    int pivot_ok;           // beta != 0 this step
    int nflag;
    int flagpos[kEx];
};

__global__ void k_et_init(TallState* st, ChainSpec* sp, int s, int64_t N) {
    for (int q = 0; q < s; ++q) {
        st->colmap[q] = q;
        st->perm[q] = q;
        sp->col[q] = q;
        sp->init[q] = 0.0;
    }
    sp->bcol = -1;
    sp->r0 = 0;
    sp->len = N;
    sp->n = s;
}

__global__ void k_et_norms(TallState* st, const ChainSpec* sp, int s) {
    for (int q = 0; q < s; ++q) st->cn[q] = st->cr[q] = sp->out[q];
}

// pivot (factor.cpp:85-93) and the sigma chain of make_householder (:28-29)
__global__ void k_et_pick(TallState* st, ChainSpec* sp, int s, int64_t N, int k, double* pnorm) {
    int piv = k;
    for (int j = k + 1; j < s; ++j)
        if (st->cn[j] > st->cn[piv]) piv = j;
    if (piv != k) {
        int64_t t64 = st->colmap[k]; st->colmap[k] = st->colmap[piv]; st->colmap[piv] = t64;
        t64 = st->perm[k]; st->perm[k] = st->perm[piv]; st->perm[piv] = t64;
        double td = st->cn[k]; st->cn[k] = st->cn[piv]; st->cn[piv] = td;
        td = st->cr[k]; st->cr[k] = st->cr[piv]; st->cr[piv] = td;
    }
    pnorm[k] = st->cn[k];
    st->jp = st->colmap[k];
    sp->col[0] = st->jp;
    sp->bcol = -1;
    sp->r0 = k + 1;
    sp->len = N - k - 1;
    sp->init[0] = 0.0;
    sp->n = N - k > 1 ? 1 : 0;
}

// make_householder's scalars (:30-37) from sigma; then the dot chains of apply_reflector (:50-51)
__global__ void k_et_house(double* work, TallState* st, ChainSpec* sp, int s, int64_t N, int k) {
    const int64_t jp = st->jp;
    const int64_t len = N - k;
    double* x = work + jp * N + k;
    double beta = 0.0;
    st->pivot_ok = 0;
    if (len > 1) {
        const double sigma = sp->out[0];
        const double alpha = x[0];
        if (sigma != 0.0) {
            const double mu = __dsqrt_rn(__dadd_rn(dsq(alpha), sigma));
            const double smu = copysign(mu, alpha);
            const double v0 = __dadd_rn(alpha, smu);
            beta = __ddiv_rn(dsq(v0), __dmul_rn(smu, v0));
            st->v0 = v0;
            st->smu = smu;
            st->pivot_ok = 1;
        }
    }
    st->beta[k] = beta;
    // dot chains for the columns at positions k+1.. (only when the reflector is non-trivial)
    int n = 0;
    if (beta != 0.0)
        for (int q = k + 1; q < s; ++q) {
            const int64_t cj = st->colmap[q];
            sp->col[n] = cj;
            sp->init[n] = work[cj * N + k];
            ++n;
        }
    sp->bcol = jp;
    sp->r0 = k + 1;
    sp->len = N - k - 1;
    sp->n = n;
}

// x[i] /= v0 (i >= 1) and x[0] = -copysign(mu, alpha) on the pivot column
__global__ void k_et_scale(double* work, const TallState* st, int64_t N, int k) {
    if (!st->pivot_ok) return;
    double* x = work + st->jp * N + k;
    const double v0 = st->v0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; i < N - k; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = __ddiv_rn(x[i], v0);
    if (blockIdx.x == 0 && threadIdx.x == 0) x[0] = -st->smu;
}

// c[0] -= t, c[i] -= t v[i] with t = dot * beta, for every column of this step's dot chains
__global__ void k_et_update(double* work, const TallState* st, const ChainSpec* sp, int64_t N, int k) {
    const int nc = sp->n;
    if (nc == 0) return;
    const double beta = st->beta[k];
    const double* v = work + st->jp * N + k;
    for (int c = 0; c < nc; ++c) {
        double* col = work + sp->col[c] * N + k;
        const double t = __dmul_rn(sp->out[c], beta);
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N - k; i += (int64_t)gridDim.x * blockDim.x)
            col[i] = i == 0 ? __dsub_rn(col[0], t) : __dsub_rn(col[i], __dmul_rn(t, v[i]));
    }
}

// downdate + guard flags (:96-107); the recompute chains are set up for the flagged positions
__global__ void k_et_downdate(const double* work, TallState* st, ChainSpec* sp, int s, int64_t N, int k) {
    int n = 0;
    for (int q = k + 1; q < s; ++q) {
        const int64_t cj = st->colmap[q];
        const double r = work[cj * N + k];
        const double nv = __dsub_rn(st->cn[q], dsq(r));
        st->cn[q] = nv;
        if (nv < __dmul_rn(1e-16, st->cr[q]) || nv < 0.0) {
            st->flagpos[n] = q;
            sp->col[n] = cj;
            sp->init[n] = 0.0;
            ++n;
        }
    }
    st->nflag = n;
    sp->bcol = -1;
    sp->r0 = k + 1;
    sp->len = N - k - 1;
    sp->n = n;
}

__global__ void k_et_guard_done(TallState* st, const ChainSpec* sp) {
    for (int f = 0; f < st->nflag; ++f) {
        const int q = st->flagpos[f];
        st->cn[q] = st->cr[q] = sp->out[f];
    }
}

// R (s x s over positions, col-major ld s) and the permutation
__global__ void k_et_out(const double* work, const TallState* st, int s, int64_t N, double* R, int64_t* perm) {
    for (int e = threadIdx.x; e < s * s; e += blockDim.x) {
        const int q = e / s, i = e - q * s;
        R[e] = i <= q ? work[st->colmap[q] * N + i] : 0.0;
    }
    for (int q = threadIdx.x; q < s; q += blockDim.x) perm[q] = st->perm[q];
}

}  // namespace

void exact_tall_qrcp(double* work, int64_t N, int64_t s, double* R, int64_t* perm, double* pnorm) {
    if (s > kEx) argument_error("bitwise pass 2 supports at most 32 columns");
    DevBuf<double> stb(sizeof(TallState) / sizeof(double) + 1), spb(sizeof(ChainSpec) / sizeof(double) + 1);
    auto* st = reinterpret_cast<TallState*>(stb.get());
    auto* sp = reinterpret_cast<ChainSpec*>(spb.get());
    const int eg = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(N, 256), (int64_t)sm_count() * 4));
    TTG_LAUNCH(k_et_init, 1, 1, 0, stream(), st, sp, (int)s, N);
    TTG_LAUNCH(k_chain, (int)s, 32, 0, stream(), work, N, sp);
    TTG_LAUNCH(k_et_norms, 1, 1, 0, stream(), st, sp, (int)s);
    const int64_t p = std::min(N, s);
    for (int k = 0; k < p; ++k) {
        TTG_LAUNCH(k_et_pick, 1, 1, 0, stream(), st, sp, (int)s, N, k, pnorm);
        TTG_LAUNCH(k_chain, 1, 32, 0, stream(), work, N, sp);
        TTG_LAUNCH(k_et_house, 1, 1, 0, stream(), work, st, sp, (int)s, N, k);
        TTG_LAUNCH(k_et_scale, eg, 256, 0, stream(), work, st, N, k);
        TTG_LAUNCH(k_chain, (int)std::max<int64_t>(1, s - k - 1), 32, 0, stream(), work, N, sp);
        TTG_LAUNCH(k_et_update, eg, 256, 0, stream(), work, st, sp, N, k);
        TTG_LAUNCH(k_et_downdate, 1, 1, 0, stream(), work, st, sp, (int)s, N, k);
        TTG_LAUNCH(k_chain, (int)std::max<int64_t>(1, s - k - 1), 32, 0, stream(), work, N, sp);
        TTG_LAUNCH(k_et_guard_done, 1, 1, 0, stream(), st, sp);
    }
    TTG_LAUNCH(k_et_out, 1, 256, 0, stream(), work, st, (int)s, N, R, perm);
}

}  // namespace ttg
