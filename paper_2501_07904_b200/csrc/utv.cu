// Factor-level device operations (utv.hpp): explicit-Q pivoted QR, the QLP/UTV engine
// state machine of factor.cpp:263-448 on device buffers, one-sided Jacobi SVD
// (factor.cpp:137-261) and truncation (factor.cpp:450-562).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <numeric>

#include "utv.hpp"

namespace ttg {
namespace {

constexpr int kT = 256;

// out(i, pos) = R1(i, perm[pos]) (R1 row i at R + i*n), i < p, pos < n.
__global__ void k_r_over_positions(const double* __restrict__ R, const int64_t* __restrict__ perm, int64_t p,
                                   int64_t n, double* out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= p * n) return;
    const int64_t pos = e / p, i = e - pos * p;
    out[i + pos * p] = R[i * n + perm[pos]];
}

// out(perm[j], c) = q(j, c), j < rows (permute_rows_from, factor.cpp:280-289)
__global__ void k_rows_from(const double* __restrict__ q, int64_t rows, int64_t cols, const int64_t* __restrict__ perm,
                            double* out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= rows * cols) return;
    const int64_t c = e / rows, j = e - c * rows;
    out[perm[j] + c * rows] = q[j + c * rows];
}

// out(:, j) = u(:, perm[j]), j < count (select_columns, factor.cpp:291-298)
__global__ void k_pick_cols(const double* __restrict__ u, int64_t rows, const int64_t* __restrict__ perm, int64_t count,
                            double* out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= rows * count) return;
    const int64_t j = e / rows, i = e - j * rows;
    out[i + j * rows] = u[i + perm[j] * rows];
}

// c[j] = a[perm[j]], j < count (permutation composition, factor.cpp:316-325)
__global__ void k_compose_perm(const int64_t* __restrict__ a, const int64_t* __restrict__ perm, int64_t count,
                               int64_t* c) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < count) c[j] = a[perm[j]];
}

// identity columns reordered: out(perm[j], j) = 1 (materialize_perm, factor.cpp:300-305)
__global__ void k_perm_matrix(const int64_t* __restrict__ perm, int64_t rows, int64_t cols, double* out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= rows * cols) return;
    const int64_t j = e / rows, i = e - j * rows;
    out[e] = (perm[j] == i) ? 1.0 : 0.0;
}

// Leading pp x pp block of R (ld = ldr) as an upper (or, transposed, lower) triangle.
__global__ void k_square(const double* __restrict__ R, int64_t ldr, int64_t pp, bool to_lower, double* out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= pp * pp) return;
    const int64_t j = e / pp, i = e - j * pp;  // out(i, j)
    double v = 0.0;
    if (!to_lower) v = i <= j ? R[i + j * ldr] : 0.0;
    else v = j <= i ? R[j + i * ldr] : 0.0;
    out[i + j * pp] = v;
}

// B(:, perm[j]) = R(:, j): undo the column pivoting (c = Q R P^T = Q B).
__global__ void k_unpivot(const double* __restrict__ R, int64_t p, int64_t n, const int64_t* __restrict__ perm,
                          double* B) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= p * n) return;
    const int64_t j = e / p, i = e - j * p;
    B[i + perm[j] * p] = R[i + j * p];
}

// One-sided cyclic Jacobi (factor.cpp:170-206) on the n x n matrix W (ld n) with V = I
// accumulated, one warp, pairs in the reference's (i, j>i) order. status[0] = sweeps run,
// status[1] = 1 if not converged.
__global__ void k_jacobi(double* W, double* V, int64_t m, int64_t n, int max_sweeps, double tol, int* status) {
    const int lane = threadIdx.x;
    for (int64_t e = lane; e < n * n; e += 32) V[e] = (e % (n + 1) == 0) ? 1.0 : 0.0;
    __syncwarp();
    int sweep = 0;
    for (; sweep < max_sweeps; ++sweep) {
        bool rotated = false;
        for (int64_t i = 0; i + 1 < n; ++i)
            for (int64_t j = i + 1; j < n; ++j) {
                double* wi = W + i * m;
                double* wj = W + j * m;
                double aii = 0.0, ajj = 0.0, aij = 0.0;
                for (int64_t r = lane; r < m; r += 32) {
                    aii = fma(wi[r], wi[r], aii);
                    ajj = fma(wj[r], wj[r], ajj);
                    aij = fma(wi[r], wj[r], aij);
                }
                aii = warp_sum(aii);
                ajj = warp_sum(ajj);
                aij = warp_sum(aij);
                if (aii == 0.0 || ajj == 0.0) continue;
                if (fabs(aij) <= tol * sqrt(aii * ajj)) continue;
                rotated = true;
                const double zeta = (ajj - aii) / (2.0 * aij);
                const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double cs = 1.0 / sqrt(1.0 + t * t);
                const double sn = cs * t;
                for (int64_t r = lane; r < m; r += 32) {
                    const double x = wi[r], y = wj[r];
                    wi[r] = cs * x - sn * y;
                    wj[r] = sn * x + cs * y;
                }
                double* vi = V + i * n;
                double* vj = V + j * n;
                for (int64_t r = lane; r < n; r += 32) {
                    const double x = vi[r], y = vj[r];
                    vi[r] = cs * x - sn * y;
                    vj[r] = sn * x + cs * y;
                }
                __syncwarp();
            }
        if (!rotated) break;
    }
    if (lane == 0) {
        status[0] = sweep;
        status[1] = sweep == max_sweeps ? 1 : 0;
    }
}

// Column norms (sequential, factor.cpp:224-226) and the worst pair cosine on failure.
__global__ void k_colnorms(const double* W, int64_t m, int64_t n, double* s) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    double a = 0.0;
    for (int64_t i = 0; i < m; ++i) a = __dadd_rn(a, __dmul_rn(W[i + j * m], W[i + j * m]));
    s[j] = sqrt(a);
}

// U(:, j) = W(:, order[j]) / s_j, V(:, j) = Vr(:, order[j]) for s_j > 0.
__global__ void k_svd_assemble(const double* W, const double* Vr, int64_t m, int64_t n, const int64_t* order,
                               const double* s, double* U, double* V) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t j = blockIdx.y;
    const int64_t src = order[j];
    const double sj = s[src];
    if (e < m) U[e + j * m] = sj > 0.0 ? W[e + src * m] / sj : 0.0;
    if (e < n) V[e + j * n] = Vr[e + src * n];
}

// complete_basis_column (factor.cpp:143-162): column j of U (m x p) as the first unit
// vector whose twice-orthogonalised remainder has norm > 0.5. One warp.
__global__ void k_complete_basis(double* U, int64_t m, int64_t j, double* r, int* ok) {
    const int lane = threadIdx.x;
    for (int64_t cand = 0; cand < m; ++cand) {
        for (int64_t i = lane; i < m; i += 32) r[i] = i == cand ? 1.0 : 0.0;
        __syncwarp();
        for (int pass = 0; pass < 2; ++pass)
            for (int64_t c = 0; c < j; ++c) {
                double proj = 0.0;
                for (int64_t i = lane; i < m; i += 32) proj = fma(U[i + c * m], r[i], proj);
                proj = warp_sum(proj);
                for (int64_t i = lane; i < m; i += 32) r[i] -= proj * U[i + c * m];
                __syncwarp();
            }
        double nn = 0.0;
        for (int64_t i = lane; i < m; i += 32) nn = fma(r[i], r[i], nn);
        nn = sqrt(warp_sum(nn));
        if (nn > 0.5) {
            for (int64_t i = lane; i < m; i += 32) U[i + j * m] = r[i] / nn;
            if (lane == 0) *ok = 1;
            return;
        }
    }
    if (lane == 0) *ok = 0;
}

// kept masses (factor.cpp:479-505): kind 0 diagonal s, 1 lower rows, 2 upper columns.
__global__ void k_kept_kind(int kind, const double* t, int64_t p, double* part, double* kept) {
    for (int64_t r = threadIdx.x; r < p; r += blockDim.x) {
        double a = 0.0;
        if (kind == 0) a = __dmul_rn(t[r], t[r]);
        else
            for (int64_t j = 0; j <= r; ++j) {
                const double x = kind == 1 ? t[r + j * p] : t[j + r * p];
                a = __dadd_rn(a, __dmul_rn(x, x));
            }
        part[r] = a;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double acc = 0.0;
        kept[0] = 0.0;
        for (int64_t r = 0; r < p; ++r) {
            acc = __dadd_rn(acc, part[r]);
            kept[r + 1] = acc;
        }
    }
}

int grid_of(int64_t n) { return (int)std::max<int64_t>(1, cdiv(n, kT)); }

DMat transposed(const double* A, int64_t m, int64_t n) {
    DMat t(n, m);
    transpose(A, m, n, m, t.get(), n);
    return t;
}

struct State {
    DMat u, v, mid;
    DevBuf<int64_t> pu, pv;  // pending permutations (size 0 = none)
    int64_t npu = 0, npv = 0;
    bool lower = false;
};

void compose_with_q(DMat& d, DevBuf<int64_t>& pp, int64_t& np, const DQr& f) {
    if (np > 0) {
        DMat o(f.q.rows, f.q.cols);
        TTG_LAUNCH(k_rows_from, grid_of(f.q.rows * f.q.cols), kT, 0, stream(), f.q.get(), f.q.rows, f.q.cols,
                   pp.get(), o.get());
        pp.release();
        np = 0;
        d = std::move(o);
    } else {
        DMat o(d.rows, f.q.cols);
        gemm(false, false, d.rows, f.q.cols, d.cols, d.get(), d.rows, f.q.get(), f.q.rows, o.get(), d.rows);
        d = std::move(o);
    }
}

void compose_with_perm(DMat& d, DevBuf<int64_t>& pp, int64_t& np, const DevBuf<int64_t>& perm, int64_t count) {
    if (np > 0) {
        DevBuf<int64_t> c((size_t)count);
        TTG_LAUNCH(k_compose_perm, grid_of(count), kT, 0, stream(), pp.get(), perm.get(), count, c.get());
        pp = std::move(c);
        np = count;
    } else {
        DMat o(d.rows, count);
        TTG_LAUNCH(k_pick_cols, grid_of(d.rows * count), kT, 0, stream(), d.get(), d.rows, perm.get(), count, o.get());
        d = std::move(o);
    }
}

void flip(State& s, bool to_lower) {
    DQr f;
    if (to_lower) {
        DMat t = transposed(s.mid.get(), s.mid.rows, s.mid.cols);
        f = qrcp_full(t.get(), t.rows, t.cols);
    } else {
        f = qrcp_full(s.mid.get(), s.mid.rows, s.mid.cols);
    }
    const int64_t pp = f.r.rows;
    if (to_lower) {
        compose_with_perm(s.u, s.pu, s.npu, f.perm, pp);
        compose_with_q(s.v, s.pv, s.npv, f);
    } else {
        compose_with_q(s.u, s.pu, s.npu, f);
        compose_with_perm(s.v, s.pv, s.npv, f.perm, pp);
    }
    DMat sq(pp, pp);
    TTG_LAUNCH(k_square, grid_of(pp * pp), kT, 0, stream(), f.r.get(), f.r.rows, pp, to_lower, sq.get());
    s.mid = std::move(sq);
    s.lower = to_lower;
}

}  // namespace

DQr qrcp_full(const double* A, int64_t m, int64_t n, bool want_q) {
    if (m <= 0 || n <= 0) argument_error("qr_col_pivot: empty matrix");
    const int64_t p = std::min(m, n);
    DQr f;
    f.r = DMat(p, n);
    f.perm.alloc((size_t)n);
    if (want_q) f.q = DMat(m, p);
    if (small_qrcp_fits(m, n)) {
        DevBuf<double> pn((size_t)p);
        small_qrcp(A, m, n, m, f.perm.get(), f.r.get(), pn.get(), want_q ? f.q.get() : nullptr);
    } else if (m <= 4096) {
        WideQrcp e1(A, m, n, m, Layout::Col, p);
        e1.run_to(p);
        if (want_q)
            TTG_CUDA(cudaMemcpyAsync(f.q.get(), e1.Q(), sizeof(double) * m * p, cudaMemcpyDeviceToDevice, stream()));
        TTG_CUDA(cudaMemcpyAsync(f.perm.get(), e1.perm(), sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, stream()));
        TTG_LAUNCH(k_r_over_positions, grid_of(p * n), kT, 0, stream(), e1.R(), f.perm.get(), p, n, f.r.get());
        sync();  // e1's buffers are released at scope exit
    } else {
        DevBuf<double> B((size_t)(m * n));
        TTG_CUDA(cudaMemcpyAsync(B.get(), A, sizeof(double) * m * n, cudaMemcpyDeviceToDevice, stream()));
        TallQrcp e2(B.get(), m, n, m);
        e2.run(p);
        e2.extract_r(f.r.get(), p);
        TTG_CUDA(cudaMemcpyAsync(f.perm.get(), e2.perm(), sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, stream()));
        if (want_q) e2.form_q(f.q.get(), p, m);
        sync();
    }
    return f;
}

DUtv utv(const double* A, int64_t m, int64_t n, bool want_lower, int refine) {
    if (refine < 0) argument_error("refine_passes must be >= 0");
    if (refine > 64) argument_error("refine_passes is unreasonably large");
    if (m <= 0 || n <= 0) argument_error("utv: empty matrix");
    int passes = refine + 1;
    const int64_t p = std::min(m, n);
    // start side fixed by pass-count parity, forced extra pass on a mismatched shape
    // (utv_engine, factor.cpp:382-395)
    bool direct = want_lower ? (passes % 2 == 0) : (passes % 2 == 1);
    if (passes == 1) {
        if (direct && m < n) { passes = 2; direct = false; }
        else if (!direct && m > n) { passes = 2; direct = true; }
    }
    State s;
    if (direct) {
        DQr f = qrcp_full(A, m, n);
        s.u = std::move(f.q);
        s.pv = std::move(f.perm);
        s.npv = n;
        s.mid = std::move(f.r);
        s.lower = false;
    } else {
        DMat at = transposed(A, m, n);
        DQr f = qrcp_full(at.get(), n, m);
        s.pu = std::move(f.perm);
        s.npu = m;
        s.v = std::move(f.q);
        s.mid = transposed(f.r.get(), f.r.rows, f.r.cols);
        s.lower = true;
    }
    for (int pass = 1; pass < passes; ++pass) flip(s, !s.lower);
    if (s.npu > 0) {
        DMat o(m, p);
        TTG_LAUNCH(k_perm_matrix, grid_of(m * p), kT, 0, stream(), s.pu.get(), m, p, o.get());
        s.u = std::move(o);
    }
    if (s.npv > 0) {
        DMat o(n, p);
        TTG_LAUNCH(k_perm_matrix, grid_of(n * p), kT, 0, stream(), s.pv.get(), n, p, o.get());
        s.v = std::move(o);
    }
    DUtv out;
    out.u = std::move(s.u);
    out.t = std::move(s.mid);
    out.v = std::move(s.v);
    return out;
}

DSvd svd(const double* A, int64_t m, int64_t n, int max_sweeps, double tol) {
    if (m <= 0 || n <= 0) argument_error("svd: empty matrix");
    if (m < n) {  // svd of the transpose with the factors swapped (factor.cpp:256-261)
        DMat at = transposed(A, m, n);
        DSvd t = svd(at.get(), n, m, max_sweeps, tol);
        DSvd out;
        out.u = std::move(t.v);
        out.v = std::move(t.u);
        out.s = std::move(t.s);
        return out;
    }
    // Tall: A P = Q R, so A = Q B with B = R P^T (n x n). Jacobi on B rotates the same
    // column pairs with the same Gram entries (B^T B = A^T A) as the reference's Jacobi
    // on A; U = Q U_B.
    DQr f = qrcp_full(A, m, n);
    const int64_t p = n;
    DMat B(p, n);
    TTG_LAUNCH(k_unpivot, grid_of(p * n), kT, 0, stream(), f.r.get(), p, n, f.perm.get(), B.get());
    DMat Vr(n, n);
    DevBuf<int> st(2);
    TTG_LAUNCH(k_jacobi, 1, 32, 0, stream(), B.get(), Vr.get(), p, n, max_sweeps, tol, st.get());
    std::vector<int> hs = st.to_host(2);
    if (hs[1]) {
        std::vector<double> hb = B.buf.to_host((size_t)(p * n));
        double worst = 0.0;
        for (int64_t i = 0; i + 1 < n; ++i)
            for (int64_t j = i + 1; j < n; ++j) {
                double num = 0.0, a = 0.0, b = 0.0;
                for (int64_t r = 0; r < p; ++r) {
                    num += hb[(size_t)(r + i * p)] * hb[(size_t)(r + j * p)];
                    a += hb[(size_t)(r + i * p)] * hb[(size_t)(r + i * p)];
                    b += hb[(size_t)(r + j * p)] * hb[(size_t)(r + j * p)];
                }
                const double den = std::sqrt(a * b);
                if (den > 0.0) worst = std::max(worst, std::abs(num) / den);
            }
        char buf[160];
        std::snprintf(buf, sizeof buf, "svd: one-sided Jacobi did not converge in %d sweeps (worst pair cosine %.3e)",
                      max_sweeps, worst);
        fail(4, buf);
    }
    DevBuf<double> s(n);
    TTG_LAUNCH(k_colnorms, grid_of(n), kT, 0, stream(), B.get(), p, n, s.get());
    std::vector<double> hsv = s.to_host(n);
    std::vector<int64_t> order((size_t)n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) { return hsv[(size_t)x] > hsv[(size_t)y]; });
    DevBuf<int64_t> ord(n);
    ord.upload(order.data(), n);
    DMat Ub(p, n);
    DSvd out;
    out.v = DMat(n, n);
    TTG_LAUNCH(k_svd_assemble, dim3((unsigned)grid_of(std::max(p, n)), (unsigned)n), kT, 0, stream(), B.get(), Vr.get(),
               p, n, ord.get(), s.get(), Ub.get(), out.v.get());
    out.s.resize((size_t)n);
    for (int64_t j = 0; j < n; ++j) out.s[(size_t)j] = hsv[(size_t)order[(size_t)j]];
    // zero singular values: complete the basis of U_B (factor.cpp:247-249)
    DevBuf<double> scratch(p);
    DevBuf<int> ok(1);
    for (int64_t j = 0; j < n; ++j)
        if (!(out.s[(size_t)j] > 0.0)) {
            TTG_LAUNCH(k_complete_basis, 1, 32, 0, stream(), Ub.get(), p, j, scratch.get(), ok.get());
            if (ok.to_host(1)[0] == 0) fail(4, "svd: failed to complete an orthonormal basis");
        }
    out.u = DMat(m, n);
    gemm(false, false, m, n, p, f.q.get(), m, Ub.get(), p, out.u.get(), m);
    return out;
}

DTrunc truncate_rank(int kind, const double* t, int64_t p, int64_t rank, double eps) {
    DevBuf<double> part(p), kept(p + 1);
    TTG_LAUNCH(k_kept_kind, 1, kT, 0, stream(), kind, t, p, part.get(), kept.get());
    DTrunc out;
    out.kept = kept.to_host(p + 1);
    int64_t r = rank;
    if (rank <= 0) {  // pick_rank (factor.cpp:512-520)
        if (eps < 0.0) argument_error("tolerance must be >= 0");
        r = p;
        if (eps != 0.0) {
            const double target = out.kept[(size_t)p] - eps * eps;
            for (int64_t c = 1; c < p; ++c)
                if (out.kept[(size_t)c] >= target) { r = c; break; }
        }
    } else if (rank > p) {
        argument_error("rank " + std::to_string(rank) + " out of range 1.." + std::to_string(p));
    }
    out.rank = r;
    out.residual = std::sqrt(std::max(0.0, out.kept[(size_t)p] - out.kept[(size_t)r]));
    return out;
}

}  // namespace ttg
