// Drop-in check: a caller written against the reference headers (ttutv/*.hpp), compiled
// unchanged against the B200 engine (-Iinclude/ttutv_b200/compat -Iinclude) and linked to
// libttutv_b200.so. Prints one PASS/FAIL line per check; exit code = failures.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "ttutv/dense_tensor.hpp"
#include "ttutv/factor.hpp"
#include "ttutv/kernels.hpp"
#include "ttutv/tensor_ops.hpp"
#include "ttutv/tt.hpp"
#include "ttutv/tt_decomp.hpp"

using namespace ttutv;

static int failures = 0;
static void report(bool ok, const char* what) {
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", what);
    if (!ok) ++failures;
}

static DenseTensor planted(const std::vector<std::int64_t>& dims, const std::vector<std::int64_t>& ranks,
                           unsigned seed, double rho) {
    std::mt19937_64 gen(seed);
    std::normal_distribution<double> nd;
    std::vector<TTCore> cores;
    for (size_t k = 0; k < dims.size(); ++k) {
        DenseTensor c{Shape({ranks[k], dims[k], ranks[k + 1]})};
        for (std::int64_t i = 0; i < c.element_count(); ++i) c[i] = nd(gen);
        cores.push_back(TTCore{std::move(c)});
    }
    DenseTensor a = reconstruct(TTTensor(std::move(cores)));
    if (rho > 0) {
        const double na = frobenius_norm(a);
        std::vector<double> e((size_t)a.element_count());
        double ne = 0;
        for (auto& x : e) { x = nd(gen); ne += x * x; }
        ne = std::sqrt(ne);
        for (std::int64_t i = 0; i < a.element_count(); ++i) a[i] += rho * na / ne * e[(size_t)i];
    }
    return a;
}

static Matrix random_matrix(std::int64_t m, std::int64_t n, std::mt19937_64& g) {
    std::normal_distribution<double> nd;
    Matrix a(m, n);
    for (std::int64_t i = 0; i < a.size(); ++i) a.data()[i] = nd(g);
    return a;
}

// max |Q^T Q - I| (test_factor.cpp's orthonormality_defect)
static double orthonormality_defect(const Matrix& q) {
    const Matrix g = kernels::matmul(q, q, true, false);
    double w = 0.0;
    for (std::int64_t j = 0; j < g.cols(); ++j)
        for (std::int64_t i = 0; i < g.rows(); ++i) w = std::max(w, std::abs(g(i, j) - (i == j ? 1.0 : 0.0)));
    return w;
}

static double diff_norm(const Matrix& a, const Matrix& b) {
    double s = 0.0;
    for (std::int64_t i = 0; i < a.size(); ++i) s += (a.data()[i] - b.data()[i]) * (a.data()[i] - b.data()[i]);
    return std::sqrt(s);
}

// The reference's own factor-level checks (tests/test_factor.cpp:103-150, 213-264),
// re-run on the device implementations through the unchanged headers.
static void factor_suite() {
    std::mt19937_64 g(101);
    {  // test_factor.cpp:103-140
        bool ok = true;
        for (auto [m, n] : {std::pair<int, int>{12, 8}, {8, 12}, {10, 10}, {1, 7}, {7, 1}}) {
            const Matrix a = random_matrix(m, n, g);
            const QrPivotResult f = qr_col_pivot(a);
            const std::int64_t p = std::min<std::int64_t>(m, n);
            ok = ok && f.q.rows() == m && f.q.cols() == p && f.r.rows() == p && f.r.cols() == n &&
                 f.perm.size() == (size_t)n;
            ok = ok && orthonormality_defect(f.q) <= 1e-12;
            for (std::int64_t j = 0; j < p; ++j)
                for (std::int64_t i = j + 1; i < p; ++i) ok = ok && f.r(i, j) == 0.0;
            for (std::int64_t j = 1; j < p; ++j)
                ok = ok && std::abs(f.r(j, j)) <= std::abs(f.r(j - 1, j - 1)) * (1.0 + 1e-12);
            std::vector<bool> seen((size_t)n, false);
            for (std::int64_t j : f.perm) {
                ok = ok && j >= 0 && j < n && !seen[(size_t)j];
                if (j >= 0 && j < n) seen[(size_t)j] = true;
            }
            const Matrix qr = kernels::matmul(f.q, f.r);
            const double norm = frobenius_norm(a);
            for (std::int64_t j = 0; j < n; ++j)
                for (std::int64_t i = 0; i < m; ++i)
                    ok = ok && std::abs(qr(i, j) - a(i, f.perm[(size_t)j])) <= 1e-12 * std::max(norm, 1.0);
        }
        report(ok, "qr_col_pivot identities (test_factor.cpp:103-140)");
    }
    {  // test_factor.cpp:142-150
        const QrPivotResult f = qr_col_pivot(Matrix(5, 3));
        bool ok = orthonormality_defect(f.q) == 0.0;
        for (std::int64_t j = 0; j < 3; ++j) {
            for (std::int64_t i = 0; i < 5; ++i) ok = ok && f.q(i, j) == (i == j ? 1.0 : 0.0);
            for (std::int64_t i = 0; i < 3; ++i) ok = ok && f.r(i, j) == 0.0;
        }
        report(ok, "qr_col_pivot of the zero matrix (test_factor.cpp:142-150)");
    }
    {  // test_factor.cpp:213-243
        bool ok = true;
        for (auto [m, n] : {std::pair<int, int>{12, 7}, {7, 12}, {9, 9}})
            for (int refine : {0, 1, 2}) {
                const Matrix a = random_matrix(m, n, g);
                const double norm = frobenius_norm(a);
                const std::int64_t p = std::min<std::int64_t>(m, n);
                const UlvFactors lf = ulv(a, refine);
                ok = ok && lf.l.rows() == p && lf.l.cols() == p;
                ok = ok && orthonormality_defect(lf.u) <= 1e-12 && orthonormality_defect(lf.v) <= 1e-12;
                for (std::int64_t j = 0; j < p; ++j)
                    for (std::int64_t i = 0; i < j; ++i) ok = ok && lf.l(i, j) == 0.0;
                const Matrix lr = kernels::matmul(kernels::matmul(lf.u, lf.l), lf.v, false, true);
                ok = ok && diff_norm(lr, a) <= 1e-10 * norm;
                const UrvFactors rf = urv(a, refine);
                ok = ok && rf.r.rows() == p && rf.r.cols() == p;
                ok = ok && orthonormality_defect(rf.u) <= 1e-12 && orthonormality_defect(rf.v) <= 1e-12;
                for (std::int64_t j = 0; j < p; ++j)
                    for (std::int64_t i = j + 1; i < p; ++i) ok = ok && rf.r(i, j) == 0.0;
                const Matrix rr = kernels::matmul(kernels::matmul(rf.u, rf.r), rf.v, false, true);
                ok = ok && diff_norm(rr, a) <= 1e-10 * norm;
            }
        bool threw = false;
        try {
            ulv(Matrix(3, 3), -1);
        } catch (const ArgumentError&) {
            threw = true;
        }
        report(ok && threw, "ulv/urv exact triangular middles, refine 0/1/2 (test_factor.cpp:213-243)");
    }
    {  // test_factor.cpp:245-264
        Matrix a(3, 3);
        a(0, 0) = 3.0;
        a(1, 1) = 2.0;
        a(2, 2) = 1.0;
        const SvdResult f = svd(a);
        const TruncatedFactorization r2 = truncate_fixed_rank(f, 2);
        bool ok = r2.rank == 2 && std::abs(r2.residual_norm - 1.0) <= 1e-12;
        ok = ok && truncate_fixed_tol(f, 1.5).rank == 2 && truncate_fixed_tol(f, 10.0).rank == 1;
        const TruncatedFactorization full = truncate_fixed_tol(f, 0.0);
        ok = ok && full.rank == 3 && full.residual_norm == 0.0;
        int throws = 0;
        for (std::int64_t bad : {0, 4}) {
            try {
                truncate_fixed_rank(f, bad);
            } catch (const ArgumentError&) {
                ++throws;
            }
        }
        report(ok && throws == 2, "truncation of diag(3,2,1) (test_factor.cpp:245-264)");
    }
    {  // rank_reveal_diag (factor.hpp:87-95): the reference's own quantities and their relations
        const Matrix a = random_matrix(10, 8, g);
        bool ok = true;
        for (std::int64_t r : {1, 3, 8}) {
            const UlvFactors lf = ulv(a);
            const UrvFactors rf = urv(a);
            const SvdResult s = svd(a);
            for (const RankRevealDiag d : {rank_reveal_diag(lf, r), rank_reveal_diag(rf, r)}) {
                ok = ok && std::abs(d.sigma_r - s.s[(size_t)r - 1]) <= 1e-12 * s.s[0];
                ok = ok && (r == 8 ? d.sigma_r_plus_1 == 0.0 : std::abs(d.sigma_r_plus_1 - s.s[(size_t)r]) <= 1e-12 * s.s[0]);
                ok = ok && d.sigma_min_t11 <= d.sigma_r * (1 + 1e-12);
                ok = ok && (r == 8 ? d.residual_spectral_norm == 0.0 : d.residual_spectral_norm >= d.sigma_r_plus_1 * (1 - 1e-12));
            }
        }
        bool threw = false;
        try {
            rank_reveal_diag(urv(a), 0);
        } catch (const ArgumentError&) {
            threw = true;
        }
        report(ok && threw, "rank_reveal_diag (sigma_r, sigma_r+1, interlacing, range check)");
    }
}

static void tensor_suite() {
    std::mt19937_64 g(7);
    std::normal_distribution<double> nd;
    {  // DenseTensor::at with an initializer list (dense_tensor.hpp:33-38), fold/unfold round trip
        DenseTensor t{Shape({3, 4, 5})};
        for (std::int64_t i = 0; i < t.element_count(); ++i) t[i] = (double)i;
        bool ok = t.at({1, 1, 1}) == 0.0 && t.at({2, 3, 4}) == 1.0 + 3.0 * 2.0 + 12.0 * 3.0;
        t.at({3, 4, 5}) = -1.0;
        ok = ok && t[59] == -1.0;
        const Matrix u = unfold(t, 2);
        ok = ok && u.rows() == 12 && u.cols() == 5 && fold(u, t.shape(), 2) == t;
        Matrix u2 = unfold(t, 1);
        ok = ok && fold(std::move(u2), t.shape(), 1) == t;
        bool threw = false;
        try {
            fold(Matrix(5, 12), t.shape(), 2);
        } catch (const ArgumentError& e) {
            threw = std::string(e.what()) == "fold: matrix is 5x12, expected 12x5";
        }
        report(ok && threw, "DenseTensor::at({..}), fold/unfold round trip and fold's error");
    }
    {  // reverse commutes with reconstruct (test_tt.cpp:120-138)
        std::vector<TTCore> cores;
        const std::vector<std::int64_t> dims{4, 3, 5, 2}, ranks{1, 2, 3, 2, 1};
        for (size_t k = 0; k < dims.size(); ++k) {
            DenseTensor c{Shape({ranks[k], dims[k], ranks[k + 1]})};
            for (std::int64_t i = 0; i < c.element_count(); ++i) c[i] = nd(g);
            cores.push_back(TTCore{std::move(c)});
        }
        const TTTensor tt(std::move(cores));
        const DenseTensor x = reconstruct(tt);
        const DenseTensor a = reverse_indices(x);
        const DenseTensor b = reconstruct(reverse_tt(tt));
        bool ok = a.shape() == b.shape() && a.shape() == Shape({2, 5, 3, 4});
        double w = 0.0;
        for (std::int64_t i = 0; ok && i < a.element_count(); ++i) w = std::max(w, std::abs(a[i] - b[i]));
        ok = ok && w <= 1e-12 * frobenius_norm(x) && reverse_indices(a) == x;
        report(ok, "reverse_indices(reconstruct(X)) == reconstruct(reverse_tt(X))");
    }
    {  // mode_product with a matrix, kron, psnr
        DenseTensor t{Shape({3, 4, 2})};
        for (std::int64_t i = 0; i < t.element_count(); ++i) t[i] = nd(g);
        const Matrix m = random_matrix(5, 4, g);
        const DenseTensor y = mode_product(t, m, 2);
        bool ok = y.shape() == Shape({3, 5, 2});
        for (std::int64_t r = 0; r < 2; ++r)
            for (std::int64_t jn = 0; jn < 5; ++jn)
                for (std::int64_t i = 0; i < 3; ++i) {
                    double s = 0.0;
                    for (std::int64_t j = 0; j < 4; ++j) s += m(jn, j) * t[i + 3 * j + 12 * r];
                    ok = ok && y[i + 3 * jn + 15 * r] == s;  // the reference's order: bitwise
                }
        const Matrix a = random_matrix(2, 3, g), b = random_matrix(3, 2, g);
        const Matrix k = kron(a, b);
        ok = ok && k.rows() == 6 && k.cols() == 6 && k(1 * 3 + 2, 2 * 2 + 1) == a(1, 2) * b(2, 1);
        DenseTensor e = t;
        e[0] += 0.01;
        const double p = psnr(e, t);
        double mx = t[0];
        for (std::int64_t i = 0; i < t.element_count(); ++i) mx = std::max(mx, t[i]);
        ok = ok && std::abs(p - 10.0 * std::log10(mx * mx / (1e-4 / 24.0))) <= 1e-6 && std::isinf(psnr(t, t));
        bool threw = false;
        try {
            mode_product(t, m, 3);
        } catch (const ArgumentError& ex) {
            threw = std::string(ex.what()) == "mode-3 product needs 2 columns, matrix has 4";
        }
        report(ok && threw, "mode_product (bitwise), kron, psnr");
    }
}

int main() {
    factor_suite();
    tensor_suite();
    const std::vector<std::int64_t> dims{12, 10, 14, 9}, ranks{1, 4, 6, 3, 1};
    const DenseTensor a = planted(dims, ranks, 7, 1e-6);

    // Alg. 3 / Alg. 1 at fixed rank: bound verified by the reference's verify_bound contract
    for (int m = 0; m < 2; ++m) {
        DecompResult r = m == 0 ? tt_urv_fixed_rank_r2l(a, ranks) : tt_ulv_fixed_rank_l2r(a, ranks);
        bool ok = r.report.ranks_chosen == ranks && r.tt.order() == 4;
        double ach = 0;
        try {
            ach = verify_bound(a, r.tt, r.report);
        } catch (const InvariantError&) {
            ok = false;
        }
        ok = ok && r.report.achieved_error.has_value() && ach <= 1e-5 * r.report.input_norm;
        report(ok, m == 0 ? "tt_urv_fixed_rank_r2l + verify_bound" : "tt_ulv_fixed_rank_l2r + verify_bound");
    }
    // prescribed accuracy (Alg. 2 and the URV analogue): rse <= eps
    {
        DecompResult u = tt_ulv_fixed_tol_l2r(a, 1e-4);
        DecompResult v = tt_urv_fixed_tol_r2l(a, 1e-4);
        const double e1 = rse(reconstruct(u.tt), a), e2 = rse(reconstruct(v.tt), a);
        report(e1 <= 1e-4 && e2 <= 1e-4 && u.report.ranks_chosen == ranks && v.report.ranks_chosen == ranks,
               "fixed tolerance sweeps meet eps with the planted ranks");
    }
    // uniform entry point, every (method, sweep) + orthogonality conventions
    {
        bool ok = true;
        for (Method meth : {Method::svd, Method::ulv, Method::urv})
            for (Sweep sw : {Sweep::left_to_right, Sweep::right_to_left}) {
                DecompConfig cfg;
                cfg.method = meth;
                cfg.sweep = sw;
                cfg.mode = FixedRank{ranks};
                DecompResult r = decompose(a, cfg);
                const OrthogonalityReport o = check_orthogonality(r.tt);
                ok = ok && (sw == Sweep::left_to_right ? o.max_left_deviation : o.max_right_deviation) <= 1e-12;
                ok = ok && rse(reconstruct(r.tt), a) <= 1e-5;
            }
        report(ok, "decompose: all six method/sweep pairs, orthogonality within 1e-12");
    }
    // factor level
    {
        Matrix m(9, 7);
        std::mt19937_64 g(3);
        std::normal_distribution<double> nd;
        for (std::int64_t i = 0; i < m.size(); ++i) m.data()[i] = nd(g);
        QrPivotResult q = qr_col_pivot(m);
        UrvFactors f = urv(m);
        TruncatedFactorization t = truncate_fixed_rank(f, 3);
        bool ok = q.q.rows() == 9 && q.r.rows() == 7 && (std::int64_t)q.perm.size() == 7;
        ok = ok && t.rank == 3 && t.u1.cols() == 3 && t.t11.rows() == 3 && t.residual_norm > 0;
        SvdResult s = svd(m);
        ok = ok && s.s.size() == 7 && s.s[0] >= s.s[6];
        report(ok, "qr_col_pivot / urv / truncate_fixed_rank / svd");
    }
    // error classes cross the boundary unchanged
    {
        bool ok = false;
        try {
            tt_urv_fixed_rank_r2l(a, {1, 2, 1});
        } catch (const ArgumentError& e) {
            ok = std::string(e.what()) == "rank chain has 3 entries, expected 5";
        }
        bool inv = false;
        DecompResult r = tt_urv_fixed_rank_r2l(a, {1, 1, 1, 1, 1});
        r.report.bound = 0.0;
        try {
            verify_bound(a, r.tt, r.report, 1e-12);
        } catch (const InvariantError&) {
            inv = true;
        }
        report(ok && inv, "ArgumentError / InvariantError mapping");
    }
    std::printf("%d failures\n", failures);
    return failures;
}
