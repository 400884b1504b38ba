// Drop-in check: a caller written against the reference headers (ttutv/*.hpp), compiled
// unchanged against the B200 engine (-Iinclude/ttutv_b200/compat -Iinclude) and linked to
// libttutv_b200.so. Prints one PASS/FAIL line per check; exit code = failures.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "ttutv/factor.hpp"
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

int main() {
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
