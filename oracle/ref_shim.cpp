// TEST INFRASTRUCTURE ONLY (oracle/). Never linked into the product.
//
// A C-ABI veneer over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/build_ref.sh into oracle/_ref/). It lets
// the Python test-suite, the golden-fixture generator and bench.py's
// `--impl reference` arm drive the reference's own public API
// (include/ttutv/{tt_decomp,factor,generators,tt,tensor_ops,kernels}.hpp)
// through ctypes. Only plain pointers and sizes cross this boundary.
//
// Error convention: every entry point returns 0 on success or the code of the
// reference exception class (same numbering as include/ttutv_b200.h):
//   1 ArgumentError 2 IndexError 3 ParseError 4 NumericalError
//   5 ResourceError 6 InvariantError 7 other ttutv::Error / std::exception
// and the message is available from ref_last_error().

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "ttutv/completion.hpp"
#include "ttutv/io.hpp"
#include "ttutv/errors.hpp"
#include "ttutv/factor.hpp"
#include "ttutv/generators.hpp"
#include "ttutv/kernels.hpp"
#include "ttutv/tensor_ops.hpp"
#include "ttutv/tt.hpp"
#include "ttutv/tt_decomp.hpp"

namespace {

thread_local std::string g_msg;

template <class F>
int guarded(F&& body) {
    try {
        body();
        g_msg.clear();
        return 0;
    } catch (const ttutv::ArgumentError& e) {
        g_msg = e.what();
        return 1;
    } catch (const ttutv::IndexError& e) {
        g_msg = e.what();
        return 2;
    } catch (const ttutv::ParseError& e) {
        g_msg = e.what();
        return 3;
    } catch (const ttutv::NumericalError& e) {
        g_msg = e.what();
        return 4;
    } catch (const ttutv::ResourceError& e) {
        g_msg = e.what();
        return 5;
    } catch (const ttutv::InvariantError& e) {
        g_msg = e.what();
        return 6;
    } catch (const std::exception& e) {
        g_msg = e.what();
        return 7;
    }
}

ttutv::Shape shape_of(const int64_t* dims, int d) {
    return ttutv::Shape(std::vector<std::int64_t>(dims, dims + d));
}

ttutv::DenseTensor tensor_of(const double* a, const int64_t* dims, int d) {
    ttutv::Shape s = shape_of(dims, d);
    std::vector<double> buf(a, a + s.element_count());
    return ttutv::DenseTensor(std::move(s), std::move(buf));
}

ttutv::Matrix matrix_of(const double* a, int64_t m, int64_t n) {
    return ttutv::Matrix(m, n, std::vector<double>(a, a + m * n));
}

void put(const ttutv::Matrix& x, double* out) {
    if (out) std::memcpy(out, x.data(), sizeof(double) * static_cast<size_t>(x.size()));
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_msg.c_str(); }

void ref_set_parallel(int enabled) { ttutv::kernels::set_parallel_enabled(enabled != 0); }

// ---- decompositions -------------------------------------------------------

// method: 0 svd, 1 ulv, 2 urv; sweep: 0 l2r, 1 r2l; retain: 0 l11_only, 1 full_column
// fixed_rank != 0 -> ranks[0..d] used; else eps + weights (nweights may be 0).
int ref_decompose(const double* a, const int64_t* dims, int d, int method, int sweep,
                  int fixed_rank, const int64_t* ranks, double eps, const double* weights,
                  int nweights, int refine, int retain, int debug_checks, void** handle) {
    *handle = nullptr;
    return guarded([&] {
        ttutv::DecompConfig cfg;
        cfg.method = static_cast<ttutv::Method>(method);
        cfg.sweep = static_cast<ttutv::Sweep>(sweep);
        cfg.refine_passes = refine;
        cfg.retain = static_cast<ttutv::Retain>(retain);
        cfg.debug_checks = debug_checks != 0;
        if (fixed_rank)
            cfg.mode = ttutv::FixedRank{std::vector<std::int64_t>(ranks, ranks + d + 1)};
        else
            cfg.mode = ttutv::FixedTol{eps, std::vector<double>(weights, weights + nweights)};
        auto* res = new ttutv::DecompResult(ttutv::decompose(tensor_of(a, dims, d), cfg));
        *handle = res;
    });
}

void ref_result_free(void* h) { delete static_cast<ttutv::DecompResult*>(h); }

int ref_result_order(void* h) {
    return static_cast<int>(static_cast<ttutv::DecompResult*>(h)->tt.order());
}

void ref_result_core_dims(void* h, int k, int64_t* out3) {
    const auto& c = static_cast<ttutv::DecompResult*>(h)->tt.cores()[static_cast<size_t>(k)];
    out3[0] = c.rank_left();
    out3[1] = c.mode_dim();
    out3[2] = c.rank_right();
}

void ref_result_core_copy(void* h, int k, double* out) {
    const auto& c = static_cast<ttutv::DecompResult*>(h)->tt.cores()[static_cast<size_t>(k)];
    std::memcpy(out, c.data.data(), sizeof(double) * static_cast<size_t>(c.data.element_count()));
}

// step_errors: d-1 entries; ranks_chosen: d+1; returns number of warnings.
int ref_result_report(void* h, double* step_errors, int64_t* ranks_chosen, double* bound,
                      int* bound_kind, double* input_norm, double* wall_ms) {
    const auto& r = static_cast<ttutv::DecompResult*>(h)->report;
    for (size_t i = 0; i < r.step_errors.size(); ++i) step_errors[i] = r.step_errors[i];
    for (size_t i = 0; i < r.ranks_chosen.size(); ++i) ranks_chosen[i] = r.ranks_chosen[i];
    *bound = r.bound;
    *bound_kind = r.bound_kind == ttutv::BoundKind::root_sum_square ? 0 : 1;
    *input_norm = r.input_norm;
    *wall_ms = r.wall_time_ms;
    return static_cast<int>(r.warnings.size());
}

const char* ref_result_warning(void* h, int i) {
    return static_cast<ttutv::DecompResult*>(h)->report.warnings[static_cast<size_t>(i)].c_str();
}

// RSE of the train in `h` against the dense tensor a (reference reconstruct + rse).
int ref_result_rse(void* h, const double* a, const int64_t* dims, int d, int64_t cap,
                   double* out) {
    return guarded([&] {
        const auto* res = static_cast<ttutv::DecompResult*>(h);
        *out = ttutv::rse(ttutv::reconstruct(res->tt, cap), tensor_of(a, dims, d));
    });
}

int ref_result_reconstruct(void* h, int64_t cap, double* out) {
    return guarded([&] {
        const auto* res = static_cast<ttutv::DecompResult*>(h);
        ttutv::DenseTensor x = ttutv::reconstruct(res->tt, cap);
        std::memcpy(out, x.data(), sizeof(double) * static_cast<size_t>(x.element_count()));
    });
}

// ---- factorizations -------------------------------------------------------

int ref_qr_col_pivot(const double* a, int64_t m, int64_t n, double* q, double* r,
                     int64_t* perm) {
    return guarded([&] {
        ttutv::QrPivotResult f = ttutv::qr_col_pivot(matrix_of(a, m, n));
        put(f.q, q);
        put(f.r, r);
        if (perm) std::memcpy(perm, f.perm.data(), sizeof(int64_t) * f.perm.size());
    });
}

// lower != 0 -> ulv (t lower), else urv (t upper). u: m x p, t: p x p, v: n x p.
int ref_utv(const double* a, int64_t m, int64_t n, int lower, int refine, double* u, double* t,
            double* v) {
    return guarded([&] {
        if (lower) {
            ttutv::UlvFactors f = ttutv::ulv(matrix_of(a, m, n), refine);
            put(f.u, u);
            put(f.l, t);
            put(f.v, v);
        } else {
            ttutv::UrvFactors f = ttutv::urv(matrix_of(a, m, n), refine);
            put(f.u, u);
            put(f.r, t);
            put(f.v, v);
        }
    });
}

// u: m x p, s: p, v: n x p
int ref_svd(const double* a, int64_t m, int64_t n, double* u, double* s, double* v) {
    return guarded([&] {
        ttutv::SvdResult f = ttutv::svd(matrix_of(a, m, n));
        put(f.u, u);
        put(f.v, v);
        std::memcpy(s, f.s.data(), sizeof(double) * f.s.size());
    });
}

// kind: 0 svd (t = diag s as p x p), 1 ulv, 2 urv. Truncation from full factors.
// fixed: rank >= 1 used; else eps. Outputs u1 (m x r), t11 (r x r), v1 (n x r).
int ref_truncate(int kind, const double* u, const double* t, const double* v, int64_t m,
                 int64_t n, int64_t p, int64_t rank, double eps, int64_t* rank_out,
                 double* residual, double* u1, double* t11, double* v1) {
    return guarded([&] {
        ttutv::TruncatedFactorization tf;
        ttutv::Matrix U = matrix_of(u, m, p), V = matrix_of(v, n, p);
        if (kind == 0) {
            ttutv::SvdResult f{U, {}, V};
            for (int64_t i = 0; i < p; ++i) f.s.push_back(t[i + i * p]);
            tf = rank > 0 ? ttutv::truncate_fixed_rank(f, rank) : ttutv::truncate_fixed_tol(f, eps);
        } else if (kind == 1) {
            ttutv::UlvFactors f{U, matrix_of(t, p, p), V};
            tf = rank > 0 ? ttutv::truncate_fixed_rank(f, rank) : ttutv::truncate_fixed_tol(f, eps);
        } else {
            ttutv::UrvFactors f{U, matrix_of(t, p, p), V};
            tf = rank > 0 ? ttutv::truncate_fixed_rank(f, rank) : ttutv::truncate_fixed_tol(f, eps);
        }
        *rank_out = tf.rank;
        *residual = tf.residual_norm;
        put(tf.u1, u1);
        put(tf.t11, t11);
        put(tf.v1, v1);
    });
}

// ---- generators and tensor ops -------------------------------------------

int ref_gen_gaussian(const int64_t* dims, int d, uint64_t seed, double* out) {
    return guarded([&] {
        ttutv::DenseTensor x = ttutv::gen_gaussian(shape_of(dims, d), seed);
        std::memcpy(out, x.data(), sizeof(double) * static_cast<size_t>(x.element_count()));
    });
}

int ref_gen_hilbert(const int64_t* dims, int d, double* out) {
    return guarded([&] {
        ttutv::DenseTensor x = ttutv::gen_hilbert(shape_of(dims, d));
        std::memcpy(out, x.data(), sizeof(double) * static_cast<size_t>(x.element_count()));
    });
}

// Dense reconstruction of gen_planted_tt(shape, ranks, seed).
int ref_gen_planted_dense(const int64_t* dims, int d, const int64_t* ranks, uint64_t seed,
                          int64_t cap, double* out) {
    return guarded([&] {
        ttutv::TTTensor tt = ttutv::gen_planted_tt(
            shape_of(dims, d), std::vector<std::int64_t>(ranks, ranks + d + 1), seed);
        ttutv::DenseTensor x = ttutv::reconstruct(tt, cap);
        std::memcpy(out, x.data(), sizeof(double) * static_cast<size_t>(x.element_count()));
    });
}

// Raw cores of gen_planted_tt, concatenated in core order.
int ref_gen_planted_cores(const int64_t* dims, int d, const int64_t* ranks, uint64_t seed,
                          double* out) {
    return guarded([&] {
        ttutv::TTTensor tt = ttutv::gen_planted_tt(
            shape_of(dims, d), std::vector<std::int64_t>(ranks, ranks + d + 1), seed);
        for (const auto& c : tt.cores()) {
            std::memcpy(out, c.data.data(), sizeof(double) * static_cast<size_t>(c.data.element_count()));
            out += c.data.element_count();
        }
    });
}

double ref_frobenius_norm(const double* a, int64_t count) {
    const int64_t dims[1] = {count};
    return ttutv::frobenius_norm(tensor_of(a, dims, 1));
}

uint64_t ref_rng_u64(uint64_t seed, int64_t skip) {
    ttutv::Rng rng(seed);
    for (int64_t i = 0; i < skip; ++i) rng.next_u64();
    return rng.next_u64();
}

// ---- binary containers (io.hpp) ---------------------------------------------
// read_tensor: status, and on ParseError its message (ref_last_error, without the
// " (at offset N)" suffix what() adds) and offset; on success order, dims and (if payload
// is not null) the elements.
int ref_read_tensor(const char* path, int64_t* offset, int* order, int64_t* dims, double* payload) {
    *offset = -1;
    try {
        ttutv::DenseTensor t = ttutv::read_tensor(path);
        *order = (int)t.order();
        for (int k = 0; k < t.order(); ++k) dims[k] = t.shape().dims()[(size_t)k];
        if (payload) std::memcpy(payload, t.data(), sizeof(double) * (size_t)t.element_count());
        g_msg.clear();
        return 0;
    } catch (const ttutv::ParseError& e) {
        const std::string w = e.what();
        const std::string suffix = " (at offset " + std::to_string(e.offset()) + ")";
        g_msg = w.size() >= suffix.size() && w.compare(w.size() - suffix.size(), suffix.size(), suffix) == 0
                    ? w.substr(0, w.size() - suffix.size())
                    : w;
        *offset = e.offset();
        return 3;
    } catch (const std::exception& e) {
        g_msg = e.what();
        return 7;
    }
}

int ref_write_tensor(const char* path, const double* a, const int64_t* dims, int d) {
    return guarded([&] { ttutv::write_tensor(path, tensor_of(a, dims, d)); });
}

// write_tt of the train with cores (ranks[k], dims[k], ranks[k+1]) back to back in `flat`
int ref_write_tt(const char* path, int d, const int64_t* ranks, const int64_t* dims, const double* flat) {
    return guarded([&] {
        std::vector<ttutv::TTCore> cores;
        const double* p = flat;
        for (int k = 0; k < d; ++k) {
            const int64_t cd[3] = {ranks[k], dims[k], ranks[k + 1]};
            cores.push_back(ttutv::TTCore{tensor_of(p, cd, 3)});
            p += cd[0] * cd[1] * cd[2];
        }
        ttutv::write_tt(path, ttutv::TTTensor(std::move(cores)));
    });
}

}  // extern "C"

// ---- tensor algebra (tensor_ops.hpp, tt.hpp, factor.hpp rank_reveal_diag) ----------------
extern "C" {

int ref_mode_product(const double* x, const int64_t* dims, int d, int k, const double* m, int64_t mr, int64_t mc,
                     double* out) {
    return guarded([&] {
        ttutv::DenseTensor y = ttutv::mode_product(tensor_of(x, dims, d), matrix_of(m, mr, mc), k);
        std::memcpy(out, y.data(), sizeof(double) * (size_t)y.element_count());
    });
}

int ref_kron(const double* a, int64_t ar, int64_t ac, const double* b, int64_t br, int64_t bc, double* out) {
    return guarded([&] { put(ttutv::kron(matrix_of(a, ar, ac), matrix_of(b, br, bc)), out); });
}

int ref_psnr(const double* e, const double* t, const int64_t* dims, int d, double* out) {
    return guarded([&] { *out = ttutv::psnr(tensor_of(e, dims, d), tensor_of(t, dims, d)); });
}

int ref_reverse_indices(const double* a, const int64_t* dims, int d, double* out) {
    return guarded([&] {
        ttutv::DenseTensor y = ttutv::reverse_indices(tensor_of(a, dims, d));
        std::memcpy(out, y.data(), sizeof(double) * (size_t)y.element_count());
    });
}

// cores packed back to back (core k: ranks[k] x dims[k] x ranks[k+1]); output packed in the
// reversed train's order
int ref_reverse_tt(const double* cores, const int64_t* dims, const int64_t* ranks, int d, double* out) {
    return guarded([&] {
        std::vector<ttutv::TTCore> cs;
        const double* p = cores;
        for (int k = 0; k < d; ++k) {
            const int64_t cd[3] = {ranks[k], dims[k], ranks[k + 1]};
            cs.push_back(ttutv::TTCore{tensor_of(p, cd, 3)});
            p += cd[0] * cd[1] * cd[2];
        }
        ttutv::TTTensor r = ttutv::reverse_tt(ttutv::TTTensor(std::move(cs)));
        for (const auto& c : r.cores()) {
            std::memcpy(out, c.data.data(), sizeof(double) * (size_t)c.data.element_count());
            out += c.data.element_count();
        }
    });
}

// lower != 0: UlvFactors{u, t, v}; else UrvFactors. out4 = sigma_min_t11, residual, sigma_r, sigma_r+1
int ref_rank_reveal_diag(const double* u, const double* t, const double* v, int64_t m, int64_t n, int64_t p,
                         int lower, int64_t rank, double* out4) {
    return guarded([&] {
        ttutv::RankRevealDiag dg;
        if (lower)
            dg = ttutv::rank_reveal_diag(ttutv::UlvFactors{matrix_of(u, m, p), matrix_of(t, p, p), matrix_of(v, n, p)},
                                         rank);
        else
            dg = ttutv::rank_reveal_diag(ttutv::UrvFactors{matrix_of(u, m, p), matrix_of(t, p, p), matrix_of(v, n, p)},
                                         rank);
        out4[0] = dg.sigma_min_t11;
        out4[1] = dg.residual_spectral_norm;
        out4[2] = dg.sigma_r;
        out4[3] = dg.sigma_r_plus_1;
    });
}

}  // extern "C"

// ---- completion (completion.hpp) ------------------------------------------------------
extern "C" {

int ref_gen_mask(const int64_t* dims, int d, double fraction, uint64_t seed, double* out) {
    return guarded([&] {
        ttutv::DenseTensor m = ttutv::gen_mask(shape_of(dims, d), fraction, seed);
        std::memcpy(out, m.data(), sizeof(double) * (size_t)m.element_count());
    });
}

// complete() with the mask given as 0/1 indicator + values (dense), fixed ranks; the trace
// arrays hold max_iters entries; returns via n_out / status_out; cores of the final train
// packed into cores_out (nullable) in core order.
int ref_complete(const double* indicator, const double* values, const int64_t* dims, int d, const int64_t* ranks,
                 int retraction, double step, int max_iters, double stop_tol, int refine, const double* truth,
                 double* obs, double* full, double* ps, int* n_out, int* status_out, double* cores_out) {
    return guarded([&] {
        ttutv::ObservationMask mask(tensor_of(indicator, dims, d), tensor_of(values, dims, d));
        ttutv::CompletionConfig cfg;
        cfg.ranks.assign(ranks, ranks + d + 1);
        cfg.retraction = static_cast<ttutv::Method>(retraction);
        cfg.step_size = step;
        cfg.max_iters = max_iters;
        cfg.stop_tol = stop_tol;
        cfg.refine_passes = refine;
        std::unique_ptr<ttutv::DenseTensor> tr;
        if (truth) tr = std::make_unique<ttutv::DenseTensor>(tensor_of(truth, dims, d));
        ttutv::CompletionResult r = ttutv::complete(mask, shape_of(dims, d), cfg, tr.get());
        const auto& t = r.trace;
        *n_out = (int)t.rse_observed.size();
        *status_out = (int)t.status;
        std::copy(t.rse_observed.begin(), t.rse_observed.end(), obs);
        if (truth) {
            std::copy(t.rse_full.begin(), t.rse_full.end(), full);
            std::copy(t.psnr.begin(), t.psnr.end(), ps);
        }
        if (cores_out)
            for (const auto& c : r.tt.cores()) {
                std::memcpy(cores_out, c.data.data(), sizeof(double) * (size_t)c.data.element_count());
                cores_out += c.data.element_count();
            }
    });
}

}  // extern "C"

// ---- sweep trace (golden fixtures) ------------------------------------------
// A restatement of sweep_l2r (ULV) / sweep_r2l (URV, l11_only) from
// src/tt_decomp.cpp:156-339 built only from the reference's public calls (ulv/urv,
// truncate_fixed_rank/tol, kernels::matmul, kernels::transpose), so every per-cut
// quantity is the reference's own bits; it additionally records what decompose() does
// not return: |diag T| (all p), the kept-mass vector (factor.cpp:479-499 order) and the
// directly computed discarded mass ||c - U1 T11 V1^T||_F per cut.
struct RefTrace {
    ttutv::DecompResult res;
    std::vector<std::vector<double>> diag, kept;
    std::vector<int64_t> m, n;
    std::vector<double> direct;
};

namespace {
std::vector<double> kept_of(const ttutv::Matrix& t, bool lower) {
    const int64_t p = t.rows();
    std::vector<double> kept((size_t)p + 1, 0.0);
    for (int64_t r = 1; r <= p; ++r) {
        double s = 0.0;
        for (int64_t j = 0; j < r; ++j) {
            const double v = lower ? t(r - 1, j) : t(j, r - 1);
            s += v * v;
        }
        kept[(size_t)r] = kept[(size_t)r - 1] + s;
    }
    return kept;
}
}  // namespace

extern "C" {

// method 1 ulv (l2r) or 2 urv (r2l); fixed_rank -> ranks[0..d], else eps (equal rss weights).
int ref_sweep_trace(const double* a, const int64_t* dims, int d, int method, int fixed_rank,
                    const int64_t* ranks, double eps, void** handle) {
    *handle = nullptr;
    return guarded([&] {
        using namespace ttutv;
        auto* tr = new RefTrace();
        const auto start = std::chrono::steady_clock::now();
        DenseTensor at = tensor_of(a, dims, d);
        const double norm_a = frobenius_norm(at);
        const Shape shp = at.shape();
        const int64_t count = shp.element_count();
        std::vector<double> budgets;
        for (int k = 0; k < d - 1; ++k) budgets.push_back(eps * norm_a / std::sqrt((double)(d - 1)));
        DecompReport& rep = tr->res.report;
        rep.input_norm = norm_a;
        rep.step_errors.assign((size_t)d - 1, 0.0);
        rep.ranks_chosen.assign((size_t)d + 1, 1);
        if (fixed_rank) rep.ranks_requested.assign(ranks, ranks + d + 1);
        tr->diag.resize((size_t)d - 1);
        tr->kept.resize((size_t)d - 1);
        tr->m.resize((size_t)d - 1);
        tr->n.resize((size_t)d - 1);
        tr->direct.resize((size_t)d - 1);
        std::vector<TTCore> cores;
        auto record = [&](int cut, const Matrix& c, const Matrix& t, bool lower, int64_t r,
                          const Matrix& u1, const Matrix& t11, const Matrix& v1) {
            std::vector<double> dg;
            for (int64_t i = 0; i < t.rows(); ++i) dg.push_back(std::abs(t(i, i)));
            tr->diag[(size_t)cut] = dg;
            tr->kept[(size_t)cut] = kept_of(t, lower);
            tr->m[(size_t)cut] = c.rows();
            tr->n[(size_t)cut] = c.cols();
            if (c.size() > 300000000) {  // memory: skip the direct residual on config 5's first cut
                tr->direct[(size_t)cut] = -1.0;
                return;
            }
            const Matrix low = kernels::matmul(kernels::matmul(u1, t11), v1, false, true);
            double s = 0.0;
            for (int64_t i = 0; i < c.size(); ++i) {
                const double e = c.data()[i] - low.data()[i];
                s += e * e;
            }
            tr->direct[(size_t)cut] = std::sqrt(s);
            (void)r;
        };
        if (method == 1) {
            Matrix c(shp.dim(1), count / shp.dim(1), at.take_storage());
            int64_t r_prev = 1;
            for (int64_t k = 1; k <= d - 1; ++k) {
                const int64_t p = std::min(c.rows(), c.cols());
                UlvFactors f = ulv(c, 1);
                TruncatedFactorization tf = fixed_rank
                    ? truncate_fixed_rank(f, std::min(ranks[k], p))
                    : truncate_fixed_tol(f, budgets[(size_t)k - 1]);
                record((int)k - 1, c, f.l, true, tf.rank, tf.u1, tf.t11, tf.v1);
                rep.step_errors[(size_t)k - 1] = tf.residual_norm;
                rep.ranks_chosen[(size_t)k] = tf.rank;
                Matrix carry = kernels::matmul(tf.t11, tf.v1, false, true);
                cores.push_back(TTCore{DenseTensor(Shape({r_prev, shp.dim(k), tf.rank}),
                                                   tf.u1.take_storage())});
                r_prev = tf.rank;
                if (k < d - 1) {
                    const int64_t nr = r_prev * shp.dim(k + 1);
                    const int64_t nc = carry.cols() / shp.dim(k + 1);
                    c = Matrix(nr, nc, carry.take_storage());
                } else {
                    cores.push_back(TTCore{DenseTensor(Shape({r_prev, shp.dim(d), 1}),
                                                       carry.take_storage())});
                }
            }
        } else {
            std::vector<TTCore> rev;
            Matrix c(count / shp.dim(d), shp.dim(d), at.take_storage());
            int64_t r_next = 1;
            for (int64_t k = d; k >= 2; --k) {
                const int64_t p = std::min(c.rows(), c.cols());
                UrvFactors f = urv(c, 1);
                TruncatedFactorization tf = fixed_rank
                    ? truncate_fixed_rank(f, std::min(ranks[k - 1], p))
                    : truncate_fixed_tol(f, budgets[(size_t)k - 2]);
                record((int)k - 2, c, f.r, false, tf.rank, tf.u1, tf.t11, tf.v1);
                rep.step_errors[(size_t)k - 2] = tf.residual_norm;
                rep.ranks_chosen[(size_t)k - 1] = tf.rank;
                Matrix carry = kernels::matmul(tf.u1, tf.t11);
                Matrix v1t = kernels::transpose(tf.v1);
                rev.push_back(TTCore{DenseTensor(Shape({tf.rank, shp.dim(k), r_next}),
                                                 v1t.take_storage())});
                r_next = tf.rank;
                if (k > 2) {
                    const int64_t nr = carry.rows() / shp.dim(k - 1);
                    c = Matrix(nr, shp.dim(k - 1) * tf.rank, carry.take_storage());
                } else {
                    rev.push_back(TTCore{DenseTensor(Shape({1, shp.dim(1), tf.rank}),
                                                     carry.take_storage())});
                }
            }
            cores.assign(std::make_move_iterator(rev.rbegin()), std::make_move_iterator(rev.rend()));
        }
        double b2 = 0.0;
        for (double e : rep.step_errors) b2 += e * e;
        rep.bound = std::sqrt(b2);
        rep.bound_kind = BoundKind::root_sum_square;
        rep.wall_time_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - start).count();
        tr->res.tt = TTTensor(std::move(cores));
        *handle = tr;
    });
}

void* ref_trace_result(void* h) { return &static_cast<RefTrace*>(h)->res; }
void ref_trace_free(void* h) { delete static_cast<RefTrace*>(h); }
// per cut (0-based unfolding index): p = diag length; kept has p+1 entries
int64_t ref_trace_cut(void* h, int cut, int64_t* m, int64_t* n, double* direct) {
    auto* t = static_cast<RefTrace*>(h);
    *m = t->m[(size_t)cut];
    *n = t->n[(size_t)cut];
    *direct = t->direct[(size_t)cut];
    return (int64_t)t->diag[(size_t)cut].size();
}
void ref_trace_cut_copy(void* h, int cut, double* diag, double* kept) {
    auto* t = static_cast<RefTrace*>(h);
    const auto& dg = t->diag[(size_t)cut];
    const auto& kp = t->kept[(size_t)cut];
    std::memcpy(diag, dg.data(), sizeof(double) * dg.size());
    std::memcpy(kept, kp.data(), sizeof(double) * kp.size());
}

}  // extern "C"
