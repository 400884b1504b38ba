// Full factor-level operations on device buffers: pivoted QR with explicit Q, the UTV
// (QLP) engine at any refine_passes, one-sided Jacobi SVD, and truncation. These back the
// factor API (ttg_utv/ttg_svd/ttg_truncate) and the general sweep path (TT-SVD, Alg. 4,
// refine_passes != 1); the refine_passes = 1 TT-URV/TT-ULV sweeps use the early-exit
// cut engine in sweep.cu instead.
#pragma once

#include "engine.hpp"

namespace ttg {

struct DMat {
    DevBuf<double> buf;
    int64_t rows = 0, cols = 0;
    DMat() = default;
    DMat(int64_t r, int64_t c) : buf((size_t)(r * c)), rows(r), cols(c) {}
    double* get() const { return buf.get(); }
};

struct DQr {
    DMat q, r;
    DevBuf<int64_t> perm;  // n entries
};

// qr_col_pivot (factor.cpp:62-135) of the m x n matrix A (ld = m), explicit economy Q.
DQr qrcp_full(const double* A, int64_t m, int64_t n, bool want_q = true);

// ulv / urv (factor.cpp:376-448): lower != 0 -> T lower-triangular.
struct DUtv {
    DMat u, t, v;
};
DUtv utv(const double* A, int64_t m, int64_t n, bool lower, int refine_passes);

// svd (factor.cpp:164-261): U m x p, s (p, descending), V n x p.
struct DSvd {
    DMat u, v;
    std::vector<double> s;
};
DSvd svd(const double* A, int64_t m, int64_t n, int max_sweeps, double pair_tol);

// truncation (factor.cpp:450-562). kind 0 svd (t = s as a device p-vector), 1 ulv, 2 urv.
struct DTrunc {
    int64_t rank = 0;
    double residual = 0.0;
    std::vector<double> kept;  // kept[0..p]
};
// rank > 0: fixed; else tolerance eps. Only computes the rank and residual; the leading
// blocks are plain column-major prefixes the caller copies.
DTrunc truncate_rank(int kind, const double* t, int64_t p, int64_t rank, double eps);

}  // namespace ttg
