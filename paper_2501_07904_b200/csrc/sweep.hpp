// Tensor-train sweep drivers (host orchestration of the device engine).
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "engine.hpp"

namespace ttg {

struct SweepConfig {
    int method = 0;  // 0 svd, 1 ulv, 2 urv
    int sweep = 0;   // 0 l2r, 1 r2l
    bool fixed_rank = true;
    std::vector<int64_t> ranks;
    double eps = 0.0;
    std::vector<double> weights;
    int refine = 1;
    int retain = 0;  // 0 l11_only, 1 full_column
    bool debug = false;
    int policy = 0;  // 0 early exit, 1 full QLP
};

struct CutInfo {
    int64_t m = 0, n = 0, p = 0, steps = 0, rank = 0, extensions = 0;
    std::vector<double> diag;  // |T_ii|, i < rank
    double direct_error = -1.0;  // directly computed discarded mass (-1: general path, not computed)
    std::vector<double> kept;    // the rank rule's kept[0..s] then kept[p] (empty: general path)
};

struct TTResult {
    std::vector<int64_t> dims;
    std::vector<DevBuf<double>> cores;
    std::vector<std::array<int64_t, 3>> core_dims;
    std::vector<double> step_errors;
    std::vector<int64_t> ranks_requested, ranks_chosen;
    double bound = 0.0;
    int bound_kind = 0;  // 0 rss, 1 plain sum
    double input_norm = 0.0;
    double wall_ms = 0.0;
    std::vector<std::string> warnings;
    std::vector<CutInfo> cuts;  // unfolding order
};

// a: device pointer to the dense tensor (first index fastest).
TTResult decompose(const double* a, const std::vector<int64_t>& dims, const SweepConfig& cfg);

// Column-sharded sweep over the ranks of `comm`. The first unfolding is
// split into comm.size() equal blocks of its pass-1 columns: TT-ULV-L2R shards the
// columns of c = A(i1; i2..id) (block g is a contiguous slice of A), TT-URV-R2L shards the
// rows of c = A(i1..i(d-1); id) (block g is an M/G x I_d column-major matrix). Each rank
// passes its own block; the cores come back replicated on every rank. Requirements: the
// sharded count divisible by comm.size(), refine_passes = 1, ULV-L2R or URV-R2L.
struct ShardRange {
    int64_t lo = 0, hi = 0;      // sharded index range [lo, hi) of this rank
    int64_t rows = 0, cols = 0;  // the local block's shape (column-major)
};
ShardRange shard_range(const std::vector<int64_t>& dims, int method, int nranks, int rank);
TTResult decompose_sharded(const double* a_local, const std::vector<int64_t>& dims, const SweepConfig& cfg,
                           Comm& comm);

// |A - reconstruct(tt)|^2 on device without materialising the full reconstruction.
double residual_squared(const TTResult& r, const double* a);
// Completion loop body on device (completion.cpp:161-186, step size 1): see
// ttg_completion_reset in include/ttutv_b200.h.
void completion_reset(double* y, const double* observed, const double* mask, const double* truth, int64_t n,
                      double stats[5]);
// Tensor algebra (tensor_ops.cu): mode_product / kron in the reference's operation order
// (bitwise), the maximum of a buffer, reverse_indices, and a reversed train's core.
void mode_product_dev(const double* x, int64_t left, int64_t mid, int64_t right, const double* m, int64_t new_mid,
                      double* out);
void kron_dev(const double* a, int64_t ar, int64_t ac, const double* b, int64_t br, int64_t bc, double* out);
double max_value_dev(const double* x, int64_t n);
void reverse_indices_dev(const double* a, const std::vector<int64_t>& dims, double* out);
void flip_core_dev(const double* in, int64_t rl, int64_t mid, int64_t rr, double* out);
// Dense reconstruction (device output of prod(dims) doubles).
void reconstruct(const std::vector<const double*>& cores, const std::vector<int64_t>& dims,
                 const std::vector<int64_t>& ranks, double* out);

}  // namespace ttg
