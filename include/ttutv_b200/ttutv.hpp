// ttutv.hpp -- C++ drop-in layer of the B200 TT-UTV engine.
//
// Declares, in namespace ttutv, the names and signatures of the reference API a caller
// of the TT-UTV path uses (/root/reference/proj/include/ttutv: errors.hpp, shape.hpp,
// matrix.hpp, dense_tensor.hpp, tt.hpp, factor.hpp, tt_decomp.hpp, tensor_ops.hpp), so
// code written against the reference recompiles against this one header and links
// libttutv_b200.so. Containers are host-side value types with the reference's storage
// conventions; every computation is forwarded to the device through the C-ABI in
// ttutv_b200.h, and device failures come back as the reference's exception classes.
#pragma once

#include <cstdint>
#include <initializer_list>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

namespace ttutv {

// ---- errors (errors.hpp) ---------------------------------------------------------
struct Error : std::runtime_error {
    explicit Error(const std::string& m) : std::runtime_error(m) {}
};
struct ArgumentError : Error { using Error::Error; };
struct IndexError : Error { using Error::Error; };
struct ParseError : Error {
    ParseError(const std::string& m, std::int64_t off)
        : Error(m + " (at offset " + std::to_string(off) + ")"), off_(off) {}
    std::int64_t offset() const noexcept { return off_; }
private:
    std::int64_t off_ = 0;
};
struct NumericalError : Error { using Error::Error; };
struct ResourceError : Error { using Error::Error; };
struct InvariantError : Error { using Error::Error; };

// ---- shapes and storage (shape.hpp, matrix.hpp, dense_tensor.hpp) -----------------
class Shape {
public:
    Shape() = default;
    explicit Shape(std::vector<std::int64_t> dims);
    std::int64_t order() const noexcept { return (std::int64_t)dims_.size(); }
    std::int64_t dim(std::int64_t k) const;  // 1-based
    std::span<const std::int64_t> dims() const noexcept { return dims_; }
    std::int64_t element_count() const noexcept { return count_; }
    std::int64_t prefix_product(std::int64_t k) const;
    bool operator==(const Shape& o) const noexcept { return dims_ == o.dims_; }
private:
    std::vector<std::int64_t> dims_;
    std::int64_t count_ = 1;
};

std::int64_t ivec(std::span<const std::int64_t> index, const Shape& shape);
void ivec_inverse(std::int64_t linear, const Shape& shape, std::span<std::int64_t> index_out);
bool next_index(std::span<std::int64_t> index, const Shape& shape);

// Column-major double matrix: (i, j) -> data[i + j * rows].
class Matrix {
public:
    Matrix() = default;
    Matrix(std::int64_t rows, std::int64_t cols);
    Matrix(std::int64_t rows, std::int64_t cols, std::vector<double> data);
    static Matrix identity(std::int64_t n);
    std::int64_t rows() const noexcept { return r_; }
    std::int64_t cols() const noexcept { return c_; }
    std::int64_t size() const noexcept { return r_ * c_; }
    bool empty() const noexcept { return v_.empty(); }
    double& operator()(std::int64_t i, std::int64_t j) noexcept { return v_[(size_t)(i + j * r_)]; }
    double operator()(std::int64_t i, std::int64_t j) const noexcept { return v_[(size_t)(i + j * r_)]; }
    double* data() noexcept { return v_.data(); }
    const double* data() const noexcept { return v_.data(); }
    double* col(std::int64_t j) noexcept { return v_.data() + j * r_; }
    const double* col(std::int64_t j) const noexcept { return v_.data() + j * r_; }
    std::vector<double>& storage() noexcept { return v_; }
    const std::vector<double>& storage() const noexcept { return v_; }
    std::vector<double> take_storage() noexcept { r_ = c_ = 0; return std::move(v_); }
private:
    std::int64_t r_ = 0, c_ = 0;
    std::vector<double> v_;
};

// Flat tensor, first index fastest; byte-identical to a Matrix of its first unfolding.
class DenseTensor {
public:
    DenseTensor() = default;
    explicit DenseTensor(Shape shape);
    DenseTensor(Shape shape, std::vector<double> data);
    const Shape& shape() const noexcept { return s_; }
    std::int64_t order() const noexcept { return s_.order(); }
    std::int64_t element_count() const noexcept { return s_.element_count(); }
    double& at(std::span<const std::int64_t> idx) { return v_[(size_t)(ivec(idx, s_) - 1)]; }
    double at(std::span<const std::int64_t> idx) const { return v_[(size_t)(ivec(idx, s_) - 1)]; }
    double& at(std::initializer_list<std::int64_t> idx) {
        return at(std::span<const std::int64_t>(idx.begin(), idx.size()));
    }
    double at(std::initializer_list<std::int64_t> idx) const {
        return at(std::span<const std::int64_t>(idx.begin(), idx.size()));
    }
    double& operator[](std::int64_t i) noexcept { return v_[(size_t)i]; }
    double operator[](std::int64_t i) const noexcept { return v_[(size_t)i]; }
    double* data() noexcept { return v_.data(); }
    const double* data() const noexcept { return v_.data(); }
    std::vector<double>& storage() noexcept { return v_; }
    const std::vector<double>& storage() const noexcept { return v_; }
    std::vector<double> take_storage() noexcept { s_ = Shape(); return std::move(v_); }
    bool operator==(const DenseTensor& o) const noexcept { return s_ == o.s_ && v_ == o.v_; }
private:
    Shape s_;
    std::vector<double> v_;
};

// ---- tensor trains (tt.hpp) ---------------------------------------------------------
struct TTCore {
    DenseTensor data;  // (r_{k-1}, I_k, r_k)
    std::int64_t rank_left() const { return data.shape().dim(1); }
    std::int64_t mode_dim() const { return data.shape().dim(2); }
    std::int64_t rank_right() const { return data.shape().dim(3); }
    Matrix left_unfolding() const;   // r_{k-1} x (I_k r_k)
    Matrix right_unfolding() const;  // (r_{k-1} I_k) x r_k
};

class TTTensor {
public:
    TTTensor() = default;
    explicit TTTensor(std::vector<TTCore> cores);
    std::int64_t order() const noexcept { return (std::int64_t)cores_.size(); }
    const std::vector<TTCore>& cores() const noexcept { return cores_; }
    const TTCore& core(std::int64_t k) const { return cores_.at((size_t)(k - 1)); }
    Shape shape() const;
    std::vector<std::int64_t> ranks() const;
private:
    std::vector<TTCore> cores_;
};

DenseTensor reconstruct(const TTTensor& tt, std::int64_t element_cap = 100'000'000);
std::int64_t param_count(const TTTensor& tt);
struct OrthogonalityReport {
    double max_left_deviation = 0.0;
    double max_right_deviation = 0.0;
};
OrthogonalityReport check_orthogonality(const TTTensor& tt);
TTTensor reverse_tt(const TTTensor& tt);
TTTensor zero_tt(const Shape& shape);

// ---- tensor ops (tensor_ops.hpp) -----------------------------------------------------
Matrix unfold(const DenseTensor& tensor, std::int64_t k);
DenseTensor fold(const Matrix& mat, const Shape& shape, std::int64_t k);
DenseTensor fold(Matrix&& mat, const Shape& shape, std::int64_t k);
DenseTensor mode_product(const DenseTensor& tensor, const Matrix& mat, std::int64_t k);
Matrix kron(const Matrix& a, const Matrix& b);
double frobenius_norm(const DenseTensor& tensor);
double frobenius_norm(const Matrix& mat);
double rse(const DenseTensor& estimate, const DenseTensor& truth);
double psnr(const DenseTensor& estimate, const DenseTensor& truth);
DenseTensor reverse_indices(const DenseTensor& tensor);

// ---- dense kernels (kernels.hpp) -------------------------------------------------------
namespace kernels {
// The device kernels are always parallel and deterministic; the switch is kept for source
// compatibility and changes nothing (kernels.hpp:13-16).
void set_parallel_enabled(bool enabled) noexcept;
bool parallel_enabled() noexcept;
// C = op(A) op(B) on the device (DMMA tiles).
Matrix matmul(const Matrix& a, const Matrix& b, bool transpose_a = false, bool transpose_b = false);
Matrix matmul_serial(const Matrix& a, const Matrix& b, bool transpose_a = false, bool transpose_b = false);
Matrix transpose(const Matrix& a);
// 4096-blocked sum of squares on the device (kernels.cpp:84-102's blocking and order).
double sum_squares(std::span<const double> values);
// Host-side BLAS-1 helpers of the reference's test API (not on the decomposition path).
double sum_squares_serial(std::span<const double> values);
double dot(std::span<const double> x, std::span<const double> y);
void axpy(double alpha, std::span<const double> x, std::span<double> y);
}  // namespace kernels

// ---- factorizations (factor.hpp) -------------------------------------------------------
struct QrPivotResult {
    Matrix q;
    Matrix r;
    std::vector<std::int64_t> perm;
};
QrPivotResult qr_col_pivot(const Matrix& a);

struct SvdResult {
    Matrix u;
    std::vector<double> s;
    Matrix v;
};
struct SvdOptions {
    int max_sweeps = 60;
    double pair_tol = 1e-14;
};
SvdResult svd(const Matrix& a, const SvdOptions& options = {});

struct UlvFactors {
    Matrix u;
    Matrix l;
    Matrix v;
};
struct UrvFactors {
    Matrix u;
    Matrix r;
    Matrix v;
};
UlvFactors ulv(const Matrix& a, int refine_passes = 1);
UrvFactors urv(const Matrix& a, int refine_passes = 1);

enum class FactorKind { svd, ulv, urv };
struct TruncatedFactorization {
    FactorKind kind = FactorKind::svd;
    std::int64_t rank = 0;
    Matrix u1;
    Matrix t11;
    Matrix v1;
    double residual_norm = 0.0;
};
TruncatedFactorization truncate_fixed_rank(const SvdResult& f, std::int64_t rank);
TruncatedFactorization truncate_fixed_rank(const UlvFactors& f, std::int64_t rank);
TruncatedFactorization truncate_fixed_rank(const UrvFactors& f, std::int64_t rank);
TruncatedFactorization truncate_fixed_tol(const SvdResult& f, double eps);
TruncatedFactorization truncate_fixed_tol(const UlvFactors& f, double eps);
TruncatedFactorization truncate_fixed_tol(const UrvFactors& f, double eps);

// Rank-revealing diagnostics at split rank r (factor.hpp:87-95): sigma_min(T11), the
// spectral norm of the discarded block, and sigma_r, sigma_{r+1} of T (0 when r == p).
struct RankRevealDiag {
    double sigma_min_t11 = 0.0;
    double residual_spectral_norm = 0.0;
    double sigma_r = 0.0;
    double sigma_r_plus_1 = 0.0;
};
RankRevealDiag rank_reveal_diag(const UlvFactors& f, std::int64_t rank);
RankRevealDiag rank_reveal_diag(const UrvFactors& f, std::int64_t rank);

// ---- sweeps (tt_decomp.hpp) -------------------------------------------------------------
enum class Method { svd, ulv, urv };
enum class Sweep { left_to_right, right_to_left };
enum class Retain { l11_only, full_column };
struct FixedRank {
    std::vector<std::int64_t> ranks;
};
struct FixedTol {
    double eps = 0.0;
    std::vector<double> weights;
};
struct DecompConfig {
    Method method = Method::svd;
    Sweep sweep = Sweep::left_to_right;
    std::variant<FixedRank, FixedTol> mode = FixedRank{};
    int refine_passes = 1;
    Retain retain = Retain::l11_only;
    bool debug_checks = false;
};
enum class BoundKind { root_sum_square, plain_sum };
struct DecompReport {
    std::vector<double> step_errors;
    std::vector<std::int64_t> ranks_requested;
    std::vector<std::int64_t> ranks_chosen;
    double bound = 0.0;
    BoundKind bound_kind = BoundKind::root_sum_square;
    std::optional<double> achieved_error;
    double input_norm = 0.0;
    double wall_time_ms = 0.0;
    std::vector<std::string> warnings;
    // Extension (not in the reference): per cut, the discarded mass computed directly on the
    // device; step_errors keep the reference's kept[p] - kept[r] subtraction (factor.cpp:507-510).
    // -1 where not computed (general path: refine != 1, TT-SVD, Alg. 4).
    std::vector<double> direct_step_errors;
};
struct DecompResult {
    TTTensor tt;
    DecompReport report;
};

DecompResult tt_svd(const DenseTensor& a, const DecompConfig& config);
DecompResult tt_ulv_fixed_rank_l2r(const DenseTensor& a, const std::vector<std::int64_t>& ranks,
                                   int refine_passes = 1);
DecompResult tt_ulv_fixed_tol_l2r(const DenseTensor& a, double eps, const std::vector<double>& weights = {},
                                  int refine_passes = 1);
DecompResult tt_urv_fixed_rank_r2l(const DenseTensor& a, const std::vector<std::int64_t>& ranks,
                                   int refine_passes = 1);
DecompResult tt_urv_fixed_tol_r2l(const DenseTensor& a, double eps, const std::vector<double>& weights = {},
                                  int refine_passes = 1);
DecompResult tt_ulv_fixed_rank_r2l(const DenseTensor& a, const std::vector<std::int64_t>& ranks,
                                   Retain retain = Retain::l11_only, int refine_passes = 1);
DecompResult left_orthogonal_via_urv(const DenseTensor& a, const DecompConfig& config);
DecompResult decompose(const DenseTensor& a, const DecompConfig& config);
double verify_bound(const DenseTensor& a, const TTTensor& tt, DecompReport& report, double slack_rel = 1e-8,
                    std::int64_t element_cap = 100'000'000);

// ---- completion (completion.hpp) ----------------------------------------------------------
class ObservationMask {
public:
    ObservationMask() = default;
    ObservationMask(const Shape& shape, const std::vector<std::vector<std::int64_t>>& indices,
                    const std::vector<double>& values);
    ObservationMask(const DenseTensor& indicator, const DenseTensor& values);
    const Shape& shape() const noexcept { return shape_; }
    std::int64_t count() const noexcept { return (std::int64_t)linear_.size(); }
    const std::vector<std::int64_t>& linear_indices() const noexcept { return linear_; }
    const std::vector<double>& values() const noexcept { return values_; }
    double values_norm() const;
private:
    Shape shape_;
    std::vector<std::int64_t> linear_;
    std::vector<double> values_;
};
DenseTensor project_observed(const DenseTensor& tensor, const ObservationMask& mask);

struct CompletionConfig {
    std::vector<std::int64_t> ranks;
    Method retraction = Method::svd;
    double step_size = 1.0;
    int max_iters = 500;
    double stop_tol = 1e-6;
    std::uint64_t seed = 42;
    int refine_passes = 2;
    std::int64_t dense_cap = 10'000'000;
    // Extension (BASELINE config 4): > 0 retracts at this prescribed accuracy (FixedTol, equal
    // rss weights) instead of the fixed-rank chain, which may then be empty.
    double retraction_eps = 0.0;
};
enum class CompletionStatus { converged, max_iters, diverged };
struct IterationTrace {
    std::vector<double> rse_observed;
    std::vector<double> rse_full;
    std::vector<double> psnr;
    std::vector<double> wall_time_ms;
    CompletionStatus status = CompletionStatus::max_iters;
    std::string note;
    // Extension: the rank chain of every iterate, [0] = the initial guess.
    std::vector<std::vector<std::int64_t>> ranks;
};
struct CompletionResult {
    TTTensor tt;
    IterationTrace trace;
};
CompletionResult complete(const ObservationMask& mask, const Shape& shape, const CompletionConfig& config,
                          const DenseTensor* truth = nullptr);
TTTensor initial_guess(const ObservationMask& mask, const Shape& shape, const CompletionConfig& config);

// ---- engine controls beyond the reference API ---------------------------------------------
namespace gpu {
// QLP policy for every subsequent sweep on this thread: false = early exit (default),
// true = all p steps of both passes like the reference (include/ttutv_b200.h).
void set_full_qlp(bool full) noexcept;
bool full_qlp() noexcept;
// Bitwise QLP (TTG_QLP_BITWISE): full QLP with narrow cuts (W of <= 32 rows) computed bitwise
// like the reference's qr_col_pivot in both passes, so ulp-decided ranks are the reference's.
void set_bitwise_qlp(bool on) noexcept;
bool bitwise_qlp() noexcept;
}  // namespace gpu

}  // namespace ttutv
