// C++ drop-in layer (include/ttutv_b200/ttutv.hpp) over the C-ABI (include/ttutv_b200.h).
// Containers and validation live here (with the reference's messages); every computation
// is a C-ABI call into the device engine.
#include "ttutv_b200/ttutv.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>

#include "ttutv_b200.h"

namespace ttutv {
namespace {

constexpr std::int64_t kMaxElements = std::numeric_limits<std::int64_t>::max() / 8;

[[noreturn]] void rethrow(int st) {
    const std::string msg = ttg_last_error();
    switch (st) {
        case TTG_ERR_ARGUMENT: throw ArgumentError(msg);
        case TTG_ERR_INDEX: throw IndexError(msg);
        case TTG_ERR_PARSE: throw ParseError(msg, 0);
        case TTG_ERR_NUMERICAL: throw NumericalError(msg);
        case TTG_ERR_RESOURCE: throw ResourceError(msg);
        case TTG_ERR_INVARIANT: throw InvariantError(msg);
        default: throw Error(msg);
    }
}

void check(ttg_status st) {
    if (st != TTG_OK) rethrow(st);
}

std::int64_t checked_size(std::int64_t rows, std::int64_t cols) {
    if (rows < 0 || cols < 0) throw ArgumentError("matrix dims must be nonnegative");
    if (rows > 0 && cols > kMaxElements / rows) throw ArgumentError("matrix element count overflows the index range");
    return rows * cols;
}

thread_local bool t_full_qlp = false;
thread_local bool t_bitwise_qlp = false;

struct ResultGuard {
    ttg_result* r = nullptr;
    ~ResultGuard() { ttg_result_free(r); }
};

DecompResult run(const DenseTensor& a, const DecompConfig& cfg) {
    const std::vector<std::int64_t> dims(a.shape().dims().begin(), a.shape().dims().end());
    ttg_config c{};
    c.method = (int)cfg.method;
    c.sweep = (int)cfg.sweep;
    c.refine_passes = cfg.refine_passes;
    c.retain = (int)cfg.retain;
    c.debug_checks = cfg.debug_checks ? 1 : 0;
    c.qlp_policy = t_bitwise_qlp ? TTG_QLP_BITWISE : t_full_qlp ? TTG_QLP_FULL : TTG_QLP_EARLY_EXIT;
    if (const auto* fr = std::get_if<FixedRank>(&cfg.mode)) {
        c.fixed_rank = 1;
        c.ranks = fr->ranks.data();
        c.nranks = (int)fr->ranks.size();
    } else {
        const auto& ft = std::get<FixedTol>(cfg.mode);
        c.fixed_rank = 0;
        c.eps = ft.eps;
        c.weights = ft.weights.data();
        c.nweights = (int)ft.weights.size();
    }
    ResultGuard g;
    check(ttg_decompose(a.data(), dims.data(), (int)dims.size(), &c, 0, &g.r));
    const int d = ttg_result_order(g.r);
    std::vector<TTCore> cores;
    for (int k = 0; k < d; ++k) {
        std::int64_t cd[3];
        ttg_result_core_dims(g.r, k, cd);
        DenseTensor t{Shape({cd[0], cd[1], cd[2]})};
        check(ttg_result_core_copy(g.r, k, t.data()));
        cores.push_back(TTCore{std::move(t)});
    }
    DecompResult out{TTTensor(std::move(cores)), {}};
    DecompReport& rep = out.report;
    rep.step_errors.resize((size_t)std::max(d - 1, 0));
    rep.ranks_chosen.resize((size_t)d + 1);
    std::vector<std::int64_t> req((size_t)d + 1);
    int bk = 0;
    const int nreq = ttg_result_report(g.r, rep.step_errors.data(), rep.ranks_chosen.data(), req.data(), &rep.bound,
                                       &bk, &rep.input_norm, &rep.wall_time_ms);
    rep.ranks_requested.assign(req.begin(), req.begin() + nreq);
    rep.bound_kind = bk == TTG_BOUND_RSS ? BoundKind::root_sum_square : BoundKind::plain_sum;
    for (int i = 0; i < ttg_result_warning_count(g.r); ++i) rep.warnings.emplace_back(ttg_result_warning(g.r, i));
    rep.direct_step_errors.resize((size_t)std::max(d - 1, 0));
    ttg_result_direct_errors(g.r, rep.direct_step_errors.data());
    return out;
}

double max_gram_deviation(const Matrix& g, bool rows_orthonormal) {
    const std::int64_t n = rows_orthonormal ? g.rows() : g.cols();
    std::vector<double> gram((size_t)(n * n));
    check(ttg_matmul(g.data(), g.rows(), g.cols(), rows_orthonormal ? 0 : 1, g.data(), g.rows(), g.cols(),
                     rows_orthonormal ? 1 : 0, gram.data()));
    double worst = 0.0;
    for (std::int64_t j = 0; j < n; ++j)
        for (std::int64_t i = 0; i < n; ++i)
            worst = std::max(worst, std::abs(gram[(size_t)(i + j * n)] - (i == j ? 1.0 : 0.0)));
    return worst;
}

}  // namespace

// ---- Shape -------------------------------------------------------------------------
Shape::Shape(std::vector<std::int64_t> dims) : dims_(std::move(dims)) {
    for (size_t k = 0; k < dims_.size(); ++k) {
        if (dims_[k] < 1)
            throw ArgumentError("shape dim " + std::to_string(k + 1) + " is " + std::to_string(dims_[k]) +
                                ", must be >= 1");
        if (count_ > kMaxElements / dims_[k]) throw ArgumentError("shape element count overflows the index range");
        count_ *= dims_[k];
    }
}

std::int64_t Shape::dim(std::int64_t k) const {
    if (k < 1 || k > order())
        throw IndexError("mode " + std::to_string(k) + " out of range 1.." + std::to_string(order()));
    return dims_[(size_t)(k - 1)];
}

std::int64_t Shape::prefix_product(std::int64_t k) const {
    if (k < 0 || k > order())
        throw IndexError("prefix length " + std::to_string(k) + " out of range 0.." + std::to_string(order()));
    std::int64_t p = 1;
    for (std::int64_t j = 0; j < k; ++j) p *= dims_[(size_t)j];
    return p;
}

std::int64_t ivec(std::span<const std::int64_t> index, const Shape& shape) {
    if ((std::int64_t)index.size() != shape.order())
        throw IndexError("multi-index has " + std::to_string(index.size()) + " entries, tensor order is " +
                         std::to_string(shape.order()));
    std::int64_t lin = 1, stride = 1;
    for (std::int64_t k = 0; k < shape.order(); ++k) {
        const std::int64_t ik = index[(size_t)k], nk = shape.dims()[(size_t)k];
        if (ik < 1 || ik > nk)
            throw IndexError("index " + std::to_string(ik) + " out of range 1.." + std::to_string(nk) + " in mode " +
                             std::to_string(k + 1));
        lin += (ik - 1) * stride;
        stride *= nk;
    }
    return lin;
}

void ivec_inverse(std::int64_t linear, const Shape& shape, std::span<std::int64_t> out) {
    if (linear < 1 || linear > shape.element_count())
        throw IndexError("linear index " + std::to_string(linear) + " out of range 1.." +
                         std::to_string(shape.element_count()));
    if ((std::int64_t)out.size() != shape.order()) throw IndexError("output multi-index has wrong order");
    std::int64_t rest = linear - 1;
    for (std::int64_t k = 0; k < shape.order(); ++k) {
        const std::int64_t nk = shape.dims()[(size_t)k];
        out[(size_t)k] = rest % nk + 1;
        rest /= nk;
    }
}

bool next_index(std::span<std::int64_t> index, const Shape& shape) {
    for (std::int64_t k = 0; k < shape.order(); ++k) {
        auto& ik = index[(size_t)k];
        if (ik < shape.dims()[(size_t)k]) {
            ++ik;
            return true;
        }
        ik = 1;
    }
    return false;
}

// ---- Matrix / DenseTensor -------------------------------------------------------------
Matrix::Matrix(std::int64_t rows, std::int64_t cols) : r_(rows), c_(cols), v_((size_t)checked_size(rows, cols), 0.0) {}

Matrix::Matrix(std::int64_t rows, std::int64_t cols, std::vector<double> data)
    : r_(rows), c_(cols), v_(std::move(data)) {
    if ((std::int64_t)v_.size() != checked_size(rows, cols))
        throw ArgumentError("matrix storage size does not match rows*cols");
}

Matrix Matrix::identity(std::int64_t n) {
    Matrix m(n, n);
    for (std::int64_t i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
}

DenseTensor::DenseTensor(Shape shape) : s_(std::move(shape)), v_((size_t)s_.element_count(), 0.0) {}

DenseTensor::DenseTensor(Shape shape, std::vector<double> data) : s_(std::move(shape)), v_(std::move(data)) {
    if ((std::int64_t)v_.size() != s_.element_count()) throw ArgumentError("tensor storage size does not match shape");
}

// ---- trains ------------------------------------------------------------------------------
Matrix TTCore::left_unfolding() const { return Matrix(rank_left(), mode_dim() * rank_right(), data.storage()); }
Matrix TTCore::right_unfolding() const { return Matrix(rank_left() * mode_dim(), rank_right(), data.storage()); }

TTTensor::TTTensor(std::vector<TTCore> cores) : cores_(std::move(cores)) {
    if (cores_.empty()) throw ArgumentError("train needs at least one core");
    for (size_t k = 0; k < cores_.size(); ++k)
        if (cores_[k].data.order() != 3)
            throw ArgumentError("core " + std::to_string(k + 1) + " has order " +
                                std::to_string(cores_[k].data.order()) + ", expected 3");
    if (cores_.front().rank_left() != 1 || cores_.back().rank_right() != 1)
        throw ArgumentError("boundary ranks must both be 1");
    for (size_t k = 0; k + 1 < cores_.size(); ++k)
        if (cores_[k].rank_right() != cores_[k + 1].rank_left())
            throw ArgumentError("rank mismatch between cores " + std::to_string(k + 1) + " and " +
                                std::to_string(k + 2) + ": " + std::to_string(cores_[k].rank_right()) + " vs " +
                                std::to_string(cores_[k + 1].rank_left()));
}

Shape TTTensor::shape() const {
    std::vector<std::int64_t> d;
    for (const auto& c : cores_) d.push_back(c.mode_dim());
    return Shape(std::move(d));
}

std::vector<std::int64_t> TTTensor::ranks() const {
    std::vector<std::int64_t> r{1};
    for (const auto& c : cores_) r.push_back(c.rank_right());
    return r;
}

DenseTensor reconstruct(const TTTensor& tt, std::int64_t element_cap) {
    const Shape shape = tt.shape();
    if (shape.element_count() > element_cap)
        throw ResourceError("reconstruct would materialize " + std::to_string(shape.element_count()) +
                            " elements (cap " + std::to_string(element_cap) + ")");
    std::int64_t left = shape.dim(1);
    for (std::int64_t k = 2; k <= tt.order(); ++k) {
        const std::int64_t grown = left * tt.core(k).mode_dim();
        if (grown * tt.core(k).rank_right() > element_cap)
            throw ResourceError("reconstruct intermediate would reach " +
                                std::to_string(grown * tt.core(k).rank_right()) + " elements (cap " +
                                std::to_string(element_cap) + ")");
        left = grown;
    }
    std::vector<double> flat;
    for (const auto& c : tt.cores()) flat.insert(flat.end(), c.data.storage().begin(), c.data.storage().end());
    const std::vector<std::int64_t> dims(shape.dims().begin(), shape.dims().end());
    const std::vector<std::int64_t> ranks = tt.ranks();
    DenseTensor out{shape};
    check(ttg_reconstruct(flat.data(), dims.data(), ranks.data(), (int)dims.size(), element_cap, out.data()));
    return out;
}

std::int64_t param_count(const TTTensor& tt) {
    std::int64_t t = 0;
    for (const auto& c : tt.cores()) t += c.rank_left() * c.mode_dim() * c.rank_right();
    return t;
}

OrthogonalityReport check_orthogonality(const TTTensor& tt) {
    OrthogonalityReport rep;
    for (std::int64_t k = 1; k <= tt.order() - 1; ++k)
        rep.max_left_deviation = std::max(rep.max_left_deviation, max_gram_deviation(tt.core(k).right_unfolding(), false));
    for (std::int64_t k = 2; k <= tt.order(); ++k)
        rep.max_right_deviation = std::max(rep.max_right_deviation, max_gram_deviation(tt.core(k).left_unfolding(), true));
    return rep;
}

TTTensor zero_tt(const Shape& shape) {
    if (shape.order() < 1) throw ArgumentError("zero train needs order >= 1");
    std::vector<TTCore> cores;
    for (std::int64_t k = 1; k <= shape.order(); ++k) cores.push_back(TTCore{DenseTensor{Shape({1, shape.dim(k), 1})}});
    return TTTensor(std::move(cores));
}

Matrix unfold(const DenseTensor& t, std::int64_t k) {
    if (t.shape().order() < 2) throw ArgumentError("unfold requires order >= 2");
    if (k < 1 || k >= t.shape().order())
        throw ArgumentError("unfold mode " + std::to_string(k) + " out of range 1.." +
                            std::to_string(t.shape().order() - 1));
    const std::int64_t rows = t.shape().prefix_product(k);
    return Matrix(rows, t.element_count() / rows, t.storage());
}

namespace {
void check_fold_mode(const Shape& shape, std::int64_t k) {
    if (shape.order() < 2) throw ArgumentError("unfold requires order >= 2");
    if (k < 1 || k >= shape.order())
        throw ArgumentError("unfold mode " + std::to_string(k) + " out of range 1.." + std::to_string(shape.order() - 1));
}
void check_fold_dims(const Matrix& mat, const Shape& shape, std::int64_t k) {
    check_fold_mode(shape, k);
    const std::int64_t rows = shape.prefix_product(k);
    if (mat.rows() != rows || mat.cols() != shape.element_count() / rows)
        throw ArgumentError("fold: matrix is " + std::to_string(mat.rows()) + "x" + std::to_string(mat.cols()) +
                            ", expected " + std::to_string(rows) + "x" + std::to_string(shape.element_count() / rows));
}
}  // namespace

// fold (tensor_ops.cpp:32-47): a reshape of the same column-major bytes
DenseTensor fold(const Matrix& mat, const Shape& shape, std::int64_t k) {
    check_fold_dims(mat, shape, k);
    return DenseTensor(shape, mat.storage());
}

DenseTensor fold(Matrix&& mat, const Shape& shape, std::int64_t k) {
    check_fold_dims(mat, shape, k);
    return DenseTensor(shape, mat.take_storage());
}

DenseTensor mode_product(const DenseTensor& t, const Matrix& mat, std::int64_t k) {
    const Shape& shape = t.shape();
    if (k < 1 || k > shape.order())
        throw ArgumentError("mode " + std::to_string(k) + " out of range 1.." + std::to_string(shape.order()));
    if (mat.cols() != shape.dim(k))
        throw ArgumentError("mode-" + std::to_string(k) + " product needs " + std::to_string(shape.dim(k)) +
                            " columns, matrix has " + std::to_string(mat.cols()));
    std::vector<std::int64_t> nd(shape.dims().begin(), shape.dims().end());
    nd[(size_t)(k - 1)] = mat.rows();
    DenseTensor out{Shape(nd)};
    const std::vector<std::int64_t> dims(shape.dims().begin(), shape.dims().end());
    check(ttg_mode_product(t.data(), dims.data(), (int)dims.size(), (int)k, mat.data(), mat.rows(), mat.cols(),
                           out.data()));
    return out;
}

Matrix kron(const Matrix& a, const Matrix& b) {
    Matrix out(a.rows() * b.rows(), a.cols() * b.cols());
    check(ttg_kron(a.data(), a.rows(), a.cols(), b.data(), b.rows(), b.cols(), out.data()));
    return out;
}

double psnr(const DenseTensor& est, const DenseTensor& truth) {
    if (!(est.shape() == truth.shape())) throw ArgumentError("psnr: shapes differ");
    double out = 0.0;
    check(ttg_psnr(est.data(), truth.data(), truth.element_count(), &out));
    return out;
}

DenseTensor reverse_indices(const DenseTensor& t) {
    const std::vector<std::int64_t> dims(t.shape().dims().begin(), t.shape().dims().end());
    DenseTensor out{Shape(std::vector<std::int64_t>(dims.rbegin(), dims.rend()))};
    check(ttg_reverse_indices(t.data(), dims.data(), (int)dims.size(), out.data()));
    return out;
}

TTTensor reverse_tt(const TTTensor& tt) {
    const std::int64_t d = tt.order();
    std::vector<std::int64_t> dims, ranks{1};
    std::vector<double> flat;
    for (const TTCore& c : tt.cores()) {
        dims.push_back(c.mode_dim());
        ranks.push_back(c.rank_right());
        flat.insert(flat.end(), c.data.storage().begin(), c.data.storage().end());
    }
    std::vector<double> out(flat.size());
    if (d > 0) check(ttg_reverse_tt(flat.data(), dims.data(), ranks.data(), (int)d, out.data()));
    std::vector<TTCore> cores;
    std::size_t off = 0;
    for (std::int64_t k = d - 1; k >= 0; --k) {  // core k of the input becomes core d-1-k
        const TTCore& src = tt.cores()[(size_t)k];
        const std::int64_t n = src.data.element_count();
        cores.push_back(TTCore{DenseTensor(Shape({src.rank_right(), src.mode_dim(), src.rank_left()}),
                                           std::vector<double>(out.begin() + (long)off, out.begin() + (long)(off + n)))});
        off += (size_t)n;
    }
    return TTTensor(std::move(cores));
}

double frobenius_norm(const DenseTensor& t) {
    double out = 0.0;
    check(ttg_frobenius_norm(t.data(), t.element_count(), 0, &out));
    return out;
}

double frobenius_norm(const Matrix& m) {
    double out = 0.0;
    check(ttg_frobenius_norm(m.data(), m.size(), 0, &out));
    return out;
}

double rse(const DenseTensor& est, const DenseTensor& truth) {
    if (!(est.shape() == truth.shape())) throw ArgumentError("rse: shapes differ");
    double out = 0.0;
    check(ttg_rse(est.data(), truth.data(), truth.element_count(), &out));
    return out;
}

// ---- completion.hpp ------------------------------------------------------------------------
ObservationMask::ObservationMask(const Shape& shape, const std::vector<std::vector<std::int64_t>>& indices,
                                 const std::vector<double>& values)
    : shape_(shape) {
    if (indices.size() != values.size()) throw ArgumentError("observation indices and values differ in length");
    std::vector<std::pair<std::int64_t, double>> entries;
    entries.reserve(indices.size());
    for (size_t i = 0; i < indices.size(); ++i) entries.emplace_back(ivec(indices[i], shape) - 1, values[i]);
    std::sort(entries.begin(), entries.end());
    for (size_t i = 1; i < entries.size(); ++i)
        if (entries[i].first == entries[i - 1].first)
            throw ArgumentError("duplicate observation at linear index " + std::to_string(entries[i].first + 1));
    for (const auto& [idx, val] : entries) {
        linear_.push_back(idx);
        values_.push_back(val);
    }
    if (linear_.empty()) throw ArgumentError("observation set is empty");
}

ObservationMask::ObservationMask(const DenseTensor& indicator, const DenseTensor& values) : shape_(indicator.shape()) {
    if (!(indicator.shape() == values.shape())) throw ArgumentError("indicator and value tensors differ in shape");
    for (std::int64_t i = 0; i < indicator.element_count(); ++i)
        if (indicator[i] != 0.0) {
            linear_.push_back(i);
            values_.push_back(values[i]);
        }
    if (linear_.empty()) throw ArgumentError("observation set is empty");
}

double ObservationMask::values_norm() const { return std::sqrt(kernels::sum_squares(values_)); }

// a scatter of the observed entries (container code, no arithmetic)
DenseTensor project_observed(const DenseTensor& tensor, const ObservationMask& mask) {
    if (!(tensor.shape() == mask.shape())) throw ArgumentError("project_observed: shapes differ");
    DenseTensor out{tensor.shape()};
    for (std::int64_t i : mask.linear_indices()) out[i] = tensor[i];
    return out;
}

namespace {
struct CompletionGuard {
    ttg_completion* c = nullptr;
    CompletionGuard() = default;
    CompletionGuard(const CompletionGuard&) = delete;
    CompletionGuard(CompletionGuard&& o) noexcept : c(o.c) { o.c = nullptr; }
    ~CompletionGuard() {
        if (c) ttg_completion_free(c);
    }
};

TTTensor tt_of(const ttg_result* r) {
    std::vector<TTCore> cores;
    for (int k = 0; k < ttg_result_order(r); ++k) {
        std::int64_t cd[3];
        ttg_result_core_dims(r, k, cd);
        DenseTensor t{Shape({cd[0], cd[1], cd[2]})};
        check(ttg_result_core_copy(r, k, t.data()));
        cores.push_back(TTCore{std::move(t)});
    }
    return TTTensor(std::move(cores));
}

CompletionGuard run_completion(const ObservationMask& mask, const Shape& shape, const CompletionConfig& config,
                               const DenseTensor* truth, int max_iters) {
    if (!(mask.shape() == shape)) throw ArgumentError("mask was built against a different shape");
    if (truth != nullptr && !(truth->shape() == shape)) throw ArgumentError("ground truth has a different shape");
    const std::vector<std::int64_t> dims(shape.dims().begin(), shape.dims().end());
    ttg_completion_config c{};
    const bool adaptive = config.retraction_eps > 0.0;
    c.ranks = adaptive ? nullptr : config.ranks.data();
    c.nranks = adaptive ? 0 : (int)config.ranks.size();
    c.eps = config.retraction_eps;
    c.retraction = (int)config.retraction;
    c.step_size = config.step_size;
    c.max_iters = max_iters;
    c.stop_tol = config.stop_tol;
    c.refine_passes = config.refine_passes;
    c.dense_cap = config.dense_cap;
    if (!adaptive && config.ranks.size() != dims.size() + 1)
        throw ArgumentError("rank chain has " + std::to_string(config.ranks.size()) + " entries, expected " +
                            std::to_string(dims.size() + 1));
    CompletionGuard g;
    check(ttg_complete(mask.linear_indices().data(), mask.values().data(), mask.count(), dims.data(),
                       (int)dims.size(), &c, truth ? truth->data() : nullptr, 0, &g.c));
    return g;
}
}  // namespace

CompletionResult complete(const ObservationMask& mask, const Shape& shape, const CompletionConfig& config,
                          const DenseTensor* truth) {
    CompletionGuard g = run_completion(mask, shape, config, truth, config.max_iters);
    CompletionResult out;
    const int n = ttg_completion_iterations(g.c);
    IterationTrace& tr = out.trace;
    tr.rse_observed.resize((size_t)n);
    tr.wall_time_ms.resize((size_t)n);
    if (truth) {
        tr.rse_full.resize((size_t)n);
        tr.psnr.resize((size_t)n);
    }
    ttg_completion_trace(g.c, tr.rse_observed.data(), truth ? tr.rse_full.data() : nullptr,
                         truth ? tr.psnr.data() : nullptr, tr.wall_time_ms.data(), nullptr);
    tr.status = (CompletionStatus)ttg_completion_status(g.c);
    tr.note = ttg_completion_note(g.c);
    std::vector<std::int64_t> rk(shape.dims().size() + 1);
    for (int it = 0; it <= n; ++it)
        if (ttg_completion_ranks(g.c, it, rk.data())) tr.ranks.push_back(rk);
    out.tt = tt_of(ttg_completion_result(g.c));
    return out;
}

TTTensor initial_guess(const ObservationMask& mask, const Shape& shape, const CompletionConfig& config) {
    // the retraction of the zero-filled observations: decompose them directly
    if (!(mask.shape() == shape)) throw ArgumentError("mask was built against a different shape");
    if (shape.element_count() > config.dense_cap)
        throw ResourceError("completion would materialize " + std::to_string(shape.element_count()) + " elements (cap " +
                            std::to_string(config.dense_cap) + ")");
    DenseTensor filled{shape};
    for (std::int64_t i = 0; i < mask.count(); ++i) filled[mask.linear_indices()[(size_t)i]] = mask.values()[(size_t)i];
    DecompConfig dc;
    dc.method = config.retraction;
    dc.sweep = config.retraction == Method::urv ? Sweep::right_to_left : Sweep::left_to_right;
    if (config.retraction_eps > 0.0) dc.mode = FixedTol{config.retraction_eps, {}};
    else dc.mode = FixedRank{config.ranks};
    dc.refine_passes = config.refine_passes;
    return decompose(filled, dc).tt;
}

// ---- kernels.hpp ---------------------------------------------------------------------------
namespace kernels {
namespace {
bool g_parallel = true;
}
void set_parallel_enabled(bool enabled) noexcept { g_parallel = enabled; }
bool parallel_enabled() noexcept { return g_parallel; }

Matrix matmul(const Matrix& a, const Matrix& b, bool ta, bool tb) {
    const std::int64_t m = ta ? a.cols() : a.rows(), k = ta ? a.rows() : a.cols();
    const std::int64_t kb = tb ? b.cols() : b.rows(), n = tb ? b.rows() : b.cols();
    if (k != kb)
        throw ArgumentError("matmul inner dimensions do not match");
    Matrix c(m, n);
    check(ttg_matmul(a.data(), a.rows(), a.cols(), ta ? 1 : 0, b.data(), b.rows(), b.cols(), tb ? 1 : 0, c.data()));
    return c;
}
Matrix matmul_serial(const Matrix& a, const Matrix& b, bool ta, bool tb) { return matmul(a, b, ta, tb); }

Matrix transpose(const Matrix& a) {
    Matrix t(a.cols(), a.rows());
    if (a.size() == 0) return t;
    Matrix id = Matrix::identity(a.cols());
    // A^T = (A^T I): one device GEMM with the transposed operand
    check(ttg_matmul(a.data(), a.rows(), a.cols(), 1, id.data(), id.rows(), id.cols(), 0, t.data()));
    return t;
}

double sum_squares(std::span<const double> v) {
    double s = 0.0;
    check(ttg_sum_squares(v.data(), (std::int64_t)v.size(), 0, &s));
    return s;
}
double sum_squares_serial(std::span<const double> v) {
    double s = 0.0;
    for (double x : v) s += x * x;
    return s;
}
double dot(std::span<const double> x, std::span<const double> y) {
    if (x.size() != y.size()) throw ArgumentError("dot operands differ in length");
    double s = 0.0;
    for (size_t i = 0; i < x.size(); ++i) s += x[i] * y[i];
    return s;
}
void axpy(double alpha, std::span<const double> x, std::span<double> y) {
    if (x.size() != y.size()) throw ArgumentError("axpy operands differ in length");
    for (size_t i = 0; i < x.size(); ++i) y[i] += alpha * x[i];
}
}  // namespace kernels

// ---- factor level --------------------------------------------------------------------------
QrPivotResult qr_col_pivot(const Matrix& a) {
    if (a.rows() == 0 || a.cols() == 0) throw ArgumentError("qr_col_pivot: empty matrix");
    const std::int64_t p = std::min(a.rows(), a.cols());
    QrPivotResult f{Matrix(a.rows(), p), Matrix(p, a.cols()), std::vector<std::int64_t>((size_t)a.cols())};
    check(ttg_qr_col_pivot(a.data(), a.rows(), a.cols(), f.q.data(), f.r.data(), f.perm.data()));
    return f;
}

SvdResult svd(const Matrix& a, const SvdOptions& o) {
    if (a.rows() == 0 || a.cols() == 0) throw ArgumentError("svd: empty matrix");
    const std::int64_t p = std::min(a.rows(), a.cols());
    SvdResult f{Matrix(a.rows(), p), std::vector<double>((size_t)p), Matrix(a.cols(), p)};
    check(ttg_svd(a.data(), a.rows(), a.cols(), o.max_sweeps, o.pair_tol, f.u.data(), f.s.data(), f.v.data()));
    return f;
}

namespace {
template <class F>
F utv_call(const Matrix& a, int refine, bool lower) {
    if (a.rows() == 0 || a.cols() == 0) throw ArgumentError("utv: empty matrix");
    const std::int64_t p = std::min(a.rows(), a.cols());
    Matrix u(a.rows(), p), t(p, p), v(a.cols(), p);
    check(ttg_utv(a.data(), a.rows(), a.cols(), lower ? 1 : 0, refine, u.data(), t.data(), v.data()));
    return F{std::move(u), std::move(t), std::move(v)};
}

TruncatedFactorization trunc(int kind, const Matrix& u, const double* t, const Matrix& v, std::int64_t p,
                             std::int64_t rank, double eps) {
    if (rank != 0 && (rank < 1 || rank > p))
        throw ArgumentError("rank " + std::to_string(rank) + " out of range 1.." + std::to_string(p));
    Matrix u1(u.rows(), p), t11(p, p), v1(v.rows(), p);
    std::int64_t r = 0;
    double res = 0.0;
    check(ttg_truncate(kind, u.data(), t, v.data(), u.rows(), v.rows(), p, rank, eps, &r, &res, u1.data(),
                       t11.data(), v1.data()));
    auto shrink = [](const Matrix& m, std::int64_t rows, std::int64_t cols) {
        std::vector<double> d(m.storage().begin(), m.storage().begin() + rows * cols);
        return Matrix(rows, cols, std::move(d));
    };
    TruncatedFactorization out;
    out.kind = (FactorKind)kind;
    out.rank = r;
    out.u1 = shrink(u1, u.rows(), r);
    out.t11 = shrink(t11, r, r);
    out.v1 = shrink(v1, v.rows(), r);
    out.residual_norm = res;
    return out;
}
}  // namespace

namespace {
// factor.cpp:568-597: singular values of T11, of the discarded block and of T (the device SVD)
RankRevealDiag reveal(const Matrix& t, std::int64_t rank, bool lower) {
    const std::int64_t p = t.rows();
    if (rank < 1 || rank > p)
        throw ArgumentError("rank " + std::to_string(rank) + " out of range 1.." + std::to_string(p));
    RankRevealDiag out;
    Matrix t11(rank, rank);
    for (std::int64_t j = 0; j < rank; ++j)
        for (std::int64_t i = 0; i < rank; ++i) t11(i, j) = t(i, j);
    out.sigma_min_t11 = svd(t11).s.back();
    if (rank < p) {
        Matrix disc = lower ? Matrix(p - rank, p) : Matrix(p, p - rank);
        if (lower) {
            for (std::int64_t j = 0; j < p; ++j)
                for (std::int64_t i = rank; i < p; ++i) disc(i - rank, j) = t(i, j);
        } else {
            for (std::int64_t j = rank; j < p; ++j)
                for (std::int64_t i = 0; i < p; ++i) disc(i, j - rank) = t(i, j);
        }
        out.residual_spectral_norm = svd(disc).s.front();
    }
    const SvdResult full = svd(t);
    out.sigma_r = full.s[(size_t)(rank - 1)];
    out.sigma_r_plus_1 = rank < p ? full.s[(size_t)rank] : 0.0;
    return out;
}
}  // namespace

RankRevealDiag rank_reveal_diag(const UlvFactors& f, std::int64_t rank) { return reveal(f.l, rank, true); }
RankRevealDiag rank_reveal_diag(const UrvFactors& f, std::int64_t rank) { return reveal(f.r, rank, false); }

UlvFactors ulv(const Matrix& a, int refine) { return utv_call<UlvFactors>(a, refine, true); }
UrvFactors urv(const Matrix& a, int refine) { return utv_call<UrvFactors>(a, refine, false); }

TruncatedFactorization truncate_fixed_rank(const SvdResult& f, std::int64_t rank) {
    if (rank < 1) throw ArgumentError("rank " + std::to_string(rank) + " out of range 1.." + std::to_string(f.s.size()));
    return trunc(0, f.u, f.s.data(), f.v, (std::int64_t)f.s.size(), rank, 0.0);
}
TruncatedFactorization truncate_fixed_rank(const UlvFactors& f, std::int64_t rank) {
    if (rank < 1) throw ArgumentError("rank " + std::to_string(rank) + " out of range 1.." + std::to_string(f.l.rows()));
    return trunc(1, f.u, f.l.data(), f.v, f.l.rows(), rank, 0.0);
}
TruncatedFactorization truncate_fixed_rank(const UrvFactors& f, std::int64_t rank) {
    if (rank < 1) throw ArgumentError("rank " + std::to_string(rank) + " out of range 1.." + std::to_string(f.r.rows()));
    return trunc(2, f.u, f.r.data(), f.v, f.r.rows(), rank, 0.0);
}
TruncatedFactorization truncate_fixed_tol(const SvdResult& f, double eps) {
    if (eps < 0.0) throw ArgumentError("tolerance must be >= 0");
    return trunc(0, f.u, f.s.data(), f.v, (std::int64_t)f.s.size(), 0, eps);
}
TruncatedFactorization truncate_fixed_tol(const UlvFactors& f, double eps) {
    if (eps < 0.0) throw ArgumentError("tolerance must be >= 0");
    return trunc(1, f.u, f.l.data(), f.v, f.l.rows(), 0, eps);
}
TruncatedFactorization truncate_fixed_tol(const UrvFactors& f, double eps) {
    if (eps < 0.0) throw ArgumentError("tolerance must be >= 0");
    return trunc(2, f.u, f.r.data(), f.v, f.r.rows(), 0, eps);
}

// ---- sweeps --------------------------------------------------------------------------------
DecompResult tt_svd(const DenseTensor& a, const DecompConfig& config) {
    DecompConfig c = config;
    c.method = Method::svd;
    return run(a, c);
}

DecompResult tt_ulv_fixed_rank_l2r(const DenseTensor& a, const std::vector<std::int64_t>& ranks, int refine) {
    DecompConfig c;
    c.method = Method::ulv;
    c.sweep = Sweep::left_to_right;
    c.mode = FixedRank{ranks};
    c.refine_passes = refine;
    return run(a, c);
}

DecompResult tt_ulv_fixed_tol_l2r(const DenseTensor& a, double eps, const std::vector<double>& w, int refine) {
    DecompConfig c;
    c.method = Method::ulv;
    c.sweep = Sweep::left_to_right;
    c.mode = FixedTol{eps, w};
    c.refine_passes = refine;
    return run(a, c);
}

DecompResult tt_urv_fixed_rank_r2l(const DenseTensor& a, const std::vector<std::int64_t>& ranks, int refine) {
    DecompConfig c;
    c.method = Method::urv;
    c.sweep = Sweep::right_to_left;
    c.mode = FixedRank{ranks};
    c.refine_passes = refine;
    return run(a, c);
}

DecompResult tt_urv_fixed_tol_r2l(const DenseTensor& a, double eps, const std::vector<double>& w, int refine) {
    DecompConfig c;
    c.method = Method::urv;
    c.sweep = Sweep::right_to_left;
    c.mode = FixedTol{eps, w};
    c.refine_passes = refine;
    return run(a, c);
}

DecompResult tt_ulv_fixed_rank_r2l(const DenseTensor& a, const std::vector<std::int64_t>& ranks, Retain retain,
                                   int refine) {
    DecompConfig c;
    c.method = Method::ulv;
    c.sweep = Sweep::right_to_left;
    c.mode = FixedRank{ranks};
    c.retain = retain;
    c.refine_passes = refine;
    return run(a, c);
}

DecompResult left_orthogonal_via_urv(const DenseTensor& a, const DecompConfig& config) {
    DecompConfig c = config;
    c.method = Method::urv;
    c.sweep = Sweep::left_to_right;
    return run(a, c);
}

DecompResult decompose(const DenseTensor& a, const DecompConfig& config) { return run(a, config); }

double verify_bound(const DenseTensor& a, const TTTensor& tt, DecompReport& report, double slack_rel,
                    std::int64_t element_cap) {
    const DenseTensor recon = reconstruct(tt, element_cap);
    if (!(recon.shape() == a.shape())) throw ArgumentError("verify_bound: shapes differ");
    double achieved = 0.0;
    check(ttg_diff_norm(recon.data(), a.data(), a.element_count(), &achieved));
    report.achieved_error = achieved;
    const double allowed = report.bound + slack_rel * report.input_norm;
    if (achieved > allowed) {
        char buf[256];
        std::snprintf(buf, sizeof buf, "achieved error %.12e exceeds bound %.12e plus slack %.3e", achieved,
                      report.bound, slack_rel * report.input_norm);
        throw InvariantError(buf);
    }
    return achieved;
}

namespace gpu {
void set_full_qlp(bool full) noexcept { t_full_qlp = full; }
bool full_qlp() noexcept { return t_full_qlp; }
void set_bitwise_qlp(bool on) noexcept { t_bitwise_qlp = on; }
bool bitwise_qlp() noexcept { return t_bitwise_qlp; }
}  // namespace gpu

}  // namespace ttutv
