// C-ABI boundary (include/ttutv_b200.h): argument marshalling, host<->device copies and
// exception -> status translation. No computation happens here.
#include <algorithm>
#include <chrono>
#include <mutex>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>

#include "../../include/ttutv_b200.h"
#include "completion.hpp"
#include "io.hpp"
#include "sweep.hpp"
#include "utv.hpp"

struct ttg_result {
    ttg::TTResult r;
};

struct ttg_completion {
    ttg::CompletionRun run;
    ttg_result res;
};

struct ttg_comm {
    std::unique_ptr<ttg::Comm> c;
};

namespace {

thread_local std::string t_msg;

template <class F>
ttg_status guard(F&& f) {
    try {
        f();
        t_msg.clear();
        return TTG_OK;
    } catch (const ttg::Failure& e) {
        t_msg = e.what();
        return static_cast<ttg_status>(e.code);
    } catch (const std::bad_alloc& e) {
        t_msg = "out of host memory";
        return TTG_ERR_RESOURCE;
    } catch (const std::exception& e) {
        t_msg = e.what();
        return TTG_ERR_INTERNAL;
    }
}

int64_t count_of(const int64_t* dims, int d) {
    int64_t n = 1;
    for (int i = 0; i < d; ++i) {
        if (dims[i] < 1)
            ttg::argument_error("shape dim " + std::to_string(i + 1) + " is " + std::to_string(dims[i]) +
                                ", must be >= 1");
        if (n > (INT64_MAX / 8) / dims[i]) ttg::argument_error("shape element count overflows the index range");
        n *= dims[i];
    }
    return n;
}

ttg::SweepConfig sweep_config(const ttg_config* cfg) {
    ttg::SweepConfig sc;
    sc.method = cfg->method;
    sc.sweep = cfg->sweep;
    if (sc.method < 0 || sc.method > 2) ttg::argument_error("unknown method");
    sc.fixed_rank = cfg->fixed_rank != 0;
    if (sc.fixed_rank && cfg->ranks && cfg->nranks > 0) sc.ranks.assign(cfg->ranks, cfg->ranks + cfg->nranks);
    sc.eps = cfg->eps;
    if (cfg->nweights > 0 && cfg->weights) sc.weights.assign(cfg->weights, cfg->weights + cfg->nweights);
    sc.refine = cfg->refine_passes;
    sc.retain = cfg->retain;
    sc.debug = cfg->debug_checks != 0;
    sc.policy = cfg->qlp_policy;
    return sc;
}

// Device view of a possibly-host buffer.
struct DeviceInput {
    ttg::DevBuf<double> buf;
    const double* ptr = nullptr;
    DeviceInput(const double* a, int64_t n, bool on_device) {
        if (on_device) {
            // the engine runs on its own non-blocking stream: order the read after any work the
            // caller queued on the legacy default stream (work on other streams of the caller's
            // must be synchronised by the caller, as ttutv_b200.h states)
            cudaEvent_t ev;
            TTG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            TTG_CUDA(cudaEventRecord(ev, cudaStreamLegacy));
            TTG_CUDA(cudaStreamWaitEvent(ttg::stream(), ev, 0));
            TTG_CUDA(cudaEventDestroy(ev));
            ptr = a;
        } else {
            // one upload at a time, completed before the next starts: each runs at the full
            // host-link rate and the next caller's upload overlaps this caller's compute
            static std::mutex mu;
            std::lock_guard<std::mutex> lk(mu);
            buf.alloc((size_t)n);
            buf.upload(a, (size_t)n);
            ttg::sync();
            ptr = buf.get();
        }
    }
};

}  // namespace

extern "C" {

const char* ttg_last_error(void) { return t_msg.c_str(); }
int ttg_abi_version(void) { return 1; }

int ttg_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

ttg_status ttg_set_device(int device) {
    return guard([&] { TTG_CUDA(cudaSetDevice(device)); });
}

int64_t ttg_kernel_launches(void) { return ttg::launches(); }

ttg_status ttg_synchronize(void) {
    return guard([&] { ttg::sync(); });
}

void* ttg_stream(void) {
    try {
        return (void*)ttg::stream();
    } catch (...) {
        return nullptr;
    }
}

ttg_status ttg_reserve(int64_t bytes) {
    return guard([&] {
        if (bytes < 0) ttg::argument_error("negative reservation");
        if (bytes == 0) return;
        void* p = nullptr;
        TTG_CUDA(cudaMallocAsync(&p, (size_t)bytes, ttg::stream()));
        TTG_CUDA(cudaFreeAsync(p, ttg::stream()));
        TTG_CUDA(cudaStreamSynchronize(ttg::stream()));
    });
}

int ttg_profile_kernels(int max, const char** names, double* ms, double* bytes, int64_t* launches) {
    try {
        return ttg::prof_kernels(max, names, ms, bytes, launches);
    } catch (...) {
        return -1;
    }
}

void ttg_profile_reset_kernels(void) { ttg::prof_reset_kernels(); }

ttg_status ttg_profile_big_phases(double* out24, int reset) {
    return guard([&] { ttg::big_phase_stats(out24, reset != 0); });
}

ttg_status ttg_profile_enable(int on) {
    return guard([&] { ttg::prof_enable(on != 0); });
}

int64_t ttg_profile_read(double* total_ms, double* algorithmic_bytes) {
    try {
        return ttg::prof_read(total_ms, algorithmic_bytes);
    } catch (...) {
        return -1;
    }
}

ttg_status ttg_decompose(const double* a, const int64_t* dims, int d, const ttg_config* cfg, int a_on_device,
                         ttg_result** out) {
    *out = nullptr;
    return guard([&] {
        if (!cfg) ttg::argument_error("null config");
        if (d < 0) ttg::argument_error("negative order");
        const auto start = std::chrono::steady_clock::now();
        std::vector<int64_t> dv(dims, dims + d);
        const int64_t n = count_of(dims, d);
        const ttg::SweepConfig sc = sweep_config(cfg);
        DeviceInput in(a, n, a_on_device != 0);
        // Decompositions issued from several host threads take the device in turn: their
        // persistent cooperative kernels each want every SM, and two of them interleaved ran
        // up to 5x slower than back to back on the B200. Uploads (above) and result reads are
        // outside the lock, so they overlap the other callers' compute.
        static std::mutex device_mu;
        std::unique_lock<std::mutex> turn(device_mu);
        auto* res = new ttg_result{ttg::decompose(in.ptr, dv, sc)};
        ttg::sync();
        turn.unlock();
        res->r.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - start).count();
        *out = res;
    });
}

void ttg_result_free(ttg_result* res) { delete res; }

// ---- files straight to and from the device (src/io.cpp:139-211) ----
int64_t ttg_last_error_offset(void) { return ttg::last_parse_offset(); }

ttg_status ttg_tensor_file_header(const char* path, int* order, int64_t* dims) {
    return guard([&] {
        if (!path) ttg::argument_error("null path");
        const ttg::TensorFileHeader h = ttg::read_tensor_header(path);
        *order = (int)h.dims.size();
        if (dims) std::copy(h.dims.begin(), h.dims.end(), dims);
    });
}

ttg_status ttg_tensor_file_to_device(const char* path, double* dst, int64_t capacity) {
    return guard([&] {
        if (!path) ttg::argument_error("null path");
        ttg::tensor_file_to_device(path, dst, capacity);
    });
}

ttg_status ttg_decompose_file(const char* path, const ttg_config* cfg, ttg_result** out) {
    *out = nullptr;
    return guard([&] {
        if (!cfg) ttg::argument_error("null config");
        if (!path) ttg::argument_error("null path");
        const auto start = std::chrono::steady_clock::now();
        const ttg::TensorFileHeader h = ttg::read_tensor_header(path);
        const ttg::SweepConfig sc = sweep_config(cfg);
        ttg::DevBuf<double> a((size_t)h.count);
        ttg::tensor_file_to_device(path, a.get(), h.count);
        auto* res = new ttg_result{ttg::decompose(a.get(), h.dims, sc)};
        res->r.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - start).count();
        *out = res;
    });
}

ttg_status ttg_result_write_file(const ttg_result* res, const char* path) {
    return guard([&] {
        if (!res || !path) ttg::argument_error("null argument");
        std::vector<const double*> cores;
        for (const auto& c : res->r.cores) cores.push_back(c.get());
        ttg::write_train_file(path, res->r.core_dims, cores);
    });
}

ttg_status ttg_comm_nccl_unique_id(unsigned char id[128]) {
    return guard([&] { ttg::nccl_unique_id(id); });
}

ttg_status ttg_comm_nccl_create(const unsigned char id[128], int nranks, int rank, ttg_comm** out) {
    *out = nullptr;
    return guard([&] { *out = new ttg_comm{ttg::make_nccl_comm(id, nranks, rank)}; });
}

ttg_status ttg_comm_callback_create(int nranks, int rank, ttg_host_allgather fn, void* user, ttg_comm** out) {
    *out = nullptr;
    return guard([&] { *out = new ttg_comm{ttg::make_callback_comm(nranks, rank, fn, user)}; });
}

ttg_status ttg_comm_loopback_create(int nranks, ttg_comm** out) {
    return guard([&] {
        auto group = ttg::make_loopback_group(nranks);
        for (int r = 0; r < nranks; ++r) out[r] = new ttg_comm{std::move(group[(size_t)r])};
    });
}

void ttg_comm_free(ttg_comm* comm) { delete comm; }

ttg_status ttg_shard_range(const int64_t* dims, int d, int method, int nranks, int rank, int64_t out[4]) {
    return guard([&] {
        if (d < 0) ttg::argument_error("negative order");
        count_of(dims, d);
        const ttg::ShardRange r = ttg::shard_range(std::vector<int64_t>(dims, dims + d), method, nranks, rank);
        out[0] = r.lo;
        out[1] = r.hi;
        out[2] = r.rows;
        out[3] = r.cols;
    });
}

ttg_status ttg_decompose_sharded(const double* a_local, const int64_t* dims, int d, const ttg_config* cfg,
                                 int a_on_device, ttg_comm* comm, ttg_result** out) {
    *out = nullptr;
    return guard([&] {
        if (!cfg) ttg::argument_error("null config");
        if (!comm || !comm->c) ttg::argument_error("null communicator");
        if (d < 0) ttg::argument_error("negative order");
        const auto start = std::chrono::steady_clock::now();
        std::vector<int64_t> dv(dims, dims + d);
        count_of(dims, d);
        const ttg::SweepConfig sc = sweep_config(cfg);
        const ttg::ShardRange sr = ttg::shard_range(dv, sc.method, comm->c->size(), comm->c->rank());
        DeviceInput in(a_local, sr.rows * sr.cols, a_on_device != 0);
        auto* res = new ttg_result{ttg::decompose_sharded(in.ptr, dv, sc, *comm->c)};
        res->r.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - start).count();
        *out = res;
    });
}

int ttg_result_order(const ttg_result* res) { return (int)res->r.cores.size(); }

void ttg_result_core_dims(const ttg_result* res, int k, int64_t dims3[3]) {
    const auto& c = res->r.core_dims[(size_t)k];
    dims3[0] = c[0];
    dims3[1] = c[1];
    dims3[2] = c[2];
}

ttg_status ttg_result_core_copy(const ttg_result* res, int k, double* host_out) {
    return guard([&] {
        const auto& c = res->r.core_dims[(size_t)k];
        res->r.cores[(size_t)k].download(host_out, (size_t)(c[0] * c[1] * c[2]));
        ttg::sync();
    });
}

const double* ttg_result_core_device(const ttg_result* res, int k) { return res->r.cores[(size_t)k].get(); }

int ttg_result_report(const ttg_result* res, double* step_errors, int64_t* ranks_chosen, int64_t* ranks_requested,
                      double* bound, int* bound_kind, double* input_norm, double* wall_time_ms) {
    const auto& r = res->r;
    if (step_errors) std::copy(r.step_errors.begin(), r.step_errors.end(), step_errors);
    if (ranks_chosen) std::copy(r.ranks_chosen.begin(), r.ranks_chosen.end(), ranks_chosen);
    if (ranks_requested) std::copy(r.ranks_requested.begin(), r.ranks_requested.end(), ranks_requested);
    if (bound) *bound = r.bound;
    if (bound_kind) *bound_kind = r.bound_kind;
    if (input_norm) *input_norm = r.input_norm;
    if (wall_time_ms) *wall_time_ms = r.wall_ms;
    return (int)r.ranks_requested.size();
}

int ttg_result_warning_count(const ttg_result* res) { return (int)res->r.warnings.size(); }
const char* ttg_result_warning(const ttg_result* res, int i) { return res->r.warnings[(size_t)i].c_str(); }

int ttg_result_cut_diag(const ttg_result* res, int cut, double* diag, int max, int64_t info[6]) {
    if (cut < 0 || (size_t)cut >= res->r.cuts.size()) return 0;
    const auto& c = res->r.cuts[(size_t)cut];
    if (info) {
        info[0] = c.steps;
        info[1] = c.p;
        info[2] = c.rank;
        info[3] = c.extensions;
        info[4] = c.m;
        info[5] = c.n;
    }
    const int n = std::min<int>(max, (int)c.diag.size());
    for (int i = 0; i < n; ++i) diag[i] = c.diag[(size_t)i];
    return n;
}

int ttg_result_direct_errors(const ttg_result* res, double* out) {
    const auto& cuts = res->r.cuts;
    if (out)
        for (size_t i = 0; i < cuts.size(); ++i) out[i] = cuts[i].direct_error;
    return (int)cuts.size();
}

int ttg_result_cut_kept(const ttg_result* res, int cut, double* kept, int max) {
    if (cut < 0 || (size_t)cut >= res->r.cuts.size()) return 0;
    const auto& k = res->r.cuts[(size_t)cut].kept;
    const int n = std::min<int>(max, (int)k.size());
    for (int i = 0; i < n; ++i) kept[i] = k[(size_t)i];
    return (int)k.size();
}

ttg_status ttg_result_rse(const ttg_result* res, const double* a, int a_on_device, double* rse) {
    return guard([&] {
        int64_t n = 1;
        for (int64_t v : res->r.dims) n *= v;
        DeviceInput in(a, n, a_on_device != 0);
        const double denom = std::sqrt(ttg::sum_squares(in.ptr, n));
        if (denom == 0.0) ttg::argument_error("rse: truth has zero norm (domain error)");
        *rse = std::sqrt(ttg::residual_squared(res->r, in.ptr)) / denom;
    });
}

ttg_status ttg_result_reconstruct(const ttg_result* res, double* out, int out_on_device) {
    return guard([&] {
        int64_t n = 1;
        for (int64_t v : res->r.dims) n *= v;
        std::vector<const double*> cores;
        std::vector<int64_t> ranks{1};
        for (size_t k = 0; k < res->r.cores.size(); ++k) {
            cores.push_back(res->r.cores[k].get());
            ranks.push_back(res->r.core_dims[k][2]);
        }
        if (out_on_device) {
            ttg::reconstruct(cores, res->r.dims, ranks, out);
        } else {
            ttg::DevBuf<double> o((size_t)n);
            ttg::reconstruct(cores, res->r.dims, ranks, o.get());
            o.download(out, (size_t)n);
        }
        ttg::sync();
    });
}

ttg_status ttg_completion_reset(double* y, const double* observed, const double* mask, const double* truth,
                                int64_t n, double stats[5]) {
    return guard([&] {
        ttg::completion_reset(y, observed, mask, truth, n, stats);
        ttg::sync();
    });
}

ttg_status ttg_verify_bound(const double* a, int a_on_device, const ttg_result* res, double slack_rel,
                            double* achieved) {
    return guard([&] {
        int64_t n = 1;
        for (int64_t v : res->r.dims) n *= v;
        DeviceInput in(a, n, a_on_device != 0);
        const double ach = std::sqrt(ttg::residual_squared(res->r, in.ptr));
        *achieved = ach;
        const double allowed = res->r.bound + slack_rel * res->r.input_norm;
        if (ach > allowed) {
            char buf[256];
            std::snprintf(buf, sizeof buf, "achieved error %.12e exceeds bound %.12e plus slack %.3e", ach,
                          res->r.bound, slack_rel * res->r.input_norm);
            ttg::fail(6, buf);
        }
    });
}

ttg_status ttg_qr_col_pivot(const double* a, int64_t m, int64_t n, double* q, double* r, int64_t* perm) {
    return guard([&] {
        if (m <= 0 || n <= 0) ttg::argument_error("qr_col_pivot: empty matrix");
        const int64_t p = std::min(m, n);
        ttg::DevBuf<double> A((size_t)(m * n));
        A.upload(a, (size_t)(m * n));
        if (m <= 4096) {
            ttg::WideQrcp e1(A.get(), m, n, m, ttg::Layout::Col, p);
            e1.run_to(p);
            if (q) {
                ttg::DevBuf<double> hq;
                TTG_CUDA(cudaMemcpyAsync(q, e1.Q(), sizeof(double) * m * p, cudaMemcpyDeviceToHost, ttg::stream()));
            }
            if (r || perm) {
                std::vector<int64_t> pm((size_t)n);
                TTG_CUDA(cudaMemcpyAsync(pm.data(), e1.perm(), sizeof(int64_t) * n, cudaMemcpyDeviceToHost,
                                         ttg::stream()));
                std::vector<double> rr((size_t)(p * n));
                TTG_CUDA(cudaMemcpyAsync(rr.data(), e1.R(), sizeof(double) * p * n, cudaMemcpyDeviceToHost,
                                         ttg::stream()));
                ttg::sync();
                if (perm) std::copy(pm.begin(), pm.end(), perm);
                if (r)  // R(i, pos) = R1 row i at column perm[pos] (exact zeros below the diagonal)
                    for (int64_t j = 0; j < n; ++j)
                        for (int64_t i = 0; i < p; ++i) r[i + j * p] = rr[(size_t)(i * n + pm[(size_t)j])];
            }
            ttg::sync();
        } else {
            ttg::TallQrcp e2(A.get(), m, n, m);
            e2.run(p);
            if (r) {
                ttg::DevBuf<double> R((size_t)(p * n));
                e2.extract_r(R.get(), p);
                R.download(r, (size_t)(p * n));
            }
            if (perm) TTG_CUDA(cudaMemcpyAsync(perm, e2.perm(), sizeof(int64_t) * n, cudaMemcpyDeviceToHost, ttg::stream()));
            if (q) {
                ttg::DevBuf<double> Q((size_t)(m * p));
                e2.form_q(Q.get(), p, m);
                Q.download(q, (size_t)(m * p));
            }
            ttg::sync();
        }
    });
}

ttg_status ttg_utv(const double* a, int64_t m, int64_t n, int lower, int refine, double* u, double* t, double* v) {
    return guard([&] {
        if (m <= 0 || n <= 0) ttg::argument_error("utv: empty matrix");
        DeviceInput in(a, m * n, false);
        ttg::DUtv f = ttg::utv(in.ptr, m, n, lower != 0, refine);
        if (u) f.u.buf.download(u, (size_t)(f.u.rows * f.u.cols));
        if (t) f.t.buf.download(t, (size_t)(f.t.rows * f.t.cols));
        if (v) f.v.buf.download(v, (size_t)(f.v.rows * f.v.cols));
        ttg::sync();
    });
}

ttg_status ttg_svd(const double* a, int64_t m, int64_t n, int max_sweeps, double pair_tol, double* u, double* s,
                   double* v) {
    return guard([&] {
        if (m <= 0 || n <= 0) ttg::argument_error("svd: empty matrix");
        DeviceInput in(a, m * n, false);
        ttg::DSvd f = ttg::svd(in.ptr, m, n, max_sweeps, pair_tol);
        if (u) f.u.buf.download(u, (size_t)(f.u.rows * f.u.cols));
        if (v) f.v.buf.download(v, (size_t)(f.v.rows * f.v.cols));
        if (s) std::copy(f.s.begin(), f.s.end(), s);
        ttg::sync();
    });
}

ttg_status ttg_truncate(int kind, const double* u, const double* t, const double* v, int64_t m, int64_t n, int64_t p,
                        int64_t rank, double eps, int64_t* rank_out, double* residual, double* u1, double* t11,
                        double* v1) {
    return guard([&] {
        if (kind < 0 || kind > 2) ttg::argument_error("unknown factor kind");
        if (rank < 0 || rank > p)
            ttg::argument_error("rank " + std::to_string(rank) + " out of range 1.." + std::to_string(p));
        DeviceInput dt(t, kind == 0 ? p : p * p, false);
        const ttg::DTrunc tr = ttg::truncate_rank(kind, dt.ptr, p, rank, eps);
        const int64_t r = tr.rank;
        *rank_out = r;
        *residual = tr.residual;
        // leading blocks (factor.cpp:458-469): column-major prefixes of the caller's factors
        if (u1) std::memcpy(u1, u, sizeof(double) * (size_t)(m * r));
        if (v1) std::memcpy(v1, v, sizeof(double) * (size_t)(n * r));
        if (t11)
            for (int64_t j = 0; j < r; ++j)
                for (int64_t i = 0; i < r; ++i)
                    t11[i + j * r] = kind == 0 ? (i == j ? t[i] : 0.0) : t[i + j * p];
    });
}

ttg_status ttg_reconstruct(const double* cores, const int64_t* dims, const int64_t* ranks, int d, int64_t element_cap,
                           double* out) {
    return guard([&] {
        if (d < 1) ttg::argument_error("train needs at least one core");
        if (ranks[0] != 1 || ranks[d] != 1) ttg::argument_error("boundary ranks must both be 1");
        const int64_t n = count_of(dims, d);
        if (n > element_cap)
            ttg::fail(5, "reconstruct would materialize " + std::to_string(n) + " elements (cap " +
                             std::to_string(element_cap) + ")");
        int64_t total = 0;
        for (int k = 0; k < d; ++k) total += ranks[k] * dims[k] * ranks[k + 1];
        ttg::DevBuf<double> C((size_t)total), O((size_t)n);
        C.upload(cores, (size_t)total);
        std::vector<const double*> cp;
        int64_t off = 0;
        for (int k = 0; k < d; ++k) {
            cp.push_back(C.get() + off);
            off += ranks[k] * dims[k] * ranks[k + 1];
        }
        ttg::reconstruct(cp, std::vector<int64_t>(dims, dims + d), std::vector<int64_t>(ranks, ranks + d + 1), O.get());
        O.download(out, (size_t)n);
        ttg::sync();
    });
}

ttg_status ttg_frobenius_norm(const double* a, int64_t count, int a_on_device, double* out) {
    return guard([&] {
        DeviceInput in(a, count, a_on_device != 0);
        *out = std::sqrt(ttg::sum_squares(in.ptr, count));
    });
}

ttg_status ttg_sum_squares(const double* a, int64_t count, int a_on_device, double* out) {
    return guard([&] {
        DeviceInput in(a, count, a_on_device != 0);
        *out = count > 0 ? ttg::sum_squares(in.ptr, count) : 0.0;
    });
}

ttg_status ttg_diff_norm(const double* x, const double* y, int64_t count, double* out) {
    return guard([&] {
        DeviceInput a(x, count, false), b(y, count, false);
        *out = std::sqrt(ttg::diff_squares(a.ptr, b.ptr, count));
    });
}

ttg_status ttg_matmul(const double* a, int64_t ar, int64_t ac, int ta, const double* b, int64_t br, int64_t bc, int tb,
                      double* c) {
    return guard([&] {
        const int64_t m = ta ? ac : ar, k = ta ? ar : ac, kb = tb ? bc : br, n = tb ? br : bc;
        if (k != kb) ttg::argument_error("matmul inner dimensions do not match");
        ttg::DevBuf<double> A((size_t)(ar * ac)), B((size_t)(br * bc)), Cc((size_t)(m * n));
        A.upload(a, (size_t)(ar * ac));
        B.upload(b, (size_t)(br * bc));
        if (k == 0) Cc.zero();
        else ttg::gemm(ta != 0, tb != 0, m, n, k, A.get(), ar, B.get(), br, Cc.get(), m);
        Cc.download(c, (size_t)(m * n));
        ttg::sync();
    });
}

ttg_status ttg_gemm_device(int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
                           int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
    return guard([&] {
        if (m < 0 || n < 0 || k < 0) ttg::argument_error("matrix dims must be nonnegative");
        if (k == 0) {
            if (beta == 0.0)
                for (int64_t j = 0; j < n; ++j)
                    TTG_CUDA(cudaMemsetAsync(C + j * ldc, 0, sizeof(double) * (size_t)m, ttg::stream()));
            return;
        }
        ttg::gemm(ta != 0, tb != 0, m, n, k, A, lda, B, ldb, C, ldc, alpha, beta);
    });
}

ttg_status ttg_rse(const double* estimate, const double* truth, int64_t count, double* out) {
    return guard([&] {
        DeviceInput e(estimate, count, false), t(truth, count, false);
        const double denom = std::sqrt(ttg::sum_squares(t.ptr, count));
        if (denom == 0.0) ttg::argument_error("rse: truth has zero norm (domain error)");
        *out = std::sqrt(ttg::diff_squares(e.ptr, t.ptr, count)) / denom;
    });
}

ttg_status ttg_mode_product(const double* x, const int64_t* dims, int d, int k, const double* m, int64_t m_rows,
                            int64_t m_cols, double* out) {
    return guard([&] {
        if (k < 1 || k > d)
            ttg::argument_error("mode " + std::to_string(k) + " out of range 1.." + std::to_string(d));
        if (m_cols != dims[k - 1])
            ttg::argument_error("mode-" + std::to_string(k) + " product needs " + std::to_string(dims[k - 1]) +
                                " columns, matrix has " + std::to_string(m_cols));
        int64_t left = 1, right = 1;
        for (int q = 0; q < k - 1; ++q) left *= dims[q];
        for (int q = k; q < d; ++q) right *= dims[q];
        const int64_t mid = dims[k - 1], n_in = left * mid * right, n_out = left * m_rows * right;
        ttg::DevBuf<double> X((size_t)std::max<int64_t>(n_in, 1)), M((size_t)std::max<int64_t>(m_rows * m_cols, 1)),
            O((size_t)std::max<int64_t>(n_out, 1));
        X.upload(x, (size_t)n_in);
        M.upload(m, (size_t)(m_rows * m_cols));
        ttg::mode_product_dev(X.get(), left, mid, right, M.get(), m_rows, O.get());
        O.download(out, (size_t)n_out);
        ttg::sync();
    });
}

ttg_status ttg_kron(const double* a, int64_t ar, int64_t ac, const double* b, int64_t br, int64_t bc, double* out) {
    return guard([&] {
        const int64_t na = ar * ac, nb = br * bc, n = na * nb;
        ttg::DevBuf<double> A((size_t)std::max<int64_t>(na, 1)), B((size_t)std::max<int64_t>(nb, 1)),
            O((size_t)std::max<int64_t>(n, 1));
        A.upload(a, (size_t)na);
        B.upload(b, (size_t)nb);
        ttg::kron_dev(A.get(), ar, ac, B.get(), br, bc, O.get());
        O.download(out, (size_t)n);
        ttg::sync();
    });
}

ttg_status ttg_psnr(const double* estimate, const double* truth, int64_t count, double* out) {
    return guard([&] {
        if (count < 1) ttg::argument_error("psnr: empty tensors");
        DeviceInput e(estimate, count, false), t(truth, count, false);
        const double max_val = ttg::max_value_dev(t.ptr, count);
        const double mse = ttg::diff_squares(e.ptr, t.ptr, count) / (double)count;
        *out = mse == 0.0 ? std::numeric_limits<double>::infinity() : 10.0 * std::log10(max_val * max_val / mse);
    });
}

ttg_status ttg_reverse_indices(const double* a, const int64_t* dims, int d, double* out) {
    return guard([&] {
        const int64_t n = count_of(dims, d);
        DeviceInput in(a, n, false);
        ttg::DevBuf<double> O((size_t)std::max<int64_t>(n, 1));
        ttg::reverse_indices_dev(in.ptr, std::vector<int64_t>(dims, dims + d), O.get());
        O.download(out, (size_t)n);
        ttg::sync();
    });
}

ttg_status ttg_reverse_tt(const double* cores, const int64_t* dims, const int64_t* ranks, int d, double* out) {
    return guard([&] {
        int64_t total = 0;
        for (int k = 0; k < d; ++k) total += ranks[k] * dims[k] * ranks[k + 1];
        ttg::DevBuf<double> C((size_t)std::max<int64_t>(total, 1)), O((size_t)std::max<int64_t>(total, 1));
        C.upload(cores, (size_t)total);
        // core k of the result is core d-1-k flipped; the output is packed in the new order
        int64_t off_out = 0;
        for (int k = 0; k < d; ++k) {
            const int src = d - 1 - k;
            int64_t off_in = 0;
            for (int q = 0; q < src; ++q) off_in += ranks[q] * dims[q] * ranks[q + 1];
            const int64_t rl = ranks[src], mid = dims[src], rr = ranks[src + 1];
            ttg::flip_core_dev(C.get() + off_in, rl, mid, rr, O.get() + off_out);
            off_out += rl * mid * rr;
        }
        O.download(out, (size_t)total);
        ttg::sync();
    });
}

ttg_status ttg_complete(const int64_t* linear, const double* values, int64_t count, const int64_t* dims, int d,
                        const ttg_completion_config* cfg, const double* truth, int on_device, ttg_completion** out) {
    *out = nullptr;
    return guard([&] {
        if (d < 1) ttg::argument_error("shape needs at least one mode");
        ttg::CompletionSpec spec;
        if (cfg->nranks > 0) spec.ranks.assign(cfg->ranks, cfg->ranks + cfg->nranks);
        spec.adaptive = cfg->nranks == 0;
        spec.eps = cfg->eps;
        spec.retraction = cfg->retraction;
        spec.step_size = cfg->step_size;
        spec.max_iters = cfg->max_iters;
        spec.stop_tol = cfg->stop_tol;
        spec.refine_passes = cfg->refine_passes;
        spec.dense_cap = cfg->dense_cap;
        const int64_t n = count_of(dims, d);
        ttg::DevBuf<int64_t> L;
        const int64_t* lp = linear;
        if (!on_device) {
            for (int64_t i = 0; i < count; ++i)
                if (linear[i] < 0 || linear[i] >= n || (i > 0 && linear[i] <= linear[i - 1]))
                    ttg::argument_error("observation indices must be 0-based, in range and strictly increasing");
            L.alloc((size_t)std::max<int64_t>(count, 1));
            L.upload(linear, (size_t)count);
            lp = L.get();
        }
        DeviceInput V(values, count, on_device != 0);
        ttg::DevBuf<double> T;
        const double* tp = truth;
        if (truth && !on_device) {
            T.alloc((size_t)n);
            T.upload(truth, (size_t)n);
            tp = T.get();
        }
        auto* c = new ttg_completion{ttg::complete(lp, V.ptr, count, std::vector<int64_t>(dims, dims + d), spec, tp), {}};
        c->res.r = std::move(c->run.tt);
        c->res.r.dims.assign(dims, dims + d);
        *out = c;
    });
}

void ttg_completion_free(ttg_completion* c) { delete c; }
int ttg_completion_iterations(const ttg_completion* c) { return (int)c->run.rse_observed.size(); }
int ttg_completion_status(const ttg_completion* c) { return c->run.status; }
const char* ttg_completion_note(const ttg_completion* c) { return c->run.note.c_str(); }

void ttg_completion_trace(const ttg_completion* c, double* rse_observed, double* rse_full, double* psnr,
                          double* wall_time_ms, double* initial3) {
    const auto& r = c->run;
    if (rse_observed) std::copy(r.rse_observed.begin(), r.rse_observed.end(), rse_observed);
    if (rse_full) std::copy(r.rse_full.begin(), r.rse_full.end(), rse_full);
    if (psnr) std::copy(r.psnr.begin(), r.psnr.end(), psnr);
    if (wall_time_ms) std::copy(r.wall_ms.begin(), r.wall_ms.end(), wall_time_ms);
    if (initial3) {
        initial3[0] = r.initial_obs.empty() ? 0.0 : r.initial_obs[0];
        initial3[1] = r.initial_full.empty() ? 0.0 : r.initial_full[0];
        initial3[2] = r.initial_psnr.empty() ? 0.0 : r.initial_psnr[0];
    }
}

int ttg_completion_ranks(const ttg_completion* c, int iter, int64_t* ranks) {
    if (iter < 0 || (size_t)iter >= c->run.ranks.size()) return 0;
    const auto& r = c->run.ranks[(size_t)iter];
    std::copy(r.begin(), r.end(), ranks);
    return (int)r.size();
}

const ttg_result* ttg_completion_result(const ttg_completion* c) { return &c->res; }

}  // extern "C"
