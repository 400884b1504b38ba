// Per-thread CUDA stream, device properties and the launch counter.
#include <mutex>
#include <string>
#include <algorithm>
#include <vector>
#include <atomic>
#include <cstdlib>

#include "common.cuh"

namespace ttg {

namespace {
std::atomic<int64_t> g_launches{0};

struct ThreadStream {
    cudaStream_t s = nullptr;
    int device = -1;
    ~ThreadStream() {
        if (s) cudaStreamDestroy(s);
    }
};
thread_local ThreadStream t_stream;
}  // namespace

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

bool debug_sync() {
    static const bool on = [] {
        const char* e = std::getenv("TTG_DEBUG_SYNC");
        return e && *e && *e != '0';
    }();
    return on;
}

void check_sync(const char* kernel, const char* file, int line) {
    const cudaError_t e = cudaStreamSynchronize(stream());
    if (e != cudaSuccess)
        fail(8, std::string("CUDA error after ") + kernel + " (" + file + ":" + std::to_string(line) +
                    "): " + cudaGetErrorString(e));
}
int64_t launches() { return g_launches.load(std::memory_order_relaxed); }

cudaStream_t stream() {
    int dev = 0;
    TTG_CUDA(cudaGetDevice(&dev));
    if (!t_stream.s || t_stream.device != dev) {
        if (t_stream.s) cudaStreamDestroy(t_stream.s);
        TTG_CUDA(cudaStreamCreateWithFlags(&t_stream.s, cudaStreamNonBlocking));
        t_stream.device = dev;
        // Keep freed blocks cached in the stream-ordered pool between calls.
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    return t_stream.s;
}

namespace {
struct Prof {
    bool on = false;
    struct Rec {
        cudaEvent_t a, b;
        double bytes;
        int kind;
        // kind chosen on the device: flag (pinned host copy) != 0 -> kind/bytes, else alt
        int* flag = nullptr;
        double alt_bytes = 0.0;
        int alt_kind = -1;
    };
    std::vector<int*> flag_pool;  // pinned host ints for device-selected records
    int* get_flag() {
        if (flag_pool.empty()) {
            int* blk = nullptr;
            TTG_CUDA(cudaMallocHost(&blk, sizeof(int) * 256));
            for (int i = 0; i < 256; ++i) flag_pool.push_back(blk + i);
        }
        int* f = flag_pool.back();
        flag_pool.pop_back();
        return f;
    }
    std::vector<Rec> pending;
    std::vector<cudaEvent_t> pool;
    cudaEvent_t open = nullptr;
    cudaEvent_t get() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        TTG_CUDA(cudaEventCreate(&e));
        return e;
    }
    // per-kernel totals of the drained records
    std::vector<std::string> names;
    std::vector<double> kms, kbytes;
    std::vector<int64_t> kcount;
    int kind_of(const char* name) {
        for (size_t i = 0; i < names.size(); ++i)
            if (names[i] == name) return (int)i;
        names.emplace_back(name);
        kms.push_back(0.0);
        kbytes.push_back(0.0);
        kcount.push_back(0);
        return (int)names.size() - 1;
    }
};
thread_local Prof t_prof;
}  // namespace

bool prof_enabled() { return t_prof.on; }
void prof_enable(bool on) { t_prof.on = on; }

void prof_begin() {
    if (!t_prof.on) return;
    t_prof.open = t_prof.get();
    TTG_CUDA(cudaEventRecord(t_prof.open, stream()));
}

void prof_end(double algorithmic_bytes, const char* kernel) {
    if (!t_prof.on || !t_prof.open) return;
    cudaEvent_t e = t_prof.get();
    TTG_CUDA(cudaEventRecord(e, stream()));
    t_prof.pending.push_back({t_prof.open, e, algorithmic_bytes, t_prof.kind_of(kernel)});
    t_prof.open = nullptr;
}

void prof_end_select(const int* dflag, double bytes1, const char* kernel1, double bytes0, const char* kernel0) {
    if (!t_prof.on || !t_prof.open) return;
    int* f = t_prof.get_flag();
    TTG_CUDA(cudaMemcpyAsync(f, dflag, sizeof(int), cudaMemcpyDeviceToHost, stream()));
    cudaEvent_t e = t_prof.get();
    TTG_CUDA(cudaEventRecord(e, stream()));
    Prof::Rec r{t_prof.open, e, bytes1, t_prof.kind_of(kernel1)};
    r.flag = f;
    r.alt_bytes = bytes0;
    r.alt_kind = t_prof.kind_of(kernel0);
    t_prof.pending.push_back(r);
    t_prof.open = nullptr;
}

int64_t prof_read(double* total_ms, double* bytes) {
    double ms = 0.0, by = 0.0;
    for (auto& r : t_prof.pending) {
        TTG_CUDA(cudaEventSynchronize(r.b));
        if (r.flag) {
            if (*r.flag == 0) {
                r.bytes = r.alt_bytes;
                r.kind = r.alt_kind;
            }
            t_prof.flag_pool.push_back(r.flag);
        }
        float x = 0.f;
        TTG_CUDA(cudaEventElapsedTime(&x, r.a, r.b));
        ms += x;
        by += r.bytes;
        t_prof.kms[(size_t)r.kind] += x;
        t_prof.kbytes[(size_t)r.kind] += r.bytes;
        t_prof.kcount[(size_t)r.kind] += 1;
        t_prof.pool.push_back(r.a);
        t_prof.pool.push_back(r.b);
    }
    const int64_t n = (int64_t)t_prof.pending.size();
    t_prof.pending.clear();
    *total_ms = ms;
    *bytes = by;
    return n;
}

int prof_kernels(int max, const char** names, double* ms, double* bytes, int64_t* launches) {
    const int n = (int)t_prof.names.size();
    for (int i = 0; i < n && i < max; ++i) {
        names[i] = t_prof.names[(size_t)i].c_str();
        ms[i] = t_prof.kms[(size_t)i];
        bytes[i] = t_prof.kbytes[(size_t)i];
        launches[i] = t_prof.kcount[(size_t)i];
    }
    return n;
}

void prof_reset_kernels() {
    std::fill(t_prof.kms.begin(), t_prof.kms.end(), 0.0);
    std::fill(t_prof.kbytes.begin(), t_prof.kbytes.end(), 0.0);
    std::fill(t_prof.kcount.begin(), t_prof.kcount.end(), 0);
}

void raise_smem_limit(const void* kernel) {
    static std::mutex mu;
    static std::vector<std::pair<const void*, int>> done;  // (kernel, device)
    int dev = 0;
    TTG_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    for (const auto& d : done)
        if (d.first == kernel && d.second == dev) return;
    int optin = 0;
    TTG_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa{};
    TTG_CUDA(cudaFuncGetAttributes(&fa, kernel));
    TTG_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  optin - (int)fa.sharedSizeBytes));
    done.emplace_back(kernel, dev);
}

void ensure_pool(size_t bytes) {
    static std::mutex mu;
    static size_t reserved[64] = {};
    int dev = 0;
    TTG_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 0 || dev >= 64 || bytes <= reserved[dev]) return;
    size_t free_b = 0, total_b = 0;
    TTG_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const size_t want = std::min(bytes, free_b / 2);
    if (want <= reserved[dev]) return;
    void* p = nullptr;
    if (cudaMallocAsync(&p, want, stream()) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    TTG_CUDA(cudaFreeAsync(p, stream()));
    reserved[dev] = want;
}

int sm_count() {
    static thread_local int cached = 0, cached_dev = -1;
    int dev = 0;
    TTG_CUDA(cudaGetDevice(&dev));
    if (cached_dev != dev) {
        TTG_CUDA(cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev));
        cached_dev = dev;
    }
    return cached;
}

}  // namespace ttg

// ---- TTG_PHASES=1: event-timed pass-1 phases (diagnostics; printed at exit) ----------
namespace ttg {
namespace {
struct Phases {
    struct Rec {
        cudaEvent_t a, b;
        int kind;
    };
    std::mutex mu;
    std::vector<Rec> recs;
    std::vector<std::string> names;
    std::vector<double> ms;
    std::vector<int64_t> n;
    ~Phases() {
        if (recs.empty()) return;
        for (auto& r : recs) {
            float x = 0.f;
            if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&x, r.a, r.b) != cudaSuccess) break;
            ms[(size_t)r.kind] += x;
            n[(size_t)r.kind] += 1;
        }
        for (size_t i = 0; i < names.size(); ++i)
            std::fprintf(stderr, "[ttg phase] %-28s n=%7lld total=%9.3f ms avg=%8.2f us\n", names[i].c_str(),
                         (long long)n[i], ms[i], n[i] ? 1e3 * ms[i] / (double)n[i] : 0.0);
    }
};
Phases g_phases;
}  // namespace

bool phases_on() {
    static const bool on = [] {
        const char* e = std::getenv("TTG_PHASES");
        return e && *e == '1';
    }();
    return on;
}

cudaEvent_t phase_mark() {
    cudaEvent_t e;
    TTG_CUDA(cudaEventCreate(&e));
    TTG_CUDA(cudaEventRecord(e, stream()));
    return e;
}

void phase_add(cudaEvent_t a, const char* name) {
    cudaEvent_t b = phase_mark();
    std::lock_guard<std::mutex> lk(g_phases.mu);
    int kind = -1;
    for (size_t i = 0; i < g_phases.names.size(); ++i)
        if (g_phases.names[i] == name) kind = (int)i;
    if (kind < 0) {
        g_phases.names.emplace_back(name);
        g_phases.ms.push_back(0.0);
        g_phases.n.push_back(0);
        kind = (int)g_phases.names.size() - 1;
    }
    g_phases.recs.push_back({a, b, kind});
}
}  // namespace ttg
