// Per-thread CUDA stream, device properties and the launch counter.
#include <mutex>
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
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
    std::vector<cudaEvent_t> pool;
    cudaEvent_t open = nullptr;
    double bytes = 0.0;
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

void prof_end(double algorithmic_bytes) {
    if (!t_prof.on || !t_prof.open) return;
    cudaEvent_t e = t_prof.get();
    TTG_CUDA(cudaEventRecord(e, stream()));
    t_prof.pending.emplace_back(t_prof.open, e);
    t_prof.open = nullptr;
    t_prof.bytes += algorithmic_bytes;
}

int64_t prof_read(double* total_ms, double* bytes) {
    double ms = 0.0;
    for (auto& pr : t_prof.pending) {
        TTG_CUDA(cudaEventSynchronize(pr.second));
        float x = 0.f;
        TTG_CUDA(cudaEventElapsedTime(&x, pr.first, pr.second));
        ms += x;
        t_prof.pool.push_back(pr.first);
        t_prof.pool.push_back(pr.second);
    }
    const int64_t n = (int64_t)t_prof.pending.size();
    t_prof.pending.clear();
    *total_ms = ms;
    *bytes = t_prof.bytes;
    t_prof.bytes = 0.0;
    return n;
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
