// Per-thread CUDA stream, device properties and the launch counter.
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
