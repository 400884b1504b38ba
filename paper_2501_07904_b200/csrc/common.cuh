// Shared host/device plumbing for the TT-UTV engine: status exceptions, the per-thread
// stream, stream-ordered device buffers and warp/block reduction helpers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace ttg {

// Internal exception carrying a ttg_status code; translated at the C-ABI boundary.
struct Failure : std::runtime_error {
    int code;
    Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Failure(code, msg); }
inline void argument_error(const std::string& msg) { fail(1, msg); }
[[noreturn]] inline void resource_error(const std::string& msg) { fail(5, msg); }
[[noreturn]] inline void invariant_error(const std::string& msg) { fail(6, msg); }

#define TTG_CUDA(expr)                                                                   \
    do {                                                                                 \
        cudaError_t _e = (expr);                                                         \
        if (_e != cudaSuccess)                                                           \
            ::ttg::fail(8, std::string("CUDA error: ") + cudaGetErrorString(_e) + " at " + \
                               __FILE__ + ":" + std::to_string(__LINE__));               \
    } while (0)

// Every kernel launch goes through this macro so the launch counter is exact and
// launch errors surface immediately.
#define TTG_LAUNCH(kernel, grid, block, smem, stream, ...)                               \
    do {                                                                                 \
        kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                      \
        ::ttg::count_launch();                                                           \
        TTG_CUDA(cudaGetLastError());                                                    \
        if (::ttg::debug_sync()) ::ttg::check_sync(#kernel, __FILE__, __LINE__);        \
    } while (0)

void count_launch();
int64_t launches();
// TTG_DEBUG_SYNC=1: synchronise after every launch and name the failing kernel.
bool debug_sync();
void check_sync(const char* kernel, const char* file, int line);

// Opt a kernel into large dynamic shared memory. Static + dynamic may not exceed 48 KB
// without the opt-in, so any request above 40 KB (kernels keep <= 8 KB static) opts in.
// The attribute is process-wide: it is raised once to the device's opt-in maximum (minus
// the kernel's static shared memory) and never lowered, so concurrent host threads
// launching the same kernel with different sizes cannot undercut each other.
void raise_smem_limit(const void* kernel);
template <class K>
inline void allow_smem(K* kernel, size_t bytes) {
    if (bytes > 40 * 1024) raise_smem_limit(reinterpret_cast<const void*>(kernel));
}

// Stream of the calling host thread (created lazily on the current device).
cudaStream_t stream();
int sm_count();
// Make sure this device's stream-ordered pool holds at least `bytes` (capped at half the
// free memory): growing the pool maps new memory at ~10-40 ms per GB, and a pool grown
// piecemeal by differently sized requests keeps growing; one up-front block does not.
void ensure_pool(size_t bytes);

// Optional event timing of the dominant (pass-1 streaming) kernel for the roofline report:
// when enabled, prof_begin/prof_end bracket each launch with CUDA events on the launching
// stream and accumulate the algorithmic bytes of that launch.
bool prof_enabled();
void prof_enable(bool on);
void prof_begin();
void prof_end(double algorithmic_bytes, const char* kernel);
// prof_end for a launch whose work is chosen on the device: the int at `dflag` (read after
// the launch, stream-ordered) selects kernel1/bytes1 (non-zero) or kernel0/bytes0 (zero).
void prof_end_select(const int* dflag, double bytes1, const char* kernel1, double bytes0, const char* kernel0);
// Drains the recorded events (host sync). Returns launches; total device ms and bytes.
// The drained records also accumulate into per-kernel totals (prof_kernels).
int64_t prof_read(double* total_ms, double* bytes);
int prof_kernels(int max, const char** names, double* ms, double* bytes, int64_t* launches);
void prof_reset_kernels();
// Persistent pass-1 loop phase totals (ms): out[v*3 + {0 reflector, 1 stream, 2 guard}]
// for k_pass1_big<v>, v < 8 (host sync); reset zeroes them.
void big_phase_stats(double* out, bool reset);

// TTG_PHASES=1 (diagnostics): event-timed phases on the thread's stream, totals printed at
// exit. Use as `PhaseTimer pt("name");` around a phase.
bool phases_on();
cudaEvent_t phase_mark();
void phase_add(cudaEvent_t begin, const char* name);
struct PhaseTimer {
    cudaEvent_t a = nullptr;
    const char* name;
    explicit PhaseTimer(const char* n) : name(n) {
        if (phases_on()) a = phase_mark();
    }
    ~PhaseTimer() {
        if (a) phase_add(a, name);
    }
};

// Stream-ordered device allocation (cudaMallocAsync on the thread's stream).
template <class T>
class DevBuf {
public:
    DevBuf() = default;
    explicit DevBuf(size_t n) { alloc(n); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); p_ = o.p_; n_ = o.n_; o.p_ = nullptr; o.n_ = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t n) {
        release();
        n_ = n;
        if (n) TTG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), n * sizeof(T), stream()));
    }
    void zero() {
        if (n_) TTG_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(T), stream()));
    }
    void release() {
        if (p_) cudaFreeAsync(p_, stream());
        p_ = nullptr;
        n_ = 0;
    }
    T* get() const { return p_; }
    size_t size() const { return n_; }
    void upload(const T* host, size_t n, size_t offset = 0) {
        if (n) TTG_CUDA(cudaMemcpyAsync(p_ + offset, host, n * sizeof(T), cudaMemcpyHostToDevice, stream()));
    }
    void download(T* host, size_t n, size_t offset = 0) const {
        if (n) TTG_CUDA(cudaMemcpyAsync(host, p_ + offset, n * sizeof(T), cudaMemcpyDeviceToHost, stream()));
    }
    std::vector<T> to_host(size_t n) const {
        std::vector<T> h(n);
        download(h.data(), n);
        sync();
        return h;
    }
    static void sync() { TTG_CUDA(cudaStreamSynchronize(stream())); }

private:
    T* p_ = nullptr;
    size_t n_ = 0;
};

inline void sync() { TTG_CUDA(cudaStreamSynchronize(stream())); }

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------------------
// Device helpers
// ---------------------------------------------------------------------------

// One FP64 tensor-core MMA, D(8x8) += A(8x4) B(4x8): lane l holds A[l/4][l%4], B[l%4][l/4]
// and D[l/4][2(l%4) + {0,1}] (mma.sync m8n8k4 f64 -> SASS DMMA on sm_100a).
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Fixed-shape block reduction (deterministic: the same tree for every call).
// `scratch` must hold blockDim.x/32 doubles. Result valid in every thread.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    double t = lane < nw ? scratch[lane] : 0.0;
    t = warp_sum(t);
    return t;
}

// Pivot candidate: larger squared norm wins, ties go to the lowest position
// (reference: strict '>' scan from the current step, factor.cpp:85-87).
struct Cand {
    double nu;
    int64_t pos;
    int64_t col;
};

__device__ __forceinline__ bool better(const Cand& a, const Cand& b) {
    return a.nu > b.nu || (a.nu == b.nu && a.pos < b.pos);
}

__device__ __forceinline__ Cand cand_none() { return Cand{-1.0, INT64_MAX, -1}; }

__device__ __forceinline__ Cand warp_best(Cand c) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        Cand x;
        x.nu = __shfl_xor_sync(0xffffffffu, c.nu, o);
        x.pos = __shfl_xor_sync(0xffffffffu, c.pos, o);
        x.col = __shfl_xor_sync(0xffffffffu, c.col, o);
        if (better(x, c)) c = x;
    }
    return c;
}

// Block-wide best candidate; `scratch` holds blockDim.x/32 Cands. Valid in all threads.
__device__ __forceinline__ Cand block_best(Cand c, Cand* scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    c = warp_best(c);
    __syncthreads();
    if (lane == 0) scratch[warp] = c;
    __syncthreads();
    Cand t = lane < nw ? scratch[lane] : cand_none();
    return warp_best(t);
}

}  // namespace ttg
