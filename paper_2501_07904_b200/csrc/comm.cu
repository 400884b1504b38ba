// Multi-GPU plumbing for the sharded sweep.
//
// The data path needs one primitive: an all-gather of a small device buffer (a pivot
// record per pass-1 step, one s x s triangle per pass-2 tree, the carry once per sweep),
// followed on every rank by the same fixed-order combine. NcclComm issues ncclAllGather
// on the engine's stream (NVLink / NVSwitch on a B200 box). NCCL is resolved with dlopen
// when a communicator is created, so the library loads without it and shares the copy
// torch already mapped. LoopbackComm serves tests on one GPU: the endpoints are host
// threads of one process and the exchange is a host barrier around device copies, so no
// kernel ever waits on another kernel.
#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <mutex>

#include "engine.hpp"

namespace ttg {
namespace {

// ---- NCCL (minimal ABI, resolved at run time) --------------------------------------------
struct NcclId {
    char internal[128];
};
using nccl_comm_t = void*;
using nccl_result_t = int;
constexpr int kNcclInt8 = 0;

struct NcclApi {
    nccl_result_t (*get_unique_id)(NcclId*) = nullptr;
    nccl_result_t (*comm_init_rank)(nccl_comm_t*, int, NcclId, int) = nullptr;
    nccl_result_t (*all_gather)(const void*, void*, size_t, int, nccl_comm_t, cudaStream_t) = nullptr;
    nccl_result_t (*comm_destroy)(nccl_comm_t) = nullptr;
    const char* (*error_string)(nccl_result_t) = nullptr;
    nccl_result_t (*send)(const void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
    nccl_result_t (*recv)(void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
    nccl_result_t (*group_start)() = nullptr;
    nccl_result_t (*group_end)() = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) resource_error(std::string("NCCL not available: ") + dlerror());
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        if (!a.get_unique_id || !a.comm_init_rank || !a.all_gather || !a.comm_destroy || !a.error_string)
            resource_error("NCCL library lacks a required symbol");
        // point-to-point (NCCL >= 2.7); absent symbols leave has_p2p() false
        a.send = reinterpret_cast<decltype(a.send)>(dlsym(h, "ncclSend"));
        a.recv = reinterpret_cast<decltype(a.recv)>(dlsym(h, "ncclRecv"));
        a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(h, "ncclGroupStart"));
        a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(h, "ncclGroupEnd"));
        return a;
    }();
    return api;
}

void nccl_check(nccl_result_t r, const char* what) {
    if (r != 0) resource_error(std::string(what) + ": " + nccl().error_string(r));
}

class NcclComm final : public Comm {
public:
    NcclComm(const unsigned char id[128], int nranks, int rank) : rank_(rank), size_(nranks) {
        NcclId uid;
        std::memcpy(uid.internal, id, sizeof(uid.internal));
        nccl_check(nccl().comm_init_rank(&comm_, nranks, uid, rank), "ncclCommInitRank");
    }
    ~NcclComm() override {
        if (comm_) nccl().comm_destroy(comm_);
    }
    int rank() const override { return rank_; }
    int size() const override { return size_; }
    void allgather(const void* send, void* recv, size_t bytes) override {
        nccl_check(nccl().all_gather(send, recv, bytes, kNcclInt8, comm_, stream()), "ncclAllGather");
    }
    bool has_p2p() const override { return nccl().send && nccl().recv && nccl().group_start && nccl().group_end; }
    void sendrecv(const void* send, int to, void* recv, int from, size_t bytes) override {
        if (to < 0 && from < 0) return;
        nccl_check(nccl().group_start(), "ncclGroupStart");
        if (to >= 0) nccl_check(nccl().send(send, bytes, kNcclInt8, to, comm_, stream()), "ncclSend");
        if (from >= 0) nccl_check(nccl().recv(recv, bytes, kNcclInt8, from, comm_, stream()), "ncclRecv");
        nccl_check(nccl().group_end(), "ncclGroupEnd");
    }

private:
    int rank_, size_;
    nccl_comm_t comm_ = nullptr;
};

// ---- in-process loopback group ------------------------------------------------------------
struct LoopShared {
    explicit LoopShared(int n) : n(n) {}
    ~LoopShared() {
        if (stage) cudaFree(stage);
    }
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const uint64_t g = gen;
        if (++arrived == n) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
    int n;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    char* stage = nullptr;
    size_t cap = 0;
};

class LoopbackComm final : public Comm {
public:
    LoopbackComm(std::shared_ptr<LoopShared> sh, int rank) : sh_(std::move(sh)), rank_(rank) {}
    int rank() const override { return rank_; }
    int size() const override { return sh_->n; }
    void allgather(const void* send, void* recv, size_t bytes) override {
        const size_t total = bytes * (size_t)sh_->n;
        sh_->barrier();
        if (rank_ == 0 && sh_->cap < total) {
            if (sh_->stage) TTG_CUDA(cudaFree(sh_->stage));
            TTG_CUDA(cudaMalloc(reinterpret_cast<void**>(&sh_->stage), total));
            sh_->cap = total;
        }
        sh_->barrier();
        TTG_CUDA(cudaMemcpyAsync(sh_->stage + bytes * rank_, send, bytes, cudaMemcpyDeviceToDevice, stream()));
        TTG_CUDA(cudaStreamSynchronize(stream()));
        sh_->barrier();
        TTG_CUDA(cudaMemcpyAsync(recv, sh_->stage, total, cudaMemcpyDeviceToDevice, stream()));
        TTG_CUDA(cudaStreamSynchronize(stream()));
        sh_->barrier();
    }
    bool has_p2p() const override { return true; }
    // every sender parks its buffer in its own stage slot; receivers copy from the sender's slot
    void sendrecv(const void* send, int to, void* recv, int from, size_t bytes) override {
        const size_t total = bytes * (size_t)sh_->n;
        sh_->barrier();
        if (rank_ == 0 && sh_->cap < total) {
            if (sh_->stage) TTG_CUDA(cudaFree(sh_->stage));
            TTG_CUDA(cudaMalloc(reinterpret_cast<void**>(&sh_->stage), total));
            sh_->cap = total;
        }
        sh_->barrier();
        if (to >= 0) {
            TTG_CUDA(cudaMemcpyAsync(sh_->stage + bytes * rank_, send, bytes, cudaMemcpyDeviceToDevice, stream()));
            TTG_CUDA(cudaStreamSynchronize(stream()));
        }
        sh_->barrier();
        if (from >= 0) {
            TTG_CUDA(cudaMemcpyAsync(recv, sh_->stage + bytes * from, bytes, cudaMemcpyDeviceToDevice, stream()));
            TTG_CUDA(cudaStreamSynchronize(stream()));
        }
        sh_->barrier();
    }

private:
    std::shared_ptr<LoopShared> sh_;
    int rank_;
};

// ---- host-callback transport (any host collective: gloo, MPI, sockets) -------------------
// The exchange leaves the device: the send buffer is copied to pinned host memory, the
// caller's all-gather runs on the host, and the gathered bytes go back to the device. Used
// with torch.distributed's gloo backend to drive the real engine from separate processes
// (tests), and as the integration point for hosts that bring their own collective library.
class CallbackComm final : public Comm {
public:
    CallbackComm(int nranks, int rank, ttg_host_allgather_fn fn, void* user)
        : rank_(rank), size_(nranks), fn_(fn), user_(user) {}
    ~CallbackComm() override {
        if (hsend_) cudaFreeHost(hsend_);
        if (hrecv_) cudaFreeHost(hrecv_);
    }
    int rank() const override { return rank_; }
    int size() const override { return size_; }
    void allgather(const void* send, void* recv, size_t bytes) override {
        const size_t total = bytes * (size_t)size_;
        if (cap_ < total) {
            if (hsend_) TTG_CUDA(cudaFreeHost(hsend_));
            if (hrecv_) TTG_CUDA(cudaFreeHost(hrecv_));
            TTG_CUDA(cudaMallocHost(&hsend_, total));
            TTG_CUDA(cudaMallocHost(&hrecv_, total));
            cap_ = total;
        }
        TTG_CUDA(cudaMemcpyAsync(hsend_, send, bytes, cudaMemcpyDeviceToHost, stream()));
        TTG_CUDA(cudaStreamSynchronize(stream()));
        const int st = fn_(hsend_, hrecv_, bytes, user_);
        if (st != 0) fail(8, "host all-gather callback failed with status " + std::to_string(st));
        TTG_CUDA(cudaMemcpyAsync(recv, hrecv_, total, cudaMemcpyHostToDevice, stream()));
        TTG_CUDA(cudaStreamSynchronize(stream()));
    }

private:
    int rank_, size_;
    ttg_host_allgather_fn fn_;
    void* user_;
    void* hsend_ = nullptr;
    void* hrecv_ = nullptr;
    size_t cap_ = 0;
};

}  // namespace

std::unique_ptr<Comm> make_callback_comm(int nranks, int rank, ttg_host_allgather_fn fn, void* user) {
    if (nranks < 1 || rank < 0 || rank >= nranks || !fn) argument_error("invalid callback communicator");
    return std::make_unique<CallbackComm>(nranks, rank, fn, user);
}

double global_sum(Comm& comm, double local) {
    DevBuf<double> one(1), all((size_t)comm.size());
    one.upload(&local, 1);
    comm.allgather(one.get(), all.get(), sizeof(double));
    std::vector<double> h = all.to_host((size_t)comm.size());
    double s = 0.0;
    for (double v : h) s += v;
    return s;
}

void nccl_unique_id(unsigned char id[128]) {
    NcclId uid;
    nccl_check(nccl().get_unique_id(&uid), "ncclGetUniqueId");
    std::memcpy(id, uid.internal, sizeof(uid.internal));
}

std::unique_ptr<Comm> make_nccl_comm(const unsigned char id[128], int nranks, int rank) {
    if (nranks < 1 || rank < 0 || rank >= nranks) argument_error("invalid NCCL rank / size");
    return std::make_unique<NcclComm>(id, nranks, rank);
}

std::vector<std::unique_ptr<Comm>> make_loopback_group(int nranks) {
    if (nranks < 1) argument_error("loopback group needs at least one rank");
    auto sh = std::make_shared<LoopShared>(nranks);
    std::vector<std::unique_ptr<Comm>> out;
    for (int r = 0; r < nranks; ++r) out.push_back(std::make_unique<LoopbackComm>(sh, r));
    return out;
}

}  // namespace ttg
