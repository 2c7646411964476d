// comm.cpp — NCCL communicator loaded with dlopen (see comm.hpp).
#include "comm.hpp"

#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace dgb {

namespace {

// Minimal NCCL ABI (nccl.h 2.x): opaque communicator, 128-byte unique id.
typedef struct ncclComm* ncclComm_t;
struct ncclUniqueId {
    char internal[128];
};
enum ncclResult_t { ncclSuccess = 0 };
enum ncclDataType_t { ncclFloat64 = 8 };
enum ncclRedOp_t { ncclSum = 0 };

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string err;
    bool load() {
        if (h) return true;
        // prefer an already-loaded copy (torch ships libnccl.so.2), else the system one
        h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = dlerror() ? dlerror() : "dlopen libnccl.so.2 failed";
            return false;
        }
        GetUniqueId = (decltype(GetUniqueId))dlsym(h, "ncclGetUniqueId");
        CommInitRank = (decltype(CommInitRank))dlsym(h, "ncclCommInitRank");
        AllReduce = (decltype(AllReduce))dlsym(h, "ncclAllReduce");
        AllGather = (decltype(AllGather))dlsym(h, "ncclAllGather");
        Broadcast = (decltype(Broadcast))dlsym(h, "ncclBroadcast");
        CommDestroy = (decltype(CommDestroy))dlsym(h, "ncclCommDestroy");
        GetErrorString = (decltype(GetErrorString))dlsym(h, "ncclGetErrorString");
        if (!GetUniqueId || !CommInitRank || !AllReduce || !AllGather || !Broadcast || !CommDestroy) {
            err = "libnccl.so.2 lacks expected symbols";
            h = nullptr;
            return false;
        }
        return true;
    }
    void check(ncclResult_t r, const char* what) const {
        if (r != ncclSuccess)
            throw CudaError(std::string("NCCL ") + what + ": " + (GetErrorString ? GetErrorString(r) : "error"));
    }
};

NcclApi& api() {
    static NcclApi a;
    return a;
}

struct NcclComm final : Comm {
    ncclComm_t comm = nullptr;
    int r = 0, n = 1;
    ~NcclComm() override {
        if (comm) api().CommDestroy(comm);
    }
    int rank() const override { return r; }
    int size() const override { return n; }
    void allreduce_sum(double* buf, int64_t cnt, cudaStream_t s) override {
        api().check(api().AllReduce(buf, buf, (size_t)cnt, ncclFloat64, ncclSum, comm, s), "allreduce");
    }
    void allgather(const double* src, double* dst, int64_t cnt, cudaStream_t s) override {
        api().check(api().AllGather(src, dst, (size_t)cnt, ncclFloat64, comm, s), "allgather");
    }
    void broadcast(double* buf, int64_t cnt, int root, cudaStream_t s) override {
        api().check(api().Broadcast(buf, buf, (size_t)cnt, ncclFloat64, root, comm, s), "broadcast");
    }
};

// ---------------------------------------------------------------- in-process ranks
struct ThreadShared {
    int world = 0;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    std::vector<std::vector<double>> stage;  // one host buffer per rank
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const uint64_t gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
            return;
        }
        if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return generation != gen; }))
            throw CudaError("thread communicator: a rank did not reach the exchange");
    }
};

struct ThreadComm final : Comm {
    std::shared_ptr<ThreadShared> sh;
    int r = 0;
    int rank() const override { return r; }
    int size() const override { return sh->world; }
    void allreduce_sum(double* buf, int64_t cnt, cudaStream_t s) override {
        auto& mine = sh->stage[r];
        mine.resize(cnt);
        DGB_CUDA(cudaMemcpyAsync(mine.data(), buf, cnt * 8, cudaMemcpyDeviceToHost, s));
        DGB_CUDA(cudaStreamSynchronize(s));
        sh->barrier();
        std::vector<double> sum(cnt, 0.0);
        for (int k = 0; k < sh->world; ++k)  // rank order, the same on every rank
            for (int64_t e = 0; e < cnt; ++e) sum[e] += sh->stage[k][e];
        sh->barrier();  // everyone has read every stage
        DGB_CUDA(cudaMemcpyAsync(buf, sum.data(), cnt * 8, cudaMemcpyHostToDevice, s));
        DGB_CUDA(cudaStreamSynchronize(s));
    }
    void allgather(const double* src, double* dst, int64_t cnt, cudaStream_t s) override {
        auto& mine = sh->stage[r];
        mine.resize(cnt);
        DGB_CUDA(cudaMemcpyAsync(mine.data(), src, cnt * 8, cudaMemcpyDeviceToHost, s));
        DGB_CUDA(cudaStreamSynchronize(s));
        sh->barrier();
        for (int k = 0; k < sh->world; ++k)
            DGB_CUDA(cudaMemcpyAsync(dst + k * cnt, sh->stage[k].data(), cnt * 8, cudaMemcpyHostToDevice, s));
        DGB_CUDA(cudaStreamSynchronize(s));
        sh->barrier();
    }
    void broadcast(double* buf, int64_t cnt, int root, cudaStream_t s) override {
        if (r == root) {
            sh->stage[root].resize(cnt);
            DGB_CUDA(cudaMemcpyAsync(sh->stage[root].data(), buf, cnt * 8, cudaMemcpyDeviceToHost, s));
            DGB_CUDA(cudaStreamSynchronize(s));
        }
        sh->barrier();
        if (r != root) {
            DGB_CUDA(cudaMemcpyAsync(buf, sh->stage[root].data(), cnt * 8, cudaMemcpyHostToDevice, s));
            DGB_CUDA(cudaStreamSynchronize(s));
        }
        sh->barrier();
    }
};

}  // namespace

Comm::~Comm() {
    if (scratch_) cudaFree(scratch_);
}

bool Comm::any(bool flag, cudaStream_t s) {
    int dev = 0;
    DGB_CUDA(cudaGetDevice(&dev));
    if (!scratch_ || scratch_dev_ != dev) {
        DGB_CUDA(cudaMalloc(&scratch_, sizeof(double)));
        scratch_dev_ = dev;
    }
    double h = flag ? 1.0 : 0.0;
    DGB_CUDA(cudaMemcpyAsync(scratch_, &h, sizeof(double), cudaMemcpyHostToDevice, s));
    allreduce_sum(scratch_, 1, s);
    DGB_CUDA(cudaMemcpyAsync(&h, scratch_, sizeof(double), cudaMemcpyDeviceToHost, s));
    DGB_CUDA(cudaStreamSynchronize(s));
    return h > 0.5;
}

std::vector<std::vector<char>> Comm::gather_bytes(const std::vector<char>& mine, cudaStream_t s) {
    const int n = size(), me = rank();
    constexpr int64_t kChunk = 8ll << 20;  // doubles per broadcast (64 MB)
    double* dev = nullptr;
    DGB_CUDA(cudaMalloc(&dev, (size_t)std::max<int64_t>(n, kChunk) * sizeof(double)));
    std::vector<double> sizes(n);
    {
        double* one = dev + kChunk - 1;  // any spare slot for this rank's size
        const double v = (double)mine.size();
        DGB_CUDA(cudaMemcpyAsync(one, &v, sizeof(double), cudaMemcpyHostToDevice, s));
        double* all = nullptr;
        DGB_CUDA(cudaMalloc(&all, n * sizeof(double)));
        allgather(one, all, 1, s);
        DGB_CUDA(cudaMemcpyAsync(sizes.data(), all, n * sizeof(double), cudaMemcpyDeviceToHost, s));
        DGB_CUDA(cudaStreamSynchronize(s));
        cudaFree(all);
    }
    std::vector<std::vector<char>> out;
    if (me == 0) {
        out.resize(n);
        out[0] = mine;
    }
    std::vector<double> host(kChunk);
    for (int k = 1; k < n; ++k) {
        const int64_t bytes = (int64_t)sizes[k];
        if (me == 0) out[k].resize((size_t)bytes);
        for (int64_t off = 0; off < bytes; off += kChunk * 8) {
            const int64_t nb = std::min<int64_t>(kChunk * 8, bytes - off), nd = (nb + 7) / 8;
            if (me == k) {
                std::memcpy(host.data(), mine.data() + off, (size_t)nb);
                DGB_CUDA(cudaMemcpyAsync(dev, host.data(), nd * 8, cudaMemcpyHostToDevice, s));
            }
            broadcast(dev, nd, k, s);
            if (me == 0) {
                DGB_CUDA(cudaMemcpyAsync(host.data(), dev, nd * 8, cudaMemcpyDeviceToHost, s));
                DGB_CUDA(cudaStreamSynchronize(s));
                std::memcpy(out[k].data() + off, host.data(), (size_t)nb);
            }
        }
    }
    DGB_CUDA(cudaStreamSynchronize(s));
    cudaFree(dev);
    return out;
}

std::vector<std::shared_ptr<Comm>> make_thread_comms(int world) {
    auto sh = std::make_shared<ThreadShared>();
    sh->world = world;
    sh->stage.resize(world);
    std::vector<std::shared_ptr<Comm>> out;
    for (int r = 0; r < world; ++r) {
        auto c = std::make_shared<ThreadComm>();
        c->sh = sh;
        c->r = r;
        out.push_back(c);
    }
    return out;
}

std::shared_ptr<Comm>& global_comm() {
    static std::shared_ptr<Comm> c;
    return c;
}

bool nccl_available(char* why, int why_len) {
    const bool ok = api().load();
    if (!ok && why) std::snprintf(why, why_len, "%s", api().err.c_str());
    return ok;
}

int nccl_unique_id(char out[128]) {
    if (!api().load()) return 1;
    ncclUniqueId id;
    api().check(api().GetUniqueId(&id), "get unique id");
    std::memcpy(out, id.internal, 128);
    return 0;
}

std::shared_ptr<Comm> make_nccl_comm(const char id_bytes[128], int rank, int world) {
    if (!api().load()) throw CudaError("NCCL unavailable: " + api().err);
    auto c = std::make_shared<NcclComm>();
    ncclUniqueId id;
    std::memcpy(id.internal, id_bytes, 128);
    c->r = rank;
    c->n = world;
    api().check(api().CommInitRank(&c->comm, world, id, rank), "comm init");
    return c;
}

}  // namespace dgb
