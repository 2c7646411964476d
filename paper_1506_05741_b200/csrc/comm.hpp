// comm.hpp — the engine's view of the multi-GPU exchange.
//
// The sampler has exactly one exchange step per batch (proj/src/runner.cpp:
// 238-245): the moment merge. Chains are block-sharded over ranks (one process
// per GPU); each rank pre-sums its chains' raw moments and an all-reduce(sum,
// f64) over NVLink pools them; per-chain PSRF inputs are all-gathered. NCCL is
// loaded lazily with dlopen so the library has no hard link dependency (the
// process's already-loaded libnccl.so.2, e.g. torch's, is reused).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <vector>

namespace dgb {

struct Comm {
    virtual ~Comm();
    virtual int rank() const = 0;
    virtual int size() const = 0;
    virtual void allreduce_sum(double* buf, int64_t n, cudaStream_t s) = 0;
    // dst holds size()*n doubles, rank r's block at r*n
    virtual void allgather(const double* src, double* dst, int64_t n, cudaStream_t s) = 0;
    // buf (n doubles, device) of rank `root` to every rank
    virtual void broadcast(double* buf, int64_t n, int root, cudaStream_t s) = 0;
    // Host byte blobs of every rank to rank 0, in rank order (every rank calls it; the other
    // ranks get an empty result). Staged through the device in 64 MB broadcasts: the
    // checkpoint of a sharded run (Engine::save_checkpoint).
    std::vector<std::vector<char>> gather_bytes(const std::vector<char>& mine, cudaStream_t s);
    // Collective OR of a host flag (every rank must call it at the same point): the
    // engine's stop decisions and rank-local failures go through it, so all ranks leave
    // the batch loop together instead of one rank waiting in a collective forever.
    bool any(bool flag, cudaStream_t s);

private:
    double* scratch_ = nullptr;  // one device double (allocated on first use)
    int scratch_dev_ = -1;

public:
    Comm() = default;
    Comm(const Comm&) = delete;
    Comm& operator=(const Comm&) = delete;
};

// Process-wide communicator used by diam_sample when set (diamx_comm_init).
std::shared_ptr<Comm>& global_comm();
// NCCL: unique id (128 bytes) from rank 0, shared out of band by the caller.
bool nccl_available(char* why, int why_len);
int nccl_unique_id(char out[128]);
std::shared_ptr<Comm> make_nccl_comm(const char id[128], int rank, int world);
// In-process communicator for `world` engines driven by `world` host threads on one GPU
// (parity tests of the sharded engine: the same exchange steps as NCCL, summed on the
// host in rank order; a rank that stops arriving makes the others fail, not hang).
std::vector<std::shared_ptr<Comm>> make_thread_comms(int world);

}  // namespace dgb
