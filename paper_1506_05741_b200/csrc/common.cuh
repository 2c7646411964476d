// common.cuh — shared device/host helpers for the B200 DIAM engine.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <stdexcept>
#include <string>

namespace dgb {

constexpr int kNumSMs = 148;  // B200: 2 dies x 74 SMs

struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& s) : std::runtime_error(s) {}
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess)
        throw CudaError(std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what + " at " +
                        file + ":" + std::to_string(line));
}
#define DGB_CUDA(x) ::dgb::cuda_check((x), #x, __FILE__, __LINE__)

// DIAM_B200_SYNC_CHECK=1: synchronize after every launch so a device fault is reported
// at the kernel that caused it (debugging only)
bool sync_check_enabled();
inline void launch_check(const char* file, int line) {
    cuda_check(cudaGetLastError(), "kernel launch", file, line);
    if (sync_check_enabled()) cuda_check(cudaDeviceSynchronize(), "kernel execution", file, line);
}
#define DGB_LAUNCH_CHECK() ::dgb::launch_check(__FILE__, __LINE__)

// Process-wide count of our own kernel launches (bench.py reports it as gpu_launches).
extern std::atomic<uint64_t> g_launch_count;
// this thread's share (a stream capture counts the kernels it records, not launches)
extern thread_local uint64_t t_launch_count;
inline void count_launch(uint64_t n = 1) {
    g_launch_count.fetch_add(n, std::memory_order_relaxed);
    t_launch_count += n;
}

// Raise a kernel's dynamic shared-memory limit to `bytes` on the CURRENT device (the
// attribute is per device; engines on several devices or threads share the table).
void set_smem_attr(const void* func, int bytes);

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Leading dimension used for every device d-vector/d×d row: a multiple of 8
// doubles (64 B) so rows stay 16-byte aligned for cp.async / vector loads and
// tiles never straddle a row end without a zero pad.
inline int64_t pad_ld(int64_t n) { return (n + 7) / 8 * 8; }

}  // namespace dgb
