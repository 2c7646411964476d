// peak.cu — live FP64 DMMA peak for the roofline denominator.
//
// MEASURED_PEAKS.json carries HBM and bf16 peaks only; the sampler's dense
// contractions run on the FP64 DMMA pipe (tcgen05 has no f64 kind), so bench.py
// measures that pipe on the same box, in the same run, with this kernel:
// independent m8n8k4 f64 MMAs per warp, 8 accumulators deep, 2 CTAs x 256
// threads per SM. (tools/fp64_peak.cu is the standalone version; 37.1 TFLOP/s
// on the pool's B200s at the time of writing.)
#include <cuda_runtime.h>

#include "../../include/diam_b200.h"
#include "common.cuh"

namespace {

__global__ void __launch_bounds__(256) dmma_peak_kernel(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-12, b = 1.0 - threadIdx.x * 1e-12;
    double c[8][2];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[k][0]), "+d"(c[k][1])
                         : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
    if (s == 12345.0) out[0] = s;  // keep the work alive
}

}  // namespace

extern "C" diam_status diamx_fp64_peak(double* tflops) {
    if (!tflops) return DIAM_ERR_INVALID_ARGUMENT;
    try {
        int sms = 0;
        DGB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
        double* out = nullptr;
        DGB_CUDA(cudaMalloc(&out, 8));
        const int grid = sms * 2, threads = 256, iters = 40000;
        dmma_peak_kernel<<<grid, threads>>>(out, 200);
        DGB_LAUNCH_CHECK();
        cudaEvent_t e0, e1;
        DGB_CUDA(cudaEventCreate(&e0));
        DGB_CUDA(cudaEventCreate(&e1));
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            DGB_CUDA(cudaEventRecord(e0));
            dmma_peak_kernel<<<grid, threads>>>(out, iters);
            DGB_CUDA(cudaEventRecord(e1));
            DGB_CUDA(cudaEventSynchronize(e1));
            float ms = 0.f;
            DGB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            best = ms < best ? ms : best;
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaFree(out);
        const double flops = double(grid) * (threads / 32) * iters * 8 * 512.0;  // 8x8x4 MACs x2
        *tflops = flops / (best * 1e-3) / 1e12;
        return DIAM_OK;
    } catch (...) {
        return DIAM_ERR_UNKNOWN;
    }
}
