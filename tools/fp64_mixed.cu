// Do the DMMA (tensor) and DFMA (FP64 ALU) pipes run concurrently? Warps of one CTA split
// between an m8n8k4 f64 MMA loop and a plain DFMA loop; the combined FP64 rate against each
// pipe alone (tools/fp64_peak.cu).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_mixed.cu -o tools/fp64_mixed
#include <cstdio>
#include <cuda_runtime.h>

// warps [0, nd) run DMMA, the rest DFMA
__global__ void mixed(double* out, int iters_mma, int iters_fma, int nd) {
    const int warp = threadIdx.x >> 5;
    double a = 1.0 + threadIdx.x * 1e-12, b = 1.0 - threadIdx.x * 1e-12;
    double s = 0.0;
    if (warp < nd) {
        double c[8][2];
#pragma unroll
        for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0.0;
        for (int i = 0; i < iters_mma; ++i) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c[k][0]), "+d"(c[k][1])
                             : "d"(a), "d"(b));
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
    } else {
        double c[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) c[k] = k;
        for (int i = 0; i < iters_fma; ++i) {
#pragma unroll
            for (int k = 0; k < 8; ++k) c[k] = fma(a, c[k], b);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) s += c[k];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, sizeof(double) * sms * 4 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int threads = 512, grid = sms * 2, warps = threads / 32;
    // per-warp work: a DMMA iteration = 8 x 512 flop, a DFMA iteration = 8 x 32 x 2 flop
    for (int nd : {16, 0, 8, 12, 4}) {
        for (int fma_scale : {4, 8, 16}) {
            const int im = 4000, ifm = im * fma_scale;
            mixed<<<grid, threads>>>(out, 10, 10, nd);
            cudaEventRecord(e0);
            mixed<<<grid, threads>>>(out, im, ifm, nd);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double fl = double(grid) * (nd * (double)im * 8 * 512 + (warps - nd) * (double)ifm * 8 * 64);
            const double fm = double(grid) * nd * (double)im * 8 * 512, ff = fl - fm;
            printf("dmma warps %2d/%d fma x%2d: %.3f ms  total %.2f TF/s (dmma %.2f + dfma %.2f)\n", nd, warps,
                   fma_scale, ms, fl / ms / 1e9, fm / ms / 1e9, ff / ms / 1e9);
            if (nd == 16) break;
        }
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
