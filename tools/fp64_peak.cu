// FP64 pipe microbenchmark for the roofline denominator (DFMA vs DMMA 8x8x4).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_peak.cu -o tools/fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void dmma_loop(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-12, b = 1.0 - threadIdx.x * 1e-12;
    double c[NACC][2];
#pragma unroll
    for (int k = 0; k < NACC; ++k) { c[k][0] = 0; c[k][1] = 0; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < NACC; ++k)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < NACC; ++k) s += c[k][0] + c[k][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-12, b = 1.0 - threadIdx.x * 1e-12;
    double c[NACC];
#pragma unroll
    for (int k = 0; k < NACC; ++k) c[k] = k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < NACC; ++k) c[k] = fma(a, c[k], b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < NACC; ++k) s += c[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out;
    cudaMalloc(&out, sizeof(double) * 148 * 8 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int blocks_per_sm : {1, 2, 4, 8}) {
        for (int threads : {128, 256}) {
            int grid = sms * blocks_per_sm;
            dmma_loop<8><<<grid, threads>>>(out, 100);
            cudaEventRecord(e0);
            dmma_loop<8><<<grid, threads>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            // one m8n8k4 per warp = 8*8*4 MAC = 512 flop
            double flops = double(grid) * (threads / 32) * iters * 8 * 512.0;
            printf("DMMA grid=%d thr=%d: %.2f TFLOP/s\n", grid, threads, flops / ms / 1e9);
            dfma_loop<8><<<grid, threads>>>(out, 100);
            cudaEventRecord(e0);
            dfma_loop<8><<<grid, threads>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            flops = double(grid) * threads * iters * 8 * 2.0;
            printf("DFMA grid=%d thr=%d: %.2f TFLOP/s\n", grid, threads, flops / ms / 1e9);
        }
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
