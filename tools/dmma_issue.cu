// dmma_issue.cu — can one warp per SM sub-partition keep the FP64 DMMA pipe busy?
// DMMA m8n8k4 loops with NACC independent accumulators, `warps` warps per SM (one CTA
// per SM), timed with CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/dmma_issue.cu -o /tmp/dmma_issue && /tmp/dmma_issue
#include <cstdio>

template <int NACC>
__global__ void dmma_loop(double* out, int iters) {
    double acc[NACC][2];
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i][0] = acc[i][1] = 0.0;
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NACC; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[i][0]), "+d"(acc[i][1])
                         : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.0) out[0] = s;
}

template <int NACC>
void run(int warps, double* out) {
    const int sms = 148, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    dmma_loop<NACC><<<sms, 32 * warps>>>(out, 16);
    cudaEventRecord(e0);
    dmma_loop<NACC><<<sms, 32 * warps>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 512.0 * NACC * iters * warps * sms;
    printf("warps/SM %2d, %2d independent accumulators: %6.2f TFLOP/s\n", warps, NACC, flops / (ms * 1e-3) / 1e12);
}

int main() {
    double* out;
    cudaMalloc(&out, 8);
    for (int w : {4, 8, 16}) {
        run<8>(w, out);
        run<16>(w, out);
        run<32>(w, out);
    }
    return 0;
}
