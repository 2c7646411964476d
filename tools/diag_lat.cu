// diag_lat.cu — latency microbenchmark of the 64x64 diagonal-block Cholesky + inverse
// (diag_tc.cuh) with its phase timestamps (DIAG_TC_PROFILE).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I paper_1506_05741_b200/csrc \
//        tools/diag_lat.cu -o tools/diag_lat && tools/diag_lat [blocks]
#define DIAG_TC_PROFILE 1
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "diag_tc.cuh"

using namespace dgb;

__global__ void __launch_bounds__(256, 2) diag_kernel(double* A, int64_t ld, double* X, long long* cyc) {
    extern __shared__ __align__(16) double smem[];
    const long long t0 = clock64();
    double* Ab = A + (int64_t)blockIdx.x * 64 * ld;
    diag64_tc_sc(*reinterpret_cast<DiagTcScratch*>(smem), Ab, ld, 64, X + (int64_t)blockIdx.x * 64 * 64, 0, 64);
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main(int argc, char** argv) {
    const int nb = argc > 1 ? atoi(argv[1]) : 64;
    const int64_t ld = 72;
    std::vector<double> h((size_t)nb * 64 * ld, 0.0);
    srand(1);
    for (int b = 0; b < nb; ++b) {
        std::vector<double> r(64 * 70);
        for (auto& v : r) v = rand() / (double)RAND_MAX - 0.5;
        for (int i = 0; i < 64; ++i)
            for (int j = 0; j <= i; ++j) {
                double s = (i == j) ? 1.0 : 0.0;
                for (int k = 0; k < 70; ++k) s += r[i * 70 + k] * r[j * 70 + k] / 70.0;
                h[((size_t)b * 64 + i) * ld + j] = s;
            }
    }
    double *A, *A0, *X;
    long long* cyc;
    cudaMalloc(&A, h.size() * 8);
    cudaMalloc(&A0, h.size() * 8);
    cudaMalloc(&X, (size_t)nb * 64 * 64 * 8);
    cudaMalloc(&cyc, nb * 8);
    cudaMemcpy(A0, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    const int smem = sizeof(DiagTcScratch);
    cudaFuncSetAttribute(diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9;
    for (int it = 0; it < 20; ++it) {
        cudaMemcpy(A, A0, h.size() * 8, cudaMemcpyDeviceToDevice);
        cudaEventRecord(e0);
        diag_kernel<<<nb, 256, smem>>>(A, ld, X, cyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    std::vector<long long> c(nb), prof(16);
    cudaMemcpy(c.data(), cyc, nb * 8, cudaMemcpyDeviceToHost);
    cudaMemcpyFromSymbol(prof.data(), g_tc_prof, 16 * 8);
    double mean = 0;
    for (auto v : c) mean += v;
    printf("blocks %d: kernel %.2f us (event, best of 20), in-kernel cycles mean %.0f\n", nb, best * 1e3, mean / nb);
    const char* names[] = {"load", "sync", "panels0-3", "panel3-factor", "panels->end", "diag-inv", "blockrow-inv", "store"};
    for (int i = 1; i < 8; ++i) printf("  mark %d (%s): +%lld cycles\n", i, names[i], prof[i] - prof[i - 1]);
    // check: L L^T = A (block 0)
    std::vector<double> L((size_t)64 * ld);
    cudaMemcpy(L.data(), A, L.size() * 8, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < 64; ++i)
        for (int j = 0; j <= i; ++j) {
            double s = 0;
            for (int k = 0; k <= j; ++k) s += L[i * ld + k] * L[j * ld + k];
            err = fmax(err, fabs(s - h[i * ld + j]));
        }
    printf("  max |L L^T - A| = %.2e\n", err);
    cudaError_t e = cudaGetLastError();
    printf("  %s\n", cudaGetErrorString(e));
    return 0;
}
