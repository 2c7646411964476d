// tma_gemm_probe.cu — feasibility probe: the DMMA GEMM tile (128x64, 32-deep stages, two
// CTAs per SM, 8 warps of 32x32) fed by 2-D TMA tensor-map copies with 128-byte swizzle
// (one thread issues 4 copies per stage) instead of per-thread cp.async, against
// libdiam's cp.async kernel (diamx_gemm) on C = A B^T, A: M x K, B: N x K, both K-major.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_1506_05741_b200/csrc -Iinclude \
//        tools/tma_gemm_probe.cu -Lpaper_1506_05741_b200 -ldiam -lcuda \
//        -Xlinker -rpath,$PWD/paper_1506_05741_b200 -o /tmp/tma_gemm_probe && /tmp/tma_gemm_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "diam_b200.h"

namespace {

constexpr int BM = 128, BN = 64, BK = 32, BOX = 16;  // BOX doubles = 128 B (the swizzle span)
constexpr int A_BOX = BM * BOX, B_BOX = BN * BOX;    // doubles per box
constexpr int A_STAGE = A_BOX * (BK / BOX), B_STAGE = B_BOX * (BK / BOX);
constexpr int STAGE_BYTES = (A_STAGE + B_STAGE) * 8;
constexpr int SMEM = 2 * STAGE_BYTES + 1024 + 64;  // 2 stages, 1 KB alignment slack, barriers

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// element (row, k) of a 128B-swizzled box of `rows` x 16 doubles
__device__ __forceinline__ int swz(int row, int k) {
    return row * 16 + ((((k >> 1) ^ (row & 7)) << 1) | (k & 1));
}

__global__ void __launch_bounds__(256, 2) tma_gemm(const __grid_constant__ CUtensorMap ta,
                                                   const __grid_constant__ CUtensorMap tb, double* C, int M, int N,
                                                   int K, int ldc) {
    extern __shared__ unsigned char raw[];
    double* base = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(base + 2 * (A_STAGE + B_STAGE));
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int KT = K / BK;
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(&ta) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tb) : "memory");
    }
    __syncthreads();
    auto issue = [&](int kt) {
        const int s = kt & 1;
        double* a_s = base + s * (A_STAGE + B_STAGE);
        double* b_s = a_s + A_STAGE;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&full[s])),
                     "r"(STAGE_BYTES)
                     : "memory");
#pragma unroll
        for (int b = 0; b < BK / BOX; ++b) {
            const int kc = kt * BK + b * BOX;
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                "[%4];\n" ::"r"(su32(a_s + b * A_BOX)),
                "l"(&ta), "r"(kc), "r"(m0), "r"(su32(&full[s]))
                : "memory");
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                "[%4];\n" ::"r"(su32(b_s + b * B_BOX)),
                "l"(&tb), "r"(kc), "r"(n0), "r"(su32(&full[s]))
                : "memory");
        }
    };
    if (tid == 0) issue(0);
    const int fr = lane >> 2, fk = lane & 3;
    const int wm0 = (warp >> 1) * 32, wn0 = (warp & 1) * 32;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kt = 0; kt < KT; ++kt) {
        const int s = kt & 1;
        asm volatile(
            "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                su32(&full[s])),
            "r"((kt >> 1) & 1)
            : "memory");
        __syncthreads();  // everyone is done with slot (kt + 1) & 1
        if (tid == 0 && kt + 1 < KT) issue(kt + 1);
        const double* a_s = base + s * (A_STAGE + B_STAGE);
        const double* b_s = a_s + A_STAGE;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            const int k = kk + fk, box = k >> 4, kin = k & 15;
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = a_s[box * A_BOX + swz(wm0 + i * 8 + fr, kin)];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = b_s[box * B_BOX + swz(wn0 + j * 8 + fr, kin)];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = m0 + wm0 + i * 8 + fr;
        if (r >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c0 = n0 + wn0 + j * 8 + fk * 2;
            if (c0 + 1 < N) *reinterpret_cast<double2*>(C + (int64_t)r * ldc + c0) = make_double2(acc[i][j][0], acc[i][j][1]);
            else if (c0 < N) C[(int64_t)r * ldc + c0] = acc[i][j][0];
        }
    }
}

void make_map(CUtensorMap* m, const double* p, int rows, int cols, int64_t ld, int box_rows) {
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
    const cuuint32_t box[2] = {BOX, (cuuint32_t)box_rows};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = cuTensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)p, dims, strides, box, es,
                                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        std::printf("cuTensorMapEncodeTiled failed: %d\n", (int)r);
        std::exit(1);
    }
}

}  // namespace

int main() {
    const int M = 32768, N = 1024;
    double peak = 0.0;
    diamx_fp64_peak(&peak);
    cudaFuncSetAttribute(tma_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    for (int K : {256, 512, 1024, 2048}) {
        std::vector<double> ha((size_t)M * K), hb((size_t)N * K);
        for (size_t i = 0; i < ha.size(); ++i) ha[i] = std::sin(0.001 * (double)i);
        for (size_t i = 0; i < hb.size(); ++i) hb[i] = std::cos(0.002 * (double)i);
        double *A, *B, *C1, *C2;
        cudaMalloc(&A, ha.size() * 8);
        cudaMalloc(&B, hb.size() * 8);
        cudaMalloc(&C1, (size_t)M * N * 8);
        cudaMalloc(&C2, (size_t)M * N * 8);
        cudaMemcpy(A, ha.data(), ha.size() * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(B, hb.data(), hb.size() * 8, cudaMemcpyHostToDevice);
        CUtensorMap ta, tb;
        make_map(&ta, A, M, K, K, BM);
        make_map(&tb, B, N, K, K, BN);
        dim3 grid(N / BN, M / BM);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        auto time = [&](auto fn) {
            for (int i = 0; i < 2; ++i) fn();
            float best = 1e30f;
            for (int r = 0; r < 3; ++r) {
                cudaEventRecord(e0);
                for (int i = 0; i < 5; ++i) fn();
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                best = std::fmin(best, ms / 5);
            }
            return best;
        };
        const float t_tma = time([&] { tma_gemm<<<grid, 256, SMEM>>>(ta, tb, C1, M, N, K, N); });
        const float t_lib = time([&] {
            diamx_gemm(A, B, C2, M, N, K, K, K, N, 1, 1, 1.0, 0.0, 0, 0, nullptr);
        });
        const cudaError_t err = cudaDeviceSynchronize();
        std::vector<double> c1((size_t)M * N), c2((size_t)M * N);
        cudaMemcpy(c1.data(), C1, c1.size() * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(c2.data(), C2, c2.size() * 8, cudaMemcpyDeviceToHost);
        double md = 0.0;
        size_t neq = 0;
        for (size_t i = 0; i < c1.size(); ++i) {
            md = std::fmax(md, std::fabs(c1[i] - c2[i]));
            neq += c1[i] != c2[i];
        }
        const double fl = 2.0 * M * N * (double)K;
        std::printf("K=%5d  TMA %8.1f us %6.2f TF (%5.1f%%)   cp.async %8.1f us %6.2f TF (%5.1f%%)   max|diff| %.3g, "
                    "%zu unequal (%s)\n",
                    K, t_tma * 1e3, fl / t_tma / 1e9, fl / t_tma / 1e9 / peak * 100, t_lib * 1e3, fl / t_lib / 1e9,
                    fl / t_lib / 1e9 / peak * 100, md, neq, cudaGetErrorString(err));
        cudaFree(A);
        cudaFree(B);
        cudaFree(C1);
        cudaFree(C2);
    }
    return 0;
}
