// tile_lab.cu -- DMMA GEMM tile experiments outside the engine: the kept tile
// (gemm_tile.cuh) against variants, on a dense 32768 x 1024 x 1024 product (both operands
// K-major, the TRMM's layout) and on the TRMM itself (64 chains x 512 x 1024, lower B).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 --expt-relaxed-constexpr \
//        -I paper_1506_05741_b200/csrc tools/tile_lab.cu -o tools/tile_lab && tools/tile_lab
#include <cstdio>
#include <vector>

#include "gemm_tile.cuh"

using namespace dgb;
using namespace dgb::tile;

// Variant mainloop: fragments double-buffered in registers, the stage hand-over one k4 step
// early (barrier + next stage's first fragments before the last DMMAs of a stage)
template <class CF, bool AK, bool BKM>
__device__ __forceinline__ void mainloop_db(const double* A, const double* B, int64_t lda, int64_t ldb, int M, int N,
                                            int K, int m0, int n0, double* smem, bool tri_b_lower,
                                            double (&acc)[CF::MI][CF::NI][2]) {
    double* sA = smem;
    double* sB = smem + CF::STAGES * CF::A_STAGE;
    const int KT = (K + CF::BK - 1) / CF::BK;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm0 = (warp / CF::WARPS_N) * CF::WM, wn0 = (warp % CF::WARPS_N) * CF::WN;
    auto issue = [&](int kt, int stage) {
        const int k0 = kt * CF::BK;
        load_tile<CF::A_ROWS, CF::A_COLS, CF::A_STRIDE, CF::THREADS>(sA + stage * CF::A_STAGE, A + (int64_t)m0 * lda + k0,
                                                                    lda, M - m0, K - k0, tid);
        load_tile<CF::B_ROWS, CF::B_COLS, CF::B_STRIDE, CF::THREADS>(sB + stage * CF::B_STAGE, B + (int64_t)n0 * ldb + k0,
                                                                    ldb, N - n0, K - k0, tid);
    };
#pragma unroll
    for (int i = 0; i < CF::MI; ++i)
#pragma unroll
        for (int j = 0; j < CF::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
    for (int st = 0; st < CF::STAGES - 1; ++st) {
        if (st < KT) issue(st, st);
        cp_async_commit();
    }
    const int fr = lane >> 2, fk = lane & 3;
    const int kt_live = tri_b_lower ? min(KT, (n0 + wn0 + CF::WN - 1) / CF::BK + 1) : KT;
    constexpr int KK = CF::BK / 4;
    double af[2][CF::MI], bf[2][CF::NI];
    auto load_frags = [&](int buf, int stage, int kk) {
        const double* a_s = sA + stage * CF::A_STAGE;
        const double* b_s = sB + stage * CF::B_STAGE;
#pragma unroll
        for (int i = 0; i < CF::MI; ++i) af[buf][i] = a_s[(wm0 + i * 8 + fr) * CF::A_STRIDE + kk + fk];
#pragma unroll
        for (int j = 0; j < CF::NI; ++j) bf[buf][j] = b_s[(wn0 + j * 8 + fr) * CF::B_STRIDE + kk + fk];
    };
    cp_async_wait<CF::STAGES - 2>();
    __syncthreads();
    if (KT > 0) load_frags(0, 0, 0);
    for (int kt = 0; kt < KT; ++kt) {
        const bool live = kt < kt_live;
#pragma unroll
        for (int kk = 0; kk < KK; ++kk) {
            const int cur = kk & 1;
            if (kk == KK - 1) {
                cp_async_wait<CF::STAGES - 2>();
                __syncthreads();
                if (kt + 1 < KT) load_frags(cur ^ 1, (kt + 1) % CF::STAGES, 0);
            } else {
                load_frags(cur ^ 1, kt % CF::STAGES, (kk + 1) * 4);
            }
            if (kk == 0) {
                const int nk = kt + CF::STAGES - 1;
                if (nk < KT) issue(nk, nk % CF::STAGES);
                cp_async_commit();
            }
            if (live) {
#pragma unroll
                for (int i = 0; i < CF::MI; ++i)
#pragma unroll
                    for (int j = 0; j < CF::NI; ++j) dmma(acc[i][j], af[cur][i], bf[cur][j]);
            }
        }
    }
    cp_async_wait<0>();
}

struct Args {
    const double* A;
    const double* B;
    double* C;
    int64_t a_stride, b_stride, c_stride;  // per batch
    int M, N, K;
    int64_t lda, ldb, ldc;
    int tri_b;
};

template <class CF, int MODE>  // MODE 0: kept mainloop, 1: double-buffered
__global__ void __launch_bounds__(CF::THREADS, CF::MINB) lab_kernel(Args p) {
    extern __shared__ __align__(16) double smem[];
    const int b = blockIdx.z;
    const int nt = p.tri_b ? (int)gridDim.x - 1 - (int)blockIdx.x : (int)blockIdx.x;
    const int n0 = nt * CF::BN, m0 = blockIdx.y * CF::BM;
    int K = p.K;
    if (p.tri_b) K = min(K, n0 + CF::BN);
    const double* A = p.A + b * p.a_stride;
    const double* B = p.B + b * p.b_stride;
    double* C = p.C + b * p.c_stride;
    double acc[CF::MI][CF::NI][2];
    if (MODE == 0) {
        gemm_mainloop<CF, true, true>(A, B, p.lda, p.ldb, p.M, p.N, K, m0, n0, false, smem, p.tri_b != 0, acc);
    } else {
        __syncthreads();
        mainloop_db<CF, true, true>(A, B, p.lda, p.ldb, p.M, p.N, K, m0, n0, smem, p.tri_b != 0, acc);
    }
    gemm_epilogue<CF>(acc, C, p.ldc, p.M, p.N, m0, n0, 1.0, 0.0, false);
}

// MODE 2 (triangular B only): CTA x takes column tiles x and NT-1-x, so every CTA has the
// same total K (64 (x+1) + 64 (NT-x)) -- one kernel of equal-length CTAs
template <class CF>
__global__ void __launch_bounds__(CF::THREADS, CF::MINB) lab_pair_kernel(Args p) {
    extern __shared__ __align__(16) double smem[];
    const int b = blockIdx.z, m0 = blockIdx.y * CF::BM;
    const int NT = (p.N + CF::BN - 1) / CF::BN;
    const double* A = p.A + b * p.a_stride;
    const double* B = p.B + b * p.b_stride;
    double* C = p.C + b * p.c_stride;
    const int tiles[2] = {NT - 1 - (int)blockIdx.x, (int)blockIdx.x};
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
        const int nt = tiles[q];
        if (q == 1 && nt == tiles[0]) break;
        const int n0 = nt * CF::BN;
        const int K = min(p.K, n0 + CF::BN);
        double acc[CF::MI][CF::NI][2];
        gemm_mainloop<CF, true, true>(A, B, p.lda, p.ldb, p.M, p.N, K, m0, n0, false, smem, true, acc);
        gemm_epilogue<CF>(acc, C, p.ldc, p.M, p.N, m0, n0, 1.0, 0.0, false);
    }
}

template <class CF>
double run_pair(const Args& a, int batch, const char* name, double flops) {
    auto k = lab_pair_kernel<CF>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM_BYTES);
    const int NT = (a.N + CF::BN - 1) / CF::BN;
    dim3 grid((NT + 1) / 2, (a.M + CF::BM - 1) / CF::BM, batch);
    for (int i = 0; i < 2; ++i) k<<<grid, CF::THREADS, CF::SMEM_BYTES>>>(a);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        for (int i = 0; i < 5; ++i) k<<<grid, CF::THREADS, CF::SMEM_BYTES>>>(a);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms / 5 < best ? ms / 5 : best;
    }
    const double tf = flops / (best * 1e-3) / 1e12;
    std::printf("%-44s %8.3f ms %6.2f TFLOP/s  (%s)\n", name, best, tf, cudaGetErrorString(cudaGetLastError()));
    return tf;
}

template <class CF, int MODE>
double run(const Args& a, int batch, const char* name, double flops) {
    auto k = lab_kernel<CF, MODE>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM_BYTES);
    dim3 grid((a.N + CF::BN - 1) / CF::BN, (a.M + CF::BM - 1) / CF::BM, batch);
    for (int i = 0; i < 2; ++i) k<<<grid, CF::THREADS, CF::SMEM_BYTES>>>(a);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        for (int i = 0; i < 5; ++i) k<<<grid, CF::THREADS, CF::SMEM_BYTES>>>(a);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms / 5 < best ? ms / 5 : best;
    }
    const double tf = flops / (best * 1e-3) / 1e12;
    std::printf("%-44s %8.3f ms %6.2f TFLOP/s  (%s)\n", name, best, tf, cudaGetErrorString(cudaGetLastError()));
    return tf;
}

int main() {
    const int M = 32768, N = 1024, K = 1024;
    double *A, *B, *C;
    cudaMalloc(&A, (size_t)M * K * 8);
    cudaMalloc(&B, (size_t)64 * N * K * 8);
    cudaMalloc(&C, (size_t)M * N * 8);
    {
        std::vector<double> h((size_t)M * K);
        for (size_t i = 0; i < h.size(); ++i) h[i] = ((i * 2654435761u) % 1000) * 1e-3 - 0.5;
        cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        std::vector<double> hb((size_t)64 * N * K);
        for (size_t i = 0; i < hb.size(); ++i) hb[i] = ((i * 40503u) % 997) * 1e-3 - 0.5;
        cudaMemcpy(B, hb.data(), hb.size() * 8, cudaMemcpyHostToDevice);
    }
    // dense: C (32768 x 1024) = A (32768 x 1024) B^T (B: 1024 x 1024, K-major)
    Args dense{A, B, C, 0, 0, 0, M, N, K, K, K, N, 0};
    const double fd = 2.0 * M * N * K;
    // TRMM: 64 batches of H (512 x 1024) = W (512 x 1024) L^T, L lower (B(k,n) = L[n][k], k <= n)
    Args trmm{A, B, C, (int64_t)512 * K, (int64_t)N * K, (int64_t)512 * N, 512, N, K, K, K, N, 1};
    const double ft = 64.0 * 512 * (double)N * (N + 1);
    using Kept = Cfg<128, 64, 32, 2, true, true, 4, 2, 2>;
    using W4 = Cfg<64, 128, 16, 3, true, true, 2, 2, 2>;
    using W4b = Cfg<128, 64, 16, 3, true, true, 2, 2, 2>;
    using W4c = Cfg<64, 128, 32, 2, true, true, 2, 2, 2>;
    run<Kept, 0>(dense, 1, "dense kept 128x64x32x2 8w", fd);
    run<Kept, 1>(dense, 1, "dense kept + frag double buffer", fd);
    run<W4, 0>(dense, 1, "dense 64x128x16x3 4w (32x64)", fd);
    run<W4, 1>(dense, 1, "dense 64x128x16x3 4w + frag db", fd);
    run<W4b, 1>(dense, 1, "dense 128x64x16x3 4w (64x32) + frag db", fd);
    run<W4c, 1>(dense, 1, "dense 64x128x32x2 4w + frag db", fd);
    {
        // the accepted-rows product of one chain group at the adapted acceptance: 4 chains x
        // ~230 rows against the shared G^-1 (lower): per chain on 64-row tiles (now) against
        // the 4 chains' rows stacked into one product on 128-row tiles
        using K64x = Cfg<64, 64, 32, 2, true, true, 2, 2, 3>;
        Args per{A, B, C, (int64_t)230 * K, 0, (int64_t)230 * N, 230, N, K, K, K, N, 1};
        Args stacked{A, B, C, 0, 0, 0, 920, N, K, K, K, N, 1};
        const double fx = 920.0 * N * (N + 1);
        run<K64x, 0>(per, 4, "xi: 4 x 230 rows, 64x64 tiles", fx);
        run<Kept, 0>(stacked, 1, "xi: 920 stacked rows, 128x64 tiles", fx);
        run_pair<Kept>(stacked, 1, "xi: 920 stacked rows, 128x64 paired", fx);
        Args per64{A, B, C, (int64_t)230 * K, 0, (int64_t)230 * N, 230, N, K, K, K, N, 1};
        Args st64{A, B, C, 0, 0, 0, 230 * 64, N, K, K, K, N, 1};
        const double fx64 = 64.0 * 230 * N * (N + 1);
        run<K64x, 0>(per64, 64, "xi 64 chains: 64x64 tiles per chain", fx64);
        run<Kept, 0>(st64, 1, "xi 64 chains stacked: 128x64 tiles", fx64);
        run_pair<Kept>(st64, 1, "xi 64 chains stacked: 128x64 paired", fx64);
    }
    run<Kept, 0>(trmm, 64, "trmm kept", ft);
    run_pair<Kept>(trmm, 64, "trmm kept, paired column tiles", ft);
    using K64 = Cfg<64, 64, 32, 2, true, true, 2, 2, 3>;
    run<K64, 0>(trmm, 64, "trmm 64x64x32x2 4w 3/SM", ft);
    run_pair<K64>(trmm, 64, "trmm 64x64 paired", ft);
    run<Kept, 1>(trmm, 64, "trmm kept + frag db", ft);
    run<W4, 0>(trmm, 64, "trmm 64x128x16x3 4w", ft);
    run<W4, 1>(trmm, 64, "trmm 64x128x16x3 4w + frag db", ft);
    run<W4b, 1>(trmm, 64, "trmm 128x64x16x3 4w + frag db", ft);
    run<W4c, 1>(trmm, 64, "trmm 64x128x32x2 4w + frag db", ft);
    return 0;
}
