// diag_bench.cu — time the POTRF diagonal-block kernel alone (64 chains, one 64x64 block
// each), against an empty launch, with CUDA events. Build + run on a B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -lineinfo \
//        -Ipaper_1506_05741_b200/csrc tools/diag_bench.cu -Lpaper_1506_05741_b200 -ldiam \
//        -Xlinker -rpath,$PWD/paper_1506_05741_b200 -o tools/diag_bench && tools/diag_bench
#include <cstdio>
#include <vector>

#define DIAG_TC_PROFILE
#include "../paper_1506_05741_b200/csrc/linalg.cu"

__global__ void empty_kernel() {}

// pure dependent-chain latencies, unrolled (no loop overhead): 128 DFMA, 128 LDS.64 chase
__global__ void lat2_kernel(long long* cyc, double* out, double a, double b) {
    __shared__ double sh[256];
    __shared__ int idx[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        sh[i] = 1.0 + i;
        idx[i] = (i * 7 + 1) & 255;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    double x = a;
    long long t0 = clock64();
#pragma unroll
    for (int i = 0; i < 128; ++i) x = fma(x, b, a);
    long long t1 = clock64();
    int j = 0;
#pragma unroll
    for (int i = 0; i < 128; ++i) j = idx[j];
    long long t2 = clock64();
    double y = x;
#pragma unroll
    for (int i = 0; i < 32; ++i) y = rsqrt(y + 1.0);
    long long t3 = clock64();
    cyc[0] = (t1 - t0) / 128;
    cyc[1] = (t2 - t1) / 128;
    cyc[2] = (t3 - t2) / 32;
    out[0] = x + j + y;
}

// barrier round trips: 256 threads, 64 iterations of (smem write by one thread, barrier,
// everyone reads it, barrier)
__global__ void barrier_kernel(long long* cyc, double* out) {
    __shared__ double v;
    double acc = 0.0;
    long long t0 = clock64();
    for (int i = 0; i < 64; ++i) {
        if (threadIdx.x == (i & 255)) v = acc + i;
        __syncthreads();
        acc += v;
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[3] = (t1 - t0) / 64;
    if (acc == -1.0) out[0] = acc;
}

// dependent-chain latencies (cycles per op), one thread
__global__ void lat_kernel(double* out, long long* cyc, double a, double b) {
    double x = a;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1000; ++i) x = fma(x, b, a);
    long long t1 = clock64();
    double y = x;
#pragma unroll 1
    for (int i = 0; i < 200; ++i) y = rsqrt(y + 2.0);
    long long t2 = clock64();
    double z = y;
#pragma unroll 1
    for (int i = 0; i < 200; ++i) z = 1.0 / (z + 3.0);
    long long t3 = clock64();
    float f = (float)a;
#pragma unroll 1
    for (int i = 0; i < 1000; ++i) f = fmaf(f, (float)b, (float)a);
    long long t4 = clock64();
    out[0] = x + y + z + f;
    cyc[0] = (t1 - t0) / 1000;
    cyc[1] = (t2 - t1) / 200;
    cyc[2] = (t3 - t2) / 200;
    cyc[3] = (t4 - t3) / 1000;
}

namespace dgb {
namespace {
// experimental copy of diag64_block: F bit 0 skips phase A, 1 phase B, 2 phase C,
// 3 the barrier after A, 4 the barrier after B (timing only: results are wrong)
template <int F>
__device__ __forceinline__ int diag_exp(double* A, int64_t ld, int jb, double* out, int zero_above,
                                        long long* cyc = nullptr) {
    long long tA = 0, tStep = 0, tPrev = 0, tB = 0;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    __shared__ double colk[2][kNb], xrow[2][kNb];
    __shared__ double piv;
    __shared__ int bad;
    double v[4][4], x[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int r = 4 * ty + a, q = 4 * tx + b;
            // rows/cols past jb are padded with the identity so the 64x64 factorization stays valid
            v[a][b] = (r < jb && q <= r) ? A[(int64_t)r * ld + q] : (r == q ? 1.0 : 0.0);
            x[a][b] = (r == q) ? 1.0 : 0.0;
        }
    // Blocked by the 4x4 register tiles: step kg finalises block column kg of L and block
    // row kg of L^{-1} with two barriers (32 in total instead of two per column):
    //   A  thread (kg,kg) factors its diagonal 4x4 tile (in registers) and publishes it
    //      with the reciprocal pivots -- the only serial piece, so nothing else happens here
    //   B  column-owners solve their tile L_ik = A_ik L_kk^-T and row-owners finish block
    //      row kg of the inverse X_k = L_kk^-1 Y_k, both by 4-step forward substitution;
    //      both publish through shared memory
    //   C  everyone applies the rank-4 updates A_ij -= L_ik L_jk^T and Y_i -= L_ik X_k
    __shared__ double s_l[4][4], s_rd[4];  // L_kk (lower) and 1 / diag(L_kk)
    __shared__ double s_col[2][kNb][4];    // block column kg of L, rows 0..63
    __shared__ double s_row[2][4][kNb];    // block row kg of L^{-1}
    (void)colk;
    (void)xrow;
    (void)piv;
    if (tid == 0) bad = 0;
    for (int kg = 0; kg < kNb / 4; ++kg) {
        const int buf = kg & 1;
        long long a0 = clock64();
        if ((F & 1) == 0 && ty == kg && tx == kg) {
            // A: 4x4 Cholesky of the diagonal tile; NotPositiveDefinite on a pivot <= 0 or
            // non-finite (proj/src/linalg.cpp:82-84) only raises `bad`, the discarded
            // arithmetic runs on
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                double p = v[cc][cc];
#pragma unroll
                for (int n = 0; n < cc; ++n) p -= v[cc][n] * v[cc][n];
                if (!(p > 0.0) || !isfinite(p)) bad = 1;
                const double rl = rsqrt(p);  // one reciprocal square root per pivot
                s_rd[cc] = rl;
                v[cc][cc] = p * rl;
#pragma unroll
                for (int rr = cc + 1; rr < 4; ++rr) {
                    double s = v[rr][cc];
#pragma unroll
                    for (int n = 0; n < cc; ++n) s -= v[rr][n] * v[cc][n];
                    v[rr][cc] = s * rl;
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (j > i) v[i][j] = 0.0;
                    s_l[i][j] = v[i][j];
                }
        }
        if (ty == kg && tx == kg) tA += clock64() - a0;
        if ((F & 8) == 0) __syncthreads();
        long long b0 = clock64();
        if (tid == 0) {
            if (kg > 0) tStep += b0 - tPrev;
            tPrev = b0;
        }
        if ((F & 2) == 0 && (F & 64) == 0 && tx == kg) {  // B: tiles of block column kg (the diagonal tile is already final)
            double lk[4][4], rd[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                rd[m] = s_rd[m];
#pragma unroll
                for (int n = 0; n < m; ++n) lk[m][n] = s_l[m][n];
            }
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const int r = 4 * ty + a;
                if (ty > kg) {
                    // row a of A_ik L_kk^-T: t L_kk^T = v  (forward substitution along the row)
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        double s = v[a][m];
#pragma unroll
                        for (int n = 0; n < m; ++n) s -= v[a][n] * lk[m][n];
                        v[a][m] = s * rd[m];
                    }
                }
                if (ty >= kg)
#pragma unroll
                    for (int m = 0; m < 4; ++m) s_col[buf][r][m] = v[a][m];
            }
        }
        if ((F & 2) == 0 && (F & 32) == 0 && ty == kg) {  // B: block row kg of L^{-1}: L_kk X_k = Y_k, column by column
            double lk[4][4], rd[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                rd[m] = s_rd[m];
#pragma unroll
                for (int n = 0; n < m; ++n) lk[m][n] = s_l[m][n];
            }
#pragma unroll
            for (int b = 0; b < 4; ++b) {
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    double s = x[a][b];
#pragma unroll
                    for (int n = 0; n < a; ++n) s -= lk[a][n] * x[n][b];
                    x[a][b] = s * rd[a];
                }
#pragma unroll
                for (int a = 0; a < 4; ++a) s_row[buf][a][4 * tx + b] = x[a][b];
            }
        }
        if ((F & 16) == 0) __syncthreads();
        if (tid == 0) tB += clock64() - b0;
        if ((F & 4) == 0 && ty > kg) {  // C: rank-4 updates of the rows below block row kg
            double lr[4][4], xk[4][4];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int m = 0; m < 4; ++m) lr[a][m] = s_col[buf][4 * ty + a][m];
#pragma unroll
            for (int m = 0; m < 4; ++m)
#pragma unroll
                for (int b = 0; b < 4; ++b) xk[m][b] = s_row[buf][m][4 * tx + b];
            if (tx > kg && tx <= ty) {
                double lq[4][4];
#pragma unroll
                for (int b = 0; b < 4; ++b)
#pragma unroll
                    for (int m = 0; m < 4; ++m) lq[b][m] = s_col[buf][4 * tx + b][m];
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        double s = v[a][b];
#pragma unroll
                        for (int m = 0; m < 4; ++m) s -= lr[a][m] * lq[b][m];
                        v[a][b] = s;
                    }
            }
            if (tx <= kg) {  // Y_i -= L_ik X_k (X_k is zero right of block column kg)
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        double s = x[a][b];
#pragma unroll
                        for (int m = 0; m < 4; ++m) s -= lr[a][m] * xk[m][b];
                        x[a][b] = s;
                    }
            }
        }
    }
    __syncthreads();
    if (cyc && blockIdx.x == 0) {
        if (tid == 0) { cyc[0] = tStep; cyc[1] = tB; }
        if (tx == ty) atomicAdd((unsigned long long*)&cyc[2], (unsigned long long)tA);
    }
    const int failed = bad;
    if (failed) return failed;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int r = 4 * ty + a;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int q = 4 * tx + b;
            // the block's strict upper part holds left-looking GEMM garbage: store exact zeros
            if (r < jb && q < jb) A[(int64_t)r * ld + q] = q <= r ? v[a][b] : 0.0;
            out[r * kNb + q] = (r < jb && q < jb && q <= r) ? x[a][b] : 0.0;
            // second half of a 128-wide block column: the 64 rows above this block were
            // also touched by the block column's GEMM and lie above the diagonal
            if (zero_above && q < jb) A[(int64_t)(r - kNb) * ld + q] = 0.0;
        }
    }
    return 0;
}

template <int F>
__global__ void __launch_bounds__(256, 2) diag_exp_kernel(double* const* Am, int64_t ld, int jb, int* status, double* inv,
                                                         long long* cyc = nullptr) {
    const int c = blockIdx.x;
    if (diag_exp<F>(Am[c], ld, jb, inv + (int64_t)c * 64 * 64, 0, cyc) && threadIdx.x == 0) status[c] = 1;
}
}  // namespace
}  // namespace dgb

int main() {
    using namespace dgb;
    const int chains = 64, n = 64, ld = 64;
    std::vector<double> h((size_t)chains * n * ld, 0.0);
    for (int c = 0; c < chains; ++c)
        for (int i = 0; i < n; ++i)
            for (int j = 0; j <= i; ++j) {
                double s = (i == j) ? n : 0.0;
                s += 1.0 / (1.0 + i + j + c);
                h[(size_t)c * n * ld + i * ld + j] = s;
            }
    double *A, *A0, *inv;
    int *status, *active;
    double** Ap;
    cudaMalloc(&A, h.size() * 8);
    cudaMalloc(&A0, h.size() * 8);
    cudaMalloc(&inv, (size_t)chains * 64 * 64 * 8);
    cudaMalloc(&status, chains * 4);
    cudaMalloc(&active, chains * 4);
    cudaMemcpy(A0, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    std::vector<double*> hp(chains);
    for (int c = 0; c < chains; ++c) hp[c] = A + (size_t)c * n * ld;
    cudaMalloc(&Ap, chains * sizeof(double*));
    cudaMemcpy(Ap, hp.data(), chains * sizeof(double*), cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](auto launch, const char* name) {
        float tot = 0.f;
        const int reps = 50;
        for (int r = 0; r < reps + 3; ++r) {
            cudaMemcpy(A, A0, h.size() * 8, cudaMemcpyDeviceToDevice);
            cudaMemset(status, 0, chains * 4);
            cudaDeviceSynchronize();
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r >= 3) tot += ms;
        }
        int st = 0;
        cudaMemcpy(&st, status, 4, cudaMemcpyDeviceToHost);
        printf("%-28s %8.2f us  (status[0]=%d, %s)\n", name, tot / reps * 1e3, st,
               cudaGetErrorString(cudaGetLastError()));
    };
    {
        double* o;
        long long* cy;
        cudaMalloc(&o, 8);
        cudaMalloc(&cy, 4 * 8);
        lat_kernel<<<1, 1>>>(o, cy, 0.5, 0.999);
        long long hc[4];
        cudaMemcpy(hc, cy, 32, cudaMemcpyDeviceToHost);
        lat2_kernel<<<1, 256>>>(cy, o, 0.5, 0.999);
        long long hl[4];
        cudaMemcpy(hl, cy, 32, cudaMemcpyDeviceToHost);
        printf("unrolled dependent latency: DFMA %lld cycles, LDS.32 chase %lld, rsqrt(double)+add %lld\n", hl[0], hl[1], hl[2]);
        barrier_kernel<<<64, 256>>>(cy, o);
        long long hb[4];
        cudaMemcpy(hb, cy, 32, cudaMemcpyDeviceToHost);
        printf("two barriers + smem broadcast per iteration: %lld cycles\n", hb[3]);
        printf("latency (cycles, incl. loop): dfma %lld, rsqrt(double)+add %lld, div(double)+add %lld, ffma %lld\n",
               hc[0], hc[1], hc[2], hc[3]);
    }
    timeit([&] { empty_kernel<<<chains, 256>>>(); }, "empty launch");
    timeit([&] { potrf_diag_kernel<2, false><<<chains, 256>>>(Ap, ld, 0, 64, nullptr, status, active, inv, 0); },
           "diag64 (minb 2)");
    timeit([&] { potrf_diag_kernel<1, false><<<chains, 256>>>(Ap, ld, 0, 64, nullptr, status, active, inv, 0); },
           "diag64 (minb 1)");
    cudaFuncSetAttribute(potrf_diag_kernel<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(DiagTcScratch));
    timeit([&] { potrf_diag_kernel<1, true><<<chains, 256, sizeof(DiagTcScratch)>>>(Ap, ld, 0, 64, nullptr, status,
                                                                                     active, inv, 0); },
           "diag64 TC");
    {
        long long pr[16];
        cudaMemcpyFromSymbol(pr, dgb::g_tc_prof, sizeof pr);
        printf("TC phases (cycles): load %lld, panels 0-2 + (a)3 %lld, (b)3 %lld, panels 4-7 %lld, diag inv %lld, "
               "block rows %lld, store %lld\n", pr[1] - pr[0], pr[2] - pr[1], pr[3] - pr[2], pr[4] - pr[3],
               pr[5] - pr[4], pr[6] - pr[5], pr[7] - pr[6]);
    }
    {  // 128x128 diagonal block (diag128_tc): phases
        const int n2 = 128;
        std::vector<double> h2((size_t)chains * n2 * n2, 0.0);
        for (int c = 0; c < chains; ++c)
            for (int i = 0; i < n2; ++i)
                for (int j = 0; j <= i; ++j)
                    h2[(size_t)c * n2 * n2 + i * n2 + j] = (i == j ? n2 : 0.0) + 1.0 / (1.0 + i + j + c);
        double *B, *inv2;
        double** Bp;
        cudaMalloc(&B, h2.size() * 8);
        cudaMalloc(&inv2, (size_t)chains * 128 * 128 * 8);
        std::vector<double*> hb(chains);
        for (int c = 0; c < chains; ++c) hb[c] = B + (size_t)c * n2 * n2;
        cudaMalloc(&Bp, chains * sizeof(double*));
        cudaMemcpy(Bp, hb.data(), chains * sizeof(double*), cudaMemcpyHostToDevice);
        cudaFuncSetAttribute(potrf_diag128_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDiag128SmemBytes);
        float tot = 0.f;
        for (int r = 0; r < 13; ++r) {
            cudaMemcpy(B, h2.data(), h2.size() * 8, cudaMemcpyHostToDevice);
            cudaMemset(status, 0, chains * 4);
            cudaDeviceSynchronize();
            cudaEventRecord(e0);
            potrf_diag128_kernel<<<chains, 256, kDiag128SmemBytes>>>(Bp, n2, 0, n2, nullptr, status, active, inv2);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r >= 3) tot += ms;
        }
        int st = 0;
        cudaMemcpy(&st, status, 4, cudaMemcpyDeviceToHost);
        long long pr[16];
        cudaMemcpyFromSymbol(pr, dgb::g_tc_prof, sizeof pr);
        printf("diag128 TC %8.2f us (status %d, %s); cycles: diag A11 %lld, L21 %lld, A22/U %lld, diag A22 %lld, "
               "X21 %lld; inside the last diag64: panels %lld, inverse %lld, store %lld\n",
               tot / 10 * 1e3, st, cudaGetErrorString(cudaGetLastError()), pr[9] - pr[8], pr[10] - pr[9],
               pr[11] - pr[10], pr[12] - pr[11], pr[13] - pr[12], pr[4] - pr[1], pr[6] - pr[4], pr[7] - pr[6]);
    }
    timeit([&] { diag_exp_kernel<0><<<chains, 256>>>(Ap, ld, 64, status, inv); }, "exp full");
    auto cyc = [&](auto launch, const char* name) {
        long long* cy;
        cudaMalloc(&cy, 4 * 8);
        cudaMemset(cy, 0, 32);
        cudaMemcpy(A, A0, h.size() * 8, cudaMemcpyDeviceToDevice);
        cudaMemset(status, 0, chains * 4);
        launch(cy);
        long long hc[4];
        cudaMemcpy(hc, cy, 32, cudaMemcpyDeviceToHost);
        printf("%-20s cycles per step %.0f, B %.0f, A %.0f\n", name, hc[0] / 15.0, hc[1] / 16.0, hc[2] / 16.0);
        cudaFree(cy);
    };
    cyc([&](long long* cy) { diag_exp_kernel<32><<<chains, 256>>>(Ap, ld, 64, status, inv, cy); }, "no row-owner B");
    cyc([&](long long* cy) { diag_exp_kernel<64><<<chains, 256>>>(Ap, ld, 64, status, inv, cy); }, "no col-owner B");
    cyc([&](long long* cy) { diag_exp_kernel<96><<<chains, 256>>>(Ap, ld, 64, status, inv, cy); }, "no B at all");
    {
        long long* cy;
        cudaMalloc(&cy, 4 * 8);
        cudaMemset(cy, 0, 32);
        cudaMemcpy(A, A0, h.size() * 8, cudaMemcpyDeviceToDevice);
        cudaMemset(status, 0, chains * 4);
        diag_exp_kernel<0><<<chains, 256>>>(Ap, ld, 64, status, inv, cy);
        long long hc[4];
        cudaMemcpy(hc, cy, 32, cudaMemcpyDeviceToHost);
        printf("cycles: 15 steps %lld (%.0f per step), phase B (barrier to barrier) %lld (%.0f per step), phase A total %lld (%.0f per step)\n",
               hc[0], hc[0] / 15.0, hc[1], hc[1] / 16.0, hc[2], hc[2] / 16.0);
    }
    timeit([&] { diag_exp_kernel<1><<<chains, 256>>>(Ap, ld, 64, status, inv); }, "exp no A");
    timeit([&] { diag_exp_kernel<2><<<chains, 256>>>(Ap, ld, 64, status, inv); }, "exp no B");
    timeit([&] { diag_exp_kernel<4><<<chains, 256>>>(Ap, ld, 64, status, inv); }, "exp no C");
    timeit([&] { diag_exp_kernel<7><<<chains, 256>>>(Ap, ld, 64, status, inv); }, "exp no ABC");
    timeit([&] { diag_exp_kernel<24><<<chains, 256>>>(Ap, ld, 64, status, inv); }, "exp no barriers");
    timeit([&] { diag_exp_kernel<31><<<chains, 256>>>(Ap, ld, 64, status, inv); }, "exp load/store only");
    return 0;
}
