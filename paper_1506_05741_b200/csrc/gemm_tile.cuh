// gemm_tile.cuh — one CTA tile of the FP64 DMMA GEMM, as a device function.
//
// Shared by the batched GEMM kernel (gemm_f64.cu) and the persistent per-chain
// Cholesky kernel (linalg.cu). C[m][n] = alpha * sum_k A(m,k) B(k,n) + beta * C[m][n]
// for the tile at (m0, n0):
//   AK : A(m,k) = A[m*lda + k]   else A[k*lda + m]
//   BKM: B(k,n) = B[n*ldb + k]   else B[k*ldb + n]
// BK-deep stages stream global->shared with 16-byte cp.async (zero-filled edges)
// through a STAGES-deep ring; 8 warps each own a WM x WN sub-tile of 8x8 DMMA
// (mma.sync.m8n8k4.f64, SASS DMMA.8x8x4) accumulators in registers; shared
// strides are 4 (mod 16) doubles so the per-lane fragment loads are conflict free.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace dgb {
namespace tile {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

template <int BM_, int BN_, int BK_, int STAGES_, bool AK, bool BKM, int WARPS_M_ = 2, int WARPS_N_ = 4,
          int MINB_ = 1>
struct Cfg {
    static constexpr int BM = BM_, BN = BN_, BK = BK_, STAGES = STAGES_;
    static constexpr int THREADS = 32 * WARPS_M_ * WARPS_N_;
    static constexpr int WARPS_M = WARPS_M_, WARPS_N = WARPS_N_;
    static constexpr int MINB = MINB_;  // CTAs resident per SM (register budget 64K / (THREADS * MINB))
    static constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;
    static constexpr int MI = WM / 8, NI = WN / 8;
    // shared layout: the global-contiguous dimension stays contiguous; stride = 4 mod 16
    static constexpr int A_ROWS = AK ? BM : BK;
    static constexpr int A_COLS = AK ? BK : BM;
    static constexpr int A_STRIDE = A_COLS + 4;
    static constexpr int B_ROWS = BKM ? BN : BK;
    static constexpr int B_COLS = BKM ? BK : BN;
    static constexpr int B_STRIDE = B_COLS + 4;
    static constexpr int A_STAGE = A_ROWS * A_STRIDE;
    static constexpr int B_STAGE = B_ROWS * B_STRIDE;
    static constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) * 8;
    static_assert(A_STRIDE % 16 == 4 && B_STRIDE % 16 == 4, "bank-conflict-free stride");
    static_assert((A_ROWS * A_COLS / 2) % THREADS == 0 && (B_ROWS * B_COLS / 2) % THREADS == 0, "copy split");
};

// Copy one rows x cols tile (cols contiguous in global) into shared memory.
// rows_valid / cols_valid are the in-bounds extents relative to the tile origin.
template <int ROWS, int COLS, int STRIDE, int THREADS>
__device__ __forceinline__ void load_tile(double* s, const double* g, int64_t ld, int rows_valid, int cols_valid,
                                          int tid) {
    constexpr int CHUNKS_PER_ROW = COLS / 2;
    constexpr int TOTAL = ROWS * CHUNKS_PER_ROW;
#pragma unroll
    for (int i = 0; i < TOTAL / THREADS; ++i) {
        const int c = tid + i * THREADS;
        const int r = c / CHUNKS_PER_ROW;
        const int cc = (c % CHUNKS_PER_ROW) * 2;
        int bytes = 0;
        if (r < rows_valid) bytes = cc + 1 < cols_valid ? 16 : (cc < cols_valid ? 8 : 0);
        const double* src = bytes ? g + r * ld + cc : g;
        cp_async16(s + r * STRIDE + cc, src, bytes);
    }
}

// The main loop of one BM x BN tile: acc = sum_k A(m,k) B(k,n) over k < K (the possibly
// triangle-clipped contraction length). Starts with a barrier so back-to-back calls may reuse
// the shared ring.
template <class CF, bool AK, bool BKM>
__device__ __forceinline__ void gemm_mainloop(const double* A, const double* B, int64_t lda, int64_t ldb, int M,
                                              int N, int K, int m0, int n0, bool tri_c_lower, double* smem,
                                              bool tri_b_lower, double (&acc)[CF::MI][CF::NI][2]) {
    __syncthreads();
    double* sA = smem;
    double* sB = smem + CF::STAGES * CF::A_STAGE;
    const int KT = (K + CF::BK - 1) / CF::BK;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int wm0 = (warp / CF::WARPS_N) * CF::WM;
    const int wn0 = (warp % CF::WARPS_N) * CF::WN;

    auto issue = [&](int kt, int stage) {
        const int k0 = kt * CF::BK;
        double* a_s = sA + stage * CF::A_STAGE;
        double* b_s = sB + stage * CF::B_STAGE;
        if (AK)
            load_tile<CF::A_ROWS, CF::A_COLS, CF::A_STRIDE, CF::THREADS>(a_s, A + (int64_t)m0 * lda + k0, lda, M - m0,
                                                                 K - k0, tid);
        else
            load_tile<CF::A_ROWS, CF::A_COLS, CF::A_STRIDE, CF::THREADS>(a_s, A + (int64_t)k0 * lda + m0, lda, K - k0,
                                                                 M - m0, tid);
        if (BKM)
            load_tile<CF::B_ROWS, CF::B_COLS, CF::B_STRIDE, CF::THREADS>(b_s, B + (int64_t)n0 * ldb + k0, ldb, N - n0,
                                                                 K - k0, tid);
        else
            load_tile<CF::B_ROWS, CF::B_COLS, CF::B_STRIDE, CF::THREADS>(b_s, B + (int64_t)k0 * ldb + n0, ldb, K - k0,
                                                                 N - n0, tid);
    };

#pragma unroll
    for (int i = 0; i < CF::MI; ++i)
#pragma unroll
        for (int j = 0; j < CF::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int s = 0; s < CF::STAGES - 1; ++s) {
        if (s < KT) issue(s, s);
        cp_async_commit();
    }

    const int fr = lane >> 2;  // fragment row (A) / col (B)
    const int fk = lane & 3;   // fragment k
    // a warp whose sub-tile lies entirely outside C (ragged edge tiles, e.g. the factor's
    // single augmented row) or, for a lower-triangular C, entirely above the diagonal only
    // helps with the copies (its DMMA issue slots go to the SM's other CTA)
    const bool compute = (m0 + wm0 < M) && (n0 + wn0 < N) && !(tri_c_lower && m0 + wm0 + CF::WM - 1 < n0 + wn0);
    for (int kt = 0; kt < KT; ++kt) {
        cp_async_wait<CF::STAGES - 2>();
        __syncthreads();
        const int nk = kt + CF::STAGES - 1;
        const double* a_s = sA + (kt % CF::STAGES) * CF::A_STAGE;
        const double* b_s = sB + (kt % CF::STAGES) * CF::B_STAGE;
        // B lower-triangular (B(k,n) = 0 for k > n): a stage entirely below this warp's
        // columns multiplies zeros only
        const bool live = compute && !(tri_b_lower && kt * CF::BK > n0 + wn0 + CF::WN - 1);
#pragma unroll
        for (int kk = 0; kk < CF::BK; kk += 4) {
            if (live) {
                double af[CF::MI], bf[CF::NI];
#pragma unroll
                for (int i = 0; i < CF::MI; ++i) {
                    const int m = wm0 + i * 8 + fr, k = kk + fk;
                    af[i] = AK ? a_s[m * CF::A_STRIDE + k] : a_s[k * CF::A_STRIDE + m];
                }
#pragma unroll
                for (int j = 0; j < CF::NI; ++j) {
                    const int n = wn0 + j * 8 + fr, k = kk + fk;
                    bf[j] = BKM ? b_s[n * CF::B_STRIDE + k] : b_s[k * CF::B_STRIDE + n];
                }
#pragma unroll
                for (int i = 0; i < CF::MI; ++i)
#pragma unroll
                    for (int j = 0; j < CF::NI; ++j) dmma(acc[i][j], af[i], bf[j]);
            }
            if (kk == 0) {
                // the next stage's copies go out behind the first DMMAs of this one, so the
                // tensor pipe restarts right after the barrier (the copy issue is ~150
                // instructions per thread). Stage nk % STAGES was consumed before the barrier.
                if (nk < KT) issue(nk, nk % CF::STAGES);
                cp_async_commit();
            }
        }
    }
    cp_async_wait<0>();
}

// C = alpha acc + beta C for the tile at (m0, n0) (lower part only if tri_c_lower).
// Epilogue in batches of IC fragment rows: all of a batch's C loads are issued before
// its stores (a store to C may alias a later load, so the compiler would otherwise
// serialise one L2 round trip per fragment).
template <class CF>
__device__ __forceinline__ void gemm_epilogue(const double (&acc)[CF::MI][CF::NI][2], double* Cp, int64_t ldc, int M,
                                              int N, int m0, int n0, double alpha, double beta, bool tri_c_lower) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm0 = (warp / CF::WARPS_N) * CF::WM;
    const int wn0 = (warp % CF::WARPS_N) * CF::WN;
    const int fr = lane >> 2, fk = lane & 3;
    constexpr int IC = CF::MI >= 2 ? 2 : 1;
#pragma unroll
    for (int i0 = 0; i0 < CF::MI; i0 += IC) {
        double2 old[IC][CF::NI];
#pragma unroll
        for (int ii = 0; ii < IC; ++ii) {
            const int r = m0 + wm0 + (i0 + ii) * 8 + fr;
#pragma unroll
            for (int j = 0; j < CF::NI; ++j) {
                const int c0 = n0 + wn0 + j * 8 + fk * 2;
                old[ii][j] = make_double2(0.0, 0.0);
                if (beta == 0.0 || r >= M) continue;
                // through L2: in the task-graph POTRF the tile may have been rewritten by
                // another SM since this one cached it
                const double* src = Cp + (int64_t)r * ldc + c0;
                const bool ok0 = c0 < N && (!tri_c_lower || c0 <= r);
                const bool ok1 = c0 + 1 < N && (!tri_c_lower || c0 + 1 <= r);
                if (ok0 && ok1) old[ii][j] = __ldcg(reinterpret_cast<const double2*>(src));
                else if (ok0) old[ii][j].x = __ldcg(src);
            }
        }
#pragma unroll
        for (int ii = 0; ii < IC; ++ii) {
            const int r = m0 + wm0 + (i0 + ii) * 8 + fr;
            if (r >= M) continue;
            double* crow = Cp + (int64_t)r * ldc;
#pragma unroll
            for (int j = 0; j < CF::NI; ++j) {
                const int c0 = n0 + wn0 + j * 8 + fk * 2;
                const bool ok0 = c0 < N && (!tri_c_lower || c0 <= r);
                const bool ok1 = c0 + 1 < N && (!tri_c_lower || c0 + 1 <= r);
                double2 v = make_double2(alpha * acc[i0 + ii][j][0], alpha * acc[i0 + ii][j][1]);
                if (beta != 0.0) {
                    v.x += beta * old[ii][j].x;
                    v.y += beta * old[ii][j].y;
                }
                if (ok0 && ok1) *reinterpret_cast<double2*>(crow + c0) = v;
                else if (ok0) crow[c0] = v.x;
            }
        }
    }
}

// One BM x BN tile of C: the main loop, then C = alpha acc + beta C.
template <class CF, bool AK, bool BKM>
__device__ __forceinline__ void gemm_tile(const double* A, const double* B, double* Cp, int64_t lda, int64_t ldb,
                                          int64_t ldc, int M, int N, int K, int m0, int n0, double alpha,
                                          double beta, bool tri_c_lower, double* smem, bool tri_b_lower = false) {
    if (beta != 0.0) {
        // read-modify-write epilogue: pull the C tile towards L2 while the main loop runs
        constexpr int LINES_PER_ROW = (CF::BN * 8 + 127) / 128;
        for (int li = threadIdx.x; li < CF::BM * LINES_PER_ROW; li += CF::THREADS) {
            const int r = m0 + li / LINES_PER_ROW, cc = n0 + (li % LINES_PER_ROW) * 16;
            if (r < M && cc < N) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(Cp + (int64_t)r * ldc + cc));
        }
    }
    double acc[CF::MI][CF::NI][2];
    gemm_mainloop<CF, AK, BKM>(A, B, lda, ldb, M, N, K, m0, n0, tri_c_lower, smem, tri_b_lower, acc);
    gemm_epilogue<CF>(acc, Cp, ldc, M, N, m0, n0, alpha, beta, tri_c_lower);
}

}  // namespace tile
}  // namespace dgb
