// diag_tc.cuh — Cholesky + inverse of one 64x64 diagonal block in shared memory, with the
// serial part on one warp and the rest on the FP64 tensor pipe (DMMA m8n8k4).
//
// The 64 columns are taken 8 at a time (left-looking, proj/src/linalg.cpp:74-93 reordered):
//   (a) panel update  A[k0:, k0:k0+8] -= L[k0:, :k0] L[k0:k0+8, :k0]^T    one 8x8 DMMA tile
//       per warp, K = k0;
//   (b) panel factor  the 8 columns of rows k0..63 by ONE warp (two rows per lane):
//       per column one rsqrt on the pivot's lane, a broadcast, and the rank-1 update of the
//       panel's remaining columns through shuffles -- no barriers inside the panel;
// then X = L^-1 by block forward substitution: the eight 8x8 diagonal inverses in
// parallel (one warp each), then block rows 1..7 in turn, each X_ij = -X_ii sum L_im X_mj
// on the DMMA pipe.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "gemm_tile.cuh"

namespace dgb {

constexpr int kDiagNb = 64;  // diagonal block size
constexpr int kD2 = 128;     // POTRF block column width (two diagonal blocks)
constexpr int kTcS = 68;
#ifdef DIAG_TC_PROFILE
__device__ long long g_tc_prof[16];
#define TC_MARK(i)                                                        \
    do {                                                                  \
        if (threadIdx.x == 0 && blockIdx.x == 0) g_tc_prof[i] = clock64(); \
    } while (0)
#else
#define TC_MARK(i) \
    do {           \
    } while (0)
#endif  // shared stride (doubles): 4 mod 16, conflict-free DMMA fragment loads

struct DiagTcScratch {
    double a[64 * kTcS];  // the block, then L
    double x[64 * kTcS];  // X = L^-1
    double t[8][64];      // per-warp staging of an 8x8 product
    double rdiag[64];     // 1 / L_kk (the panel's rsqrt of each pivot)
    int bad;
};

// 8x8 DMMA tile C (+)= A_rows[r0.., k..] * B_rows[n0.., k..]^T over k in [0, K), both
// operands row-major in shared memory with stride kTcS. acc: lane holds C[lane/4][2(lane%4)+{0,1}].
__device__ __forceinline__ void tc_tile(double (&acc)[2], const double* A, int r0, const double* B, int n0, int K,
                                        int lane) {
    const int fr = lane >> 2, fk = lane & 3;
    double e[2] = {0.0, 0.0}, o[2] = {0.0, 0.0};  // two chains: halve the dependent DMMA latency
    int k = 0;
    for (; k + 8 <= K; k += 8) {
        tile::dmma(e, A[(r0 + fr) * kTcS + k + fk], B[(n0 + fr) * kTcS + k + fk]);
        tile::dmma(o, A[(r0 + fr) * kTcS + k + 4 + fk], B[(n0 + fr) * kTcS + k + 4 + fk]);
    }
    if (k < K) tile::dmma(e, A[(r0 + fr) * kTcS + k + fk], B[(n0 + fr) * kTcS + k + fk]);
    acc[0] = e[0] + o[0];
    acc[1] = e[1] + o[1];
}

// pre_L (optional): the 64 columns left of the block (same rows, stride ld); the block is
// first updated A -= pre_L pre_L^T (the right-looking step a 128-wide block column's
// second half needs), in shared memory. With pre_X (64x64 lower, stride px_ld) pre_L still
// holds A's entries and is first solved in place, pre_L <- pre_L pre_X^T (the TRSM of
// those rows against the first half's inverse).
__device__ __forceinline__ int diag64_tc_sc(DiagTcScratch& sc, double* A, int64_t ld, int jb, double* out,
                                            int zero_above, int out_ld, double* pre_L = nullptr,
                                            const double* pre_X = nullptr, int px_ld = 64) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int fr = lane >> 2, fk = lane & 3;
    constexpr unsigned kAll = 0xffffffffu;
    double* sa = sc.a;
    double* sx = sc.x;
    // load the lower part; rows/cols past jb are the identity (a valid 64x64 factorization).
    // All 16 loads of a thread are in flight together (a loop that stores each value
    // before the next load would pay one L2 round trip per element: ~9000 cycles).
    {
        double v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int e = tid + 256 * i, r = e >> 6, q = e & 63;
            v[i] = (r < jb && q <= r) ? __ldcg(A + (int64_t)r * ld + q) : (r == q ? 1.0 : 0.0);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int e = tid + 256 * i;
            sa[(e >> 6) * kTcS + (e & 63)] = v[i];
        }
        if (pre_L) {  // stage pre_L (rows past jb: zero) in the inverse's buffer, free until then
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int e = tid + 256 * i, r = e >> 6, q = e & 63;
                v[i] = r < jb ? __ldcg(pre_L + (int64_t)r * ld + q) : 0.0;
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int e = tid + 256 * i;
                sx[(e >> 6) * kTcS + (e & 63)] = v[i];
            }
        }
    }
    if (pre_L && pre_X) {
        __syncthreads();
        // L = pre_L pre_X^T: warp w the 8 tiles of row tile w (pre_X[n][k] = 0 for k > n)
        const int r = 8 * warp + fr;
        double res[8][2];
#pragma unroll
        for (int ct = 0; ct < 8; ++ct) {
            double e[2] = {0.0, 0.0}, o[2] = {0.0, 0.0};
#pragma unroll
            for (int k = 0; k < 8 * ct + 8; k += 8) {
                tile::dmma(e, sx[r * kTcS + k + fk], __ldcg(pre_X + (8 * ct + fr) * px_ld + k + fk));
                tile::dmma(o, sx[r * kTcS + k + 4 + fk], __ldcg(pre_X + (8 * ct + fr) * px_ld + k + 4 + fk));
            }
            res[ct][0] = e[0] + o[0];
            res[ct][1] = e[1] + o[1];
        }
        __syncthreads();  // every warp has read its rows of sx
#pragma unroll
        for (int ct = 0; ct < 8; ++ct) {
            const int q = 8 * ct + 2 * fk;
            sx[r * kTcS + q] = res[ct][0];
            sx[r * kTcS + q + 1] = res[ct][1];
            if (r < jb) *reinterpret_cast<double2*>(pre_L + (int64_t)r * ld + q) = make_double2(res[ct][0], res[ct][1]);
        }
    }
    if (pre_L) {
        __syncthreads();
        // lower 8x8 tiles (ct <= rt) of A -= pre_L pre_L^T, up to 5 per warp
        for (int t = warp; t < 36; t += 8) {
            int rt = 0, base = 0;
            while (base + rt + 1 <= t) {
                base += rt + 1;
                ++rt;
            }
            const int ct = t - base;
            double acc[2];
            tc_tile(acc, sx, 8 * rt, sx, 8 * ct, 64, lane);
            sa[(8 * rt + fr) * kTcS + 8 * ct + 2 * fk] -= acc[0];
            sa[(8 * rt + fr) * kTcS + 8 * ct + 2 * fk + 1] -= acc[1];
        }
    }
    if (tid == 0) sc.bad = 0;
    TC_MARK(0);
    __syncthreads();
    TC_MARK(1);
    for (int p = 0; p < 8; ++p) {
        const int k0 = 8 * p;
        if (p > 0 && warp < 8 - p) {  // (a) row tile i = p + warp of the panel
            const int i = p + warp;
            double acc[2];
            tc_tile(acc, sa, 8 * i, sa, k0, k0, lane);
            sa[(8 * i + fr) * kTcS + k0 + 2 * fk] -= acc[0];
            sa[(8 * i + fr) * kTcS + k0 + 2 * fk + 1] -= acc[1];
        }
        __syncthreads();
        if (p == 3) TC_MARK(2);
        if (warp == 0) {  // (b) the panel: rows k0 + lane and k0 + 32 + lane
            const int r1 = k0 + lane, r2 = k0 + 32 + lane;
            const bool v1 = r1 < 64, v2 = r2 < 64;
            double pa[8], pb[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                pa[j] = v1 ? sa[r1 * kTcS + k0 + j] : 0.0;
                pb[j] = v2 ? sa[r2 * kTcS + k0 + j] : 0.0;
            }
            int bad = 0;
            // the pivot chain per column: shuffle the pivot, rsqrt, scale, and the next pivot's
            // own update (lane c+1: L[c+1][c]^2 from its own register, no shuffle); the other
            // columns' updates (one shuffle each) are off that chain
            double piv = __shfl_sync(kAll, pa[0], 0);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                if (!(piv > 0.0) || !isfinite(piv)) bad = 1;  // proj/src/linalg.cpp:82-84
                const double rl = rsqrt(piv);
                pa[c] = lane == c ? piv * rl : pa[c] * rl;
                pb[c] *= rl;
                if (lane == 0) sc.rdiag[k0 + c] = rl;
                if (c + 1 < 8) piv = __shfl_sync(kAll, pa[c + 1] - pa[c] * pa[c], c + 1);
#pragma unroll
                for (int j = c + 1; j < 8; ++j) {
                    const double lj = __shfl_sync(kAll, pa[c], j);  // L[k0+j][k0+c]
                    pa[j] -= pa[c] * lj;
                    pb[j] -= pb[c] * lj;
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (v1) sa[r1 * kTcS + k0 + j] = (lane >= j) ? pa[j] : 0.0;
                if (v2) sa[r2 * kTcS + k0 + j] = pb[j];
            }
            bad = __any_sync(kAll, bad);
            if (lane == 0 && bad) sc.bad = 1;
        }
        if (p == 3) TC_MARK(3);
        __syncthreads();
    }
    TC_MARK(4);
    if (sc.bad) return 1;
    // X = L^-1. Diagonal blocks: warp w inverts L_ww by columns (lane j < 8: column j).
    {
        const int b0 = 8 * warp;
        if (lane < 8) {
            const int j = lane;
            double xcol[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                double s = (i == j) ? 1.0 : 0.0;
#pragma unroll
                for (int k = 0; k < i; ++k) s -= sa[(b0 + i) * kTcS + b0 + k] * xcol[k];
                xcol[i] = s * sc.rdiag[b0 + i];  // 1 / L_ii from the panel (no division chain)
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) sx[(b0 + i) * kTcS + b0 + j] = (i >= j) ? xcol[i] : 0.0;
        }
        // the strict upper blocks of X are zero
        for (int e = lane; e < 8 * 64; e += 32) {
            const int r = b0 + (e >> 6), q = e & 63;
            if (q >= b0 + 8) sx[r * kTcS + q] = 0.0;
        }
    }
    __syncthreads();
    TC_MARK(5);
    // block rows i = 1..7: X_ij = -X_ii sum_{m=j}^{i-1} L_im X_mj, j < i (tile j by warp j)
    for (int i = 1; i < 8; ++i) {
        if (warp < i) {
            const int j = warp;
            // T = sum_m L_im X_mj: rows 8i.. of L times columns 8j.. of X, K over 8j..8i
            const double* Lr = sa + 8 * i * kTcS;
            double te[2] = {0.0, 0.0}, to[2] = {0.0, 0.0};
            for (int k = 8 * j; k < 8 * i; k += 8) {
                // A(m,k) = L[8i+m][k], B(k,n) = X[k][8j+n]
                tile::dmma(te, Lr[fr * kTcS + k + fk], sx[(k + fk) * kTcS + 8 * j + fr]);
                tile::dmma(to, Lr[fr * kTcS + k + 4 + fk], sx[(k + 4 + fk) * kTcS + 8 * j + fr]);
            }
            double* st = sc.t[warp];
            st[fr * 8 + 2 * fk] = te[0] + to[0];
            st[fr * 8 + 2 * fk + 1] = te[1] + to[1];
            __syncwarp();
            // X_ij = -X_ii T: A(m,k) = X[8i+m][8i+k], B(k,n) = T[k][n]
            double xe[2] = {0.0, 0.0};
            tile::dmma(xe, sx[(8 * i + fr) * kTcS + 8 * i + fk], st[fk * 8 + fr]);
            tile::dmma(xe, sx[(8 * i + fr) * kTcS + 8 * i + 4 + fk], st[(4 + fk) * 8 + fr]);
            sx[(8 * i + fr) * kTcS + 8 * j + 2 * fk] = -xe[0];
            sx[(8 * i + fr) * kTcS + 8 * j + 2 * fk + 1] = -xe[1];
        }
        __syncthreads();
    }
    TC_MARK(6);
    // store L (exact zeros above the diagonal: the left-looking GEMM's garbage) and X
    for (int e = 2 * tid; e < 64 * 64; e += 512) {  // pairs of columns (ld, out_ld even)
        const int r = e >> 6, q = e & 63;
        const bool v0 = r < jb && q < jb, v1 = r < jb && q + 1 < jb;
        const double2 l = make_double2(q <= r ? sa[r * kTcS + q] : 0.0, q + 1 <= r ? sa[r * kTcS + q + 1] : 0.0);
        const double2 x = make_double2(v0 && q <= r ? sx[r * kTcS + q] : 0.0, v1 && q + 1 <= r ? sx[r * kTcS + q + 1] : 0.0);
        if (v1) *reinterpret_cast<double2*>(A + (int64_t)r * ld + q) = l;
        else if (v0) A[(int64_t)r * ld + q] = l.x;
        *reinterpret_cast<double2*>(out + r * out_ld + q) = x;
        if (zero_above) {
            if (v1) *reinterpret_cast<double2*>(A + (int64_t)(r - kDiagNb) * ld + q) = make_double2(0.0, 0.0);
            else if (v0) A[(int64_t)(r - kDiagNb) * ld + q] = 0.0;
        }
    }
    TC_MARK(7);
    return 0;
}



}  // namespace dgb
