// diag_block.cuh — register-blocked Cholesky + inverse of one 64x64 diagonal block by a
// 256-thread CTA (device function shared by the launch-per-phase POTRF in linalg.cu and
// the task-graph POTRF in potrf_dag.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace dgb {

constexpr int kDiagNb = 64;

// Loads go through L2 (__ldcg): in the task-graph POTRF another SM may have rewritten the
// block since this SM last cached it.
// Register-blocked right-looking Cholesky of one 64x64 diagonal block (at A, stride ld,
// jb <= 64 valid rows/cols), fused with the explicit inverse of the factor (for the DMMA
// TRSM that follows), by the 256 threads of a CTA. Thread (ty, tx) of a 16x16 grid owns
// the contiguous 4x4 sub-block rows 4ty+a, columns 4tx+b of both L and L^{-1} in
// registers. Writes L (zero strict upper part) back to A and the inverse to `out`
// (64x64 row-major). Returns nonzero (uniformly) on a bad pivot.
// shared scratch of one diagonal-block factorization (8.3 KB)
struct DiagScratch {
    double l[4][4], rd[4];        // L_kk (lower) and 1 / diag(L_kk)
    double col[2][kDiagNb][4];    // block column kg of L, rows 0..63
    double row[2][4][kDiagNb];    // block row kg of L^{-1}
    int bad;
};

__device__ __forceinline__ int diag64_block_sc(DiagScratch& sc, double* A, int64_t ld, int jb, double* out,
                                               int zero_above, int out_ld) {
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    double v[4][4], x[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int r = 4 * ty + a, q = 4 * tx + b;
            // rows/cols past jb are padded with the identity so the 64x64 factorization stays valid
            v[a][b] = (r < jb && q <= r) ? __ldcg(A + (int64_t)r * ld + q) : (r == q ? 1.0 : 0.0);
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
    if (tid == 0) sc.bad = 0;
    for (int kg = 0; kg < kDiagNb / 4; ++kg) {
        const int buf = kg & 1;
        if (ty == kg && tx == kg) {
            // A: 4x4 Cholesky of the diagonal tile; NotPositiveDefinite on a pivot <= 0 or
            // non-finite (proj/src/linalg.cpp:82-84) only raises `bad`, the discarded
            // arithmetic runs on
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                double p = v[cc][cc];
#pragma unroll
                for (int n = 0; n < cc; ++n) p -= v[cc][n] * v[cc][n];
                if (!(p > 0.0) || !isfinite(p)) sc.bad = 1;
                const double rl = rsqrt(p);  // one reciprocal square root per pivot
                sc.rd[cc] = rl;
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
                    sc.l[i][j] = v[i][j];
                }
        }
        __syncthreads();
        if (tx == kg) {  // B: tiles of block column kg (the diagonal tile is already final)
            double lk[4][4], rd[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                rd[m] = sc.rd[m];
#pragma unroll
                for (int n = 0; n < m; ++n) lk[m][n] = sc.l[m][n];
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
                    for (int m = 0; m < 4; ++m) sc.col[buf][r][m] = v[a][m];
            }
        }
        if (ty == kg) {  // B: block row kg of L^{-1}: L_kk X_k = Y_k, column by column
            double lk[4][4], rd[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                rd[m] = sc.rd[m];
#pragma unroll
                for (int n = 0; n < m; ++n) lk[m][n] = sc.l[m][n];
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
                for (int a = 0; a < 4; ++a) sc.row[buf][a][4 * tx + b] = x[a][b];
            }
        }
        __syncthreads();
        if (ty > kg) {  // C: rank-4 updates of the rows below block row kg
            double lr[4][4], xk[4][4];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int m = 0; m < 4; ++m) lr[a][m] = sc.col[buf][4 * ty + a][m];
#pragma unroll
            for (int m = 0; m < 4; ++m)
#pragma unroll
                for (int b = 0; b < 4; ++b) xk[m][b] = sc.row[buf][m][4 * tx + b];
            if (tx > kg && tx <= ty) {
                double lq[4][4];
#pragma unroll
                for (int b = 0; b < 4; ++b)
#pragma unroll
                    for (int m = 0; m < 4; ++m) lq[b][m] = sc.col[buf][4 * tx + b][m];
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
    const int failed = sc.bad;
    if (failed) return failed;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int r = 4 * ty + a;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int q = 4 * tx + b;
            // the block's strict upper part holds left-looking GEMM garbage: store exact zeros
            if (r < jb && q < jb) A[(int64_t)r * ld + q] = q <= r ? v[a][b] : 0.0;
            out[r * out_ld + q] = (r < jb && q < jb && q <= r) ? x[a][b] : 0.0;
            // second half of a 128-wide block column: the 64 rows above this block were
            // also touched by the block column's GEMM and lie above the diagonal
            if (zero_above && q < jb) A[(int64_t)(r - kDiagNb) * ld + q] = 0.0;
        }
    }
    return 0;
}

// the same with the scratch in static shared memory
__device__ __forceinline__ int diag64_block(double* A, int64_t ld, int jb, double* out, int zero_above,
                                            int out_ld = kDiagNb) {
    __shared__ DiagScratch sc;
    return diag64_block_sc(sc, A, ld, jb, out, zero_above, out_ld);
}

}  // namespace dgb
