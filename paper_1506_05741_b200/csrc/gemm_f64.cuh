// gemm_f64.cuh — batched FP64 tensor-core GEMM for sm_100a.
//
// tcgen05.mma has no f64 kind, so FP64 work on B200 runs on the DMMA pipe
// (SASS DMMA.8x8x4, PTX mma.sync.m8n8k4.f64), which we measured at 37.1
// TFLOP/s against 33.9 TFLOP/s for plain DFMA (tools/fp64_peak.cu,
// profiles/r01_fp64_peaks.txt). This kernel is the dense-contraction engine
// behind every window-level operation of the sampler:
//
//   TRMM   Xi_c  = s_c * W_c * L_c^T      (B lower-triangular: K-loop clipped)
//   GEMM   H     = Xi * G^T               (G = precision or eigvecs^T, shared)
//   SYRK   S_c   = a*X_c^T X_c + b*S_c    (C lower: upper tiles skipped)
//   POTRF  A22  -= L21 L21^T, L21 = A21 L11^-T
//
// C[m][n] = alpha_b * sum_k A(m,k) B(k,n) + beta * C[m][n]
//   A_KMAJOR: A(m,k) = A[m*lda + k]   else A(m,k) = A[k*lda + m]
//   B_KMAJOR: B(k,n) = B[n*ldb + k]   else B(k,n) = B[k*ldb + n]
//
// Tiles: BM x BN per CTA, BK-deep stages streamed global->shared with
// cp.async (16 B, zero-filled at the edges) through a STAGES-deep ring, 8
// warps each owning a (BM/2) x (BN/4) sub-tile of 8x8 DMMA accumulators in
// registers. Shared-memory strides are padded to 4 (mod 16) doubles so the
// per-lane fragment loads (A: row lane/4, k lane%4) are bank-conflict free.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace dgb {

struct GemmBatch {
    // per-batch operand pointers (device arrays of device pointers)
    const double* const* A;
    const double* const* B;
    double* const* C;
    int64_t a_off, b_off, c_off;  // element offset added to every batch pointer
    int64_t lda, ldb, ldc;
    int M, N, K;
    double alpha;              // global scale
    const double* alpha_vec;   // optional per-batch scale (multiplied in)
    double alpha_vec_mul;      // multiplier on alpha_vec entries
    double beta;               // 0: C is write-only
    const int* active;         // optional per-batch mask (0 = skip)
    int tri_b_lower;           // B(k,n) == 0 for k > n  (K-loop clipped per n-tile)
    int tri_c_lower;           // compute/store only n <= m
    const int* k_vec;          // optional per-batch contraction length (<= K); 0 leaves
                               // C = beta C
    const int* m_vec;          // optional per-batch row count (<= M): rows past it untouched
};

// Launch the batched GEMM on `stream`. Layout flags select the template instance.
void gemm_f64(const GemmBatch& g, int batch, bool a_kmajor, bool b_kmajor, cudaStream_t stream);
// the same with 64 x 64 tiles (both operands K-major): shorter per-CTA latency for long K
void gemm_f64_small(const GemmBatch& g, int batch, cudaStream_t stream);

}  // namespace dgb
