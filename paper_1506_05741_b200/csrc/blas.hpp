// blas.hpp — the one plain library GEMM of the engine: the window's target product
// H = Xi G^T (one (C L) x d x d GEMM, no fused epilogue) through cuBLAS, which is dlopen'ed
// (the library loads without it; the engine then uses its own DMMA kernel).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace dgb {

// C = A B^T for row-major A (m x k, lda), B (n x k, ldb), C (m x n, ldc), FP64, on `s`.
// Returns false (nothing launched) when cuBLAS is unavailable.
bool cublas_gemm_abt(cudaStream_t s, int m, int n, int k, const double* A, int64_t lda, const double* B, int64_t ldb,
                     double* C, int64_t ldc);

}  // namespace dgb
