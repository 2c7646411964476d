// blas.cpp — see blas.hpp.
#include "blas.hpp"

#include <cublas_v2.h>
#include <dlfcn.h>

#include <mutex>
#include <string>

#include "common.cuh"

namespace dgb {

namespace {

struct Cublas {
    void* h = nullptr;
    cublasHandle_t handle = nullptr;
    cublasStatus_t (*create)(cublasHandle_t*) = nullptr;
    cublasStatus_t (*set_stream)(cublasHandle_t, cudaStream_t) = nullptr;
    cublasStatus_t (*dgemm)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int, const double*,
                            const double*, int, const double*, int, const double*, double*, int) = nullptr;
    std::mutex mu;  // one handle, stream set per call
};

Cublas* lib() {
    static Cublas* c = [] {
        auto* r = new Cublas;
        // a libcublas already in the process (e.g. PyTorch's) first, then the loader's search
        r->h = dlopen("libcublas.so.12", RTLD_NOW | RTLD_NOLOAD);
        if (!r->h) r->h = dlopen("libcublas.so.12", RTLD_NOW | RTLD_LOCAL);
        if (!r->h) r->h = dlopen("/usr/local/cuda/lib64/libcublas.so.12", RTLD_NOW | RTLD_LOCAL);
        if (!r->h) return r;
        r->create = (decltype(r->create))dlsym(r->h, "cublasCreate_v2");
        r->set_stream = (decltype(r->set_stream))dlsym(r->h, "cublasSetStream_v2");
        r->dgemm = (decltype(r->dgemm))dlsym(r->h, "cublasDgemm_v2");
        if (!r->create || !r->set_stream || !r->dgemm || r->create(&r->handle) != CUBLAS_STATUS_SUCCESS)
            r->handle = nullptr;
        return r;
    }();
    return c->handle ? c : nullptr;
}

}  // namespace

bool cublas_gemm_abt(cudaStream_t s, int m, int n, int k, const double* A, int64_t lda, const double* B, int64_t ldb,
                     double* C, int64_t ldc) {
    Cublas* c = lib();
    if (!c) return false;
    // column-major view: C^T (n x m) = B (n x k as B^T col-major, transposed) * A^T (k x m)
    const double one = 1.0, zero = 0.0;
    std::lock_guard<std::mutex> lk(c->mu);
    if (c->set_stream(c->handle, s) != CUBLAS_STATUS_SUCCESS) return false;
    const cublasStatus_t st = c->dgemm(c->handle, CUBLAS_OP_T, CUBLAS_OP_N, n, m, k, &one, B, (int)ldb, A, (int)lda,
                                       &zero, C, (int)ldc);
    if (st != CUBLAS_STATUS_SUCCESS)
        throw CudaError("cublasDgemm failed (status " + std::to_string((int)st) + ")");
    return true;
}

}  // namespace dgb
