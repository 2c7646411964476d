// target_gpu.cu — the O(d^3) pieces of diam_target_build on the GPU.
//
// The reference builds targets with a cyclic Jacobi eigensolver and column-by-column
// inverse (proj/src/target.cpp:66-152, proj/src/linalg.cpp:95-115, 178-250): exact, but
// hours at d = 4096. Here, for the benchmark sizes:
//   gram           A A^T: A drawn on the host exactly as the reference (same Philox
//                  stream, host libm), the product as a lower-triangle DMMA GEMM
//                  (gemm_f64) mirrored to a symmetric matrix;
//   inverse+eigen  P = V diag(lambda) V^T by cuSOLVER's divide-and-conquer syevd (the
//                  one library call: an eigensolver is off the sampler's hot path),
//                  then covariance = P^-1 = V diag(1/lambda) V^T as a DMMA GEMM; the
//                  covariance's eigenpairs are P's, reversed (ascending 1/lambda), with
//                  the reference's sign convention (largest-|component| positive);
//   eigen_product  V diag(w) V^T as a lower-triangle DMMA GEMM, mirrored.
// Results agree with the host restatement to rounding (tests/test_gpu_kernels.py), not
// bit-for-bit: DIAMTGT files of this builder differ from the reference's in the last
// bits. cuSOLVER is dlopen'ed so the library loads without it.
#include <dlfcn.h>

#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "common.cuh"
#include "gemm_f64.cuh"
#include "host.hpp"

namespace dgb {

namespace {

struct Solver {
    void* h = nullptr;
    std::string err;
    cusolverStatus_t (*create)(cusolverDnHandle_t*) = nullptr;
    cusolverStatus_t (*destroy)(cusolverDnHandle_t) = nullptr;
    cusolverStatus_t (*set_stream)(cusolverDnHandle_t, cudaStream_t) = nullptr;
    cusolverStatus_t (*bufsize)(cusolverDnHandle_t, cusolverEigMode_t, cublasFillMode_t, int, const double*, int,
                                const double*, int*) = nullptr;
    cusolverStatus_t (*syevd)(cusolverDnHandle_t, cusolverEigMode_t, cublasFillMode_t, int, double*, int, double*,
                              double*, int, int*) = nullptr;
    bool ok() const { return h && create && destroy && set_stream && bufsize && syevd; }
};

// The process may already hold a libcublas.so.12 (PyTorch's wheel): prefer a cuSOLVER
// that is already loaded, then the one next to that cuBLAS, then the system's.
Solver& solver() {
    static Solver s = [] {
        Solver r;
        std::vector<std::string> cands;
        if (void* cb = dlopen("libcublas.so.12", RTLD_NOW | RTLD_NOLOAD)) {
            Dl_info info{};
            void* sym = dlsym(cb, "cublasCreate_v2");
            if (sym && dladdr(sym, &info) && info.dli_fname) {
                std::string p = info.dli_fname;  // .../nvidia/cublas/lib/libcublas.so.12
                const size_t cut = p.rfind("/cublas/lib/");
                if (cut != std::string::npos) cands.push_back(p.substr(0, cut) + "/cusolver/lib/libcusolver.so.11");
            }
            dlclose(cb);
        }
        cands.push_back("libcusolver.so.11");
        cands.push_back("/usr/local/cuda/lib64/libcusolver.so.11");
        if (void* h = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_NOLOAD)) r.h = h;
        for (size_t i = 0; !r.h && i < cands.size(); ++i) {
            r.h = dlopen(cands[i].c_str(), RTLD_NOW | RTLD_LOCAL);
            if (!r.h) {
                const char* e = dlerror();
                r.err += cands[i] + ": " + (e ? e : "?") + "; ";
            }
        }
        if (!r.h) return r;
        r.create = (decltype(r.create))dlsym(r.h, "cusolverDnCreate");
        r.destroy = (decltype(r.destroy))dlsym(r.h, "cusolverDnDestroy");
        r.set_stream = (decltype(r.set_stream))dlsym(r.h, "cusolverDnSetStream");
        r.bufsize = (decltype(r.bufsize))dlsym(r.h, "cusolverDnDsyevd_bufferSize");
        r.syevd = (decltype(r.syevd))dlsym(r.h, "cusolverDnDsyevd");
        if (!r.ok()) r.err += "cuSOLVER symbols missing";
        return r;
    }();
    return s;
}

void sol_check(cusolverStatus_t st, const char* what) {
    require(st == CUSOLVER_STATUS_SUCCESS, Err::Unknown, std::string("cuSOLVER ") + what + " failed (status " +
                                                              std::to_string((int)st) + ")");
}

struct DevBuf {
    double* p = nullptr;
    explicit DevBuf(size_t n) { DGB_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(double))); }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

// host rows x cols (row-major) <-> device rows x ld
void upload(double* dst, int64_t ld, const double* src, size_t rows, size_t cols) {
    DGB_CUDA(cudaMemcpy2D(dst, ld * 8, src, cols * 8, cols * 8, rows, cudaMemcpyHostToDevice));
}
void download(double* dst, const double* src, int64_t ld, size_t rows, size_t cols) {
    DGB_CUDA(cudaMemcpy2D(dst, cols * 8, src, ld * 8, cols * 8, rows, cudaMemcpyDeviceToHost));
}

// lower triangle of X Y^T (both n x k row-major on the device, leading dimension ld)
// -> symmetric host matrix
Mat sym_product(const double* X, const double* Y, int64_t ld, size_t n, size_t k) {
    const int64_t ldc = pad_ld((int64_t)n);
    DevBuf out((size_t)n * ldc);
    double** ptrs = nullptr;
    DGB_CUDA(cudaMalloc(&ptrs, 3 * sizeof(double*)));
    const double* hp[3] = {X, Y, out.p};
    DGB_CUDA(cudaMemcpy(ptrs, hp, sizeof hp, cudaMemcpyHostToDevice));
    GemmBatch g{};
    g.A = (const double* const*)ptrs;
    g.B = (const double* const*)(ptrs + 1);
    g.C = ptrs + 2;
    g.lda = g.ldb = ld;
    g.ldc = ldc;
    g.M = g.N = (int)n;
    g.K = (int)k;
    g.alpha = 1.0;
    g.beta = 0.0;
    g.tri_c_lower = 1;
    gemm_f64(g, 1, true, true, 0);  // A(m,k) = X[m ld + k], B(k,n) = Y[n ld + k]
    DGB_CUDA(cudaStreamSynchronize(0));
    cudaFree(ptrs);
    Mat m(n, n);
    download(m.a.data(), out.p, ldc, n, n);
    for (size_t i = 0; i < n; ++i)
        for (size_t j = 0; j < i; ++j) m(j, i) = m(i, j);
    return m;
}

class GpuOps final : public TargetOps {
public:
    Mat gram(size_t d, size_t r, uint64_t seed) const override {
        std::vector<double> a(d * r);
        target_normals(d, r, seed, a.data());
        const int64_t ld = pad_ld((int64_t)r);
        DevBuf A(d * ld);
        DGB_CUDA(cudaMemset(A.p, 0, d * ld * 8));
        upload(A.p, ld, a.data(), d, r);
        return sym_product(A.p, A.p, ld, d, r);
    }

    void inverse_and_eigen(const Mat& P, Mat& cov, Mat& vecs, Vec& vals) const override {
        Solver& s = solver();
        require(s.ok(), Err::Unknown, "cuSOLVER unavailable for the GPU target builder: " + s.err);
        const size_t n = P.rows;
        const int64_t ld = pad_ld((int64_t)n);
        DevBuf A(n * ld), w(n);
        DGB_CUDA(cudaMemset(A.p, 0, n * ld * 8));
        upload(A.p, ld, P.a.data(), n, n);
        cusolverDnHandle_t h = nullptr;
        sol_check(s.create(&h), "create");
        std::unique_ptr<void, void (*)(void*)> guard(h, [](void* p) {
            solver().destroy(static_cast<cusolverDnHandle_t>(p));
        });
        sol_check(s.set_stream(h, 0), "set_stream");
        // P is symmetric: its row-major array is its column-major array
        int lwork = 0;
        sol_check(s.bufsize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)n, A.p, (int)ld, w.p, &lwork),
                  "syevd_bufferSize");
        DevBuf work((size_t)lwork);
        int* info = nullptr;
        DGB_CUDA(cudaMalloc(&info, sizeof(int)));
        sol_check(s.syevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)n, A.p, (int)ld, w.p, work.p, lwork,
                          info),
                  "syevd");
        int hinfo = 0;
        DGB_CUDA(cudaMemcpy(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost));
        cudaFree(info);
        require(hinfo == 0, Err::ConvergenceFailure, "sym_eigen: syevd info " + std::to_string(hinfo));
        // eigenvector j of P (ascending lambda_j) is column j of the column-major result,
        // i.e. row j of the row-major array
        Vec lam(n);
        DGB_CUDA(cudaMemcpy(lam.data(), w.p, n * 8, cudaMemcpyDeviceToHost));
        Mat rows(n, n);  // rows(j, i) = component i of P's eigenvector j
        download(rows.a.data(), A.p, ld, n, n);
        for (size_t j = 0; j < n; ++j)
            require(lam[j] > 0.0 && std::isfinite(lam[j]), Err::NotPositiveDefinite,
                    "precision not positive definite (eigenvalue " + std::to_string(lam[j]) + ")");
        // covariance eigenpairs: mu_j = 1 / lambda_{n-1-j} ascending; sign: largest-|component|
        // positive (proj/src/linalg.cpp:238-247)
        vals.assign(n, 0.0);
        vecs = Mat(n, n);
        for (size_t j = 0; j < n; ++j) {
            const size_t src = n - 1 - j;
            vals[j] = 1.0 / lam[src];
            const double* v = &rows.a[src * n];
            size_t arg = 0;
            double best = 0.0;
            for (size_t i = 0; i < n; ++i)
                if (std::abs(v[i]) > best) {
                    best = std::abs(v[i]);
                    arg = i;
                }
            const double sg = v[arg] < 0.0 ? -1.0 : 1.0;
            for (size_t i = 0; i < n; ++i) vecs(i, j) = sg * v[i];
        }
        cov = eigen_product(vecs, vals);
    }

    Mat eigen_product(const Mat& v, const Vec& wv) const override {
        // V diag(w) V^T = X V^T with X = V diag(w): lower triangle as one GEMM
        const size_t n = v.rows;
        const int64_t ld = pad_ld((int64_t)n);
        std::vector<double> x(v.a);
        for (size_t i = 0; i < n; ++i)
            for (size_t k = 0; k < n; ++k) x[i * n + k] *= wv[k];
        DevBuf X(n * ld), V(n * ld);
        DGB_CUDA(cudaMemset(X.p, 0, n * ld * 8));
        DGB_CUDA(cudaMemset(V.p, 0, n * ld * 8));
        upload(X.p, ld, x.data(), n, n);
        upload(V.p, ld, v.a.data(), n, n);
        return sym_product(X.p, V.p, ld, n, n);
    }
};

}  // namespace

const TargetOps* gpu_target_ops() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return nullptr;
    }
    if (!solver().ok()) return nullptr;
    static GpuOps ops;
    return &ops;
}

}  // namespace dgb
