// ref_shim.cpp — TEST INFRASTRUCTURE. Exposes a few internal C++ functions of
// the reference (compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libdiam_ref.so) through plain C symbols, so that the oracle
// restatement (oracle/diam_oracle.c) can be pinned against the reference
// itself. Nothing here is product code.
#include <cstring>
#include <span>
#include <vector>

#include "diam/linalg.hpp"
#include "diam/moments.hpp"
#include "diam/proposal.hpp"
#include "diam/rng.hpp"

using namespace diam;

extern "C" {

void shim_fill_u64(uint64_t seed, uint64_t idx, const char* purpose, uint64_t start, size_t n,
                   uint64_t* out) {
    RngStream s = make_rng_stream(seed, idx, purpose);
    s.set_draw_count(start);
    for (size_t i = 0; i < n; ++i) out[i] = s.next_u64();
}

void shim_fill_uniform_open(uint64_t seed, uint64_t idx, const char* purpose, uint64_t start,
                            size_t n, double* out) {
    RngStream s = make_rng_stream(seed, idx, purpose);
    s.set_draw_count(start);
    for (size_t i = 0; i < n; ++i) out[i] = s.uniform_open();
}

void shim_fill_normal(uint64_t seed, uint64_t idx, const char* purpose, uint64_t start, size_t n,
                      double* out) {
    RngStream s = make_rng_stream(seed, idx, purpose);
    s.set_draw_count(start);
    for (size_t i = 0; i < n; ++i) out[i] = s.normal();
}

static LowerTriangular lower_from(const double* l, size_t n) {
    LowerTriangular t(n);
    std::memcpy(t.a.data(), l, n * n * sizeof(double));
    return t;
}

void shim_tri_matvec(const double* l, size_t n, const double* v, double* y) {
    const Vector r = tri_matvec(lower_from(l, n), std::span<const double>(v, n));
    std::memcpy(y, r.data(), n * sizeof(double));
}

int shim_tri_solve(const double* l, size_t n, const double* v, double* y) {
    try {
        const Vector r = tri_solve(lower_from(l, n), std::span<const double>(v, n));
        std::memcpy(y, r.data(), n * sizeof(double));
        return 0;
    } catch (const Error& e) {
        return 1 + static_cast<int>(e.code());
    }
}

void shim_sym_matvec(const double* m, size_t n, const double* v, double* y) {
    Matrix mm(n, n);
    std::memcpy(mm.a.data(), m, n * n * sizeof(double));
    const Vector r = sym_matvec(mm, std::span<const double>(v, n));
    std::memcpy(y, r.data(), n * sizeof(double));
}

// 0 ok; else 1 + ErrorCode
int shim_cholesky(const double* m, size_t n, double* l, int jittered) {
    Matrix mm(n, n);
    std::memcpy(mm.a.data(), m, n * n * sizeof(double));
    try {
        KernelConfig cfg = KernelConfig::defaults(KernelKind::DIAM, n);
        const LowerTriangular f = jittered ? jittered_cholesky(mm, cfg) : cholesky(mm);
        std::memcpy(l, f.a.data(), n * n * sizeof(double));
        return 0;
    } catch (const Error& e) {
        return 1 + static_cast<int>(e.code());
    }
}

// running accumulate of `rows` samples into fresh moments
void shim_accumulate(size_t d, size_t rows, const double* x, double* mean, double* second) {
    MomentAccumulator acc(d);
    for (size_t r = 0; r < rows; ++r) acc.accumulate(std::span<const double>(x + r * d, d));
    std::memcpy(mean, acc.mean.data(), d * sizeof(double));
    std::memcpy(second, acc.second.a.data(), d * d * sizeof(double));
}

}  // extern "C"
