// host.hpp — host-side pieces behind the diam.h ABI that are not on the GPU
// hot path: synthetic targets (construction, DIAMTGT v1 IO, scalar log
// density), post-hoc trace diagnostics, the quadratic fit, error codes, and
// the run configuration / result types shared with the engine.
#pragma once

#include <cstdint>
#include <fstream>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace dgb {

// Error codes in diam_status order (proj/include/diam/error.hpp:8-19 semantics).
enum class Err { InvalidArgument = 1, InvalidDimension, DimensionMismatch, NotPositiveDefinite,
                 SingularDiagonal, ConvergenceFailure, DegenerateTrace, ZeroWithinVariance,
                 UnequalBatchSizes, Io, Unknown };

struct Error : std::runtime_error {
    Error(Err c, const std::string& what) : std::runtime_error(what), code(c) {}
    Err code;
};
[[noreturn]] inline void fail(Err c, const std::string& w) { throw Error(c, w); }
inline void require(bool ok, Err c, const std::string& w) {
    if (!ok) fail(c, w);
}

using Vec = std::vector<double>;

// Dense row-major square helpers (host).
struct Mat {
    size_t rows = 0, cols = 0;
    Vec a;
    Mat() = default;
    Mat(size_t r, size_t c) : rows(r), cols(c), a(r * c, 0.0) {}
    double& operator()(size_t i, size_t j) { return a[i * cols + j]; }
    double operator()(size_t i, size_t j) const { return a[i * cols + j]; }
};

// ---------------------------------------------------------------- little-endian binary IO
// (the DIAMTGT / DIAMCKPT field encodings of proj/src/binio.hpp: u32/u64/f64 raw,
// vectors as u64 length + data, matrices as u64 rows, u64 cols + row-major data)
struct BinOut {
    std::ofstream f;
    std::string path;
    std::vector<char> mem;  // memory mode (no path): the bytes a rank contributes to a file
    bool to_mem = false;
    explicit BinOut(const std::string& p) : f(p, std::ios::binary), path(p) {
        require(f.good(), Err::Io, "cannot open for writing: " + p);
    }
    BinOut() : to_mem(true) {}
    void raw(const void* p, size_t n) {
        if (to_mem) mem.insert(mem.end(), static_cast<const char*>(p), static_cast<const char*>(p) + n);
        else f.write(static_cast<const char*>(p), (std::streamsize)n);
    }
    template <class T>
    void pod(T v) {
        raw(&v, sizeof v);
    }
    void vec(const Vec& v) {
        pod<uint64_t>(v.size());
        raw(v.data(), v.size() * 8);
    }
    void mat(const Mat& m) {
        pod<uint64_t>(m.rows);
        pod<uint64_t>(m.cols);
        raw(m.a.data(), m.a.size() * 8);
    }
    void str(const std::string& s) {
        pod<uint64_t>(s.size());
        raw(s.data(), s.size());
    }
    void close() {
        if (to_mem) return;
        f.flush();
        require(f.good(), Err::Io, "write failed: " + path);
        f.close();
    }
};

struct BinIn {
    std::ifstream f;
    std::string path;
    explicit BinIn(const std::string& p) : f(p, std::ios::binary), path(p) {
        require(f.good(), Err::Io, "cannot open for reading: " + p);
    }
    void raw(void* p, size_t n) {
        f.read(static_cast<char*>(p), (std::streamsize)n);
        require(f.gcount() == (std::streamsize)n, Err::Io, "truncated file: " + path);
    }
    template <class T>
    T pod() {
        T v;
        raw(&v, sizeof v);
        return v;
    }
    size_t count() {
        const uint64_t n = pod<uint64_t>();
        require(n <= (1ull << 32), Err::Io, "implausible field size in " + path);
        return (size_t)n;
    }
    Vec vec() {
        Vec v(count());
        raw(v.data(), v.size() * 8);
        return v;
    }
    void skip(size_t n) {
        f.seekg((std::streamoff)n, std::ios::cur);
        require(f.good(), Err::Io, "truncated file: " + path);
    }
    void skip_vec() { skip(count() * 8); }
    void skip_mat() {
        const size_t r = count(), c = count();
        skip(r * c * 8);
    }
    Mat mat() {
        const size_t r = count(), c = count();
        Mat m(r, c);
        raw(m.a.data(), m.a.size() * 8);
        return m;
    }
    std::string str() {
        std::string s(count(), '\0');
        raw(s.data(), s.size());
        return s;
    }
    bool at_end() {
        return f.peek() == std::char_traits<char>::eof();
    }
};

// ---------------------------------------------------------------- targets
enum class TKind { Pi1 = 0, Pi2, Pi3, Pi4, Pi5, Pi6 };
const char* tkind_name(TKind k);
TKind tkind_from_name(const std::string& s);

struct HostTarget {
    TKind kind = TKind::Pi1;
    size_t dim = 0;
    uint64_t seed = 0;
    double sigma2 = 0.0, twist_b = 0.0;
    Mat precision;   // Gaussian kinds
    Mat covariance;  // analytic
    Mat eigvecs;     // columns, ascending eigenvalues
    Vec eigvals, b_coeffs, mean, eigen_mean, eigen_var;
    bool twisted() const { return kind == TKind::Pi5 || kind == TKind::Pi6; }
    double log_density(const double* x, size_t n) const;
};

// The O(d^3) pieces of target construction. The default (null) is the host restatement
// of the reference (bit-identical files, cyclic Jacobi: practical up to d ~ 1000);
// gpu_target_ops() runs them on the GPU for the benchmark sizes (target_gpu.cu).
struct TargetOps {
    virtual ~TargetOps() = default;
    // A A^T, A = d x r standard normals of the (seed, 0, "target") stream
    virtual Mat gram(size_t d, size_t r, uint64_t seed) const = 0;
    // covariance = precision^-1 and its eigenpairs (ascending, largest-|component| positive)
    virtual void inverse_and_eigen(const Mat& precision, Mat& covariance, Mat& eigvecs, Vec& eigvals) const = 0;
    // v diag(w) v^T
    virtual Mat eigen_product(const Mat& v, const Vec& w) const = 0;
};
const TargetOps* gpu_target_ops();  // null when no GPU / no cuSOLVER
void target_normals(size_t d, size_t r, uint64_t seed, double* out);  // the reference's A, bit-exact

HostTarget build_target(TKind kind, size_t dim, uint64_t seed, double sigma2, double twist_b,
                        const TargetOps* ops = nullptr);
void save_target(const HostTarget& t, const std::string& path);
HostTarget load_target(const std::string& path);
void write_target_blob(BinOut& o, const HostTarget& t);  // embedded in DIAMCKPT files
HostTarget read_target_blob(BinIn& r);

// ---------------------------------------------------------------- diagnostics
Vec acf(const double* x, size_t n, size_t max_lag);
double iact(const double* x, size_t n);
double ess(const double* x, size_t n);
struct QuadFit {
    double coeffs[3] = {0, 0, 0};
    double quad_share = 0.0, rss = 0.0;
};
QuadFit fit_quadratic(const double* xs, const double* ys, size_t n);
// max_i sqrt(R_i) from per-chain cumulative means / second-moment diagonals
// (proj/src/diagnostics.cpp:72-119); throws ZeroWithinVariance / InvalidArgument.
double psrf_max(const std::vector<const double*>& means, const std::vector<const double*>& diags, size_t d,
                uint64_t n_per_chain);

// ---------------------------------------------------------------- multi-GPU host logic
// Block sharding of P global chains over `world` ranks: rank r owns
// [r P / world, (r+1) P / world). RNG streams stay keyed by the global index.
void shard_range(int64_t P, int world, int rank, int64_t* first, int64_t* count);
// Weights of the batch merge (proj/src/moments.cpp:63-74): global <- keep*global
// + wp * sum_p local_p, with every chain holding `per_chain` samples.
void merge_weights(uint64_t global_count, uint64_t chains, uint64_t per_chain, double* keep, double* wp);

// ---------------------------------------------------------------- run config / result
enum class KKind { RW = 0, PCN, AM, DIAM };
const char* kkind_name(KKind k);
KKind kkind_from_name(const std::string& s);

struct KernelCfg {
    KKind kind = KKind::DIAM;
    size_t dim = 0;
    double beta_init = 0.0, inflation = 1.0;
    bool adaptive_ref = false;
    size_t n_lag = 0;
    double band_lo = 0.0, band_hi = 0.0;
    uint64_t n0 = 0, n_ref_start = 0;
    double beta_adapt_factor = 1.1, beta_min = 1e-6, beta_max = 1.0;
    bool adapt_beta = true, use_explicit_inverse = false;
    bool pcn_form() const { return kind == KKind::PCN || kind == KKind::DIAM; }
    bool adapts_cov() const { return kind == KKind::AM || kind == KKind::DIAM; }
    double noise_infl() const { return kind == KKind::DIAM ? inflation : 1.0; }
    static KernelCfg defaults(KKind k, size_t dim);  // proj/src/proposal.cpp:24-45
};

struct RunCfg {
    KernelCfg kernel;
    size_t chains = 1, intervals_per_batch = 1, max_batches = 100;
    std::optional<double> cov_tol, mean_tol, psrf_tol, max_wall_seconds;
    std::optional<uint64_t> max_samples;
    double init_dispersion = 1.0;
    uint64_t master_seed = 0;
    bool record_traces = true;
    size_t trace_thin = 1;
    bool trace_eigen_projections = true;
    std::string checkpoint_path;
    size_t threads = 0;
};
void validate_run_cfg(const RunCfg& c, const HostTarget& t);  // proj/src/runner.cpp:507-533

struct RunResult {
    std::string target_kind, kernel_name;
    size_t dim = 0, chains = 0, intervals_per_batch = 0, n_lag = 0;
    uint64_t master_seed = 0, total_samples = 0, accumulated_samples = 0;
    size_t batches = 0;
    double wall_seconds = 0.0;
    Vec batch_seconds;
    std::string stop_reason;
    Vec global_mean;
    Mat global_cov;
    double final_cov_error = 0, final_mean_error = 0, final_max_psrf = 0;
    Vec cov_error_history, mean_error_history, psrf_history;
    std::vector<Vec> beta_history, acceptance_history;  // [chain][boundary]
    std::vector<std::string> functional_names;
    std::vector<std::vector<Vec>> traces;  // [chain][functional]
};
std::string result_to_json(const RunResult& r);

}  // namespace dgb
