// host.cpp — host-side target construction/IO, diagnostics and JSON report.
//
// Target construction restates proj/src/target.cpp:18-152 and the dense helpers
// it relies on (proj/src/linalg.cpp) with the same arithmetic order, so that a
// target built here from (kind, d, seed) is bit-identical to the reference's
// (checked in tests/test_host_abi.py by comparing saved DIAMTGT files). It is
// O(d^3) host work (cyclic Jacobi), usable up to d of a few hundred exactly as
// in the reference; larger targets are loaded from DIAMTGT fixture files.
#include "host.hpp"

#include <algorithm>
#include <bit>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <numeric>
#include <sstream>
#include <thread>

#include "philox.cuh"

namespace dgb {

namespace {

// four interleaved lanes, folded ((l0+l1)+l2)+l3 — proj/src/linalg.cpp:43-54
double dot4(const double* a, const double* b, size_t n) {
    double s[4] = {0, 0, 0, 0};
    size_t j = 0;
    for (; j + 4 <= n; j += 4)
        for (int q = 0; q < 4; ++q) s[q] += a[j + q] * b[j + q];
    for (; j < n; ++j) s[0] += a[j] * b[j];
    return ((s[0] + s[1]) + s[2]) + s[3];
}

double host_normal(const PhiloxKey& k, uint64_t ctr) {
    // same as philox_normal, but through the host libm (as the reference)
    const Block4 b = philox_block(k, ctr);
    const uint64_t w0 = (static_cast<uint64_t>(b.w[1]) << 32) | b.w[0];
    const uint64_t w1 = (static_cast<uint64_t>(b.w[3]) << 32) | b.w[2];
    const double u1 = (static_cast<double>(w0 >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = static_cast<double>(w1 >> 11) * 0x1.0p-53;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
}

void check_sym(const Mat& m, const char* who) {
    require(m.rows == m.cols, Err::InvalidArgument, std::string(who) + ": matrix must be square");
    double mx = 0.0;
    for (double v : m.a) mx = std::max(mx, std::abs(v));
    const double tol = 1e-12 * std::max(mx, 1.0);
    for (size_t i = 0; i < m.rows; ++i)
        for (size_t j = i + 1; j < m.cols; ++j)
            require(std::abs(m(i, j) - m(j, i)) <= tol, Err::InvalidArgument,
                    std::string(who) + ": matrix not symmetric");
}

Mat chol(const Mat& m) {  // left-looking column Cholesky, proj/src/linalg.cpp:74-93
    check_sym(m, "cholesky");
    const size_t n = m.rows;
    Mat l(n, n);
    for (size_t j = 0; j < n; ++j) {
        double sq = 0.0;
        for (size_t k = 0; k < j; ++k) sq += l(j, k) * l(j, k);
        const double piv = m(j, j) - sq;
        if (piv <= 0.0 || !std::isfinite(piv))
            fail(Err::NotPositiveDefinite, "cholesky: pivot " + std::to_string(piv) + " at column " + std::to_string(j));
        l(j, j) = std::sqrt(piv);
        for (size_t i = j + 1; i < n; ++i) {
            double s = 0.0;
            for (size_t k = 0; k < j; ++k) s += l(i, k) * l(j, k);
            l(i, j) = (m(i, j) - s) / l(j, j);
        }
    }
    return l;
}

Vec fwd_solve(const Mat& l, const Vec& v) {
    const size_t n = l.rows;
    Vec y(n, 0.0);
    for (size_t i = 0; i < n; ++i) {
        require(l(i, i) != 0.0, Err::SingularDiagonal, "tri_solve: zero diagonal");
        y[i] = (v[i] - dot4(&l.a[i * n], y.data(), i)) / l(i, i);
    }
    return y;
}

Vec back_solve_t(const Mat& l, const Vec& v) {  // l^T y = v
    const size_t n = l.rows;
    Vec y(n, 0.0);
    for (size_t ii = n; ii-- > 0;) {
        require(l(ii, ii) != 0.0, Err::SingularDiagonal, "tri_solve_transposed: zero diagonal");
        double s = v[ii];
        for (size_t j = ii + 1; j < n; ++j) s -= l(j, ii) * y[j];
        y[ii] = s / l(ii, ii);
    }
    return y;
}

Mat spd_inverse(const Mat& m) {  // proj/src/linalg.cpp:95-115
    const Mat l = chol(m);
    const size_t n = l.rows;
    Mat inv(n, n);
    Vec e(n, 0.0);
    for (size_t j = 0; j < n; ++j) {
        e[j] = 1.0;
        const Vec col = back_solve_t(l, fwd_solve(l, e));
        for (size_t i = 0; i < n; ++i) inv(i, j) = col[i];
        e[j] = 0.0;
    }
    for (size_t i = 0; i < n; ++i)
        for (size_t j = i + 1; j < n; ++j) inv(i, j) = inv(j, i) = 0.5 * (inv(i, j) + inv(j, i));
    return inv;
}

double frob(const Mat& m) {
    double s = 0.0;
    for (double v : m.a) s += v * v;
    return std::sqrt(s);
}

// cyclic Jacobi, proj/src/linalg.cpp:178-250 (ascending, largest-|component| positive)
void jacobi_eigen(const Mat& m, Mat& vecs, Vec& vals) {
    check_sym(m, "sym_eigen");
    const size_t n = m.rows;
    Mat a = m;
    Mat v(n, n);
    for (size_t i = 0; i < n; ++i) v(i, i) = 1.0;
    auto off = [&] {
        double s = 0.0;
        for (size_t i = 0; i < n; ++i)
            for (size_t j = i + 1; j < n; ++j) s += a(i, j) * a(i, j);
        return std::sqrt(2.0 * s);
    };
    const double tol = 1e-14 * std::max(frob(m), 1.0);
    int sweeps = 0;
    while (off() > tol) {
        if (++sweeps > 64) fail(Err::ConvergenceFailure, "sym_eigen: Jacobi sweep cap exceeded");
        for (size_t p = 0; p + 1 < n; ++p)
            for (size_t q = p + 1; q < n; ++q) {
                const double apq = a(p, q);
                if (apq == 0.0) continue;
                const double th = (a(q, q) - a(p, p)) / (2.0 * apq);
                const double t = (th >= 0.0 ? 1.0 : -1.0) / (std::abs(th) + std::sqrt(1.0 + th * th));
                const double c = 1.0 / std::sqrt(1.0 + t * t);
                const double s = t * c;
                const double app = a(p, p), aqq = a(q, q);
                a(p, p) = app - t * apq;
                a(q, q) = aqq + t * apq;
                a(p, q) = a(q, p) = 0.0;
                for (size_t k = 0; k < n; ++k) {
                    if (k != p && k != q) {
                        const double akp = a(k, p), akq = a(k, q);
                        a(k, p) = c * akp - s * akq;
                        a(p, k) = a(k, p);
                        a(k, q) = s * akp + c * akq;
                        a(q, k) = a(k, q);
                    }
                    const double vkp = v(k, p), vkq = v(k, q);
                    v(k, p) = c * vkp - s * vkq;
                    v(k, q) = s * vkp + c * vkq;
                }
            }
    }
    std::vector<size_t> ord(n);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](size_t i, size_t j) { return a(i, i) < a(j, j); });
    vals.assign(n, 0.0);
    vecs = Mat(n, n);
    for (size_t j = 0; j < n; ++j) {
        const size_t src = ord[j];
        vals[j] = a(src, src);
        size_t arg = 0;
        double best = 0.0;
        for (size_t i = 0; i < n; ++i)
            if (std::abs(v(i, src)) > best) {
                best = std::abs(v(i, src));
                arg = i;
            }
        const double sg = v(arg, src) < 0.0 ? -1.0 : 1.0;
        for (size_t i = 0; i < n; ++i) vecs(i, j) = sg * v(i, src);
    }
}

Mat eigen_product(const Mat& v, const Vec& w) {  // v diag(w) v^T, proj/src/linalg.cpp:291-303
    const size_t n = v.rows;
    Mat out(n, n);
    for (size_t i = 0; i < n; ++i)
        for (size_t j = 0; j < n; ++j) {
            double s = 0.0;
            for (size_t k = 0; k < n; ++k) s += v(i, k) * w[k] * v(j, k);
            out(i, j) = s;
        }
    return out;
}

}  // namespace

// d x r standard normals of the target stream, element e = i r + k at counter e
// (proj/src/target.cpp:18-31), through the host libm as the reference
void target_normals(size_t d, size_t r, uint64_t seed, double* out) {
    const PhiloxKey key = make_philox_key(seed, 0, "target");
    const size_t n = d * r;
    // counter-indexed draws: split over host threads for the large targets
    const size_t nt = n < (size_t(1) << 20) ? 1 : std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (size_t t = 0; t < nt; ++t)
        pool.emplace_back([&, t] {
            for (size_t e = n * t / nt; e < n * (t + 1) / nt; ++e) out[e] = host_normal(key, e);
        });
    for (auto& th : pool) th.join();
}

namespace {

Mat gram(size_t d, size_t r, uint64_t seed) {  // A A^T with A ~ N(0,1) d x r, proj/src/target.cpp:18-31
    Mat a(d, r);
    target_normals(d, r, seed, a.a.data());
    Mat b(d, d);
    for (size_t i = 0; i < d; ++i)
        for (size_t j = 0; j <= i; ++j) {
            double s = 0.0;
            for (size_t k = 0; k < r; ++k) s += a(i, k) * a(j, k);
            b(i, j) = b(j, i) = s;
        }
    return b;
}

void finish_gaussian(HostTarget& t, const TargetOps* ops) {
    if (ops) {
        ops->inverse_and_eigen(t.precision, t.covariance, t.eigvecs, t.eigvals);
    } else {
        t.covariance = spd_inverse(t.precision);
        jacobi_eigen(t.covariance, t.eigvecs, t.eigvals);
    }
    t.mean.assign(t.dim, 0.0);
    t.eigen_mean.assign(t.dim, 0.0);
    t.eigen_var = t.eigvals;
    t.b_coeffs.assign(t.dim, 0.0);
}

using Out = BinOut;
using In = BinIn;

static_assert(std::endian::native == std::endian::little, "DIAMTGT is little-endian");
constexpr char kMagic[8] = {'D', 'I', 'A', 'M', 'T', 'G', 'T', '\0'};

}  // namespace

const char* tkind_name(TKind k) {
    static const char* names[] = {"pi1", "pi2", "pi3", "pi4", "pi5", "pi6"};
    return names[static_cast<int>(k)];
}

TKind tkind_from_name(const std::string& s) {
    for (int k = 0; k < 6; ++k)
        if (s == tkind_name(static_cast<TKind>(k))) return static_cast<TKind>(k);
    fail(Err::InvalidArgument, "unknown target kind: " + s);
}

double HostTarget::log_density(const double* x, size_t n) const {  // proj/src/target.cpp:154-165
    require(n == dim, Err::DimensionMismatch, "log_density: wrong dimension");
    Vec tmp(dim);
    if (!twisted()) {
        for (size_t i = 0; i < dim; ++i) tmp[i] = dot4(&precision.a[i * dim], x, dim);
        return -0.5 * dot4(x, tmp.data(), dim);
    }
    // z = V^T x, row i of V^T is column i of V
    Vec col(dim);
    for (size_t i = 0; i < dim; ++i) {
        for (size_t k = 0; k < dim; ++k) col[k] = eigvecs(k, i);
        tmp[i] = dot4(col.data(), x, dim);
    }
    double s = 0.0;
    for (size_t i = 0; i < dim; ++i) {
        double w = tmp[i];
        if ((i & 1) && b_coeffs[i - 1] != 0.0) w += b_coeffs[i - 1] * tmp[i - 1] * tmp[i - 1];
        s += w * w / eigvals[i];
    }
    return -0.5 * s;
}

HostTarget build_target(TKind kind, size_t dim, uint64_t seed, double sigma2, double twist_b, const TargetOps* ops) {
    require(dim >= 2, Err::InvalidDimension, "target dimension must be >= 2");
    HostTarget t;
    t.kind = kind;
    t.dim = dim;
    t.seed = seed;
    switch (kind) {
        case TKind::Pi1:
        case TKind::Pi2:
        case TKind::Pi3: {
            size_t rank = dim;
            if (kind == TKind::Pi3) {
                require(dim >= 10, Err::InvalidDimension, "pi3 needs d >= 10 so that r = d/10 >= 1");
                rank = dim / 10;
            }
            Mat b = ops ? ops->gram(dim, rank, seed) : gram(dim, rank, seed);
            if (kind == TKind::Pi2) {
                const double s = 1.0 / static_cast<double>(dim);
                for (double& v : b.a) v *= s;
            }
            for (size_t i = 0; i < dim; ++i) b(i, i) += 1.0;
            t.precision = std::move(b);
            finish_gaussian(t, ops);
            break;
        }
        case TKind::Pi4: {
            t.sigma2 = sigma2 > 0.0 ? sigma2 : 1.0 / static_cast<double>(dim);
            HostTarget base = build_target(TKind::Pi1, dim, seed, 0.0, -1.0, ops);
            const double inv_s2 = 1.0 / t.sigma2;
            Vec ce(dim), pe(dim);
            for (size_t n = 1; n <= dim; ++n) {
                const double nd = static_cast<double>(n);
                pe[n - 1] = inv_s2 / (nd * nd * nd * nd) + 1.0;
                ce[n - 1] = 1.0 / pe[n - 1];
            }
            t.precision = ops ? ops->eigen_product(base.eigvecs, pe) : eigen_product(base.eigvecs, pe);
            t.covariance = ops ? ops->eigen_product(base.eigvecs, ce) : eigen_product(base.eigvecs, ce);
            t.eigvecs = std::move(base.eigvecs);
            t.eigvals = ce;
            t.mean.assign(dim, 0.0);
            t.eigen_mean.assign(dim, 0.0);
            t.eigen_var = t.eigvals;
            t.b_coeffs.assign(dim, 0.0);
            break;
        }
        case TKind::Pi5:
        case TKind::Pi6: {
            require(dim % 20 == 0, Err::InvalidDimension, "twisted targets need d divisible by 20");
            t.twist_b = twist_b >= 0.0 ? twist_b : (kind == TKind::Pi5 ? 0.3 : 2.0);
            HostTarget base = build_target(TKind::Pi1, dim, seed, 0.0, -1.0, ops);
            t.eigvecs = std::move(base.eigvecs);
            t.eigvals = std::move(base.eigvals);
            const size_t m = dim / 10;
            const double rd = std::sqrt(static_cast<double>(dim));
            t.b_coeffs.assign(dim, 0.0);
            for (size_t i = 1; i < m; i += 2) t.b_coeffs[i - 1] = t.twist_b / (t.eigvals[i - 1] * rd);
            t.eigen_mean.assign(dim, 0.0);
            t.eigen_var = t.eigvals;
            for (size_t i = 2; i <= m; i += 2) {
                const double bp = t.b_coeffs[i - 2], sp = t.eigvals[i - 2];
                t.eigen_mean[i - 1] = -bp * sp;
                t.eigen_var[i - 1] = t.eigvals[i - 1] + 2.0 * bp * bp * sp * sp;
            }
            t.mean.assign(dim, 0.0);
            for (size_t i = 0; i < dim; ++i) t.mean[i] = dot4(&t.eigvecs.a[i * dim], t.eigen_mean.data(), dim);
            t.covariance = ops ? ops->eigen_product(t.eigvecs, t.eigen_var) : eigen_product(t.eigvecs, t.eigen_var);
            break;
        }
    }
    return t;
}

void save_target(const HostTarget& t, const std::string& path) {
    Out o(path);
    write_target_blob(o, t);
    o.close();
}

HostTarget load_target(const std::string& path) {
    In r(path);
    return read_target_blob(r);
}

void write_target_blob(BinOut& o, const HostTarget& t) {  // proj/src/target.cpp:187-204
    o.raw(kMagic, 8);
    o.pod<uint32_t>(1);
    o.pod<uint32_t>(0x01020304u);
    o.pod<uint32_t>(static_cast<uint32_t>(t.kind));
    o.pod<uint64_t>(t.dim);
    o.pod<uint64_t>(t.seed);
    o.pod<double>(t.sigma2);
    o.pod<double>(t.twist_b);
    o.mat(t.precision);
    o.mat(t.covariance);
    o.mat(t.eigvecs);
    o.vec(t.eigvals);
    o.vec(t.b_coeffs);
    o.vec(t.mean);
    o.vec(t.eigen_mean);
    o.vec(t.eigen_var);
}

HostTarget read_target_blob(BinIn& r) {  // proj/src/target.cpp:206-231
    char magic[8];
    r.raw(magic, 8);
    require(std::memcmp(magic, kMagic, 8) == 0, Err::Io, "not a target file");
    require(r.pod<uint32_t>() == 1, Err::Io, "unsupported target file version");
    require(r.pod<uint32_t>() == 0x01020304u, Err::Io, "endianness mismatch in target data");
    HostTarget t;
    const uint32_t k = r.pod<uint32_t>();
    require(k < 6, Err::Io, "corrupt target data");
    t.kind = static_cast<TKind>(k);
    t.dim = r.pod<uint64_t>();
    t.seed = r.pod<uint64_t>();
    t.sigma2 = r.pod<double>();
    t.twist_b = r.pod<double>();
    t.precision = r.mat();
    t.covariance = r.mat();
    t.eigvecs = r.mat();
    t.eigvals = r.vec();
    t.b_coeffs = r.vec();
    t.mean = r.vec();
    t.eigen_mean = r.vec();
    t.eigen_var = r.vec();
    require(t.dim >= 2 && t.covariance.rows == t.dim && t.eigvals.size() == t.dim, Err::Io, "corrupt target data");
    require(t.eigvecs.rows == t.dim && t.eigvecs.cols == t.dim && t.b_coeffs.size() == t.dim &&
                t.mean.size() == t.dim && (t.twisted() || t.precision.rows == t.dim),
            Err::Io, "corrupt target data");
    return t;
}

// ------------------------------------------------------------------ diagnostics (proj/src/diagnostics.cpp)
namespace {
double trace_mean(const double* x, size_t n) {
    double m = 0.0;
    for (size_t i = 0; i < n; ++i) m += x[i];
    return m / static_cast<double>(n);
}
double autocov(const double* x, size_t n, double m, size_t lag) {
    double c = 0.0;
    for (size_t t = 0; t + lag < n; ++t) c += (x[t] - m) * (x[t + lag] - m);
    return c / static_cast<double>(n);
}
double lag0(const double* x, size_t n, double m) {
    require(n >= 2, Err::DegenerateTrace, "trace too short");
    const double c0 = autocov(x, n, m, 0);
    require(c0 > 1e-20 * std::max(1.0, m * m) && std::isfinite(c0), Err::DegenerateTrace, "trace has zero variance");
    return c0;
}
double iact_capped(const double* x, size_t n, size_t max_lag) {
    const double m = trace_mean(x, n);
    const double c0 = lag0(x, n, m);
    double th = 0.0;
    for (size_t lag = 1; lag <= max_lag; ++lag) {
        const double rho = autocov(x, n, m, lag) / c0;
        if (rho < 0.05) break;
        th += rho;
    }
    return 1.0 + 2.0 * th;
}
}  // namespace

Vec acf(const double* x, size_t n, size_t max_lag) {
    require(max_lag < n / 2, Err::InvalidArgument, "acf: max_lag must be below half the trace length");
    const double m = trace_mean(x, n);
    const double c0 = lag0(x, n, m);
    Vec rho(max_lag + 1);
    rho[0] = 1.0;
    for (size_t lag = 1; lag <= max_lag; ++lag) rho[lag] = autocov(x, n, m, lag) / c0;
    return rho;
}

double iact(const double* x, size_t n) {
    require(n >= 2, Err::DegenerateTrace, "trace too short");
    return iact_capped(x, n, std::min<size_t>(n / 2 - 1, 10000));
}

double ess(const double* x, size_t n) { return static_cast<double>(n) / iact(x, n); }

QuadFit fit_quadratic(const double* xs, const double* ys, size_t n) {  // proj/src/fit.cpp:7-50
    require(n >= 3, Err::InvalidArgument, "fit_quadratic: need at least 3 points");
    Mat xtx(3, 3);
    Vec xty(3, 0.0);
    for (size_t i = 0; i < n; ++i) {
        const double row[3] = {1.0, xs[i], xs[i] * xs[i]};
        for (int a = 0; a < 3; ++a) {
            for (int b = 0; b <= a; ++b) {
                xtx(a, b) += row[a] * row[b];
                if (a != b) xtx(b, a) = xtx(a, b);
            }
            xty[a] += row[a] * ys[i];
        }
    }
    const Mat l = chol(xtx);
    const Vec beta = back_solve_t(l, fwd_solve(l, xty));
    QuadFit f;
    for (int a = 0; a < 3; ++a) f.coeffs[a] = beta[a];
    double ym = 0.0, qm = 0.0;
    for (size_t i = 0; i < n; ++i) {
        ym += ys[i];
        qm += beta[2] * xs[i] * xs[i];
    }
    ym /= static_cast<double>(n);
    qm /= static_cast<double>(n);
    double yv = 0.0, qv = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double pred = beta[0] + beta[1] * xs[i] + beta[2] * xs[i] * xs[i];
        const double res = ys[i] - pred;
        f.rss += res * res;
        yv += (ys[i] - ym) * (ys[i] - ym);
        const double q = beta[2] * xs[i] * xs[i];
        qv += (q - qm) * (q - qm);
    }
    f.quad_share = yv > 0.0 ? qv / yv : 0.0;
    return f;
}

double psrf_max(const std::vector<const double*>& means, const std::vector<const double*>& diags, size_t d,
                uint64_t n_per_chain) {
    const size_t p = means.size();
    require(p >= 2, Err::InvalidArgument, "psrf needs at least 2 chains");
    require(n_per_chain >= 2, Err::InvalidArgument, "psrf needs at least 2 samples per chain");
    Vec gm(d, 0.0);
    const double inv_p = 1.0 / static_cast<double>(p);
    for (size_t c = 0; c < p; ++c)
        for (size_t i = 0; i < d; ++i) gm[i] += inv_p * means[c][i];
    const double n = static_cast<double>(n_per_chain), pd = static_cast<double>(p);
    double mx = 0.0;
    for (size_t i = 0; i < d; ++i) {
        double between = 0.0, within = 0.0;
        for (size_t c = 0; c < p; ++c) {
            const double dl = means[c][i] - gm[i];
            between += dl * dl;
            within += diags[c][i] - means[c][i] * means[c][i];
        }
        const double b = n / (pd - 1.0) * between;
        const double w = n / ((n - 1.0) * pd) * within;
        require(w > 0.0, Err::ZeroWithinVariance, "psrf: zero within-chain variance in direction " + std::to_string(i));
        mx = std::max(mx, std::sqrt((n - 1.0) / n + (pd + 1.0) / (pd * n) * b / w));
    }
    return mx;
}

// ------------------------------------------------------------------ multi-GPU host logic
void shard_range(int64_t P, int world, int rank, int64_t* first, int64_t* count) {
    const int64_t a = P * rank / world, b = P * (rank + 1) / world;
    *first = a;
    *count = b - a;
}

void merge_weights(uint64_t global_count, uint64_t chains, uint64_t per_chain, double* keep, double* wp) {
    const uint64_t incoming = chains * per_chain;
    const double total = static_cast<double>(global_count + incoming);
    *keep = incoming ? static_cast<double>(global_count) / total : 1.0;
    *wp = incoming ? static_cast<double>(per_chain) / total : 0.0;
}

// ------------------------------------------------------------------ configuration
const char* kkind_name(KKind k) {
    static const char* names[] = {"rw", "pcn", "am", "diam"};
    return names[static_cast<int>(k)];
}

KKind kkind_from_name(const std::string& s) {
    for (int k = 0; k < 4; ++k)
        if (s == kkind_name(static_cast<KKind>(k))) return static_cast<KKind>(k);
    fail(Err::InvalidArgument, "unknown kernel: " + s);
}

KernelCfg KernelCfg::defaults(KKind k, size_t dim) {
    KernelCfg c;
    c.kind = k;
    c.dim = dim;
    c.beta_init = std::min(2.4 / std::sqrt(static_cast<double>(dim)), 0.5);
    c.n_lag = std::max<size_t>(1, dim / 2);
    const bool pcn = c.pcn_form();
    c.band_lo = pcn ? 0.3 : 0.1;
    c.band_hi = pcn ? 0.5 : 0.3;
    c.beta_max = pcn ? 1.0 : 10.0;
    c.n0 = 25 * static_cast<uint64_t>(dim);  // the code's default, not the header's 5d
    c.n_ref_start = 10 * static_cast<uint64_t>(dim);
    return c;
}

void validate_run_cfg(const RunCfg& c, const HostTarget& t) {
    const KernelCfg& k = c.kernel;
    require(k.dim == t.dim, Err::DimensionMismatch, "kernel dimension does not match the target");
    require(c.chains >= 1, Err::InvalidArgument, "need at least one chain");
    require(c.intervals_per_batch >= 1, Err::InvalidArgument, "M must be positive");
    require(k.n_lag >= 1, Err::InvalidArgument, "n_lag must be positive");
    require(k.beta_init > 0.0 && k.beta_init <= k.beta_max, Err::InvalidArgument, "beta_init must lie in (0, beta_max]");
    require(k.band_lo > 0.0 && k.band_lo < k.band_hi && k.band_hi < 1.0, Err::InvalidArgument,
            "acceptance band must satisfy 0 < lo < hi < 1");
    require(k.inflation >= 1.0, Err::InvalidArgument, "inflation must be >= 1");
    require(c.init_dispersion > 0.0, Err::InvalidArgument, "dispersion must be positive");
    require(c.trace_thin >= 1, Err::InvalidArgument, "trace thinning must be >= 1");
    if (c.psrf_tol) require(c.chains >= 2, Err::InvalidArgument, "the PSRF stopping rule needs at least 2 chains");
}

// ------------------------------------------------------------------ JSON report
namespace {
void jnum(std::ostringstream& o, double v) {
    if (!std::isfinite(v)) {
        o << "null";
        return;
    }
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    // keep a decimal point so the value reads back as a float
    std::string s(buf);
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    o << s;
}
void jarr(std::ostringstream& o, const Vec& v) {
    o << '[';
    for (size_t i = 0; i < v.size(); ++i) {
        if (i) o << ", ";
        jnum(o, v[i]);
    }
    o << ']';
}
void jstr(std::ostringstream& o, const std::string& s) {
    o << '"';
    for (char ch : s) {
        if (ch == '"' || ch == '\\') o << '\\';
        o << ch;
    }
    o << '"';
}
}  // namespace

std::string result_to_json(const RunResult& r) {  // field set of proj/src/report.cpp:18-77
    std::ostringstream o;
    o << "{\n  \"schema\": \"diam-run-result/1\",\n  \"target_kind\": ";
    jstr(o, r.target_kind);
    o << ",\n  \"kernel\": ";
    jstr(o, r.kernel_name);
    o << ",\n  \"dim\": " << r.dim << ",\n  \"chains\": " << r.chains << ",\n  \"intervals_per_batch\": "
      << r.intervals_per_batch << ",\n  \"n_lag\": " << r.n_lag << ",\n  \"master_seed\": " << r.master_seed
      << ",\n  \"total_samples\": " << r.total_samples << ",\n  \"batches\": " << r.batches
      << ",\n  \"wall_seconds\": ";
    jnum(o, r.wall_seconds);
    o << ",\n  \"batch_seconds\": ";
    jarr(o, r.batch_seconds);
    o << ",\n  \"stop_reason\": ";
    jstr(o, r.stop_reason);
    o << ",\n  \"accumulated_samples\": " << r.accumulated_samples << ",\n  \"global_mean\": ";
    jarr(o, r.global_mean);
    o << ",\n  \"final_cov_error\": ";
    jnum(o, r.final_cov_error);
    o << ",\n  \"final_mean_error\": ";
    jnum(o, r.final_mean_error);
    o << ",\n  \"final_max_psrf\": ";
    jnum(o, r.final_max_psrf);
    o << ",\n  \"cov_error_history\": ";
    jarr(o, r.cov_error_history);
    o << ",\n  \"mean_error_history\": ";
    jarr(o, r.mean_error_history);
    o << ",\n  \"psrf_history\": ";
    jarr(o, r.psrf_history);
    auto rows = [&](const std::vector<Vec>& m) {
        o << '[';
        for (size_t i = 0; i < m.size(); ++i) {
            if (i) o << ", ";
            jarr(o, m[i]);
        }
        o << ']';
    };
    o << ",\n  \"beta_history\": ";
    rows(r.beta_history);
    o << ",\n  \"acceptance_history\": ";
    rows(r.acceptance_history);
    o << ",\n  \"functionals\": [";
    for (size_t i = 0; i < r.functional_names.size(); ++i) {
        if (i) o << ", ";
        jstr(o, r.functional_names[i]);
    }
    o << "]";
    std::vector<Vec> ia, es;
    for (const auto& ch : r.traces) {
        Vec a, e;
        for (const Vec& tr : ch) {
            double tau = NAN;
            if (tr.size() >= 8) {
                try {
                    tau = iact(tr.data(), tr.size());
                } catch (const Error&) {
                    tau = NAN;
                }
            }
            a.push_back(tau);
            e.push_back(std::isfinite(tau) ? static_cast<double>(tr.size()) / tau : NAN);
        }
        ia.push_back(a);
        es.push_back(e);
    }
    o << ",\n  \"iact\": ";
    rows(ia);
    o << ",\n  \"ess\": ";
    rows(es);
    o << "\n}\n";
    return o.str();
}

}  // namespace dgb
