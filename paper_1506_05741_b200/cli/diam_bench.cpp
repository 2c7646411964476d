// diam_bench — the reference CLI's `benchmark` subcommand (proj/tools/diam_cli.cpp:427-505)
// as a standalone driver over the C ABI (include/diam/diam.h) and nothing else, so the same
// source links against this library (paper_1506_05741_b200/diam_bench) or against the
// reference's own libdiam (oracle/_ref/diam_bench_ref, oracle/Makefile) unchanged.
//
//   diam_bench [benchmark] --target pi1 --kernel diam --dims 256 512 1024 --samples 200000
//              [--chain-sweep 1 2 4 ...] [--out benchmark.csv] [sampler options]
//
// Dimension sweep: one run per d with traces, checkpoints and stopping tolerances off, n0 = 0
// unless given, and max_batches = ceil(samples / (chains * intervals * n_lag)); CSV rows
// "d,total_samples,wall_seconds,sec_per_sample,sec_per_batch", then the per-sample cost fit
// T(d) = c0 + c1 d + c2 d^2 (diam_fit_quadratic). Chain sweep: one run per P with the given
// options; rows "P,total_seconds,sec_per_batch,N". The reference's CLI11 option parser is
// absent from this image, so options are parsed by hand with the same names.
// Exit codes as the reference CLI: 0 ok, 1 configuration error, 2 runtime error.
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "diam/diam.h"

namespace {

constexpr int kExitOk = 0, kExitConfig = 1, kExitRuntime = 2;

int exit_code_for(diam_status s) {
    if (s == DIAM_OK) return kExitOk;
    if (s == DIAM_ERR_INVALID_ARGUMENT || s == DIAM_ERR_INVALID_DIMENSION || s == DIAM_ERR_DIMENSION_MISMATCH)
        return kExitConfig;
    return kExitRuntime;
}

int report_failure(const char* what, diam_status s) {
    std::fprintf(stderr, "error: %s: %s (%s)\n", what, diam_status_string(s), diam_last_error());
    return exit_code_for(s);
}

std::string fmt(double v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

struct Target {
    diam_target* t = nullptr;
    ~Target() { diam_target_free(t); }
};
struct Result {
    diam_result* r = nullptr;
    ~Result() { diam_result_free(r); }
};

struct Options {
    std::string target = "pi1", kernel = "diam", out = "benchmark.csv";
    int64_t dim = 100, n_lag = -1, n0 = -1, n_ref_start = -1, chains = 1, intervals = 10, max_batches = 1000;
    int64_t samples = 20000, threads = 0, max_samples = -1;
    uint64_t target_seed = 1, seed = 0;
    double sigma2 = -1.0, twist_b = -1.0, beta = -1.0, inflation = -1.0, band_lo = -1.0, band_hi = -1.0;
    double dispersion = 1.0, max_wall = -1.0;
    bool adaptive_ref = false, explicit_inverse = false, no_adapt_beta = false;
    std::vector<int64_t> dims, chain_sweep;

    int build(int64_t d, Target& out_t) const {
        const bool kind = target.rfind("pi", 0) == 0 && target.size() == 3;
        const diam_status st = kind ? diam_target_build(target.c_str(), d, target_seed, sigma2, twist_b, &out_t.t)
                                    : diam_target_load(target.c_str(), &out_t.t);
        return st == DIAM_OK ? kExitOk : report_failure("building target", st);
    }
    void fill(diam_run_options& o) const {  // proj/tools/diam_cli.cpp:141-178
        diam_run_options_init(&o);
        o.kernel = kernel.c_str();
        o.beta_init = beta;
        o.inflation = inflation;
        o.band_lo = band_lo;
        o.band_hi = band_hi;
        o.n_lag = n_lag;
        o.n0 = n0;
        o.n_ref_start = n_ref_start;
        o.adaptive_ref = adaptive_ref ? 1 : 0;
        o.use_explicit_inverse = explicit_inverse ? 1 : 0;
        o.adapt_beta = no_adapt_beta ? 0 : 1;
        o.chains = chains;
        o.intervals_per_batch = intervals;
        o.max_batches = max_batches;
        o.max_samples = max_samples;
        o.max_wall_seconds = max_wall;
        o.master_seed = seed;
        o.init_dispersion = dispersion;
        o.threads = threads;
    }
};

bool parse(int argc, char** argv, Options& o) {
    auto num = [&](int& i, auto& dst) {
        if (i + 1 >= argc) return false;
        const char* v = argv[++i];
        char* end = nullptr;
        if constexpr (std::is_floating_point_v<std::remove_reference_t<decltype(dst)>>) dst = std::strtod(v, &end);
        else dst = static_cast<std::remove_reference_t<decltype(dst)>>(std::strtoll(v, &end, 10));
        return end && *end == '\0';
    };
    auto list = [&](int& i, std::vector<int64_t>& dst) {
        bool any = false;
        while (i + 1 < argc && argv[i + 1][0] != '-') {
            dst.push_back(std::strtoll(argv[++i], nullptr, 10));
            any = true;
        }
        return any;
    };
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        bool ok = true;
        if (a == "benchmark" && i == 1) continue;
        else if (a == "--target" && i + 1 < argc) o.target = argv[++i];
        else if (a == "--kernel" && i + 1 < argc) {
            o.kernel = argv[++i];
            ok = o.kernel == "rw" || o.kernel == "pcn" || o.kernel == "am" || o.kernel == "diam";
        } else if (a == "--out" && i + 1 < argc) o.out = argv[++i];
        else if (a == "--dim") ok = num(i, o.dim);
        else if (a == "--target-seed") ok = num(i, o.target_seed);
        else if (a == "--sigma2") ok = num(i, o.sigma2);
        else if (a == "--twist-b") ok = num(i, o.twist_b);
        else if (a == "--beta") ok = num(i, o.beta);
        else if (a == "--inflation") ok = num(i, o.inflation);
        else if (a == "--band-lo") ok = num(i, o.band_lo);
        else if (a == "--band-hi") ok = num(i, o.band_hi);
        else if (a == "--n-lag") ok = num(i, o.n_lag);
        else if (a == "--n0") ok = num(i, o.n0);
        else if (a == "--n-ref-start") ok = num(i, o.n_ref_start);
        else if (a == "--adaptive-ref") o.adaptive_ref = true;
        else if (a == "--explicit-inverse") o.explicit_inverse = true;
        else if (a == "--no-adapt-beta") o.no_adapt_beta = true;
        else if (a == "--chains") ok = num(i, o.chains);
        else if (a == "--intervals") ok = num(i, o.intervals);
        else if (a == "--max-batches") ok = num(i, o.max_batches);
        else if (a == "--max-samples") ok = num(i, o.max_samples);
        else if (a == "--max-wall") ok = num(i, o.max_wall);
        else if (a == "--seed") ok = num(i, o.seed);
        else if (a == "--dispersion") ok = num(i, o.dispersion);
        else if (a == "--threads") ok = num(i, o.threads);
        else if (a == "--samples") ok = num(i, o.samples);
        else if (a == "--dims") ok = list(i, o.dims);
        else if (a == "--chain-sweep") ok = list(i, o.chain_sweep);
        else ok = false;
        if (!ok) {
            std::fprintf(stderr, "error: bad option '%s'\n", a.c_str());
            return false;
        }
    }
    return true;
}

int benchmark(const Options& base) {  // proj/tools/diam_cli.cpp:427-505
    if (base.dims.empty() && base.chain_sweep.empty()) {
        std::fprintf(stderr, "error: benchmark needs --dims or --chain-sweep\n");
        return kExitConfig;
    }
    std::ofstream out(base.out);
    if (!out.good()) {
        std::fprintf(stderr, "error: cannot open %s\n", base.out.c_str());
        return kExitRuntime;
    }
    if (!base.dims.empty()) {
        out << "d,total_samples,wall_seconds,sec_per_sample,sec_per_batch\n";
        std::vector<double> xs, ys;
        for (int64_t d : base.dims) {
            Target target;
            if (int rc = base.build(d, target); rc != kExitOk) return rc;
            diam_run_options o;
            base.fill(o);
            o.record_traces = 0;
            o.checkpoint_path = nullptr;
            o.cov_tol = o.mean_tol = o.psrf_tol = -1.0;
            const int64_t n_lag = o.n_lag > 0 ? o.n_lag : std::max<int64_t>(1, d / 2);
            const int64_t per_batch = o.chains * o.intervals_per_batch * n_lag;
            o.max_batches = std::max<int64_t>(1, (base.samples + per_batch - 1) / per_batch);
            o.max_samples = -1;
            o.n0 = o.n0 >= 0 ? o.n0 : 0;
            Result res;
            if (diam_status st = diam_sample(target.t, &o, &res.r); st != DIAM_OK)
                return report_failure("benchmark run", st);
            const double wall = diam_result_wall_seconds(res.r);
            const auto total = static_cast<double>(diam_result_total_samples(res.r));
            const auto batches = static_cast<double>(diam_result_batches(res.r));
            out << d << ',' << static_cast<uint64_t>(total) << ',' << fmt(wall) << ',' << fmt(wall / total) << ','
                << fmt(wall / batches) << '\n';
            xs.push_back(static_cast<double>(d));
            ys.push_back(wall / total);
        }
        if (xs.size() >= 3) {
            double coeffs[3], share = 0.0, rss = 0.0;
            if (diam_status st = diam_fit_quadratic(xs.data(), ys.data(), static_cast<int64_t>(xs.size()), coeffs,
                                                    &share, &rss);
                st != DIAM_OK)
                return report_failure("fitting scaling curve", st);
            std::printf("per-sample seconds fit: T = %.6g + %.6g*d + %.6g*d^2\n", coeffs[0], coeffs[1], coeffs[2]);
            std::printf("quadratic variance share = %.3f, rss = %.6g\n", share, rss);
        }
    }
    if (!base.chain_sweep.empty()) {
        out << "P,total_seconds,sec_per_batch,N\n";
        for (int64_t p : base.chain_sweep) {
            Target target;
            if (int rc = base.build(base.dim, target); rc != kExitOk) return rc;
            diam_run_options o;
            base.fill(o);
            o.record_traces = 0;
            o.checkpoint_path = nullptr;
            o.chains = p;
            Result res;
            if (diam_status st = diam_sample(target.t, &o, &res.r); st != DIAM_OK)
                return report_failure("benchmark run", st);
            const double wall = diam_result_wall_seconds(res.r);
            const auto batches = static_cast<double>(diam_result_batches(res.r));
            out << p << ',' << fmt(wall) << ',' << fmt(batches > 0 ? wall / batches : 0.0) << ','
                << diam_result_total_samples(res.r) << '\n';
        }
    }
    std::printf("benchmark table written to %s\n", base.out.c_str());
    return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
    Options o;
    if (!parse(argc, argv, o)) return kExitConfig;
    return benchmark(o);
}
