/*
 * diam_oracle — CPU restatement of the reference DIAM sampler hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This library is the checker for the B200 path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it. The product (paper_1506_05741_b200/libdiam.so) never links it.
 *
 * Every function restates one reference function with the same arithmetic
 * order (so that, compiled with the reference's flags, results are
 * bit-identical to the reference; tests/test_oracle.py pins that against
 * oracle/_ref and the reference's golden vectors). The cited lines are in
 * /root/reference/proj/.
 *
 * Layout conventions follow the reference: row-major doubles, lower
 * triangular factors stored as full d×d squares with a zero upper part.
 */
#ifndef DIAM_ORACLE_H
#define DIAM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror diam_status (include/diam/diam.h) */
enum { OR_OK = 0, OR_INVALID_ARGUMENT = 1, OR_DIMENSION_MISMATCH = 3,
       OR_NOT_POSITIVE_DEFINITE = 4, OR_SINGULAR_DIAGONAL = 5,
       OR_ZERO_WITHIN_VARIANCE = 8, OR_UNEQUAL_BATCH_SIZES = 9 };

/* ---- Philox4x32-10 streams: src/rng.cpp:38-94 ---------------------------- */
typedef struct or_stream {
    uint32_t key[2];
    uint32_t stream[2];
    uint64_t counter;
} or_stream;

void or_stream_init(or_stream* s, uint64_t master_seed, uint64_t stream_index, const char* purpose);
void or_block(or_stream* s, uint32_t out[4]);
uint64_t or_next_u64(or_stream* s);
double or_uniform(or_stream* s);
double or_uniform_open(or_stream* s);
double or_normal(or_stream* s);
/* n consecutive draws starting at draw counter `start` */
void or_fill_u64(uint64_t seed, uint64_t idx, const char* purpose, uint64_t start, size_t n, uint64_t* out);
void or_fill_uniform_open(uint64_t seed, uint64_t idx, const char* purpose, uint64_t start, size_t n, double* out);
void or_fill_normal(uint64_t seed, uint64_t idx, const char* purpose, uint64_t start, size_t n, double* out);

/* ---- dense kernels: src/linalg.cpp ---------------------------------------- */
double or_lane_dot(const double* a, const double* b, size_t n);
void or_sym_matvec(const double* m, size_t n, const double* v, double* y);
void or_matvec(const double* m, size_t rows, size_t cols, const double* v, double* y);
void or_tri_matvec(const double* l, size_t n, const double* v, double* y);
int or_tri_solve(const double* l, size_t n, const double* v, double* y);
int or_cholesky(const double* m, size_t n, double* l);
int or_jittered_cholesky(const double* cov, size_t n, double* l);

/* ---- targets: src/target.cpp:154-173 --------------------------------------- */
typedef struct or_target {
    size_t dim;
    int twisted;             /* pi5 / pi6 */
    const double* precision; /* d×d, Gaussian kinds */
    const double* eigvecs_t; /* d×d, Vᵀ row-major (twisted kinds) */
    const double* eigvals;   /* d */
    const double* b_coeffs;  /* d */
    const double* proj_min;  /* d: eigvecs column 0 (trace functional) */
    const double* proj_max;  /* d: eigvecs column d-1 */
    const double* covariance;/* d×d analytic */
    const double* mean;      /* d analytic */
} or_target;

double or_log_density(const or_target* t, const double* x);

/* ---- moments: src/moments.cpp ---------------------------------------------- */
typedef struct or_moments {
    size_t dim;
    uint64_t count;
    double* mean;   /* d */
    double* second; /* d×d */
} or_moments;

void or_accumulate(or_moments* acc, const double* x);
/* blend local with global; writes mean (d), second (d×d), cov (d×d); returns count */
uint64_t or_blend(const or_moments* local, const or_moments* global, double* mean, double* second,
                  double* cov);
void or_covariance(const double* second, const double* mean, size_t d, double* cov);
int or_merge_batch(or_moments* global, uint64_t* global_batches, const or_moments* locals, size_t p);
void or_merge_into(or_moments* into, const or_moments* from);

/* ---- diagnostics: src/diagnostics.cpp:72-142 ------------------------------- */
int or_psrf_max(const or_moments* chains, size_t p, double* out_max);
double or_cov_error(const double* emp, const double* truth, size_t d);
double or_mean_error(const double* emp, const double* truth, size_t d);

/* ---- kernel configuration: src/proposal.cpp:24-45 -------------------------- */
enum { OR_RW = 0, OR_PCN = 1, OR_AM = 2, OR_DIAM = 3 };
typedef struct or_kernel_cfg {
    int kind;
    size_t dim;
    double beta_init, inflation;
    int adaptive_ref;  /* RefMode::AdaptiveMean, else Zero */
    size_t n_lag;
    double band_lo, band_hi;
    uint64_t n0, n_ref_start;
    double beta_adapt_factor, beta_min, beta_max;
    int adapt_beta;
    int use_explicit_inverse;
} or_kernel_cfg;

void or_kernel_defaults(or_kernel_cfg* c, int kind, size_t dim);

/* ---- one chain: src/proposal.cpp:87-266 ------------------------------------ */
typedef struct or_chain {
    size_t dim, n_lag;
    double* x;
    double log_pi, quad, beta;
    uint64_t n, n_accepted;
    double* factor;      /* d×d lower */
    double* factor_inv;  /* d×d lower or NULL */
    double* x_ref;
    double* noise;       /* n_lag×d pre-scaled increments */
    size_t noise_pos;
    uint64_t noise_ctr_at_batch;
    or_moments batch_acc, cum_acc;
    or_stream noise_rng, uniform_rng;
} or_chain;

/* Draw provider: when `inject_w` is non-NULL the next window's standard normals
 * are taken from it (n_lag×d, row-major) instead of the noise stream, and the
 * stream counter is advanced by n_lag·d exactly as if they had been drawn.
 * This is how the GPU path and the oracle are run on identical draws. */
int or_chain_init(or_chain* c, const or_kernel_cfg* cfg, const or_target* t, const double* x0,
                  uint64_t seed, uint64_t chain_index, const double* inject_w);
void or_chain_free(or_chain* c);
double or_quad_term(const or_kernel_cfg* cfg, const or_chain* c, const double* z);
/* one MH transition (src/proposal.cpp:137-157); u taken from the chain's uniform stream
 * unless `u_override` >= 0. Returns 1 if accepted, negative on error. *log_ratio_out
 * receives log alpha. */
int or_mh_step(const or_kernel_cfg* cfg, const or_target* t, or_chain* c, double u_override,
               double* log_ratio_out);
/* src/proposal.cpp:159-216. `global` is the frozen batch snapshot. */
int or_lag_update(const or_kernel_cfg* cfg, or_chain* c, const or_moments* global,
                  const double* inject_w, double* rate_out);
void or_regenerate_noise(const or_kernel_cfg* cfg, or_chain* c, const double* inject_w);

/* ---- engine: src/runner.cpp:122-279 (single thread; the reference is thread-count
 * invariant, tests/test_runner.cpp:92-108) --------------------------------- */
typedef struct or_run_cfg {
    or_kernel_cfg kernel;
    size_t chains, intervals_per_batch, max_batches;
    double cov_tol, mean_tol, psrf_tol; /* <= 0: disabled */
    int64_t max_samples;                /* < 0: disabled */
    double init_dispersion;
    uint64_t master_seed;
    int record_traces;
    size_t trace_thin;
    int trace_eigen_projections;
} or_run_cfg;

typedef struct or_run_out {
    size_t batches;
    uint64_t total_samples, accumulated_samples;
    int stop_reason; /* 0 batch_cap 1 max_samples 2 psrf 3 cov_tol 4 mean_tol */
    double* global_mean;      /* d  (caller-allocated) */
    double* global_cov;       /* d×d (caller-allocated) */
    double* cov_error_hist;   /* max_batches (caller-allocated) */
    double* mean_error_hist;
    double* psrf_hist;
    double* beta_hist;        /* chains × (max_batches·M) */
    double* acc_hist;         /* chains × (max_batches·M) */
    double* accept_bits;      /* optional: chains × total steps (1/0) or NULL */
    double* log_ratio;        /* optional: chains × total steps or NULL */
    double* log_u;            /* optional: chains × total steps or NULL */
    double* final_x;          /* optional: chains × d or NULL */
    /* optional traces (src/runner.cpp:363-379): chains × 3 × trace_cap, functional f of
     * chain p at traces[(p·3 + f)·trace_cap + i]; trace_len = entries per chain */
    double* traces;
    size_t trace_cap, trace_len;
} or_run_out;

/* Run options beyond the reference's: `threads` workers run the chains of a batch
 * concurrently (chains are independent within a batch; results do not depend on it);
 * `chain_ids` (n_ids > 0) runs only those global chain indices, their RNG streams keyed
 * by the global index -- valid for per-chain quantities of the FIRST batch only (the
 * merge pools just the listed chains). Per-chain outputs are indexed by position in
 * chain_ids. */
typedef struct or_run_opts {
    int threads;
    const size_t* chain_ids;
    size_t n_ids;
} or_run_opts;
int or_run_ex(const or_run_cfg* cfg, const or_target* t, const double* const* inject_w, or_run_out* out,
              const or_run_opts* opts);

/* Full run. `inject_w`, when non-NULL, supplies every window's normals:
 * inject_w[p] points at chain p's stream of windows, each n_lag×d, in the order
 * the chain consumes them (init window first). */
int or_run(const or_run_cfg* cfg, const or_target* t, const double* const* inject_w,
           or_run_out* out);

const char* or_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
