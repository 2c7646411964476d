/*
 * diam_oracle.c — CPU restatement of the reference DIAM hot path.
 *
 * TEST INFRASTRUCTURE (the checker, never the thing measured or shipped).
 * See diam_oracle.h. Each function cites the reference lines it restates
 * (paths relative to /root/reference/proj/). Summation orders are kept
 * identical to the reference so that the restatement is bit-identical to
 * it when built with the reference's flags (-O3, no -march, no fast-math);
 * tests/test_oracle.py checks this against oracle/_ref.
 */
#include "diam_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];
const char* or_last_error(void) { return g_err; }
static int fail_with(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 + key/stream derivation: src/rng.cpp:9-49, 51-70            */
/* ------------------------------------------------------------------------- */
static uint64_t splitmix64(uint64_t* state) { /* src/rng.cpp:14-19 */
    uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static uint64_t fnv1a64(const char* s) { /* src/rng.cpp:21-28 */
    uint64_t h = 0xcbf29ce484222325ull;
    for (; *s; ++s) {
        h ^= (unsigned char)*s;
        h *= 0x100000001b3ull;
    }
    return h;
}

void or_stream_init(or_stream* st, uint64_t master_seed, uint64_t stream_index,
                    const char* purpose) { /* src/rng.cpp:38-49 */
    uint64_t s = master_seed;
    const uint64_t k = splitmix64(&s);
    st->key[0] = (uint32_t)k;
    st->key[1] = (uint32_t)(k >> 32);
    uint64_t id = splitmix64(&s) ^ (stream_index * 0xA24BAED4963EE407ull) ^ fnv1a64(purpose);
    const uint64_t sid = splitmix64(&id);
    st->stream[0] = (uint32_t)sid;
    st->stream[1] = (uint32_t)(sid >> 32);
    st->counter = 0;
}

void or_block(or_stream* st, uint32_t out[4]) { /* src/rng.cpp:51-70 */
    uint32_t c0 = (uint32_t)st->counter, c1 = (uint32_t)(st->counter >> 32);
    uint32_t c2 = st->stream[0], c3 = st->stream[1];
    uint32_t k0 = st->key[0], k1 = st->key[1];
    st->counter++;
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

uint64_t or_next_u64(or_stream* st) { /* src/rng.cpp:72-75 */
    uint32_t b[4];
    or_block(st, b);
    return ((uint64_t)b[1] << 32) | b[0];
}

double or_uniform(or_stream* st) { /* src/rng.cpp:77-79 */
    return (double)(or_next_u64(st) >> 11) * 0x1.0p-53;
}

double or_uniform_open(or_stream* st) { /* src/rng.cpp:81-83 */
    return ((double)(or_next_u64(st) >> 11) + 0.5) * 0x1.0p-53;
}

double or_normal(or_stream* st) { /* src/rng.cpp:85-94 */
    uint32_t b[4];
    or_block(st, b);
    const uint64_t w0 = ((uint64_t)b[1] << 32) | b[0];
    const uint64_t w1 = ((uint64_t)b[3] << 32) | b[2];
    const double u1 = ((double)(w0 >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = (double)(w1 >> 11) * 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u1));
    return r * cos(6.283185307179586476925286766559 * u2);
}

void or_fill_u64(uint64_t seed, uint64_t idx, const char* purpose, uint64_t start, size_t n,
                 uint64_t* out) {
    or_stream s;
    or_stream_init(&s, seed, idx, purpose);
    s.counter = start;
    for (size_t i = 0; i < n; ++i) out[i] = or_next_u64(&s);
}

void or_fill_uniform_open(uint64_t seed, uint64_t idx, const char* purpose, uint64_t start,
                          size_t n, double* out) {
    or_stream s;
    or_stream_init(&s, seed, idx, purpose);
    s.counter = start;
    for (size_t i = 0; i < n; ++i) out[i] = or_uniform_open(&s);
}

void or_fill_normal(uint64_t seed, uint64_t idx, const char* purpose, uint64_t start, size_t n,
                    double* out) {
    or_stream s;
    or_stream_init(&s, seed, idx, purpose);
    s.counter = start;
    for (size_t i = 0; i < n; ++i) out[i] = or_normal(&s);
}

/* ------------------------------------------------------------------------- */
/* dense kernels: src/linalg.cpp                                              */
/* ------------------------------------------------------------------------- */
double or_lane_dot(const double* a, const double* b, size_t n) { /* src/linalg.cpp:43-54 */
    double l0 = 0.0, l1 = 0.0, l2 = 0.0, l3 = 0.0;
    size_t j = 0;
    for (; j + 4 <= n; j += 4) {
        l0 += a[j] * b[j];
        l1 += a[j + 1] * b[j + 1];
        l2 += a[j + 2] * b[j + 2];
        l3 += a[j + 3] * b[j + 3];
    }
    for (; j < n; ++j) l0 += a[j] * b[j];
    return ((l0 + l1) + l2) + l3;
}

void or_sym_matvec(const double* m, size_t n, const double* v, double* y) { /* :117-124 */
    for (size_t i = 0; i < n; ++i) y[i] = or_lane_dot(m + i * n, v, n);
}

void or_matvec(const double* m, size_t rows, size_t cols, const double* v, double* y) { /* :126-131 */
    for (size_t i = 0; i < rows; ++i) y[i] = or_lane_dot(m + i * cols, v, cols);
}

void or_tri_matvec(const double* l, size_t n, const double* v, double* y) { /* :133-139 */
    for (size_t i = 0; i < n; ++i) y[i] = or_lane_dot(l + i * n, v, i + 1);
}

int or_tri_solve(const double* l, size_t n, const double* v, double* y) { /* :141-151 */
    for (size_t i = 0; i < n; ++i) y[i] = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double* row = l + i * n;
        if (row[i] == 0.0) return fail_with(OR_SINGULAR_DIAGONAL, "tri_solve: zero diagonal");
        y[i] = (v[i] - or_lane_dot(row, y, i)) / row[i];
    }
    return OR_OK;
}

int or_cholesky(const double* m, size_t n, double* l) { /* :62-93 (symmetry check + column loop) */
    double scale = 0.0;
    for (size_t i = 0; i < n * n; ++i) scale = fmax(scale, fabs(m[i]));
    const double tol = 1e-12 * fmax(scale, 1.0);
    for (size_t i = 0; i < n; ++i)
        for (size_t j = i + 1; j < n; ++j)
            if (!(fabs(m[i * n + j] - m[j * n + i]) <= tol))
                return fail_with(OR_INVALID_ARGUMENT, "cholesky: matrix not symmetric");
    memset(l, 0, sizeof(double) * n * n);
    for (size_t j = 0; j < n; ++j) {
        double sum_sq = 0.0;
        for (size_t k = 0; k < j; ++k) sum_sq += l[j * n + k] * l[j * n + k];
        const double pivot = m[j * n + j] - sum_sq;
        if (pivot <= 0.0 || !isfinite(pivot))
            return fail_with(OR_NOT_POSITIVE_DEFINITE, "cholesky: non-positive pivot");
        l[j * n + j] = sqrt(pivot);
        for (size_t i = j + 1; i < n; ++i) {
            double sum = 0.0;
            for (size_t k = 0; k < j; ++k) sum += l[i * n + k] * l[j * n + k];
            l[i * n + j] = (m[i * n + j] - sum) / l[j * n + j];
        }
    }
    return OR_OK;
}

int or_jittered_cholesky(const double* cov, size_t n, double* l) { /* src/proposal.cpp:218-239 */
    int st = or_cholesky(cov, n, l);
    if (st != OR_NOT_POSITIVE_DEFINITE) return st;
    double trace = 0.0;
    for (size_t i = 0; i < n; ++i) trace += cov[i * n + i];
    const double scale = trace / (double)n;
    double* padded = (double*)malloc(sizeof(double) * n * n);
    for (double eps = 1e-10; eps <= 1e-4; eps *= 100.0) {
        memcpy(padded, cov, sizeof(double) * n * n);
        for (size_t i = 0; i < n; ++i) padded[i * n + i] += eps * scale;
        st = or_cholesky(padded, n, l);
        if (st != OR_NOT_POSITIVE_DEFINITE) {
            free(padded);
            return st;
        }
    }
    free(padded);
    return fail_with(OR_NOT_POSITIVE_DEFINITE, "covariance not factorizable after jitter escalation");
}

/* ------------------------------------------------------------------------- */
/* targets: src/target.cpp:154-173                                            */
/* ------------------------------------------------------------------------- */
double or_log_density(const or_target* t, const double* x) {
    const size_t d = t->dim;
    double* tmp = (double*)malloc(sizeof(double) * d);
    double out;
    if (!t->twisted) {
        or_sym_matvec(t->precision, d, x, tmp);
        out = -0.5 * or_lane_dot(x, tmp, d);
    } else {
        or_matvec(t->eigvecs_t, d, d, x, tmp); /* z = Vᵀx */
        /* twist_map: w_{i+1} += b_i z_i², i even (0-based), b_i != 0 */
        double s = 0.0;
        for (size_t i = 0; i < d; ++i) {
            double w = tmp[i];
            if (i % 2 == 1 && t->b_coeffs[i - 1] != 0.0) w += t->b_coeffs[i - 1] * tmp[i - 1] * tmp[i - 1];
            s += w * w / t->eigvals[i];
        }
        out = -0.5 * s;
    }
    free(tmp);
    return out;
}

/* ------------------------------------------------------------------------- */
/* moments: src/moments.cpp                                                   */
/* ------------------------------------------------------------------------- */
static void moments_alloc(or_moments* m, size_t d) {
    m->dim = d;
    m->count = 0;
    m->mean = (double*)calloc(d, sizeof(double));
    m->second = (double*)calloc(d * d, sizeof(double));
}
static void moments_free(or_moments* m) {
    free(m->mean);
    free(m->second);
    m->mean = m->second = NULL;
}
static void moments_reset(or_moments* m) {
    m->count = 0;
    memset(m->mean, 0, sizeof(double) * m->dim);
    memset(m->second, 0, sizeof(double) * m->dim * m->dim);
}

void or_accumulate(or_moments* acc, const double* x) { /* src/moments.cpp:5-20 */
    const size_t d = acc->dim;
    const double n = (double)acc->count;
    const double keep = n / (n + 1.0);
    const double add = 1.0 / (n + 1.0);
    for (size_t i = 0; i < d; ++i) acc->mean[i] = acc->mean[i] * keep + x[i] * add;
    for (size_t i = 0; i < d; ++i) {
        const double xi = x[i] * add;
        for (size_t j = 0; j <= i; ++j) {
            const double v = acc->second[i * d + j] * keep + xi * x[j];
            acc->second[i * d + j] = v;
            acc->second[j * d + i] = v;
        }
    }
    acc->count++;
}

void or_covariance(const double* second, const double* mean, size_t d, double* cov) { /* :90-101 */
    for (size_t i = 0; i < d; ++i)
        for (size_t j = 0; j <= i; ++j) {
            const double v = 0.5 * (second[i * d + j] + second[j * d + i]) - mean[i] * mean[j];
            cov[i * d + j] = v;
            cov[j * d + i] = v;
        }
}

uint64_t or_blend(const or_moments* local, const or_moments* global, double* mean, double* second,
                  double* cov) { /* src/moments.cpp:28-49 */
    const size_t d = local->dim;
    const uint64_t count = local->count + global->count;
    if (count == 0) {
        memcpy(mean, local->mean, sizeof(double) * d);
        memcpy(second, local->second, sizeof(double) * d * d);
        or_covariance(second, mean, d, cov);
        return 0;
    }
    const double total = (double)count;
    const double wg = (double)global->count / total;
    const double wl = (double)local->count / total;
    for (size_t i = 0; i < d; ++i) mean[i] = wg * global->mean[i] + wl * local->mean[i];
    for (size_t i = 0; i < d * d; ++i) second[i] = wg * global->second[i] + wl * local->second[i];
    or_covariance(second, mean, d, cov);
    return count;
}

int or_merge_batch(or_moments* global, uint64_t* global_batches, const or_moments* locals,
                   size_t p) { /* src/moments.cpp:51-75 */
    if (p == 0) return fail_with(OR_INVALID_ARGUMENT, "merge_batch: no chains");
    const uint64_t per_chain = locals[0].count;
    for (size_t c = 0; c < p; ++c)
        if (locals[c].count != per_chain)
            return fail_with(OR_UNEQUAL_BATCH_SIZES, "merge_batch: unequal counts");
    (*global_batches)++;
    const uint64_t incoming = per_chain * p;
    if (incoming == 0) return OR_OK;
    const double total = (double)(global->count + incoming);
    const double keep = (double)global->count / total;
    const double wp = (double)per_chain / total;
    const size_t d = global->dim;
    for (size_t i = 0; i < d; ++i) global->mean[i] *= keep;
    for (size_t i = 0; i < d * d; ++i) global->second[i] *= keep;
    for (size_t c = 0; c < p; ++c) {
        for (size_t i = 0; i < d; ++i) global->mean[i] += wp * locals[c].mean[i];
        for (size_t i = 0; i < d * d; ++i) global->second[i] += wp * locals[c].second[i];
    }
    global->count += incoming;
    return OR_OK;
}

void or_merge_into(or_moments* into, const or_moments* from) { /* src/moments.cpp:77-88 */
    if (from->count == 0) return;
    const size_t d = into->dim;
    const double total = (double)(into->count + from->count);
    const double keep = (double)into->count / total;
    const double add = (double)from->count / total;
    for (size_t i = 0; i < d; ++i) into->mean[i] = keep * into->mean[i] + add * from->mean[i];
    for (size_t i = 0; i < d * d; ++i) into->second[i] = keep * into->second[i] + add * from->second[i];
    into->count += from->count;
}

/* ------------------------------------------------------------------------- */
/* diagnostics: src/diagnostics.cpp:72-142                                    */
/* ------------------------------------------------------------------------- */
int or_psrf_max(const or_moments* chains, size_t p, double* out_max) {
    if (p < 2) return fail_with(OR_INVALID_ARGUMENT, "psrf needs at least 2 chains");
    const size_t d = chains[0].dim;
    const uint64_t nsc = chains[0].count;
    for (size_t c = 0; c < p; ++c)
        if (chains[c].count != nsc) return fail_with(OR_UNEQUAL_BATCH_SIZES, "psrf: unequal counts");
    if (nsc < 2) return fail_with(OR_INVALID_ARGUMENT, "psrf needs at least 2 samples per chain");
    double* gmean = (double*)calloc(d, sizeof(double));
    const double inv_p = 1.0 / (double)p;
    for (size_t c = 0; c < p; ++c) /* make_psrf_input :90-91 */
        for (size_t i = 0; i < d; ++i) gmean[i] += inv_p * chains[c].mean[i];
    const double n = (double)nsc;
    const double pd = (double)p;
    double mx = 0.0;
    for (size_t i = 0; i < d; ++i) { /* psrf :104-117 */
        double between = 0.0, within = 0.0;
        for (size_t c = 0; c < p; ++c) {
            const double delta = chains[c].mean[i] - gmean[i];
            between += delta * delta;
            within += chains[c].second[i * d + i] - chains[c].mean[i] * chains[c].mean[i];
        }
        const double b_i = n / (pd - 1.0) * between;
        const double w_i = n / ((n - 1.0) * pd) * within;
        if (!(w_i > 0.0)) {
            free(gmean);
            return fail_with(OR_ZERO_WITHIN_VARIANCE, "psrf: zero within-chain variance");
        }
        const double r = (n - 1.0) / n + (pd + 1.0) / (pd * n) * b_i / w_i;
        mx = fmax(mx, sqrt(r)); /* runner.cpp:387-389 */
    }
    free(gmean);
    *out_max = mx;
    return OR_OK;
}

double or_cov_error(const double* emp, const double* truth, size_t d) { /* :121-132 */
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < d * d; ++i) {
        const double diff = emp[i] - truth[i];
        num += diff * diff;
        den += truth[i] * truth[i];
    }
    return sqrt(num / den);
}

double or_mean_error(const double* emp, const double* truth, size_t d) { /* :134-142 */
    double s = 0.0;
    for (size_t i = 0; i < d; ++i) {
        const double diff = emp[i] - truth[i];
        s += diff * diff;
    }
    return sqrt(s);
}

/* ------------------------------------------------------------------------- */
/* proposals: src/proposal.cpp                                                */
/* ------------------------------------------------------------------------- */
static int pcn_form(int kind) { return kind == OR_PCN || kind == OR_DIAM; }
static int adapts_cov(int kind) { return kind == OR_AM || kind == OR_DIAM; }
static double noise_infl(const or_kernel_cfg* c) { return c->kind == OR_DIAM ? c->inflation : 1.0; }

void or_kernel_defaults(or_kernel_cfg* c, int kind, size_t dim) { /* src/proposal.cpp:24-45 */
    memset(c, 0, sizeof *c);
    c->kind = kind;
    c->dim = dim;
    c->beta_init = fmin(2.4 / sqrt((double)dim), 0.5);
    c->inflation = 1.0;
    c->n_lag = dim / 2 > 1 ? dim / 2 : 1;
    if (pcn_form(kind)) {
        c->band_lo = 0.3;
        c->band_hi = 0.5;
        c->beta_max = 1.0;
    } else {
        c->band_lo = 0.1;
        c->band_hi = 0.3;
        c->beta_max = 10.0;
    }
    c->n0 = 25 * (uint64_t)dim;
    c->n_ref_start = 10 * (uint64_t)dim;
    c->beta_adapt_factor = 1.1;
    c->beta_min = 1e-6;
    c->adapt_beta = 1;
}

static void invert_lower(const double* l, size_t n, double* inv) { /* :241-252 */
    double* e = (double*)calloc(n, sizeof(double));
    double* col = (double*)malloc(sizeof(double) * n);
    memset(inv, 0, sizeof(double) * n * n);
    for (size_t j = 0; j < n; ++j) {
        e[j] = 1.0;
        or_tri_solve(l, n, e, col);
        for (size_t i = j; i < n; ++i) inv[i * n + j] = col[i];
        e[j] = 0.0;
    }
    free(e);
    free(col);
}

double or_quad_term(const or_kernel_cfg* cfg, const or_chain* c, const double* z) { /* :51-61 */
    const size_t d = cfg->dim;
    double* centered = (double*)malloc(sizeof(double) * d);
    double* y = (double*)malloc(sizeof(double) * d);
    for (size_t i = 0; i < d; ++i) centered[i] = z[i] - c->x_ref[i];
    if (c->factor_inv)
        or_tri_matvec(c->factor_inv, d, centered, y);
    else
        or_tri_solve(c->factor, d, centered, y);
    double s = 0.0;
    for (size_t i = 0; i < d; ++i) s += y[i] * y[i];
    const double infl = noise_infl(cfg);
    free(centered);
    free(y);
    return 0.5 * s / (infl * infl);
}

void or_regenerate_noise(const or_kernel_cfg* cfg, or_chain* c, const double* inject_w) { /* :254-266 */
    const size_t d = cfg->dim;
    const double scale = c->beta * noise_infl(cfg);
    double* w = (double*)malloc(sizeof(double) * d);
    double* xi = (double*)malloc(sizeof(double) * d);
    for (size_t r = 0; r < cfg->n_lag; ++r) {
        if (inject_w) {
            memcpy(w, inject_w + r * d, sizeof(double) * d);
            c->noise_rng.counter += d;
        } else {
            for (size_t i = 0; i < d; ++i) w[i] = or_normal(&c->noise_rng);
        }
        or_tri_matvec(c->factor, d, w, xi);
        for (size_t i = 0; i < d; ++i) c->noise[r * d + i] = scale * xi[i];
    }
    c->noise_pos = 0;
    free(w);
    free(xi);
}

int or_chain_init(or_chain* c, const or_kernel_cfg* cfg, const or_target* t, const double* x0,
                  uint64_t seed, uint64_t chain_index, const double* inject_w) { /* :87-113 */
    const size_t d = cfg->dim;
    memset(c, 0, sizeof *c);
    c->dim = d;
    c->n_lag = cfg->n_lag;
    c->x = (double*)malloc(sizeof(double) * d);
    memcpy(c->x, x0, sizeof(double) * d);
    c->beta = cfg->beta_init;
    c->factor = (double*)calloc(d * d, sizeof(double));
    for (size_t i = 0; i < d; ++i) c->factor[i * d + i] = 1.0;
    if (cfg->use_explicit_inverse) {
        c->factor_inv = (double*)malloc(sizeof(double) * d * d);
        invert_lower(c->factor, d, c->factor_inv);
    }
    c->x_ref = (double*)calloc(d, sizeof(double));
    c->noise = (double*)malloc(sizeof(double) * cfg->n_lag * d);
    or_stream_init(&c->noise_rng, seed, chain_index, "noise");
    or_stream_init(&c->uniform_rng, seed, chain_index, "uniform");
    c->log_pi = or_log_density(t, c->x);
    c->quad = pcn_form(cfg->kind) ? or_quad_term(cfg, c, c->x) : 0.0;
    moments_alloc(&c->batch_acc, d);
    moments_alloc(&c->cum_acc, d);
    c->noise_ctr_at_batch = c->noise_rng.counter;
    or_regenerate_noise(cfg, c, inject_w);
    return OR_OK;
}

void or_chain_free(or_chain* c) {
    free(c->x);
    free(c->factor);
    free(c->factor_inv);
    free(c->x_ref);
    free(c->noise);
    moments_free(&c->batch_acc);
    moments_free(&c->cum_acc);
    memset(c, 0, sizeof *c);
}

int or_mh_step(const or_kernel_cfg* cfg, const or_target* t, or_chain* c, double u_override,
               double* log_ratio_out) { /* :137-157 with evaluate :70-83, propose :115-127 */
    const size_t d = cfg->dim;
    if (c->noise_pos >= cfg->n_lag)
        return -fail_with(OR_INVALID_ARGUMENT, "mh_step: noise batch exhausted");
    const double* xi = c->noise + c->noise_pos * d;
    c->noise_pos++;
    double* cand = (double*)malloc(sizeof(double) * d);
    if (pcn_form(cfg->kind)) {
        const double contract = sqrt(fmax(0.0, 1.0 - c->beta * c->beta));
        for (size_t i = 0; i < d; ++i) cand[i] = c->x_ref[i] + contract * (c->x[i] - c->x_ref[i]) + xi[i];
    } else {
        for (size_t i = 0; i < d; ++i) cand[i] = c->x[i] + xi[i];
    }
    const double lp = or_log_density(t, cand);
    double q = 0.0, ratio;
    if (pcn_form(cfg->kind)) {
        q = or_quad_term(cfg, c, cand);
        ratio = (lp + q) - (c->log_pi + c->quad);
    } else {
        ratio = lp - c->log_pi;
    }
    const double u = u_override >= 0.0 ? u_override : or_uniform_open(&c->uniform_rng);
    const int accepted = log(u) < ratio;
    if (accepted) {
        memcpy(c->x, cand, sizeof(double) * d);
        c->log_pi = lp;
        c->quad = q;
        c->n_accepted++;
    }
    c->n++;
    if (c->n > cfg->n0) or_accumulate(&c->batch_acc, c->x);
    free(cand);
    if (log_ratio_out) *log_ratio_out = ratio;
    return accepted;
}

int or_lag_update(const or_kernel_cfg* cfg, or_chain* c, const or_moments* global,
                  const double* inject_w, double* rate_out) { /* :159-216 */
    const size_t d = cfg->dim;
    if (c->n % cfg->n_lag != 0) return fail_with(OR_INVALID_ARGUMENT, "lag_update: not at a boundary");
    const double rate = (double)c->n_accepted / (double)cfg->n_lag;
    if (cfg->adapt_beta) {
        if (rate > cfg->band_hi)
            c->beta *= cfg->beta_adapt_factor;
        else if (rate < cfg->band_lo)
            c->beta /= cfg->beta_adapt_factor;
        c->beta = c->beta < cfg->beta_min ? cfg->beta_min : (c->beta > cfg->beta_max ? cfg->beta_max : c->beta);
    }
    c->n_accepted = 0;

    const int wants_moments = adapts_cov(cfg->kind) || cfg->adaptive_ref;
    if (wants_moments && c->n >= cfg->n0) {
        double* mean = (double*)malloc(sizeof(double) * d);
        double* second = (double*)malloc(sizeof(double) * d * d);
        double* cov = (double*)malloc(sizeof(double) * d * d);
        const uint64_t count = or_blend(&c->batch_acc, global, mean, second, cov);
        if (adapts_cov(cfg->kind) && count >= 2) {
            double trace = 0.0;
            for (size_t i = 0; i < d; ++i) trace += cov[i * d + i];
            const double floor = 1e-12 * (1.0 + or_lane_dot(mean, mean, d));
            if (trace > floor && isfinite(trace)) {
                double* factor = (double*)malloc(sizeof(double) * d * d);
                int st = or_jittered_cholesky(cov, d, factor);
                if (st != OR_OK) {
                    free(factor);
                    free(mean);
                    free(second);
                    free(cov);
                    return st;
                }
                int usable = 1;
                if (pcn_form(cfg->kind)) {
                    double* centered = (double*)malloc(sizeof(double) * d);
                    double* y = (double*)malloc(sizeof(double) * d);
                    for (size_t i = 0; i < d; ++i) centered[i] = c->x[i] - c->x_ref[i];
                    or_tri_solve(factor, d, centered, y);
                    const double infl = noise_infl(cfg);
                    const double q = 0.5 * or_lane_dot(y, y, d) / (infl * infl);
                    usable = q <= 5.0 * (double)d;
                    free(centered);
                    free(y);
                }
                if (usable) {
                    memcpy(c->factor, factor, sizeof(double) * d * d);
                    if (cfg->use_explicit_inverse) invert_lower(c->factor, d, c->factor_inv);
                }
                free(factor);
            }
        }
        if (cfg->adaptive_ref && c->n >= cfg->n_ref_start && count > 0) memcpy(c->x_ref, mean, sizeof(double) * d);
        free(mean);
        free(second);
        free(cov);
    }
    if (pcn_form(cfg->kind)) c->quad = or_quad_term(cfg, c, c->x);
    c->noise_ctr_at_batch = c->noise_rng.counter;
    or_regenerate_noise(cfg, c, inject_w);
    if (rate_out) *rate_out = rate;
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* engine: src/runner.cpp:122-279, 326-396                                    */
/* ------------------------------------------------------------------------- */
/* One chain's batch (run_chain_batch, src/runner.cpp:359-373, + record_trace :375-379). */
typedef struct or_batch_job {
    const or_run_cfg* cfg;
    const or_target* t;
    or_chain* ch;
    const double* const* inject_w;
    size_t* win_used;
    or_run_out* out;
    const or_moments* global;
    size_t P, batches, step_idx, total_steps_cap;
    int threads, tid;
    int status;
} or_batch_job;

static int run_chain_batch(or_batch_job* j, size_t p) {
    const or_run_cfg* cfg = j->cfg;
    const or_kernel_cfg* k = &cfg->kernel;
    const size_t d = k->dim, M = cfg->intervals_per_batch, win = k->n_lag * d;
    or_run_out* out = j->out;
    or_chain* c = &j->ch[p];
    size_t s_local = j->step_idx;
    for (size_t m = 0; m < M; ++m) {
        for (size_t s = 0; s < k->n_lag; ++s) {
            double lr = 0.0;
            double u = -1.0;
            if (out->log_u) {
                or_stream peek = c->uniform_rng;
                u = or_uniform_open(&peek);
            }
            const int acc = or_mh_step(k, j->t, c, -1.0, &lr);
            if (acc < 0) return -acc;
            if (out->accept_bits) out->accept_bits[p * j->total_steps_cap + s_local] = acc;
            if (out->log_ratio) out->log_ratio[p * j->total_steps_cap + s_local] = lr;
            if (out->log_u) out->log_u[p * j->total_steps_cap + s_local] = log(u);
            ++s_local;
            if (out->traces && cfg->record_traces && c->n > k->n0 && (c->n - k->n0 - 1) % cfg->trace_thin == 0) {
                /* the entry index is the same for every chain (same n) */
                const size_t i = (size_t)((c->n - k->n0 - 1) / cfg->trace_thin);
                if (i < out->trace_cap) {
                    double* tr = out->traces + p * 3 * out->trace_cap;
                    tr[i] = c->log_pi;
                    if (cfg->trace_eigen_projections) {
                        tr[out->trace_cap + i] = or_lane_dot(j->t->proj_min, c->x, d);
                        tr[2 * out->trace_cap + i] = or_lane_dot(j->t->proj_max, c->x, d);
                    }
                }
            }
        }
        double rate = 0.0;
        const double* w = j->inject_w ? j->inject_w[p] + j->win_used[p] * win : NULL;
        const int st = or_lag_update(k, c, j->global, w, &rate);
        if (st != OR_OK) return st;
        j->win_used[p]++;
        const size_t h = j->batches * M + m;
        out->beta_hist[p * cfg->max_batches * M + h] = c->beta;
        out->acc_hist[p * cfg->max_batches * M + h] = rate;
    }
    return OR_OK;
}

static void* batch_worker(void* arg) {
    or_batch_job* j = (or_batch_job*)arg;
    j->status = OR_OK;
    for (size_t p = (size_t)j->tid; p < j->P; p += (size_t)j->threads) {
        const int st = run_chain_batch(j, p);
        if (st != OR_OK) {
            j->status = st;
            break;
        }
    }
    return NULL;
}

int or_run(const or_run_cfg* cfg, const or_target* t, const double* const* inject_w, or_run_out* out) {
    return or_run_ex(cfg, t, inject_w, out, NULL);
}

int or_run_ex(const or_run_cfg* cfg, const or_target* t, const double* const* inject_w, or_run_out* out,
              const or_run_opts* opts) {
    const or_kernel_cfg* k = &cfg->kernel;
    const size_t d = k->dim, M = cfg->intervals_per_batch;
    const size_t P = opts && opts->n_ids ? opts->n_ids : cfg->chains; /* chains run here */
    const int threads = opts && opts->threads > 1 ? (opts->threads < (int)P ? opts->threads : (int)P) : 1;
    or_chain* ch = (or_chain*)calloc(P, sizeof(or_chain));
    size_t* win_used = (size_t*)calloc(P, sizeof(size_t));
    double* x0 = (double*)malloc(sizeof(double) * d);
    or_batch_job* jobs = (or_batch_job*)calloc((size_t)threads, sizeof(or_batch_job));
    pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    int st = OR_OK;
    for (size_t p = 0; p < P; ++p) { /* Engine ctor :122-137 */
        const size_t gp = opts && opts->n_ids ? opts->chain_ids[p] : p; /* global chain index */
        or_stream init;
        or_stream_init(&init, cfg->master_seed, gp, "init");
        for (size_t i = 0; i < d; ++i) x0[i] = cfg->init_dispersion * or_normal(&init);
        or_chain_init(&ch[p], k, t, x0, cfg->master_seed, gp, inject_w ? inject_w[p] : NULL);
        win_used[p] = 1;
    }
    or_moments global;
    moments_alloc(&global, d);
    uint64_t global_batches = 0;
    size_t batches = 0, step_idx = 0;
    const size_t total_steps_cap = cfg->max_batches * M * k->n_lag;
    int reason = 0;
    for (;;) { /* Engine::run :216-279 */
        const uint64_t iters = (uint64_t)cfg->chains * M * batches * k->n_lag;
        if (cfg->max_samples >= 0 && iters >= (uint64_t)cfg->max_samples) {
            reason = 1;
            break;
        }
        if (batches >= cfg->max_batches) {
            reason = 0;
            break;
        }
        /* run_batch :326-357: the chains of a batch are independent (they read only the
         * frozen global snapshot), so workers take them round-robin */
        for (int i = 0; i < threads; ++i) {
            or_batch_job* j = &jobs[i];
            j->cfg = cfg;
            j->t = t;
            j->ch = ch;
            j->inject_w = inject_w;
            j->win_used = win_used;
            j->out = out;
            j->global = &global;
            j->P = P;
            j->batches = batches;
            j->step_idx = step_idx;
            j->total_steps_cap = total_steps_cap;
            j->threads = threads;
            j->tid = i;
            if (threads > 1) pthread_create(&th[i], NULL, batch_worker, j);
            else batch_worker(j);
        }
        for (int i = 0; i < threads; ++i) {
            if (threads > 1) pthread_join(th[i], NULL);
            if (jobs[i].status != OR_OK && st == OR_OK) st = jobs[i].status;
        }
        if (st != OR_OK) goto done;
        step_idx += M * k->n_lag;
        { /* merge :237-245 */
            or_moments* locals = (or_moments*)malloc(sizeof(or_moments) * P);
            for (size_t p = 0; p < P; ++p) locals[p] = ch[p].batch_acc;
            st = or_merge_batch(&global, &global_batches, locals, P);
            free(locals);
            if (st != OR_OK) goto done;
            for (size_t p = 0; p < P; ++p) {
                or_merge_into(&ch[p].cum_acc, &ch[p].batch_acc);
                moments_reset(&ch[p].batch_acc);
            }
        }
        ++batches;
        double cov_err = NAN, mean_err = NAN, psrf = NAN;
        if (global.count >= 2) { /* :249-256 */
            double* cov = (double*)malloc(sizeof(double) * d * d);
            or_covariance(global.second, global.mean, d, cov);
            cov_err = or_cov_error(cov, t->covariance, d);
            mean_err = or_mean_error(global.mean, t->mean, d);
            free(cov);
        }
        if (P >= 2) { /* compute_max_psrf :381-396 */
            or_moments* cums = (or_moments*)malloc(sizeof(or_moments) * P);
            for (size_t p = 0; p < P; ++p) cums[p] = ch[p].cum_acc;
            double mx;
            if (or_psrf_max(cums, P, &mx) == OR_OK) psrf = mx;
            free(cums);
        }
        out->cov_error_hist[batches - 1] = cov_err;
        out->mean_error_hist[batches - 1] = mean_err;
        out->psrf_hist[batches - 1] = psrf;
        if (cfg->psrf_tol > 0 && isfinite(psrf) && psrf <= cfg->psrf_tol) {
            reason = 2;
            break;
        }
        if (cfg->cov_tol > 0 && isfinite(cov_err) && cov_err <= cfg->cov_tol) {
            reason = 3;
            break;
        }
        if (cfg->mean_tol > 0 && isfinite(mean_err) && mean_err <= cfg->mean_tol) {
            reason = 4;
            break;
        }
    }
    out->batches = batches;
    out->total_samples = (uint64_t)cfg->chains * M * batches * k->n_lag;
    out->accumulated_samples = global.count;
    out->stop_reason = reason;
    if (out->traces && cfg->record_traces) {
        const uint64_t n = (uint64_t)batches * M * k->n_lag;
        out->trace_len = n > k->n0 ? (size_t)((n - k->n0 - 1) / cfg->trace_thin + 1) : 0;
    }
    memcpy(out->global_mean, global.mean, sizeof(double) * d);
    or_covariance(global.second, global.mean, d, out->global_cov);
    if (out->final_x)
        for (size_t p = 0; p < P; ++p) memcpy(out->final_x + p * d, ch[p].x, sizeof(double) * d);
done:
    for (size_t p = 0; p < P; ++p) or_chain_free(&ch[p]);
    free(ch);
    free(win_used);
    free(x0);
    free(jobs);
    free(th);
    moments_free(&global);
    return st;
}
