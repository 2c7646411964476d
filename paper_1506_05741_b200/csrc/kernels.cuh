// kernels.cuh — device kernels of the B200 DIAM engine (launch wrappers).
//
// Data layout in HBM (per GPU, C local chains, dimension d, ld = pad_ld(d),
// window length Lw = n_lag):
//   target G        d x ld        precision P (Gaussian) or V^T (twisted), shared
//   factor L_c      d x ld        lower factor, zero upper part (one per chain)
//   factor' L'_c    d x ld        refactor workspace (blend -> POTRF in place)
//   moments S_c     d x ld        raw second moment, lower triangle (per chain)
//   window W_c      Lw x ld       standard normals of the window
//   window Xi_c     Lw x ld       increments s*W*L^T; overwritten in place by
//                                 the post-step states X (SYRK input)
//   window H_c      Lw x ld       G * xi rows (target contraction of Xi)
//   vectors         C x ld        x, g = G x, y = L^-1 (x - x_ref), x_ref, g_ref,
//                                 local mean, cumulative mean / diag
// All pad columns [d, ld) stay zero; every kernel writes only [0, d).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "philox.cuh"

namespace dgb {

// ---------------------------------------------------------------- draws
// W[c][r][i] = normal(key_c, start + r*d + i), r < rows (every chain is at the same
// noise-stream position); if Xi is non-null also Xi = (beta_c * infl) * W, which is
// exactly tri_matvec(I, w) * scale (identity-factor fast path, bit-exact).
void launch_normals(double* W, double* Xi, int64_t chain_stride, int chains, int rows, int d,
                    int64_t ld, const PhiloxKey* keys, uint64_t start, const double* beta,
                    double infl, cudaStream_t s);
// out[c][i] = scale * normal(key_c, start + i), i < n   (init dispersion draws)
void launch_normal_vec(double* out, int64_t stride, int chains, int n, const PhiloxKey* keys,
                       uint64_t start, double scale, cudaStream_t s);
// kernel-level parity entry: raw draws of one stream
void launch_draws(int kind, double* out_f64, uint64_t* out_u64, int64_t n, PhiloxKey key,
                  uint64_t start, cudaStream_t s);

// ---------------------------------------------------------------- MH window
struct StepParams {
    int d, n_lag, chains;
    int64_t ld, win_stride;
    int dg;               // entries of g = G x and of the H rows (d + the twisted rows)
    int64_t ldg;          // their stride
    int64_t hwin_stride;  // per-chain stride of the H window
    double* W;        // in: the window's normals; out: row j = z_j (the j-th distinct counted
                      // state's whitened coordinates, the moment SYRK's B operand)
    double* Xi;       // out: row k = the z part of h_t of the k-th accepted step
    double* H;        // in: h_t = G xi_t rows (s W L_z^T); out: row j = m_j z_j, m_j = the
                      // counted steps spent in state j
    int first;        // first counted step of this chunk (proj/src/proposal.cpp:153-155)
    int* kcount;      // [chain]: distinct counted states of the chunk
    int* acc_count;   // [chain]: accepted steps of the chunk
    int* state_src;   // [chain][out_ld]: distinct state j = the state after accepted step src_j (-1: start)
    int* state_mult;  // [chain][out_ld]: m_j
    int* row_of;      // [chain][out_ld], nullable: the distinct state after step t
    double* g;
    double* y;
    const double* gr;  // null: zero reference point
    double* log_pi;
    double* quad;
    const double* beta;
    uint64_t* n_accepted;
    const PhiloxKey* ukeys;
    uint64_t* uctr;  // advanced by n_lag
    double infl;
    int pcn;  // pCN-form kernels (pCN, DIAM)
    const double* inv_eig;  // per g entry: the whitened log density's weights (Engine::upload_target)
    const double* bcoef;    // per g entry: twist coefficients / subtraction flags
    double* trace_lp;       // [chain][out_ld], nullable
    uint8_t* accept_out;    // [chain][out_ld], nullable
    double* log_ratio_out;  // [chain][out_ld], nullable (parity tests)
    int out_ld;             // per-chain stride of the outputs above (the window length: a
                            // chunk of a window writes at its row offset); 0 = n_lag
};
void launch_mh_window(const StepParams& p, cudaStream_t s);
// x-space states of a chunk from its accepted increments XA (rows k, xi_k = G^-1 h_k): the final
// x, the distinct counted states x_j into Xout rows, and the running x-space mean / raw
// diagonal over the chunk's kc counted steps after n_prev earlier ones
void launch_reconstruct(double* x, const double* xr, const double* beta, int pcn, const double* XA, int64_t xa_stride,
                        int64_t xa_ld, double* Xout, int64_t xo_stride, int64_t ld, const int* state_src,
                        const int* state_mult, int out_ld, const int* kcount, const int* acc_count, double* mean_x,
                        double* diag_x, double n_prev, int kc, int chains, int d, const double* Z, int64_t z_stride,
                        double* mean_z, cudaStream_t s);

// ---------------------------------------------------------------- moments
// (The running means are updated by reconstruct_kernel; the second moment is the weighted
// SYRK through gemm_f64.)
// Blend (count weights) and covariance, written as a lower matrix with zero upper part
// into C_out (the refactor workspace); blended mean -> mb. jitter_eps > 0 adds
// eps*trace_c/d on the diagonal (trace from tr[c]). mask: chains to process.
void launch_blend_cov(double* const* C_out, const double* Sg, const double* mg,
                      const double* Sl, int64_t sl_stride, const double* ml, int64_t ml_stride,
                      double wg, double wl, double* mb, int64_t mb_stride, int chains, int d,
                      int64_t ld, const int* mask, double jitter_eps, const double* tr,
                      const double* jitter_mat, cudaStream_t s, const double* aug_x = nullptr,
                      const double* aug_xr = nullptr, int64_t aug_stride = 0, const struct TraceX* tx = nullptr);
// The x-space side of a refactor's first attempt, done by one extra CTA per chain of the blend
// launch: the blended mean mb, trace tr and trace-floor flag try from the x-space statistics
// (proj/src/proposal.cpp:177-183), and the factorization status reset
struct TraceX {
    const double* Sg;
    const double* mg;
    const double* dl;
    const double* ml;
    double* mb;
    double* tr;
    int* try_flag;
    int* status;
};
// Merge helpers (proj/src/moments.cpp:51-88)
void launch_sum_chains(double* out, const double* in, int64_t chain_stride, int chains, int64_t n,
                       double weight, cudaStream_t s);
// packed lower triangle of sum_c S_c (chains ascending), and the merge of such a sum into Sg
void launch_sum_chains_lower(double* out, const double* S, int64_t stride, int chains, int d, int64_t ld,
                             cudaStream_t s);
void launch_merge_lower(double* Sg, int64_t ld, const double* packed, int d, double keep, double wp,
                        cudaStream_t s);
void launch_axpby(double* y, const double* x, int64_t n, double a, double b, cudaStream_t s);
// cum mean/diag fold (merge_into restricted to the PSRF inputs)
// cumulative per-chain x-space mean and raw diagonal (PSRF inputs) from the batch's
// (ldiag: chain c's diagonal at ldiag + c s_stride)
void launch_cum_fold(double* cmean, double* cdiag, const double* lmean, const double* ldiag,
                     int64_t s_stride, int chains, int d, int64_t ld, double keep, double add,
                     cudaStream_t s);
// the batch's convergence statistics on the device (single GPU): out4 = {cov error, mean
// error, max sqrt(R) (PSRF), flags: 1 zero reference norm, 2 zero within-chain variance}
void launch_batch_stats(const double* part2, const double* mg, const double* tmean, int d, const double* cmean,
                        const double* cdiag, int64_t ld, int chains, uint64_t n_per_chain, bool want_err,
                        bool want_psrf, double* out4, cudaStream_t s);
// cov/mean error partial sums for cov_error (proj/src/diagnostics.cpp:121-142)
void launch_cov_error(const double* Sg, const double* mg, const double* Ctrue, int d, int64_t ld,
                      double* out2, cudaStream_t s);

// ---------------------------------------------------------------- triangular
// y_c = L_c^{-1} (x_c - xr_c); quad_c = half_inv_infl2 * sum y^2 (pcn) and, if
// qmax >= 0, usable_c &= (0.5*y.y/infl^2 <= qmax). mask: chains to process.
// explicit inverse (use_explicit_inverse): X = L^{-1} for the masked chains (T: r2 x d/2
// scratch per chain), and y = X (x - xr), quad = hq |y|^2
void trtri_batched(double* const* L, double* const* X, double* const* T, int64_t ld, int d, int chains,
                   const int* mask, cudaStream_t s);
void launch_trmv_quad(double* const* X, int64_t ld, const double* x, const double* xr, int64_t vstride, double* y,
                      int64_t ystride, double* quad_out, int chains, int d, double half_inv_infl2, cudaStream_t s);
void launch_trsv(double* const* L, int64_t ld, const double* x, const double* xr, int64_t vstride,
                 double* y, int64_t ystride, double* quad_out, int chains, int d, double half_inv_infl2,
                 const int* mask, cudaStream_t s);
// y_c = x_c (rows of stride ld), quad_c = hq |x_c|^2: the identity factor's y and quad
void launch_init_yq(const double* x, int64_t ld, double* y, double* quad, int chains, int d, double hq,
                    cudaStream_t s);
// Cholesky of the lower part of A_c (in place), blocked right-looking with the
// diagonal blocks factored in shared memory, TRSM and SYRK through gemm_f64.
// status[c] = 0 ok, 1 not positive definite. Only chains with mask[c] != 0.
struct PotrfWork {
    double* inv;           // potrf_work_doubles(chains): per chain a 128x128 slot holding the two
                           // 64x64 inverse diagonal blocks of a block column, then int active[chains]
    double** inv128_ptrs;  // chain i: inv + i * 128 * 128
};
inline size_t potrf_work_doubles(int chains) { return (size_t)chains * 128 * 128 + chains; }
void potrf_batched(double* const* A, int64_t ld, int d, int chains, const int* mask, int* status,
                   PotrfWork& w, cudaStream_t s, int extra_rows = 0);
// F = the symmetric matrix whose lower triangle S holds (d x ld)
void launch_mirror_lower(const double* S, double* F, int d, int64_t ld, cudaStream_t s);
// G (lower, G^T G = P) from the precision reversed in P_rev (J P J, overwritten by its
// factor); the whitened Gaussian target of the engine (Engine::upload_target)
void whitening_factor(double* P_rev, double* G, int d, int64_t ld, cudaStream_t s);

// ---------------------------------------------------------------- lag update
// beta adaptation + rate (proj/src/proposal.cpp:163-173)
void launch_beta_update(double* beta, uint64_t* n_acc, double* rate_out, double* beta_out,
                        int chains, int n_lag, int adapt, double lo, double hi, double factor,
                        double bmin, double bmax, cudaStream_t s);
// The adoption of a refactor's new factors in one launch (proposal.cpp:185-202): q_c =
// hq |row d of Lnew_c|^2 (the augmented row L'^-1 (x - x_ref); hq < 0: no augmented row),
// usable[c] = try[c] && (q_c <= qmax or qmax < 0), pointers swapped where usable, status reset;
// with y: y_c = that row and quad_c = q_c for the usable chains
void launch_adopt_factor(double** L, double** Lnew, int64_t ld, int d, int chains, const int* try_flag, int* status,
                         double hq, double qmax, int* usable, double* y, double* quad, cudaStream_t s);
// L_c = I
void launch_set_identity(double* base, int64_t mat_stride, int chains, int d, int64_t ld, cudaStream_t s);
// log pi from x and g = G x (Gaussian: -1/2 x.g; twisted: -1/2 sum twist(g)^2 / sigma^2)
// log pi = -1/2 sum over pairs (e, e+1) of ie_e w_e^2 + ie_{e+1} (w_{e+1}^2 - bc_{e+1} g_{e+1}^2),
// w = (g_e, g_{e+1} + bc_e g_e^2): the whitened form of every target (Engine::upload_target)
void launch_eval_logpi(const double* g, const double* inv_eig, const double* bcoef, double* out, int chains, int dg,
                       int64_t ldg, cudaStream_t s);
// mb_c = wg*mg + wl*ml_c
void launch_blend_mean(const double* mg, const double* ml, double wg, double wl, double* mb, int chains,
                       int d, int64_t ld, cudaStream_t s);
// out[c][t][0..1] = proj[0..1] . X_c[t], t in [t0, rows)
// out[c] = G X[c] (G d x d row-major; X, out: one row per chain; stride ld)
// out[c][n] = sum_k G[n][k] X[c][k], n < nrows (G rows and X rows of stride ld, out rows of out_ld)
void launch_gemv_rows(const double* G, int64_t ld, int d, int nrows, const double* X, double* out, int64_t out_ld,
                      int chains, cudaStream_t s);
// through row_of (the compacted window): out[c][t] = proj . X_c[row_of[c][t]]
void launch_project_rows(const double* X, int64_t win_stride, int64_t ld, int chains, int rows, int t0,
                         int d, const double* proj, double* out, int out_ld, const int* row_of, cudaStream_t s);
void launch_copy_vecs(double* dst, const double* src, int64_t n, const int* mask_per_chain,
                      int64_t stride, int chains, cudaStream_t s);

}  // namespace dgb
