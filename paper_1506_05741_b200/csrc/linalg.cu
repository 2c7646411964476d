// linalg.cu — batched triangular solve, blocked Cholesky, moment and lag-update kernels.
#include <cmath>

#include <cstdlib>

#include "gemm_f64.cuh"
#include "gemm_tile.cuh"
#include "diag_tc.cuh"
#include "kernels.cuh"

namespace dgb {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// The x-space trace floor of the blended covariance (proj/src/proposal.cpp:177-183) from the
// x-space statistics the whitened engine keeps: mb = wg mg + wl ml (the blended mean, also the
// adaptive reference), tr = sum_i (wg Sg_ii + wl dl_i) - mb_i^2, try = tr > 1e-12 (1 + mb.mb)
__device__ __forceinline__ void trace_x_block(const double* Sg, const double* mg, const double* dl, const double* ml,
                                              double wg, double wl, double* mb, double* tr, int* try_flag, int d,
                                              int64_t ld, int c) {
    double t = 0.0, mm = 0.0;
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        const double m = wg * mg[i] + wl * ml[c * ld + i];
        const double sii = wg * Sg[(int64_t)i * ld + i] + wl * dl[c * ld + i];
        mb[c * ld + i] = m;
        t += sii - m * m;
        mm += m * m;
    }
    __shared__ double red[2][8];
    t = warp_sum(t);
    mm = warp_sum(mm);
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = t;
        red[1][threadIdx.x >> 5] = mm;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < 8; ++w) {
            a += red[0][w];
            b += red[1][w];
        }
        tr[c] = a;
        if (try_flag) try_flag[c] = (a > 1e-12 * (1.0 + b) && isfinite(a)) ? 1 : 0;
    }
}

constexpr int kBlendPairs = 4;  // row pairs per CTA

// C = wg*Sg + wl*Sl - mb mb^T on the lower triangle, 0 above; optional jitter on the diagonal.
// Rows are taken in pairs (p, d-1-p): the two hold d+1 lower entries together, so every
// pair moves the same bytes and all threads work; a CTA handles kBlendPairs pairs of one
// chain (a CTA per pair made d/2 short-lived CTAs per chain: 42% warps active, 3.1 TB/s).
__global__ void blend_cov_kernel(double* const* C_out, const double* Sg, const double* mg, const double* Sl,
                                 int64_t sl_stride, const double* ml, int64_t ml_stride, double wg, double wl,
                                 double* mb, int64_t mb_stride, int d, int64_t ld, const int* mask,
                                 double jitter_eps, const double* tr, const double* jm, const double* ax,
                                 const double* axr, int64_t ax_stride, TraceX tx, int has_tx) {
    const int c = blockIdx.z;
    if (mask && !mask[c]) return;
    const int npairs = (d + 1) / 2, nblk = (npairs + kBlendPairs - 1) / kBlendPairs;
    const int p = blockIdx.y;
    if (has_tx && p == (int)gridDim.y - 1) {
        trace_x_block(tx.Sg, tx.mg, tx.dl, tx.ml, wg, wl, tx.mb, tx.tr, tx.try_flag, d, ld, c);
        if (threadIdx.x == 0) tx.status[c] = 0;
        return;
    }
    if (p == nblk) {  // augmented row r = x - x_ref (solved by the POTRF for the usable guard)
        double* Crow = C_out[c] + (int64_t)d * ld;
        for (int j = threadIdx.x; j < d; j += blockDim.x)
            Crow[j] = ax[c * ax_stride + j] - (axr ? axr[c * ax_stride + j] : 0.0);
        return;
    }
    const double* mlc = ml + c * ml_stride;
    // jitter eps (tr / d) (proposal.cpp:229-231); with jm, eps (tr / d) J -- the whitened
    // space's image of eps (tr / d) I -- read only when there is jitter
    const double jit = jitter_eps > 0.0 ? jitter_eps * (tr[c] / (double)d) : 0.0;
    for (int pp = p * kBlendPairs; pp < min(npairs, (p + 1) * kBlendPairs); ++pp) {
        const int r1 = pp, r2 = d - 1 - pp;  // r1 == r2: the middle row of an odd d
        // blended mean (proj/src/moments.cpp:44)
        const double mb1 = wg * mg[r1] + wl * mlc[r1];
        const double mb2 = wg * mg[r2] + wl * mlc[r2];
        if (threadIdx.x == 0 && mb) {
            mb[c * mb_stride + r1] = mb1;
            mb[c * mb_stride + r2] = mb2;
        }
        // Lower triangle only. The strict upper part of a workspace factor is zero already
        // (zeroed at allocation and by set_identity; the POTRF zeroes the strict upper part
        // of every diagonal block it factors, the only upper entries its GEMMs touch), and
        // it stays zero through factor/workspace pointer swaps.
        // Column pairs (rows are 64-byte aligned: ld is a multiple of 8), both rows flattened.
        const int q1 = (r1 + 2) / 2, q2 = r2 == r1 ? 0 : (r2 + 2) / 2;
        for (int q = threadIdx.x; q < q1 + q2; q += blockDim.x) {
            const bool first = q < q1;
            const int i = first ? r1 : r2;
            const int j = 2 * (first ? q : q - q1);
            const double mbi = first ? mb1 : mb2;
            // the pair (j, j+1) is loaded as one double2 unless j+1 lies past the diagonal: at
            // j = i = d-1 with ld == d it would be past the end of the row (and of the buffer)
            const bool pair = j + 1 <= i;
            const double* sgp = Sg + (int64_t)i * ld + j;
            const double* slp = Sl + c * sl_stride + (int64_t)i * ld + j;
            double2 sg, sl, g2, l2;
            if (pair) {
                sg = *reinterpret_cast<const double2*>(sgp);
                sl = __ldcs(reinterpret_cast<const double2*>(slp));  // read once: stream it
                g2 = *reinterpret_cast<const double2*>(mg + j);
                l2 = *reinterpret_cast<const double2*>(mlc + j);
            } else {
                sg = make_double2(*sgp, 0.0);
                sl = make_double2(*slp, 0.0);
                g2 = make_double2(mg[j], 0.0);
                l2 = make_double2(mlc[j], 0.0);
            }
            // covariance :90-101 (S exactly symmetric) of the blend :45-46
            double v0 = (wg * sg.x + wl * sl.x) - mbi * (wg * g2.x + wl * l2.x);
            double v1 = (wg * sg.y + wl * sl.y) - mbi * (wg * g2.y + wl * l2.y);
            if (jit != 0.0) {
                if (jm) {
                    v0 += jit * jm[(int64_t)i * ld + j];
                    if (pair) v1 += jit * jm[(int64_t)i * ld + j + 1];
                } else {
                    if (j == i) v0 += jit;
                    if (j + 1 == i) v1 += jit;
                }
            }
            double* Crow = C_out[c] + (int64_t)i * ld;
            if (pair)
                *reinterpret_cast<double2*>(Crow + j) = make_double2(v0, v1);
            else
                Crow[j] = v0;
        }
    }
}

__global__ void sum_chains_kernel(double* out, const double* in, int64_t chain_stride, int chains, int64_t n,
                                  double weight) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int c = 0; c < chains; ++c) s += in[c * chain_stride + e];
        out[e] = weight * s;
    }
}

// out[i (i+1) / 2 + j] = sum_c S_c[i][j] for j <= i (chains in ascending order): the
// packed lower triangle of the local moment sum, the only part the merge needs (half the
// bytes of the square, and of the all-reduce on several GPUs). CTA p takes rows p and
// d-1-p, so every CTA moves the same number of entries.
__global__ void sum_chains_lower_kernel(double* out, const double* S, int64_t stride, int chains, int d,
                                        int64_t ld) {
    const int p = blockIdx.x, r1 = p, r2 = d - 1 - p;
    const int q1 = r1 + 1, q2 = r2 == r1 ? 0 : r2 + 1;
    for (int q = threadIdx.x; q < q1 + q2; q += blockDim.x) {
        const bool first = q < q1;
        const int i = first ? r1 : r2, j = first ? q : q - q1;
        const double* src = S + (int64_t)i * ld + j;
        double s = 0.0;
        for (int c = 0; c < chains; ++c) s += src[c * stride];
        out[(int64_t)i * (i + 1) / 2 + j] = s;
    }
}

// Sg[i][j] = keep Sg[i][j] + wp packed[i (i+1) / 2 + j], j <= i (proj/src/moments.cpp:63-74)
__global__ void merge_lower_kernel(double* Sg, int64_t ld, const double* packed, int d, double keep, double wp) {
    const int p = blockIdx.x, r1 = p, r2 = d - 1 - p;
    const int q1 = r1 + 1, q2 = r2 == r1 ? 0 : r2 + 1;
    for (int q = threadIdx.x; q < q1 + q2; q += blockDim.x) {
        const bool first = q < q1;
        const int i = first ? r1 : r2, j = first ? q : q - q1;
        double* y = Sg + (int64_t)i * ld + j;
        *y = keep * *y + wp * packed[(int64_t)i * (i + 1) / 2 + j];
    }
}

__global__ void axpby_kernel(double* y, const double* x, int64_t n, double a, double b) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        y[e] = b * y[e] + a * x[e];
}

__global__ void cum_fold_kernel(double* cmean, double* cdiag, const double* lmean, const double* ldiag,
                                int64_t s_stride, int d, int64_t ld, double keep, double add) {
    const int c = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= d) return;
    const int64_t v = c * ld + i;
    cmean[v] = keep * cmean[v] + add * lmean[v];
    cdiag[v] = keep * cdiag[v] + add * ldiag[c * s_stride + i];
}

// partial sums for ||C_emp - C*||_F^2 and ||C*||_F^2 over the full symmetric matrix
__global__ void cov_error_kernel(const double* Sg, const double* mg, const double* Ct, int d, int64_t ld,
                                 double* partial) {
    double num = 0.0, den = 0.0;
    const int i = blockIdx.x;
    for (int j = threadIdx.x; j <= i; j += blockDim.x) {
        const double emp = Sg[(int64_t)i * ld + j] - mg[i] * mg[j];
        const double t = Ct[(int64_t)i * d + j];
        const double t2 = Ct[(int64_t)j * d + i];
        num += (emp - t) * (emp - t);
        den += t * t;
        if (j != i) {
            num += (emp - t2) * (emp - t2);
            den += t2 * t2;
        }
    }
    __shared__ double sn[32], sd[32];
    num = warp_sum(num);
    den = warp_sum(den);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        sn[warp] = num;
        sd[warp] = den;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) {
            a += sn[w2];
            b += sd[w2];
        }
        partial[2 * i] = a;
        partial[2 * i + 1] = b;
    }
}

// ------------------------------------------------------------------ triangular solve
// One CTA per chain: blocked forward substitution y = L^{-1}(x - xr), 64-row blocks.
constexpr int kTrsvThreads = 256;
constexpr int kTrsvB = 64;

__global__ void __launch_bounds__(kTrsvThreads) trsv_kernel(double* const* Lm, int64_t ld, const double* x,
                                                            const double* xr, int64_t vstride, double* y,
                                                            int64_t ystride, double* quad_out, int d, double hq,
                                                            const int* mask) {
    const int c = blockIdx.x;
    if (mask && !mask[c]) return;
    extern __shared__ double sh[];
    double* ys = sh;                       // d
    double* blk = sh + ((d + 1) & ~1);     // 64 x 65
    double* rhs = blk + kTrsvB * (kTrsvB + 1);
    const double* L = Lm[c];
    const double* xc = x + c * vstride;
    const double* xrc = xr ? xr + c * vstride : nullptr;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = kTrsvThreads / 32;

    for (int b0 = 0; b0 < d; b0 += kTrsvB) {
        const int bs = min(kTrsvB, d - b0);
        // diagonal block -> shared (coalesced rows)
        for (int e = tid; e < bs * kTrsvB; e += kTrsvThreads) {
            const int r = e / kTrsvB, j = e % kTrsvB;
            blk[r * (kTrsvB + 1) + j] = (j <= r && j < bs) ? L[(int64_t)(b0 + r) * ld + b0 + j] : 0.0;
        }
        // rhs_i = (x_i - xr_i) - L[i, 0:b0] . y[0:b0]
        for (int r = warp; r < bs; r += NW) {
            const double* Lr = L + (int64_t)(b0 + r) * ld;
            double s = 0.0;
            for (int j = lane; j < b0; j += 32) s += Lr[j] * ys[j];
            s = warp_sum(s);
            if (lane == 0) {
                const double xi = xc[b0 + r] - (xrc ? xrc[b0 + r] : 0.0);
                rhs[r] = xi - s;
            }
        }
        __syncthreads();
        if (warp == 0) {
            // column-oriented substitution inside the block: lane owns rows lane, lane+32
            double r0 = lane < bs ? rhs[lane] : 0.0;
            double r1 = lane + 32 < bs ? rhs[lane + 32] : 0.0;
            for (int j = 0; j < bs; ++j) {
                const int owner = j & 31;
                double yj;
                if (j < 32) yj = __shfl_sync(0xffffffffu, r0, owner);
                else yj = __shfl_sync(0xffffffffu, r1, owner);
                yj = yj / blk[j * (kTrsvB + 1) + j];
                if (lane == owner) {
                    if (j < 32) r0 = yj;
                    else r1 = yj;
                }
                if (lane > j && lane < bs) r0 -= blk[lane * (kTrsvB + 1) + j] * yj;
                if (lane + 32 > j && lane + 32 < bs) r1 -= blk[(lane + 32) * (kTrsvB + 1) + j] * yj;
            }
            if (lane < bs) ys[b0 + lane] = r0;
            if (lane + 32 < bs) ys[b0 + lane + 32] = r1;
        }
        __syncthreads();
    }
    // write y and the quad term
    double s = 0.0;
    for (int i = tid; i < d; i += kTrsvThreads) {
        const double v = ys[i];
        if (y) y[c * ystride + i] = v;
        s += v * v;
    }
    __shared__ double red[NW];
    s = warp_sum(s);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < NW; ++w) t += red[w];
        quad_out[c] = hq * t;
    }
}

// ------------------------------------------------------------------ G x for a chain group
// out[c] = G X[c] for C chains (G: d x d row-major; X, out: one row per chain; all with
// stride ld): a CTA takes 16 rows of G
// and 8 chains, a warp two rows; lanes stride along k with 16-byte loads, and the 16
// (row, chain) partial sums are combined by recursive halving (16 shuffles per warp).
// One pass over G per 8 chains instead of a 128-row DMMA tile with 4 valid rows.
__global__ void __launch_bounds__(256) gemv_rows_kernel(const double* G, int64_t ld, int d, int nrows,
                                                        const double* X, double* out, int64_t out_ld, int chains) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n0 = blockIdx.x * 16 + 2 * warp;
    const int c0 = blockIdx.y * 8;
    const int nc = min(8, chains - c0);
    const double* xs[8];
#pragma unroll
    for (int ch = 0; ch < 8; ++ch) xs[ch] = ch < nc ? X + (int64_t)(c0 + ch) * ld : nullptr;
    const double* g0 = G + (int64_t)min(n0, nrows - 1) * ld;
    const double* g1 = G + (int64_t)min(n0 + 1, nrows - 1) * ld;
    double v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = 0.0;
    const int dk = (d + 1) & ~1;  // rows are zero-padded to ld (a multiple of 8)
    for (int k = 2 * lane; k < dk; k += 64) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(g0 + k));
        const double2 b = __ldg(reinterpret_cast<const double2*>(g1 + k));
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
            if (ch >= nc) break;
            const double2 x = *reinterpret_cast<const double2*>(xs[ch] + k);
            v[ch] = fma(a.y, x.y, fma(a.x, x.x, v[ch]));
            v[8 + ch] = fma(b.y, x.y, fma(b.x, x.x, v[8 + ch]));
        }
    }
    // recursive halving: after the xor-16/8/4/2 steps lane l holds slot l >> 1 summed over 16
    // lanes; the xor-1 step completes the sum over the warp
#pragma unroll
    for (int w = 8; w >= 1; w >>= 1) {
        const int x = w * 2;  // partner distance 16, 8, 4, 2
        const bool upper = lane & x;
#pragma unroll
        for (int i = 0; i < w; ++i) {
            const double send = upper ? v[i] : v[i + w];
            const double keep = upper ? v[i + w] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, x);
        }
    }
    const double tot = v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
    const int slot = lane >> 1, r = slot >> 3, ch = slot & 7;
    if (!(lane & 1) && ch < nc && n0 + r < nrows) out[(int64_t)(c0 + ch) * out_ld + n0 + r] = tot;
}

// ------------------------------------------------------------------ Cholesky diagonal block
constexpr int kNb = kDiagNb;


// The 128 x 128 diagonal block of block column J = [j0, j0 + n1 + n2) in one CTA per chain
// (n1 = 64, n2 <= 64; n2 = 0 for a last block column of width <= 64), from shared memory:
//   (1) L11 = chol(A11), X11 = L11^-1 (diag_tc.cuh)
//   (2) L21 = A21 X11^T, A22 -= L21 L21^T, L22 = chol(A22), X22 = L22^-1 (the same routine
//       with its pre-solve and pre-update)
//   (3) X21 = -X22 (L21 X11), completing X_J = L_JJ^{-1} in the chain's 128 x 128 slot (row
//       stride 128) for the block column's one 128-deep TRSM
// Two CTAs per SM (<= 128 registers) so a diagonal-block CTA can share its SM with a GEMM
// CTA of another chain group.
using X21Tile = tile::Cfg<64, 64, 32, 2, true, false, 2, 4, 1>;  // X21's two 64 x 64 products (8 warps)
static_assert(X21Tile::SMEM_BYTES <= (int)sizeof(DiagTcScratch), "X21 products reuse the diagonal scratch");

__global__ void __launch_bounds__(256, 2) potrf_diag_kernel(double* const* Am, int64_t ld, int j0, int n1, int n2,
                                                            const int* mask, int* status, int* active,
                                                            double* inv_base) {
    extern __shared__ __align__(16) double dyn_smem[];
    const int c = blockIdx.x;
    const bool run = (!mask || mask[c]) && status[c] == 0;
    if (threadIdx.x == 0) active[c] = run ? 1 : 0;
    if (!run) return;
    DiagTcScratch& sc = *reinterpret_cast<DiagTcScratch*>(dyn_smem);
    double* A11 = Am[c] + (int64_t)j0 * ld + j0;
    // the chain's 128 x 128 inverse slot X_J (row stride 128): X11 at [0, 0), X22 at [64, 64)
    double* xj = inv_base + (int64_t)c * kD2 * kD2;
    int bad = diag64_tc_sc(sc, A11, ld, n1, xj, 0, kD2);
    if (!bad && n2 > 0) {
        __syncthreads();  // the first block's stores have read the scratch; X11 is in the slot
        double* A22 = A11 + (int64_t)kNb * ld + kNb;
        bad = diag64_tc_sc(sc, A22, ld, n2, xj + kNb * kD2 + kNb, j0 > 0 ? 1 : 0, kD2, A22 - kNb, xj, kD2);
        if (!bad) {
            // X21 = -X22 (L21 X11): T = L21 X11 into X21's place, then in place (L21 was
            // solved by this CTA)
            __threadfence_block();
            tile::gemm_tile<X21Tile, true, false>(A22 - kNb, xj, xj + kNb * kD2, ld, kD2, kD2, n2, kNb, kNb, 0, 0,
                                                  1.0, 0.0, false, dyn_smem);
            __threadfence_block();
            tile::gemm_tile<X21Tile, true, false>(xj + kNb * kD2 + kNb, xj + kNb * kD2, xj + kNb * kD2, kD2, kD2, kD2,
                                                  n2, kNb, n2, 0, 0, -1.0, 0.0, false, dyn_smem);
        }
    }
    if (bad && threadIdx.x == 0) {
        status[c] = 1;
        active[c] = 0;
    }
}

// The rows below a block column's diagonal block: L[r, J] = A[r, J] X_J^T, one 128-deep
// triangular DMMA product per 64-row tile (B(k, n) = X_J[n][k] = 0 for k > n), in place:
// a CTA owns all of J's columns for its rows, so it reads its whole A tile before writing.
// Column n needs k <= n only, so a warp owning 32 consecutive columns would do between 1/4
// and all of the work and the per-stage barrier would pace every warp at the slowest: each
// warp instead owns two 16-column blocks from opposite ends, {w, 7 - w} (w = warp % 4), and
// skips the k steps past each 8-column fragment's last column: 272 DMMAs for every warp (and
// every SM sub-partition, which hosts warps w and w + 4) against 128 (w + 1) before.
using TrsmTile = tile::Cfg<64, 128, 32, 2, true, true, 2, 4, 2>;  // stage layout: 64 x 32 A, 128 x 32 B

// fragment j of warp column wn, in descending column order: the fragments still live at a
// given k are always the first ones
__device__ __forceinline__ int trsm_frag_col(int wn, int j) {
    return j < 2 ? 16 * (7 - wn) + 8 * (1 - j) : 16 * wn + 8 * (3 - j);
}

// 8 k (two k4 steps) of the NL live fragments: a separate body per live count, selected by a
// warp-uniform switch, so the dead fragments' DMMAs are not issued (if-converted, they would
// still occupy the tensor pipe)
template <int NL>
__device__ __forceinline__ void trsm_chunk(double (&acc)[4][4][2], const double* a_s, const double* b_s, int kk0,
                                           int wm0, int wn, int fr, int fk) {
#pragma unroll
    for (int kk = kk0; kk < kk0 + 8; kk += 4) {
        double af[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = a_s[(wm0 + i * 8 + fr) * TrsmTile::A_STRIDE + kk + fk];
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            const double bf = b_s[(trsm_frag_col(wn, j) + fr) * TrsmTile::B_STRIDE + kk + fk];
#pragma unroll
            for (int i = 0; i < 4; ++i) tile::dmma(acc[i][j], af[i], bf);
        }
    }
}

__global__ void __launch_bounds__(256, 2) potrf_trsm_kernel(double* const* Am, int64_t ld, int r0, int c0, int rows,
                                                            int nb, const int* active, double* const* inv) {
    using CF = TrsmTile;
    const int c = blockIdx.z;
    if (!active[c]) return;
    extern __shared__ __align__(16) double smem[];
    double* a = Am[c] + (int64_t)r0 * ld + c0;
    const double* X = inv[c];  // B(k, n) = X[n * kD2 + k]
    const int m0 = blockIdx.y * CF::BM;
    const int N = nb, K = nb;
    double* sA = smem;
    double* sB = smem + CF::STAGES * CF::A_STAGE;
    const int KT = (K + CF::BK - 1) / CF::BK;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm0 = (warp / 4) * 32, wn = warp % 4;
    const int fr = lane >> 2, fk = lane & 3;
    auto issue = [&](int kt, int stage) {
        const int k0 = kt * CF::BK;
        tile::load_tile<CF::A_ROWS, CF::A_COLS, CF::A_STRIDE, CF::THREADS>(sA + stage * CF::A_STAGE,
                                                                        a + (int64_t)m0 * ld + k0, ld, rows - m0,
                                                                        K - k0, tid);
        tile::load_tile<CF::B_ROWS, CF::B_COLS, CF::B_STRIDE, CF::THREADS>(sB + stage * CF::B_STAGE, X + k0, kD2, N,
                                                                        K - k0, tid);
    };
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    issue(0, 0);
    tile::cp_async_commit();
    const bool compute = m0 + wm0 < rows;
    for (int kt = 0; kt < KT; ++kt) {
        tile::cp_async_wait<0>();
        __syncthreads();
        if (kt + 1 < KT) issue(kt + 1, (kt + 1) % CF::STAGES);
        tile::cp_async_commit();
        const double* a_s = sA + (kt % CF::STAGES) * CF::A_STAGE;
        const double* b_s = sB + (kt % CF::STAGES) * CF::B_STAGE;
        if (compute) {
#pragma unroll
            for (int kk0 = 0; kk0 < CF::BK; kk0 += 8) {
                // fragments with a column >= k (B(k, n) = 0 for k > n)
                const int kg = kt * CF::BK + kk0;
                int nl = 0;
#pragma unroll
                for (int j = 0; j < 4; ++j) nl += trsm_frag_col(wn, j) + 8 > kg ? 1 : 0;
                switch (nl) {
                    case 4: trsm_chunk<4>(acc, a_s, b_s, kk0, wm0, wn, fr, fk); break;
                    case 3: trsm_chunk<3>(acc, a_s, b_s, kk0, wm0, wn, fr, fk); break;
                    case 2: trsm_chunk<2>(acc, a_s, b_s, kk0, wm0, wn, fr, fk); break;
                    case 1: trsm_chunk<1>(acc, a_s, b_s, kk0, wm0, wn, fr, fk); break;
                    default: break;
                }
            }
        }
    }
    tile::cp_async_wait<0>();
    __syncthreads();  // every warp has read its A rows: the tile may be overwritten
    if (!compute) return;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = m0 + wm0 + i * 8 + fr;
        if (r >= rows) continue;
        double* crow = a + (int64_t)r * ld;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int q = trsm_frag_col(wn, j) + 2 * fk;
            if (q + 1 < N) *reinterpret_cast<double2*>(crow + q) = make_double2(acc[i][j][0], acc[i][j][1]);
            else if (q < N) crow[q] = acc[i][j][0];
        }
    }
}

__global__ void beta_update_kernel(double* beta, uint64_t* n_acc, double* rate_out, double* beta_out, int chains,
                                   int n_lag, int adapt, double lo, double hi, double factor, double bmin,
                                   double bmax) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= chains) return;
    const double rate = (double)n_acc[c] / (double)n_lag;  // proj/src/proposal.cpp:162-172
    double b = beta[c];
    if (adapt) {
        if (rate > hi) b *= factor;
        else if (rate < lo) b /= factor;
        b = b < bmin ? bmin : (b > bmax ? bmax : b);
    }
    beta[c] = b;
    n_acc[c] = 0;
    if (rate_out) rate_out[c] = rate;
    if (beta_out) beta_out[c] = b;
}

__global__ void __launch_bounds__(256) adopt_factor_kernel(double** L, double** Lnew, int64_t ld, int d,
                                                           const int* try_flag, int* status, double hq, double qmax,
                                                           int* usable, double* y, double* quad) {
    const int c = blockIdx.x;
    const bool tried = try_flag[c] != 0;
    const double* row = Lnew[c] + (int64_t)d * ld;  // read before thread 0 may swap the pointers
    __shared__ double red[8];
    __shared__ int s_ok;
    double q = 0.0;
    if (hq >= 0.0 && tried) {  // proj/src/proposal.cpp:190-196
        double t = 0.0;
        for (int i = threadIdx.x; i < d; i += blockDim.x) t += row[i] * row[i];
        t = warp_sum(t);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
        __syncthreads();
        if (threadIdx.x == 0) {
            double u = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) u += red[w];
            q = hq * u;
        }
    }
    if (threadIdx.x == 0) {
        bool ok = tried;
        if (ok && qmax >= 0.0) ok = q <= qmax;  // proj/src/proposal.cpp:197-199
        if (ok) {
            double* t = L[c];
            L[c] = Lnew[c];
            Lnew[c] = t;
        }
        usable[c] = ok ? 1 : 0;
        status[c] = 0;
        if (ok && quad) quad[c] = q;
        s_ok = ok;
    }
    __syncthreads();
    if (s_ok && y)
        for (int i = threadIdx.x; i < d; i += blockDim.x) y[c * ld + i] = row[i];
}

__global__ void copy_vecs_kernel(double* dst, const double* src, int64_t n, const int* mask, int64_t stride) {
    const int c = blockIdx.y;
    if (mask && !mask[c]) return;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        dst[c * stride + e] = src[c * stride + e];
}

__global__ void set_identity_kernel(double* base, int64_t mat_stride, int d, int64_t ld) {
    const int c = blockIdx.y;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)d * ld;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / ld, j = e % ld;
        base[c * mat_stride + e] = (i == j) ? 1.0 : 0.0;
    }
}

__global__ void eval_logpi_kernel(const double* g, const double* inv_eig, const double* bcoef, double* out, int dg,
                                  int64_t ldg) {
    const int c = blockIdx.x;
    const double* gc = g + c * ldg;
    double s = 0.0;
    for (int i = 2 * threadIdx.x; i < dg; i += 2 * blockDim.x) {
        const double g0 = gc[i], g1 = i + 1 < dg ? gc[i + 1] : 0.0;
        const double w1 = g1 + bcoef[i] * g0 * g0;
        s += g0 * g0 * inv_eig[i] + (i + 1 < dg ? (w1 * w1 - bcoef[i + 1] * g1 * g1) * inv_eig[i + 1] : 0.0);
    }
    __shared__ double red[32];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        out[c] = -0.5 * t;
    }
}

__global__ void blend_mean_kernel(const double* mg, const double* ml, double wg, double wl, double* mb, int d,
                                  int64_t ld) {
    const int c = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < d) mb[c * ld + i] = wg * mg[i] + wl * ml[c * ld + i];
}

__global__ void project_rows_kernel(const double* X, int64_t win_stride, int64_t ld, int rows, int t0, int d,
                                    const double* proj, double* out, int out_ld, const int* row_of) {
    const int c = blockIdx.y;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int t = t0 + warp;
    if (t >= rows) return;
    const double* xr = X + c * win_stride + (int64_t)row_of[(int64_t)c * out_ld + t] * ld;
    double a = 0.0, b = 0.0;
    for (int i = lane; i < d; i += 32) {
        a += proj[i] * xr[i];
        b += proj[ld + i] * xr[i];
    }
    a = warp_sum(a);
    b = warp_sum(b);
    if (lane == 0) {
        out[((int64_t)c * out_ld + t) * 2] = a;
        out[((int64_t)c * out_ld + t) * 2 + 1] = b;
    }
}

unsigned grid_for(int64_t n, int threads, int cap_per_sm = 8) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), (int64_t)kNumSMs * cap_per_sm));
}

}  // namespace

void launch_gemv_rows(const double* G, int64_t ld, int d, int nrows, const double* X, double* out, int64_t out_ld,
                      int chains, cudaStream_t s) {
    if (chains <= 0 || d <= 0) return;
    dim3 grid((unsigned)ceil_div(nrows, 16), (unsigned)ceil_div(chains, 8));
    gemv_rows_kernel<<<grid, 256, 0, s>>>(G, ld, d, nrows, X, out, out_ld, chains);
    DGB_LAUNCH_CHECK();
    count_launch();
}

void launch_blend_cov(double* const* C_out, const double* Sg, const double* mg, const double* Sl,
                      int64_t sl_stride, const double* ml, int64_t ml_stride, double wg, double wl, double* mb,
                      int64_t mb_stride, int chains, int d, int64_t ld, const int* mask, double jitter_eps,
                      const double* tr, const double* jitter_mat, cudaStream_t s, const double* aug_x,
                      const double* aug_xr, int64_t aug_stride, const TraceX* tx) {
    const int nblk = ((d + 1) / 2 + kBlendPairs - 1) / kBlendPairs;
    dim3 grid(1, (unsigned)(nblk + (aug_x ? 1 : 0) + (tx ? 1 : 0)), chains);
    blend_cov_kernel<<<grid, 256, 0, s>>>(C_out, Sg, mg, Sl, sl_stride, ml, ml_stride, wg, wl, mb, mb_stride, d, ld,
                                          mask, jitter_eps, tr, jitter_mat, aug_x, aug_xr,
                                          aug_stride > 0 ? aug_stride : ld, tx ? *tx : TraceX{}, tx ? 1 : 0);
    DGB_LAUNCH_CHECK();
    count_launch();
}

void launch_sum_chains(double* out, const double* in, int64_t chain_stride, int chains, int64_t n, double weight,
                       cudaStream_t s) {
    sum_chains_kernel<<<grid_for(n, 256), 256, 0, s>>>(out, in, chain_stride, chains, n, weight);
    DGB_LAUNCH_CHECK();
    count_launch();
}

void launch_sum_chains_lower(double* out, const double* S, int64_t stride, int chains, int d, int64_t ld,
                             cudaStream_t s) {
    sum_chains_lower_kernel<<<(d + 1) / 2, 256, 0, s>>>(out, S, stride, chains, d, ld);
    DGB_LAUNCH_CHECK();
    count_launch();
}

void launch_merge_lower(double* Sg, int64_t ld, const double* packed, int d, double keep, double wp,
                        cudaStream_t s) {
    merge_lower_kernel<<<(d + 1) / 2, 256, 0, s>>>(Sg, ld, packed, d, keep, wp);
    DGB_LAUNCH_CHECK();
    count_launch();
}

void launch_axpby(double* y, const double* x, int64_t n, double a, double b, cudaStream_t s) {
    axpby_kernel<<<grid_for(n, 256), 256, 0, s>>>(y, x, n, a, b);
    DGB_LAUNCH_CHECK();
    count_launch();
}

void launch_cum_fold(double* cmean, double* cdiag, const double* lmean, const double* ldiag, int64_t s_stride,
                     int chains, int d, int64_t ld, double keep, double add, cudaStream_t s) {
    dim3 grid((unsigned)ceil_div(d, 128), chains);
    cum_fold_kernel<<<grid, 128, 0, s>>>(cmean, cdiag, lmean, ldiag, s_stride, d, ld, keep, add);
    DGB_LAUNCH_CHECK();
    count_launch();
}

// out[0] cov error, out[1] mean error, out[2] max sqrt(R), out[3] flags (1: zero reference
// norm, 2: zero within-chain variance). The same summation orders as the host versions
// (Engine::batch_stats, psrf_max in host.cpp), no FMA contraction.
__global__ void batch_stats_kernel(const double* part2, const double* mg, const double* tmean, int d,
                                   const double* cmean, const double* cdiag, int64_t ld, int chains, double n,
                                   int want_err, int want_psrf, double* out) {
    __shared__ double smax[256];
    __shared__ int sbad[256];
    const int tid = threadIdx.x;
    if (tid == 0) {
        out[0] = out[1] = out[2] = nan("");
        out[3] = 0.0;
        if (want_err) {  // proj/src/diagnostics.cpp:121-142, proj/src/runner.cpp:249-256
            double num = 0.0, den = 0.0;
            for (int i = 0; i < d; ++i) {
                num = __dadd_rn(num, part2[2 * i]);
                den = __dadd_rn(den, part2[2 * i + 1]);
            }
            if (den > 0.0) out[0] = sqrt(__ddiv_rn(num, den));
            else out[3] = 1.0;
            double s = 0.0;
            for (int i = 0; i < d; ++i) {
                const double df = __dadd_rn(mg[i], -tmean[i]);
                s = __dadd_rn(s, __dmul_rn(df, df));
            }
            out[1] = sqrt(s);
        }
    }
    if (!want_psrf) return;
    // proj/src/diagnostics.cpp:72-119 per direction, then the max
    const double pd = (double)chains, inv_p = __ddiv_rn(1.0, pd);
    double mx = 0.0;
    int bad = 0;
    for (int i = tid; i < d; i += blockDim.x) {
        double gm = 0.0;
        for (int c = 0; c < chains; ++c) gm = __dadd_rn(gm, __dmul_rn(inv_p, cmean[(int64_t)c * ld + i]));
        double between = 0.0, within = 0.0;
        for (int c = 0; c < chains; ++c) {
            const double m = cmean[(int64_t)c * ld + i];
            const double dl = __dadd_rn(m, -gm);
            between = __dadd_rn(between, __dmul_rn(dl, dl));
            within = __dadd_rn(within, __dadd_rn(cdiag[(int64_t)c * ld + i], -__dmul_rn(m, m)));
        }
        const double b = __dmul_rn(__ddiv_rn(n, __dadd_rn(pd, -1.0)), between);
        const double w = __dmul_rn(__ddiv_rn(n, __dmul_rn(__dadd_rn(n, -1.0), pd)), within);
        if (!(w > 0.0)) bad = 1;
        const double r = sqrt(__dadd_rn(__ddiv_rn(__dadd_rn(n, -1.0), n),
                                        __dmul_rn(__ddiv_rn(__dadd_rn(pd, 1.0), __dmul_rn(pd, n)), __ddiv_rn(b, w))));
        mx = r > mx ? r : mx;  // std::max(mx, r): a NaN r leaves mx
    }
    smax[tid] = mx;
    sbad[tid] = bad;
    __syncthreads();
    if (tid == 0) {
        double m = 0.0;
        int anybad = 0;
        for (int k = 0; k < (int)blockDim.x; ++k) {
            m = smax[k] > m ? smax[k] : m;
            anybad |= sbad[k];
        }
        if (anybad) out[3] = (double)((int)out[3] | 2);
        else out[2] = m;
    }
}

void launch_batch_stats(const double* part2, const double* mg, const double* tmean, int d, const double* cmean,
                        const double* cdiag, int64_t ld, int chains, uint64_t n_per_chain, bool want_err,
                        bool want_psrf, double* out4, cudaStream_t s) {
    batch_stats_kernel<<<1, 256, 0, s>>>(part2, mg, tmean, d, cmean, cdiag, ld, chains, (double)n_per_chain,
                                         want_err ? 1 : 0, want_psrf ? 1 : 0, out4);
    DGB_LAUNCH_CHECK();
    count_launch();
}

void launch_cov_error(const double* Sg, const double* mg, const double* Ctrue, int d, int64_t ld, double* out2,
                      cudaStream_t s) {
    cov_error_kernel<<<d, 256, 0, s>>>(Sg, mg, Ctrue, d, ld, out2);
    DGB_LAUNCH_CHECK();
    count_launch();
}

void launch_trsv(double* const* L, int64_t ld, const double* x, const double* xr, int64_t vstride, double* y,
                 int64_t ystride, double* quad_out, int chains, int d, double half_inv_infl2, const int* mask,
                 cudaStream_t s) {
    const size_t smem = sizeof(double) * (((d + 1) & ~1) + kTrsvB * (kTrsvB + 1) + kTrsvB);
    if (smem > 48 * 1024) set_smem_attr(reinterpret_cast<const void*>(trsv_kernel), (int)smem);
    trsv_kernel<<<chains, kTrsvThreads, smem, s>>>(L, ld, x, xr, vstride, y, ystride, quad_out, d, half_inv_infl2,
                                                   mask);
    DGB_LAUNCH_CHECK();
    count_launch();
}

// ------------------------------------------------------------------ explicit inverse
// use_explicit_inverse (proj/src/proposal.cpp:98, 202, 241-252): X = L^{-1} kept beside the
// factor, and the quadratic term taken as |X (x - x_ref)|^2 (proposal.cpp:51-61) instead of a
// triangular solve. The reference inverts by d column solves; here by recursive doubling of
// 64x64 diagonal inverses, [L11 0; L21 L22]^{-1} = [X11 0; -X22 L21 X11  X22], the two
// products of every level on the DMMA GEMM.
constexpr int kInvB = 64;

// one CTA per (64-block, chain): thread j solves column j of the block by forward substitution
__global__ void __launch_bounds__(kInvB) trtri_diag_kernel(double* const* Lm, double* const* Xm, int64_t ld, int d,
                                                           const int* mask) {
    const int c = blockIdx.y;
    if (mask && !mask[c]) return;
    const int b0 = blockIdx.x * kInvB, n = min(kInvB, d - b0);
    extern __shared__ double inv_smem[];
    auto sl = reinterpret_cast<double(*)[kInvB + 1]>(inv_smem);
    auto sx = reinterpret_cast<double(*)[kInvB + 1]>(inv_smem + kInvB * (kInvB + 1));
    const double* L = Lm[c] + (int64_t)b0 * ld + b0;
    for (int e = threadIdx.x; e < kInvB * kInvB; e += kInvB) {
        const int r = e / kInvB, q = e % kInvB;
        sl[r][q] = (r < n && q <= r) ? L[(int64_t)r * ld + q] : 0.0;
    }
    __syncthreads();
    const int j = threadIdx.x;
    for (int i = 0; i < n; ++i) {
        if (i >= j) {
            double s = i == j ? 1.0 : 0.0;
            for (int k = j; k < i; ++k) s -= sl[i][k] * sx[k][j];
            sx[i][j] = s / sl[i][i];
        }
    }
    __syncthreads();
    double* X = Xm[c] + (int64_t)b0 * ld + b0;
    for (int e = threadIdx.x; e < n * kInvB; e += kInvB) {
        const int r = e / kInvB, q = e % kInvB;
        if (q < n) X[(int64_t)r * ld + q] = q <= r ? sx[r][q] : 0.0;
    }
}

// y = X (x - xr) (lower-triangular X), quad = hq |y|^2: one CTA per chain, a warp per row
__global__ void __launch_bounds__(256) trmv_quad_kernel(double* const* Xm, int64_t ld, const double* x,
                                                        const double* xr, int64_t vstride, double* y, int64_t ystride,
                                                        double* quad_out, int d, double hq) {
    const int c = blockIdx.x;
    extern __shared__ double rs[];
    const double* X = Xm[c];
    const double* xc = x + c * vstride;
    const double* xrc = xr ? xr + c * vstride : nullptr;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < d; i += blockDim.x) rs[i] = xc[i] - (xrc ? xrc[i] : 0.0);
    __syncthreads();
    double q = 0.0;
    for (int i = warp; i < d; i += 8) {
        const double* Xr = X + (int64_t)i * ld;
        double s = 0.0;
        for (int j = lane; j <= i; j += 32) s += Xr[j] * rs[j];
        s = warp_sum(s);
        if (lane == 0) {
            y[c * ystride + i] = s;
            q += s * s;
        }
    }
    __shared__ double red[8];
    if (lane == 0) red[warp] = q;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w];
        quad_out[c] = hq * t;
    }
}

void trtri_batched(double* const* L, double* const* X, double* const* T, int64_t ld, int d, int chains,
                   const int* mask, cudaStream_t s) {
    const int smem = 2 * kInvB * (kInvB + 1) * (int)sizeof(double);
    set_smem_attr(reinterpret_cast<const void*>(trtri_diag_kernel), smem);
    trtri_diag_kernel<<<dim3((unsigned)ceil_div(d, kInvB), (unsigned)chains), kInvB, smem, s>>>(L, X, ld, d, mask);
    DGB_LAUNCH_CHECK();
    count_launch();
    for (int h = kInvB; h < d; h *= 2) {
        for (int b0 = 0; b0 + h < d; b0 += 2 * h) {
            const int r2 = std::min(h, d - b0 - h);
            GemmBatch t{};  // T = L21 X11 (r2 x h)
            t.A = (const double* const*)L;
            t.B = (const double* const*)X;
            t.C = T;
            t.a_off = (int64_t)(b0 + h) * ld + b0;
            t.b_off = (int64_t)b0 * ld + b0;
            t.lda = t.ldb = t.ldc = ld;
            t.M = r2;
            t.N = h;
            t.K = h;
            t.alpha = 1.0;
            t.active = mask;
            gemm_f64(t, chains, true, false, s);
            GemmBatch x{};  // X21 = -X22 T
            x.A = (const double* const*)X;
            x.B = (const double* const*)T;
            x.C = X;
            x.a_off = (int64_t)(b0 + h) * ld + b0 + h;
            x.c_off = (int64_t)(b0 + h) * ld + b0;
            x.lda = x.ldb = x.ldc = ld;
            x.M = r2;
            x.N = h;
            x.K = r2;
            x.alpha = -1.0;
            x.active = mask;
            gemm_f64(x, chains, true, false, s);
        }
    }
}

void launch_trmv_quad(double* const* X, int64_t ld, const double* x, const double* xr, int64_t vstride, double* y,
                      int64_t ystride, double* quad_out, int chains, int d, double half_inv_infl2, cudaStream_t s) {
    const size_t smem = sizeof(double) * (size_t)d;
    if (smem > 48 * 1024) set_smem_attr(reinterpret_cast<const void*>(trmv_quad_kernel), (int)smem);
    trmv_quad_kernel<<<chains, 256, smem, s>>>(X, ld, x, xr, vstride, y, ystride, quad_out, d, half_inv_infl2);
    DGB_LAUNCH_CHECK();
    count_launch();
}

void potrf_batched(double* const* A, int64_t ld, int d, int chains, const int* mask, int* status, PotrfWork& w,
                   cudaStream_t s, int extra_rows) {
    // Left-looking blocked Cholesky over 128-wide block columns J = [j0, j0+128):
    //   (1) A[j0:, J] -= L[j0:, :j0] L[J, :j0]^T    one long-K DMMA GEMM (lower tiles of the
    //                                               diagonal block only)
    //   (2) the first 64x64 diagonal block: L11 = chol, X11 = L11^-1 (one CTA per chain,
    //       shared memory, diag_tc.cuh)
    //   (3) the second one: its rows of the first half-column solved against X11 and their
    //       64-deep update applied first, then L22, X22, and X21 = -X22 L21 X11, so the
    //       chain's slot holds X_J = L_JJ^{-1} (128 x 128)
    //   (4) everything below (potrf_trsm_kernel): L[r, J] = A[r, J] X_J^T, one 128-deep
    //       triangular DMMA product per 64-row tile, in place
    // A last block column of width <= 64 is a diagonal block + one TRSM GEMM.
    // `extra_rows` augmented rows r^T below row d-1 ride along as ordinary rows of the
    // GEMMs and TRSMs and come out as (L^{-1} r)^T: the forward substitution of the
    // usable-factor guard (proj/src/proposal.cpp:185-199) costs no extra pass over L.
    // w.inv holds chains*128*128 doubles (X_J per chain), followed by an int active[chains]
    int* active = reinterpret_cast<int*>(w.inv + (int64_t)chains * kD2 * kD2);

    const int rows = d + extra_rows;
    set_smem_attr(reinterpret_cast<const void*>(potrf_diag_kernel), (int)sizeof(DiagTcScratch));
    set_smem_attr(reinterpret_cast<const void*>(potrf_trsm_kernel), TrsmTile::SMEM_BYTES);
    for (int j0 = 0; j0 < d; j0 += 2 * kNb) {
        const int jb = std::min(2 * kNb, d - j0);
        if (j0 > 0) {
            // A[j0:rows, J] -= L[j0:rows, :j0] L[J, :j0]^T; the warps above the diagonal of
            // the diagonal tile skip their DMMAs and its upper quarter keeps its zeros
            GemmBatch p{};
            p.A = (const double* const*)A;
            p.B = (const double* const*)A;
            p.C = A;
            p.a_off = (int64_t)j0 * ld;
            p.b_off = (int64_t)j0 * ld;
            p.c_off = (int64_t)j0 * ld + j0;
            p.lda = p.ldb = p.ldc = ld;
            p.M = rows - j0;
            p.N = jb;
            p.K = j0;
            p.alpha = -1.0;
            p.beta = 1.0;
            p.active = active;
            p.tri_c_lower = 1;
            // 64 x 64 tiles: this update's per-CTA K loop (K = j0) is the longest latency on
            // the refactor's critical path, halved against 128 x 64 tiles (d=1024, 4 chains:
            // 0.83 -> 0.72 ms per factorization; 22.45 -> 22.21 ms per 16-group batch)
            gemm_f64_small(p, chains, s);
        }
        const int n1 = std::min(kNb, jb), n2 = jb - n1;
        potrf_diag_kernel<<<chains, 256, sizeof(DiagTcScratch), s>>>(A, ld, j0, n1, n2, mask, status, active, w.inv);
        DGB_LAUNCH_CHECK();
        count_launch();
        if (n2 == 0) {  // a last, narrow block column: TRSM L21 = A21 X11^T below it
            const int rest = rows - j0 - jb;
            if (rest <= 0) continue;
            GemmBatch t{};
            t.A = (const double* const*)A;
            t.B = (const double* const*)w.inv128_ptrs;  // X11 at the slot start (row stride 128)
            t.C = A;
            t.a_off = (int64_t)(j0 + jb) * ld + j0;
            t.c_off = t.a_off;
            t.lda = ld;
            t.ldb = kD2;
            t.ldc = ld;
            t.M = rest;
            t.N = jb;
            t.K = jb;
            t.alpha = 1.0;
            t.beta = 0.0;
            t.active = active;
            gemm_f64(t, chains, true, true, s);  // one 64-wide column tile per CTA: safe in place
            continue;
        }
        const int c1 = j0 + kNb;
        const int rest = rows - c1 - n2;
        if (rest <= 0) continue;
        dim3 grid(1, (unsigned)ceil_div(rest, TrsmTile::BM), (unsigned)chains);
        potrf_trsm_kernel<<<grid, 256, TrsmTile::SMEM_BYTES, s>>>(A, ld, c1 + n2, j0, rest, jb, active,
                                                                  w.inv128_ptrs);
        DGB_LAUNCH_CHECK();
        count_launch();
    }
}


// G[i][j] = F[d-1-j][d-1-i] (j <= i), zero above: from the Cholesky factor F of the reversed
// precision J P J = F F^T, G = (J F J)^T is lower triangular with G^T G = P
__global__ void reverse_factor_kernel(const double* F, double* G, int d, int64_t ld) {
    const int i = blockIdx.x;
    for (int j = threadIdx.x; j < ld; j += blockDim.x)
        G[(int64_t)i * ld + j] = (j <= i && j < d) ? F[(int64_t)(d - 1 - j) * ld + (d - 1 - i)] : 0.0;
}

void whitening_factor(double* P_rev, double* G, int d, int64_t ld, cudaStream_t s) {
    // P_rev: the reversed precision (lower part used), factored in place
    double** pa = nullptr;
    int* status = nullptr;
    double* inv = nullptr;
    double** invp = nullptr;
    // stream-ordered pool allocations: a plain cudaFree synchronises the device and can make
    // the driver trim the pool the previous engine left (measured: 450 ms per engine init)
    DGB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&pa), 2 * sizeof(double*), s));
    invp = pa + 1;
    DGB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&status), sizeof(int), s));
    DGB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&inv), potrf_work_doubles(1) * sizeof(double), s));
    DGB_CUDA(cudaMemcpyAsync(pa, &P_rev, sizeof(double*), cudaMemcpyHostToDevice, s));
    DGB_CUDA(cudaMemcpyAsync(invp, &inv, sizeof(double*), cudaMemcpyHostToDevice, s));
    DGB_CUDA(cudaMemsetAsync(status, 0, sizeof(int), s));
    PotrfWork w{inv, invp};
    potrf_batched(pa, ld, d, 1, nullptr, status, w, s, 0);
    reverse_factor_kernel<<<d, 256, 0, s>>>(P_rev, G, d, ld);
    DGB_LAUNCH_CHECK();
    count_launch();
    int st = 0;
    DGB_CUDA(cudaMemcpyAsync(&st, status, sizeof(int), cudaMemcpyDeviceToHost, s));
    cudaFreeAsync(inv, s);
    cudaFreeAsync(status, s);
    cudaFreeAsync(pa, s);
    DGB_CUDA(cudaStreamSynchronize(s));
    if (st != 0) throw CudaError("target precision is not positive definite");
}

__global__ void init_yq_kernel(const double* x, int64_t ld, double* y, double* quad, int d, double hq) {
    const int c = blockIdx.x;
    double s = 0.0;
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        const double v = x[c * ld + i];
        y[c * ld + i] = v;
        s += v * v;
    }
    __shared__ double red[8];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w];
        quad[c] = hq * t;
    }
}

void launch_init_yq(const double* x, int64_t ld, double* y, double* quad, int chains, int d, double hq,
                    cudaStream_t s) {
    init_yq_kernel<<<chains, 256, 0, s>>>(x, ld, y, quad, d, hq);
    DGB_LAUNCH_CHECK();
    count_launch();
}

__global__ void mirror_lower_kernel(const double* S, double* F, int d, int64_t ld) {
    const int i = blockIdx.x;
    for (int j = threadIdx.x; j < ld; j += blockDim.x)
        F[(int64_t)i * ld + j] = j >= d ? 0.0 : (j <= i ? S[(int64_t)i * ld + j] : S[(int64_t)j * ld + i]);
}

void launch_mirror_lower(const double* S, double* F, int d, int64_t ld, cudaStream_t s) {
    mirror_lower_kernel<<<d, 256, 0, s>>>(S, F, d, ld);
    DGB_LAUNCH_CHECK();
    count_launch();
}

void launch_beta_update(double* beta, uint64_t* n_acc, double* rate_out, double* beta_out, int chains, int n_lag,
                        int adapt, double lo, double hi, double factor, double bmin, double bmax, cudaStream_t s) {
    beta_update_kernel<<<(unsigned)ceil_div(chains, 128), 128, 0, s>>>(beta, n_acc, rate_out, beta_out, chains, n_lag,
                                                                      adapt, lo, hi, factor, bmin, bmax);
    DGB_LAUNCH_CHECK();
    count_launch();
}

void launch_adopt_factor(double** L, double** Lnew, int64_t ld, int d, int chains, const int* try_flag, int* status,
                         double hq, double qmax, int* usable, double* y, double* quad, cudaStream_t s) {
    adopt_factor_kernel<<<chains, 256, 0, s>>>(L, Lnew, ld, d, try_flag, status, hq, qmax, usable, y, quad);
    DGB_LAUNCH_CHECK();
    count_launch();
}

void launch_set_identity(double* base, int64_t mat_stride, int chains, int d, int64_t ld, cudaStream_t s) {
    dim3 grid(grid_for((int64_t)d * ld, 256, 1), chains);
    set_identity_kernel<<<grid, 256, 0, s>>>(base, mat_stride, d, ld);
    DGB_LAUNCH_CHECK();
    count_launch();
}

void launch_eval_logpi(const double* g, const double* inv_eig, const double* bcoef, double* out, int chains, int dg,
                       int64_t ldg, cudaStream_t s) {
    eval_logpi_kernel<<<chains, 256, 0, s>>>(g, inv_eig, bcoef, out, dg, ldg);
    DGB_LAUNCH_CHECK();
    count_launch();
}

void launch_blend_mean(const double* mg, const double* ml, double wg, double wl, double* mb, int chains, int d,
                       int64_t ld, cudaStream_t s) {
    dim3 grid((unsigned)ceil_div(d, 128), chains);
    blend_mean_kernel<<<grid, 128, 0, s>>>(mg, ml, wg, wl, mb, d, ld);
    DGB_LAUNCH_CHECK();
    count_launch();
}

void launch_project_rows(const double* X, int64_t win_stride, int64_t ld, int chains, int rows, int t0, int d,
                         const double* proj, double* out, int out_ld, const int* row_of, cudaStream_t s) {
    if (t0 >= rows) return;
    const int warps = rows - t0;
    dim3 grid((unsigned)ceil_div((int64_t)warps * 32, 256), chains);
    project_rows_kernel<<<grid, 256, 0, s>>>(X, win_stride, ld, rows, t0, d, proj, out, out_ld, row_of);
    DGB_LAUNCH_CHECK();
    count_launch();
}

void launch_copy_vecs(double* dst, const double* src, int64_t n, const int* mask, int64_t stride, int chains,
                      cudaStream_t s) {
    dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 32)), chains);
    copy_vecs_kernel<<<grid, 256, 0, s>>>(dst, src, n, mask, stride);
    DGB_LAUNCH_CHECK();
    count_launch();
}

}  // namespace dgb
