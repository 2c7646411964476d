// window.cu — Philox draws and the sequential MH window kernel.
//
// The MH window is the only inherently sequential part of the sampler: step
// t+1 of a chain depends on step t's accept decision. Everything O(d^2) per
// step in the reference (SYMV log density, TRSV quad term, SYR moments) has
// been moved into window-level dense contractions (gemm_f64), so one step is
// O(d) work: with x' = x_ref + c (x - x_ref) + xi_t,
//   G x'            = G x_ref + c (G x - G x_ref) + (G Xi^T)_t      [H rows]
//   L^-1 (x'-x_ref) = c y + s w_t   (xi_t = s L w_t, y = L^-1 (x - x_ref))
//   log pi(x')      = -1/2 x'.(G x')  or  -1/2 sum twist(z')^2/sigma^2
//   quad(x')        = 1/2 |L^-1(x'-x_ref)|^2 / infl^2
// One CTA owns one chain for the whole window, its state vectors in registers;
// each step is one fused pass (candidate, two dot products, CTA reduction with
// a single barrier, accept/reject from the chain's Philox uniform) — the
// "fused warp-level accept/reject" of the design.
#include <cooperative_groups.h>

#include "kernels.cuh"

namespace dgb {

namespace {

// grid: x over rows, y over chains; threads over the row's d entries (no index division)
__global__ void normals_kernel(double* W, double* Xi, int64_t chain_stride, int rows, int d, int64_t ld,
                               const PhiloxKey* keys, uint64_t start, const double* beta, double infl) {
    const int c = blockIdx.y;
    const PhiloxKey key = keys[c];
    const double scale = Xi ? beta[c] * infl : 0.0;
    double* Wc = W + c * chain_stride;
    double* Xc = Xi ? Xi + c * chain_stride : nullptr;
    for (int r = blockIdx.x; r < rows; r += gridDim.x) {
        const uint64_t base = start + (uint64_t)r * d;
        for (int i = threadIdx.x; i < d; i += blockDim.x) {
            const double z = philox_normal(key, base + (uint64_t)i);
            Wc[(int64_t)r * ld + i] = z;
            if (Xc) Xc[(int64_t)r * ld + i] = scale * z;
        }
    }
}

__global__ void normal_vec_kernel(double* out, int64_t stride, int chains, int n, const PhiloxKey* keys,
                                  uint64_t start, double scale) {
    const int c = blockIdx.y;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[c * stride + i] = scale * philox_normal(keys[c], start + (uint64_t)i);
}

__global__ void draws_kernel(int kind, double* out_f64, uint64_t* out_u64, int64_t n, PhiloxKey key,
                             uint64_t start) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (kind == 0) out_u64[i] = philox_u64(key, start + i);
        else if (kind == 1) out_f64[i] = philox_uniform_open(key, start + i);
        else out_f64[i] = philox_normal(key, start + i);
    }
}

#ifdef MH_PROFILE  // tools/mh_lat.cu: per-phase cycle sums of block 0, thread 0
__device__ long long g_mh_prof[8];
#define MH_PROF(i)                                                       \
    do {                                                                 \
        const long long now = clock64();                                 \
        mh_acc[i] += now - mh_t0;                                        \
        mh_t0 = now;                                                     \
    } while (0)
#else
#define MH_PROF(i) \
    do {           \
    } while (0)
#endif

constexpr int kMaxStages = 8;  // TMA ring depth bound (one mbarrier per stage)

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void st2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }

// The window in whitened coordinates. The proposal factor is kept as L_z = G L (the Cholesky
// factor of the whitened covariance G C G^T, Engine::enqueue_refactor), so the window's
// product H = s W L_z^T gives h_t = G xi_t directly and the step needs no x-space row:
//   g' = G x_ref + c (g - G x_ref) + h_t      (g = G x, the target's whitened coordinates)
//   y' = c y + s w_t                          (y = L^-1 (x - x_ref) = L_z^-1 (g - g_ref))
//   log pi(x') = -1/2 sum ie (twisted) g'^2,  quad = 1/2 |y'|^2 / infl^2
// Only ACCEPTED steps need the x-space candidate x' = x_ref + c (x - x_ref) + xi_t (the
// reference's exact operations, proposal.cpp:119-124): the kernel keeps each accepted h_t
// (row k of Xi, k = accepted count), xi_t = G^-1 h_t for those rows is one small GEMM, and
// reconstruct_kernel replays the x recursion over them.
//
// Compaction of the counted post-step states (steps t >= first; proposal.cpp:153-155): a
// rejected step repeats the previous state, so a window holds about acceptance x n_lag
// DISTINCT states. Row j of W gets the j-th distinct state's whitened z_j, row j of H the
// weighted m_j z_j (m_j = the counted steps spent in it), and the moment SYRK runs over those
// rows in whitened space: S_z += sum_j m_j z_j z_j^T. All writes go to rows the TMA ring has
// already consumed (j, k <= t).
struct Compactor {
    int j = -1;         // current distinct row
    double mult = 0.0;  // counted steps spent in it so far
};

// Two partial sums of a warp in one butterfly: the first exchange leaves lanes 0-15 with
// partial sums of `a` and lanes 16-31 with partial sums of `b`, four more levels finish each
// (5 double shuffles instead of 10); lane 0 ends with sum(a), lane 16 with sum(b).
__device__ __forceinline__ double warp_sum2(double a, double b, int lane) {
    const bool hi = lane & 16;
    double v = (hi ? b : a) + __shfl_xor_sync(0xffffffffu, hi ? a : b, 16);
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// One elected thread streams the window rows (h_t, w_t) into an NS-deep shared-memory ring
// with cp.async.bulk (1-D TMA) and mbarrier transaction counts.
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_row(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

// PRE: the parts of the candidate that change only on acceptance (ga = G x_ref + c (g - G x_ref),
// cy = c y) are kept ready (2 pairs per thread at most: registers). ZREF: the reference point
// is the origin (G x_ref = 0, no registers). TWG: the per-entry log-density constants are
// read through L1 each step instead of held in registers (4 pairs per thread).
// pairs of entries per CTA when a chain of dg entries is split over CL CTAs: an even split,
// rounded up to 4 pairs (64-byte slices for the bulk copies)
__host__ __device__ inline int cluster_span(int dg, int CL) {
    const int pairs = (dg + 1) / 2;
    return ((pairs + CL - 1) / CL + 3) & ~3;
}

// CL > 1: a chain is split over a thread-block cluster of CL CTAs, CTA r owning an even slice
// of the entries (cluster_span; every CTA keeps R <= 2 pairs per thread in registers and its
// own TMA ring of row slices); the per-step partial sums are exchanged through
// distributed shared memory -- every warp stores its partial into each CTA of the cluster --
// and one cluster barrier per step replaces the CTA barrier. Every CTA sums the CL x NW
// partials in the same order, so all take the same accept decision.
template <int R, int T, bool PRE, bool ZREF, int CL>
__global__ void __launch_bounds__(T, 1) mh_window_kernel(StepParams p, int NS) {
    constexpr bool TWG = R >= 4;
    constexpr int NW = T / 32;
    namespace cg = cooperative_groups;
    const int rank = CL > 1 ? (int)cg::this_cluster().block_rank() : 0;
    const int c = blockIdx.x / CL;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int d = p.d, dg = p.dg;
    const int64_t ld = p.ld, ldg = p.ldg;
    const bool pcn = p.pcn != 0;
    extern __shared__ __align__(128) double ring[];  // NS stages, then the log-uniform table
    __shared__ __align__(8) uint64_t full[kMaxStages];
    __shared__ __align__(16) double red[2][CL * NW][2];
    // a stage: this CTA's slice of the h row (ldg: d + the twisted rows) and, for the pCN
    // form, of the w row (ld); e0 = the slice's first entry
    const int span = CL > 1 ? cluster_span(dg, CL) : R * T;  // pairs of this CTA's slice
    const int e0 = CL > 1 ? rank * 2 * span : 0, e_end = CL > 1 ? e0 + 2 * span : 2 * R * T;
    auto clip = [](int64_t v, int64_t hi) -> int64_t { return v < 0 ? 0 : (v > hi ? hi : v); };
    const int64_t h_len = CL > 1 ? clip(ldg - e0, 2 * span) : ldg;
    const int64_t w_len = CL > 1 ? clip(ld - e0, 2 * span) : ld;
    const int64_t stage_h = CL > 1 ? 2 * span : ldg;
    const uint32_t hrow_bytes = (uint32_t)(h_len * sizeof(double)), wrow_bytes = (uint32_t)(w_len * sizeof(double));
    double* stage0 = ring;
    const int64_t stage_len = stage_h + (pcn ? (CL > 1 ? 2 * span : ld) : 0);
    const bool lead = rank == 0;  // writes the chain's scalars

    const double beta = p.beta[c];
    const double cc = pcn ? sqrt(fmax(0.0, 1.0 - beta * beta)) : 1.0;  // proj/src/proposal.cpp:120
    const double sc = beta * p.infl;
    const double hq = 0.5 / (p.infl * p.infl);
    double* Wc = p.W + c * p.win_stride;
    double* Xc = p.Xi + c * p.win_stride;
    double* Hc = p.H + c * p.hwin_stride;
    int* src = p.state_src + (int64_t)c * p.out_ld;
    int* mul = p.state_mult + (int64_t)c * p.out_ld;
    Compactor cp;

    auto issue = [&](int t, int s) {  // producer: row t of the window into stage s = t % NS
        double* st = stage0 + s * stage_len;
        const uint32_t wb = (pcn && w_len > 0) ? wrow_bytes : 0u;
        mbar_expect_tx(&full[s], hrow_bytes + wb);
        if (hrow_bytes) tma_row(st, Hc + (int64_t)t * ldg + e0, hrow_bytes, &full[s]);
        if (wb) tma_row(st + stage_h, Wc + (int64_t)t * ld + e0, wb, &full[s]);
    };
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if constexpr (CL > 1)  // every CTA of the cluster runs before any stores into its shared memory
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    if (tid == 0)
        for (int t = 0; t < NS && t < p.n_lag; ++t) issue(t, t);

    // GRL: the reference point read through L1 each step (4+ pairs per thread: registers would spill)
    constexpr bool GRL = !ZREF && R >= 4;
    // (value-initialised: the accessor lambdas below capture them before the loading loop)
    double2 g[R] = {}, y[R] = {}, grv[(ZREF || GRL) ? 1 : R] = {}, iev[TWG ? 1 : R] = {}, bcv[TWG ? 1 : R] = {},
            ga[R] = {}, cy[R] = {};
    bool vx[R], vg[R];  // entry pair e in x-space (e < d) / in g-space (e < dg)
    auto GR = [&](int r) -> double2 {
        if (ZREF) return make_double2(0.0, 0.0);
        if (GRL) {
            const int e = e0 + 2 * (tid + r * T);
            return e < dg ? __ldg(reinterpret_cast<const double2*>(p.gr + c * ldg + e)) : make_double2(0.0, 0.0);
        }
        return grv[(ZREF || GRL) ? 0 : r];
    };
    auto IE = [&](int r) -> double2 {
        return TWG ? __ldg(reinterpret_cast<const double2*>(p.inv_eig) + e0 / 2 + tid + r * T) : iev[TWG ? 0 : r];
    };
    auto BC = [&](int r) -> double2 {
        return TWG ? __ldg(reinterpret_cast<const double2*>(p.bcoef) + e0 / 2 + tid + r * T) : bcv[TWG ? 0 : r];
    };
    auto refresh = [&](int r) {
        if (!PRE) return;
        const double2 gr = GR(r);
        ga[r].x = gr.x + cc * (g[r].x - gr.x);
        ga[r].y = gr.y + cc * (g[r].y - gr.y);
        cy[r].x = cc * y[r].x;
        cy[r].y = cc * y[r].y;
    };
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int e = e0 + 2 * (tid + r * T);
        vx[r] = e < d && e < e_end;
        vg[r] = e < dg && e < e_end;
        const double2 z2 = make_double2(0.0, 0.0);
        g[r] = vg[r] ? ld2(p.g + c * ldg + e) : z2;
        y[r] = (vx[r] && pcn) ? ld2(p.y + c * ld + e) : z2;
        if (!ZREF && !GRL) grv[(ZREF || GRL) ? 0 : r] = (vg[r] && p.gr) ? ld2(p.gr + c * ldg + e) : z2;
        if (!TWG) {
            iev[TWG ? 0 : r] = vg[r] ? ld2(p.inv_eig + e) : z2;
            bcv[TWG ? 0 : r] = vg[r] ? ld2(p.bcoef + e) : z2;
        }
        refresh(r);
    }
    double lp = p.log_pi[c], q = pcn ? p.quad[c] : 0.0;
    uint64_t nacc = p.n_accepted[c];
    const PhiloxKey uk = p.ukeys[c];
    const uint64_t u0 = p.uctr[c];
    // log u of every step of the window, from the chain's uniform stream (bit-exact u),
    // computed once in parallel instead of redundantly by every thread every step
    double* logu_tab = ring + (int64_t)NS * stage_len;
    for (int t = tid; t < p.n_lag; t += T) logu_tab[t] = log(philox_uniform_open(uk, u0 + (uint64_t)t));
    __syncthreads();

    // one entry pair's candidate from the h and w rows: the same operations whether called for
    // the dot products or, after the decision, to adopt the candidate (bit-identical)
    auto cand = [&](const double* ph, const double* pw, int r, double2& gc, double2& yc) {
        const int e = e0 + 2 * (tid + r * T);
        const double2 h = vg[r] ? ld2(ph + e) : make_double2(0.0, 0.0);
        if (PRE) {
            gc.x = ga[r].x + h.x;
            gc.y = ga[r].y + h.y;
        } else {
            const double2 gr = GR(r);
            gc.x = gr.x + cc * (g[r].x - gr.x) + h.x;
            gc.y = gr.y + cc * (g[r].y - gr.y) + h.y;
        }
        if (pcn) {
            const double2 w = vx[r] ? ld2(pw + e) : make_double2(0.0, 0.0);
            if (PRE) {
                yc.x = cy[r].x + sc * w.x;
                yc.y = cy[r].y + sc * w.y;
            } else {
                yc.x = cc * y[r].x + sc * w.x;
                yc.y = cc * y[r].y + sc * w.y;
            }
        }
    };
    // the z part (first d entries) of the thread's g, scaled, into a window row
    auto store_z = [&](double* row, double scale) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int e = e0 + 2 * (tid + r * T);
            if (!vx[r]) continue;
            const double2 v = make_double2(scale * g[r].x, scale * g[r].y);
            if (e + 1 < d) st2(row + e, v);
            else row[e] = v.x;
        }
    };
    // With 3 or more stages a stage is refilled one step late, so an accepted candidate is
    // re-read from shared memory; with fewer (wide rows) the refill cannot wait and the
    // accepted rows are re-read from global memory (row t of H / W is overwritten by the
    // compaction only after the adoption, j <= t)
    const bool late = NS >= 3;
    int acc_k = 0;  // accepted steps of this chunk so far
#ifdef MH_PROFILE
    long long mh_t0 = clock64(), mh_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
    int s = 0;           // t % NS, kept incrementally (no integer division in the step)
    uint32_t phase = 0;  // (t / NS) & 1
    for (int t = 0; t < p.n_lag; ++t) {
        const double logu = logu_tab[t];
        MH_PROF(0);
        mbar_wait(&full[s], phase);
        MH_PROF(1);
        const double* st = stage0 + s * stage_len;
        double sa0 = 0.0, sa1 = 0.0, sb0 = 0.0, sb1 = 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            double2 gc, yc;
            cand(st - e0, st + stage_h - e0, r, gc, yc);
            // whitened log density: ie w0^2 + ie' (w1^2 - bc' g1^2), w1 = g1 + bc g0^2
            // (Engine::upload_target)
            const double2 ie = IE(r), bc = BC(r);
            const double w1 = gc.y + bc.x * gc.x * gc.x;
            sa0 += gc.x * gc.x * ie.x;
            sa1 += (w1 * w1 - bc.y * gc.y * gc.y) * ie.y;
            if (pcn) {
                sb0 += yc.x * yc.x;
                sb1 += yc.y * yc.y;
            }
        }
        MH_PROF(2);
        const double ws = warp_sum2(sa0 + sa1, sb0 + sb1, lane);
        const int buf = t & 1;
        if constexpr (CL > 1) {
            // this warp's partial into slot (rank, warp) of every CTA of the cluster
            if ((lane & 15) == 0) {
                namespace cg = cooperative_groups;
                cg::cluster_group cl = cg::this_cluster();
#pragma unroll
                for (int q = 0; q < CL; ++q) cl.map_shared_rank(&red[buf][rank * NW + warp][0], q)[lane >> 4] = ws;
            }
            MH_PROF(3);
            asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
        } else {
            if ((lane & 15) == 0) red[buf][warp][lane >> 4] = ws;
            MH_PROF(3);
            __syncthreads();
        }
        MH_PROF(4);
        // every thread is done with step t-1 (its stage may be re-read for an adoption until
        // this barrier): refill that stage NS - 1 steps ahead
        if (tid == 0) {
            if (late && t > 0 && t - 1 + NS < p.n_lag) issue(t - 1 + NS, s == 0 ? NS - 1 : s - 1);
            if (!late && t + NS < p.n_lag) issue(t + NS, s);
        }
        double ta = 0.0, tb = 0.0;
        {
            // the warps' partial sums in 4 independent chains (few registers even at 16 warps)
            constexpr int NA = NW < 4 ? NW : 4;
            double2 v[NA];
#pragma unroll
            for (int k = 0; k < NA; ++k) v[k] = *reinterpret_cast<const double2*>(&red[buf][k][0]);
#pragma unroll
            for (int k = NA; k < CL * NW; ++k) {
                const double2 u = *reinterpret_cast<const double2*>(&red[buf][k][0]);
                v[k % NA].x += u.x;
                v[k % NA].y += u.y;
            }
#pragma unroll
            for (int k = NA / 2; k > 0; k >>= 1)
#pragma unroll
                for (int i = 0; i < k; ++i) {
                    v[i].x += v[i + k].x;
                    v[i].y += v[i + k].y;
                }
            ta = v[0].x;
            tb = v[0].y;
        }
        MH_PROF(5);
        const double lpc = -0.5 * ta;
        const double qc = pcn ? hq * tb : 0.0;
        const double ratio = pcn ? (lpc + qc) - (lp + q) : lpc - lp;  // proj/src/proposal.cpp:77-82
        const bool acc = logu < ratio;                               // strict, :146
        // counted post-step state -> the compacted window (Compactor)
        const bool counted = t >= p.first;
        const bool fresh = counted && (acc || t == p.first);
        if (fresh) {
            if (cp.j >= 0) {
                store_z(Hc + (int64_t)cp.j * ldg, cp.mult);
                if (tid == 0 && lead) mul[cp.j] = (int)cp.mult;
            }
            ++cp.j;
            cp.mult = 0.0;
        }
        if (acc) {
            const double* ph = late ? st - e0 : Hc + (int64_t)t * ldg;
            const double* pw = late ? st + stage_h - e0 : Wc + (int64_t)t * ld;
            // keep h_t (its z part) for the x-space increment xi_t = G^-1 h_t of this step
            double* keep = Xc + (int64_t)acc_k * ld;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int e = e0 + 2 * (tid + r * T);
                if (vx[r]) {
                    if (e + 1 < d) st2(keep + e, ld2(ph + e));
                    else keep[e] = ph[e];
                }
                double2 gc, yc;
                cand(ph, pw, r, gc, yc);
                g[r] = gc;
                if (pcn) y[r] = yc;
                refresh(r);
            }
            ++acc_k;
            lp = lpc;
            q = qc;
            ++nacc;
        }
        if (fresh) {
            store_z(Wc + (int64_t)cp.j * ld, 1.0);
            if (tid == 0 && lead) src[cp.j] = acc_k - 1;  // the state after accepted step acc_k - 1 (-1: the start)
        }
        if (counted) cp.mult += 1.0;
        if (tid == 0 && lead) {
            if (p.trace_lp) p.trace_lp[(int64_t)c * p.out_ld + t] = lp;
            if (p.accept_out) p.accept_out[(int64_t)c * p.out_ld + t] = acc ? 1 : 0;
            if (p.log_ratio_out) p.log_ratio_out[(int64_t)c * p.out_ld + t] = ratio;
            if (p.row_of && counted) p.row_of[(int64_t)c * p.out_ld + t] = cp.j;
        }
        MH_PROF(6);
        if (++s == NS) {
            s = 0;
            phase ^= 1u;
        }
    }
#ifdef MH_PROFILE
    if (blockIdx.x == 0 && tid == 32)  // a thread of warp 1: not the TMA producer
        for (int i = 0; i < 7; ++i) g_mh_prof[i] = mh_acc[i];
#endif
    if (cp.j >= 0) {
        store_z(Hc + (int64_t)cp.j * ldg, cp.mult);
        if (tid == 0 && lead) mul[cp.j] = (int)cp.mult;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int e = e0 + 2 * (tid + r * T);
        if (vg[r]) {
            if (e + 1 < dg) st2(p.g + c * ldg + e, g[r]);
            else p.g[c * ldg + e] = g[r].x;
        }
        if (vx[r] && pcn) {
            if (e + 1 < d) st2(p.y + c * ld + e, y[r]);
            else p.y[c * ld + e] = y[r].x;
        }
    }
    if constexpr (CL > 1)  // no CTA leaves while a partner may still store into its shared memory
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    if (tid == 0 && lead) {
        p.log_pi[c] = lp;
        if (pcn) p.quad[c] = q;
        p.n_accepted[c] = nacc;
        p.uctr[c] = u0 + (uint64_t)p.n_lag;
        p.kcount[c] = cp.j + 1;
        p.acc_count[c] = acc_k;
    }
}

template <int R, int T, bool PRE = (R * T <= 512), int CL = 1>
bool try_tma(const StepParams& p, cudaStream_t s) {
    if (CL > 1 && cluster_span(p.dg, CL) > R * T) return false;
    const size_t stage = (CL > 1 ? (size_t)2 * cluster_span(p.dg, CL) * (p.pcn ? 2 : 1)
                                 : (size_t)(p.ldg + (p.pcn ? p.ld : 0))) *
                         sizeof(double);
    const size_t table = (size_t)p.n_lag * sizeof(double);
    constexpr size_t kMaxSmem = 220 * 1024;
    if (table + stage > kMaxSmem) return false;
    // ring depth: deep enough to hide HBM latency (>= 3 steps ahead), shallow enough that a
    // 110 KB GEMM CTA of another chain group can share the SM (the step loop leaves the DMMA
    // pipe idle); at most kMaxStages (the mbarrier array)
    static const int env_ns = [] {
        const char* e = std::getenv("DIAM_B200_STEP_STAGES");
        return e ? std::atoi(e) : 0;
    }();
    constexpr size_t kShareBudget = 112 * 1024;  // 227 KB - one 110.6 KB GEMM CTA - reserves
    int NS = (int)std::min<size_t>(kMaxStages, (kMaxSmem - table) / stage);
    if (table + 3 * stage <= kShareBudget) NS = std::min<int>(NS, (int)((kShareBudget - table) / stage));
    NS = std::min(NS, 6);
    if (env_ns > 0) NS = std::min<int>(env_ns, (int)std::min<size_t>(kMaxStages, (kMaxSmem - table) / stage));
    const size_t smem = NS * stage + table;
    auto kern = p.gr ? mh_window_kernel<R, T, PRE, false, CL> : mh_window_kernel<R, T, PRE, true, CL>;
    set_smem_attr(reinterpret_cast<const void*>(kern), (int)smem);
    if constexpr (CL == 1) {
        kern<<<p.chains, T, smem, s>>>(p, NS);
    } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(p.chains * CL));
        cfg.blockDim = dim3(T);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CL;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        DGB_CUDA(cudaLaunchKernelEx(&cfg, kern, p, NS));
    }
    return true;
}

void launch_r(const StepParams& p, cudaStream_t s) {
    const int pairs = (p.dg + 1) / 2;  // the g-space entries (d + the twisted rows) set the width
    // 256 threads (up to 2 double2 pairs each) up to d = 1024, then 512 threads: fewer warps
    // per step barrier and reduction for the small dimensions where the step loop matters most.
    // Wider rows (d > 4096) split each chain over a cluster of 4 CTAs of 512 threads x 2 pairs:
    // no thread holds more than 2 pairs of each state vector (one CTA with 8 pairs per thread
    // spilled 420 B) and the chain's row stream is read by 4 SMs. (A 2-CTA cluster at
    // d = 2040 -- 1122 pairs with the twisted rows -- measured 4% slower per batch than one
    // CTA with 4 pairs per thread: twice the CTAs of the 1-CTA-per-SM step kernel.)
    bool done = false;
    // small d (the time-to-cov-error workloads): as few warps as cover the row, so the
    // per-step reduction and barrier span 2 or 4 warps instead of 8
    if (pairs <= 64) done = try_tma<1, 64>(p, s);
    else if (pairs <= 128) done = try_tma<1, 128>(p, s);
    else if (pairs <= 256) done = try_tma<1, 256>(p, s);
    else if (pairs <= 512) done = try_tma<2, 256>(p, s);
    else if (pairs <= 1024) done = try_tma<2, 512>(p, s);
    else if (pairs <= 2048) done = try_tma<4, 512>(p, s);
    else if (pairs <= 4096) done = try_tma<2, 512, false, 4>(p, s);
    if (!done) throw CudaError("mh_window: dimension above 8192 is not supported by this build");
    DGB_LAUNCH_CHECK();
    count_launch();
}

// The x-space states of a chunk, in the reference's exact operations (proposal.cpp:119-124):
// x <- x_ref + c (x - x_ref) + xi_k over the chunk's accepted steps k (xi_k = G^-1 h_k, rows of
// XA); the distinct counted states x_j (rows of Xout, for the eigen-projection traces), the
// x-space running mean and raw diagonal (PSRF, trace floor, adaptive reference) and the
// whitened running mean (from the z_j rows of Z, the blend's mean), with their multiplicities. Threads over the entries (no cross-thread dependence), 128 per CTA so a
// chain spreads over d/128 CTAs.
__global__ void __launch_bounds__(128) reconstruct_kernel(double* x, const double* xr, const double* beta, int pcn,
                                                          const double* __restrict__ XA, int64_t xa_stride,
                                                          int64_t xa_ld, double* __restrict__ Xout, int64_t xo_stride,
                                                          int64_t ld, const int* state_src, const int* state_mult,
                                                          int out_ld, const int* kcount, const int* acc_count,
                                                          double* mean_x, double* diag_x, double keep, double add,
                                                          int d, const double* __restrict__ Z, int64_t z_stride,
                                                          double* mean_z) {
    // the chain's (src, mult) lists in shared memory: every thread walks them
    extern __shared__ int rec_sm[];
    const int c = blockIdx.y;
    const double b = beta[c];
    const double cc = pcn ? sqrt(fmax(0.0, 1.0 - b * b)) : 1.0;
    const int nk = acc_count[c], nj = kcount[c];
    int* src = rec_sm;
    int* mul = rec_sm + out_ld;
    for (int j = threadIdx.x; j < nj; j += blockDim.x) {
        src[j] = state_src[(int64_t)c * out_ld + j];
        mul[j] = state_mult[(int64_t)c * out_ld + j];
    }
    __syncthreads();
    const double* xa = XA + c * xa_stride;
    double* xo = Xout + c * xo_stride;
    const double* zc = Z + c * z_stride;  // row j: the distinct state's whitened z_j
    constexpr int PF = 8;                 // accepted increments in flight per thread
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < d; e += gridDim.x * blockDim.x) {
        double v = x[c * ld + e];
        const double r = xr ? xr[c * ld + e] : 0.0;
        double s1 = 0.0, s2 = 0.0;
        int j = 0;
        // states that predate the chunk's first acceptance
        for (; j < nj && src[j] < 0; ++j) {
            xo[(int64_t)j * ld + e] = v;
            s1 += mul[j] * v;
            s2 += mul[j] * (v * v);
        }
        // the recursion is serial in v, its increments are not: PF loads issued per block
        for (int k0 = 0; k0 < nk; k0 += PF) {
            double inc[PF];
#pragma unroll
            for (int i = 0; i < PF; ++i) inc[i] = k0 + i < nk ? xa[(int64_t)(k0 + i) * xa_ld + e] : 0.0;
#pragma unroll
            for (int i = 0; i < PF; ++i) {
                const int k = k0 + i;
                if (k >= nk) break;
                v = __dadd_rn(__dadd_rn(r, __dmul_rn(cc, __dadd_rn(v, -r))), inc[i]);
                for (; j < nj && src[j] == k; ++j) {
                    xo[(int64_t)j * ld + e] = v;
                    s1 += mul[j] * v;
                    s2 += mul[j] * (v * v);
                }
            }
        }
        x[c * ld + e] = v;
        if (nj > 0) {
            // the whitened running mean (the blend's) from the z_j rows, loads in flight together
            double sz[4] = {0.0, 0.0, 0.0, 0.0};
            int jj = 0;
            for (; jj + 4 <= nj; jj += 4) {
#pragma unroll
                for (int i = 0; i < 4; ++i) sz[i] += mul[jj + i] * zc[(int64_t)(jj + i) * ld + e];
            }
            for (; jj < nj; ++jj) sz[0] += mul[jj] * zc[(int64_t)jj * ld + e];
            mean_x[c * ld + e] = keep * mean_x[c * ld + e] + add * s1;
            diag_x[c * ld + e] = keep * diag_x[c * ld + e] + add * s2;
            mean_z[c * ld + e] = keep * mean_z[c * ld + e] + add * ((sz[0] + sz[1]) + (sz[2] + sz[3]));
        }
    }
}

}  // namespace

void launch_normals(double* W, double* Xi, int64_t chain_stride, int chains, int rows, int d, int64_t ld,
                    const PhiloxKey* keys, uint64_t start, const double* beta, double infl,
                    cudaStream_t s) {
    if ((int64_t)chains * rows * d == 0) return;
    const int threads = 256;
    // about 16 resident 256-thread blocks per SM over all chains
    const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(rows, ceil_div((int64_t)kNumSMs * 16, chains)));
    normals_kernel<<<dim3((unsigned)gx, (unsigned)chains), threads, 0, s>>>(W, Xi, chain_stride, rows, d, ld, keys,
                                                                          start, beta, infl);
    DGB_LAUNCH_CHECK();
    count_launch();
}

void launch_normal_vec(double* out, int64_t stride, int chains, int n, const PhiloxKey* keys, uint64_t start,
                       double scale, cudaStream_t s) {
    dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 64)), chains);
    normal_vec_kernel<<<grid, 256, 0, s>>>(out, stride, chains, n, keys, start, scale);
    DGB_LAUNCH_CHECK();
    count_launch();
}

void launch_draws(int kind, double* out_f64, uint64_t* out_u64, int64_t n, PhiloxKey key, uint64_t start,
                  cudaStream_t s) {
    if (n <= 0) return;
    const int64_t blocks = std::min<int64_t>(ceil_div(n, 256), (int64_t)kNumSMs * 8);
    draws_kernel<<<(unsigned)blocks, 256, 0, s>>>(kind, out_f64, out_u64, n, key, start);
    DGB_LAUNCH_CHECK();
    count_launch();
}

void launch_mh_window(const StepParams& p, cudaStream_t s) {
    if (p.chains <= 0 || p.n_lag <= 0) return;
    StepParams q = p;
    if (q.out_ld <= 0) q.out_ld = q.n_lag;
    launch_r(q, s);
}

void launch_reconstruct(double* x, const double* xr, const double* beta, int pcn, const double* XA, int64_t xa_stride,
                        int64_t xa_ld, double* Xout, int64_t xo_stride, int64_t ld, const int* state_src,
                        const int* state_mult, int out_ld, const int* kcount, const int* acc_count, double* mean_x,
                        double* diag_x, double n_prev, int kc, int chains, int d, const double* Z, int64_t z_stride,
                        double* mean_z, cudaStream_t s) {
    if (chains <= 0) return;
    const double total = n_prev + kc;
    const dim3 grid((unsigned)std::max(1, (d + 127) / 128), (unsigned)chains);
    const size_t smem = 2 * (size_t)out_ld * sizeof(int);
    if (smem > 48 * 1024) set_smem_attr(reinterpret_cast<const void*>(reconstruct_kernel), (int)smem);
    reconstruct_kernel<<<grid, 128, smem, s>>>(x, xr, beta, pcn, XA, xa_stride, xa_ld, Xout, xo_stride, ld, state_src,
                                              state_mult, out_ld, kcount, acc_count, mean_x, diag_x,
                                              total > 0 ? n_prev / total : 0.0, total > 0 ? 1.0 / total : 0.0, d, Z,
                                              z_stride, mean_z);
    DGB_LAUNCH_CHECK();
    count_launch();
}

}  // namespace dgb
