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

constexpr int kStepThreads = 512;
constexpr int kMaxStages = 8;  // TMA ring depth bound (one mbarrier per stage)
constexpr int kStepWarps = kStepThreads / 32;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void st2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }

// scale * v (this thread's pairs of a state vector) -> one window row
template <int R, int T>
__device__ __forceinline__ void store_row(double* row, const double2 (&v)[R], const bool (&valid)[R], int tid, int d,
                                          double scale) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int e = 2 * (tid + r * T);
        if (!valid[r]) continue;
        const double2 w = make_double2(scale * v[r].x, scale * v[r].y);
        if (e + 1 < d) st2(row + e, w);
        else row[e] = w.x;
    }
}

// Window compaction of the counted post-step states (steps t >= first; the reference
// accumulates x after every such step, proj/src/proposal.cpp:153-155): a rejected step
// repeats the previous state, so the window holds only about acceptance x n_lag DISTINCT
// states. Row j of Xi gets the j-th distinct state x_j, row j of H the weighted m_j x_j
// (m_j = the number of counted steps spent in it), and the moment SYRK and mean run over
// those rows: S += sum_j m_j x_j x_j^T -- the same sum, in fewer, exact-integer-weighted
// terms. Both rows are written only once consumed (j <= t), so the TMA ring and the
// register prefetch of the rows ahead are never overwritten.
struct Compactor {
    int j = -1;         // current distinct row
    double mult = 0.0;  // counted steps spent in it so far
};

// R = double2 pairs per thread; PREF = prefetch the next step's rows into registers
template <int R, bool TWISTED, bool PREF>
__global__ void __launch_bounds__(kStepThreads, 1) mh_window_kernel(StepParams p) {
    const int c = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int d = p.d;
    const int64_t ld = p.ld;
    __shared__ double red[2][kStepWarps][2];

    const double beta = p.beta[c];
    const bool pcn = p.pcn != 0;
    const double cc = pcn ? sqrt(fmax(0.0, 1.0 - beta * beta)) : 1.0;  // proj/src/proposal.cpp:120
    const double sc = beta * p.infl;
    const double hq = 0.5 / (p.infl * p.infl);

    const int dg = p.dg;
    const int64_t ldg = p.ldg;
    const double* Wc = p.W + c * p.win_stride;
    double* Xc = p.Xi + c * p.win_stride;
    double* Hc = p.H + c * p.hwin_stride;
    Compactor cp;

    double2 x[R], g[R], y[R], xr[R], gr[R], ie[R], bc[R];
    bool valid[R], vg[R];  // entry pair e in x-space (e < d) / in g-space (e < dg)
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int e = 2 * (tid + r * kStepThreads);
        valid[r] = e < d;
        vg[r] = e < dg;
        const double2 z2 = make_double2(0.0, 0.0);
        x[r] = valid[r] ? ld2(p.x + c * ld + e) : z2;
        g[r] = vg[r] ? ld2(p.g + c * ldg + e) : z2;
        y[r] = (valid[r] && pcn) ? ld2(p.y + c * ld + e) : z2;
        xr[r] = (valid[r] && p.xr) ? ld2(p.xr + c * ld + e) : z2;
        gr[r] = (vg[r] && p.gr) ? ld2(p.gr + c * ldg + e) : z2;
        if (TWISTED) {
            ie[r] = vg[r] ? ld2(p.inv_eig + e) : z2;
            bc[r] = vg[r] ? ld2(p.bcoef + e) : z2;
        }
    }
    double lp = p.log_pi[c], q = pcn ? p.quad[c] : 0.0;
    uint64_t nacc = p.n_accepted[c];
    const PhiloxKey uk = p.ukeys[c];
    const uint64_t u0 = p.uctr[c];

    double2 xi[R], w[R], h[R];
    auto load_row = [&](int t, double2 (&a)[R], double2 (&b)[R], double2 (&hh)[R]) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int e = 2 * (tid + r * kStepThreads);
            const double2 z2 = make_double2(0.0, 0.0);
            a[r] = valid[r] ? ld2(Xc + (int64_t)t * ld + e) : z2;
            b[r] = (valid[r] && pcn) ? ld2(Wc + (int64_t)t * ld + e) : z2;
            hh[r] = vg[r] ? ld2(Hc + (int64_t)t * ldg + e) : z2;
        }
    };
    load_row(0, xi, w, h);

    for (int t = 0; t < p.n_lag; ++t) {
        double2 nxi[R], nw[R], nh[R];
        if (PREF && t + 1 < p.n_lag) load_row(t + 1, nxi, nw, nh);
        const double logu = log(philox_uniform_open(uk, u0 + (uint64_t)t));

        double2 xc[R], gc[R], yc[R];
        double sa = 0.0, sb = 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            // candidate exactly as proj/src/proposal.cpp:119-124 (x_ref + c (x - x_ref) + xi)
            // explicit _rn ops: no FMA contraction, so x' has the reference's exact bits
            xc[r].x = __dadd_rn(__dadd_rn(xr[r].x, __dmul_rn(cc, __dadd_rn(x[r].x, -xr[r].x))), xi[r].x);
            xc[r].y = __dadd_rn(__dadd_rn(xr[r].y, __dmul_rn(cc, __dadd_rn(x[r].y, -xr[r].y))), xi[r].y);
            gc[r].x = gr[r].x + cc * (g[r].x - gr[r].x) + h[r].x;
            gc[r].y = gr[r].y + cc * (g[r].y - gr[r].y) + h[r].y;
            if (TWISTED) {
                // w_{2j+1} = z_{2j+1} + b_{2j} z_{2j}^2 (proj/src/target.cpp:167-173)
                const double w0 = gc[r].x;
                const double w1 = gc[r].y + bc[r].x * gc[r].x * gc[r].x;
                // whitened form: ie w0^2 + ie' (w1^2 - bc' g1^2) (Engine::upload_target)
                sa += w0 * w0 * ie[r].x + (w1 * w1 - bc[r].y * gc[r].y * gc[r].y) * ie[r].y;
            } else {
                sa += xc[r].x * gc[r].x + xc[r].y * gc[r].y;
            }
            if (pcn) {
                yc[r].x = cc * y[r].x + sc * w[r].x;
                yc[r].y = cc * y[r].y + sc * w[r].y;
                sb += yc[r].x * yc[r].x + yc[r].y * yc[r].y;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            sa += __shfl_xor_sync(0xffffffffu, sa, o);
            sb += __shfl_xor_sync(0xffffffffu, sb, o);
        }
        const int buf = t & 1;
        if (lane == 0) {
            red[buf][warp][0] = sa;
            red[buf][warp][1] = sb;
        }
        __syncthreads();
        double ta = 0.0, tb = 0.0;
#pragma unroll
        for (int k = 0; k < kStepWarps; ++k) {
            ta += red[buf][k][0];
            tb += red[buf][k][1];
        }
        const double lpc = -0.5 * ta;
        const double qc = pcn ? hq * tb : 0.0;
        const double ratio = pcn ? (lpc + qc) - (lp + q) : lpc - lp;  // proj/src/proposal.cpp:77-82
        const bool acc = logu < ratio;                               // strict, :146
        // counted post-step state -> the compacted window (Compactor)
        const bool counted = t >= p.first;
        const bool fresh = counted && (acc || t == p.first);
        if (fresh) {
            if (cp.j >= 0) store_row<R, kStepThreads>(Hc + (int64_t)cp.j * ldg, x, valid, tid, d, cp.mult);
            ++cp.j;
            cp.mult = 0.0;
        }
        if (acc) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                x[r] = xc[r];
                g[r] = gc[r];
                if (pcn) y[r] = yc[r];
            }
            lp = lpc;
            q = qc;
            ++nacc;
        }
        if (fresh) store_row<R, kStepThreads>(Xc + (int64_t)cp.j * ld, x, valid, tid, d, 1.0);
        if (counted) cp.mult += 1.0;
        if (tid == 0) {
            if (p.trace_lp) p.trace_lp[(int64_t)c * p.out_ld + t] = lp;
            if (p.accept_out) p.accept_out[(int64_t)c * p.out_ld + t] = acc ? 1 : 0;
            if (p.log_ratio_out) p.log_ratio_out[(int64_t)c * p.out_ld + t] = ratio;
            if (p.row_of && counted) p.row_of[(int64_t)c * p.out_ld + t] = cp.j;
        }
        if (PREF) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                xi[r] = nxi[r];
                w[r] = nw[r];
                h[r] = nh[r];
            }
        } else if (t + 1 < p.n_lag) {
            load_row(t + 1, xi, w, h);
        }
    }
    if (cp.j >= 0) store_row<R, kStepThreads>(Hc + (int64_t)cp.j * ldg, x, valid, tid, d, cp.mult);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int e = 2 * (tid + r * kStepThreads);
        if (vg[r]) {
            if (e + 1 < dg) st2(p.g + c * ldg + e, g[r]);
            else p.g[c * ldg + e] = g[r].x;
        }
        if (!valid[r]) continue;
        if (e + 1 < d) {
            st2(p.x + c * ld + e, x[r]);
            if (pcn) st2(p.y + c * ld + e, y[r]);
        } else {
            p.x[c * ld + e] = x[r].x;
            if (pcn) p.y[c * ld + e] = y[r].x;
        }
    }
    if (tid == 0) {
        p.log_pi[c] = lp;
        if (pcn) p.quad[c] = q;
        p.n_accepted[c] = nacc;
        p.uctr[c] = u0 + (uint64_t)p.n_lag;
        p.kcount[c] = cp.j + 1;
    }
}

// ---------------------------------------------------------------------------------------
// TMA-fed variant: one elected thread streams the window rows (xi_t, w_t, h_t) into an
// NS-deep shared-memory ring with cp.async.bulk (1-D TMA) and mbarrier transaction
// counts, NS-1 steps ahead of the consumers, so the step loop never waits on HBM.
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

// PRE: the parts of the candidate that only change on acceptance are kept ready --
// a = x_ref + c (x - x_ref) (the reference's exact bits), ga = G x_ref + c (G x - G x_ref) and
// cy = c y -- so a step is xc = a + xi, gc = ga + h, yc = cy + s w: 5 FP64 ops per entry
// instead of 10 (the register cost rules it out above 2 pairs per thread).
// ZREF: the reference point is the origin (p.xr == nullptr): x_ref and G x_ref are the
// constant 0 instead of registers. TWG: the twisted target's per-entry constants are read
// through L1 each step instead of held in registers (wide rows: 4 pairs per thread).
template <int R, bool TWISTED, int T, bool PRE, bool ZREF>
__global__ void __launch_bounds__(T, 1) mh_window_tma_kernel(StepParams p, int NS) {
    constexpr bool TWG = TWISTED && R >= 4;
    constexpr int NW = T / 32;
    const int c = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int d = p.d;
    const int64_t ld = p.ld;
    const bool pcn = p.pcn != 0;
    const int nrows = pcn ? 3 : 2;  // xi, h (+ w for the pCN-form y recursion)
    (void)nrows;
    const int dg = p.dg;
    const int64_t ldg = p.ldg;
    extern __shared__ __align__(128) double ring[];  // NS stages, then the log-uniform table
    __shared__ __align__(8) uint64_t full[kMaxStages];
    __shared__ __align__(16) double red[2][NW][2];
    // a stage: the xi row (ld), the h row (ldg: d + the twisted rows), the w row (ld)
    const uint32_t row_bytes = (uint32_t)(ld * sizeof(double)), hrow_bytes = (uint32_t)(ldg * sizeof(double));
    double* stage0 = ring;
    const int64_t stage_len = ld + ldg + (pcn ? ld : 0);

    const double beta = p.beta[c];
    const double cc = pcn ? sqrt(fmax(0.0, 1.0 - beta * beta)) : 1.0;  // proj/src/proposal.cpp:120
    const double sc = beta * p.infl;
    const double hq = 0.5 / (p.infl * p.infl);
    const double* Wc = p.W + c * p.win_stride;
    double* Xc = p.Xi + c * p.win_stride;
    double* Hc = p.H + c * p.hwin_stride;
    Compactor cp;

    auto issue = [&](int t, int s) {  // producer: row t of the window into stage s = t % NS
        double* st = stage0 + s * stage_len;
        mbar_expect_tx(&full[s], row_bytes * (pcn ? 2 : 1) + hrow_bytes);
        tma_row(st, Xc + (int64_t)t * ld, row_bytes, &full[s]);
        tma_row(st + ld, Hc + (int64_t)t * ldg, hrow_bytes, &full[s]);
        if (pcn) tma_row(st + ld + ldg, Wc + (int64_t)t * ld, row_bytes, &full[s]);
    };
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (tid == 0)
        for (int t = 0; t < NS && t < p.n_lag; ++t) issue(t, t);

    double2 x[R], g[R], y[R], xrv[ZREF ? 1 : R], grv[ZREF ? 1 : R], iev[TWG ? 1 : R], bcv[TWG ? 1 : R], a[R], ga[R],
        cy[R];
    bool valid[R], vg[R];  // entry pair e in x-space (e < d) / in g-space (e < dg)
    auto XR = [&](int r) -> double2 { return ZREF ? make_double2(0.0, 0.0) : xrv[ZREF ? 0 : r]; };
    auto GR = [&](int r) -> double2 { return ZREF ? make_double2(0.0, 0.0) : grv[ZREF ? 0 : r]; };
    auto IE = [&](int r) -> double2 {
        return TWG ? __ldg(reinterpret_cast<const double2*>(p.inv_eig) + tid + r * T) : iev[TWG ? 0 : r];
    };
    auto BC = [&](int r) -> double2 {
        return TWG ? __ldg(reinterpret_cast<const double2*>(p.bcoef) + tid + r * T) : bcv[TWG ? 0 : r];
    };
    // candidate parts that change only on acceptance (exact reference bits for a)
    auto refresh = [&](int r) {
        if (!PRE) return;
        const double2 xr = XR(r), gr = GR(r);
        a[r].x = __dadd_rn(xr.x, __dmul_rn(cc, __dadd_rn(x[r].x, -xr.x)));
        a[r].y = __dadd_rn(xr.y, __dmul_rn(cc, __dadd_rn(x[r].y, -xr.y)));
        ga[r].x = gr.x + cc * (g[r].x - gr.x);
        ga[r].y = gr.y + cc * (g[r].y - gr.y);
        cy[r].x = cc * y[r].x;
        cy[r].y = cc * y[r].y;
    };
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int e = 2 * (tid + r * T);
        valid[r] = e < d;
        vg[r] = e < dg;
        const double2 z2 = make_double2(0.0, 0.0);
        x[r] = valid[r] ? ld2(p.x + c * ld + e) : z2;
        g[r] = vg[r] ? ld2(p.g + c * ldg + e) : z2;
        y[r] = (valid[r] && pcn) ? ld2(p.y + c * ld + e) : z2;
        if (!ZREF) {
            xrv[ZREF ? 0 : r] = (valid[r] && p.xr) ? ld2(p.xr + c * ld + e) : z2;
            grv[ZREF ? 0 : r] = (vg[r] && p.gr) ? ld2(p.gr + c * ldg + e) : z2;
        }
        if (TWISTED && !TWG) {
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

    // one entry's candidate from the stage (xi, h, w rows): the same operations whether called
    // for the dot products or, after the decision, to adopt the candidate (bit-identical)
    auto cand = [&](const double* pxi, const double* ph, const double* pw, int r, double2& xc, double2& gc,
                    double2& yc) {
        const int e = 2 * (tid + r * T);
        const double2 xi = valid[r] ? ld2(pxi + e) : make_double2(0.0, 0.0);
        const double2 h = vg[r] ? ld2(ph + e) : make_double2(0.0, 0.0);
        // exact reference candidate (proj/src/proposal.cpp:119-124), no FMA contraction
        if (PRE) {
            xc.x = __dadd_rn(a[r].x, xi.x);
            xc.y = __dadd_rn(a[r].y, xi.y);
            gc.x = ga[r].x + h.x;
            gc.y = ga[r].y + h.y;
        } else {
            const double2 xr = XR(r), gr = GR(r);
            xc.x = __dadd_rn(__dadd_rn(xr.x, __dmul_rn(cc, __dadd_rn(x[r].x, -xr.x))), xi.x);
            xc.y = __dadd_rn(__dadd_rn(xr.y, __dmul_rn(cc, __dadd_rn(x[r].y, -xr.y))), xi.y);
            gc.x = gr.x + cc * (g[r].x - gr.x) + h.x;
            gc.y = gr.y + cc * (g[r].y - gr.y) + h.y;
        }
        if (pcn) {
            const double2 w = valid[r] ? ld2(pw + e) : make_double2(0.0, 0.0);
            if (PRE) {
                yc.x = cy[r].x + sc * w.x;
                yc.y = cy[r].y + sc * w.y;
            } else {
                yc.x = cc * y[r].x + sc * w.x;
                yc.y = cc * y[r].y + sc * w.y;
            }
        }
    };
    // With 3 or more stages a stage is refilled one step late, so an accepted candidate is
    // re-read from shared memory; with 2 (wide rows) the refill cannot wait and the accepted
    // row is re-read from global memory (row t of Xi / H is overwritten by the compaction
    // only after the adoption, j <= t)
    const bool late = NS >= 3;
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
            double2 xc, gc, yc;
            cand(st, st + ld, st + ld + ldg, r, xc, gc, yc);
            if (TWISTED) {
                // whitened form: ie w0^2 + ie' (w1^2 - bc' g1^2), w1 = g1 + bc g0^2 (upload_target)
                const double2 ie = IE(r), bc = BC(r);
                const double w0 = gc.x;
                const double w1 = gc.y + bc.x * gc.x * gc.x;
                sa0 += w0 * w0 * ie.x;
                sa1 += (w1 * w1 - bc.y * gc.y * gc.y) * ie.y;
            } else {
                sa0 += xc.x * gc.x;
                sa1 += xc.y * gc.y;
            }
            if (pcn) {
                sb0 += yc.x * yc.x;
                sb1 += yc.y * yc.y;
            }
        }
        MH_PROF(2);
        const double ws = warp_sum2(sa0 + sa1, sb0 + sb1, lane);
        const int buf = t & 1;
        if ((lane & 15) == 0) red[buf][warp][lane >> 4] = ws;
        MH_PROF(3);
        __syncthreads();
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
            for (int k = NA; k < NW; ++k) {
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
            if (cp.j >= 0) store_row<R, T>(Hc + (int64_t)cp.j * ldg, x, valid, tid, d, cp.mult);
            ++cp.j;
            cp.mult = 0.0;
        }
        if (acc) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                double2 xc, gc, yc;
                if (late) cand(st, st + ld, st + ld + ldg, r, xc, gc, yc);
                else cand(Xc + (int64_t)t * ld, Hc + (int64_t)t * ldg, Wc + (int64_t)t * ld, r, xc, gc, yc);
                x[r] = xc;
                g[r] = gc;
                if (pcn) y[r] = yc;
                refresh(r);
            }
            lp = lpc;
            q = qc;
            ++nacc;
        }
        if (fresh) store_row<R, T>(Xc + (int64_t)cp.j * ld, x, valid, tid, d, 1.0);
        if (counted) cp.mult += 1.0;
        if (tid == 0) {
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
    if (cp.j >= 0) store_row<R, T>(Hc + (int64_t)cp.j * ldg, x, valid, tid, d, cp.mult);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int e = 2 * (tid + r * T);
        if (vg[r]) {
            if (e + 1 < dg) st2(p.g + c * ldg + e, g[r]);
            else p.g[c * ldg + e] = g[r].x;
        }
        if (!valid[r]) continue;
        if (e + 1 < d) {
            st2(p.x + c * ld + e, x[r]);
            if (pcn) st2(p.y + c * ld + e, y[r]);
        } else {
            p.x[c * ld + e] = x[r].x;
            if (pcn) p.y[c * ld + e] = y[r].x;
        }
    }
    if (tid == 0) {
        p.log_pi[c] = lp;
        if (pcn) p.quad[c] = q;
        p.n_accepted[c] = nacc;
        p.uctr[c] = u0 + (uint64_t)p.n_lag;
        p.kcount[c] = cp.j + 1;
    }
}

template <int R, bool TW, int T, bool PRE = (R * T <= 512)>
bool try_tma(const StepParams& p, cudaStream_t s) {
    const size_t stage = (size_t)(p.ld * (p.pcn ? 2 : 1) + p.ldg) * sizeof(double);
    const size_t table = (size_t)p.n_lag * sizeof(double);
    constexpr size_t kMaxSmem = 220 * 1024;
    if (table + 2 * stage > kMaxSmem) return false;
    // ring depth: deep enough to hide HBM latency (>= 3 steps ahead), shallow enough that a
    // 110 KB GEMM CTA of another chain group can share the SM: the step loop leaves the DMMA
    // pipe idle, so an MH CTA that fills the SM's shared memory idles it for the whole window
    // (d=1024 pCN form: 3 rows of 8 KB per stage -> 4 stages + the log-u table = 100 KB);
    // at most kMaxStages (the mbarrier array)
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
    auto kern = p.xr ? mh_window_tma_kernel<R, TW, T, PRE, false> : mh_window_tma_kernel<R, TW, T, PRE, true>;
    set_smem_attr(reinterpret_cast<const void*>(kern), (int)smem);
    kern<<<p.chains, T, smem, s>>>(p, NS);
    return true;
}

template <bool TW>
void launch_r(const StepParams& p, cudaStream_t s) {
    const int pairs = (p.dg + 1) / 2;  // the g-space entries (d + the twisted rows) set the width
    const int R = (pairs + kStepThreads - 1) / kStepThreads;
    dim3 grid(p.chains), block(kStepThreads);
    // 256 threads (2 double2 pairs each) up to d = 1024, then 512 threads: fewer warps per
    // step barrier and reduction for the small dimensions where the step loop matters most
    // (128 threads measured slower at d = 1024)
    bool done = false;
    if (pairs <= 256) done = try_tma<1, TW, 256>(p, s);
    else if (pairs <= 512) done = try_tma<2, TW, 256>(p, s);
    else if (R <= 2) done = try_tma<2, TW, 512>(p, s);
    else if (R <= 4) done = try_tma<4, TW, 512>(p, s);
    if (done) {
        DGB_LAUNCH_CHECK();
        count_launch();
        return;
    }
    if (R <= 1) mh_window_kernel<1, TW, true><<<grid, block, 0, s>>>(p);
    else if (R <= 2) mh_window_kernel<2, TW, true><<<grid, block, 0, s>>>(p);
    else if (R <= 4) mh_window_kernel<4, TW, true><<<grid, block, 0, s>>>(p);
    else if (R <= 8) mh_window_kernel<8, TW, false><<<grid, block, 0, s>>>(p);
    else throw CudaError("mh_window: dimension above 8192 is not supported by this build");
    DGB_LAUNCH_CHECK();
    count_launch();
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

void launch_mh_window(const StepParams& p, bool twisted, cudaStream_t s) {
    if (p.chains <= 0 || p.n_lag <= 0) return;
    StepParams q = p;
    if (q.out_ld <= 0) q.out_ld = q.n_lag;
    if (twisted) launch_r<true>(q, s);
    else launch_r<false>(q, s);
}

}  // namespace dgb
