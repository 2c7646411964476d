// potrf_dag.cu — batched Cholesky as a task graph run by a persistent kernel.
//
// The launch-per-phase left-looking POTRF (linalg.cu) issues ~47 dependent launches per
// factorization at d=1024; each is small (a diagonal block per chain, a few tiles per
// chain), so most of the GPU idles while one chain group refactors, and the groups all
// refactor at about the same time. Here the factorization of every chain of a group is
// one tiled right-looking DAG over 128x128 tiles (reference algorithm:
// proj/src/linalg.cpp:74-93, left-looking column Cholesky; same factor, different
// summation order):
//   POTRF(k)     L_kk = chol(A_kk) and X_kk = L_kk^-1     (register-blocked, one CTA)
//   TRSM(i,k)    L_ik = A_ik X_kk^T                      (one DMMA tile, in place)
//   UPDATE(i,j,k) A_ij -= L_ik L_jk^T                    (one DMMA tile, lower if i == j)
// with the augmented row (x - x_ref, the usable-guard solve) as an extra 1-row block row.
// The tasks of all the group's chains are put in one order on the host (critical-path
// list scheduling), and `workers` persistent CTAs take them in that order from an
// atomic ticket counter. A CTA waits (acquire loads on per-tile counters) only for tasks
// with smaller tickets, which running CTAs already hold, so the schedule cannot
// deadlock; a spin limit turns a bug into an error instead of a hung GPU.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <queue>
#include <string>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "diag_block.cuh"
#include "diag_tc.cuh"
#include "gemm_tile.cuh"
#include "host.hpp"
#include "kernels.cuh"

namespace dgb {

namespace {

constexpr int kTb = 128;  // tile size of the task graph
// 128 x 64 half tiles, two CTAs per SM (the batched GEMM's configuration): one CTA's
// dependency wait, prologue and epilogue overlap the other's DMMA main loop
using DagTile = tile::Cfg<128, 64, 32, 2, true, true, 4, 2, 2>;
static_assert((3 * 64 * 65) * 8 + sizeof(DiagScratch) <= DagTile::SMEM_BYTES, "diag128 staging fits the ring");
enum : uint8_t { kPotrf = 0, kTrsm = 1, kUpdate = 2 };

struct DagTask {
    uint16_t c;
    uint8_t type, i, j, k, h, pad;  // h: column half of an UPDATE's 128 x 128 tile
};
static_assert(sizeof(DagTask) == 8, "task record");

struct DagArgs {
    double* const* A;
    int64_t ld;
    int d, rows, n;  // n = block columns; block row n (if rows > d) is the augmented row
    const DagTask* tasks;
    int ntasks;
    int* counter;
    int* abort_flag;
    int* flags;  // per chain: upd[(n+1) n 2] | trsm[(n+1) n] | potrf[n]
    int fstride;
    double* inv;  // per chain: n blocks of 128 x 128 (X_kk)
    const int* mask;
    int* status;
    unsigned long long* trace;  // DIAM_B200_DAG_TRACE: per ticket {grab, deps met, done} (ns)
    int tc_diag;                // diagonal tiles on the DMMA path (diag128_tc)
};

__device__ __forceinline__ unsigned long long now_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
    return t;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// true once *p >= v; false if the run was aborted (spin limit reached here or elsewhere)
__device__ bool wait_ge(const int* p, int v, int* abort_flag) {
    unsigned spins = 0;
    while (ld_acquire(p) < v) {
        if (*(volatile int*)abort_flag) return false;
        __nanosleep(64);
        if (++spins > (1u << 25)) {  // seconds: a dependency that never arrives
            atomicExch(abort_flag, 1);
            return false;
        }
    }
    return true;
}

// L = chol(A) and X = L^-1 of one diagonal tile (jb <= 128 valid rows) by the whole CTA:
// two 64x64 register-blocked diagonal factorizations (diag64_block) joined by three
// small products staged in shared memory. X is 128 x 128 row-major (ld 128), zero
// outside the lower jb x jb part. Returns nonzero on a bad pivot.
__device__ int diag128(double* A, int64_t ld, int jb, double* X, double* smem) {
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int j1 = min(kDiagNb, jb);
    constexpr int S = 65;  // padded stride of the 64 x 64 staging blocks
    // the diagonal factorizations' scratch sits after the three staging blocks: no static
    // shared memory, so two CTAs fit per SM
    DiagScratch& sc = *reinterpret_cast<DiagScratch*>(smem + 3 * 64 * S);
    if (diag64_block_sc(sc, A, ld, j1, X, 0, kTb)) return 1;
    for (int e = tid; e < 64 * 64; e += 256) X[(e >> 6) * kTb + 64 + (e & 63)] = 0.0;  // upper-right block
    if (jb <= kDiagNb) {
        for (int e = tid; e < 64 * kTb; e += 256) X[64 * kTb + e] = 0.0;
        return 0;
    }
    const int j2 = jb - kDiagNb;
    double* sX = smem;           // X11
    double* sL = sX + 64 * S;    // A21, then L21
    double* sT = sL + 64 * S;    // L21 X11
    double* sY = sX;             // X22 (X11 is no longer needed once L21 X11 is formed)
    __syncthreads();  // diag64_block's global writes of L11 / X11 are visible to the CTA
    for (int e = tid; e < 64 * 64; e += 256) {
        const int r = e >> 6, q = e & 63;
        sX[r * S + q] = __ldcg(X + r * kTb + q);
        sL[r * S + q] = r < j2 ? __ldcg(A + (int64_t)(64 + r) * ld + q) : 0.0;
    }
    __syncthreads();
    double acc[4][4];
    // L21 = A21 X11^T (X11 lower: only m <= q contributes)
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int m = 0; m < 64; ++m) {
        double ar[4], br[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) ar[a] = sL[(4 * ty + a) * S + m];
#pragma unroll
        for (int b = 0; b < 4; ++b) br[b] = sX[(4 * tx + b) * S + m];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] += ar[a] * br[b];
    }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int r = 4 * ty + a, q = 4 * tx + b;
            sL[r * S + q] = acc[a][b];
            if (r < j2) A[(int64_t)(64 + r) * ld + q] = acc[a][b];
        }
    __syncthreads();
    // A22 -= L21 L21^T on the lower triangle
    if (tx <= ty) {
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
        for (int m = 0; m < 64; ++m) {
            double ar[4], br[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) ar[a] = sL[(4 * ty + a) * S + m];
#pragma unroll
            for (int b = 0; b < 4; ++b) br[b] = sL[(4 * tx + b) * S + m];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] += ar[a] * br[b];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int r = 4 * ty + a, q = 4 * tx + b;
                if (r < j2 && q <= r) {
                    double* p = A + (int64_t)(64 + r) * ld + 64 + q;
                    *p = __ldcg(p) - acc[a][b];
                }
            }
    }
    __syncthreads();
    if (diag64_block_sc(sc, A + 64 * ld + 64, ld, j2, X + 64 * kTb + 64, 0, kTb)) return 1;
    // X21 = -X22 (L21 X11)
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int m = 0; m < 64; ++m) {  // (L21 X11)[r][q] = sum_m L21[r][m] X11[m][q]
        double ar[4], br[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) ar[a] = sL[(4 * ty + a) * S + m];
#pragma unroll
        for (int b = 0; b < 4; ++b) br[b] = sX[m * S + 4 * tx + b];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] += ar[a] * br[b];
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) sT[(4 * ty + a) * S + 4 * tx + b] = acc[a][b];
    __syncthreads();  // also: diag64_block's X22 stores are visible to the CTA
    for (int e = tid; e < 64 * 64; e += 256) {
        const int r = e >> 6, q = e & 63;
        sY[r * S + q] = __ldcg(X + (64 + r) * kTb + 64 + q);
    }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int m = 0; m < 64; ++m) {
        double ar[4], br[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) ar[a] = sY[(4 * ty + a) * S + m];
#pragma unroll
        for (int b = 0; b < 4; ++b) br[b] = sT[m * S + 4 * tx + b];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] += ar[a] * br[b];
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int r = 4 * ty + a, q = 4 * tx + b;
            X[(64 + r) * kTb + q] = r < j2 ? -acc[a][b] : 0.0;
        }
    return 0;
}

// diag128_tc (diag_tc.cuh) works in the ring
static_assert(sizeof(DiagTcScratch) + 64 * kL21S * 8 <= DagTile::SMEM_BYTES, "diag128_tc fits the ring");

__global__ void __launch_bounds__(256, 2) potrf_dag_kernel(DagArgs a) {
    extern __shared__ __align__(16) double smem[];
    __shared__ int s_task, s_state;
    const int tid = threadIdx.x;
    const int n = a.n;
    for (;;) {
        if (tid == 0) s_task = atomicAdd(a.counter, 1);
        __syncthreads();
        const int t = s_task;
        if (t >= a.ntasks) return;
        const DagTask tk = a.tasks[t];
        const int c = tk.c, ti = tk.i, tj = tk.j, tkk = tk.k, th = tk.h;
        int* upd = a.flags + (int64_t)c * a.fstride;  // [i][j][half]
        int* trsm = upd + 2 * (n + 1) * n;
        int* potrf = trsm + (n + 1) * n;
        unsigned long long t_grab = 0;
        if (tid == 0) {
            if (a.trace) t_grab = now_ns();
            // a tile column has a second 64-wide half unless it is the last, narrow one
            const bool two = min(kTb, a.d - tkk * kTb) > 64;
            bool ok;
            if (tk.type == kPotrf)
                ok = wait_ge(upd + 2 * (tkk * n + tkk), tkk, a.abort_flag) &&
                     (!two || wait_ge(upd + 2 * (tkk * n + tkk) + 1, tkk, a.abort_flag));
            else if (tk.type == kTrsm)
                ok = wait_ge(potrf + tkk, 1, a.abort_flag) && wait_ge(upd + 2 * (ti * n + tkk), tkk, a.abort_flag) &&
                     (!two || wait_ge(upd + 2 * (ti * n + tkk) + 1, tkk, a.abort_flag));
            else
                ok = wait_ge(trsm + ti * n + tkk, 1, a.abort_flag) &&
                     (ti == tj || wait_ge(trsm + tj * n + tkk, 1, a.abort_flag)) &&
                     wait_ge(upd + 2 * (ti * n + tj) + th, tkk, a.abort_flag);
            __threadfence();
            const bool live = ok && (!a.mask || a.mask[c]) && *(volatile int*)(a.status + c) == 0;
            s_state = !ok ? -1 : (live ? 1 : 0);
            if (a.trace) {
                a.trace[3 * (int64_t)t] = t_grab;
                a.trace[3 * (int64_t)t + 1] = now_ns();
            }
        }
        __syncthreads();
        const int state = s_state;
        if (state < 0) return;  // aborted: the host reports it
        if (state == 1) {
            double* A = a.A[c];
            const int k0 = tkk * kTb, kb = min(kTb, a.d - k0);
            double* X = a.inv + ((int64_t)c * n + tkk) * kTb * kTb;
            // block rows 0..n-1 hold rows [0, d); block row n is the augmented row
            const int i0 = ti < n ? ti * kTb : a.d;
            const int mrows = ti < n ? min(kTb, a.d - i0) : a.rows - a.d;
            if (tk.type == kPotrf) {
                const int bad = a.tc_diag ? diag128_tc(A + (int64_t)k0 * a.ld + k0, a.ld, kb, X, smem)
                                          : diag128(A + (int64_t)k0 * a.ld + k0, a.ld, kb, X, smem);
                if (bad && tid == 0) atomicExch(a.status + c, 1);
            } else if (tk.type == kTrsm) {
                // in place, right half first: it reads all of A_ik, the left half only
                // A_ik[:, :64] (X_kk is lower triangular)
                double* Ab = A + (int64_t)i0 * a.ld + k0;
                if (kb > 64)
                    tile::gemm_tile<DagTile, true, true>(Ab, X, Ab, a.ld, kTb, a.ld, mrows, kb, kb, 0, 64, 1.0, 0.0,
                                                         false, smem);
                tile::gemm_tile<DagTile, true, true>(Ab, X, Ab, a.ld, kTb, a.ld, mrows, kb, min(kb, 64), 0, 0, 1.0,
                                                     0.0, false, smem);
            } else {
                const int j0 = tj * kTb, jbj = min(kTb, a.d - j0);
                tile::gemm_tile<DagTile, true, true>(A + (int64_t)i0 * a.ld + k0, A + (int64_t)j0 * a.ld + k0,
                                                     A + (int64_t)i0 * a.ld + j0, a.ld, a.ld, a.ld, mrows, jbj, kb, 0,
                                                     64 * th, -1.0, 1.0, ti == tj, smem);
            }
        }
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            if (a.trace) a.trace[3 * (int64_t)t + 2] = now_ns();
            if (tk.type == kPotrf)
                st_release(potrf + tkk, 1);
            else if (tk.type == kTrsm)
                st_release(trsm + ti * n + tkk, 1);
            else
                st_release(upd + 2 * (ti * n + tj) + th, tkk + 1);
        }
    }
}

// ---------------------------------------------------------------- host: the task order
// Critical-path list scheduling over all chains (HLFET): a simulated run on `workers`
// CTAs with estimated task costs; the order in which the simulation starts tasks is the
// ticket order. Dependencies always precede their consumers, as the kernel requires.
std::vector<DagTask> build_order(int n, int aug, int d, int chains, int workers) {
    const int nr = n + aug;  // block rows
    struct Node {
        uint8_t type, i, j, k, h;
        double cost, blevel = 0.0;
        std::vector<int> succ;
        int ndeps = 0;
    };
    std::vector<Node> g;
    std::map<std::tuple<int, int, int, int, int>, int> id;
    auto halves = [&](int j) { return std::min(kTb, d - j * kTb) > 64 ? 2 : 1; };
    auto add = [&](int type, int i, int j, int k, int h, double cost) {
        id[{type, i, j, k, h}] = (int)g.size();
        g.push_back(Node{(uint8_t)type, (uint8_t)i, (uint8_t)j, (uint8_t)k, (uint8_t)h, cost});
    };
    // estimated costs (us, two CTAs per SM)
    for (int k = 0; k < n; ++k) {
        add(kPotrf, k, k, k, 0, 90.0);
        for (int i = k + 1; i < nr; ++i) add(kTrsm, i, k, k, 0, i < n ? 24.0 : 4.0);
        for (int j = k + 1; j < n; ++j)
            for (int i = j; i < nr; ++i)
                for (int h = 0; h < halves(j); ++h) add(kUpdate, i, j, k, h, i >= n ? 3.0 : (i == j ? 10.0 : 18.0));
    }
    auto edge = [&](int from, int to) {
        g[from].succ.push_back(to);
        g[to].ndeps++;
    };
    for (int k = 0; k < n; ++k) {
        const int pk = id[{kPotrf, k, k, k, 0}];
        if (k > 0)
            for (int h = 0; h < halves(k); ++h) edge(id[{kUpdate, k, k, k - 1, h}], pk);
        for (int i = k + 1; i < nr; ++i) {
            const int t = id[{kTrsm, i, k, k, 0}];
            edge(pk, t);
            if (k > 0)
                for (int h = 0; h < halves(k); ++h) edge(id[{kUpdate, i, k, k - 1, h}], t);
        }
        for (int j = k + 1; j < n; ++j)
            for (int i = j; i < nr; ++i)
                for (int h = 0; h < halves(j); ++h) {
                    const int u = id[{kUpdate, i, j, k, h}];
                    edge(id[{kTrsm, i, k, k, 0}], u);
                    if (i != j) edge(id[{kTrsm, j, k, k, 0}], u);
                    if (k > 0) edge(id[{kUpdate, i, j, k - 1, h}], u);
                }
    }
    // bottom levels: nodes were created in a topological order, so walk it backwards
    for (int v = (int)g.size() - 1; v >= 0; --v) {
        double m = 0.0;
        for (int s : g[v].succ) m = std::max(m, g[s].blevel);
        g[v].blevel = g[v].cost + m;
    }
    // simulate: ready heap by (-blevel, chain); workers free at given times
    const int V = (int)g.size();
    std::vector<int> deps((size_t)V * chains);
    std::vector<double> ready_at((size_t)V * chains, 0.0);
    for (int c = 0; c < chains; ++c)
        for (int v = 0; v < V; ++v) deps[(size_t)c * V + v] = g[v].ndeps;
    using Item = std::tuple<double, int, int>;  // (-blevel, chain, node)
    std::priority_queue<Item, std::vector<Item>, std::greater<Item>> ready;
    for (int c = 0; c < chains; ++c) ready.push({-g[0].blevel, c, 0});  // POTRF(0) of every chain
    std::priority_queue<std::pair<double, int64_t>, std::vector<std::pair<double, int64_t>>, std::greater<>> running;
    std::priority_queue<double, std::vector<double>, std::greater<double>> free_at;
    for (int w = 0; w < workers; ++w) free_at.push(0.0);
    std::vector<DagTask> order;
    order.reserve((size_t)V * chains);
    double now = 0.0;
    auto complete_until = [&](double t) {  // finish running tasks up to time t
        while (!running.empty() && running.top().first <= t) {
            const auto [ft, key] = running.top();
            running.pop();
            const int c = (int)(key / V), v = (int)(key % V);
            for (int s : g[v].succ) {
                const size_t idx = (size_t)c * V + s;
                ready_at[idx] = std::max(ready_at[idx], ft);
                if (--deps[idx] == 0) ready.push({-g[s].blevel, c, s});
            }
        }
    };
    while (order.size() < (size_t)V * chains) {
        now = std::max(now, free_at.top());
        complete_until(now);
        while (ready.empty()) {  // idle until the next completion
            now = running.top().first;
            complete_until(now);
        }
        const auto [nb, c, v] = ready.top();
        ready.pop();
        free_at.pop();
        const double start = std::max(now, ready_at[(size_t)c * V + v]);
        running.push({start + g[v].cost, (int64_t)c * V + v});
        free_at.push(start + g[v].cost);
        order.push_back(DagTask{(uint16_t)c, g[v].type, g[v].i, g[v].j, g[v].k, g[v].h, 0});
    }
    return order;
}

}  // namespace

struct DagState {
    int n = -1, aug = -1, chains = -1, workers = -1, d = -1;
    int ntasks = 0, fstride = 0;
    std::vector<DagTask> order;
    unsigned long long* trace = nullptr;
    DagTask* tasks = nullptr;
    int* flags = nullptr;  // + counter + abort at the end
    double* inv = nullptr;
    int* h_abort = nullptr;
};

void potrf_work_release(PotrfWork& w) {
    if (!w.dag) return;
    cudaFree(w.dag->tasks);
    cudaFree(w.dag->flags);
    cudaFree(w.dag->inv);
    cudaFree(w.dag->trace);
    if (w.dag->h_abort) cudaFreeHost(w.dag->h_abort);
    delete w.dag;
    w.dag = nullptr;
}

int potrf_dag_workers_default() { return kNumSMs; }

size_t potrf_dag_bytes(int d, int chains) {
    const int n = (d + kTb - 1) / kTb;
    return (size_t)chains * n * kTb * kTb * 8;
}

void potrf_dag(double* const* A, int64_t ld, int d, int chains, const int* mask, int* status, PotrfWork& w,
               cudaStream_t s, int extra_rows) {
    const int n = (d + kTb - 1) / kTb;
    const int aug = extra_rows > 0 ? 1 : 0;
    require(extra_rows <= 1 && n <= 255 && chains <= 65535, Err::InvalidArgument, "potrf_dag: unsupported shape");
    const int workers = std::max(1, w.workers > 0 ? w.workers : 2 * kNumSMs);
    if (!w.dag) w.dag = new DagState();
    DagState& st = *w.dag;
    if (st.n != n || st.d != d || st.aug != aug || st.chains != chains || st.workers != workers) {
        st.order = build_order(n, aug, d, chains, workers);
        const std::vector<DagTask>& order = st.order;
        cudaFree(st.tasks);
        cudaFree(st.flags);
        cudaFree(st.inv);
        st.ntasks = (int)order.size();
        st.fstride = 3 * (n + 1) * n + n;
        DGB_CUDA(cudaMalloc(&st.tasks, order.size() * sizeof(DagTask)));
        DGB_CUDA(cudaMemcpy(st.tasks, order.data(), order.size() * sizeof(DagTask), cudaMemcpyHostToDevice));
        DGB_CUDA(cudaMalloc(&st.flags, ((size_t)chains * st.fstride + 2) * sizeof(int)));
        DGB_CUDA(cudaMalloc(&st.inv, potrf_dag_bytes(d, chains)));
        if (!st.h_abort) DGB_CUDA(cudaMallocHost(&st.h_abort, sizeof(int)));
        st.n = n;
        st.d = d;
        st.aug = aug;
        st.chains = chains;
        st.workers = workers;
        static bool attr = false;
        if (!attr) {
            DGB_CUDA(cudaFuncSetAttribute(potrf_dag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          DagTile::SMEM_BYTES));
            attr = true;
        }
    }
    DGB_CUDA(cudaMemsetAsync(st.flags, 0, ((size_t)chains * st.fstride + 2) * sizeof(int), s));
    DagArgs a{};
    a.A = A;
    a.ld = ld;
    a.d = d;
    a.rows = d + extra_rows;
    a.n = n;
    a.tasks = st.tasks;
    a.ntasks = st.ntasks;
    a.flags = st.flags;
    a.fstride = st.fstride;
    a.counter = st.flags + (size_t)chains * st.fstride;
    a.abort_flag = a.counter + 1;
    a.inv = st.inv;
    a.mask = mask;
    a.status = status;
    {
        const char* de = std::getenv("DIAM_B200_DIAG");
        a.tc_diag = !(de && std::string(de) == "block");
    }
    static const char* trace_path = std::getenv("DIAM_B200_DAG_TRACE");  // CSV of the next launch
    if (trace_path && !st.trace) {
        DGB_CUDA(cudaMalloc(&st.trace, (size_t)st.ntasks * 3 * sizeof(unsigned long long)));
        a.trace = st.trace;
    }
    potrf_dag_kernel<<<std::min(workers, st.ntasks), 256, DagTile::SMEM_BYTES, s>>>(a);
    DGB_LAUNCH_CHECK();
    count_launch();
    // an aborted schedule (a dependency that never arrived) must not pass silently
    DGB_CUDA(cudaMemcpyAsync(st.h_abort, a.abort_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    if (a.trace) {  // one traced launch per work set: type,chain,i,j,k,grab,deps,done
        std::vector<unsigned long long> h((size_t)st.ntasks * 3);
        DGB_CUDA(cudaMemcpyAsync(h.data(), st.trace, h.size() * 8, cudaMemcpyDeviceToHost, s));
        DGB_CUDA(cudaStreamSynchronize(s));
        if (FILE* f = std::fopen(trace_path, "a")) {
            for (int t = 0; t < st.ntasks; ++t) {
                const DagTask& k = st.order[t];
                std::fprintf(f, "%d,%d,%d,%d,%d,%llu,%llu,%llu\n", k.type, k.c, k.i, k.j, k.k, h[3 * t],
                             h[3 * t + 1], h[3 * t + 2]);
            }
            std::fclose(f);
        }
    }
}

bool potrf_dag_aborted(const PotrfWork& w) { return w.dag && w.dag->h_abort && *w.dag->h_abort != 0; }

}  // namespace dgb
