// engine.cu — B200 sampler engine (see engine.hpp). Reference semantics cited inline
// (paths relative to /root/reference/proj/).
#include "engine.hpp"

#include <algorithm>
#include <chrono>
#include <set>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>

#include <nvtx3/nvToolsExt.h>

#include "gemm_f64.cuh"

namespace dgb {

std::atomic<uint64_t> g_launch_count{0};
thread_local uint64_t t_launch_count = 0;

bool sync_check_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("DIAM_B200_SYNC_CHECK");
        return e && std::atoi(e) != 0;
    }();
    return on;
}

void set_smem_attr(const void* func, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> set;  // (device, kernel) -> bytes allowed
    int dev = 0;
    DGB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    int& cur = set[{dev, func}];
    if (bytes <= cur) return;
    DGB_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    cur = bytes;
}

namespace {

// Engine buffers come from the device's stream-ordered memory pool, kept resident
// between runs (release threshold = max): a second diam_sample on the same GPU reuses
// the first one's HBM instead of paying cudaMalloc/cudaFree for gigabytes again.
void keep_pool_resident() {
    // per device (the attribute belongs to the device's default pool); engines of several
    // rank threads may get here concurrently
    static std::mutex mu;
    static std::set<int> done;
    int dev = 0;
    DGB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (done.count(dev)) return;
    cudaMemPool_t pool;
    DGB_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t keep = ~0ull;
    DGB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    done.insert(dev);
}

// While an engine is being built, allocations are zeroed on stream 0 without a sync
// each; the constructor synchronizes once before the engine's (non-blocking) streams
// touch them. Later allocations synchronize at once.
thread_local bool g_defer_alloc_sync = false;

template <class M, class T = double>
T* dalloc_impl(M& mem, size_t count) {
    if (count == 0) count = 1;
    const size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
    void* p = nullptr;
    if (mem.arena && mem.used + bytes <= mem.size) {  // carve (the arena is zeroed once)
        p = mem.arena + mem.used;
        mem.used += bytes;
        return static_cast<T*>(p);
    }
    keep_pool_resident();
    DGB_CUDA(cudaMallocAsync(&p, bytes, 0));
    DGB_CUDA(cudaMemsetAsync(p, 0, bytes, 0));
    if (!g_defer_alloc_sync) DGB_CUDA(cudaStreamSynchronize(0));
    mem.blocks.push_back(p);
    return static_cast<T*>(p);
}
template <class T, class M>
T* dalloc(M& mem, size_t count) {
    return dalloc_impl<M, T>(mem, count);
}

template <class M>
double** ptr_array(M& list, double* base, int64_t stride, int n) {
    std::vector<double*> h(n);
    for (int i = 0; i < n; ++i) h[i] = base + stride * i;
    double** d = dalloc<double*>(list, n);
    // from pageable memory: returns once h is staged, so h may go out of scope
    DGB_CUDA(cudaMemcpyAsync(d, h.data(), n * sizeof(double*), cudaMemcpyHostToDevice, 0));
    if (!g_defer_alloc_sync) DGB_CUDA(cudaStreamSynchronize(0));
    return d;
}

// Pinned host buffers are kept for the process and handed from engine to engine:
// cudaMallocHost / cudaFreeHost per run cost milliseconds to hundreds of milliseconds
// (page pinning, an implicit device synchronization) at random.
std::mutex g_pinned_mu;
std::multimap<size_t, void*> g_pinned_free;
std::map<void*, size_t> g_pinned_size;

void* pinned_acquire(size_t bytes, bool zero = true) {
    bytes = (bytes + 4095) & ~size_t(4095);
    {
        std::lock_guard<std::mutex> lk(g_pinned_mu);
        auto it = g_pinned_free.lower_bound(bytes);
        if (it != g_pinned_free.end()) {
            void* p = it->second;
            g_pinned_free.erase(it);
            if (zero) std::memset(p, 0, bytes);
            return p;
        }
    }
    void* p = nullptr;
    DGB_CUDA(cudaMallocHost(&p, bytes));
    std::memset(p, 0, bytes);
    std::lock_guard<std::mutex> lk(g_pinned_mu);  // engines of several rank threads share the maps
    g_pinned_size[p] = bytes;
    return p;
}

void pinned_release(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    const auto it = g_pinned_size.find(p);
    if (it != g_pinned_size.end()) g_pinned_free.emplace(it->second, p);
}

// Streams are kept for the process too (creating and destroying the 33 prioritised streams
// of a 16-group engine costs ~3 ms per diam_sample call); an engine returns its streams
// idle. Keyed by device and priority.
std::mutex g_stream_mu;
std::multimap<std::pair<int, int>, cudaStream_t> g_stream_free;

cudaStream_t stream_acquire(int priority) {
    int dev = 0;
    DGB_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(g_stream_mu);
        auto it = g_stream_free.find({dev, priority});
        if (it != g_stream_free.end()) {
            cudaStream_t st = it->second;
            g_stream_free.erase(it);
            return st;
        }
    }
    cudaStream_t st = nullptr;
    DGB_CUDA(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, priority));
    return st;
}

void stream_release(cudaStream_t st, int priority) {
    if (!st) return;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess) {
        cudaStreamDestroy(st);
        return;
    }
    std::lock_guard<std::mutex> lk(g_stream_mu);
    g_stream_free.emplace(std::make_pair(dev, priority), st);
}

struct DeferAllocSync {
    DeferAllocSync() { g_defer_alloc_sync = true; }
    ~DeferAllocSync() { g_defer_alloc_sync = false; }
};

// host matrix (rows x cols, row-major) -> device rows x ld
void upload_padded(double* dst, int64_t ld, const Mat& m) {
    DGB_CUDA(cudaMemcpy2D(dst, ld * sizeof(double), m.a.data(), m.cols * sizeof(double), m.cols * sizeof(double),
                          m.rows, cudaMemcpyHostToDevice));
}

}  // namespace

Engine::Engine(std::shared_ptr<const HostTarget> t, const RunCfg& cfg, std::shared_ptr<Comm> comm)
    : tgtp_(std::move(t)), tgt_(*tgtp_), cfg_(cfg), k_(cfg.kernel), comm_(std::move(comm)) {
    const auto tctor = std::chrono::steady_clock::now();
    validate_run_cfg(cfg_, tgt_);
    if (const char* e = std::getenv("DIAM_B200_TWICE")) {
        const std::string v = e;
        const char* names[] = {"normals", "trmm", "target", "mh", "syrk", "potrf"};
        for (int i = 0; i < 6; ++i)
            if (v.find(names[i]) != std::string::npos) twice_ |= 1u << i;
    }
    {
        static const bool graphs_off = [] {
            const char* e = std::getenv("DIAM_B200_GRAPHS");
            return e && std::atoi(e) == 0;
        }();
        use_graphs_ = !graphs_off && !sync_check_enabled();
    }
    if (comm_) {
        rank_ = comm_->rank();
        world_ = comm_->size();
    }
    d_ = static_cast<int>(tgt_.dim);
    Lw_ = static_cast<int>(k_.n_lag);
    P_ = static_cast<int>(cfg_.chains);
    require(P_ >= world_, Err::InvalidArgument, "fewer chains than GPUs");
    // block sharding of global chain indices: rank r owns [r P / N, (r+1) P / N)
    int64_t first = 0, count = 0;
    shard_range(P_, world_, rank_, &first, &count);
    c0_ = static_cast<int>(first);
    C_ = static_cast<int>(count);
    ld_ = pad_ld(d_);
    mat_ = (int64_t)d_ * ld_;
    fmat_ = (int64_t)(d_ + 1) * ld_;
    twisted_ = tgt_.twisted();
    require(d_ <= 8192, Err::InvalidDimension, "the B200 engine supports d <= 8192");
    {
        int T = 0;  // the twist pairs (i, i+1), b_i != 0 (proj/src/target.cpp:167-173)
        if (twisted_)
            for (size_t i = 0; i < tgt_.b_coeffs.size(); ++i)
                if (tgt_.b_coeffs[i] != 0.0) T = std::max(T, (int)i + 2);
        T = (T + 1) & ~1;
        require(d_ % 2 == 0 || T == 0, Err::InvalidDimension, "twisted targets need an even dimension");
        dg_ = d_ + T;
        ldg_ = pad_ld(dg_);
    }
    {  // the main stream (batch merge, statistics) at the highest priority: the next
       // batch's moment updates wait for it
        int least = 0, greatest = 0;
        DGB_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        stream_prio_ = greatest;
        stream_ = stream_acquire(stream_prio_);
    }
    DGB_CUDA(cudaEventCreateWithFlags(&main_ev_, cudaEventDisableTiming));
    DeferAllocSync defer;
    static const bool tinit = std::getenv("DIAM_B200_INIT_TIMING") != nullptr;  // phases to stderr
    auto t0 = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!tinit) return;
        DGB_CUDA(cudaDeviceSynchronize());
        const auto t1 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "engine init %-14s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
        t0 = t1;
    };
    if (tinit)
        std::fprintf(stderr, "engine init %-14s %8.3f ms\n", "prologue",
                     std::chrono::duration<double, std::milli>(t0 - tctor).count());
    upload_target();
    mark("upload_target");
    const int ng = plan_memory();
    {  // the arena: everything init_chains / make_groups allocate, plus slack
        size_t bytes = arena_bytes_ + ((size_t)64 << 20);
        bytes = (bytes + 255) & ~size_t(255);
        keep_pool_resident();
        void* p = nullptr;
        DGB_CUDA(cudaMallocAsync(&p, bytes, 0));
        DGB_CUDA(cudaMemsetAsync(p, 0, bytes, 0));
        allocs_.blocks.push_back(p);
        allocs_.arena = static_cast<char*>(p);
        allocs_.size = bytes;
    }
    mark("plan_memory");
    init_chains();
    mark("init_chains");
    make_groups(ng);
    DGB_CUDA(cudaStreamSynchronize(0));
    mark("make_groups");
    if (tinit)
        std::fprintf(stderr, "engine init %-14s %8.3f ms\n", "total",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tctor).count());
}

int Engine::plan_memory() {
    // chain groups on separate streams overlap one group's latency-bound pieces (MH steps,
    // diagonal factorizations) with the others' GEMMs; small problems are launch-latency
    // bound and keep one stream (DIAM_B200_GROUPS overrides, 1 = a single stream)
    // (d=1024, 64 chains, each group on a low-priority steps stream and a high-priority
    // refactor stream, 32 hardware queues: 4 groups 28.5, 8: 27.9, 12: 27.8, 16: 27.4,
    // 24: 27.4, 32: 32.0 ms per batch; neutral at d=2040 / 4096)
    int ng = d_ < 256 ? 1 : d_ >= 512 ? std::max(1, std::min(16, C_ / 4)) : (C_ >= 8 ? 2 : 1);
    const char* eg = std::getenv("DIAM_B200_GROUPS");
    if (eg) ng = std::max(1, std::min(C_, std::atoi(eg)));

    // Device bytes for a window of lc rows per chain, with or without a shared refactor
    // workspace. Free memory counts what the (resident) stream-ordered pool holds unused.
    size_t free_b = 0, total_b = 0;
    DGB_CUDA(cudaMemGetInfo(&free_b, &total_b));
    {
        int dev = 0;
        DGB_CUDA(cudaGetDevice(&dev));
        cudaMemPool_t mp;
        DGB_CUDA(cudaDeviceGetDefaultMemPool(&mp, dev));
        uint64_t reserved = 0, used = 0;
        DGB_CUDA(cudaMemPoolGetAttribute(mp, cudaMemPoolAttrReservedMemCurrent, &reserved));
        DGB_CUDA(cudaMemPoolGetAttribute(mp, cudaMemPoolAttrUsedMemCurrent, &used));
        if (reserved > used) free_b += reserved - used;
    }
    const double budget = 0.97 * (double)free_b - 1.5e9;  // context growth, NCCL, small buffers
    const double M = (double)cfg_.intervals_per_batch;
    auto need = [&](int lc, int ws_factors) {
        double n = (double)C_ * fmat_;            // factors L
        n += (double)ws_factors * fmat_;          // refactor workspace
        n += (double)C_ * mat_;                   // local moments S
        n += (double)C_ * lc * (2.0 * ld_ + ldg_);  // W, Xi, H
        if (!cfg_.checkpoint_path.empty()) n += (double)C_ * mat_;  // cumulative S
        if (k_.use_explicit_inverse) n += (double)C_ * (mat_ + (double)((d_ + 1) / 2) * ld_);  // X, TRTRI scratch
        n += 2.0 * mat_ + 3.0 * ld_;              // global snapshot, reduction buffer
        n += 3.0 * M * C_ * Lw_ + 0.5 * C_ * Lw_;  // per-batch traces, compacted-row map
        n += 16.0 * C_ * ld_ + 16400.0 * C_;      // chain vectors, POTRF inverse blocks
        return 8.0 * n;
    };
    auto gmax = [&](int groups) { return (C_ + groups - 1) / groups; };

    int lc = Lw_;
    bool pool = false;
    const char* ec = std::getenv("DIAM_B200_CHUNK");  // rows per window chunk (experiments, tests)
    const char* ep = std::getenv("DIAM_B200_POOL");   // 1: shared refactor workspace
    if (ec || ep) {
        if (ec) lc = std::max(1, std::min(Lw_, std::atoi(ec)));
        pool = ep && std::atoi(ep) != 0;
    } else if (need(Lw_, C_) > budget) {
        // 1) chunk the window (a divisor of n_lag keeps the target GEMM one matrix);
        // 2) then share one refactor workspace between the groups, which refactor in turn
        std::vector<int> divs;
        for (int c = Lw_; c >= 1; --c)
            if (Lw_ % c == 0) divs.push_back(c);
        bool found = false;
        for (int pass = 0; pass < 2 && !found; ++pass) {
            const bool pl = pass == 1;
            const int groups = pl && !eg ? std::min(8, C_) : ng;  // refactors take turns: 8 groups
            for (int c : divs) {
                if (c < (pl ? 64 : 256)) break;
                if (need(c, pl ? gmax(groups) : C_) <= budget) {
                    lc = c;
                    pool = pl;
                    ng = groups;
                    found = true;
                    break;
                }
            }
        }
        require(found, Err::InvalidArgument,
                "run does not fit in device memory: " + std::to_string(C_) + " chains of dim " + std::to_string(d_) +
                    " need " + std::to_string(need(64, gmax(std::min(8, C_))) / 1e9) + " GB, " +
                    std::to_string(std::max(0.0, budget) / 1e9) + " GB available");
    }
    Lc_ = lc;
    win_ = (int64_t)Lc_ * ld_;
    winh_ = (int64_t)Lc_ * ldg_;
    pool_ = pool && ng > 1;
    pool_n_ = pool_ ? gmax(ng) : 0;
    arena_bytes_ = (size_t)need(lc, pool_ ? pool_n_ : C_);
    return ng;
}

Engine::~Engine() {
    static const bool tinit = std::getenv("DIAM_B200_INIT_TIMING") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (tinit)
            std::fprintf(stderr, "engine free %-14s %8.3f ms\n", what,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    };
    if (stream_) cudaStreamSynchronize(stream_);
    for (auto& g : groups_) {
        if (g.potrf_exec) cudaGraphExecDestroy(g.potrf_exec);
        if (g.sr) stream_release(g.sr, g.prio_sr);
        if (g.s) stream_release(g.s, g.prio_s);
        if (g.ev_steps) cudaEventDestroy(g.ev_steps);
        if (g.ev_ref) cudaEventDestroy(g.ev_ref);
        if (g.done) cudaEventDestroy(g.done);
        if (g.pool_ev) cudaEventDestroy(g.pool_ev);
    }
    mark("streams");
    for (void* p : allocs_.blocks) cudaFreeAsync(p, 0);
    cudaStreamSynchronize(0);
    mark("buffers");
    for (auto& e : event_pool_) cudaEventDestroy(e);
    for (auto& pe : pending_) {
        cudaEventDestroy(pe.a);
        cudaEventDestroy(pe.b);
    }
    if (main_ev_) cudaEventDestroy(main_ev_);
    for (auto& g : groups_)
        if (g.status_ev) cudaEventDestroy(g.status_ev);
    pinned_release(h_flags_);
    pinned_release(h_stats_);
    pinned_release(h_out_);
    if (out_ev_) cudaEventDestroy(out_ev_);
    if (join_ev_) cudaEventDestroy(join_ev_);
    if (merge_ev_) cudaEventDestroy(merge_ev_);
    stream_release(stream_, stream_prio_);
    mark("done");
}

void Engine::upload_target() {
    auto& A = allocs_;
    // whitened form of every target: G (dg x ld) with rows 0..d-1 = a lower-triangular factor of
    // the precision P (G^T G = P, reversed Cholesky on the GPU), so that x^T P x = |G x|^2, and
    // for twisted targets rows d..d+T-1 = the first T eigenvectors (z_i = (V^T x)_i). Then
    //   log pi(x) = -1/2 [ |G x|_d^2 + sum_{i<T} (w_i^2 - z_i^2) / sigma_i^2 ],
    // w the twisted z (proj/src/target.cpp:154-173): one step formula for every target, and a
    // window target product of d(d+1) + 2dT flops per row instead of 2d^2
    G_ = dalloc<double>(A, (size_t)dg_ * ld_);
    double* prev = nullptr;
    // transient buffers from the engine's stream-ordered pool (freed with it): a plain
    // cudaMalloc/cudaFree pair here synchronised the device and let the driver trim the pool
    // the previous engine left -- 450 ms of engine construction, every other diam_sample
    prev = dalloc<double>(A, mat_);
    if (twisted_) {
        // P_rev = A_rev A_rev^T, A_rev[i][k] = V[d-1-i][k] / sigma_k
        Mat ar(d_, d_);
        for (int i = 0; i < d_; ++i)
            for (int k = 0; k < d_; ++k) ar(i, k) = tgt_.eigvecs(d_ - 1 - i, k) / std::sqrt(tgt_.eigvals[k]);
        double* dar = nullptr;
        dar = dalloc<double>(A, mat_);
        upload_padded(dar, ld_, ar);
        double** pp = nullptr;
        pp = dalloc<double*>(A, 2);
        const double* hp[2] = {dar, prev};
        DGB_CUDA(cudaMemcpy(pp, hp, sizeof(hp), cudaMemcpyHostToDevice));
        GemmBatch g{};
        g.A = (const double* const*)pp;
        g.B = (const double* const*)pp;
        g.C = pp + 1;
        g.lda = g.ldb = g.ldc = ld_;
        g.M = g.N = g.K = d_;
        g.alpha = 1.0;
        gemm_f64(g, 1, true, true, stream_);
        DGB_CUDA(cudaStreamSynchronize(stream_));

    } else {
        Mat rev(d_, d_);
        for (int i = 0; i < d_; ++i)
            for (int j = 0; j < d_; ++j) rev(i, j) = tgt_.precision(d_ - 1 - i, d_ - 1 - j);
        upload_padded(prev, ld_, rev);
    }
    whitening_factor(prev, G_, d_, ld_, stream_);
    const int T = dg_ - d_;
    std::vector<double> ie(ldg_, 0.0), bc(ldg_, 0.0);
    for (int i = 0; i < d_; ++i) ie[i] = 1.0;
    if (T > 0) {
        Mat vt(T, d_);  // rows d.. of G: V^T
        for (int i = 0; i < T; ++i)
            for (int k = 0; k < d_; ++k) vt(i, k) = tgt_.eigvecs(k, i);
        upload_padded(G_ + (size_t)d_ * ld_, ld_, vt);
        // pair (d + i, d + i + 1), i even: w_{i+1} = z_{i+1} + b_i z_i^2 contributes
        // (w_{i+1}^2 - z_{i+1}^2) / sigma_{i+1}^2; w_i = z_i contributes nothing
        for (int i = 0; i < T; i += 2) {
            bc[d_ + i] = tgt_.b_coeffs[i];
            ie[d_ + i + 1] = 1.0 / tgt_.eigvals[i + 1];
            bc[d_ + i + 1] = 1.0;  // subtract z_{i+1}^2 (its Gaussian term is inside |G x|^2)
        }
    }
    inv_eig_ = dalloc<double>(A, ldg_);
    bcoef_ = dalloc<double>(A, ldg_);
    DGB_CUDA(cudaMemcpy(inv_eig_, ie.data(), ldg_ * 8, cudaMemcpyHostToDevice));
    DGB_CUDA(cudaMemcpy(bcoef_, bc.data(), ldg_ * 8, cudaMemcpyHostToDevice));
    tri_target_ = true;
    // G^-1 (accepted increments xi = G^-1 h, the x-space snapshot), G G^T (the jitter of the
    // whitened covariance: G (C + eps I) G^T = C_z + eps G G^T) and, for twisted targets,
    // B_T = V_T^T G^-1 (the twisted coordinates of an increment from its whitened h)
    Ginv_ = dalloc<double>(A, mat_);
    GG_ = dalloc<double>(A, mat_);
    {
        double** pa = ptr_array(A, G_, 0, 1);
        Ginvp_ = ptr_array(A, Ginv_, 0, 1);
        double* tscr = nullptr;
        tscr = dalloc<double>(A, (size_t)((d_ + 1) / 2) * ld_);
        double** tp = nullptr;
        tp = dalloc<double*>(A, 1);
        DGB_CUDA(cudaMemcpy(tp, &tscr, sizeof(double*), cudaMemcpyHostToDevice));
        trtri_batched(pa, Ginvp_, tp, ld_, d_, 1, nullptr, stream_);
        GemmBatch gg{};
        gg.A = (const double* const*)pa;
        gg.B = (const double* const*)pa;
        gg.C = ptr_array(A, GG_, 0, 1);
        gg.lda = gg.ldb = gg.ldc = ld_;
        gg.M = gg.N = gg.K = d_;
        gg.alpha = 1.0;
        gg.tri_b_lower = 1;
        gg.tri_c_lower = 1;
        gemm_f64(gg, 1, true, true, stream_);
        if (T > 0) {
            BT_ = dalloc<double>(A, (size_t)T * ld_);
            GemmBatch b{};
            b.A = (const double* const*)ptr_array(A, G_ + (size_t)d_ * ld_, 0, 1);
            b.B = (const double* const*)Ginvp_;
            b.C = ptr_array(A, BT_, 0, 1);
            b.lda = b.ldb = b.ldc = ld_;
            b.M = T;
            b.N = d_;
            b.K = d_;
            b.alpha = 1.0;
            gemm_f64(b, 1, true, false, stream_);
        }
        DGB_CUDA(cudaStreamSynchronize(stream_));

    }
    Ct_ = dalloc<double>(A, (size_t)d_ * d_);
    DGB_CUDA(cudaMemcpy(Ct_, tgt_.covariance.a.data(), (size_t)d_ * d_ * 8, cudaMemcpyHostToDevice));
    std::vector<double> pj(2 * ld_, 0.0);
    for (int i = 0; i < d_; ++i) {
        pj[i] = tgt_.eigvecs(i, 0);
        pj[ld_ + i] = tgt_.eigvecs(i, d_ - 1);
    }
    tmean_ = dalloc<double>(A, ld_);
    DGB_CUDA(cudaMemcpy(tmean_, tgt_.mean.data(), d_ * 8, cudaMemcpyHostToDevice));
    dstats_ = dalloc<double>(A, 4);
    h_stats_ = static_cast<double*>(pinned_acquire(4 * sizeof(double)));
    proj_ = dalloc<double>(A, 2 * ld_);
    DGB_CUDA(cudaMemcpy(proj_, pj.data(), 2 * ld_ * 8, cudaMemcpyHostToDevice));
    Gp_ = ptr_array(A, G_, 0, 1);
}

void Engine::init_chains() {
    auto& A = allocs_;
    const int C = C_;
    L_ = dalloc<double>(A, (size_t)C * fmat_);
    const int nws = pool_ ? pool_n_ : C;  // refactor workspace factors
    Lw2_ = dalloc<double>(A, (size_t)nws * fmat_);
    S_ = dalloc<double>(A, (size_t)C * mat_);
    W_ = dalloc<double>(A, (size_t)C * win_);
    Xi_ = dalloc<double>(A, (size_t)C * win_);
    H_ = dalloc<double>(A, (size_t)C * winh_);
    x_ = dalloc<double>(A, (size_t)C * ld_);
    g_ = dalloc<double>(A, (size_t)C * ldg_);
    y_ = dalloc<double>(A, (size_t)C * ld_);
    xr_ = dalloc<double>(A, (size_t)C * ld_);
    gr_ = dalloc<double>(A, (size_t)C * ldg_);
    mean_ = dalloc<double>(A, (size_t)C * ld_);
    cmean_ = dalloc<double>(A, (size_t)C * ld_);
    cdiag_ = dalloc<double>(A, (size_t)C * ld_);
    mb_ = dalloc<double>(A, (size_t)C * ld_);
    logpi_ = dalloc<double>(A, C);
    quad_ = dalloc<double>(A, C);
    beta_ = dalloc<double>(A, C);
    tr_ = dalloc<double>(A, C);
    qtmp_ = dalloc<double>(A, C);
    nacc_ = dalloc<uint64_t>(A, C);
    uctr_ = dalloc<uint64_t>(A, C);
    status_ = dalloc<int>(A, C);
    try_ = dalloc<int>(A, C);
    usable_ = dalloc<int>(A, C);
    mask_ = dalloc<int>(A, C);
    h_flags_ = static_cast<int*>(pinned_acquire(3 * (size_t)C * sizeof(int)));
    Sg_ = dalloc<double>(A, mat_);
    mg_ = dalloc<double>(A, ld_);
    Ssum_ = dalloc<double>(A, (size_t)d_ * (d_ + 1) / 2 + 2 * ld_);  // packed lower sum, z mean, x mean
    cov_part_ = dalloc<double>(A, 2 * (size_t)d_);
    if (!cfg_.checkpoint_path.empty()) cS_ = dalloc<double>(A, (size_t)C * mat_);
    if (k_.use_explicit_inverse) {
        Xinv_ = dalloc<double>(A, (size_t)C * mat_);
        Tinv_ = dalloc<double>(A, (size_t)C * ((d_ + 1) / 2) * ld_);
    }
    mean_x_ = dalloc<double>(A, (size_t)C * ld_);
    diag_x_ = dalloc<double>(A, (size_t)C * ld_);
    Sgz_ = dalloc<double>(A, mat_);
    mgz_ = dalloc<double>(A, ld_);
    Sfull_ = dalloc<double>(A, mat_);
    Stmp_ = dalloc<double>(A, mat_);
    state_src_ = dalloc<int>(A, (size_t)C * Lw_);
    state_mult_ = dalloc<int>(A, (size_t)C * Lw_);
    acc_cnt_ = dalloc<int>(A, C);
    const size_t M = cfg_.intervals_per_batch;
    trace_lp_ = dalloc<double>(A, M * C * Lw_);
    kcount_ = dalloc<int>(A, C);
    row_of_ = dalloc<int>(A, (size_t)C * Lw_);
    trace_pj_ = dalloc<double>(A, M * C * Lw_ * 2);
    hist_rate_ = dalloc<double>(A, M * C);
    hist_beta_ = dalloc<double>(A, M * C);

    Lp_ = ptr_array(A, L_, fmat_, C);
    Lnp_ = ptr_array(A, Lw2_, fmat_, nws);
    Wp_ = ptr_array(A, W_, win_, C);
    Xip_ = ptr_array(A, Xi_, win_, C);
    Hp_ = ptr_array(A, H_, winh_, C);
    Gpc_ = ptr_array(A, G_, 0, C);  // G once per chain (batched GEMMs)
    Ginvpc_ = ptr_array(A, Ginv_, 0, C);
    ptr_gen_ = ptr_array(A, Sfull_, 0, 3);
    ptr_tmp_[0] = ptr_array(A, Sfull_, 0, 1);
    ptr_tmp_[1] = ptr_array(A, Stmp_, 0, 1);
    ptr_tmp_[2] = ptr_array(A, Sg_, 0, 1);
    if (BT_) BTpc_ = ptr_array(A, BT_, 0, C);
    Sp_ = ptr_array(A, S_, mat_, C);
    if (Xinv_) {
        Xinvp_ = ptr_array(A, Xinv_, mat_, C);
        Tinvp_ = ptr_array(A, Tinv_, ((d_ + 1) / 2) * ld_, C);
    }

    // RNG keys: global chain index p = c0 + i (runner.cpp:128-130, 556-559)
    std::vector<PhiloxKey> nk(C), uk(C), ik(C);
    for (int i = 0; i < C; ++i) {
        const uint64_t p = (uint64_t)(c0_ + i);
        nk[i] = make_philox_key(cfg_.master_seed, p, "noise");
        uk[i] = make_philox_key(cfg_.master_seed, p, "uniform");
        ik[i] = make_philox_key(cfg_.master_seed, p, "init");
    }
    nkeys_ = dalloc<PhiloxKey>(A, C);
    ukeys_ = dalloc<PhiloxKey>(A, C);
    ikeys_ = dalloc<PhiloxKey>(A, C);
    DGB_CUDA(cudaMemcpy(nkeys_, nk.data(), C * sizeof(PhiloxKey), cudaMemcpyHostToDevice));
    DGB_CUDA(cudaMemcpy(ukeys_, uk.data(), C * sizeof(PhiloxKey), cudaMemcpyHostToDevice));
    DGB_CUDA(cudaMemcpy(ikeys_, ik.data(), C * sizeof(PhiloxKey), cudaMemcpyHostToDevice));

    DGB_CUDA(cudaStreamSynchronize(0));  // the buffers above are zeroed before stream_ uses them
    // x0 = dispersion * N(0, I) from the "init" stream (runner.cpp:131-132)
    launch_normal_vec(x_, ld_, C, d_, ikeys_, 0, cfg_.init_dispersion, stream_);
    // factor = I, beta = beta_init (proposal.cpp:95-97): in whitened space L_z = G I = G, and the
    // explicit inverse L_z^-1 = G^-1
    for (int c = 0; c < C; ++c) {
        DGB_CUDA(cudaMemcpyAsync(L_ + (size_t)c * fmat_, G_, (size_t)mat_ * 8, cudaMemcpyDeviceToDevice, stream_));
        if (Xinv_)
            DGB_CUDA(cudaMemcpyAsync(Xinv_ + (size_t)c * mat_, Ginv_, (size_t)mat_ * 8, cudaMemcpyDeviceToDevice,
                                     stream_));
    }
    std::vector<double> b(C, k_.beta_init);
    DGB_CUDA(cudaMemcpyAsync(beta_, b.data(), C * 8, cudaMemcpyHostToDevice, stream_));
    identity_ = false;
    // log pi(x0), quad(x0) (proposal.cpp:107-108); with the identity factor y = x - 0 exactly
    refresh_g(x_, g_, C, stream_);
    launch_eval_logpi(g_, inv_eig_, bcoef_, logpi_, C, dg_, ldg_, stream_);  // whitened form
    if (k_.pcn_form()) {
        const double infl = k_.noise_infl();
        launch_init_yq(x_, ld_, y_, quad_, C, d_, 0.5 / (infl * infl), stream_);
    }
    DGB_CUDA(cudaStreamSynchronize(stream_));

    // functionals (runner.cpp:292-309)
    fnames_ = {"log_density"};
    if (cfg_.trace_eigen_projections) {
        fnames_.push_back("proj_min");
        fnames_.push_back("proj_max");
    }
    beta_hist_.assign(C, {});
    acc_hist_.assign(C, {});
    traces_.assign(C, std::vector<std::vector<double>>(fnames_.size()));
}

void Engine::make_groups(int n) {
    auto& A = allocs_;
    groups_.resize(n);
    for (int i = 0; i < n; ++i) {
        Group& g = groups_[i];
        g.off = (int)((int64_t)C_ * i / n);
        g.C = (int)((int64_t)C_ * (i + 1) / n) - g.off;
        {
            // steps at the lowest priority, the refactorization at the highest: the
            // latency-bound POTRF launches of one group are scheduled ahead of the other
            // groups' GEMM tiles
            int least = 0, greatest = 0;
            DGB_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
            g.s = stream_acquire(least);
            g.prio_s = least;
            g.sr = stream_acquire(greatest);
            g.prio_sr = greatest;
            DGB_CUDA(cudaEventCreateWithFlags(&g.ev_steps, cudaEventDisableTiming));
            DGB_CUDA(cudaEventCreateWithFlags(&g.ev_ref, cudaEventDisableTiming));
        }
        DGB_CUDA(cudaEventCreateWithFlags(&g.done, cudaEventDisableTiming));
        DGB_CUDA(cudaEventCreateWithFlags(&g.status_ev, cudaEventDisableTiming));
        DGB_CUDA(cudaEventCreateWithFlags(&g.pool_ev, cudaEventDisableTiming));
        g.Lp = Lp_ + g.off;
        // pool mode: every group factors into the same workspace (slot i <-> the group's
        // chain i); accepted factors swap pointers with their slot as before
        g.Lnp = pool_ ? Lnp_ : Lnp_ + g.off;
        g.Wp = Wp_ + g.off;
        g.Xip = Xip_ + g.off;
        g.Sp = Sp_ + g.off;
        g.Xib = ptr_array(A, Xi_ + g.off * win_, 0, 1);
        g.Hb = ptr_array(A, H_ + g.off * winh_, 0, 1);
        // per-group inverse-block scratch (+ int active[C] tail): groups factor concurrently
        g.pw.inv = dalloc<double>(A, potrf_work_doubles(g.C));
        g.pw.inv128_ptrs = ptr_array(A, g.pw.inv, 128 * 128, g.C);
    }
}

void Engine::refresh_g(const double* x, double* out, int chains, cudaStream_t s) {
    // out = x G^T: G x for every chain of the group (rows of stride ld)
    timed_begin(s);
    launch_gemv_rows(G_, ld_, d_, dg_, x, out, ldg_, chains, s);
    timed_end("gemv_state", 2.0 * chains * (double)d_ * dg_, s);
}

void Engine::gemm(const char* name, const GemmBatch& g, int batch, bool ak, bool bk, cudaStream_t s, double flops,
                  bool small) {
    if (flops < 0.0) {
        flops = 2.0 * g.M * (double)g.N * g.K * batch;
        if (g.tri_c_lower) flops *= 0.5 * (1.0 + 1.0 / std::max(1, g.N));
        if (g.tri_b_lower) flops *= 0.5 * (1.0 + 1.0 / std::max(1, g.N));
    }
    nvtxRangePushA(name);  // `ncu --nvtx --nvtx-include "<name>/"` selects one GEMM class
    timed_begin(s);
    if (small) gemm_f64_small(g, batch, s);
    else gemm_f64(g, batch, ak, bk, s);
    timed_end(name, flops, s);
    nvtxRangePop();
}

void Engine::timed_begin(cudaStream_t s) {
    if (!profiling_) return;
    if (event_pool_.size() < 2) {
        for (int i = 0; i < 64; ++i) {
            cudaEvent_t e;
            DGB_CUDA(cudaEventCreate(&e));
            event_pool_.push_back(e);
        }
    }
    cudaEvent_t a = event_pool_.back();
    event_pool_.pop_back();
    DGB_CUDA(cudaEventRecord(a, s));
    open_[s] = a;
}

void Engine::timed_end(const char* name, double flops, cudaStream_t s) {
    if (!profiling_) return;
    cudaEvent_t b = event_pool_.back();
    event_pool_.pop_back();
    DGB_CUDA(cudaEventRecord(b, s));
    pending_.push_back({name, open_.at(s), b, flops, s});
    if (pending_.size() > 4096) resolve_events();
}

void Engine::resolve_events() {
    if (pending_.empty()) return;
    DGB_CUDA(cudaDeviceSynchronize());
    static const char* tl_path = std::getenv("DIAM_B200_TIMELINE");  // CSV: name,stream,start_ms,end_ms
    FILE* tl = nullptr;
    if (tl_path && timeline_base_) tl = std::fopen(tl_path, "a");
    for (auto& p : pending_) {
        float ms = 0.f;
        DGB_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
        auto& st = stats_[p.name];
        st.ms += ms;
        st.flops += p.flops;
        st.launches += 1;
        if (tl) {
            float t0 = 0.f;
            DGB_CUDA(cudaEventElapsedTime(&t0, timeline_base_, p.a));
            std::fprintf(tl, "%s,%p,%.4f,%.4f\n", p.name.c_str(), (void*)p.s, t0, t0 + ms);
        }
        event_pool_.push_back(p.a);
        event_pool_.push_back(p.b);
    }
    if (tl) std::fclose(tl);
    pending_.clear();
}

const std::map<std::string, KernelStat>& Engine::stats() {
    resolve_events();
    return stats_;
}

double Engine::flops_per_batch() const {
    // algorithmic FP64 flops of one batch over the local chains, upper bound:
    // the window product H = s W L_z^T d(d+1) per row, the twisted rows 2dT, the SYRK d(d+1)
    // and the accepted increments d(d+1) per row if every step were accepted (bench.py counts
    // the rows they actually ran over), POTRF d^3/3 per window
    const double d = d_, L = Lw_, C = C_, M = (double)cfg_.intervals_per_batch;
    const double per_row = d * (d + 1) + 2.0 * d * (dg_ - d_) + 2.0 * d * (d + 1);
    return M * C * (L * per_row + d * d * d / 3.0);
}

void Engine::fork_groups() {
    DGB_CUDA(cudaEventRecord(main_ev_, stream_));
    for (auto& g : groups_) DGB_CUDA(cudaStreamWaitEvent(g.s, main_ev_, 0));
}

void Engine::join_groups() {
    for (auto& g : groups_) {
        DGB_CUDA(cudaEventRecord(g.done, g.s));
        DGB_CUDA(cudaStreamWaitEvent(stream_, g.done, 0));
    }
}

Engine::WindowPlan Engine::plan_window(size_t w, bool record) const {
    WindowPlan p;
    p.w = w;
    p.record = record;
    p.n_start = n_;
    p.n_end = n_ + Lw_;
    p.nctr = nctr_;
    p.identity = identity_;
    // post-burn-in rows: step t counts iff n_start + t + 1 > n0 (proposal.cpp:153-155)
    p.first = (int)std::clamp<int64_t>((int64_t)k_.n0 - (int64_t)p.n_start, 0, Lw_);
    p.k = Lw_ - p.first;
    p.cnt_before = cnt_local_;
    p.cnt_after = cnt_local_ + (uint64_t)p.k;
    const bool wants = k_.adapts_cov() || k_.adaptive_ref;
    if (wants && p.n_end >= k_.n0) {  // proposal.cpp:174-209, with counts after this window
        const uint64_t count = p.cnt_after + cnt_g_;
        p.wg = count ? (double)cnt_g_ / (double)count : 0.0;
        p.wl = count ? (double)p.cnt_after / (double)count : 1.0;
        p.refactor = k_.adapts_cov() && count >= 2;
        p.move_ref = k_.adaptive_ref && p.n_end >= k_.n_ref_start && count > 0;
    }
    return p;
}

void Engine::commit_window(const WindowPlan& p) {
    n_ = p.n_end;
    nctr_ += (uint64_t)Lw_ * d_;
    cnt_local_ = p.cnt_after;
    window_n_start_[p.w] = p.n_start;
    if (p.refactor) identity_ = false;
}

void Engine::run_batch_windows(bool record) {
    const size_t M = cfg_.intervals_per_batch;
    std::vector<WindowPlan> plans;
    plans.reserve(M);
    auto next_plan = [&](size_t m) {
        plans.push_back(plan_window(m, record));
        commit_window(plans.back());
    };
    if (capture_) {
        // parity capture: strictly ordered windows and groups (W is copied chunk by chunk)
        for (size_t m = 0; m < M; ++m) {
            next_plan(m);
            for (auto& g : groups_) {
                enqueue_head(g, plans[m]);
                enqueue_tail(g, plans[m]);
            }
            capture_window(m);
        }
        return;
    }
    if (pool_) {
        // shared refactor workspace: group g refactors after group g-1's tail released the
        // workspace, so g's refactor is enqueued after that tail; the other groups' steps
        // keep the GPU busy meanwhile
        next_plan(0);
        for (auto& g : groups_) enqueue_steps(g, plans[0]);
        for (size_t m = 0; m < M; ++m) {
            if (m + 1 < M) next_plan(m + 1);
            for (auto& g : groups_) {
                enqueue_refactor(g, plans[m]);
                enqueue_tail(g, plans[m]);
                if (m + 1 < M) enqueue_steps(g, plans[m + 1]);
            }
        }
        return;
    }
    // software pipeline over groups: while the host reads group g's POTRF statuses for
    // window m, the other group's kernels keep the GPU busy; g's next head follows at once.
    // Groups whose factorization needs the jitter ladder are set aside and stepped
    // together, so their retries run concurrently instead of one group after another.
    // (Measured and dropped: staggering the groups' start by half a window, and drawing
    // the next window's noise on a side stream during the refactorization -- neither
    // beat this plain order at d=1024 or d=4096.)
    begin_windows(record);
    end_windows();
}

void Engine::begin_windows(bool record) {
    const size_t M = cfg_.intervals_per_batch;
    bplans_.clear();
    bplans_.reserve(M);
    for (size_t m = 0; m < M; ++m) {
        bplans_.push_back(plan_window(m, record));
        commit_window(bplans_.back());
    }
    for (auto& g : groups_) enqueue_head(g, bplans_[0]);
}

void Engine::end_windows() {
    const size_t M = cfg_.intervals_per_batch;
    const std::vector<WindowPlan>& plans = bplans_;
    std::vector<Ladder> lad(groups_.size());
    for (size_t m = 0; m < M; ++m) {
        std::vector<size_t> pending;
        // groups in the order their factorizations finish (polled), not in index order: a
        // group whose refactor is done gets its next window at once
        std::vector<size_t> todo(groups_.size());
        for (size_t i = 0; i < todo.size(); ++i) todo[i] = i;
        while (!todo.empty()) {
            const auto tw0 = std::chrono::steady_clock::now();
            const size_t before = todo.size();
            for (auto it = todo.begin(); it != todo.end();) {
                const size_t i = *it;
                if (plans[m].refactor) {
                    const cudaError_t q = cudaEventQuery(groups_[i].status_ev);
                    if (q == cudaErrorNotReady) {
                        ++it;
                        continue;
                    }
                    DGB_CUDA(q);
                }
                it = todo.erase(it);
                if (!tail_begin(groups_[i], plans[m], lad[i])) {
                    pending.push_back(i);
                    continue;
                }
                tail_finish(groups_[i], plans[m]);
                if (m + 1 < M) enqueue_head(groups_[i], plans[m + 1]);
            }
            if (todo.size() == before)  // a pass with nothing ready: the host waited
                host_wait_s_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - tw0).count();
        }
        while (!pending.empty()) {
            std::vector<size_t> still;
            for (size_t i : pending) {
                if (!tail_step(groups_[i], plans[m], lad[i])) {
                    still.push_back(i);
                    continue;
                }
                tail_finish(groups_[i], plans[m]);
                if (m + 1 < M) enqueue_head(groups_[i], plans[m + 1]);
            }
            pending.swap(still);
        }
    }
}

void Engine::enqueue_steps(Group& g, const WindowPlan& p) {
    for (int r0 = 0; r0 < Lw_; r0 += Lc_) enqueue_chunk(g, p, r0, std::min(Lc_, Lw_ - r0));
    // ---- lag update (proposal.cpp:159-216): beta from the window's acceptance rate
    const int o = g.off;
    launch_beta_update(beta_ + o, nacc_ + o, hist_rate_ + p.w * C_ + o, hist_beta_ + p.w * C_ + o, g.C, Lw_,
                       k_.adapt_beta ? 1 : 0, k_.band_lo, k_.band_hi, k_.beta_adapt_factor, k_.beta_min, k_.beta_max,
                       g.s);
}

// Rows [r0, r0 + rows) of the window: noise, target GEMM, the MH steps, and the moments
// of the chunk's post-burn-in states. The step recursion's state (x, G x, y, log pi,
// counters) lives in global memory, so consecutive chunks continue one another exactly;
// only the running-average moment update is split at chunk boundaries (rounding).
void Engine::enqueue_chunk(Group& g, const WindowPlan& p, int r0, int rows) {
    const int C = g.C, o = g.off;
    const cudaStream_t s = g.s;
    const double infl = k_.noise_infl();
    // ---- noise (proposal.cpp:254-266): W from Philox, row r of the window drawing counters
    // nctr + r d .. nctr + (r + 1) d - 1 of the chain's stream; then H = s W L_z^T, i.e.
    // h_t = G xi_t with xi_t = s L w_t: the factor is kept in whitened space (L_z = G L), so
    // this one triangular product gives the target's coordinates of every increment
    timed_begin(s);
    for (int rep = (twice_ & kTwiceNormals) ? 2 : 1; rep > 0; --rep)
        launch_normals(W_ + o * win_, nullptr, win_, C, rows, d_, ld_, nkeys_ + o, p.nctr + (uint64_t)r0 * d_,
                       beta_ + o, infl, s);
    timed_end("normals", 0.0, s);
    {
        GemmBatch t{};
        t.A = (const double* const*)g.Wp;
        t.B = (const double* const*)g.Lp;
        t.C = Hp_ + o;
        t.lda = ld_;
        t.ldb = ld_;
        t.ldc = ldg_;
        t.M = rows;
        t.N = d_;
        t.K = d_;
        t.alpha = 1.0;
        t.alpha_vec = beta_ + o;
        t.alpha_vec_mul = infl;
        t.beta = 0.0;
        t.tri_b_lower = 1;
        gemm("trmm_noise", t, C, true, true, s);
        if (twice_ & kTwiceTrmm) gemm("trmm_noise", t, C, true, true, s);
    }
    if (BT_) {
        // twisted targets: the T twisted coordinates of each increment, V_T^T xi = B_T h
        // (B_T = V_T^T G^-1), into columns d.. of the H rows
        GemmBatch b{};
        b.A = (const double* const*)(Hp_ + o);
        b.B = (const double* const*)(BTpc_ + o);
        b.C = Hp_ + o;
        b.c_off = d_;
        b.lda = ldg_;
        b.ldb = ld_;
        b.ldc = ldg_;
        b.M = rows;
        b.N = dg_ - d_;
        b.K = d_;
        b.alpha = 1.0;
        gemm("gemm_target", b, C, true, true, s);
        if (twice_ & kTwiceTarget) gemm("gemm_target", b, C, true, true, s);
    }
    // parity capture: W before the steps reuse its consumed rows
    if (capture_) capture_chunk(g, r0, rows);

    // ---- the chunk's MH steps (proposal.cpp:137-157, runner.cpp:363-368), in whitened space
    StepParams sp{};
    sp.d = d_;
    sp.n_lag = rows;
    sp.out_ld = Lw_;
    sp.chains = C;
    sp.ld = ld_;
    sp.win_stride = win_;
    sp.W = W_ + o * win_;
    sp.Xi = Xi_ + o * win_;
    sp.H = H_ + o * winh_;
    sp.dg = dg_;
    sp.ldg = ldg_;
    sp.hwin_stride = winh_;
    sp.g = g_ + o * ldg_;
    sp.y = y_ + o * ld_;
    sp.gr = k_.adaptive_ref ? gr_ + o * ldg_ : nullptr;
    sp.log_pi = logpi_ + o;
    sp.quad = quad_ + o;
    sp.beta = beta_ + o;
    sp.n_accepted = nacc_ + o;
    sp.ukeys = ukeys_ + o;
    sp.uctr = uctr_ + o;
    sp.infl = infl;
    sp.pcn = k_.pcn_form() ? 1 : 0;
    sp.inv_eig = inv_eig_;
    sp.bcoef = bcoef_;
    sp.trace_lp = p.record ? trace_lp_ + (p.w * C_ + o) * (size_t)Lw_ + r0 : nullptr;
    sp.accept_out = capture_ ? dbg_acc_ + (size_t)o * Lw_ + r0 : nullptr;
    sp.log_ratio_out = capture_ ? dbg_ratio_ + (size_t)o * Lw_ + r0 : nullptr;
    // post-burn-in rows: window rows t >= first count (proj/src/proposal.cpp:153-155), so the
    // chunk holds rows [lf, rows) after cb earlier samples
    const int lf = std::clamp(p.first - r0, 0, rows);
    const int kc = rows - lf;
    const uint64_t cb = p.cnt_before + (uint64_t)std::max(0, r0 - p.first);
    const bool project = p.record && cfg_.trace_eigen_projections;
    sp.first = lf;
    sp.kcount = kcount_ + o;
    sp.acc_count = acc_cnt_ + o;
    sp.state_src = state_src_ + (size_t)o * Lw_;
    sp.state_mult = state_mult_ + (size_t)o * Lw_;
    sp.row_of = project ? row_of_ + (size_t)o * Lw_ + r0 : nullptr;
    // the previous batch's trace copies read the buffers the MH steps write
    if (merge_pending_ && p.record) DGB_CUDA(cudaStreamWaitEvent(s, merge_ev_, 0));
    timed_begin(s);
    launch_mh_window(sp, s);
    timed_end("mh_window", 0.0, s);

    // ---- moments of the chunk's counted states (proposal.cpp:153-155, moments.cpp:5-20) in
    // whitened space: the MH kernel compacted them into kcount_c distinct states z_j (rows of W)
    // and their weighted copies m_j z_j (rows of H), so S_z <- (cb S_z + sum_j m_j z_j z_j^T)
    // / (cb + kc) is a SYRK over about acceptance x kc rows instead of kc
    // the merge reads S_ / mean_ and clears mean_; the histories' copies read hist_*
    if (merge_pending_) DGB_CUDA(cudaStreamWaitEvent(s, merge_ev_, 0));
    auto device_count = [&](const int* v) {  // profiling: the rows a data-dependent GEMM ran over
        std::vector<int> h(C);
        DGB_CUDA(cudaStreamSynchronize(s));
        DGB_CUDA(cudaMemcpy(h.data(), v, C * sizeof(int), cudaMemcpyDeviceToHost));
        double n = 0.0;
        for (int x : h) n += x;
        return n;
    };
    if (kc > 0) {
        const double total = (double)(cb + (uint64_t)kc);
        GemmBatch m{};
        m.A = (const double* const*)(Hp_ + o);
        m.B = (const double* const*)g.Wp;
        m.C = g.Sp;
        m.lda = ldg_;
        m.ldb = ld_;
        m.ldc = ld_;
        m.M = d_;
        m.N = d_;
        m.K = kc;
        m.k_vec = kcount_ + o;
        m.alpha = 1.0 / total;
        m.beta = (double)cb / total;
        m.tri_c_lower = 1;
        const double fl = profiling_ ? device_count(kcount_ + o) * d_ * (d_ + 1.0) : -1.0;
        gemm("syrk_moments", m, C, false, false, s, fl);
    }
    // ---- the chunk's x-space states: xi_k = G^-1 h_k for its accepted steps only (rows of Xi
    // into rows of H), then the reference's exact recursion x <- x_ref + c (x - x_ref) + xi_k
    {
        GemmBatch a{};
        a.A = (const double* const*)g.Xip;
        a.B = (const double* const*)(Ginvpc_ + o);
        a.C = Hp_ + o;
        a.lda = ld_;
        a.ldb = ld_;
        a.ldc = ldg_;
        a.M = rows;
        a.m_vec = acc_cnt_ + o;
        a.N = d_;
        a.K = d_;
        a.alpha = 1.0;
        a.tri_b_lower = 1;
        const double fl = profiling_ ? device_count(acc_cnt_ + o) * d_ * (d_ + 1.0) : -1.0;
        // 64-row tiles: a chain's accepted rows (about acceptance x n_lag, ~50 at the d=1024
        // bench) fill one such tile, where a 128-row tile would leave half its warps idle
        gemm("xi_accepted", a, C, true, true, s, fl, true);
        timed_begin(s);
        launch_reconstruct(x_ + o * ld_, k_.adaptive_ref ? xr_ + o * ld_ : nullptr, beta_ + o, k_.pcn_form() ? 1 : 0,
                           H_ + o * winh_, winh_, ldg_, Xi_ + o * win_, win_, ld_, state_src_ + (size_t)o * Lw_,
                           state_mult_ + (size_t)o * Lw_, Lw_, kcount_ + o, acc_cnt_ + o, mean_x_ + o * ld_,
                           diag_x_ + o * ld_, (double)cb, kc, C, d_, W_ + o * win_, win_, mean_ + o * ld_, s);
        timed_end("reconstruct", 0.0, s);
    }
    if (project)
        launch_project_rows(Xi_ + o * win_, win_, ld_, C, rows, lf, d_, proj_,
                            trace_pj_ + ((p.w * C_ + o) * (size_t)Lw_ + r0) * 2, Lw_, row_of_ + (size_t)o * Lw_ + r0,
                            s);
}

// The group's first attempt at a window's factorization. Its ~3 launches per 128-wide block
// column take the same arguments every window (device pointer arrays, the group's masks and
// workspace), so from the second window on they run as one CUDA graph captured on the
// refactor stream: one host call instead of 22 (d=1024), and graph-internal dependencies
// instead of stream ones. (The jitter ladder's retries, with their own masks, launch directly.)
void Engine::factor(Group& g, cudaStream_t s, bool aug) {
    const int C = g.C, o = g.off;
    if (!use_graphs_ || g.potrf_calls++ == 0) {  // the first call also sets kernel attributes
        potrf_batched(g.Lnp, ld_, d_, C, try_ + o, status_ + o, g.pw, s, aug ? 1 : 0);
        return;
    }
    if (!g.potrf_exec) {
        cudaGraph_t graph = nullptr;
        DGB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        const uint64_t n0 = t_launch_count;
        try {
            potrf_batched(g.Lnp, ld_, d_, C, try_ + o, status_ + o, g.pw, s, aug ? 1 : 0);
        } catch (...) {  // leave the stream out of capture mode before reporting
            cudaStreamEndCapture(s, &graph);
            if (graph) cudaGraphDestroy(graph);
            throw;
        }
        g.potrf_nodes = t_launch_count - n0;
        DGB_CUDA(cudaStreamEndCapture(s, &graph));
        g_launch_count.fetch_sub(g.potrf_nodes, std::memory_order_relaxed);  // recorded, not launched
        t_launch_count -= g.potrf_nodes;
        DGB_CUDA(cudaGraphInstantiate(&g.potrf_exec, graph, 0));
        DGB_CUDA(cudaGraphDestroy(graph));
    }
    DGB_CUDA(cudaGraphLaunch(g.potrf_exec, s));
    count_launch(g.potrf_nodes);
}

void Engine::enqueue_refactor(Group& g, const WindowPlan& p) {
    const int C = g.C, o = g.off;
    const cudaStream_t s = g.sr;
    // the refactor stream continues after the window's steps
    DGB_CUDA(cudaEventRecord(g.ev_steps, g.s));
    DGB_CUDA(cudaStreamWaitEvent(g.sr, g.ev_steps, 0));
    // g = G x re-anchored from the reconstructed x-space state at every boundary (the steps
    // carry g by recursion); the augmented row, the quad and the next window start from it
    refresh_g(x_ + o * ld_, g_ + o * ldg_, C, s);
    if (p.refactor) {
        // blend -> covariance into the workspace factor, trace floor, POTRF (proposal.cpp:176-184),
        // in whitened space: C_z = G C G^T from the whitened moments, so the factor is L_z = G L;
        // the trace floor and the blended mean (adaptive reference) from the x-space statistics.
        // pCN-form kernels append r = z - z_ref (the whitened x - x_ref) as row d: the
        // factorization then also delivers L_z'^{-1} r = L'^{-1} (x - x_ref) for the usable guard.
        const bool aug = k_.pcn_form();
        const double* ax = aug ? g_ + o * ldg_ : nullptr;
        const double* axr = aug && k_.adaptive_ref ? gr_ + o * ldg_ : nullptr;
        // shared workspace: wait until the previous group's tail has released it
        if (pool_ && pool_last_) DGB_CUDA(cudaStreamWaitEvent(s, pool_last_, 0));
        // one launch: the z-space covariance (and augmented row) plus, per chain, the x-space
        // trace floor (tr, try, the blended mean mb) and the status reset
        const TraceX tx{Sg_, mg_, diag_x_ + o * ld_, mean_x_ + o * ld_, mb_ + o * ld_, tr_ + o, try_ + o, status_ + o};
        auto blend = [&] {
            launch_blend_cov(g.Lnp, Sgz_, mgz_, S_ + o * mat_, mat_, mean_ + o * ld_, ld_, p.wg, p.wl, nullptr, ld_, C,
                             d_, ld_, nullptr, 0.0, nullptr, GG_, s, ax, axr, ldg_, &tx);
        };
        timed_begin(s);
        blend();
        timed_end("blend_cov", 0.0, s);
        nvtxRangePushA("potrf");
        timed_begin(s);
        factor(g, s, aug);
        if (twice_ & kTwicePotrf) {  // blend + factorization again: same inputs, same factor
            blend();
            factor(g, s, aug);
        }
        timed_end("potrf", (double)C * d_ * (double)d_ * d_ / 3.0, s);
        nvtxRangePop();
        DGB_CUDA(cudaMemcpyAsync(h_flags_ + o, status_ + o, C * sizeof(int), cudaMemcpyDeviceToHost, s));
        DGB_CUDA(cudaMemcpyAsync(h_flags_ + C_ + o, try_ + o, C * sizeof(int), cudaMemcpyDeviceToHost, s));
        DGB_CUDA(cudaEventRecord(g.status_ev, s));
    }
}

void Engine::enqueue_tail(Group& g, const WindowPlan& p) {
    Ladder st;
    if (!tail_begin(g, p, st))
        while (!tail_step(g, p, st)) {
        }
    tail_finish(g, p);
}

// Jitter escalation for chains whose factorization failed (proposal.cpp:218-239):
// eps = 1e-10, 1e-8, 1e-6, 9.999e-5 -- the reference's floating loop -- with the same
// blocked POTRF restricted to the failing chains. tail_begin reads the first attempt's
// statuses; each tail_step reads one retry's and enqueues the next; true = every tried
// chain of the group has factored.
bool Engine::tail_begin(Group& g, const WindowPlan& p, Ladder& st) {
    if (!p.refactor) return true;
    const int C = g.C, o = g.off;
    const auto tw0 = std::chrono::steady_clock::now();
    DGB_CUDA(cudaEventSynchronize(g.status_ev));
    host_wait_s_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - tw0).count();
    st.failing.assign(C, 0);
    bool any = false;
    for (int c = 0; c < C; ++c) {
        st.failing[c] = h_flags_[C_ + o + c] && h_flags_[o + c];
        any |= st.failing[c] != 0;
    }
    if (!any) return true;
    st.eps = 1e-10;
    ladder_retry(g, p, st);
    return false;
}

bool Engine::tail_step(Group& g, const WindowPlan& p, Ladder& st) {
    const int C = g.C, o = g.off;
    DGB_CUDA(cudaEventSynchronize(g.status_ev));
    bool any = false;
    for (int c = 0; c < C; ++c) {
        if (st.failing[c] && !h_flags_[o + c]) st.failing[c] = 0;
        any |= st.failing[c] != 0;
    }
    if (!any) return true;
    st.eps *= 100.0;
    if (st.eps > 1e-4) {
        int c = 0;
        while (!st.failing[c]) ++c;
        double trh = 0.0;
        DGB_CUDA(cudaMemcpy(&trh, tr_ + o + c, 8, cudaMemcpyDeviceToHost));
        fail(Err::NotPositiveDefinite, "chain " + std::to_string(c0_ + o + c) +
                                           ": covariance not factorizable after jitter escalation (dim " +
                                           std::to_string(d_) + ", trace " + std::to_string(trh) + ")");
    }
    ladder_retry(g, p, st);
    return false;
}

void Engine::ladder_retry(Group& g, const WindowPlan& p, Ladder& st) {
    const int C = g.C, o = g.off;
    const cudaStream_t s = g.sr;
    const bool aug = k_.pcn_form();
    const double* ax = aug ? g_ + o * ldg_ : nullptr;
    const double* axr = aug && k_.adaptive_ref ? gr_ + o * ldg_ : nullptr;
    // mask through the pinned status mirror's third block (the copy is stream-ordered)
    int* hm = h_flags_ + 2 * C_ + o;
    std::copy(st.failing.begin(), st.failing.end(), hm);
    DGB_CUDA(cudaMemcpyAsync(mask_ + o, hm, C * sizeof(int), cudaMemcpyHostToDevice, s));
    // C_z + eps (tr / d) G G^T = G (C + eps (tr / d) I) G^T: the reference's jitter, whitened
    launch_blend_cov(g.Lnp, Sgz_, mgz_, S_ + o * mat_, mat_, mean_ + o * ld_, ld_, p.wg, p.wl, nullptr, ld_, C, d_,
                     ld_, mask_ + o, st.eps, tr_ + o, GG_, s, ax, axr, ldg_);
    DGB_CUDA(cudaMemsetAsync(status_ + o, 0, C * sizeof(int), s));
    potrf_batched(g.Lnp, ld_, d_, C, mask_ + o, status_ + o, g.pw, s, aug ? 1 : 0);
    DGB_CUDA(cudaMemcpyAsync(h_flags_ + o, status_ + o, C * sizeof(int), cudaMemcpyDeviceToHost, s));
    DGB_CUDA(cudaEventRecord(g.status_ev, s));
}

void Engine::tail_finish(Group& g, const WindowPlan& p) {
    const int C = g.C, o = g.off;
    const cudaStream_t s = g.sr;
    const double infl = k_.noise_infl();
    if (p.refactor) {
        const bool aug = k_.pcn_form();
        // every tried chain has factored by now. Usable guard (pCN forms, proposal.cpp:185-199):
        // 1/2 |L'^-1 (x - x_ref)|^2 / infl^2 <= 5 d, L'^-1 (x - x_ref) being the augmented row
        // the POTRF just solved; adopted factors come with y = that row and the quad term for
        // free when the reference point is fixed and no explicit inverse is kept
        const bool adopt_y = aug && !Xinv_ && !k_.adaptive_ref;
        launch_adopt_factor(g.Lp, g.Lnp, ld_, d_, C, try_ + o, status_ + o, aug ? 0.5 / (infl * infl) : -1.0,
                            aug ? 5.0 * d_ : -1.0, usable_ + o, adopt_y ? y_ + o * ld_ : nullptr,
                            adopt_y ? quad_ + o : nullptr, s);
        if (pool_) {  // the shared workspace is free for the next group
            DGB_CUDA(cudaEventRecord(g.pool_ev, s));
            pool_last_ = g.pool_ev;
        }
        // explicit inverse: X = L^{-1} of every adopted factor (proposal.cpp:202)
        if (Xinv_) trtri_batched(g.Lp, Xinvp_ + o, Tinvp_ + o, ld_, d_, C, usable_ + o, s);
    }
    // adaptive reference point (proposal.cpp:206-208)
    if (p.move_ref) {
        if (!p.refactor) launch_blend_mean(mg_, mean_x_ + o * ld_, p.wg, p.wl, mb_ + o * ld_, C, d_, ld_, s);
        DGB_CUDA(cudaMemcpyAsync(xr_ + o * ld_, mb_ + o * ld_, (size_t)C * ld_ * 8, cudaMemcpyDeviceToDevice, s));
        refresh_g(xr_ + o * ld_, gr_ + o * ldg_, C, s);
    }
    // quad with the current factor (proposal.cpp:211) and y for the next window's recursion.
    // With a fixed reference point y = L^-1 (x - x_ref) is carried exactly through the
    // steps (c y + s w) and re-anchored from the augmented POTRF row whenever the factor
    // changes, so only a moving reference point needs a fresh triangular solve.
    // In whitened coordinates: L^-1 (x - x_ref) = L_z^-1 (z - z_ref), z = G x.
    if (k_.pcn_form() && Xinv_) {
        // the reference's quad_term through factor_inv (tri_matvec, proposal.cpp:55) at every
        // boundary, whether or not the factor changed (X_z = L_z^-1)
        launch_trmv_quad(Xinvp_ + o, ld_, g_ + o * ldg_, k_.adaptive_ref ? gr_ + o * ldg_ : nullptr, ldg_,
                         y_ + o * ld_, ld_, quad_ + o, C, d_, 0.5 / (infl * infl), s);
    } else if (k_.pcn_form() && k_.adaptive_ref) {
        timed_begin(s);
        launch_trsv(g.Lp, ld_, g_ + o * ldg_, gr_ + o * ldg_, ldg_, y_ + o * ld_, ld_, quad_ + o, C, d_,
                    0.5 / (infl * infl), nullptr, s);
        timed_end("trsv", 0.0, s);
    }
    // the next window's steps follow the tail
    DGB_CUDA(cudaEventRecord(g.ev_ref, g.sr));
    DGB_CUDA(cudaStreamWaitEvent(g.s, g.ev_ref, 0));
}

void Engine::capture_chunk(const Group& g, int r0, int rows) {
    // parity-test capture: the chunk's W rows of the group's chains, before the next
    // chunk overwrites them
    DGB_CUDA(cudaStreamSynchronize(g.s));
    if (cap_wbuf_.empty()) cap_wbuf_.assign((size_t)C_ * Lw_ * d_, 0.0);
    for (int c = 0; c < g.C; ++c)
        DGB_CUDA(cudaMemcpy2D(cap_wbuf_.data() + ((size_t)(g.off + c) * Lw_ + r0) * d_, (size_t)d_ * 8,
                              W_ + (g.off + c) * win_, (size_t)ld_ * 8, (size_t)d_ * 8, rows,
                              cudaMemcpyDeviceToHost));
}

void Engine::capture_window(size_t) {
    // parity-test capture: the window's W (captured chunk by chunk) and the step records
    DGB_CUDA(cudaDeviceSynchronize());
    const int C = C_;
    if (cap_w_.empty()) {
        cap_w_.assign(C, {});
        cap_ratio_.assign(C, {});
        cap_acc_.assign(C, {});
    }
    std::vector<double> r((size_t)C * Lw_);
    std::vector<uint8_t> a((size_t)C * Lw_);
    DGB_CUDA(cudaMemcpy(r.data(), dbg_ratio_, r.size() * 8, cudaMemcpyDeviceToHost));
    DGB_CUDA(cudaMemcpy(a.data(), dbg_acc_, a.size(), cudaMemcpyDeviceToHost));
    for (int c = 0; c < C; ++c) {
        cap_w_[c].insert(cap_w_[c].end(), cap_wbuf_.begin() + (size_t)c * Lw_ * d_,
                         cap_wbuf_.begin() + (size_t)(c + 1) * Lw_ * d_);
        cap_ratio_[c].insert(cap_ratio_[c].end(), r.begin() + (size_t)c * Lw_, r.begin() + (size_t)(c + 1) * Lw_);
        cap_acc_[c].insert(cap_acc_[c].end(), a.begin() + (size_t)c * Lw_, a.begin() + (size_t)(c + 1) * Lw_);
    }
}

void Engine::merge_batch() {
    // proj/src/moments.cpp:51-88 with the P-chain sum pooled across GPUs: each GPU sums its
    // chains' packed lower triangles and means, one all-reduce (sum) of d(d+1)/2 + d doubles
    // over NVLink, and every rank applies the merge weights to its replica of the snapshot
    const uint64_t incoming = (uint64_t)P_ * cnt_local_;
    if (incoming > 0) {
        double keep = 1.0, wp = 0.0;
        merge_weights(cnt_g_, (uint64_t)P_, cnt_local_, &keep, &wp);
        // whitened packed S_z and mean m_z (the blend's snapshot), the x-space mean and raw
        // diagonal (the reported snapshot's mean, the trace floor); one all-reduce
        const int64_t tri = (int64_t)d_ * (d_ + 1) / 2;
        timed_begin(stream_);
        launch_sum_chains_lower(Ssum_, S_, mat_, C_, d_, ld_, stream_);
        launch_sum_chains(Ssum_ + tri, mean_, ld_, C_, ld_, 1.0, stream_);
        launch_sum_chains(Ssum_ + tri + ld_, mean_x_, ld_, C_, ld_, 1.0, stream_);
        if (comm_) comm_->allreduce_sum(Ssum_, tri + 2 * ld_, stream_);
        launch_merge_lower(Sgz_, ld_, Ssum_, d_, keep, wp, stream_);
        launch_axpby(mgz_, Ssum_ + tri, ld_, wp, keep, stream_);
        launch_axpby(mg_, Ssum_ + tri + ld_, ld_, wp, keep, stream_);
        update_x_snapshot();  // Sg_ = G^-1 Sgz_ G^-T
        timed_end("merge", 0.0, stream_);
        cnt_g_ += incoming;
        const double ct = (double)(cum_cnt_ + cnt_local_);
        launch_cum_fold(cmean_, cdiag_, mean_x_, diag_x_, ld_, C_, d_, ld_, (double)cum_cnt_ / ct,
                        (double)cnt_local_ / ct, stream_);
        // full cumulative second moments only when they must be checkpointed (merge_into,
        // proj/src/moments.cpp:77-88); the PSRF needs just the diagonal kept above
        if (cS_) launch_axpby(cS_, S_, (int64_t)C_ * mat_, (double)cnt_local_ / ct, (double)cum_cnt_ / ct, stream_);
        cum_cnt_ += cnt_local_;
    }
    // S_ needs no clearing (C x d^2 doubles, ~0.1 ms at d=1024): the batch's first moment
    // update runs with weight cb/total = 0 on the old value, which the GEMM then never reads
    // (beta = 0), and nothing reads S_ with a nonzero weight before that update
    DGB_CUDA(cudaMemsetAsync(mean_, 0, (size_t)C_ * ld_ * 8, stream_));
    DGB_CUDA(cudaMemsetAsync(mean_x_, 0, (size_t)C_ * ld_ * 8, stream_));
    DGB_CUDA(cudaMemsetAsync(diag_x_, 0, (size_t)C_ * ld_ * 8, stream_));
    cnt_local_ = 0;
}

void Engine::update_x_snapshot() {
    // the reported snapshot from the whitened one: Sg_ = G^-1 Sgz_ G^-T (raw second moments
    // transform by congruence; mg_ is merged directly). Sgz_ holds the lower triangle: mirrored
    // into Sfull_, then Stmp_ = Sfull_ G^-T and Sg_ = lower(G^-1 Stmp_)
    launch_mirror_lower(Sgz_, Sfull_, d_, ld_, stream_);
    GemmBatch a{};
    a.A = (const double* const*)ptr_tmp_[0];
    a.B = (const double* const*)Ginvp_;
    a.C = ptr_tmp_[1];
    a.lda = a.ldb = a.ldc = ld_;
    a.M = a.N = a.K = d_;
    a.alpha = 1.0;
    a.tri_b_lower = 1;
    gemm_f64(a, 1, true, true, stream_);
    GemmBatch b{};
    b.A = (const double* const*)Ginvp_;
    b.B = (const double* const*)ptr_tmp_[1];
    b.C = ptr_tmp_[2];
    b.lda = b.ldb = b.ldc = ld_;
    b.M = b.N = b.K = d_;
    b.alpha = 1.0;
    b.tri_c_lower = 1;
    gemm_f64(b, 1, true, false, stream_);
}

void Engine::collect_histories(size_t windows, const std::vector<uint64_t>& n_start, const double* rate,
                               const double* beta, const double* lp, const double* pj) {
    const int C = C_;
    for (size_t w = 0; w < windows; ++w)
        for (int c = 0; c < C; ++c) {
            beta_hist_[c].push_back(beta[w * C + c]);
            acc_hist_[c].push_back(rate[w * C + c]);
        }
    if (!cfg_.record_traces) return;
    for (size_t w = 0; w < windows; ++w) {
        const uint64_t ns = n_start[w];
        for (int t = 0; t < Lw_; ++t) {
            const uint64_t n = ns + t + 1;
            if (!(n > k_.n0 && (n - k_.n0 - 1) % cfg_.trace_thin == 0)) continue;
            for (int c = 0; c < C; ++c) {
                const size_t idx = (w * C + c) * (size_t)Lw_ + t;
                traces_[c][0].push_back(lp[idx]);
                if (cfg_.trace_eigen_projections) {
                    traces_[c][1].push_back(pj[idx * 2]);
                    traces_[c][2].push_back(pj[idx * 2 + 1]);
                }
            }
        }
    }
}

void Engine::enqueue_batch_outputs(size_t windows) {
    // The batch statistics (cov / mean error from the merged snapshot, the PSRF over every
    // chain's cumulative mean and diagonal) on the device, and every per-batch output's copy
    // into pinned memory, in stream order; read_batch_outputs waits for them. With several
    // ranks the PSRF inputs are all-gathered first (device to device, stream-ordered) and
    // compacted into global chain order, so the statistics kernel sums over the same chains
    // in the same order as a one-GPU run (runner.cpp:249-256, 381-396).
    const int C = C_;
    const size_t mc = windows * C, tr = cfg_.record_traces ? mc * (size_t)Lw_ : 0;
    if (!h_out_) {
        h_out_ = static_cast<double*>(pinned_acquire((2 * mc + 3 * tr + 1) * sizeof(double), false));
        DGB_CUDA(cudaEventCreateWithFlags(&out_ev_, cudaEventDisableTiming));
    }
    const bool want_err = cnt_g_ >= 2, want_psrf = P_ >= 2 && cum_cnt_ >= 2;
    if (want_err) launch_cov_error(Sg_, mg_, Ct_, d_, ld_, cov_part_, stream_);
    const double* cm = cmean_;
    const double* cd = cdiag_;
    if (comm_ && want_psrf) {
        const int64_t maxc = (P_ + world_ - 1) / world_, blk = 2 * maxc * ld_;
        if (!gather_) gather_ = dalloc<double>(allocs_, (size_t)blk * (world_ + 1) + 2 * (size_t)P_ * ld_);
        double* src = gather_;
        double* dst = gather_ + blk;
        double* all = dst + blk * world_;  // P x ld cumulative means, then P x ld diagonals
        DGB_CUDA(cudaMemcpyAsync(src, cmean_, (size_t)C_ * ld_ * 8, cudaMemcpyDeviceToDevice, stream_));
        DGB_CUDA(cudaMemcpyAsync(src + maxc * ld_, cdiag_, (size_t)C_ * ld_ * 8, cudaMemcpyDeviceToDevice, stream_));
        comm_->allgather(src, dst, blk, stream_);
        for (int r = 0; r < world_; ++r) {
            int64_t f = 0, cr = 0;
            shard_range(P_, world_, r, &f, &cr);
            DGB_CUDA(cudaMemcpyAsync(all + f * ld_, dst + r * blk, (size_t)cr * ld_ * 8, cudaMemcpyDeviceToDevice,
                                     stream_));
            DGB_CUDA(cudaMemcpyAsync(all + (P_ + f) * ld_, dst + r * blk + maxc * ld_, (size_t)cr * ld_ * 8,
                                     cudaMemcpyDeviceToDevice, stream_));
        }
        cm = all;
        cd = all + (int64_t)P_ * ld_;
    }
    launch_batch_stats(cov_part_, mg_, tmean_, d_, cm, cd, ld_, comm_ ? P_ : C_, cum_cnt_, want_err, want_psrf,
                       dstats_, stream_);
    DGB_CUDA(cudaMemcpyAsync(h_stats_, dstats_, 4 * sizeof(double), cudaMemcpyDeviceToHost, stream_));
    DGB_CUDA(cudaMemcpyAsync(h_out_, hist_rate_, mc * 8, cudaMemcpyDeviceToHost, stream_));
    DGB_CUDA(cudaMemcpyAsync(h_out_ + mc, hist_beta_, mc * 8, cudaMemcpyDeviceToHost, stream_));
    if (tr) {
        DGB_CUDA(cudaMemcpyAsync(h_out_ + 2 * mc, trace_lp_, tr * 8, cudaMemcpyDeviceToHost, stream_));
        if (cfg_.trace_eigen_projections)
            DGB_CUDA(cudaMemcpyAsync(h_out_ + 2 * mc + tr, trace_pj_, 2 * tr * 8, cudaMemcpyDeviceToHost, stream_));
    }
    DGB_CUDA(cudaEventRecord(out_ev_, stream_));
    out_n_start_ = window_n_start_;  // the next batch's plans overwrite window_n_start_
}

void Engine::read_batch_outputs(size_t windows, double& cov_err, double& mean_err, double& psrf) {
    const size_t mc = windows * C_, tr = cfg_.record_traces ? mc * (size_t)Lw_ : 0;
    DGB_CUDA(cudaEventSynchronize(out_ev_));
    require(!((int)h_stats_[3] & 1), Err::InvalidArgument, "cov_error: zero reference norm");
    cov_err = h_stats_[0];
    mean_err = h_stats_[1];
    psrf = h_stats_[2];
    collect_histories(windows, out_n_start_, h_out_, h_out_ + mc, h_out_ + 2 * mc, h_out_ + 2 * mc + tr);
}

double Engine::run_batches_timed(int k) {
    const size_t M = cfg_.intervals_per_batch;
    window_n_start_.assign(M, 0);
    cudaEvent_t a, b;
    DGB_CUDA(cudaEventCreate(&a));
    DGB_CUDA(cudaEventCreate(&b));
    DGB_CUDA(cudaDeviceSynchronize());
    DGB_CUDA(cudaEventRecord(a, stream_));
    const auto th0 = std::chrono::steady_clock::now();
    host_wait_s_ = 0.0;
    if (profiling_) {
        resolve_events();
        if (!timeline_base_) DGB_CUDA(cudaEventCreate(&timeline_base_));
        DGB_CUDA(cudaEventRecord(timeline_base_, stream_));
    }
    // as the pipelined run loop: batch i + 1's first windows start at batch i's join
    const bool early = !capture_ && !pool_;
    if (early && !join_ev_) {
        DGB_CUDA(cudaEventCreateWithFlags(&join_ev_, cudaEventDisableTiming));
        DGB_CUDA(cudaEventCreateWithFlags(&merge_ev_, cudaEventDisableTiming));
    }
    for (int i = 0; i < k; ++i) {
        if (early && i > 0) {
            for (auto& g : groups_) DGB_CUDA(cudaStreamWaitEvent(g.s, join_ev_, 0));
            merge_pending_ = true;
            begin_windows(false);
            merge_pending_ = false;
            end_windows();
        } else {
            fork_groups();
            run_batch_windows(false);
        }
        join_groups();
        if (early) DGB_CUDA(cudaEventRecord(join_ev_, stream_));
        merge_batch();
        // the batch statistics and the history copies of a diam_sample batch (the host reads
        // nothing here)
        enqueue_batch_outputs(M);
        if (early) DGB_CUDA(cudaEventRecord(merge_ev_, stream_));
        ++batches_done_;
    }
    DGB_CUDA(cudaEventRecord(b, stream_));
    {  // host time to enqueue the k batches, and how much of it was spent waiting on the GPU
        const double enq = std::chrono::duration<double>(std::chrono::steady_clock::now() - th0).count();
        stats_["host_enqueue"].ms += 1e3 * enq;
        stats_["host_enqueue"].launches += k;
        stats_["host_wait"].ms += 1e3 * host_wait_s_;
    }
    DGB_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    DGB_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms;
}

RunResult Engine::run() {  // runner.cpp:216-279
    const auto t0 = std::chrono::steady_clock::now();
    // wall time includes earlier segments of a resumed run (runner.cpp:217-218)
    auto elapsed = [&] {
        return wall_accum_ + std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    };
    const size_t M = cfg_.intervals_per_batch;
    window_n_start_.assign(M, 0);
    if (capture_ && !dbg_ratio_) {
        dbg_ratio_ = dalloc<double>(allocs_, (size_t)C_ * Lw_);
        dbg_acc_ = dalloc<uint8_t>(allocs_, (size_t)C_ * Lw_);
    }
    // Pipelined when no rule needs a batch's statistics or state before the next batch may
    // start (no tolerance, wall-clock limit or checkpoint): the next batch's first windows
    // are enqueued before the host waits for this batch's outputs, so the GPU does not idle
    // while the host reads them. Otherwise batch by batch, as runner.cpp:216-279.
    const bool pipelined = !capture_ && !pool_ && cfg_.checkpoint_path.empty() && !cfg_.max_wall_seconds &&
                           !cfg_.psrf_tol && !cfg_.cov_tol && !cfg_.mean_tol;
    auto cap_reason = [&](size_t done) -> const char* {  // loop-top rules known without the GPU
        const uint64_t iters = (uint64_t)P_ * M * done * k_.n_lag;
        if (cfg_.max_samples && iters >= *cfg_.max_samples) return "max_samples";
        if (done >= cfg_.max_batches) return "batch_cap";
        return nullptr;
    };
    // Several ranks: every decision to leave the loop is collective. The wall-clock rule is
    // OR-ed over the ranks at the top of each batch (each rank reads its own clock), and a
    // rank-local failure (jitter ladder exhausted, a launch error) is announced to the others
    // at the point where they check, right before the merge's all-reduce, so every rank
    // throws instead of waiting in a collective the failed rank never joins.
    bool announced = false;  // this rank's failure has been announced
    auto check_peers = [&] {
        if (comm_ && comm_->any(false, stream_)) {
            announced = true;  // the others know already
            fail(Err::Unknown, "sampling failed on another rank (rank " + std::to_string(rank_) + " stops too)");
        }
    };
    bool head_queued = false;  // the next batch's plans and first windows are enqueued
    std::string reason;
    try {
        for (;;) {
            if (const char* cr = cap_reason(batches_done_)) {
                reason = cr;
                break;
            }
            if (cfg_.max_wall_seconds) {
                bool stop = elapsed() >= *cfg_.max_wall_seconds;
                if (comm_) stop = comm_->any(stop, stream_);
                if (stop) {
                    reason = "wall_time";
                    break;
                }
            }
            const auto b0 = std::chrono::steady_clock::now();
            double ce, me, ps;
            if (pipelined) {
                if (!head_queued) {
                    fork_groups();
                    begin_windows(cfg_.record_traces);
                }
                end_windows();
                join_groups();
                if (!join_ev_) {
                    DGB_CUDA(cudaEventCreateWithFlags(&join_ev_, cudaEventDisableTiming));
                    DGB_CUDA(cudaEventCreateWithFlags(&merge_ev_, cudaEventDisableTiming));
                }
                DGB_CUDA(cudaEventRecord(join_ev_, stream_));
                check_peers();
                merge_batch();
                enqueue_batch_outputs(M);
                DGB_CUDA(cudaEventRecord(merge_ev_, stream_));
                ++batches_done_;
                head_queued = cap_reason(batches_done_) == nullptr;
                if (head_queued) {
                    // the next batch's first windows start at the join, not after the merge
                    for (auto& g : groups_) DGB_CUDA(cudaStreamWaitEvent(g.s, join_ev_, 0));
                    merge_pending_ = true;
                    begin_windows(cfg_.record_traces);
                    merge_pending_ = false;
                }
                read_batch_outputs(M, ce, me, ps);
            } else {
                fork_groups();
                run_batch_windows(cfg_.record_traces);
                join_groups();
                check_peers();
                merge_batch();
                enqueue_batch_outputs(M);
                ++batches_done_;
                read_batch_outputs(M, ce, me, ps);
            }
            batch_seconds_.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - b0).count());
            cov_hist_.push_back(ce);
            mean_hist_.push_back(me);
            psrf_hist_.push_back(ps);
            if (!cfg_.checkpoint_path.empty()) save_checkpoint(elapsed());  // runner.cpp:259
            // the tolerance rules read statistics that are identical on every rank (the
            // snapshot is all-reduced, the PSRF inputs all-gathered): no exchange needed
            if (cfg_.psrf_tol && std::isfinite(ps) && ps <= *cfg_.psrf_tol) {
                reason = "psrf";
                break;
            }
            if (cfg_.cov_tol && std::isfinite(ce) && ce <= *cfg_.cov_tol) {
                reason = "cov_tol";
                break;
            }
            if (cfg_.mean_tol && std::isfinite(me) && me <= *cfg_.mean_tol) {
                reason = "mean_tol";
                break;
            }
        }
    } catch (...) {
        if (comm_ && !announced) {
            announced = true;
            try {
                comm_->any(true, stream_);
            } catch (...) {
            }
        }
        throw;
    }
    const double wall = elapsed();
    wall_accum_ = wall;
    if (!cfg_.checkpoint_path.empty()) save_checkpoint(wall);  // runner.cpp:276-277
    return build_result(reason, wall);
}

RunResult Engine::build_result(const std::string& reason, double wall) {  // runner.cpp:459-489
    RunResult r;
    r.target_kind = tkind_name(tgt_.kind);
    r.kernel_name = kkind_name(k_.kind);
    r.dim = d_;
    r.chains = P_;
    r.intervals_per_batch = cfg_.intervals_per_batch;
    r.n_lag = k_.n_lag;
    r.master_seed = cfg_.master_seed;
    r.total_samples = (uint64_t)P_ * cfg_.intervals_per_batch * batches_done_ * k_.n_lag;
    r.batches = batches_done_;
    r.wall_seconds = wall;
    r.batch_seconds = batch_seconds_;
    r.stop_reason = reason;
    r.accumulated_samples = cnt_g_;
    // moments through a pinned staging buffer (a pageable d2h of d^2 doubles plus the
    // element-wise mirror cost ~10 ms at d=1024); the result matrix is allocated while
    // the copy runs
    double* hs = static_cast<double*>(pinned_acquire((size_t)(mat_ + ld_) * 8, false));
    const double* sg = hs;
    const double* mg = hs + mat_;
    DGB_CUDA(cudaMemcpyAsync(hs, Sg_, mat_ * 8, cudaMemcpyDeviceToHost, stream_));
    DGB_CUDA(cudaMemcpyAsync(hs + mat_, mg_, ld_ * 8, cudaMemcpyDeviceToHost, stream_));
    r.global_cov = Mat(d_, d_);
    DGB_CUDA(cudaStreamSynchronize(stream_));
    r.global_mean.assign(mg, mg + d_);
    // covariance(), moments.cpp:90-101: lower triangle of S - m m^T, mirrored by 64x64 tiles
    constexpr int kT = 64;
    double* cv = r.global_cov.a.data();
    for (int i0 = 0; i0 < d_; i0 += kT)
        for (int j0 = 0; j0 <= i0; j0 += kT) {
            const int i1 = std::min(d_, i0 + kT), j1 = std::min(d_, j0 + kT);
            for (int i = i0; i < i1; ++i)
                for (int j = j0; j < std::min(j1, i + 1); ++j) cv[(size_t)i * d_ + j] = sg[(size_t)i * ld_ + j] - mg[i] * mg[j];
            for (int j = j0; j < j1; ++j)
                for (int i = std::max(i0, j + 1); i < i1; ++i) cv[(size_t)j * d_ + i] = cv[(size_t)i * d_ + j];
        }
    pinned_release(hs);
    r.final_cov_error = cov_hist_.empty() ? NAN : cov_hist_.back();
    r.final_mean_error = mean_hist_.empty() ? NAN : mean_hist_.back();
    r.final_max_psrf = psrf_hist_.empty() ? NAN : psrf_hist_.back();
    r.cov_error_history = cov_hist_;
    r.mean_error_history = mean_hist_;
    r.psrf_history = psrf_hist_;
    r.functional_names = fnames_;
    // histories and traces of every chain: with several ranks each rank's chains are
    // all-gathered (runner.cpp:459-489 returns every chain's). Every chain has the same
    // number of history entries and of trace entries per functional.
    r.beta_history.assign(P_, {});
    r.acceptance_history.assign(P_, {});
    r.traces.assign(P_, std::vector<std::vector<double>>(fnames_.size()));
    const size_t nb = beta_hist_.empty() ? 0 : beta_hist_[0].size();
    const size_t nf = fnames_.size();
    const size_t nt = (traces_.empty() || traces_[0].empty()) ? 0 : traces_[0][0].size();
    if (comm_) {
        const int64_t maxc = (P_ + world_ - 1) / world_;
        const int64_t per = 2 * (int64_t)nb + (int64_t)(nf * nt);  // doubles per chain
        const int64_t blk = std::max<int64_t>(maxc * per, 1);
        std::vector<double> mine(blk, 0.0);
        for (int c = 0; c < C_; ++c) {
            double* o = mine.data() + c * per;
            std::copy(beta_hist_[c].begin(), beta_hist_[c].end(), o);
            std::copy(acc_hist_[c].begin(), acc_hist_[c].end(), o + nb);
            for (size_t f = 0; f < nf; ++f) std::copy(traces_[c][f].begin(), traces_[c][f].end(), o + 2 * nb + f * nt);
        }
        double* dsrc = dalloc<double>(allocs_, blk);
        double* ddst = dalloc<double>(allocs_, blk * world_);
        DGB_CUDA(cudaMemcpyAsync(dsrc, mine.data(), blk * 8, cudaMemcpyHostToDevice, stream_));
        comm_->allgather(dsrc, ddst, blk, stream_);
        std::vector<double> all(blk * world_);
        DGB_CUDA(cudaMemcpyAsync(all.data(), ddst, all.size() * 8, cudaMemcpyDeviceToHost, stream_));
        DGB_CUDA(cudaStreamSynchronize(stream_));
        for (int rk = 0; rk < world_; ++rk) {
            int64_t base = 0, cr = 0;
            shard_range(P_, world_, rk, &base, &cr);
            for (int c = 0; c < cr; ++c) {
                const double* b = all.data() + rk * blk + c * per;
                r.beta_history[base + c].assign(b, b + nb);
                r.acceptance_history[base + c].assign(b + nb, b + 2 * nb);
                for (size_t f = 0; f < nf; ++f)
                    r.traces[base + c][f].assign(b + 2 * nb + f * nt, b + 2 * nb + (f + 1) * nt);
            }
        }
    } else {
        for (int c = 0; c < C_; ++c) {
            r.beta_history[c0_ + c] = beta_hist_[c];
            r.acceptance_history[c0_ + c] = acc_hist_[c];
            r.traces[c0_ + c] = std::move(traces_[c]);
        }
    }
    return r;
}

}  // namespace dgb
