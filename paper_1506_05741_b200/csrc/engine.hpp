// engine.hpp — the B200 sampler engine (C++ host driver over sm_100a kernels).
//
// Mirrors the reference Engine (proj/src/runner.cpp:122-279): P chains, batches
// of M lag windows, a frozen global snapshot per batch, merge at the barrier,
// convergence diagnostics and OR-composed stopping rules. The per-chain loop
// of the reference (mh_step x n_lag, lag_update) becomes a per-window sequence
// of batched kernels over a GROUP of local chains on the group's CUDA stream:
//
//   noise    W = Philox normals                 (launch_normals)
//   TRMM     Xi = s * W * L^T                   (gemm_f64, tri B)
//   target   H = Xi * G^T                       (gemm_f64, the group's windows as one GEMM)
//   steps    n_lag MH steps, O(d) each          (launch_mh_window, TMA-fed ring)
//   moments  S = a X^T X + b S, mean            (gemm_f64 tri C + launch_mean_update)
//   adapt    beta, blend -> POTRF (+ jitter ladder stepped by the host, augmented usable-guard row)
//            -> swap, x_ref, g = G x            (potrf_batched, gemm_f64)
//
// The local chains are split into groups on separate streams with no host
// round trip inside a batch, so one group's latency-bound pieces (MH steps,
// diagonal factorizations) overlap the other group's DMMA GEMMs. Per batch:
// join the groups, local moment sum -> all-reduce (multi-GPU) -> merge,
// cumulative PSRF statistics, cov/mean error.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "comm.hpp"
#include "gemm_f64.cuh"
#include "host.hpp"
#include "kernels.cuh"

namespace dgb {

struct KernelStat {
    double ms = 0.0;
    double flops = 0.0;
    uint64_t launches = 0;
};

class Engine {
public:
    // The target is shared, not copied (3 d x d matrices): a blocking call passes a
    // non-owning pointer (borrow()), an engine handle that outlives the call an owning one.
    Engine(std::shared_ptr<const HostTarget> t, const RunCfg& cfg, std::shared_ptr<Comm> comm);
    static std::shared_ptr<const HostTarget> borrow(const HostTarget& t) {
        return std::shared_ptr<const HostTarget>(&t, [](const HostTarget*) {});
    }
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    RunResult run();                  // full run with the reference's stopping rules
    double run_batches_timed(int k);  // k batches, no stopping rules; device ms (CUDA events)

    // DIAMCKPT v1 checkpoints (proj/src/runner.cpp:398-457 / 139-207), written after every
    // batch when cfg.checkpoint_path is set. The file is the reference's layout followed by
    // a "B200EXT1" block carrying each chain's y = L^-1 (x - x_ref) so that a resumed run
    // continues bit-for-bit; a reference-written file (no block) gets y re-solved.
    static void read_checkpoint_header(BinIn& r, HostTarget& t, RunCfg& cfg);
    void restore(BinIn& r);  // after construction from the header's target/config
    void override_stop(const RunCfg& c);
    void override_max_batches(size_t k) { cfg_.max_batches = k; }

    // profiling: per-kernel-class CUDA-event timing (adds events around launches)
    void set_profiling(bool on) { profiling_ = on; }
    const std::map<std::string, KernelStat>& stats();

    // debug capture for parity tests: W of every window, accept bits / log ratios of every step
    void set_capture(bool on) { capture_ = on; }
    const std::vector<double>& captured_w(int chain) const { return cap_w_.at(chain); }
    const std::vector<double>& captured_ratio(int chain) const { return cap_ratio_.at(chain); }
    const std::vector<uint8_t>& captured_accept(int chain) const { return cap_acc_.at(chain); }

    cudaStream_t stream() const { return stream_; }
    int local_chains() const { return C_; }
    int dim() const { return d_; }
    int n_lag() const { return Lw_; }
    int groups() const { return (int)groups_.size(); }
    int chunk_rows() const { return Lc_; }
    int pool_factors() const { return pool_ ? pool_n_ : 0; }
    double flops_per_batch() const;  // algorithmic FP64 flops of one batch (all local chains)

private:
    struct Group {
        int off = 0, C = 0;
        cudaStream_t s = nullptr;
        int prio_s = 0, prio_sr = 0;  // stream priorities (the pool's keys)
        cudaEvent_t done = nullptr;
        double **Lp = nullptr, **Lnp = nullptr, **Wp = nullptr, **Xip = nullptr, **Sp = nullptr;
        double **Xib = nullptr, **Hb = nullptr;                                     // 1-element arrays
        PotrfWork pw{};
        cudaEvent_t status_ev = nullptr;  // POTRF statuses of the group's last window landed in h_status_
        cudaEvent_t pool_ev = nullptr;    // shared refactor workspace released (pool mode)
        // refactorization + tail on their own high-priority stream: the latency-bound
        // POTRF launches of one group are scheduled ahead of the other groups' GEMMs
        cudaStream_t sr = nullptr;
        cudaEvent_t ev_steps = nullptr, ev_ref = nullptr;
        cudaGraphExec_t potrf_exec = nullptr;  // the factorization's launches (Engine::factor)
        uint64_t potrf_nodes = 0, potrf_calls = 0;
    };
    // host-side scalars of one lag window, identical for every chain
    struct WindowPlan {
        size_t w = 0;
        uint64_t n_start = 0, n_end = 0, nctr = 0;
        int first = 0, k = 0;  // accumulated rows [first, n_lag)
        uint64_t cnt_before = 0, cnt_after = 0;
        bool record = false, refactor = false, move_ref = false;
        bool identity = false;  // every factor is still the initial identity (noise = s W)
        double wg = 0.0, wl = 1.0;
    };

    void upload_target();
    int plan_memory();  // window chunk rows, shared refactor workspace; returns the group count
    void init_chains();
    void make_groups(int n);
    WindowPlan plan_window(size_t w, bool record) const;
    void commit_window(const WindowPlan& p);
    // a window is enqueued in two parts: the head (noise .. POTRF, statuses copied to the
    // host asynchronously) and the tail (jitter ladder if any chain failed, usable guard,
    // factor swap, reference point, G x). Between them the host reads the group's
    // statuses while the other group keeps the GPU busy. The head is the window's steps
    // (chunk by chunk) followed by the refactorization.
    void enqueue_head(Group& g, const WindowPlan& p) {
        enqueue_steps(g, p);
        enqueue_refactor(g, p);
    }
    void enqueue_steps(Group& g, const WindowPlan& p);
    void enqueue_chunk(Group& g, const WindowPlan& p, int r0, int rows);
    void enqueue_refactor(Group& g, const WindowPlan& p);
    void enqueue_tail(Group& g, const WindowPlan& p);  // tail_begin/step.../finish, blocking
    struct Ladder {  // one group's jitter escalation in flight
        std::vector<int> failing;
        double eps = 0.0;
    };
    bool tail_begin(Group& g, const WindowPlan& p, Ladder& st);
    bool tail_step(Group& g, const WindowPlan& p, Ladder& st);
    void ladder_retry(Group& g, const WindowPlan& p, Ladder& st);
    void tail_finish(Group& g, const WindowPlan& p);
    void run_batch_windows(bool record);
    // run_batch_windows split for the pipelined run loop (no capture, no shared workspace):
    // begin_windows plans the batch and enqueues every group's first window; end_windows
    // runs the tails and the remaining windows
    void begin_windows(bool record);
    void end_windows();
    std::vector<WindowPlan> bplans_;
    void capture_chunk(const Group& g, int r0, int rows);
    void capture_window(size_t w);
    void fork_groups();  // groups wait for the main stream
    // pipelined loop: the next batch's first windows start right after the join; only
    // their moment updates (and MH steps when traces are recorded) wait for merge_ev_,
    // the end of the batch's merge, statistics and output copies
    cudaEvent_t join_ev_ = nullptr, merge_ev_ = nullptr;
    bool merge_pending_ = false;
    void join_groups();  // main stream waits for every group
    void merge_batch();
    // per batch: enqueue the statistics kernels and every per-batch output's copy into
    // pinned memory (stream order), then read them once the stream got there
    void enqueue_batch_outputs(size_t windows);
    void read_batch_outputs(size_t windows, double& cov_err, double& mean_err, double& psrf);
    void collect_histories(size_t windows, const std::vector<uint64_t>& n_start, const double* rate,
                           const double* beta, const double* lp, const double* pj);
    std::vector<uint64_t> out_n_start_;  // window start counts of the batch in h_out_
    void save_checkpoint(double wall);
    // flops < 0: the algorithmic count from the shape (triangular halves included)
    void gemm(const char* name, const GemmBatch& g, int batch, bool ak, bool bk, cudaStream_t s,
              double flops = -1.0, bool small = false);
    void refresh_g(const double* x, double* out, int chains, cudaStream_t s);
    void timed_begin(cudaStream_t s);
    void timed_end(const char* name, double flops, cudaStream_t s);
    void resolve_events();
    RunResult build_result(const std::string& reason, double wall);

    std::shared_ptr<const HostTarget> tgtp_;
    const HostTarget& tgt_;
    RunCfg cfg_;
    KernelCfg k_;
    std::shared_ptr<Comm> comm_;
    int rank_ = 0, world_ = 1;
    int d_ = 0, Lw_ = 0, C_ = 0, P_ = 0, c0_ = 0;
    // memory plan (plan_memory): window buffers hold Lc_ rows per chain (Lc_ < Lw_: the
    // window runs in chunks); pool_: the chain groups share one refactor workspace of
    // pool_n_ factors and refactor one after another
    int Lc_ = 0;
    bool pool_ = false;
    int pool_n_ = 0;
    size_t arena_bytes_ = 0;  // device bytes the plan needs after the target upload
    cudaEvent_t pool_last_ = nullptr;  // latest release of the shared workspace
    int64_t ld_ = 0, win_ = 0, mat_ = 0;
    int64_t fmat_ = 0;  // factor stride: d rows + the augmented row r = x - x_ref
    bool twisted_ = false, identity_ = true;
    // Gaussian targets are stepped in whitened form: G = a lower-triangular factor of the
    // precision (G^T G = P), log pi(x) = -1/2 |G x|^2 -- the target product H = Xi G^T is
    // then triangular (half the flops of the full product with P)
    bool tri_target_ = false;
    // twisted targets add the T = d/10 twisted coordinates z_i = (V^T x)_i as rows of G below
    // the whitening factor: g = G x has dg_ = d + T entries (stride ldg_; H rows likewise)
    int dg_ = 0;
    int64_t ldg_ = 0, winh_ = 0;
    cudaStream_t stream_ = nullptr;
    int stream_prio_ = 0;
    cudaEvent_t main_ev_ = nullptr;
    std::vector<Group> groups_;

    // device memory
    // device memory: one arena per engine sized by the memory plan (a single block that
    // the stream-ordered pool hands to the next engine of the same shape, instead of
    // dozens of buffers that fragment it), plus individual blocks for what does not fit
    struct DevMem {
        std::vector<void*> blocks;
        char* arena = nullptr;
        size_t size = 0, used = 0;
    };
    DevMem allocs_;
    double* G_ = nullptr;      // d x ld
    double* Ct_ = nullptr;     // d x d analytic covariance
    double* inv_eig_ = nullptr;
    double* bcoef_ = nullptr;
    double* proj_ = nullptr;   // 2 x ld
    double *L_ = nullptr, *Lw2_ = nullptr, *S_ = nullptr;  // C x ((d+1) or d) x ld
    double *W_ = nullptr, *Xi_ = nullptr, *H_ = nullptr;   // C x (Lc x ld)
    double *x_ = nullptr, *g_ = nullptr, *y_ = nullptr, *xr_ = nullptr, *gr_ = nullptr;
    double *mean_ = nullptr, *cmean_ = nullptr, *cdiag_ = nullptr, *mb_ = nullptr;
    double *logpi_ = nullptr, *quad_ = nullptr, *beta_ = nullptr, *tr_ = nullptr, *qtmp_ = nullptr;
    uint64_t *nacc_ = nullptr, *uctr_ = nullptr;
    int *status_ = nullptr, *try_ = nullptr, *usable_ = nullptr, *mask_ = nullptr;
    int* kcount_ = nullptr;  // per chain: distinct counted states of the last window chunk
    int* row_of_ = nullptr;  // C x n_lag: compacted row of each step's state (trace projections)
    int* h_flags_ = nullptr;  // pinned host mirror: status[C], try[C], ladder mask[C]
    PhiloxKey *nkeys_ = nullptr, *ukeys_ = nullptr, *ikeys_ = nullptr;
    double **Lp_ = nullptr, **Lnp_ = nullptr;  // factor / workspace pointer arrays (swapped on device)
    double **Wp_ = nullptr, **Xip_ = nullptr, **Hp_ = nullptr, **Sp_ = nullptr, **Gp_ = nullptr, **Gpc_ = nullptr;
    double *Sg_ = nullptr, *mg_ = nullptr, *Ssum_ = nullptr;  // global snapshot, reduction buffer
    double *trace_lp_ = nullptr, *trace_pj_ = nullptr;      // per batch: M x C x Lw (x2)
    double *hist_rate_ = nullptr, *hist_beta_ = nullptr;    // per batch: M x C
    double* cov_part_ = nullptr;                              // d x 2
    double *tmean_ = nullptr, *dstats_ = nullptr;             // target mean; batch statistics (4)
    double* h_stats_ = nullptr;                               // pinned mirror of dstats_
    double* h_out_ = nullptr;  // pinned per-batch outputs: rate, beta (M x C), traces (M x C x Lw x 3)
    cudaEvent_t out_ev_ = nullptr;  // the copies into h_out_ / h_stats_ are done
    double* gather_ = nullptr;                                // PSRF all-gather buffer
    double* cS_ = nullptr;  // cumulative raw second moments (whitened, lower), kept only for checkpoints
    // whitened-space factorization: the factors L_ are L_z = G L, the local and
    // global second moments S_ / Sgz_ and means mean_ / mgz_ are in whitened coordinates; the
    // x-space statistics the reference reports are kept beside them: per chain the running mean
    // and raw diagonal (mean_x_, diag_x_; PSRF, trace floor, adaptive reference), globally the
    // snapshot Sg_ / mg_ (Sg_ = G^-1 Sgz_ G^-T once per batch; cov error, results, checkpoints)
    double *Ginv_ = nullptr, *GG_ = nullptr, *BT_ = nullptr;  // G^-1, G G^T (jitter), V_T^T G^-1
    double **Ginvp_ = nullptr, **Ginvpc_ = nullptr, **BTpc_ = nullptr;
    double *mean_x_ = nullptr, *diag_x_ = nullptr, *Sgz_ = nullptr, *mgz_ = nullptr;
    double *Sfull_ = nullptr, *Stmp_ = nullptr;  // per-batch x-space transform scratch
    double** ptr_tmp_[3] = {nullptr, nullptr, nullptr};  // Sfull_, Stmp_, Sg_ as GEMM operands
    int *state_src_ = nullptr, *state_mult_ = nullptr, *acc_cnt_ = nullptr;
    void update_x_snapshot();  // Sg_ = G^-1 Sgz_ G^-T
    double** ptr_gen_ = nullptr;  // 3 device pointers for dev_gemm
    void dev_gemm(const double* A, const double* B, bool bk, double* out, bool tri);
    void congruence(const double* S, const double* M, double* out);
    // use_explicit_inverse: X = L^{-1} per chain (upper part zero) and the TRTRI scratch
    double* Xinv_ = nullptr;
    double* Tinv_ = nullptr;
    double** Xinvp_ = nullptr;
    double** Tinvp_ = nullptr;
    double wall_accum_ = 0.0;  // wall seconds of earlier (checkpointed) segments of the run

    // host-side counters (uniform across chains)
    uint64_t n_ = 0;          // iterations per chain
    uint64_t nctr_ = 0;       // noise stream draw counter
    uint64_t cnt_local_ = 0;  // samples in the batch accumulators (per chain)
    uint64_t cnt_g_ = 0;      // global moments count
    uint64_t cum_cnt_ = 0;    // cumulative per-chain count
    size_t batches_done_ = 0;
    std::vector<uint64_t> window_n_start_;  // per window of the current batch

    // result accumulation
    std::vector<double> batch_seconds_, cov_hist_, mean_hist_, psrf_hist_;
    std::vector<std::vector<double>> beta_hist_, acc_hist_;  // local chains
    std::vector<std::vector<std::vector<double>>> traces_;   // local chains x functionals
    std::vector<std::string> fnames_;

    // profiling
    bool profiling_ = false;
    struct Pending {
        std::string name;
        cudaEvent_t a, b;
        double flops;
        cudaStream_t s;
    };
    cudaEvent_t timeline_base_ = nullptr;  // profiling: origin of the optional timeline dump
    std::vector<Pending> pending_;
    std::vector<cudaEvent_t> event_pool_;
    std::map<std::string, KernelStat> stats_;
    std::map<cudaStream_t, cudaEvent_t> open_;

    bool capture_ = false;
    // timing tool (DIAM_B200_TWICE=normals,trmm,target,potrf; tools/twice_sweep.py): the named
    // idempotent steps are launched twice -- the second launch recomputes the same values, so
    // the run is unchanged and the batch time grows by what one more instance costs in the
    // overlapped schedule
    unsigned twice_ = 0;
    bool use_graphs_ = true;  // DIAM_B200_GRAPHS=0 or DIAM_B200_SYNC_CHECK: direct launches
    void factor(Group& g, cudaStream_t s, bool aug);
    enum : unsigned { kTwiceNormals = 1, kTwiceTrmm = 2, kTwiceTarget = 4, kTwicePotrf = 32 };
    double host_wait_s_ = 0.0;  // run_batches_timed: host time blocked on the GPU (statuses)
    std::vector<std::vector<double>> cap_w_, cap_ratio_;
    std::vector<std::vector<uint8_t>> cap_acc_;
    std::vector<double> cap_wbuf_;  // C x n_lag x d: the current window's W, filled chunk by chunk
    double* dbg_ratio_ = nullptr;
    uint8_t* dbg_acc_ = nullptr;
};

}  // namespace dgb
