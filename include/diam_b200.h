/*
 * diam_b200.h — B200 engine extensions exported next to the diam.h ABI.
 *
 * None of these replace a reference entry point; they are what a caller needs
 * to (a) place the engine on several GPUs (one process per GPU, NCCL over
 * NVLink), (b) time the device-resident hot path, and (c) check individual
 * kernels against the CPU oracle. Pointer arguments named d_* are DEVICE
 * pointers (e.g. torch CUDA tensors' data_ptr()); `stream` is a cudaStream_t
 * (0 = legacy default stream). Plain C types only.
 */
#ifndef DIAM_B200_H
#define DIAM_B200_H

#include <stdint.h>

#include "diam/diam.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- build identification ------------------------------------------------- */
const char* diamx_build_info(void);       /* arch, CUDA version */
/* FP64 DMMA (mma.sync m8n8k4 f64) throughput of this GPU, TFLOP/s: the roofline
 * denominator for the sampler's dense contractions, measured live */
diam_status diamx_fp64_peak(double* tflops);
uint64_t diamx_launch_count(void);        /* kernels this process launched through the engine */

/* ---- multi-GPU: one process per GPU ---------------------------------------- */
/* rank 0 creates the id, the caller broadcasts the 128 bytes out of band
 * (e.g. torch.distributed), every rank then calls diamx_comm_init. While a
 * communicator is set, diam_sample shards `chains` over the ranks and pools the
 * batch moments with an NCCL all-reduce (the reference's merge_batch,
 * proj/src/moments.cpp:51-75). */
/* host logic the engine uses for the sharded path (CPU-callable, tested with gloo):
 * block sharding of global chain indices and the batch-merge weights */
void diamx_shard_range(int64_t chains, int world, int rank, int64_t* first, int64_t* count);
void diamx_merge_weights(uint64_t global_count, uint64_t chains, uint64_t per_chain, double* keep,
                         double* wp);
/* max_i sqrt(R_i) from per-chain cumulative means / second-moment diagonals
 * (chains x d each, row-major), as the engine computes it after the all-gather */
diam_status diamx_psrf_max(const double* means, const double* diags, int64_t chains, int64_t d,
                           uint64_t samples_per_chain, double* out);
diam_status diamx_nccl_unique_id(char out[128]);
diam_status diamx_comm_init(const char id[128], int rank, int world);
void diamx_comm_destroy(void);
/* ranks of the communicator diam_sample uses (0 = none set) */
diam_status diamx_comm_size(int* out);

/* ---- engine handle for device-resident timing (bench.py) ------------------- */
typedef struct diamx_engine diamx_engine;
diam_status diamx_engine_create(const diam_target* target, const diam_run_options* options,
                                diamx_engine** out);
/* run k full batches (M windows + merge each) without stopping rules;
 * *device_ms = CUDA-event time on the engine stream */
diam_status diamx_engine_run_batches(diamx_engine* e, int64_t k, double* device_ms);
diam_status diamx_engine_set_profiling(diamx_engine* e, int on);
/* per-kernel-class CUDA-event totals; name = "gemm_target" | "trmm_noise" | "syrk_moments" |
 * "potrf" | "mh_window" | "normals" | "trsv" | "blend_cov" | "merge" | "gemv_state" */
diam_status diamx_engine_stat(diamx_engine* e, const char* name, double* ms, double* flops,
                              int64_t* launches);
double diamx_engine_flops_per_batch(const diamx_engine* e);
int64_t diamx_engine_local_chains(const diamx_engine* e);
/* memory plan of an engine: chain groups (streams), rows per window chunk (= n_lag when
 * the whole window is resident) and the shared refactor workspace size (0 = one
 * workspace factor per chain) */
diam_status diamx_engine_layout(const diamx_engine* e, int64_t* groups, int64_t* chunk_rows,
                                int64_t* pool_factors);
void diamx_engine_free(diamx_engine* e);

/* the sharded multi-GPU engine path on ONE GPU: `world` engines (ranks) driven by host
 * threads, exchanging through an in-process communicator instead of NCCL; returns rank
 * 0's result (chain histories all-gathered, traces merged). For parity tests. */
diam_status diamx_sample_threads(const diam_target* target, const diam_run_options* options, int world,
                                 diam_result** out);
/* diam_resume with `world` in-process ranks: the sharded restore of a DIAMCKPT file (every
 * rank reads the file and keeps its block of chains) */
diam_status diamx_resume_threads(const char* path, const diam_run_options* overrides, int world,
                                 diam_result** out);

/* parity capture: run a full diam_sample-equivalent and keep every window's
 * standard normals W (n_windows x n_lag x d per chain) and per-step log alpha /
 * accept bits, so the CPU oracle can be driven on identical draws. */
diam_status diamx_sample_capture(const diam_target* target, const diam_run_options* options,
                                 diam_result** out, diamx_engine** capture_out);
int64_t diamx_capture_len(const diamx_engine* e, int64_t chain, const char* which);
diam_status diamx_capture_copy(const diamx_engine* e, int64_t chain, const char* which, double* out,
                               int64_t capacity);

/* ---- kernel-level entry points (device pointers) ---------------------------- */
/* kind 0: raw u64 (out_u64), 1: uniform_open, 2: normal; stream (seed, idx, purpose) at `start` */
diam_status diamx_draws(int kind, double* d_out_f64, uint64_t* d_out_u64, int64_t n, uint64_t seed,
                        uint64_t stream_index, const char* purpose, uint64_t start, void* stream);
/* C = alpha*A(op)B(op) + beta*C, row-major FP64 on the DMMA GEMM;
 * a_kmajor: A(m,k)=A[m*lda+k] else A[k*lda+m]; b_kmajor: B(k,n)=B[n*ldb+k] else B[k*ldb+n];
 * stream-ordered (returns without waiting for the kernel) */
diam_status diamx_gemm(const double* d_a, const double* d_b, double* d_c, int m, int n, int k,
                       int64_t lda, int64_t ldb, int64_t ldc, int a_kmajor, int b_kmajor, double alpha,
                       double beta, int tri_b_lower, int tri_c_lower, void* stream);
/* batched in-place lower Cholesky of `batch` matrices d_a + i*stride (ld), status per matrix
 * (0 ok, 1 not positive definite) into d_status (int32, device) */
diam_status diamx_potrf(double* d_a, int64_t stride, int64_t ld, int d, int batch, int* d_status,
                        void* stream);
/* timing tool: `groups` concurrent streams each refactoring `chains` copies of the SPD matrix
 * d_src (d + extra_rows rows of stride ld) `rounds` times; device milliseconds */
diam_status diamx_potrf_bench(const double* d_src, int64_t ld, int d, int extra_rows, int groups, int chains,
                              int rounds, double* ms);
/* y_i = L_i^{-1} x_i (batched, L_i = d_l + i*stride), quad_i = 0.5*|y_i|^2 */
diam_status diamx_trsv(const double* d_l, int64_t stride, int64_t ld, const double* d_x, double* d_y,
                       double* d_quad, int d, int batch, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DIAM_B200_H */
