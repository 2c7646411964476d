"""Benchmark: DIAM chain-samples/s on B200 (BASELINE.json metric).

Default workload (N=1): BASELINE.json configs[1] — DIAM, d=1024 anisotropic
Gaussian (pi1), 64 concurrent synchronised chains per GPU, n_lag = d/2 = 512,
M = 4 lag windows per batch, burn-in n0 = 0 and traces
off as in the reference's own `benchmark` command (proj/tools/diam_cli.cpp:
446-458). One bench "step" = one batch = 64 x 4 x 512 = 131072 chain-samples
(windows of Philox noise -> TRMM -> target GEMM -> MH steps -> SYRK moments ->
blend/POTRF/usable guard per window, then the moment merge).

  value  : device-resident throughput, CUDA events on the engine stream,
           max over ranks (diamx_engine_run_batches)
  e2e    : the same metric through the reference-facing C ABI (diam_sample)
           with the target in host memory: H2D upload, engine init, K batches,
           D2H of the result, all inside the timed region (host clock)
  roofline: the dominant kernel class (the FP64 DMMA GEMM: TRMM + target GEMM +
           SYRK + POTRF updates) against the FP64 DMMA peak measured live on
           this GPU (tcgen05 has no f64 kind)
  cpu_baseline: the reference itself (oracle/_ref, built from
           /root/reference/proj/src) on the host cores, bounded sample.

`--impl reference` times the reference's CPU implementation of the same
workload (oracle/_ref, all host threads) and prints its own line.
Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N (weak scaling: 64
chains per GPU, NCCL all-reduce of the batch moments over NVLink).
"""
from __future__ import annotations

import argparse
import json
import os

# before any CUDA context exists: 32 hardware queues for the engine's 2 streams per chain
# group (libdiam.so sets the same default when it loads; see csrc/capi.cpp)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (target kind, d, chains per GPU, n_lag, M)
    "d1024": ("pi1", 1024, 64, 512, 4),
    "d4096": ("pi1", 4096, 64, 2048, 1),
    "d2040": ("pi5", 2040, 256, 1020, 1),
    "d8192": ("pi1", 8192, 128, 4096, 1),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (time, fields)
        self.window = None
        self._proc = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        try:
            self._proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                           "--format=csv,noheader,nounits", "-lms", "50"],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            for line in self._proc.stdout:
                parts = [p.strip() for p in line.strip().split(",")]
                if len(parts) == 6:
                    self.samples.append((time.perf_counter(), parts))
        except Exception:
            pass

    def start(self):
        self._t.start()
        time.sleep(0.3)  # nvidia-smi start-up
        return self

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def stop(self):
        if self._proc:
            self._proc.terminate()
        self._t.join(timeout=10)

    def summary(self):
        samples = self.samples
        if self.window and samples:
            t0, t1 = self.window
            inside = [s for s in samples if t0 <= s[0] <= t1]
            # a sample is a snapshot: keep the ones inside, else the nearest after the start
            samples = inside or [min(samples, key=lambda s: abs(s[0] - t0))]
        rows = [s[1] for s in samples]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(s[0]) for s in rows if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in rows if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in rows for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def make_target_file(kind, d, seed=1):
    from paper_1506_05741_b200 import fixtures
    path = os.path.join(tempfile.gettempdir(), f"diam_bench_{kind}_{d}_{seed}_{os.getpid()}.bin")
    fixtures.make(path, kind, d, seed)
    return path


def run_options(cfg, chains, **over):
    kind, d, _, n_lag, M = cfg
    o = dict(kernel="diam", chains=chains, intervals_per_batch=M, n_lag=n_lag, n0=0, record_traces=0,
             trace_eigen_projections=0, master_seed=2026)
    o.update(over)
    return o


def ncu_gemm_traffic(cfg_name, chains, d, n_lag, distinct=1.0, accepted=0.0):
    """DRAM bytes per launch of the DMMA GEMM classes from the committed `ncu --set full`
    captures (profiles/r02c_ncu_<class>.csv, tools/ncu_capture.sh: d=1024, 64 chains, single
    stream), against their algorithmic bytes (operands in once, results out once)."""
    import csv
    if cfg_name != "d1024" or chains != 64:
        return None
    out, alg = {}, {}
    w = chains * n_lag * d * 8       # one window matrix (W, Xi or H) of all chains
    tri = chains * d * (d + 1) // 2 * 8  # the lower triangles of all chains' L_z or S_z
    # trmm_noise: W in, H out, the factors' lower triangles once
    # syrk_moments: the window's distinct states (rows of H and W) in, the lower S_z read and
    # written
    # xi_accepted: the accepted h rows in, their increments out, the shared G^-1 once
    # (the SYRK's and the accepted-rows product's bytes depend on the window's distinct and
    # accepted rows, which drift as the chains adapt; the captures are of early batches, so
    # only the state-independent TRMM is compared)
    alg_bytes = {"trmm_noise": 2 * w + tri}
    for cls in ("trmm_noise",):
        path = os.path.join(ROOT, "profiles", f"r02c_ncu_{cls}.csv")
        if not os.path.exists(path):
            return None
        rows = list(csv.reader(open(path)))
        h, u, v = rows[0], rows[1], rows[2]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(m)
            tot += float(v[i].replace(",", "")) * scale.get(u[i], 1)
        out[cls] = tot
        alg[cls] = alg_bytes[cls]
    return {"dram_bytes_per_launch": out, "algorithmic_bytes_per_launch": alg,
            "source": "profiles/r02c_ncu_trmm_noise.csv (one launch, single stream; writes still in L2 when "
                      "the kernel ends are not counted)"}


def time_to_cov_error(lib, with_reference: bool):
    """BASELINE.json's second metric: wall time until the pooled covariance error first
    reaches a tolerance. d=100 pi2 (config 1's target), 8 chains, M=2, n0=0, cov_tol 0.3 —
    reachable by the reference in seconds (it converges slowly) — same seeds
    on both sides; the reference on 8 host threads."""
    kw = dict(kernel="diam", chains=8, intervals_per_batch=2, max_batches=5000, n0=0, cov_tol=0.3,
              master_seed=3, record_traces=0, trace_eigen_projections=0)
    t = lib.target_build("pi2", 100, 1)
    lib.sample(t, **dict(kw, max_batches=1))  # warm
    secs = []
    for _ in range(3):  # median of 3 full runs (identical results: same seeds)
        t0 = time.perf_counter()
        r = lib.sample(t, **kw)
        secs.append(time.perf_counter() - t0)
    out = {"target": "pi2 d=100 seed 1", "chains": 8, "cov_tol": 0.3, "gpu_seconds": statistics.median(secs),
           "gpu_runs_seconds": secs, "gpu_samples": r.total_samples, "gpu_stop": r.stop_reason,
           "gpu_final_cov_error": r.final_cov_error}
    if with_reference:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import _oracle as O
        from paper_1506_05741_b200.abi import DiamABI
        if O.ref_available():
            ref = DiamABI(O.REF_SO)
            tr = ref.target_build("pi2", 100, 1)
            rsecs = []
            for _ in range(3):
                t0 = time.perf_counter()
                rr = ref.sample(tr, threads=8, **kw)
                rsecs.append(time.perf_counter() - t0)
            out.update(reference_seconds=statistics.median(rsecs), reference_runs_seconds=rsecs,
                       reference_samples=rr.total_samples,
                       reference_stop=rr.stop_reason, reference_final_cov_error=rr.final_cov_error,
                       reference_threads=8)
    return out


def time_to_cov_error_d1024(lib, cpu):
    """Time-to-cov-error at the benchmark dimension (a reachable tolerance at
    d <= 1024): config 2 (pi1 d=1024, 64 chains, M=4, n0=0) until cov_err <= 0.5, end to end
    through diam_sample. The reference would need the same number of samples at its measured
    rate (cpu_baseline, the same run's host cores): hours, so its time is the composed
    samples / rate, labelled as such."""
    path = make_target_file("pi1", 1024)
    t = lib.target_load(path)
    kw = dict(kernel="diam", chains=64, intervals_per_batch=4, max_batches=3000, n0=0, cov_tol=0.5, master_seed=3,
              record_traces=0, trace_eigen_projections=0)
    t0 = time.perf_counter()
    r = lib.sample(t, **kw)
    secs = time.perf_counter() - t0
    os.unlink(path)
    out = {"target": "pi1 d=1024 (config 2)", "chains": 64, "cov_tol": 0.5, "gpu_seconds": secs,
           "gpu_samples": r.total_samples, "gpu_batches": r.batches, "gpu_stop": r.stop_reason,
           "gpu_final_cov_error": r.final_cov_error}
    if cpu and cpu.get("value"):
        out["reference_seconds_composed"] = r.total_samples / cpu["value"]
        out["reference_note"] = ("composed: the GPU run's sample count at the reference's measured "
                                 f"{cpu['value']:.0f} chain-samples/s on {cpu.get('cores')} host cores")
    return out


# ---------------------------------------------------------------------------- reference CPU arm
def reference_sample(cfg_name, target_path, threads, chains, windows=1):
    """One bounded reference run: `chains` chains x `windows` lag windows on the host cores."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import _oracle as O
    from paper_1506_05741_b200.abi import DiamABI
    if not O.ref_available():
        return None
    kind, d, _, n_lag, _ = CONFIGS[cfg_name]
    ref = DiamABI(O.REF_SO)
    t = ref.target_load(target_path)
    t0 = time.perf_counter()
    r = ref.sample(t, **run_options(CONFIGS[cfg_name], chains, intervals_per_batch=windows, max_batches=1,
                                    threads=threads))
    wall = time.perf_counter() - t0
    return r.total_samples, wall


def impl_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    kind, d, per_gpu, n_lag, M = cfg
    threads = os.cpu_count() or 1
    target = make_target_file(kind, d)
    chains = threads  # one chain per host thread (thread-count invariant results, runner.cpp:316-324)
    samples, times = 0, []
    for i in range(args.warmup + args.steps):
        res = reference_sample(args.config, target, threads, chains)
        if res is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libdiam_ref.so not built"}))
            return 0
        if i >= args.warmup:
            samples += res[0]
            times.append(res[1])
    os.unlink(target)
    total = sum(times)
    value = samples / total
    line = {
        "impl": "reference", "metric": f"chain-samples/s (DIAM, {kind} d={d}, n_lag={n_lag})", "value": value,
        "unit": "chain-samples/s", "n_gpus": int(os.environ.get("WORLD_SIZE", args.gpus)), "device": "host cpu", "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (pi1 target from the reference's Philox stream)",
        "config": {"workload": f"{args.config}: {chains} chains x 1 window of {n_lag} steps per step "
                               f"(reference diam_sample, {threads} threads)", "d": d, "chains": chains,
                   "n_lag": n_lag, "kernel": "diam", "n0": 0},
        "cpu_baseline": {"value": value, "unit": "chain-samples/s", "cores": threads, "kind": "reference",
                         "sample": f"{args.steps} x diam_sample({chains} chains, 1 window of {n_lag}) at d={d}"},
        "e2e": {"value": value, "unit": "chain-samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------- B200 arm
def impl_b200(args):
    import ctypes as C

    import numpy as np
    import torch

    import paper_1506_05741_b200 as pkg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    lib = pkg.load()
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            buf = C.create_string_buffer(128)
            lib.check(lib.lib.diamx_nccl_unique_id(buf))
            uid = torch.frombuffer(bytearray(buf.raw), dtype=torch.uint8).clone()
        uid = uid.cuda()
        dist.broadcast(uid, 0)
        lib.check(lib.lib.diamx_comm_init(bytes(uid.cpu().numpy().tobytes()), rank, world))
        ranks = C.c_int(0)
        lib.check(lib.lib.diamx_comm_size(C.byref(ranks)))
        assert ranks.value == world, f"NCCL communicator has {ranks.value} ranks, expected {world}"
        log(f"rank {rank}: NCCL communicator of {ranks.value} ranks on cuda:{local}")

    cfg = CONFIGS[args.config]
    kind, d, per_gpu, n_lag, M = cfg
    chains = per_gpu * world
    # identical target file on every rank (deterministic generator)
    target_path = make_target_file(kind, d)
    t = lib.target_load(target_path)

    # ---- device-resident throughput
    clocks = ClockSampler(local).start()
    eng = lib.engine(t, **run_options(cfg, chains))
    eng.run_batches(args.warmup)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches0 = lib.launch_count()
    t_start = time.perf_counter()
    ms = eng.run_batches(args.steps)
    clocks.mark(t_start, time.perf_counter())
    clocks.stop()
    launches = lib.launch_count() - launches0
    if dist:
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
        dist.barrier()
    samples_per_step = chains * M * n_lag
    value = samples_per_step * args.steps / (ms / 1e3)

    layout = eng.layout
    alg_flops = eng.flops_per_batch
    del eng
    # ---- roofline of the dominant kernel class: a profiled pass on a single-stream engine
    # (CUDA events around every launch; with one chain group nothing overlaps, so each
    # event pair times its kernel alone). A run that needed the shared refactor workspace
    # (d=8192) is profiled with half the chains, which fit on one stream.
    prof_chains = chains if layout["pool_factors"] == 0 else max(1, chains // 2)
    os.environ["DIAM_B200_GROUPS"] = "1"
    eng = lib.engine(t, **run_options(cfg, prof_chains))
    del os.environ["DIAM_B200_GROUPS"]
    # the same trajectory as the timed run (the chains are independent of the grouping): the
    # same warm-up, then every timed step profiled -- the work per batch grows as the chains
    # adapt (acceptance and with it the distinct and accepted rows: d=1024 from ~10% to ~45%
    # over the first ~10 batches), so the flop count must cover the steps that were timed
    eng.run_batches(max(1, args.warmup))
    eng.set_profiling(True)
    prof_steps = max(1, args.steps)
    eng.run_batches(prof_steps)
    classes = ["gemm_target", "trmm_noise", "syrk_moments", "potrf", "mh_window", "normals", "trsv", "blend_cov",
               "merge", "gemv_state", "xi_accepted", "reconstruct"]
    st = {c: tuple(v / prof_steps for v in eng.stat(c)[:2]) for c in classes}  # per batch
    prof_total = sum(v[0] for v in st.values())
    gemm_cls = ["gemm_target", "trmm_noise", "syrk_moments", "xi_accepted"]
    g_ms = sum(st[c][0] for c in gemm_cls)
    g_fl = sum(st[c][1] for c in gemm_cls)
    peak = C.c_double()
    lib.check(lib.lib.diamx_fp64_peak(C.byref(peak)))
    achieved = g_fl / (g_ms / 1e3) / 1e12 if g_ms > 0 else 0.0
    t_ms, t_fl = st["trmm_noise"][0], st["trmm_noise"][1]
    t_achieved = t_fl / (t_ms / 1e3) / 1e12 if t_ms > 0 else 0.0
    f_achieved = st["potrf"][1] / (st["potrf"][0] / 1e3) / 1e12 if st["potrf"][0] > 0 else 0.0
    # the step's algorithmic flops: every class's count from the profiled batch (the SYRK over
    # the window's distinct states and the accepted steps' increments count the rows they ran
    # over), scaled to the timed run's chains per GPU
    syrk_full = prof_chains * M * n_lag * d * (d + 1.0)
    distinct = st["syrk_moments"][1] / syrk_full if syrk_full else 1.0
    accepted = st["xi_accepted"][1] / syrk_full if syrk_full else 0.0
    alg_flops = sum(v[1] for v in st.values()) * (chains / world) / prof_chains
    traffic = ncu_gemm_traffic(args.config, per_gpu, d, n_lag, distinct, accepted)
    del eng

    # ---- end-to-end through the C ABI (host target, result back to host)
    torch.cuda.synchronize()
    lib.sample(t, **run_options(cfg, chains, max_batches=1))  # warm (module load, allocator)
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    r = lib.sample(t, **run_options(cfg, chains, max_batches=args.steps))
    t1 = time.perf_counter()
    mean = r.mean()
    cov = r.cov()
    wall = time.perf_counter() - t0
    if dist:
        tt = torch.tensor([wall], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        wall = float(tt.item())
    bsec = r.history("batch_seconds")
    log(f"e2e: {wall * 1e3:.1f} ms wall, batches {bsec.sum() * 1e3:.1f} ms "
        f"(first {bsec[0] * 1e3:.1f}, median {float(sorted(bsec)[len(bsec) // 2]) * 1e3:.1f}), "
        f"fixed costs {(wall - bsec.sum()) * 1e3:.1f} ms (diam_sample {(t1 - t0) * 1e3:.1f} ms, "
        f"result copies {(wall - (t1 - t0)) * 1e3:.1f} ms)")
    e2e = r.total_samples / wall
    h2d = (d * d * 8 * 2 + 4 * d * 8) / args.steps  # precision + analytic covariance + vectors, once per run
    d2h = (mean.nbytes + cov.nbytes) / args.steps + chains * M * 16 + 24
    os.unlink(target_path)

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            cpu_t = make_target_file(kind, d)
            threads = os.cpu_count() or 1
            res = reference_sample(args.config, cpu_t, threads, threads)
            os.unlink(cpu_t)
            if res:
                cpu = {"value": res[0] / res[1], "unit": "chain-samples/s", "cores": threads, "kind": "reference",
                       "sample": f"reference diam_sample: {threads} chains x 1 window of {n_lag} steps at d={d} "
                                 f"({res[0]} chain-samples in {res[1]:.1f} s, incl. its init window)"}
        line = {
            "metric": f"chain-samples/s (DIAM, {kind} d={d}, n_lag={n_lag})",
            "value": value, "unit": "chain-samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (pi1 target, Philox stream of the reference, random chains)",
            "config": {"workload": f"{args.config}: DIAM {kind} d={d}, {per_gpu} chains/GPU, n_lag={n_lag}, "
                                   f"M={M} windows per step, n0=0, traces off",
                       "d": d, "chains": chains, "chains_per_gpu": per_gpu, "n_lag": n_lag,
                       "intervals_per_batch": M, "kernel": "diam", "parallelism": f"chains sharded dp{world}",
                       "memory_plan": layout,
                       "l2": "no flush needed: per-step working set "
                             f"{(3 * d * d + 3 * n_lag * d) * 8 * per_gpu / 1e9:.1f} GB >> 126 MB L2"},
            "roofline": {"bound": "tensor", "pipe": "FP64 DMMA (mma.sync.m8n8k4.f64; tcgen05 has no f64 kind)",
                         "achieved": t_achieved, "peak": peak.value, "unit": "TFLOP/s",
                         "frac": t_achieved / peak.value if peak.value else None,
                         "traffic": traffic["dram_bytes_per_launch"]["trmm_noise"] if traffic else None,
                         "traffic_detail": traffic,
                         "kernel": "trmm_noise: the window TRMM H = s W L_z^T (the step's largest kernel)",
                         "share_of_step": t_ms / prof_total if prof_total else None,
                         "gemm_class": {"kernels": "TRMM + twisted rows + SYRK moments + accepted increments",
                                        "achieved": achieved, "frac": achieved / peak.value if peak.value else None,
                                        "share_of_step": g_ms / prof_total if prof_total else None},
                         "factorization_class": {"kernels": "long-K updates + diagonal blocks + TRSMs (d^3/3 flops)",
                                                 "achieved": f_achieved,
                                                 "frac": f_achieved / peak.value if peak.value else None,
                                                 "share_of_step": st["potrf"][0] / prof_total if prof_total else None},
                         "peak_source": "diamx_fp64_peak: DMMA m8n8k4 loop measured live (MEASURED_PEAKS.json "
                                        "has no FP64 entry)",
                         "step_alg_tflops": alg_flops / (ms / args.steps / 1e3) / 1e12,
                         "syrk_distinct_row_fraction": distinct,
                         "accepted_row_fraction": accepted,
                         "profile_chains": prof_chains,
                         "per_class_ms": {c: round(v[0], 4) for c, v in st.items()}},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": "chain-samples/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "note": "diam_sample via the C ABI: target upload + engine init + K batches + result copy"},
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            line["time_to_cov_error"] = time_to_cov_error(lib, with_reference=True)
            if args.config == "d1024":
                line["time_to_cov_error_d1024"] = time_to_cov_error_d1024(lib, cpu)
        print(json.dumps(line))
    if dist:
        lib.lib.diamx_comm_destroy()
        dist.destroy_process_group()
    return 0


def relaunch(args) -> int:
    """`bench.py --gpus N` run directly (no torchrun): start the N ranks ourselves, one
    process per GPU, with the same arguments (the driver's own launch line is the same
    torch.distributed.run command)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    log(f"bench.py: launching {args.gpus} ranks: {' '.join(cmd)}")
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="d1024")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    if args.impl == "reference":
        return impl_reference(args)
    return impl_b200(args)


if __name__ == "__main__":
    sys.exit(main())
