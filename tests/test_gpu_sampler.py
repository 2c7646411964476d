"""End-to-end parity of the B200 sampler through the diam.h ABI.

1. Lockstep on identical draws: the engine records every window's standard
   normals W (GPU Philox + CUDA libm); the CPU oracle (restating
   proj/src/proposal.cpp + runner.cpp) is then driven with exactly those W and
   its own bit-exact Philox uniforms. Accept/reject decisions and accept counts
   (hence every beta/acceptance history entry) must be identical; log alpha
   must agree to 1e-9 (absolute, |log alpha| ~ O(1)); any decision difference
   is allowed only at a near-tie |log u - log alpha| <= 1e-9 and is reported.
   Global moments must agree to 1e-10 relative (FP64, different summation
   order: DMMA GEMMs vs sequential loops).
2. Chain-level statistics vs the reference library on its own draws
   (independent seeds): acceptance rate and covariance error within 3 sigma
   of the Monte Carlo spread.
3. ABI semantics on the GPU path: stopping rules, histories, traces, JSON.
"""
import json
import os

import numpy as np
import pytest

import _oracle as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def lockstep(b200, tmp_path, target_kind, d, kern, P, M, K, n_lag, n0, seed, lr_tol=1e-9, **extra):
    t = b200.target_build(target_kind, d, 17) if isinstance(target_kind, str) else target_kind
    path = str(tmp_path / "t.bin")
    t.save(path)
    td = O.read_target(path)
    res, cap = b200.sample_capture(t, kernel=kern, chains=P, intervals_per_batch=M, max_batches=K, n_lag=n_lag,
                                   n0=n0, master_seed=seed, record_traces=0, **extra)
    windows = K * M
    ws = []
    for p in range(P):
        w = cap.get(p, "w")
        assert w.size == windows * n_lag * d
        ws.append(np.concatenate([w, np.zeros(n_lag * d)]))  # + the never-consumed final window
    o = O.run(td, kind=kern, chains=P, M=M, K=K, seed=seed, inject_w=ws, record_decisions=True, n_lag=n_lag,
              n0=n0, **extra)
    ties = 0
    for p in range(P):
        acc_g = cap.get(p, "accept")
        lr_g = cap.get(p, "log_ratio")
        acc_o = o["accept_bits"][p]
        lr_o = o["log_ratio"][p]
        lu = o["log_u"][p]
        diff = np.nonzero(acc_g != acc_o)[0]
        if diff.size:
            first = diff[0]
            assert abs(lu[first] - lr_o[first]) <= 1e-9, f"chain {p}: decision mismatch at step {first} off a tie"
            ties += 1
            continue  # trajectories legitimately diverge after a tie flip
        assert np.max(np.abs(lr_g - lr_o)) <= lr_tol * max(1.0, np.max(np.abs(lr_o)))
        assert np.array_equal(res.chain_history(p, "beta"), o["beta_hist"][p])
        assert np.array_equal(res.chain_history(p, "acceptance"), o["acc_hist"][p])
    if ties == 0 and lr_tol <= 1e-9:
        gm, om = res.mean(), o["global_mean"]
        gc, oc = res.cov(), o["global_cov"]
        assert np.linalg.norm(gm - om) <= 1e-10 * max(1.0, np.linalg.norm(om))
        assert np.linalg.norm(gc - oc) <= 1e-10 * np.linalg.norm(oc)
        ce = res.history("cov_error")
        assert np.allclose(ce, o["cov_error_hist"], rtol=1e-9, equal_nan=True)
        assert np.allclose(res.history("psrf"), o["psrf_hist"], rtol=1e-9, equal_nan=True)
        assert res.accumulated_samples == o["accumulated_samples"]
    return res, o, ties


@pytest.mark.parametrize("kern", ["diam", "am", "rw", "pcn"])
def test_lockstep_gaussian(b200, tmp_path, kern):
    # n_lag >> d and n0 on a window boundary: even at RW/AM acceptance rates the first
    # adapted covariance has far more distinct states than d, i.e. it is full rank and
    # no factorization depends on rounding (no jitter ladder)
    _, _, ties = lockstep(b200, tmp_path, "pi2", 12, kern, P=3, M=2, K=3, n_lag=200, n0=200, seed=11)
    assert ties == 0


def test_lockstep_rank_deficient_jitter(b200, tmp_path):
    # the first adaptation sees 10 < d samples: the covariance is singular and whether
    # the jitter ladder stops at eps=1e-10 or 1e-8 is decided by rounding;
    # decisions must still agree, log alpha to the jitter scale
    _, _, ties = lockstep(b200, tmp_path, "pi2", 16, "am", P=4, M=3, K=3, n_lag=40, n0=30, seed=11, lr_tol=1e-6)
    assert ties == 0


def test_lockstep_twisted_pi5(b200, tmp_path):
    _, _, ties = lockstep(b200, tmp_path, "pi5", 20, "diam", P=3, M=2, K=3, n_lag=48, n0=0, seed=5, inflation=1.2)
    assert ties == 0


def test_lockstep_adaptive_reference(b200, tmp_path):
    _, _, ties = lockstep(b200, tmp_path, "pi1", 12, "diam", P=2, M=2, K=3, n_lag=30, n0=0, seed=3,
                          adaptive_ref=1, n_ref_start=40)
    assert ties == 0


def test_lockstep_odd_dimension_and_multi_tile(b200, tmp_path):
    # d not a multiple of 8 (padded rows) and > one 128-wide GEMM tile
    _, _, ties = lockstep(b200, tmp_path, "pi2", 133, "diam", P=2, M=2, K=2, n_lag=150, n0=0, seed=9)
    assert ties == 0


@pytest.mark.parametrize("d,P,n_lag,M,K,kern,n0", [
    (2, 1, 1, 3, 4, "diam", 0),     # smallest dimension, one chain, one-step windows
    (3, 2, 5, 2, 3, "am", 3),       # burn-in inside the first window
    (9, 5, 7, 1, 4, "pcn", 0),      # fixed-factor pCN, odd sizes
    (17, 3, 64, 2, 2, "rw", 100),   # burn-in spanning windows, RW form
    (256, 33, 16, 1, 2, "diam", 0),  # odd chain count split over two chain groups (streams)
])
def test_lockstep_edge_cases(b200, tmp_path, d, P, n_lag, M, K, kern, n0):
    # early adaptations see fewer samples than d: rank-deficient covariances factor only
    # with the 1e-10 * tr/d jitter, whose ~1e-5 pivots carry O(eps ||C||) rounding, i.e.
    # ~1e-6 relative in the proposal scale -- decisions must agree, log alpha to 1e-4
    _, _, ties = lockstep(b200, tmp_path, "pi2", d, kern, P=P, M=M, K=K, n_lag=n_lag, n0=n0, seed=d + P,
                          lr_tol=1e-4)
    assert ties == 0


@pytest.mark.parametrize("chunk,pool,groups", [(37, 0, 1), (37, 1, 2), (50, 1, 4)])
def test_lockstep_chunked_windows_shared_workspace(b200, tmp_path, monkeypatch, chunk, pool, groups):
    # the large-d memory plan: windows run in chunks of `chunk` rows (37: ragged last
    # chunk) and the chain groups share one refactor workspace, refactoring in turn
    monkeypatch.setenv("DIAM_B200_CHUNK", str(chunk))
    monkeypatch.setenv("DIAM_B200_POOL", str(pool))
    monkeypatch.setenv("DIAM_B200_GROUPS", str(groups))
    _, _, ties = lockstep(b200, tmp_path, "pi2", 133, "diam", P=4, M=2, K=2, n_lag=150, n0=60, seed=9)
    assert ties == 0


@pytest.mark.parametrize("d", [133, 180, 200])
def test_lockstep_potrf_block_shapes(b200, tmp_path, monkeypatch, d):
    # the blocked factorization's edge shapes under the full engine (augmented usable-guard
    # row, two chain groups): 133 = 128 + 5 (a narrow last block column), 180 = 128 + 52,
    # 200 = 128 + 64 + 8 (a last block column with two diagonal blocks, the second ragged)
    monkeypatch.setenv("DIAM_B200_GROUPS", "2")
    _, _, ties = lockstep(b200, tmp_path, "pi2", d, "diam", P=4, M=2, K=2, n_lag=150, n0=0, seed=9)
    assert ties == 0


def test_chunked_run_matches_resident_run(b200, monkeypatch):
    """Chunked windows + shared workspace change only the moment update's rounding:
    decisions, histories and traces (log density, eigen projections) match the
    resident-window run; moments agree to 1e-12."""
    t = b200.target_build("pi1", 40, 3)
    kw = dict(kernel="diam", chains=6, intervals_per_batch=3, max_batches=2, n_lag=64, n0=50, master_seed=21,
              trace_thin=3)
    monkeypatch.setenv("DIAM_B200_GROUPS", "3")
    r0 = b200.sample(t, **kw)
    monkeypatch.setenv("DIAM_B200_CHUNK", "24")
    monkeypatch.setenv("DIAM_B200_POOL", "1")
    eng = b200.engine(t, **kw)
    assert eng.layout == {"groups": 3, "chunk_rows": 24, "pool_factors": 2}
    del eng
    r1 = b200.sample(t, **kw)
    for p in range(6):
        assert np.array_equal(r0.chain_history(p, "acceptance"), r1.chain_history(p, "acceptance"))
        assert np.array_equal(r0.chain_history(p, "beta"), r1.chain_history(p, "beta"))
        for f in range(3):
            a, b = r0.trace(p, f), r1.trace(p, f)
            assert a.shape == b.shape
            assert np.max(np.abs(a - b)) <= 1e-9 * max(1.0, np.max(np.abs(a)))
    assert np.linalg.norm(r0.cov() - r1.cov()) <= 1e-12 * np.linalg.norm(r0.cov())
    assert np.linalg.norm(r0.mean() - r1.mean()) <= 1e-12 * max(1.0, np.linalg.norm(r0.mean()))


@pytest.mark.parametrize("kern", ["diam", "am"])
def test_pipelined_run_matches_batch_by_batch(b200, kern):
    """The pipelined run loop (next batch enqueued before a batch's outputs are read; used
    when no rule needs the statistics first) and the batch-by-batch loop (forced here by a
    wall-clock limit that never fires) give bit-identical results: histories, statistics,
    traces and moments."""
    t = b200.target_build("pi1", 48, 5)
    kw = dict(kernel=kern, chains=6, intervals_per_batch=3, max_batches=4, n_lag=24, n0=30, master_seed=8,
              trace_thin=2)
    r0 = b200.sample(t, **kw)
    r1 = b200.sample(t, max_wall_seconds=1e6, **kw)
    assert r0.batches == r1.batches == 4
    for h in ("cov_error", "mean_error", "psrf"):
        assert np.array_equal(r0.history(h), r1.history(h), equal_nan=True)
    for p in range(6):
        assert np.array_equal(r0.chain_history(p, "acceptance"), r1.chain_history(p, "acceptance"))
        assert np.array_equal(r0.chain_history(p, "beta"), r1.chain_history(p, "beta"))
        for f in range(3):
            assert np.array_equal(r0.trace(p, f), r1.trace(p, f))
    assert np.array_equal(r0.cov(), r1.cov()) and np.array_equal(r0.mean(), r1.mean())


def test_golden_target_runs_statistics(b200):
    """The reference's own golden runs (tests/golden/runs.npz, written by the reference with
    its own draws and libm): the same configurations on the GPU. The normals differ only in
    the last bits (CUDA vs glibc log/cos), so decisions -- hence the beta / acceptance
    histories and sample counts -- are identical, and every statistic and trace value agrees
    to rounding."""
    import sys
    sys.path.insert(0, GOLD)
    from make_golden import RUNS
    g = np.load(os.path.join(GOLD, "runs.npz"))
    for i, (tf, kern, P, M, K, nl, n0, seed, extra) in enumerate(RUNS):
        t = b200.target_load(os.path.join(GOLD, tf))
        r = b200.sample(t, kernel=kern, chains=P, intervals_per_batch=M, max_batches=K, n_lag=nl, n0=n0,
                        master_seed=seed, record_traces=1, **extra)
        assert r.accumulated_samples == int(g[f"r{i}_accumulated"][0])
        for p in range(P):
            assert np.array_equal(r.chain_history(p, "beta"), g[f"r{i}_beta"][p]), (i, p)
            assert np.array_equal(r.chain_history(p, "acceptance"), g[f"r{i}_acc"][p]), (i, p)
        for h in ("cov_error", "psrf"):
            assert np.allclose(r.history(h), g[f"r{i}_{h}"], rtol=1e-8, atol=1e-12, equal_nan=True), (i, h)
        # the factor amplifies the last-bit differences of the normals by its condition
        # number (RW / AM walk them along): relative Frobenius bounds, reported
        em = np.linalg.norm(r.mean() - g[f"r{i}_mean"]) / max(1.0, np.linalg.norm(g[f"r{i}_mean"]))
        ec = np.linalg.norm(r.cov() - g[f"r{i}_cov"]) / np.linalg.norm(g[f"r{i}_cov"])
        tr, tg = r.trace(0, 0), g[f"r{i}_trace_logpi_c0"]
        assert tr.shape == tg.shape
        et = np.max(np.abs(tr - tg)) / max(1.0, np.max(np.abs(tg)))
        print(f"golden run {i} ({kern}): mean {em:.2e} cov {ec:.2e} trace {et:.2e}")
        assert em <= 1e-8 and ec <= 1e-8 and et <= 1e-8, i


@pytest.mark.parametrize("target", ["pi2", "pi1"])
def test_chain_statistics_vs_reference(b200, ref_abi, tmp_path, target):
    """north_star's chain-level bar: acceptance rate, cov error, mean error and ESS per sample
    of log pi (proj/src/diagnostics.cpp:50-70, the reference's own estimator applied to both
    sides' traces) agree with the reference within Monte Carlo error: 12 independent seeds
    per side (the same seeds -- the normals differ in the last bits, so after a few hundred
    steps the trajectories are independent draws of the same process), 3 standard errors."""
    d = 32
    t_ref = ref_abi.target_build(target, d, 4)
    p = str(tmp_path / "t.bin")
    t_ref.save(p)
    t = b200.target_load(p)
    kw = dict(kernel="diam", chains=4, intervals_per_batch=4, max_batches=6, n_lag=64, n0=0, record_traces=1,
              trace_thin=1, trace_eigen_projections=0)
    stats = {"gpu": [], "ref": []}
    for seed in range(12):
        for name, lib, tt in (("gpu", b200, t), ("ref", ref_abi, t_ref)):
            r = lib.sample(tt, master_seed=100 + seed, threads=4, **kw) if name == "ref" else \
                lib.sample(tt, master_seed=100 + seed, **kw)
            acc = np.mean([r.chain_history(c, "acceptance")[-8:].mean() for c in range(4)])
            # ESS/N of the second half of each chain's log-density trace (post-adaptation)
            ess = []
            for c in range(4):
                tr = r.trace(c, 0)
                tail = np.ascontiguousarray(tr[tr.size // 2:])
                ess.append(ref_abi.ess(tail) / tail.size)
            stats[name].append((acc, r.final_cov_error, r.final_mean_error, float(np.mean(ess))))
    a = np.array(stats["gpu"])
    b = np.array(stats["ref"])
    for j, what in enumerate(["acceptance", "cov_error", "mean_error", "ess_per_sample"]):
        se = np.sqrt(a[:, j].var(ddof=1) / len(a) + b[:, j].var(ddof=1) / len(b))
        print(f"{what}: gpu {a[:, j].mean():.4f} ref {b[:, j].mean():.4f} (3se {3 * se:.4f})")
        assert abs(a[:, j].mean() - b[:, j].mean()) <= 3 * se + 1e-12


def test_stopping_rules_and_histories(b200, tmp_path):
    t = b200.target_build("pi2", 10, 2)
    r = b200.sample(t, kernel="diam", chains=3, intervals_per_batch=2, max_batches=50, n_lag=20, n0=0,
                    cov_tol=0.5, master_seed=1)
    assert r.stop_reason in ("cov_tol", "batch_cap")
    n = r.batches
    assert r.history("cov_error").shape == (n,)
    assert r.history("psrf").shape == (n,)
    assert r.history("batch_seconds").shape == (n,)
    assert r.total_samples == 3 * 2 * n * 20
    assert r.chain_history(2, "beta").shape == (2 * n,)
    if r.stop_reason == "cov_tol":
        assert r.final_cov_error <= 0.5
    r2 = b200.sample(t, kernel="rw", chains=2, max_batches=100, n_lag=10, max_samples=200, master_seed=1)
    assert r2.stop_reason == "max_samples" and r2.total_samples == 200
    # traces: log density + two eigen projections, recorded after burn-in only
    r3 = b200.sample(t, kernel="diam", chains=2, intervals_per_batch=2, max_batches=3, n_lag=10, n0=15,
                     trace_thin=2, master_seed=4)
    assert r3.functional_names() == ["log_density", "proj_min", "proj_max"]
    total = 2 * 3 * 10
    want = len([n for n in range(1, total + 1) if n > 15 and (n - 15 - 1) % 2 == 0])
    assert r3.trace(1, 0).shape == (want,) and r3.trace(1, 2).shape == (want,)
    assert np.all(r3.trace(1, 0) <= 0)
    js = str(tmp_path / "r.json")
    r3.write_json(js)
    doc = json.load(open(js))
    assert doc["schema"] == "diam-run-result/1" and doc["batches"] == 3 and len(doc["iact"]) == 2


def test_engines_reuse_pooled_streams_and_host_buffers(b200, monkeypatch):
    """Engines of different shapes created back to back (and concurrently alive) reuse
    the process-wide stream and pinned-buffer pools; every run equals a fresh one."""
    t = b200.target_build("pi1", 24, 2)
    kw = dict(kernel="diam", chains=8, intervals_per_batch=2, max_batches=2, n_lag=12, n0=0, master_seed=5)
    ref = b200.sample(t, **kw)
    for groups in ("1", "2", "4", "8", "3"):
        monkeypatch.setenv("DIAM_B200_GROUPS", groups)
        held = b200.engine(t, **kw)  # alive while the next run takes streams from the pool
        held.run_batches(1)
        r = b200.sample(t, **kw)
        del held
        assert np.array_equal(r.cov(), ref.cov()) and np.array_equal(r.mean(), ref.mean())
        for p in range(8):
            assert np.array_equal(r.chain_history(p, "acceptance"), ref.chain_history(p, "acceptance"))


def test_launch_counter_moves(b200):
    t = b200.target_build("pi1", 8, 1)
    before = b200.launch_count()
    b200.sample(t, chains=2, max_batches=1, n_lag=4, record_traces=0)
    assert b200.launch_count() > before


@pytest.mark.parametrize("world,P,kern", [(2, 6, "diam"), (3, 7, "diam"), (4, 9, "pcn")])
def test_sharded_engine_in_process_ranks(b200, world, P, kern):
    """The multi-GPU engine path -- block-sharded chains, the batch-moment all-reduce,
    the PSRF and history all-gathers, merge weights over ranks -- with `world` engines on
    one GPU exchanging in process (uneven shards for P % world != 0). Draws are keyed by
    global chain index, so every chain's decisions and histories equal the single-engine
    run; pooled moments agree to summation order (parity across G is at
    tolerance)."""
    t = b200.target_build("pi1", 48, 6)
    kw = dict(kernel=kern, chains=P, intervals_per_batch=2, max_batches=3, n_lag=40, n0=20, master_seed=12,
              trace_thin=5)
    r1 = b200.sample(t, **kw)
    rw = b200.sample_threads(t, world, **kw)
    assert rw.total_samples == r1.total_samples and rw.accumulated_samples == r1.accumulated_samples
    for p in range(P):
        assert np.array_equal(rw.chain_history(p, "beta"), r1.chain_history(p, "beta"))
        assert np.array_equal(rw.chain_history(p, "acceptance"), r1.chain_history(p, "acceptance"))
        a, b = r1.trace(p, 0), rw.trace(p, 0)
        assert a.shape == b.shape and np.max(np.abs(a - b)) <= 1e-9 * max(1.0, np.max(np.abs(a)))
    assert np.linalg.norm(rw.cov() - r1.cov()) <= 1e-12 * np.linalg.norm(r1.cov())
    assert np.linalg.norm(rw.mean() - r1.mean()) <= 1e-12 * max(1.0, np.linalg.norm(r1.mean()))
    assert np.allclose(rw.history("cov_error"), r1.history("cov_error"), rtol=1e-10, equal_nan=True)
    assert np.allclose(rw.history("psrf"), r1.history("psrf"), rtol=1e-10, equal_nan=True)


def test_nccl_sharded_path_single_rank(b200, tmp_path):
    """The multi-GPU code path (NCCL all-reduce of the batch moments, all-gather of the
    PSRF inputs and of the chain histories) on a one-rank communicator must reproduce
    the single-GPU run exactly: a one-rank all-reduce is the identity."""
    import ctypes as C
    t = b200.target_build("pi2", 24, 5)
    kw = dict(kernel="diam", chains=4, intervals_per_batch=2, max_batches=3, n_lag=30, n0=0, master_seed=8,
              record_traces=0)
    r0 = b200.sample(t, **kw)
    uid = C.create_string_buffer(128)
    b200.check(b200.lib.diamx_nccl_unique_id(uid))
    b200.check(b200.lib.diamx_comm_init(uid.raw, 0, 1))
    try:
        r1 = b200.sample(t, **kw)
    finally:
        b200.lib.diamx_comm_destroy()
    assert np.array_equal(r0.mean(), r1.mean()) and np.array_equal(r0.cov(), r1.cov())
    assert np.array_equal(r0.history("psrf"), r1.history("psrf"), equal_nan=True)
    for p in range(4):
        assert np.array_equal(r0.chain_history(p, "beta"), r1.chain_history(p, "beta"))


def test_engine_error_paths(b200):
    """Errors surface as diam statuses with messages, never as crashes: unknown kernel,
    a run that cannot fit in device memory (the memory planner refuses it up front)."""
    from paper_1506_05741_b200.abi import DiamError
    t = b200.target_build("pi1", 64, 2)
    with pytest.raises(DiamError) as e:
        b200.sample(t, kernel="nope", chains=2, max_batches=1, n_lag=8)
    assert e.value.status == 1
    big = b200.target_build("pi1", 1024, 2)
    with pytest.raises(DiamError) as e:
        b200.sample(big, kernel="diam", chains=200000, max_batches=1, n_lag=512, n0=0)
    assert "does not fit in device memory" in e.value.message
    # the library stays usable afterwards
    r = b200.sample(t, kernel="diam", chains=2, max_batches=1, n_lag=8, n0=0)
    assert r.batches == 1


@pytest.mark.parametrize("kern,n_lag,n0,extra", [("diam", 40, 0, {}), ("pcn", 40, 0, {}),
                                                 ("diam", 60, 60, dict(adaptive_ref=1, n_ref_start=120))])
def test_lockstep_explicit_inverse(b200, tmp_path, kern, n_lag, n0, extra):
    # use_explicit_inverse (proj/src/proposal.cpp:98, 202, 241-252): the factor's inverse is
    # kept (GPU: recursive-doubling TRTRI on the DMMA GEMM) and the boundary quad term goes
    # through it (tri_matvec, proposal.cpp:55); the oracle runs the reference's own
    # invert_lower path on the same draws. The option changes rounding only, amplified by
    # cond(L): the moving-reference case uses a burn-in so the first adapted covariance is
    # well conditioned (with n0 = 0 and a 40-step first window the reference's own two modes
    # already differ by 5e-8 in log alpha, and the step recursion vs a per-step TRSV by 1e-5)
    _, _, ties = lockstep(b200, tmp_path, "pi1", 12, kern, P=3, M=2, K=3, n_lag=n_lag, n0=n0, seed=9,
                          use_explicit_inverse=1, **extra)
    assert ties == 0


def test_lockstep_explicit_inverse_multi_level(b200, tmp_path):
    # d = 150: three 64-blocks (a ragged last one) -> two doubling levels of the TRTRI
    _, _, ties = lockstep(b200, tmp_path, "pi2", 150, "diam", P=2, M=2, K=2, n_lag=160, n0=0, seed=4,
                          use_explicit_inverse=1)
    assert ties == 0


@pytest.mark.parametrize("case", ["diam_traces", "am_no_traces", "rw_stop_max_samples", "pcn_psrf_single_chain",
                                  "pi5_projections"])
def test_json_report_matches_contract(b200, tmp_path, case):
    """diam_result_write_json of GPU runs satisfies the reference's report schema
    (proj/docs/result.schema.json via tests/golden/result_contract.json), including NaN
    statistics written as null (one chain: PSRF undefined) and runs without traces."""
    import _schema
    t = b200.target_build("pi5", 20, 3) if case == "pi5_projections" else b200.target_build("pi2", 10, 2)
    kw = dict(diam_traces=dict(kernel="diam", chains=3, intervals_per_batch=2, max_batches=3, n_lag=12, n0=10),
              am_no_traces=dict(kernel="am", chains=2, intervals_per_batch=2, max_batches=2, n_lag=12, n0=0,
                                record_traces=0),
              rw_stop_max_samples=dict(kernel="rw", chains=2, max_batches=50, n_lag=10, max_samples=120),
              pcn_psrf_single_chain=dict(kernel="pcn", chains=1, intervals_per_batch=2, max_batches=2, n_lag=10,
                                         n0=0),
              pi5_projections=dict(kernel="diam", chains=2, intervals_per_batch=1, max_batches=2, n_lag=20, n0=0,
                                   trace_thin=3, inflation=1.2))[case]
    r = b200.sample(t, master_seed=8, **kw)
    js = str(tmp_path / "r.json")
    r.write_json(js)
    doc = json.load(open(js))
    assert _schema.violations(doc) == []
    assert doc["chains"] == kw["chains"] and doc["batches"] == r.batches
    assert len(doc["beta_history"]) == kw["chains"] and len(doc["ess"]) == kw["chains"]
    if case == "pcn_psrf_single_chain":
        assert all(v is None for v in doc["psrf_history"])
