"""Lockstep parity at the benchmarked configurations (SURVEY §8c protocol (3)).

The small-d lockstep runs of test_gpu_sampler.py do not reach the regime the bench
measures: d = 1024, n_lag = 512 steps between re-anchors of the carried G x and
y = L^-1 (x - x_ref) recursions, the 16-group engine, a rank-deficient first
adaptation (512 < d samples), the d >= 1024 GPU target builder, and the chunked,
shared-workspace memory plan of d = 8192. Here the CUDA path runs at those shapes and the
oracle (oracle/diam_oracle.c, on the host's cores) replays chains on the engine's own
captured normals W; the uniforms are bit-exact from the seeds on both sides.

Bars: accept/reject decisions identical, |Delta log alpha| <= 1e-9 max(1, |log alpha|);
beta and acceptance histories bit-equal; pooled moments <= 1e-10 relative; traces
(log pi, the two eigen projections) <= 1e-9 relative.
"""
import os

import numpy as np
import pytest

import _oracle as O

pytestmark = pytest.mark.gpu
THREADS = max(1, min(16, os.cpu_count() or 1))


@pytest.fixture(scope="module")
def pi1_1024(b200, tmp_path_factory):
    """The bench's d=1024 target (bench.make_target_file: fixtures.make('pi1', 1024, 1))."""
    from paper_1506_05741_b200 import fixtures
    path = str(tmp_path_factory.mktemp("bench") / "pi1_1024.bin")
    fixtures.make(path, "pi1", 1024, 1)
    return b200.target_load(path), O.read_target(path)


def captured_windows(cap, p, windows, n_lag, d):
    w = cap.get(p, "w")
    assert w.size == windows * n_lag * d
    return np.concatenate([w, np.zeros(n_lag * d)])  # + the never-consumed final window


def check_chain(res, cap, o, p, i, traces=False):
    """GPU chain p against oracle row i: decisions, log alpha, histories (and traces)."""
    acc_g, lr_g = cap.get(p, "accept"), cap.get(p, "log_ratio")
    acc_o, lr_o, lu = o["accept_bits"][i], o["log_ratio"][i], o["log_u"][i]
    diff = np.nonzero(acc_g != acc_o)[0]
    assert diff.size == 0, (f"chain {p}: {diff.size} decision(s) differ, first at step {diff[0]} "
                            f"(|log u - log alpha| = {abs(lu[diff[0]] - lr_o[diff[0]]):.3e})")
    scale = max(1.0, float(np.max(np.abs(lr_o))))
    err = float(np.max(np.abs(lr_g - lr_o)))
    assert err <= 1e-9 * scale, f"chain {p}: max |Delta log alpha| {err:.3e}"
    assert np.array_equal(res.chain_history(p, "beta"), o["beta_hist"][i])
    assert np.array_equal(res.chain_history(p, "acceptance"), o["acc_hist"][i])
    if traces:
        for f in range(3):
            a, b = res.trace(p, f), o["traces"][i, f]
            assert a.shape == b.shape
            assert np.max(np.abs(a - b)) <= 1e-9 * max(1.0, float(np.max(np.abs(b)))), (p, f)
    return int(acc_g.sum())


def test_bench_config_first_batch_chains_replayed(b200, pi1_1024):
    """The bench workload itself (config 2: pi1 d=1024, 64 chains on 16 chain groups,
    n_lag=512, M=4, n0=0, the bench's seed), one batch; chains 0, 31 and 63 replayed on the
    oracle from their captured W. Inside the first batch every chain reads only the empty
    snapshot, so a chain subset replays exactly. Covers the rank-deficient adaptations of
    windows 1-2 (jitter ladder, usable guard) and the adapted factor of windows 3-4, the
    512-step recursions, and the trace values."""
    t, td = pi1_1024
    P, M, nl, seed = 64, 4, 512, 2026
    res, cap = b200.sample_capture(t, kernel="diam", chains=P, intervals_per_batch=M, max_batches=1, n_lag=nl,
                                   n0=0, master_seed=seed, record_traces=1, trace_thin=1,
                                   trace_eigen_projections=1)
    ids = [0, 31, 63]
    ws = [captured_windows(cap, p, M, nl, 1024) for p in ids]
    o = O.run(td, kind="diam", chains=P, M=M, K=1, seed=seed, inject_w=ws, record_decisions=True, n_lag=nl, n0=0,
              chain_ids=ids, threads=min(THREADS, len(ids)), traces=True)
    accepted = [check_chain(res, cap, o, p, i, traces=True) for i, p in enumerate(ids)]
    assert min(accepted) > 0
    # the adapted factor was adopted by window 3 (count 1536 > d): beta moved off its start
    assert not np.all(o["beta_hist"] == o["beta_hist"][:, :1])


_merge_oracle = {}


@pytest.mark.parametrize("plan", ["resident", "chunked_pool"])
def test_bench_dimension_two_batches_with_merge(b200, pi1_1024, monkeypatch, plan):
    """d=1024, n_lag=512, 4 chains, two batches of two windows: the second batch blends every
    chain with the merged snapshot of the first (moments.cpp:51-88), so pooled moments,
    cov-error and PSRF histories are compared too. 'chunked_pool' forces the d=8192 memory
    plan at this size: 256-row window chunks and one refactor workspace shared by two
    chain groups that refactor in turn."""
    t, td = pi1_1024
    P, M, K, nl, seed = 4, 2, 2, 512, 77
    if plan == "chunked_pool":
        monkeypatch.setenv("DIAM_B200_CHUNK", "256")
        monkeypatch.setenv("DIAM_B200_POOL", "1")
        monkeypatch.setenv("DIAM_B200_GROUPS", "2")
        eng = b200.engine(t, kernel="diam", chains=P, intervals_per_batch=M, n_lag=nl, n0=0, master_seed=seed)
        assert eng.layout == {"groups": 2, "chunk_rows": 256, "pool_factors": 2}
        del eng
    res, cap = b200.sample_capture(t, kernel="diam", chains=P, intervals_per_batch=M, max_batches=K, n_lag=nl,
                                   n0=0, master_seed=seed, record_traces=0)
    ws = [captured_windows(cap, p, M * K, nl, 1024) for p in range(P)]
    key = (P, M, K, nl, seed)
    if key not in _merge_oracle:  # the draws are the same under either plan
        _merge_oracle[key] = O.run(td, kind="diam", chains=P, M=M, K=K, seed=seed, inject_w=ws,
                                   record_decisions=True, n_lag=nl, n0=0, threads=min(THREADS, P))
    o = _merge_oracle[key]
    for p in range(P):
        check_chain(res, cap, o, p, p)
    gm, om = res.mean(), o["global_mean"]
    gc, oc = res.cov(), o["global_cov"]
    assert np.linalg.norm(gm - om) <= 1e-10 * max(1.0, np.linalg.norm(om))
    assert np.linalg.norm(gc - oc) <= 1e-10 * np.linalg.norm(oc)
    assert np.allclose(res.history("cov_error"), o["cov_error_hist"], rtol=1e-9, equal_nan=True)
    assert np.allclose(res.history("psrf"), o["psrf_hist"], rtol=1e-9, equal_nan=True)
    assert res.accumulated_samples == o["accumulated_samples"]


def test_twisted_pi5_d2040_window(b200, tmp_path):
    """Config 4's shape: twisted pi5 at d=2040 (d % 20 == 0, target.cpp:124-125) built by the
    GPU target builder, one window of n_lag = d/2 = 1020 DIAM steps with inflation 1.2 on
    two chains; the oracle loads the same DIAMTGT file. Covers the 2040 x 2040 V^T target
    GEMM and the twisted log-density recursion over 1020 steps."""
    t = b200.target_build("pi5", 2040, 4)
    path = str(tmp_path / "pi5_2040.bin")
    t.save(path)
    td = O.read_target(path)
    P, nl, seed = 2, 1020, 31
    res, cap = b200.sample_capture(t, kernel="diam", chains=P, intervals_per_batch=1, max_batches=1, n_lag=nl, n0=0,
                                   master_seed=seed, inflation=1.2, record_traces=1, trace_thin=7,
                                   trace_eigen_projections=1)
    ws = [captured_windows(cap, p, 1, nl, 2040) for p in range(P)]
    o = O.run(td, kind="diam", chains=P, M=1, K=1, seed=seed, inject_w=ws, record_decisions=True, n_lag=nl, n0=0,
              inflation=1.2, threads=min(THREADS, P), traces=True, trace_thin=7)
    for p in range(P):
        assert check_chain(res, cap, o, p, p, traces=True) > 0


@pytest.mark.parametrize("d,adaptive", [(4100, False), (4100, True), (2100, True)])
def test_wide_rows_window(b200, tmp_path, d, adaptive):
    """The wide-row MH kernels. d = 4100 > 4096 entries: each chain is split over a 4-CTA
    cluster (partial sums through distributed shared memory, one cluster barrier per step,
    every CTA deciding from the same ordered sum); d = 2100: one CTA with 4 pairs per thread,
    the reference point read through L1. Two short windows on two chains, the GPU-built pi1
    target loaded by the oracle; with the adaptive reference point the second window steps
    around a moved x_ref (the kernel variants that carry G x_ref)."""
    t = b200.target_build("pi1", d, 5)
    path = str(tmp_path / f"pi1_{d}.bin")
    t.save(path)
    td = O.read_target(path)
    P, nl, M, seed = 2, 48, 2, 17
    extra = dict(adaptive_ref=1, n_ref_start=nl) if adaptive else {}
    res, cap = b200.sample_capture(t, kernel="diam", chains=P, intervals_per_batch=M, max_batches=1, n_lag=nl,
                                   n0=0, master_seed=seed, record_traces=1, trace_thin=5,
                                   trace_eigen_projections=1, **extra)
    ws = [captured_windows(cap, p, M, nl, d) for p in range(P)]
    o = O.run(td, kind="diam", chains=P, M=M, K=1, seed=seed, inject_w=ws, record_decisions=True, n_lag=nl, n0=0,
              threads=min(THREADS, P), traces=True, trace_thin=5, **extra)
    for p in range(P):
        check_chain(res, cap, o, p, p, traces=True)
