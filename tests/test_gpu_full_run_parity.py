"""Whole adaptive runs against the reference library itself (oracle/_ref, built from
/root/reference): the time-to-cov-error workload of the bench -- d=100 pi2, 8 chains, two
windows per batch, cov_tol 0.3, the same seeds. DIAM stops after ~400 batches of adaptation
(beta, factors, jitter ladder, merges): the stopping batch, the sample count, the final
covariance error and the per-batch error history must agree (the trajectories differ only
by rounding: 1e-9 relative). AM needs ~2000 batches; its trajectory amplifies rounding
differences ~10x per 100 batches (tools/am_divergence.py: 1e-10 at batch 0, 2e-9 at 200,
3e-4 at 400 -- chaotic, as between any two builds of the reference with different
rounding), so it is held to the same bar over its first 200 batches and to a statistically
equivalent stop after that."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kernel,extra,strict", [("diam", {}, None), ("diam", dict(adaptive_ref=1, n_ref_start=500), None),
                                                 ("am", {}, 200)])
def test_time_to_cov_error_run_matches_reference(b200, ref_abi, kernel, extra, strict):
    kw = dict(kernel=kernel, chains=8, intervals_per_batch=2, max_batches=3000, n0=0, cov_tol=0.3, master_seed=3,
              record_traces=0, trace_eigen_projections=0, **extra)
    tg = b200.target_build("pi2", 100, 1)
    tr = ref_abi.target_build("pi2", 100, 1)
    g = b200.sample(tg, **kw)
    r = ref_abi.sample(tr, threads=8, **kw)
    assert g.stop_reason == r.stop_reason == "cov_tol"
    hg, hr = g.history("cov_error"), r.history("cov_error")
    n = min(len(hg), len(hr)) if strict is None else min(strict, len(hg), len(hr))
    ok = np.isfinite(hr[:n])
    assert np.array_equal(np.isfinite(hg[:n]), ok)
    assert np.max(np.abs(hg[:n][ok] - hr[:n][ok]) / np.abs(hr[:n][ok])) <= 1e-8
    if strict is not None:
        assert abs(g.batches - r.batches) <= 0.1 * r.batches
        return
    assert g.batches == r.batches and g.total_samples == r.total_samples
    assert abs(g.final_cov_error - r.final_cov_error) <= 1e-9 * abs(r.final_cov_error)
