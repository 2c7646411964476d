"""DIAMCKPT checkpoint / resume on the GPU engine.

* resume is bit-exact: K batches in one go == K1 batches, checkpoint, resume to K
  (proj/tests/test_runner.cpp:154-183 asks the same of the reference);
* the file is the reference's format: the reference library resumes a checkpoint
  written by the B200 engine, and the B200 engine resumes one written by the
  reference (proj/src/runner.cpp:398-457, 139-207).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same(r0, r1, chains):
    assert r0.batches == r1.batches and r0.total_samples == r1.total_samples
    assert np.array_equal(r0.mean(), r1.mean())
    assert np.array_equal(r0.cov(), r1.cov())
    for h in ("cov_error", "mean_error", "psrf"):
        assert np.array_equal(r0.history(h), r1.history(h), equal_nan=True)
    for p in range(chains):
        assert np.array_equal(r0.chain_history(p, "beta"), r1.chain_history(p, "beta"))
        assert np.array_equal(r0.chain_history(p, "acceptance"), r1.chain_history(p, "acceptance"))
        for f in range(3):
            assert np.array_equal(r0.trace(p, f), r1.trace(p, f))


@pytest.mark.parametrize("kern", ["diam", "am"])
def test_resume_is_bit_exact(b200, tmp_path, kern):
    t = b200.target_build("pi2", 20, 6)
    kw = dict(kernel=kern, chains=4, intervals_per_batch=2, n_lag=30, n0=40, master_seed=12)
    full = b200.sample(t, max_batches=5, **kw)
    ck = str(tmp_path / "run.ckpt")
    part = b200.sample(t, max_batches=2, checkpoint_path=ck, **kw)
    assert part.batches == 2 and part.stop_reason == "batch_cap"
    resumed = b200.resume(ck, b200.options(max_batches=5))
    _same(full, resumed, 4)
    assert resumed.stop_reason == "batch_cap"


def test_reference_resumes_b200_checkpoint_and_vice_versa(b200, ref_abi, tmp_path):
    t_ref = ref_abi.target_build("pi2", 16, 3)
    tp = str(tmp_path / "t.bin")
    t_ref.save(tp)
    t = b200.target_load(tp)
    kw = dict(kernel="diam", chains=3, intervals_per_batch=2, n_lag=40, n0=0, master_seed=5)
    # B200 writes, reference resumes
    ck1 = str(tmp_path / "b200.ckpt")
    b200.sample(t, max_batches=2, checkpoint_path=ck1, **kw)
    r_ref = ref_abi.resume(ck1, ref_abi.options(max_batches=4))
    assert r_ref.batches == 4 and r_ref.total_samples == 3 * 2 * 4 * 40
    assert np.isfinite(r_ref.final_cov_error)
    # reference writes, B200 resumes
    ck2 = str(tmp_path / "ref.ckpt")
    ref_abi.sample(t_ref, max_batches=2, checkpoint_path=ck2, threads=1, **kw)
    r_b = b200.resume(ck2, b200.options(max_batches=4))
    assert r_b.batches == 4 and r_b.total_samples == 3 * 2 * 4 * 40
    # the first two batches' histories come from the reference's run unchanged
    r_ref2 = ref_abi.sample(t_ref, max_batches=2, threads=1, **kw)
    assert np.array_equal(r_b.history("cov_error")[:2], r_ref2.history("cov_error"))
    for p in range(3):
        assert np.array_equal(r_b.chain_history(p, "beta")[:4], r_ref2.chain_history(p, "beta"))
    # and the continuation is statistically the same process
    assert np.isfinite(r_b.final_cov_error) and r_b.final_cov_error < 10 * r_ref.final_cov_error + 1.0


def test_explicit_inverse_checkpoint(b200, ref_abi, tmp_path):
    # factor_inv travels in the DIAMCKPT file (proj/src/runner.cpp:186, 444-445): resume is
    # bit-exact, and the reference resumes the file
    t = b200.target_build("pi2", 70, 6)
    kw = dict(kernel="diam", chains=3, intervals_per_batch=2, n_lag=40, n0=0, master_seed=12, use_explicit_inverse=1)
    full = b200.sample(t, max_batches=4, **kw)
    ck = str(tmp_path / "inv.ckpt")
    b200.sample(t, max_batches=2, checkpoint_path=ck, **kw)
    import shutil
    ck2 = str(tmp_path / "inv_copy.ckpt")
    shutil.copy(ck, ck2)  # the resumed run keeps checkpointing into `ck`
    _same(full, b200.resume(ck, b200.options(max_batches=4)), 3)
    r_ref = ref_abi.resume(ck2, ref_abi.options(max_batches=3))
    assert r_ref.batches == 3 and np.isfinite(r_ref.final_cov_error)


def _close(r0, r1, chains):
    """A sharded run against the single engine: per-chain decisions identical, pooled moments
    to rounding (the merge sums in a different order)."""
    assert r0.batches == r1.batches and r0.total_samples == r1.total_samples
    for p in range(chains):
        assert np.array_equal(r0.chain_history(p, "beta"), r1.chain_history(p, "beta")), p
        assert np.array_equal(r0.chain_history(p, "acceptance"), r1.chain_history(p, "acceptance")), p
    assert np.linalg.norm(r0.cov() - r1.cov()) <= 1e-12 * np.linalg.norm(r0.cov())
    assert np.linalg.norm(r0.mean() - r1.mean()) <= 1e-12 * max(1.0, np.linalg.norm(r0.mean()))
    assert np.allclose(r0.history("cov_error"), r1.history("cov_error"), rtol=1e-10)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_checkpoint_resume(b200, ref_abi, tmp_path, world):
    # a run sharded over `world` ranks (in-process exchange, uneven shards for 3) checkpoints
    # into ONE reference-format file written by rank 0 (runner.cpp:398-457 for any P); the
    # file resumes on one engine, on `world` ranks again, and in the reference library
    import shutil
    t = b200.target_build("pi2", 24, 6)
    kw = dict(kernel="diam", chains=5, intervals_per_batch=2, n_lag=30, n0=20, master_seed=12)
    full = b200.sample(t, max_batches=4, **kw)
    ck = str(tmp_path / "shard.ckpt")
    part = b200.sample_threads(t, world, max_batches=2, checkpoint_path=ck, **kw)
    assert part.batches == 2 and part.chains == 5
    copies = []
    for i in range(3):
        copies.append(str(tmp_path / f"c{i}.ckpt"))
        shutil.copy(ck, copies[-1])
    _close(full, b200.resume(copies[0], b200.options(max_batches=4)), 5)
    _close(full, b200.resume_threads(copies[1], world, b200.options(max_batches=4)), 5)
    r_ref = ref_abi.resume(copies[2], ref_abi.options(max_batches=3))
    assert r_ref.batches == 3 and np.isfinite(r_ref.final_cov_error)
