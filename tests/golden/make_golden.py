"""Regenerate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (needs oracle/_ref/libdiam_ref.so, built from
/root/reference/proj/src by oracle/Makefile):

    python tests/golden/make_golden.py

Outputs (committed, small):
  rng.json            Philox u64 / uniform_open goldens of proj/tests/test_rng.cpp:31-45
                      plus more draws of the same stream, and host-libm normals
  target_pi1_d12.bin  DIAMTGT v1 file written by the reference (pi1, d=12, seed 5)
  target_pi5_d20.bin  DIAMTGT v1 file written by the reference (pi5, d=20, seed 3)
  runs.npz            reference diam_sample outputs for the four kernels on those targets
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import _oracle as O  # noqa: E402
from paper_1506_05741_b200.abi import DiamABI  # noqa: E402

RUNS = [
    # (target file, kernel, chains, M, K, n_lag, n0, seed, extra)
    ("target_pi1_d12.bin", "diam", 3, 2, 4, 24, 30, 5, {}),
    ("target_pi1_d12.bin", "am", 2, 2, 3, 20, 0, 6, {}),
    ("target_pi1_d12.bin", "rw", 2, 1, 3, 16, 10, 7, {}),
    ("target_pi1_d12.bin", "pcn", 2, 1, 3, 16, 10, 8, {}),
    ("target_pi5_d20.bin", "diam", 2, 2, 3, 40, 0, 9, {"inflation": 1.2}),
    ("target_pi1_d12.bin", "diam", 2, 2, 3, 24, 0, 10, {"adaptive_ref": 1, "n_ref_start": 30}),
]


def main():
    ref = DiamABI(O.REF_SO)
    rng = {
        "stream": [42, 0, "noise"],
        "u64_test_rng_cpp": ["10100362237944140226", "18187497329872721372", "5864986178550710854",
                             "15965594040270767174"],
        "uniform_test_rng_cpp": [0.54754173406347939, 0.9859462058561157, 0.31794153781910683,
                                 0.86549658717415934],
        "u64_more": [str(v) for v in O.fill("u64", 42, 0, "noise", 0, 64, "ref")],
        "uniform_open_7_3_uniform_100": list(O.fill("uniform_open", 7, 3, "uniform", 100, 64, "ref")),
        "normal_9_3_noise_17": list(O.fill("normal", 9, 3, "noise", 17, 64, "ref")),
    }
    with open(os.path.join(HERE, "rng.json"), "w") as f:
        json.dump(rng, f, indent=1)
    ref.target_build("pi1", 12, 5).save(os.path.join(HERE, "target_pi1_d12.bin"))
    ref.target_build("pi5", 20, 3).save(os.path.join(HERE, "target_pi5_d20.bin"))
    out = {}
    for i, (tf, kern, P, M, K, nl, n0, seed, extra) in enumerate(RUNS):
        t = ref.target_load(os.path.join(HERE, tf))
        r = ref.sample(t, kernel=kern, chains=P, intervals_per_batch=M, max_batches=K, n_lag=nl, n0=n0,
                       master_seed=seed, threads=1, record_traces=1, **extra)
        out[f"r{i}_mean"] = r.mean()
        out[f"r{i}_cov"] = r.cov()
        out[f"r{i}_cov_error"] = r.history("cov_error")
        out[f"r{i}_psrf"] = r.history("psrf")
        out[f"r{i}_beta"] = np.stack([r.chain_history(p, "beta") for p in range(P)])
        out[f"r{i}_acc"] = np.stack([r.chain_history(p, "acceptance") for p in range(P)])
        out[f"r{i}_trace_logpi_c0"] = r.trace(0, 0)
        out[f"r{i}_accumulated"] = np.array([r.accumulated_samples])
    np.savez(os.path.join(HERE, "runs.npz"), **out)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
