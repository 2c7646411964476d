"""The reference CLI's `benchmark` subcommand (proj/tools/diam_cli.cpp:
427-505) as paper_1506_05741_b200/cli/diam_bench.cpp: one driver source over the C ABI,
built against this library (paper_1506_05741_b200/diam_bench) and against the reference's
own diam.h + libdiam (oracle/_ref/diam_bench_ref). The checks are the reference's own
end-to-end ones (proj/tests/cli_e2e.sh:125-137): CSV header, the chain sweep, an empty
sweep rejected with exit code 1; on the GPU both libraries produce the same sample counts."""
import csv
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OURS = os.path.join(ROOT, "paper_1506_05741_b200", "diam_bench")
REF = os.path.join(ROOT, "oracle", "_ref", "diam_bench_ref")
DIMS = ["--target", "pi1", "--kernel", "diam", "--dims", "16", "24", "32", "--samples", "1500", "--seed", "2"]
CHAINS = ["--target", "pi1", "--dim", "12", "--kernel", "diam", "--chain-sweep", "1", "2", "--intervals", "5",
          "--max-batches", "8", "--seed", "2"]


def run(exe, args, out):
    return subprocess.run([exe, "benchmark", *args, "--out", str(out)], capture_output=True, text=True, timeout=300)


def rows(path):
    return list(csv.reader(open(path)))


def test_driver_rejects_empty_sweep_without_a_gpu(tmp_path):
    assert os.path.exists(OURS), "paper_1506_05741_b200/diam_bench not built"
    r = run(OURS, [], tmp_path / "nothing.csv")
    assert r.returncode == 1 and "needs --dims or --chain-sweep" in r.stderr
    assert run(OURS, ["--kernel", "hmc", "--dims", "8"], tmp_path / "x.csv").returncode == 1


@pytest.mark.skipif(not os.path.exists(REF), reason="reference library not built (oracle/Makefile ref)")
def test_reference_driver_e2e(tmp_path):
    r = run(REF, DIMS, tmp_path / "bench.csv")
    assert r.returncode == 0, r.stderr
    t = rows(tmp_path / "bench.csv")
    assert t[0] == ["d", "total_samples", "wall_seconds", "sec_per_sample", "sec_per_batch"]
    assert [int(x[0]) for x in t[1:]] == [16, 24, 32]
    assert "per-sample seconds fit: T =" in r.stdout
    r = run(REF, CHAINS, tmp_path / "bench_p.csv")
    assert r.returncode == 0, r.stderr
    t = rows(tmp_path / "bench_p.csv")
    assert t[0] == ["P", "total_seconds", "sec_per_batch", "N"] and [int(x[3]) for x in t[1:]] == [240, 480]
    assert run(REF, [], tmp_path / "n.csv").returncode == 1


@pytest.mark.gpu
def test_driver_on_b200_matches_reference_tables(tmp_path):
    r = run(OURS, DIMS, tmp_path / "bench.csv")
    assert r.returncode == 0, r.stderr
    ours = rows(tmp_path / "bench.csv")
    assert ours[0] == ["d", "total_samples", "wall_seconds", "sec_per_sample", "sec_per_batch"]
    # n0 = 0, max_batches = ceil(1500 / (1 chain x 10 intervals x d/2)): the reference's counts
    assert [(int(x[0]), int(x[1])) for x in ours[1:]] == [(16, 1520), (24, 1560), (32, 1600)]
    assert all(float(x[2]) > 0 and float(x[3]) > 0 for x in ours[1:])
    assert "per-sample seconds fit: T =" in r.stdout and "quadratic variance share" in r.stdout
    r = run(OURS, CHAINS, tmp_path / "bench_p.csv")
    assert r.returncode == 0, r.stderr
    p = rows(tmp_path / "bench_p.csv")
    assert p[0] == ["P", "total_seconds", "sec_per_batch", "N"] and [int(x[3]) for x in p[1:]] == [240, 480]
    # the bench dimension through the same driver: a d-sweep at the configs' sizes
    r = run(OURS, ["--target", "pi1", "--kernel", "diam", "--dims", "256", "512", "1024", "--chains", "64",
                   "--intervals", "4", "--samples", "400000", "--seed", "3"], tmp_path / "big.csv")
    assert r.returncode == 0, r.stderr
    big = rows(tmp_path / "big.csv")
    print("\n".join(",".join(x) for x in big) + "\n" + r.stdout)
    assert [int(x[0]) for x in big[1:]] == [256, 512, 1024]
