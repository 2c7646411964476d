"""Kernel-class shares of one steady-state batch from an `ncu --metrics
gpu__time_duration.sum` launch list (cold-cache, serialised), next to bench.py's own
CUDA-event per-class times (`roofline.per_class_ms`, single stream).

    python tools/launch_shares.py profiles/r02_launches_d1024.csv profiles/r02_bench_d1024_groups1.json

(round 1's CSV classified with round 1's kernel names: git show 306b434:tools/launch_shares.py)
"""
import collections
import csv
import json
import sys


def cls(name, grid):
    if "gemm_f64_kernel" in name:
        gx, gy, gz = eval(grid)  # "(x, y, z)"
        if ", 0, 0," in name:
            return "syrk_moments"  # the only MN-major x MN-major GEMM
        if "Cfg<64, 64," in name:
            # 64 x 64 tiles: the accepted-rows product (d/64 column tiles) or the
            # factorization's long-K updates (128 columns: 2 tiles)
            return "xi_accepted" if gx > 2 else "potrf"
        if gz == 1 and gy >= 8:
            return "merge"  # the x-space snapshot G^-1 S_gz G^-T (two d x d products per batch)
        if gz > 1 and gx == 16 and gy == 4:
            return "trmm_noise"  # batched n_lag x d per chain
        if gz == 1 and gy == 1:
            return "gemv_state"
        return "potrf"  # the narrow last block column's TRSM
    for k in ("potrf_diag", "potrf_trsm", "gemv_rows", "mh_window", "normals", "blend_cov", "mean_update",
              "reconstruct", "sum_chains", "merge_lower", "adopt_factor"):
        if k in name:
            return "potrf" if k.startswith("potrf") else "gemv_state" if k == "gemv_rows" else k
    return "other"


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    h, rows = rows[0], rows[1:]
    ki, gi, vi = h.index("Kernel Name"), h.index("Grid Size"), h.index("Metric Value")
    starts = [i for i, r in enumerate(rows) if "normals_kernel" in r[ki]]
    # exactly the second batch: its 4 windows start at the 5th..8th normals launch, the next
    # batch (or the bench's later phases: the live DMMA peak, the profile pass) at the 9th
    first = starts[4] if len(starts) > 4 else 0
    last = starts[8] if len(starts) > 8 else len(rows)
    agg = collections.defaultdict(float)
    for r in rows[first:last]:
        agg[cls(r[ki], r[gi])] += float(r[vi].replace(",", ""))
    tot = sum(agg.values())
    bench = json.load(open(sys.argv[2]))["roofline"]["per_class_ms"]
    btot = sum(bench.values())
    print("| class | ncu launch list share | bench CUDA-event share |")
    print("|---|---:|---:|")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
        b = bench.get(k)
        print(f"| {k} | {100 * v / tot:.1f}% | " + (f"{100 * b / btot:.1f}% |" if b else "– |"))


if __name__ == "__main__":
    main()
