"""Summarise the ncu captures of tools/ncu_capture.sh into profiles/.

    python tools/ncu_summary.py r01

For every gpurun_out/<tag>_<kernel>.ncu-rep: the raw-page metrics that the roofline
needs (duration, DRAM bytes, pipe utilisation, occupancy) -> profiles/<tag>_ncu_<kernel>.csv,
and one table of all kernels -> profiles/<tag>_ncu_summary.md.
"""
import csv
import glob
import io
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_shared_mem",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_sector_hit_rate.pct",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    return rows[0], rows[1], rows[2:]


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    reps = sorted(glob.glob(os.path.join(ROOT, "gpurun_out", f"{tag}_*.ncu-rep")))
    lines = ["| kernel | launch | time (us) | DRAM read MB | DRAM write MB | SM thr % | FP64 tensor ops % of peak | warps active % |",
             "|---|---|---:|---:|---:|---:|---:|---:|"]
    for rep in reps:
        name = os.path.basename(rep)[len(tag) + 1:-len(".ncu-rep")]
        hdr, units, rows = raw(rep)
        # section-prefixed names ("TPC.TriageCompute.sm__...") -> bare metric names
        hdr = [next((m for m in METRICS if h == m or h.endswith("." + m)), h) for h in hdr]
        keep = [i for i, h in enumerate(hdr) if h in METRICS or h in ("Kernel Name", "Grid Size", "Block Size")]
        path = os.path.join(ROOT, "profiles", f"{tag}_ncu_{name}.csv")
        with open(path, "w", newline="") as f:
            w = csv.writer(f)
            w.writerow([hdr[i] for i in keep])
            w.writerow([units[i] for i in keep])
            for r in rows:
                w.writerow([r[i] for i in keep])
        r = rows[0]

        def get(m, scale=1.0):
            if m not in hdr:
                return ""
            v = r[hdr.index(m)].replace(",", "")
            u = units[hdr.index(m)]
            try:
                x = float(v)
            except ValueError:
                return v
            if u == "ms":
                x *= 1e3
            elif u == "ns":
                x *= 1e-3
            elif u == "Gbyte":
                x *= 1e3
            elif u == "Kbyte":
                x *= 1e-3
            elif u == "byte":
                x *= 1e-6
            return f"{x * scale:.1f}"
        kname = r[hdr.index("Kernel Name")][:60]
        lines.append(f"| {name} | `{kname}` | {get('gpu__time_duration.sum')} | {get('dram__bytes_read.sum')} | "
                     f"{get('dram__bytes_write.sum')} | {get('sm__throughput.avg.pct_of_peak_sustained_elapsed')} | "
                     f"{get('sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed')} | "
                     f"{get('sm__warps_active.avg.pct_of_peak_sustained_active')} |")
        print("wrote", path)
    md = os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md")
    with open(md, "w") as f:
        f.write(f"# ncu --set full summaries ({tag}), tools/ncu_capture.sh on one B200, --clock-control none\n\n")
        f.write("\n".join(lines) + "\n")
    print("wrote", md)


if __name__ == "__main__":
    main()
