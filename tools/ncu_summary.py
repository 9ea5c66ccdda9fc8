"""Compact per-launch summary of an ncu report (key throughput / stall metrics).

    python tools/ncu_summary.py gpurun_out/prof_aca.ncu-rep > profiles/r01_ncu_full_aca_U32k.csv
"""
import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    w = csv.writer(sys.stdout)
    keep = ["Kernel Name"] + [m for m in METRICS if m in hdr]
    w.writerow(keep)
    w.writerow([""] + [units[hdr.index(m)] for m in keep[1:]])
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"]
        name = name.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")
        w.writerow([name] + [d[m] for m in keep[1:]])


if __name__ == "__main__":
    main(sys.argv[1])
