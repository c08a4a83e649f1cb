"""Key metrics of `ncu --set full` captures (raw CSV pages, one file per capture):
  python tools/ncu_key_metrics.py gpurun_out/prof_*_raw.csv > profiles/rNN_ncu_full_key_metrics.csv"""
import csv
import os
import sys

COLS = ["Kernel Name", "launch__grid_size", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__cycles_elapsed.avg.per_second", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"]


def main(paths):
    w = csv.writer(sys.stdout)
    w.writerow(["capture"] + COLS)
    for p in paths:
        rows = list(csv.reader(open(p)))
        if len(rows) < 3:
            continue
        head, units = rows[0], rows[1]
        for r in rows[2:]:
            out = [os.path.basename(p).replace("_raw.csv", "")]
            for c in COLS:
                if c in head:
                    i = head.index(c)
                    out.append(f"{r[i]} {units[i]}".strip() if units[i] else r[i])
                else:
                    out.append("")
            w.writerow(out)


if __name__ == "__main__":
    main(sys.argv[1:])
