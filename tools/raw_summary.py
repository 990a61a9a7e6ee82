"""Key metrics from an ncu raw-page CSV: python tools/raw_summary.py raw.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, u, v = rows[0], rows[1], rows[2]
for k in ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed.avg.per_cycle_active",
          "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
          "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum",
          "dram__bytes_write.sum"]:
    if k in h:
        print(f"  {k:60s} {v[h.index(k)]:>14s} {u[h.index(k)]}")
