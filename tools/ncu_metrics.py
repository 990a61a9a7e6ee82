"""Key walk-kernel metrics from an ncu raw-page CSV (header, units, values
rows) as "metric,value,unit" lines -- the per-config files bench.py reads
(profiles/r02_cfg*_walk_f32_ncu_metrics.csv):
    python tools/ncu_metrics.py raw.csv > profiles/r02_cfgC_walk_f32_ncu_metrics.csv"""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "sm__inst_executed.sum",
        "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "lts__t_bytes.sum",
        "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
        "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__occupancy_limit_registers"]

rows = list(csv.reader(open(sys.argv[1])))
h, u, v = rows[0], rows[1], rows[2]
print("metric,value,unit")
for k in KEYS:
    if k in h:
        print(f"{k},{v[h.index(k)].replace(',', '')},{u[h.index(k)]}")
