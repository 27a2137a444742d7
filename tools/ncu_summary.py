"""Per-launch summary of an ncu --set full report: time, DRAM traffic, FP64 pipe, occupancy.

python tools/ncu_summary.py REPORT.ncu-rep
"""
import csv
import io
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
     "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
     "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
     "launch__grid_size", "launch__block_size",
     "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
     "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
     "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
     "sm__ops_path_tensor_src_fp64.sum", "lts__t_sector_hit_rate.pct"]
SHORT = {"gpu__time_duration.sum": "time", "dram__bytes_read.sum": "dram_rd",
         "dram__bytes_write.sum": "dram_wr",
         "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe%",
         "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_inst%",
         "sm__issue_active.avg.pct_of_peak_sustained_elapsed": "issue%",
         "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
         "launch__registers_per_thread": "regs", "launch__grid_size": "grid",
         "launch__block_size": "block",
         "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum": "dfma",
         "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum": "dadd",
         "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum": "dmul",
         "sm__ops_path_tensor_src_fp64.sum": "dmma_ops", "lts__t_sector_hit_rate.pct": "l2_hit%"}

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics", ",".join(M)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
for r in rows[2:]:
    d, u = dict(zip(h, r)), dict(zip(h, units))
    name = d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")
    cols = [f"{SHORT[m]}={d[m]}{u[m] if u[m] not in ('', '%') else ''}" for m in M if m in d]
    print(name[:34].ljust(34), " ".join(cols))
