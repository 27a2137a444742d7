"""Selected raw metrics of one kernel in an ncu report (L1/shared-memory pipeline, pipes, stalls).

python tools/ncu_raw.py REPORT.ncu-rep KERNEL_REGEX [METRIC_REGEX]
"""
import csv
import io
import re
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
pat = re.compile(sys.argv[3] if len(sys.argv) > 3 else
                 r"l1tex__(data_pipe|data_bank|lsu_writeback|throughput|f_wavefronts|t_sectors_pipe_lsu_mem_global_op_(ld|st)\.sum$|m_xbar)"
                 r"|shared|smsp__inst_executed_pipe|sm__inst_executed_pipe|sm__pipe_fp64|smsp__inst_executed\.sum$|"
                 r"gpu__time_duration|sm__throughput|lts__throughput|smsp__warp_issue_stalled.*_per_warp_active")
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", "regex:" + kern],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
names, units = rows[0], rows[1]
for r in rows[2:]:
    print("==", r[names.index("Kernel Name")][:60])
    for n, u, v in zip(names, units, r):
        if pat.search(n) and v not in ("", "0", "0.0", "n/a"):
            print(f"{n:90s} {v:>18s} {u}")
