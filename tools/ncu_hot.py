"""Top SASS lines by warp-stall samples for one kernel of an .ncu-rep.

python tools/ncu_hot.py REPORT KERNEL_REGEX [launch_skip] [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}", "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1] if len(rows) > 1 else sys.exit("no rows")
data = [r for r in rows[2:] if len(r) == len(h)]
si = h.index("Warp Stall Sampling (All Samples)")
src = h.index("Source")
ie = h.index("Instructions Executed")
stall = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
tot = sum(int(r[si]) for r in data if r[si].isdigit())
print("samples", tot, "warp-instructions", sum(int(r[ie]) for r in data if r[ie].isdigit()))
agg = {}
for r in data:
    for i in stall:
        if r[i].isdigit():
            agg[h[i]] = agg.get(h[i], 0) + int(r[i])
print(sorted(agg.items(), key=lambda x: -x[1])[:8])
for r in sorted(data, key=lambda r: -int(r[si]) if r[si].isdigit() else 0)[:top]:
    st = sorted([(int(r[i]), h[i][6:]) for i in stall if r[i].isdigit() and int(r[i]) > 0], reverse=True)[:3]
    print(r[si].rjust(6), r[ie].rjust(9), r[src].strip()[:58].ljust(58), st)
