"""Loop bodies of one kernel in an ncu --set full report: SASS instructions grouped by their
executed count (one group per loop), with the opcode mix and the stall samples of each group.

python tools/ncu_loops.py REPORT.ncu-rep KERNEL_REGEX [MIN_INSTRUCTIONS]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    min_n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern, "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    src = list(csv.reader(io.StringIO(out)))
    h = src[1]
    i_s = h.index("Warp Stall Sampling (All Samples)")
    i_e = h.index("Instructions Executed")
    data = [r for r in src[2:] if len(r) > i_s]
    tot = sum(float(r[i_s] or 0) for r in data)
    groups = {}
    for r in data:
        e = int((r[i_e] or "0").replace(",", ""))
        groups.setdefault(e, []).append(r)
    for e, rs in sorted(groups.items(), key=lambda kv: -kv[0] * len(kv[1])):
        if len(rs) < min_n or e == 0:
            continue
        mix = {}
        for r in rs:
            t = r[1].split()
            op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
            mix[op] = mix.get(op, 0) + 1
        st = sum(float(r[i_s] or 0) for r in rs)
        print(f"exec {e:>10d} x {len(rs):4d} instr  stall samples {st / tot * 100:5.1f}%  "
              + ", ".join(f"{k} {v}" for k, v in sorted(mix.items(), key=lambda x: -x[1])))
        # stall reasons of the group (share of the group's samples)
        reasons = {}
        for i, nme in enumerate(h):
            if nme.startswith("stall_") and "Not Issued" not in nme:
                v = sum(float(r[i] or 0) for r in rs if i < len(r))
                if v:
                    reasons[nme[6:]] = v
        tr = sum(reasons.values()) or 1.0
        print("      " + ", ".join(f"{k} {v / tr * 100:.0f}%" for k, v in sorted(reasons.items(), key=lambda x: -x[1])[:7]))


if __name__ == "__main__":
    main()
