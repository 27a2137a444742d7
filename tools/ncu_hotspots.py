"""Stall reasons and the hottest SASS instructions of one kernel in an ncu --set full report.

python tools/ncu_hotspots.py REPORT.ncu-rep KERNEL_REGEX [N]
"""
import csv
import io
import subprocess
import sys


def ncu(*args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True, check=True).stdout


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv", "-k", "regex:" + kern))))
    hdr, row = raw[0], raw[2]
    print(f"kernel: {row[hdr.index('Kernel Name')][:90]}")
    stalls = []
    for k, v in zip(hdr, row):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v.replace(",", "")), k[len("smsp__average_warps_issue_stalled_"):-len(
                    "_per_issue_active.ratio")]))
            except ValueError:
                pass
    print("warp stall cycles per issued instruction:")
    for v, k in sorted(stalls, reverse=True)[:10]:
        print(f"  {k:28s} {v:7.3f}")
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "-k", "regex:" + kern,
                                          "--print-source", "sass"))))
    h = src[1]
    i_s = h.index("Warp Stall Sampling (All Samples)")
    i_e = h.index("Instructions Executed")
    data = [r for r in src[2:] if len(r) > i_s]
    tot = sum(float(r[i_s] or 0) for r in data)
    print(f"SASS: {len(data)} instructions, {int(tot)} stall samples; top {top}:")
    for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:top]:
        print(f"  {float(r[i_s] or 0) / tot * 100:5.1f}%  exec {r[i_e]:>10s}  {r[1][:80]}")
    mix = {}
    for r in data:
        op = r[1].split()[0] if not r[1].startswith("@") else r[1].split()[1]
        op = op.split(".")[0]
        mix[op] = mix.get(op, 0) + float((r[i_e] or "0").replace(",", ""))
    n = sum(mix.values())
    print("executed warp instructions by opcode (share):")
    print("  " + ", ".join(f"{k} {v / n * 100:.1f}%" for k, v in sorted(mix.items(), key=lambda x: -x[1])[:14]))


if __name__ == "__main__":
    main()
