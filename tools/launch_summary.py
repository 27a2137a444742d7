"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

Usage: python tools/launch_summary.py gpurun_out/launches.csv [--skip-setup] [--tail N]
Prints kernel, launches, total/avg duration (us) and share of the listed time.
ncu launch times are cold-cache and serialised: compare SHARES, not absolutes.
"""

import collections
import csv
import sys

SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
SETUP = ("k_bbox", "k_path_keys", "k_classify", "k_heads", "k_emit", "k_child_counts",
         "k_leaf_", "k_finish_bodies", "k_fill_half", "k_traverse", "k_igrid", "k_rshift",
         "k_cutoffs", "k_grid_keys", "k_cell_ranges", "k_near", "k_corr_values",
         "k_sorted_sources", "cub::", "k_dfma_probe", "at::", "k_permute")


def main(path, skip_setup=False, tail=0):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    data = [d for d in data if d["Metric Name"] == "gpu__time_duration.sum"]
    for d in data[-tail:] if tail else data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("fmmbem::", "").replace("<unnamed>::", "")
        if skip_setup and any(s in name for s in SETUP):
            continue
        v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values()) or 1.0
    print(f"{'kernel':48s} {'n':>5s} {'total_us':>10s} {'share':>6s} {'avg_us':>9s}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:48]:48s} {n:5d} {t:10.1f} {100 * t / tot:5.1f}% {t / n:9.2f}")


if __name__ == "__main__":
    a = sys.argv
    main(a[1], "--skip-setup" in a, int(a[a.index("--tail") + 1]) if "--tail" in a else 0)
