"""Relaxed-vs-fixed comparison with an n_crit sweep on the device.

  python tools/relaxation_study.py [--problem laplace2] [--level 6] [--out profiles/x]

Writes <out>.txt (StudyReport format) and <out>.csv and prints the derived values.
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1506_05957_b200.study import run_relaxation_comparison  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--problem", default="laplace2")
    ap.add_argument("--level", type=int, default=6)
    ap.add_argument("--tol", type=float, default=1e-6)
    ap.add_argument("--p-initial", type=int, default=12)
    ap.add_argument("--p-min", type=int, default=3)
    ap.add_argument("--ncrit", default="32,64,128,256")
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--out", default="gpurun_out/relaxation_study")
    a = ap.parse_args()
    rep = run_relaxation_comparison(a.problem, a.level, tol=a.tol, p_initial=a.p_initial,
                                    p_min=a.p_min, ncrit_candidates=[int(v) for v in a.ncrit.split(",")],
                                    repeats=a.repeats, max_iter=200)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    rep.write(a.out + ".txt")
    rep.write_csv(a.out + ".csv")
    for r in rep.records:
        print(json.dumps(r))
    print(json.dumps(rep.derived))


if __name__ == "__main__":
    main()
