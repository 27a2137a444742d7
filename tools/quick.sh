#!/bin/bash
# quick GPU check: gpu tests, bench summary, per-kernel launch times of one bench run
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --steps 20 --warmup 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); [print(k, d[k]) for k in (\"value\",\"stage_ms_per_apply\") if k in d]"
ncu --metrics gpu__time_duration.sum --clock-control none -c 220 --csv --log-file gpurun_out/lq.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/lq.csv --tail 60 2>/dev/null | head -${1:-16}
