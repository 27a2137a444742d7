#!/bin/bash
# bench value + isolated stage times per env variant (quick A/B on the GPU box)
for cfg in ${VARIANTS:-"X=1" "FMMBEM_SERIAL=1"}; do
  for r in 1 2; do
  echo "$cfg: $(env $cfg python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["e2e"]["value"]), {k: round(v*1e3,1) for k,v in d["roofline"]["stage_ms_per_apply"].items()})')"
  done
done
