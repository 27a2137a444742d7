#!/bin/bash
# bench variants: VARIANTS="NAME:ENV=VAL,ENV2=VAL ..." CONFIGS="cfg5 cfg2"
mkdir -p gpurun_out
for cfg in ${CONFIGS:-cfg5}; do
for v in ${VARIANTS:-base:}; do
  name=${v%%:*}; envs=${v#*:}
  env $(echo $envs | tr ',' ' ') timeout 600 python bench.py --config $cfg --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline > gpurun_out/var_${cfg}_${name}.json 2> gpurun_out/var_${cfg}_${name}.err
  python - "$cfg" "$name" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/var_{sys.argv[1]}_{sys.argv[2]}.json").read().strip().splitlines()[-1])
    r = d["roofline"]
    print(sys.argv[1], sys.argv[2], "value %.1f e2e %.1f" % (d["value"], d["e2e"]["value"]), "orders", d["orders"],
          "stage", {k: round(v, 4) for k, v in r["stage_ms_per_apply"].items()},
          "iso", {k: round(v, 4) for k, v in r["stage_ms_per_apply_isolated"].items()}, "p2p_frac %.3f" % r["frac"])
except Exception as e:
    print(sys.argv[1], sys.argv[2], "FAILED", e)
PY
done; done
