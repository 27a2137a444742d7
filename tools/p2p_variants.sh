#!/bin/bash
# P2P kernel time (ncu launch list, serialised) per variant (env assignments) on one config.
cfg=${1:-cfg2}; p=${2:-12}
for v in ${VARIANTS:-FMMBEM_P2P_STAGES=2 FMMBEM_P2P_STAGES=3}; do
  env $v ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_p2p --csv \
      --log-file gpurun_out/var.csv python tools/apply_once.py $cfg $p 3 > /dev/null 2>&1
  echo "$cfg $v $(python tools/launch_summary.py gpurun_out/var.csv | sed -n 2p)"
done
