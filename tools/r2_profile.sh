#!/bin/bash
# Round-2 GPU session: gpu tests, the cfg5 bench line, the launch list, ncu --set full of the
# apply kernels and of the setup / vector kernels (verdict: per-kernel roofline evidence).
# Outputs under gpurun_out/r2prof/ (copy the summaries worth keeping into profiles/).
O=gpurun_out/r2prof
R=/tmp/r2rep; mkdir -p $R
mkdir -p $O
if [ "${TESTS:-1}" = 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo "gpu tests exit $?"; tail -2 $O/gputests.log
fi
if [ "${BENCH:-1}" = 1 ]; then
  timeout 1200 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench exit $?"
  timeout 1200 python bench.py --impl reference --steps ${REF_STEPS:-3} --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref exit $?"
fi
if [ "${NCU:-1}" = 1 ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "launch list exit $?"
  python tools/launch_summary.py $O/launches.csv --tail 160 > $O/launch_summary.txt 2>&1
  head -30 $O/launch_summary.txt
  # apply kernels of a p = 14 apply (skip the warm-up solves' launches)
  ncu --set full --import-source on --clock-control none \
      -k regex:"k_p2p_lapd|k_m2l_rot|k_p2m_basis_cl|k_vrot|k_epilogue|k_arnoldi|k_m2l_gather|k_children_sum" \
      --launch-skip 40 -c 14 -o $R/apply -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_apply.log 2>&1
  echo "ncu apply exit $?"
  python tools/ncu_summary.py $R/apply.ncu-rep > $O/apply_summary.txt 2>&1
  # setup kernels (tree build, traversal, near pairs, correction assembly)
  ncu --set full --clock-control none \
      -k regex:"k_bbox|k_path_keys|k_heads|k_emit|k_finish_bodies|k_traverse|k_near|k_corr_values|k_grid_keys|Onesweep" \
      -c 24 -o $R/setup -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_setup.log 2>&1
  echo "ncu setup exit $?"
  python tools/ncu_summary.py $R/setup.ncu-rep > $O/setup_summary.txt 2>&1
  cat $O/apply_summary.txt $O/setup_summary.txt | cut -c1-220
fi
