#!/bin/bash
# One GPU session: gpu tests, bench line, launch list, ncu --set full of the hot kernels.
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "gpu tests exit $?" >> gpurun_out/gputests.log
tail -3 gpurun_out/gputests.log
python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
tail -1 gpurun_out/bench.json
[ "${REF:-1}" = 1 ] && python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv --tail 200 | head -25
if [ "${FULL:-1}" = 1 ]; then
ncu --set full --clock-control none --import-source on -k regex:"k_p2p|k_m2l_rot|k_p2m_basis|k_epilogue|k_arnoldi|k_m2l_gather" \
    --launch-skip 10 -c 8 -o gpurun_out/full -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "ncu full exit $?"
fi
