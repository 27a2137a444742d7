#!/bin/bash
# round-2 GPU check: gpu tests, cfg5 bench line (with the CPU leg), a short reference arm
mkdir -p gpurun_out
nproc > gpurun_out/r2_nproc.txt; free -g >> gpurun_out/r2_nproc.txt
( time timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:-} ) > gpurun_out/r2_gputests.log 2>&1; echo "gpu tests exit $?"
tail -5 gpurun_out/r2_gputests.log
( time timeout 1200 python bench.py --steps 20 --warmup 5 ) > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench exit $?"
tail -4 gpurun_out/r2_bench.err
if [ "${REF:-1}" = 1 ]; then
( time timeout 1500 python bench.py --impl reference --steps ${REF_STEPS:-3} --warmup 1 ) > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err; echo "ref exit $?"
tail -4 gpurun_out/r2_bench_ref.err
fi
