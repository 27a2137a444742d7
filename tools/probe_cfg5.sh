mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/p1_smi.txt
python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/p1_cfg5.json 2> gpurun_out/p1_cfg5.err
echo "bench rc $?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/p1_launches_cfg5.csv python bench.py --config cfg5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/p1_ncu.log 2>&1
echo "ncu rc $?"
python tools/launch_summary.py gpurun_out/p1_launches_cfg5.csv --tail 120 | head -30
