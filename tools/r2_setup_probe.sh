CONFIGS="cfg5" VARIANTS="base: c100:FMMBEM_P2P_CARVEOUT=100 c100r:FMMBEM_P2P_CARVEOUT=100,FMMBEM_NEAR_PRIO_HIGH=1" STEPS=10 bash tools/variants.sh
CONFIGS="cfg2" VARIANTS="base: c100:FMMBEM_P2P_CARVEOUT=100" STEPS=10 bash tools/variants.sh
mkdir -p gpurun_out/r2prof /tmp/r2rep
ncu --set full --clock-control none -k regex:"k_traverse|k_near|k_corr_values|k_cutoffs|k_cell_ranges|k_grid_keys|k_finish_bodies|k_leaf" -c 40 -o /tmp/r2rep/setup2 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2prof/ncu_setup2.log 2>&1
python tools/ncu_summary.py /tmp/r2rep/setup2.ncu-rep > gpurun_out/r2prof/setup2_summary.txt 2>&1
cut -c1-200 gpurun_out/r2prof/setup2_summary.txt | head -40
