# round-end evidence with the final code: bench (driver shape, MIXED + FP64) + ncu launch list and
# full capture of the bench step, the per-config results table, the Table 1 analogue, C4 band sweep
TAG=${TAG:-r02c}
bash scripts/gpu_bench_profiles.sh
timeout 1500 python scripts/results_table.py --out gpurun_out/${TAG}_results_table.json > gpurun_out/${TAG}_results.log 2>&1; echo results rc $?
timeout 600 python scripts/studies.py table1 --config C5 > gpurun_out/${TAG}_next3_t1_c5.json 2> gpurun_out/t1.err; echo t1 rc $?
timeout 900 python scripts/band_sweep.py --config C4 --quick 1 2 4 8 > gpurun_out/${TAG}_band_sweep_c4.txt 2>&1; echo sweep rc $?
timeout 900 python scripts/band_sweep.py --config C5 --quick 1 2 4 8 > gpurun_out/${TAG}_band_sweep_c5.txt 2>&1; echo sweep5 rc $?
