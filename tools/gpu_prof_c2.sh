# ncu --set full (source) of the C2 batch kernels + launch list -> gpurun_out/prof_c2_r2.ncu-rep, launches_r2.csv
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tri_setup|k_samples|k_texels|k_coarse|k_level1|k_mark' -s 16 -c 8 -o gpurun_out/prof_c2_r2 -f python bench.py --fixations 6144 --steps 1 --warmup 1 --no-cpu --no-e2e --no-stats --no-cold > gpurun_out/ncu_full_r2.log 2>&1
echo "ncu full rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_r2.csv python bench.py --fixations 10240 --steps 1 --warmup 2 --no-cpu --no-e2e --no-stats --no-cold > gpurun_out/ncu_launches_r2.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_texels' -s 4 -c 2 -o gpurun_out/prof_c2off_r2 -f python bench.py --config c2off --fixations 4096 --steps 1 --warmup 1 --no-cpu --no-e2e --no-stats --no-cold > gpurun_out/ncu_off_r2.log 2>&1
echo "ncu off rc=$?"
