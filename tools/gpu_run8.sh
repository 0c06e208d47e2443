mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
VARIANTS="_v_prev _gazemap_b200 _v_tsvec" CONFIGS="c2 c2off c5" REPS=1 EXTRA="--no-cold" bash tools/gpu_ab.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_tri_setup' -s 3 -c 1 -o gpurun_out/prof_ts_c5 -f python bench.py --config c5 --fixations 4096 --steps 1 --warmup 1 --no-cpu --no-e2e --no-stats --no-cold > gpurun_out/ncu_ts.log 2>&1
echo "ncu rc=$?"
timeout 600 python tools/accum_loop_bench.py > gpurun_out/accum_loop.json 2>&1; cat gpurun_out/accum_loop.json
