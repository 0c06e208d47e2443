mkdir -p gpurun_out
VARIANTS="_gazemap_b200 _v_cap64 _v_full16" CONFIGS="c2 c2off c5" REPS=1 EXTRA="--no-cold" bash tools/gpu_ab.sh
GM_BENCH_DEVICE_MOD=1 GM_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config c4 --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_g2_c4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_g2_c4.log
tail -c 1500 gpurun_out/bench_g2_c4.log
