mkdir -p gpurun_out
VARIANTS="_v_base _gazemap_b200 _v_rank32 _v_rank0" CONFIGS="c2 c2off c5" REPS=1 EXTRA="--no-cold" bash tools/gpu_ab.sh
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo "rc=$?" >> gpurun_out/bench_full.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
GM_BENCH_DEVICE_MOD=1 GM_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --fixations 20000 --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_g2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_g2.log
