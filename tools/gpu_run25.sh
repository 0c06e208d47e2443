mkdir -p gpurun_out
VARIANTS="_gazemap_b200 _v_rc128 _v_rc256" CONFIGS="c2 c5 c2off" REPS=1 EXTRA="--no-cold" bash tools/gpu_ab.sh
timeout 600 python tools/accum_loop_bench.py
