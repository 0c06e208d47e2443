mkdir -p gpurun_out
VARIANTS="_gazemap_b200 _v_tl" CONFIGS="c2 c5 c2off" REPS=2 EXTRA="--no-cold" bash tools/gpu_ab.sh
