mkdir -p gpurun_out
VARIANTS="_v_prev _gazemap_b200 _v_tw2" CONFIGS="c2 c5 c2off" REPS=2 EXTRA="--no-cold" bash tools/gpu_ab.sh
