mkdir -p gpurun_out
VARIANTS="_v_prev _gazemap_b200" CONFIGS="c2 c2off c5" REPS=2 EXTRA="--no-cold" bash tools/gpu_ab.sh
