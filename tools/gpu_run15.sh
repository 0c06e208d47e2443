mkdir -p gpurun_out
VARIANTS="_v_prev _gazemap_b200 _v_agg12 _v_agg32" CONFIGS="c2 c5" REPS=1 EXTRA="--no-cold" bash tools/gpu_ab.sh
