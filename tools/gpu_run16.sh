mkdir -p gpurun_out
VARIANTS="_gazemap_b200 _v_th32 _v_tw4 _v_tw1" CONFIGS="c2 c2off c5" REPS=1 EXTRA="--no-cold" bash tools/gpu_ab.sh
