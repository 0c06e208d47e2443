mkdir -p gpurun_out
VARIANTS="_gazemap_b200 _v_cap96 _v_cap128 _v_cap64r32" CONFIGS="c2 c5 c2off" REPS=1 EXTRA="--no-cold" bash tools/gpu_ab.sh
