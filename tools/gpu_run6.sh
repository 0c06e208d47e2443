mkdir -p gpurun_out
VARIANTS="_v_prev _v_crowdall _v_crowdall4 _v_hv4" CONFIGS="c2off c2 c5" REPS=1 EXTRA="--no-cold" bash tools/gpu_ab.sh
