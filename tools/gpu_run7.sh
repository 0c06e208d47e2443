mkdir -p gpurun_out
VARIANTS="_v_prev _v_ca1 _v_ca2 _v_crowdall4 _v_hv1" CONFIGS="c2 c5" REPS=1 EXTRA="--no-cold" bash tools/gpu_ab.sh
