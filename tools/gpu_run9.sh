mkdir -p gpurun_out
bash tools/gpu_checkfull.sh
bash tools/gpu_sanitize.sh
