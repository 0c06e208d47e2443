mkdir -p gpurun_out
VARIANTS="_v_prev _gazemap_b200" CONFIGS="c2 c5 c2off" REPS=1 EXTRA="--no-cold" bash tools/gpu_ab.sh
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "scale_parity or fullsize or parity" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
