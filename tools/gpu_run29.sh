mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
VARIANTS="_v_prev _gazemap_b200" CONFIGS="c2 c5 c2off" REPS=2 EXTRA="--no-cold" bash tools/gpu_ab.sh
