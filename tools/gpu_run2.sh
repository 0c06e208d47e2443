mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
VARIANTS="_v_base _gazemap_b200" CONFIGS="c2 c2off c5" REPS=2 bash tools/gpu_ab.sh
