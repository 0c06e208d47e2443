mkdir -p gpurun_out
python tools/check_crowded.py > gpurun_out/crowded.log 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu8.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu8.log
