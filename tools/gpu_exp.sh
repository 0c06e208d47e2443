mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu5.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu5.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench5.log 2>&1
