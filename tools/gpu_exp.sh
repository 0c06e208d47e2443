mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu7.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu7.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench8.log 2>&1
timeout 600 python bench.py --config c5 --steps 2 --warmup 2 --no-cpu --no-e2e > gpurun_out/bench8_c5.log 2>&1
timeout 600 python bench.py --config c3k100 --steps 2 --warmup 2 --no-cpu > gpurun_out/bench8_c3.log 2>&1
