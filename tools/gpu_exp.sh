mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu3.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu3.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c2.log 2>&1
for c in c2off c3k1 c3k3 c3k10 c3k30 c3k100 c5; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_$c.log 2>&1
done
timeout 900 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu > gpurun_out/bench_c4.log 2>&1
