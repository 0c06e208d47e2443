mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_rb.log 2>&1; echo rc=$? >> gpurun_out/pytest_rb.log
for c in c2 c3k100 c3k30 c5; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/rb_$c.log 2>&1; done
