mkdir -p gpurun_out
timeout 600 python bench.py --steps 1 --warmup 3 --fixations 20000 --no-cpu --no-e2e > gpurun_out/bench3.log 2>&1
