mkdir -p gpurun_out
for b in 512 1024 256; do
timeout 600 python bench.py --steps 2 --warmup 3 --batch $b --no-cpu --no-e2e > gpurun_out/bench_b$b.log 2>&1
done
