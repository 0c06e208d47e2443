mkdir -p gpurun_out; rm -f gpurun_out/variants.txt
for b in 1024 512 768 1024; do
  timeout 600 python bench.py --steps 2 --warmup 2 --batch $b --no-cpu --no-e2e --no-stats > gpurun_out/bb_$b.log 2>&1
  echo "c2 b$b $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bb_$b.log)" >> gpurun_out/variants.txt
done
