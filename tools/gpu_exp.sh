mkdir -p gpurun_out; rm -f gpurun_out/variants.txt


for v in _gazemap_b200 _v_ks4 _v_ks5 _gazemap_b200; do
  GAZEMAP_B200_SO=paper_2601_07571_b200/$v.so timeout 600 python bench.py --steps 2 --warmup 2 --fixations 30720 --no-cpu --no-e2e --no-stats > gpurun_out/bv_$v.log 2>&1
  echo "c2 $v $(grep -o '"phases_ms": {[^}]*}' gpurun_out/bv_$v.log | cut -c1-130) $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bv_$v.log)" >> gpurun_out/variants.txt
done
GAZEMAP_B200_SO=paper_2601_07571_b200/_gazemap_b200.so timeout 600 python bench.py --steps 1 --warmup 1 --fixations 10240 --no-cpu --no-e2e > gpurun_out/bv_stats.log 2>&1
