mkdir -p gpurun_out; rm -f gpurun_out/variants.txt
for v in _gazemap_b200 _v_cb5 _gazemap_b200 _v_cb5; do
  GAZEMAP_B200_SO=paper_2601_07571_b200/$v.so timeout 600 python bench.py --config c5 --steps 2 --warmup 1 --fixations 10000 --no-cpu --no-e2e --no-stats > gpurun_out/bv5_$v.log 2>&1
  echo "c5 $v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bv5_$v.log)" >> gpurun_out/variants.txt
  GAZEMAP_B200_SO=paper_2601_07571_b200/$v.so timeout 600 python bench.py --steps 2 --warmup 2 --fixations 30720 --no-cpu --no-e2e --no-stats > gpurun_out/bv_$v.log 2>&1
  echo "c2 $v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bv_$v.log)" >> gpurun_out/variants.txt
done
