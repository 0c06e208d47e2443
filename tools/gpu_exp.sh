mkdir -p gpurun_out; rm -f gpurun_out/variants.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu17.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu17.log
for v in _v_head _gazemap_b200 _v_head _gazemap_b200; do
  GAZEMAP_B200_SO=paper_2601_07571_b200/$v.so timeout 600 python bench.py --steps 2 --warmup 2 --fixations 30720 --no-cpu --no-e2e --no-stats > gpurun_out/bv_$v.log 2>&1
  echo "c2 $v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bv_$v.log) $(grep -o '"mark": [0-9.]*' gpurun_out/bv_$v.log | tail -1)" >> gpurun_out/variants.txt
done
