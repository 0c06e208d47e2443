mkdir -p gpurun_out; rm -f gpurun_out/variants.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu11.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu11.log
GAZEMAP_B200_SO=paper_2601_07571_b200/_v_n4.so timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu11_n3.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu11_n3.log
for v in _gazemap_b200 _v_n4 _gazemap_b200 _v_n4; do
  GAZEMAP_B200_SO=paper_2601_07571_b200/$v.so timeout 600 python bench.py --steps 2 --warmup 2 --fixations 30720 --no-cpu --no-e2e --no-stats > gpurun_out/bv_$v.log 2>&1
  echo "c2 $v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bv_$v.log)" >> gpurun_out/variants.txt
done
