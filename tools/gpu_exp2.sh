mkdir -p gpurun_out; rm -f gpurun_out/variants.txt
for rep in 1 2; do
for v in _gazemap_b200 _v_d2 _v_d3 _v_d5; do
  for cfg in c2 c2off c5; do
  GAZEMAP_B200_SO=paper_2601_07571_b200/$v.so timeout 600 python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu --no-e2e --no-stats > gpurun_out/bv_$v.log 2>&1
  echo "$cfg $v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bv_$v.log | head -1)" >> gpurun_out/variants.txt
  done
done
done
GAZEMAP_B200_SO=paper_2601_07571_b200/_v_d3.so timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_d3.log 2>&1; echo rc=$? >> gpurun_out/pytest_d3.log
