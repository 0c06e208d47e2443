mkdir -p gpurun_out; rm -f gpurun_out/variants.txt
for rep in 1 2; do
for v in _gazemap_b200 _v_ts1 _v_ts4 _v_ts8; do
  for cfg in c2 c5; do
  GAZEMAP_B200_SO=paper_2601_07571_b200/$v.so timeout 600 python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu --no-e2e --no-stats > gpurun_out/bv_$v.log 2>&1
  echo "$cfg $v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bv_$v.log | head -1)" >> gpurun_out/variants.txt
  done
done
done
