mkdir -p gpurun_out; rm -f gpurun_out/variants.txt
for v in _gazemap_b200; do
  for cfg in c2 c2off c5; do
  GAZEMAP_B200_SO=paper_2601_07571_b200/$v.so timeout 600 python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/bv_$v.log 2>&1
  echo "$cfg $v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bv_$v.log | head -1) $(grep -o '"phases_single_stream_ms": {[^}]*}' gpurun_out/bv_$v.log) $(grep -o '"texel_pairs": [0-9]*' gpurun_out/bv_$v.log)" >> gpurun_out/variants.txt
  done
done
