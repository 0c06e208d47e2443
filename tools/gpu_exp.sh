mkdir -p gpurun_out; rm -f gpurun_out/variants.txt
for rep in 1 2; do
for v in _v_ck1 _gazemap_b200 _v_ck4 _v_ck8; do
  GAZEMAP_B200_SO=paper_2601_07571_b200/$v.so timeout 600 python bench.py --steps 3 --warmup 2 --fixations 30720 --no-cpu --no-e2e --no-stats > gpurun_out/bv_$v.log 2>&1
  echo "c2 $v $(grep -o '"phases_ms": {[^}]*}' gpurun_out/bv_$v.log | cut -c1-120) $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bv_$v.log)" >> gpurun_out/variants.txt
done; done
