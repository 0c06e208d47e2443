# A/B timing of build variants on the B200 (scratch runner; edit the variant list).
#   python -c "from paper_2601_07571_b200 import build as b; b.build(defines=['-DX=1'], out=b.PKG/'_v_x.so')"
#   gpurun -- 'bash tools/gpu_exp.sh'   -> gpurun_out/variants.txt
mkdir -p gpurun_out; rm -f gpurun_out/variants.txt
for rep in 1 2; do
for v in _v_base _gazemap_b200; do
  for cfg in c2 c5; do
  GAZEMAP_B200_SO=paper_2601_07571_b200/$v.so timeout 600 python bench.py --config $cfg --steps 3 --warmup 2 \
      --no-cpu --no-e2e --no-stats > gpurun_out/bv_$v.log 2>&1
  echo "$cfg $v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bv_$v.log)" >> gpurun_out/variants.txt
  done
done
done
