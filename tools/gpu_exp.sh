# A/B timing of build variants on the B200 (scratch runner; edit the variant list).
#   python -c "from paper_2601_07571_b200 import build as b; b.build(defines=['-DX=1'], out=b.PKG/'_v_x.so')"
#   gpurun -- 'bash tools/gpu_exp.sh'   -> gpurun_out/variants.txt
mkdir -p gpurun_out; rm -f gpurun_out/variants.txt
for v in _gazemap_b200; do
  GAZEMAP_B200_SO=paper_2601_07571_b200/$v.so timeout 600 python bench.py --steps 2 --warmup 2 --fixations 30720 \
      --no-cpu --no-e2e --no-stats > gpurun_out/bv_$v.log 2>&1
  echo "c2 $v $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bv_$v.log)" >> gpurun_out/variants.txt
done
