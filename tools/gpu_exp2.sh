mkdir -p gpurun_out; rm -f gpurun_out/variants.txt
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_cd.log 2>&1; echo rc=$? >> gpurun_out/pytest_cd.log
for cfg in c2 c2off c5; do
  timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu > gpurun_out/cd_$cfg.log 2>&1
  echo "$cfg $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/cd_$cfg.log | head -2 | tr '\n' ' ')" >> gpurun_out/variants.txt
done
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_cd.log 2>&1
