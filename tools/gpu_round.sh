# One GPU round: parity tests, smoke, bench (both arms), every BASELINE config, launch list, one ncu --set full capture.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x --durations=12 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1
echo "rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
echo "rc=$?" >> gpurun_out/bench_ref.log
rm -f gpurun_out/configs.jsonl
for c in c2off c3k1 c3k3 c3k10 c3k30 c3k100 c5; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_$c.log 2>&1
  grep '^{' gpurun_out/bench_$c.log >> gpurun_out/configs.jsonl
done
timeout 900 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu > gpurun_out/bench_c4.log 2>&1
grep '^{' gpurun_out/bench_c4.log >> gpurun_out/configs.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches.csv python bench.py --fixations 10240 --steps 1 --warmup 2 --no-cpu --no-e2e --no-stats > gpurun_out/ncu_launches.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tri_setup|k_samples|k_texels|k_coarse|k_level1|k_mark' -s 80 -c 8 -o gpurun_out/prof_r1b -f python bench.py --fixations 4096 --steps 1 --warmup 3 --no-cpu --no-e2e --no-stats > gpurun_out/ncu_full.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full.log
