# Round-end evidence: GPU suite, smoke, bench (both arms), configs, launch list, ncu --set full capture
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 4 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
rm -f gpurun_out/configs.jsonl
for c in c1 c2off c3k1 c3k3 c3k10 c3k30 c3k100 c4 c5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_$c.log 2>&1
  grep '^{' gpurun_out/bench_$c.log >> gpurun_out/configs.jsonl
done
for c in c2off c5; do
  timeout 900 python bench.py --impl reference --config $c --steps 2 --warmup 1 > gpurun_out/bench_ref_$c.log 2>&1
  grep '^{' gpurun_out/bench_ref_$c.log >> gpurun_out/configs_ref.jsonl
done
timeout 600 python tools/accum_loop_bench.py > gpurun_out/accum_loop.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_final.csv python bench.py --fixations 10240 --steps 1 --warmup 2 --no-cpu --no-e2e --no-stats --no-cold > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tri_setup|k_samples|k_texels|k_coarse|k_level1|k_mark' -s 16 -c 8 -o gpurun_out/prof_final -f python bench.py --fixations 6144 --steps 1 --warmup 1 --no-cpu --no-e2e --no-stats --no-cold > gpurun_out/ncu_full.log 2>&1
echo "done"
