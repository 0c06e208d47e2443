mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_texels' -s 4 -c 2 -o gpurun_out/prof_tx -f python bench.py --fixations 4096 --steps 1 --warmup 1 --no-cpu --no-e2e --no-stats > gpurun_out/ncu_tx.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_tx.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_texels' -s 4 -c 1 -o gpurun_out/prof_tx_off -f python bench.py --config c2off --fixations 4096 --steps 1 --warmup 1 --no-cpu --no-e2e --no-stats > gpurun_out/ncu_tx_off.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_tx_off.log
