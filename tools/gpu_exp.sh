mkdir -p gpurun_out
timeout 600 python bench.py --steps 2 --warmup 2 --fixations 20480 --no-cpu > gpurun_out/bench7.log 2>&1
GM_BENCH_BACKEND=gloo GM_BENCH_DEVICE_MOD=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 2 --warmup 1 --fixations 8192 > gpurun_out/bench7_2rank.log 2>&1
echo "rc=$?" >> gpurun_out/bench7_2rank.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 --cpu-fixations 20 > gpurun_out/bench7_ref2.log 2>&1
echo "rc=$?" >> gpurun_out/bench7_ref2.log
