mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_p2p.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_p2p.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p2p.log
tail -3 gpurun_out/pytest_p2p.log
VARIANTS="_gazemap_b200 _v_c96 _v_nw4 _v_tw1 _v_tw4" CONFIGS="c2 c5" REPS=1 EXTRA="--no-cold" bash tools/gpu_ab.sh
