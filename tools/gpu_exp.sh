mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -p no:cacheprovider -k "generate_vs_oracle" --durations=8 > gpurun_out/pytest_gpu16.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu16.log
