mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
VARIANTS="_v_prev _gazemap_b200" CONFIGS="c2 c2off c5 c3k100" REPS=1 EXTRA="--no-cold" bash tools/gpu_ab.sh
CS=compute-sanitizer
timeout 900 $CS --tool initcheck python tools/check_run.py --config c1 --any-build > gpurun_out/sanitize_initcheck_c1.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_initcheck_c1.log
timeout 900 $CS --tool memcheck --leak-check full python tools/check_run.py --config c1 --any-build > gpurun_out/sanitize_memcheck_c1.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_memcheck_c1.log
grep "ERROR SUMMARY" gpurun_out/sanitize_*c1.log
