mkdir -p gpurun_out
bash tools/gpu_checkfull.sh
CS=compute-sanitizer
timeout 900 $CS --tool initcheck python tools/check_run.py --config c1 --any-build > gpurun_out/sanitize_initcheck_c1.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_initcheck_c1.log
timeout 900 $CS --tool initcheck python tools/check_run.py --config c2 --fixations 1024 --any-build > gpurun_out/sanitize_initcheck_c2.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_initcheck_c2.log
timeout 900 $CS --tool memcheck --leak-check full python tools/check_run.py --config c1 --any-build > gpurun_out/sanitize_memcheck_c1.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_memcheck_c1.log
timeout 900 $CS --tool racecheck python tools/check_run.py --config c5 --fixations 256 --any-build > gpurun_out/sanitize_racecheck_c5.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_racecheck_c5.log
timeout 900 $CS --tool racecheck python tools/check_run.py --config c2 --fixations 1024 --unfiltered --any-build > gpurun_out/sanitize_racecheck_c2off.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_racecheck_c2off.log
grep "ERROR SUMMARY\|RACECHECK SUMMARY" gpurun_out/sanitize_*.log
bash tools/gpu_prof_c2.sh
