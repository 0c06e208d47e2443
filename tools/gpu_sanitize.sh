# compute-sanitizer memcheck / racecheck / synccheck on C1 and a C2 slice -> gpurun_out/sanitize_*.log
mkdir -p gpurun_out
CS=compute-sanitizer
run() { name=$1; shift; timeout 1500 $CS "$@" > gpurun_out/sanitize_$name.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_$name.log; tail -4 gpurun_out/sanitize_$name.log; }
run memcheck_c1 --tool memcheck --leak-check full python tools/check_run.py --config c1 --any-build
run memcheck_c2 --tool memcheck python tools/check_run.py --config c2 --fixations 2048 --any-build
run memcheck_c2off --tool memcheck python tools/check_run.py --config c2 --fixations 512 --unfiltered --any-build
run racecheck_c1 --tool racecheck python tools/check_run.py --config c1 --any-build
run racecheck_c2 --tool racecheck python tools/check_run.py --config c2 --fixations 2048 --any-build
run synccheck_c2 --tool synccheck python tools/check_run.py --config c2 --fixations 512 --any-build
run initcheck_c1 --tool initcheck python tools/check_run.py --config c1 --any-build
