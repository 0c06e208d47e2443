# compute-sanitizer re-run on the final round-2 build (crowded-pass shared list head + warp sort, 80-byte TriF32)
mkdir -p gpurun_out
CS=compute-sanitizer
run() { name=$1; shift; timeout 1200 $CS "$@" > gpurun_out/sanitize_$name.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_$name.log; echo "== $name"; grep "ERROR SUMMARY\|RACECHECK SUMMARY\|rc=" gpurun_out/sanitize_$name.log | tail -3; }
run racecheck_c5 --tool racecheck python tools/check_run.py --config c5 --fixations 256 --any-build
run racecheck_c2 --tool racecheck python tools/check_run.py --config c2 --fixations 2048 --any-build
run racecheck_c2off --tool racecheck python tools/check_run.py --config c2 --fixations 1024 --unfiltered --any-build
run memcheck_c2 --tool memcheck python tools/check_run.py --config c2 --fixations 2048 --any-build
run memcheck_c1 --tool memcheck --leak-check full python tools/check_run.py --config c1 --any-build
run initcheck_c2 --tool initcheck python tools/check_run.py --config c2 --fixations 1024 --any-build
run synccheck_c2 --tool synccheck python tools/check_run.py --config c2 --fixations 512 --any-build
