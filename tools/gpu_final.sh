# Final check of a build: GPU parity suite, smoke, default bench line (both arms).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 900 > gpurun_out/pytest_final.log 2>&1; echo rc=$? >> gpurun_out/pytest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo rc=$? >> gpurun_out/smoke_final.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_final.log 2>&1; echo rc=$? >> gpurun_out/bench_final.log
