mkdir -p gpurun_out; rm -f gpurun_out/rep.log
GAZEMAP_B200_SO=paper_2601_07571_b200/_v_chk.so timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/chk_all.log 2>&1
GAZEMAP_B200_SO=paper_2601_07571_b200/_v_chk.so timeout 600 python bench.py --steps 1 --warmup 0 --fixations 4096 --no-cpu --no-e2e --no-stats > gpurun_out/chk_bench.log 2>&1
GAZEMAP_B200_SO=paper_2601_07571_b200/_v_chk.so timeout 600 python bench.py --config c2off --steps 1 --warmup 0 --fixations 2048 --no-cpu --no-e2e --no-stats > gpurun_out/chk_bench2.log 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu10.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu10.log
for i in 1 2; do timeout 600 python bench.py --steps 2 --warmup 2 --fixations 30720 --no-cpu --no-e2e --no-stats 2>&1 | grep -o '"ms_per_step": [0-9.]*' >> gpurun_out/rep.log; done
