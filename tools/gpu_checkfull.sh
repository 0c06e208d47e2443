# Full-stream self-check runs of the GM_CHECK build -> gpurun_out/check_full.jsonl
mkdir -p gpurun_out; rm -f gpurun_out/check_full.jsonl gpurun_out/check_rc.txt
export GAZEMAP_B200_SO=paper_2601_07571_b200/_gazemap_b200_check.so
for args in "--config c2" "--config c2 --unfiltered" "--config c5" "--config c3k100" "--config c3k30" "--config c4"; do
  timeout 1800 python tools/check_run.py $args >> gpurun_out/check_full.jsonl 2>> gpurun_out/check_err.log
  echo "rc=$? $args" >> gpurun_out/check_rc.txt
  tail -1 gpurun_out/check_full.jsonl | cut -c1-400
done
