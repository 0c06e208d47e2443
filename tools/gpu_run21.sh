mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
VARIANTS="_v_prev _gazemap_b200 _v_ns4 _v_ns2" CONFIGS="c2 c2off c5" REPS=1 EXTRA="" bash tools/gpu_ab.sh
for v in _v_prev _gazemap_b200; do for c in c2 c2off c5; do python - $v $c <<'PY'
import json, sys
v, c = sys.argv[1:3]
d = json.loads([l for l in open(f"gpurun_out/ab_{v}_{c}.log") if l.startswith("{")][-1])
print(v, c, "cold", d["e2e"]["cold"]["ms"], d["e2e"]["cold"]["reps_ms"], "e2e", d["e2e"]["ms_per_step"], "retries", d["phases_ms"]["retries"])
PY
done; done
timeout 600 python tools/accum_loop_bench.py
