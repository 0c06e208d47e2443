# A/B timing of build variants on the B200.
#   VARIANTS="_v_base _gazemap_b200" CONFIGS="c2 c2off c5" REPS=2 bash tools/gpu_ab.sh
#   -> gpurun_out/ab.txt (ms_per_step and single-stream texel ms per variant/config)
mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
VARIANTS=${VARIANTS:-"_v_base _gazemap_b200"}
CONFIGS=${CONFIGS:-"c2 c5"}
REPS=${REPS:-2}
EXTRA=${EXTRA:-}
for rep in $(seq $REPS); do
for cfg in $CONFIGS; do
for v in $VARIANTS; do
  GAZEMAP_B200_SO=paper_2601_07571_b200/$v.so timeout 600 python bench.py --config $cfg --steps 3 --warmup 2 \
      --no-cpu $EXTRA > gpurun_out/ab_${v}_$cfg.log 2>&1
  python - "$cfg" "$v" >> gpurun_out/ab.txt <<'PY'
import json, sys
cfg, v = sys.argv[1:3]
try:
    line = [l for l in open(f"gpurun_out/ab_{v}_{cfg}.log") if l.startswith("{")][-1]
    d = json.loads(line)
    ss = d.get("phases_single_stream_ms") or {}
    print(f"{cfg:6s} {v:22s} step {d['ms_per_step']:8.2f} ms  1s: total {ss.get('total',0):7.1f} texels {ss.get('texels',0):7.1f} "
          f"mark {ss.get('mark',0):6.1f} acc {ss.get('accumulate',0):6.1f} cull {ss.get('cull',0):6.1f}  gmax {d.get('global_max')}")
except Exception as e:
    print(cfg, v, "FAILED", e)
PY
done; done; done
cat gpurun_out/ab.txt
