mkdir -p gpurun_out
VARIANTS="_gazemap_b200 _v_fill" CONFIGS="c2 c5 c2off" REPS=1 EXTRA="--no-cold" bash tools/gpu_ab.sh
for v in _gazemap_b200 _v_fill; do
GAZEMAP_B200_SO=paper_2601_07571_b200/$v.so timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:'k_texels' -s 8 -c 4 --csv python bench.py --fixations 6144 --steps 1 --warmup 1 --no-cpu --no-e2e --no-stats --no-cold > gpurun_out/ncu_fill_$v.csv 2>&1
echo "== $v"; grep -E "k_texels" gpurun_out/ncu_fill_$v.csv | grep -E "dram__bytes|gpu__time|lts__t_sector_hit" | awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}' | head -16
done
