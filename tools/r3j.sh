# lane-buffer capacity / CTA size A/B on B (k = 40)
for v in "" variants/lib_cap96.so variants/lib_cap96w1.so variants/lib_cap64w1.so; do echo "lib=${v:-default}"; FG_LIB_PATH=$v timeout 300 python tools/hd_stats.py B 2>&1 | grep -E "B force_hd"; done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_fix_big" --csv python bench.py --config north_star --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-strong 2>/dev/null | grep k_fix_big | awk -F'","' '{print $NF}'
