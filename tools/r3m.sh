timeout 900 python -m pytest tests/test_gpu_hd.py tests/test_gpu_f64.py -q -p no:cacheprovider -x 2>&1 | tail -2
timeout 300 python tools/hd_stats.py B C 2>&1 | grep -E "B force_hd|C default"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_hd_tiles" --csv python bench.py --config B --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-strong 2>/dev/null | grep -E "k_hd_tiles" | awk -F'","' '{split($5,a,"("); print a[1], $NF}' | head -4
