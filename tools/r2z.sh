# interpolated cuts: parity + B / C A/B
timeout 900 python -m pytest tests/test_gpu_hd.py tests/test_gpu_f64.py -q -p no:cacheprovider -x 2>&1 | tail -2
for v in "" variants/lib_nointerp.so; do echo "lib=${v:-default}"; FG_LIB_PATH=$v timeout 300 python tools/hd_stats.py B C 2>&1 | grep -E "C default|B force_hd"; done
