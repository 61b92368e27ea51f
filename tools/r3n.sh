# hd dispatch order (widest boxes first): parity + A/B on B and C
timeout 900 python -m pytest tests/test_gpu_hd.py tests/test_gpu_f64.py tests/test_capi.py -q -p no:cacheprovider -x 2>&1 | tail -2
for v in "" variants/lib_noorder.so; do echo "lib=${v:-default}"; FG_LIB_PATH=$v timeout 300 python tools/hd_stats.py B C 2>&1 | grep -E "B force_hd|C default"; done
