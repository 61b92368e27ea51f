# thread-level cuts: parity + B / C
timeout 900 python -m pytest tests/test_gpu_hd.py tests/test_gpu_f64.py -q -p no:cacheprovider -x 2>&1 | tail -2
timeout 300 python tools/hd_stats.py B C 2>&1 | grep -E "C default|B force_hd"
