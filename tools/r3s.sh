timeout 900 python -m pytest tests/test_gpu_hd.py tests/test_gpu_f64.py tests/test_gpu_verify.py -q -p no:cacheprovider -x 2>&1 | tail -2
timeout 300 python tools/hd_stats.py B C 2>&1 | grep -E "B force_hd|C default"
F="--kernel-name-exclude kns=at::,kns=elementwise,kns=vectorized,kns=reduce_kernel,kns=distribution"
timeout 600 compute-sanitizer --tool initcheck --print-limit 3 $F python tools/init_min.py 0 2>&1 | grep -E "ERROR SUMMARY|Uninit|at void" | head -5
