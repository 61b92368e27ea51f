timeout 600 python tools/hd_stats.py C B north_star E 2>&1 | tee gpurun_out/hd_stats.txt
timeout 600 python -m pytest tests/test_gpu_hd.py tests/test_gpu_f64.py -q -p no:cacheprovider 2>&1 | tail -3
