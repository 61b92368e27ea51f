timeout 900 python -m pytest tests/test_gpu_hd.py tests/test_gpu_f64.py -q -p no:cacheprovider -x 2>&1 | tail -2
for v in variants/lib_seed0.so variants/lib_seed256.so; do echo $v; FG_LIB_PATH=$v timeout 300 python tools/hd_stats.py C B 2>&1 | grep -E "C default|B force_hd|B no_hd"; done
