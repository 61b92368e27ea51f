F="--kernel-name-exclude kns=at::,kns=elementwise,kns=vectorized,kns=reduce_kernel,kns=distribution,kns=k_tile_finish"
timeout 600 compute-sanitizer --tool initcheck --print-limit 3 $F python tools/init_min.py 0 2>&1 | grep -E "ERROR SUMMARY|Uninit|at void|queries" | head -8
timeout 600 compute-sanitizer --tool initcheck --print-limit 3 $F python tools/init_min.py 4096 2>&1 | grep -E "ERROR SUMMARY|Uninit|at void|queries" | head -8
for v in variants/lib_s120.so variants/lib_s184.so variants/lib_cap96w1.so ""; do echo "lib=${v:-default}"; FG_LIB_PATH=$v timeout 300 python tools/hd_stats.py B 2>&1 | grep -E "B force_hd"; done
