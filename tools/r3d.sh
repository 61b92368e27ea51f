for v in "" variants/lib_seedall.so; do echo "lib=${v:-default}"; FG_LIB_PATH=$v timeout 300 python tools/hd_stats.py B C 2>&1 | grep -E "B force_hd|C default"; done
