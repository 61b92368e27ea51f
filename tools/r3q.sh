for v in "" variants/lib_s120.so variants/lib_s184.so variants/lib_cap96w1.so; do echo "lib=${v:-default}"; FG_LIB_PATH=$v timeout 300 python tools/hd_stats.py B 2>&1 | grep -E "B force_hd"; done
