# stage-0 seed window A/B on B (hd filter build)
for v in "" variants/lib_s512.so variants/lib_s1024.so variants/lib_nofilt.so; do echo "lib=${v:-default}"; FG_LIB_PATH=$v timeout 300 python tools/hd_stats.py B 2>&1 | grep -E "B force_hd"; done
