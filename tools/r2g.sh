for v in variants/lib_cap96.so variants/lib_cap128.so; do echo $v; FG_LIB_PATH=$v timeout 300 python tools/hd_stats.py C 2>&1 | grep "C default"; done
