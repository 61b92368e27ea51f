timeout 300 python tools/hd_stats.py B C 2>&1 | grep -E "B force_hd|C default"
