# C regression check + full ncu source capture of the hd search on config B
timeout 300 python tools/hd_stats.py C 2>&1 | grep -E "C default"
bash tools/ncu_src.sh hd_B B k_hd_search
ls -la gpurun_out/hd_B*
