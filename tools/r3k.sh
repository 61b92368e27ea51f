bash tools/ncu_src.sh hd_B3 B k_hd_search
grep -E '"Duration"|"Executed Ipc Active"' gpurun_out/hd_B3.details.csv | head -3
