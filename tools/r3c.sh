bash tools/ncu_src.sh hd_B2 B k_hd_search
grep -E "Duration|Executed Ipc A" gpurun_out/hd_B2.details.csv | head -3
