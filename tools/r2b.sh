bash tools/ncu_src.sh ns_bwd north_star k_knn_bwd_pipe
bash tools/ncu_src.sh ns_finish north_star k_tile_finish
bash tools/ncu_src.sh ns_scan north_star k_tile_search
for f in ns_bwd ns_finish ns_scan; do echo "== $f"; grep -E '"(Duration|Executed Ipc Active|Issue Slots Busy|Achieved Occupancy|Theoretical Occupancy|Warp Cycles Per Issued Instruction|L1/TEX Hit Rate|L2 Hit Rate|DRAM Throughput|Memory Throughput|Registers Per Thread|Compute \(SM\) Throughput|Mem Busy|Max Bandwidth|L2 Compression Ratio)"' gpurun_out/$f.details.csv | awk -F'","' '{print $(NF-2)" | "$NF}'; python tools/sass_hot.py gpurun_out/$f.sass.csv 25 | tail -30; done
