for kn in k_gn_fwd_pairs k_gn_rows1 k_gn_cols; do
ncu --set full --clock-control none -k regex:$kn -s 0 -c 1 -o gpurun_out/E_$kn python bench.py --config E --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-strong > /dev/null 2>&1
ncu -i gpurun_out/E_$kn.ncu-rep --page details --csv > gpurun_out/E_$kn.details.csv 2>&1
echo "== $kn"; grep -E '"(Duration|Executed Ipc Active|Issue Slots Busy|Achieved Occupancy|Theoretical Occupancy|Warp Cycles Per Issued Instruction|L1/TEX Hit Rate|L2 Hit Rate|DRAM Throughput|Memory Throughput|Registers Per Thread|Mem Busy|Max Bandwidth)"' gpurun_out/E_$kn.details.csv | awk -F'","' '{print $(NF-2)" | "$NF}'
done
