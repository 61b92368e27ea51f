mkdir -p gpurun_out/r4
bash tools/ncu_launches.sh north_star r4/launches_ns > gpurun_out/r4/launches_ns.txt 2>&1
cat gpurun_out/r4/launches_ns.txt
ncu --set full --clock-control none --import-source on -k 'regex:k_assign|k_scan|k_place|k_fix_small' -s 8 -c 4 -o gpurun_out/r4/bin python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-strong > gpurun_out/r4/bin.log 2>&1
ncu -i gpurun_out/r4/bin.ncu-rep --page details --csv > gpurun_out/r4/bin.details.csv 2>&1
ncu -i gpurun_out/r4/bin.ncu-rep --page raw --csv > gpurun_out/r4/bin.raw.csv 2>&1
