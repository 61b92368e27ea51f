# per-kernel ncu metrics of one backward call: bash tools/ncu_bwd.sh CFG
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed
for c in "$@"; do
ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/bwd_$c.csv python tools/prof_bwd.py $c > /dev/null 2>&1
echo "== $c"; python tools/ncu_table.py gpurun_out/bwd_$c.csv
done
