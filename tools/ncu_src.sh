# full ncu capture (with source) of one kernel of the bench workload + raw/source CSV exports
OUT=${1:-knn_src}; CFG=${2:-north_star}; KRE=${3:-k_knn_fwd}
ncu --set full --clock-control none --import-source on -k regex:$KRE -s 0 -c 1 -o gpurun_out/$OUT \
    python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-strong > gpurun_out/$OUT.log 2>&1
ncu -i gpurun_out/$OUT.ncu-rep --page raw --csv > gpurun_out/$OUT.raw.csv 2>&1
ncu -i gpurun_out/$OUT.ncu-rep --page source --csv --print-source sass > gpurun_out/$OUT.sass.csv 2>&1
ncu -i gpurun_out/$OUT.ncu-rep --page details --csv > gpurun_out/$OUT.details.csv 2>&1
