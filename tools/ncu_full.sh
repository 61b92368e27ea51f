# full ncu capture (with source) of the first launch of kernels matching KRE in
# an arbitrary command: bash tools/ncu_full.sh OUT KRE cmd args...
OUT=$1; KRE=$2; shift 2
ncu --set full --clock-control none --import-source on -k regex:$KRE -s 0 -c 1 -o gpurun_out/$OUT "$@" > gpurun_out/$OUT.log 2>&1
ncu -i gpurun_out/$OUT.ncu-rep --page raw --csv > gpurun_out/$OUT.raw.csv 2>&1
ncu -i gpurun_out/$OUT.ncu-rep --page source --csv --print-source sass > gpurun_out/$OUT.sass.csv 2>&1
ncu -i gpurun_out/$OUT.ncu-rep --page details --csv > gpurun_out/$OUT.details.csv 2>&1
