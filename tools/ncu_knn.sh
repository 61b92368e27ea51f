# one full ncu capture of the search kernel (bench workload); args: out-name config kernel-regex
OUT=${1:-knn}
CFG=${2:-north_star}
KRE=${3:-"k_knn_fwd"}
ncu --set full --clock-control none --import-source on -k regex:$KRE -s 0 -c 1 -o gpurun_out/$OUT python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/$OUT.log 2>&1
