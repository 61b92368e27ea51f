# A/B the experimental builds in variants/ on the bench workload
CFG=${1:-north_star}
for v in variants/lib_*.so; do
  for i in 1 2; do
    FG_LIB_PATH=$v python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['breakdown_ms'].items()})"
  done
done
