timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_f64.py tests/test_gpu_shard.py -q -p no:cacheprovider -x 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-strong 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ns', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['breakdown_ms'].items()})"; done
bash tools/ncu_launches.sh north_star r2u > gpurun_out/r2u.txt; grep -E "bbox|assign|scan|scatter|fix" gpurun_out/r2u.txt
