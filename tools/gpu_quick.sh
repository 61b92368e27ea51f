python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -3
python tools/knn_stats.py north_star B 2>&1 | tail -2
for c in north_star B E A; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:40], round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['breakdown_ms'].items()}, round(d['roofline']['frac'],3))"; done
