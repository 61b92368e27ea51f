# redo beside finish (side stream) + hd seed/filter changes: parity and benches
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
for c in north_star B E; do
timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-strong 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['breakdown_ms'].items()})"
done
