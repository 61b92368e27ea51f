timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "bin" 2>&1 | tail -2
for c in B north_star; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-strong 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['breakdown_ms'].items()})"
done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_fix|k_dense|k_cell|k_hd|k_block" --csv python bench.py --config B --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-strong 2>/dev/null | grep -E "k_fix|k_dense|k_cell|k_hd|k_block" | awk -F'","' '{print $5, $NF}' | sort | uniq | head -20
