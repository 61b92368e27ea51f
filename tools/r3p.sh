for c in B E; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-strong 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['breakdown_ms'].items()})"
done
bash tools/ncu_src.sh gn_rows E k_gn_rows1
grep -E '"Duration"|"Executed Ipc Active"|"Executed Instructions"|"Issue Slots Busy"' gpurun_out/gn_rows.details.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
