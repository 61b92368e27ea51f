nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv
for i in 1 2 3; do python bench.py --config ${1:-north_star} --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['breakdown_ms'].items()}, d['clocks'])"; done
nvidia-smi --query-compute-apps=pid,name,used_memory --format=csv
