for i in 1 2 3; do timeout 300 python tools/e2e_prof.py B 4 2>&1 | grep -E "alone|pipelined" ; done
for i in 1 2; do timeout 300 python bench.py --config B --steps 5 --warmup 3 --no-cpu-baseline --no-strong | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['latency_ms_per_step'])"; done
