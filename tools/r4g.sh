# hd lane buffers 80 entries (9 warps/SM), cut rounds fixed for CAP % 32 != 0
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --config B --steps 10 --warmup 5 --no-e2e --no-strong --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('B', d['ms_per_step'], d['breakdown_ms'])"; done
timeout 600 python bench.py --config C --steps 2 --warmup 3 --no-e2e --no-strong --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C', d['ms_per_step'], d['breakdown_ms'])"
