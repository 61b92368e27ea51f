# GravNet rows pass: slot data staged in shared memory
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_tile.py -x -q -k "gravnet or GravNet" 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --config E --steps 10 --warmup 5 --no-e2e --no-strong --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('E', d['ms_per_step'], d['breakdown_ms'])"; done
