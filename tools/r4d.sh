# binning rework: ranked assign + place pass
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-strong --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['breakdown_ms'])"
timeout 300 python bench.py --config B --steps 10 --warmup 5 --no-e2e --no-strong --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['breakdown_ms'])"
bash tools/ncu_launches.sh north_star r4/launches_ns2 > gpurun_out/launches_ns2.txt 2>&1; head -12 gpurun_out/launches_ns2.txt
