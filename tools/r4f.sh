mkdir -p gpurun_out/r4
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-strong --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['breakdown_ms'])"
bash tools/ncu_launches.sh north_star r4/launches_ns3 > gpurun_out/r4/launches_ns3.txt 2>&1; head -9 gpurun_out/r4/launches_ns3.txt
