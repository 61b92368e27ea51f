timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
mkdir -p gpurun_out/r2
timeout 600 python bench.py --config B --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench_B.json 2> /dev/null
tail -1 gpurun_out/r2/bench_B.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B', d['ms_per_step'], d['breakdown_ms'], d['e2e']['ms_per_step'])"
bash tools/ncu_launches.sh B r2/launches_B > gpurun_out/r2/launches_B.txt 2>&1
