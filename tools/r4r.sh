# binning: cells of <= 8192 points by the CTA bitonic fix-up (was 4096)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hd.py -x -q -k "bin or dense" 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --config B --steps 10 --warmup 5 --no-e2e --no-strong --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('B', d['ms_per_step'], d['breakdown_ms'])"; done
bash tools/ncu_launches.sh B r4/launches_B2 > gpurun_out/r4/launches_B2.txt 2>&1; grep -E "fix_" gpurun_out/r4/launches_B2.txt
