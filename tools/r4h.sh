# dense-cell Morton order by a bucketed counting sort
mkdir -p gpurun_out/r4
timeout 900 python -m pytest tests/test_gpu_hd.py tests/test_gpu_verify.py tests/test_gpu_tile.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --config B --steps 10 --warmup 5 --no-e2e --no-strong --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('B', d['ms_per_step'], d['breakdown_ms'])"; done
bash tools/ncu_launches.sh B r4/launches_B > gpurun_out/r4/launches_B.txt 2>&1; grep -E "morton|cell_split|hd_search" gpurun_out/r4/launches_B.txt
