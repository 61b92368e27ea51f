set -x
./tools/micro/red_locality > gpurun_out/red_locality.txt 2>&1; cat gpurun_out/red_locality.txt
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --deterministic 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('det', d['ms_per_step'], d['breakdown_ms'])"
bash tools/ncu_src.sh ns_finish north_star k_tile_finish
bash tools/ncu_src.sh ns_scan north_star k_tile_search
bash tools/ncu_src.sh ns_bwd north_star k_knn_bwd_pipe
ls -la gpurun_out
