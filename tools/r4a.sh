# scan padding + e2e timeline of config B back to back
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_backward.py -x -q -k "bin or scan or gravnet or backward" 2>&1 | tail -2
timeout 300 python tools/e2e_prof.py B 4 > gpurun_out/e2e_B.txt 2>&1
head -3 gpurun_out/e2e_B.txt
timeout 300 python tools/e2e_prof.py north_star 4 2>&1 | head -2
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-strong --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['breakdown_ms'])"
bash tools/ncu_launches.sh north_star r4/launches_ns > gpurun_out/launches_ns.txt 2>&1; head -12 gpurun_out/launches_ns.txt
