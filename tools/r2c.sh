nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests/test_gpu_hd.py tests/test_gpu_f64.py tests/test_fileio_cli.py -m gpu -q -p no:cacheprovider > gpurun_out/t_new.log 2>&1; echo "new rc=$?"; tail -30 gpurun_out/t_new.log
timeout 1500 python -m pytest tests/test_gpu_reference_suite.py -q -p no:cacheprovider -rA > gpurun_out/t_refsuite.log 2>&1; echo "refsuite rc=$?"; grep -E "passed|failed|FAILED|ERROR" gpurun_out/t_refsuite.log | head -60
timeout 300 python bench.py --config C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C_hd.json 2>gpurun_out/bench_C_hd.err; echo "benchC rc=$?"; python -c "import json; d=json.loads(open('gpurun_out/bench_C_hd.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['breakdown_ms'])"
./tools/micro/red_locality 2>&1 | tee gpurun_out/red_locality.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x --deselect tests/test_gpu_reference_suite.py > gpurun_out/t_all.log 2>&1; echo "all rc=$?"; tail -5 gpurun_out/t_all.log
