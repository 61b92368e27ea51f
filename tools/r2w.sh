# A/B: expanded-form filtered scan (variants/lib_exp.so) vs default on north_star
timeout 600 python -m pytest tests/test_gpu_tile.py tests/test_gpu_parity.py -q -p no:cacheprovider -x 2>&1 | tail -2
FG_LIB_PATH=variants/lib_exp.so timeout 600 python -m pytest tests/test_gpu_tile.py tests/test_gpu_parity.py tests/test_gpu_verify.py -q -p no:cacheprovider -x 2>&1 | tail -2
for r in 1 2; do for v in "" variants/lib_exp.so; do
FG_LIB_PATH=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-strong 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ns ${v:-default}', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['breakdown_ms'].items()})"
done; done
