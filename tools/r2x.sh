# hd candidate filter: parity + B / C A/B against the unfiltered build
timeout 900 python -m pytest tests/test_gpu_hd.py tests/test_gpu_f64.py -q -p no:cacheprovider -x 2>&1 | tail -2
for v in "" variants/lib_nofilt.so; do echo "lib=${v:-default}"; FG_LIB_PATH=$v timeout 300 python tools/hd_stats.py B C 2>&1 | grep -E "C default|B force_hd"; done
for v in "" variants/lib_nofilt.so; do
FG_LIB_PATH=$v timeout 300 python bench.py --config B --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-strong 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('B ${v:-default}', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['breakdown_ms'].items()})"
done
