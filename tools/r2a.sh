nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_ns.json 2> gpurun_out/bench_ns.err; echo "bench rc=$?"; cat gpurun_out/bench_ns.json
for c in B C E D; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; tail -c 600 gpurun_out/bench_$c.json; echo; done
