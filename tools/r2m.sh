mkdir -p gpurun_out/san2
F="--kernel-name-exclude kns=at::,kns=elementwise,kns=vectorized,kns=reduce_kernel,kns=distribution"
timeout 1500 compute-sanitizer --tool initcheck --print-limit 20 $F python tools/sanitize_workload.py > gpurun_out/san2/initcheck2.log 2>&1; echo "initcheck rc=$?"; tail -3 gpurun_out/san2/initcheck2.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 $F python tools/sanitize_workload.py --hd > gpurun_out/san2/racecheck2.log 2>&1; echo "racecheck rc=$?"; tail -2 gpurun_out/san2/racecheck2.log
