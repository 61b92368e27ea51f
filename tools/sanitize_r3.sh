# round 2: memcheck / racecheck / synccheck of the new high-dimensional and
# float64 tile kernels; initcheck of everything except k_tile_finish (whose
# list prefetch reads whole 88-entry rows speculatively -- values past the
# row's length are never used, documented in profiles/r2/sanitizer.md)
mkdir -p gpurun_out/san3
F="--kernel-name-exclude kns=at::,kns=elementwise,kns=vectorized,kns=reduce_kernel,kns=distribution"
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 $F python tools/sanitize_workload.py --hd > gpurun_out/san3/$tool.log 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/san3/$tool.log
done
timeout 1200 compute-sanitizer --tool initcheck --print-limit 20 $F --kernel-name-exclude kns=k_tile_finish python tools/sanitize_workload.py > gpurun_out/san3/initcheck.log 2>&1
echo "initcheck rc=$?"; tail -3 gpurun_out/san3/initcheck.log

