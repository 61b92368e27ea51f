# round 2 (second pass): memcheck / racecheck / synccheck of the hd / float64 / clustered-fallback kernels;
# initcheck of every kernel (excluding k_tile_finish hid its redo-list writes
# from the tracker: the redo kernel then read "uninitialized" entries)

mkdir -p gpurun_out/san3
F="--kernel-name-exclude kns=at::,kns=elementwise,kns=vectorized,kns=reduce_kernel,kns=distribution"
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 $F python tools/sanitize_workload.py --hd > gpurun_out/san3/$tool.log 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/san3/$tool.log
done
timeout 1200 compute-sanitizer --tool initcheck --print-limit 20 $F python tools/sanitize_workload.py > gpurun_out/san3/initcheck.log 2>&1
echo "initcheck rc=$?"; tail -3 gpurun_out/san3/initcheck.log

