# compute-sanitizer over tools/sanitize_workload.py (one tool per pass); logs
# to gpurun_out/sanitizer_<tool>.log, summaries copied to profiles/ by hand.
# Only the library's kernels are checked (torch's own are excluded by name).
mkdir -p gpurun_out
FILTER="--kernel-name-exclude kns=at::,kns=elementwise,kns=vectorized,kns=reduce_kernel,kns=distribution"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 $FILTER \
      python tools/sanitize_workload.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitizer_$tool.log
done
