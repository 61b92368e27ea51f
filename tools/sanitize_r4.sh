# round 2 (final build): memcheck / racecheck / synccheck / initcheck over the
# whole workload incl. the clustered fallback (dense-cell counting sort, 80-entry
# lane buffers) and the rank/place binning
mkdir -p gpurun_out/san4
F="--kernel-name-exclude kns=at::,kns=elementwise,kns=vectorized,kns=reduce_kernel,kns=distribution"
for tool in memcheck racecheck synccheck; do
  for mode in "" "--hd"; do
    tag=$tool${mode:+_hd}
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 $F python tools/sanitize_workload.py $mode > gpurun_out/san4/$tag.log 2>&1
    echo "$tag rc=$?"; tail -2 gpurun_out/san4/$tag.log
  done
done
timeout 1200 compute-sanitizer --tool initcheck --print-limit 20 $F python tools/sanitize_workload.py > gpurun_out/san4/initcheck.log 2>&1
echo "initcheck rc=$?"; tail -3 gpurun_out/san4/initcheck.log
