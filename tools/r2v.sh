timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t_all2.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/t_all2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
