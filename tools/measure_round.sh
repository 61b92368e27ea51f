# Round measurement set: bench line (N=1, default config) + reference arm +
# per-launch list + one full ncu capture of the search kernel.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_north_star.json 2> gpurun_out/bench_north_star.err
for c in A B E D C; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2>/dev/null; done
python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_reference.json 2>/dev/null
bash tools/ncu_launches.sh north_star launches_north_star > gpurun_out/launches_north_star.txt
bash tools/ncu_knn.sh knn_fwd_north_star north_star k_knn_fwd
bash tools/ncu_knn.sh knn_bwd_north_star north_star k_knn_bwd
bash tools/ncu_knn.sh bin_assign_north_star north_star k_assign
