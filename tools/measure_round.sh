# Round measurement set: bench lines, reference arm, per-launch list, full ncu
# captures of the search (scan + finish) and backward kernels (-> profiles/ via
# tools/ncu_summary.py).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_north_star.json 2> gpurun_out/bench_north_star.err
for c in A B E D C; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2>/dev/null; done
python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_reference.json 2>/dev/null
bash tools/ncu_launches.sh north_star launches_north_star > gpurun_out/launches_north_star.txt
bash tools/ncu_launches.sh E launches_E > gpurun_out/launches_E.txt
for k in k_tile_search k_tile_finish k_knn_bwd k_tiles; do bash tools/ncu_src.sh ns_$k north_star $k; done
bash tools/ncu_src.sh ns_k_knn_fwd north_star "k_knn_fwd"
