# ncu --set full of the north_star search + backward kernels and B's hd search (current build)
mkdir -p gpurun_out/r4n
for kk in k_tiles k_tile_search k_tile_finish k_knn_fwd k_knn_bwd_stream; do
  bash tools/ncu_src.sh r4n/ns_$kk north_star $kk
done
bash tools/ncu_src.sh r4n/B_k_hd_search B k_hd_search
rm -f gpurun_out/r4n/*.sass.csv
ls -la gpurun_out/r4n | head -30
