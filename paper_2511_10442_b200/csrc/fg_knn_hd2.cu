// High-dimensional / float64-coordinate tile path (fg_knn_hd.cuh) for
// coordinates stored as NV = 2 float4 per point; one translation unit per NV
// (parallel builds).
#include "fg_knn_hd.cuh"

namespace fg {
namespace hd {

int dispatch_hd_nv2(tile::TileArgs& t, const search::KnnArgs& a, int d_bin, cudaStream_t st) {
    return a.x64 ? dispatch_db<2, true>(t, a, d_bin, st) : dispatch_db<2, false>(t, a, d_bin, st);
}

}  // namespace hd
}  // namespace fg
