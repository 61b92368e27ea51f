// Search kernels for coordinates of 5..8 dims (NV = 2 float4 per point).
#include "fg_knn_impl.cuh"

namespace fg {
namespace search {
int dispatch_nv2(const KnnArgs& a, int d_bin, cudaStream_t st) { return dispatch_db<2>(a, d_bin, st); }
}  // namespace search
}  // namespace fg
