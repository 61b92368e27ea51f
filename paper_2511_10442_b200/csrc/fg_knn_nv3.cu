// Search kernels for coordinates of 9..12 dims (NV = 3 float4 per point).
#include "fg_knn_impl.cuh"

namespace fg {
namespace search {
int dispatch_nv3(const KnnArgs& a, int d_bin, cudaStream_t st) { return dispatch_db<3>(a, d_bin, st); }
}  // namespace search
}  // namespace fg
