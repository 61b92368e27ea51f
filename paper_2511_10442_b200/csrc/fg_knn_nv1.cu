// Search kernels for coordinates of 1..4 dims (NV = 1 float4 per point).
#include "fg_knn_impl.cuh"

namespace fg {
namespace search {
int dispatch_nv1(const KnnArgs& a, int d_bin, cudaStream_t st) { return dispatch_db<1>(a, d_bin, st); }
}  // namespace search
}  // namespace fg
