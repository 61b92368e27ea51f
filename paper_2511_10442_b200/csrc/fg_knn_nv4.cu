// Search kernels for coordinates of 13..16 dims (NV = 4 float4 per point).
#include "fg_knn_impl.cuh"

namespace fg {
namespace search {
int dispatch_nv4(const KnnArgs& a, int d_bin, cudaStream_t st) { return dispatch_db<4>(a, d_bin, st); }
}  // namespace search
}  // namespace fg
