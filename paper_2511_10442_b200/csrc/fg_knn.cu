// fg_knn.cu -- C ABI entry of binned_select_knn forward (kernels: fg_knn_impl.cuh).
#include <mutex>

#include "fg_knn_impl.cuh"

using namespace fg;
using namespace fg::search;

namespace {
unsigned long long* g_stats_dev = nullptr;  // FG_KNN_STATS counters (lazily allocated)
std::mutex g_stats_mu;
}  // namespace

extern "C" int fg_knn_fwd(const float* sorted_coords, const int32_t* sort_order,
                          const int64_t* bin_idx, const int32_t* bin_bounds,
                          const int64_t* row_splits, const double* dim_mins, const double* widths,
                          int64_t n, int32_t n_coords, int32_t n_splits, int32_t d_bin,
                          int32_t n_bins, int32_t k, const int8_t* dir_mask, double max_radius2,
                          uint32_t flags, int32_t* out_idx, void* out_d2, void* stream) {
    if (k < 1 || k > 960) return FG_ERR_BAD_K;
    if (n < 0 || n >= ((int64_t)1 << 31) || n_splits < 1 || n_bins < 1) return FG_ERR_BAD_SHAPE;
    if (n_coords < 1) return FG_ERR_BAD_SHAPE;
    if (n_coords > 16) return FG_ERR_TOO_MANY_DIMS;
    if (d_bin < 1 || d_bin > 5 || d_bin > n_coords) return FG_ERR_TOO_FEW_DIMS;
    if ((flags & FG_KNN_USE_MAX_R2) && !(max_radius2 >= 0.0)) return FG_ERR_BAD_RADIUS;
    int64_t total = 1;
    for (int i = 0; i < d_bin; ++i) total *= n_bins;
    if (total >= ((int64_t)1 << 31)) return FG_ERR_BAD_SHAPE;
    if (n == 0) return 0;
    if (!sorted_coords || !sort_order || !bin_idx || !bin_bounds || !row_splits || !dim_mins ||
        !widths || !out_idx || !out_d2)
        return FG_ERR_NULL;
    if ((flags & FG_KNN_USE_DIRECTION) && !dir_mask) return FG_ERR_NULL;
    KnnArgs a;
    a.sc = reinterpret_cast<const float4*>(sorted_coords);
    a.sid = sort_order;
    a.bin_idx = bin_idx;
    a.bounds = bin_bounds;
    a.rs = row_splits;
    a.mins = dim_mins;
    a.widths = widths;
    a.n = n;
    a.total = total;
    a.n_c = n_coords;
    a.n_splits = n_splits;
    a.nb = n_bins;
    a.k = k;
    a.dir = dir_mask;
    a.max_r2 = max_radius2;
    a.flags = flags;
    a.out_idx = out_idx;
    a.out_d2 = out_d2;
    a.stats = nullptr;
    if (flags & FG_KNN_STATS) {
        std::lock_guard<std::mutex> lk(g_stats_mu);
        if (!g_stats_dev) {
            FG_CUDA(cudaMalloc(&g_stats_dev, sizeof(unsigned long long) * ST_COUNT));
            FG_CUDA(cudaMemset(g_stats_dev, 0, sizeof(unsigned long long) * ST_COUNT));
        }
        a.stats = g_stats_dev;
    }
    cudaStream_t st = (cudaStream_t)stream;
    switch ((n_coords + 3) / 4) {
        case 1: return dispatch_nv1(a, d_bin, st);
        case 2: return dispatch_nv2(a, d_bin, st);
        case 3: return dispatch_nv3(a, d_bin, st);
        default: return dispatch_nv4(a, d_bin, st);
    }
}

extern "C" int fg_knn_stats(uint64_t* out, int32_t n, int32_t reset) {
    std::lock_guard<std::mutex> lk(g_stats_mu);
    unsigned long long h[ST_COUNT] = {0};
    if (g_stats_dev) {
        FG_CUDA(cudaMemcpy(h, g_stats_dev, sizeof(h), cudaMemcpyDeviceToHost));
        if (reset) FG_CUDA(cudaMemset(g_stats_dev, 0, sizeof(h)));
    }
    for (int i = 0; i < n && i < ST_COUNT; ++i) out[i] = h[i];
    return 0;
}
