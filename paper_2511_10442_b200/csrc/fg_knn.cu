// fg_knn.cu -- C ABI entry of binned_select_knn forward (kernels: fg_knn_impl.cuh).
#include <mutex>

#include "fg_knn_hd.cuh"

using namespace fg;
using namespace fg::search;

namespace fg {
namespace tile {
int launch(TileArgs& t, const search::KnnArgs& a, int d_bin, cudaStream_t st, TileArgs* clustered);
}
namespace gravnet {
int reducer_bits(const int32_t* reducers, int n_red, unsigned* bits);
}  // namespace gravnet
}  // namespace fg

namespace {
unsigned long long* g_stats_dev = nullptr;  // FG_KNN_STATS counters (lazily allocated)

// Per-device host-mapped "the last tile-path call was clustered" flag (see
// TileArgs::hint).  It only picks which exact path is launched; results are
// identical either way.
constexpr int kMaxDevices = 64;
std::mutex g_hint_mu;
volatile int* g_hint_host[kMaxDevices] = {};
int* g_hint_dev[kMaxDevices] = {};

int clustered_hint(int** dev_ptr, bool* last_clustered) {
    int dev = 0;
    FG_CUDA(cudaGetDevice(&dev));
    *dev_ptr = nullptr;
    *last_clustered = true;  // unknown: launch the (gated) fallback
    if (dev < 0 || dev >= kMaxDevices) return 0;
    std::lock_guard<std::mutex> lk(g_hint_mu);
    if (!g_hint_host[dev]) {
        int* h = nullptr;
        if (cudaHostAlloc((void**)&h, sizeof(int), cudaHostAllocMapped) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
        *h = 1;
        int* d = nullptr;
        FG_CUDA(cudaHostGetDevicePointer((void**)&d, h, 0));
        g_hint_host[dev] = h;
        g_hint_dev[dev] = d;
    }
    *dev_ptr = g_hint_dev[dev];
    *last_clustered = *g_hint_host[dev] != 0;
    return 0;
}
std::mutex g_stats_mu;
constexpr int kStatsTotal = ST_COUNT + tile::TS_COUNT + hd::HS_COUNT;

// The lane-per-query tile path (fg_knn_tile.cuh) serves every coordinate
// binned, d <= 4, k - 1 <= 40, no mask / radius / exhaustive / float64 output.
bool tile_path(int32_t n_coords, int32_t n_splits, int32_t d_bin, int32_t n_bins, int32_t k,
               uint32_t flags) {
    const uint32_t off = FG_KNN_USE_DIRECTION | FG_KNN_USE_MAX_R2 | FG_KNN_EXHAUSTIVE |
                         FG_KNN_D2_F64 | FG_KNN_NO_TILE | FG_KNN_FORCE_HD;  // FG_KNN_FUSED_EPI / _GN: tile variants
    if (!(n_coords == d_bin && n_coords <= 4 && n_bins <= 32 && k >= 2 &&
          k - 1 <= tile::kMaxNeed && !(flags & off)))
        return false;
    int64_t blocks = n_splits;  // lead blocks must fit the int32 tile descriptors
    for (int i = 0; i < d_bin - 1; ++i) blocks *= (n_bins + 1) / 2;
    return blocks < ((int64_t)1 << 30);
}

// The lane-per-query high-dimensional tile path (fg_knn_hd.cuh) serves what the
// d <= 4 tile path does not: n_coords > 4 or d_bin < n_coords, k <= 64, no
// mask / radius / exhaustive (float64 distances are fine).
bool hd_shape(int32_t n_splits, int32_t d_bin, int32_t n_bins, int32_t k) {
    if (!(n_bins <= 32 && k >= 1 && k <= hd::kMaxK64)) return false;
    int64_t blocks = n_splits;
    for (int i = 0; i < d_bin - 1; ++i) blocks *= (n_bins + 1) / 2;
    return blocks < ((int64_t)1 << 30);
}
bool hd_path(int32_t n_coords, int32_t n_splits, int32_t d_bin, int32_t n_bins, int32_t k,
             uint32_t flags) {
    const uint32_t off = FG_KNN_EXHAUSTIVE | FG_KNN_NO_TILE | FG_KNN_NO_HD;
    if (tile_path(n_coords, n_splits, d_bin, n_bins, k, flags)) return false;
    return k >= 2 && k <= hd::kMaxNeed1 && !(flags & off) && hd_shape(n_splits, d_bin, n_bins, k);
}

// Argument validation shared by both entry points (before any CUDA call).
int check_args(const float* sorted_coords, const int32_t* sort_order, const int64_t* bin_idx,
               const int32_t* bin_bounds, const int64_t* row_splits, const double* dim_mins,
               const double* widths, int64_t n, int32_t n_coords, int32_t n_splits, int32_t d_bin,
               int32_t n_bins, int32_t k, const int8_t* dir_mask, double max_radius2,
               uint32_t flags, const int32_t* out_idx, const void* out_d2) {
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
    return 0;
}

struct TileWs {
    int* ctr;
    int2* tiles;
    int32_t* redo;
    float4* sc2;     // hd path: search copies (dense cells in Morton order)
    int32_t* sid2;
    int32_t* dense;
    float4* boxes;   // hd path, d <= 4: per-32-position bounding boxes
    uint8_t* tcnt;   // hd path: points per tile
    uint8_t* tkey;   //          cost bucket per tile
    int* hist;       //          bucket counts / cursors
    int32_t* order;  //          dispatch order
    int32_t* lists;  // split epilogue: n * kCap sorted positions
    float2* meta;    //                 n * (tau, m)
    size_t bytes;
    int64_t n_blocks;
};

TileWs tile_ws(void* base, int64_t n, int32_t n_splits, int32_t d_bin, int32_t n_bins) {
    TileWs w;
    const int64_t nblk = (n_bins + 1) / 2;
    int64_t bps = 1;
    for (int i = 0; i < d_bin - 1; ++i) bps *= nblk;
    w.n_blocks = bps * n_splits;
    // a tile holds >= 1 point: at most min(blocks x columns, n) tiles
    const int64_t max_tiles = std::min<int64_t>(w.n_blocks * n_bins, std::max<int64_t>(n, 1));
    char* p = static_cast<char*>(base);
    size_t off = 0;
    w.ctr = reinterpret_cast<int*>(p + off);
    off += 64;
    w.tiles = reinterpret_cast<int2*>(p + off);
    off = align_up(off + sizeof(int2) * (size_t)max_tiles, 256);
    w.redo = reinterpret_cast<int32_t*>(p + off);
    off = align_up(off + sizeof(int32_t) * (size_t)std::max<int64_t>(n, 1), 256);
    w.lists = reinterpret_cast<int32_t*>(p + off);
    off = align_up(off + sizeof(int32_t) * (size_t)tile::kCap * (size_t)std::max<int64_t>(n, 1), 256);
    w.meta = reinterpret_cast<float2*>(p + off);
    off = align_up(off + sizeof(float2) * (size_t)std::max<int64_t>(n, 1), 256);
    w.bytes = off;
    return w;
}
TileWs hd_ws(void* base, int64_t n, int32_t n_coords, int32_t n_splits, int32_t d_bin, int32_t n_bins) {
    TileWs w{};
    const int64_t nblk = (n_bins + 1) / 2;
    int64_t bps = 1;
    for (int i = 0; i < d_bin - 1; ++i) bps *= nblk;
    w.n_blocks = bps * n_splits;
    // runs of <= 32 per block, a run never spanning more than hd::kTileSpan
    // columns: at most one short run per column of a block
    const int64_t max_tiles = n / 32 + w.n_blocks * n_bins + 1;
    char* p = static_cast<char*>(base);
    size_t off = 0;
    w.ctr = reinterpret_cast<int*>(p + off);
    off += 64;
    w.tiles = reinterpret_cast<int2*>(p + off);
    off = align_up(off + sizeof(int2) * (size_t)max_tiles, 256);
    w.redo = reinterpret_cast<int32_t*>(p + off);
    off = align_up(off + sizeof(int32_t) * (size_t)std::max<int64_t>(n, 1), 256);
    // the search's copies of the sorted coordinates / ids (dense cells re-ordered)
    const int nv = (n_coords + 3) / 4;
    w.sc2 = reinterpret_cast<float4*>(p + off);
    off = align_up(off + sizeof(float4) * nv * (size_t)std::max<int64_t>(n, 1), 256);
    w.sid2 = reinterpret_cast<int32_t*>(p + off);
    off = align_up(off + sizeof(int32_t) * (size_t)std::max<int64_t>(n, 1), 256);
    w.dense = reinterpret_cast<int32_t*>(p + off);
    off = align_up(off + sizeof(int32_t) * (size_t)(n / (hd::kDenseCell + 1) + 1), 256);
    w.tcnt = reinterpret_cast<uint8_t*>(p + off);
    off = align_up(off + (size_t)max_tiles, 256);
    w.tkey = reinterpret_cast<uint8_t*>(p + off);
    off = align_up(off + (size_t)max_tiles, 256);
    w.hist = reinterpret_cast<int*>(p + off);
    off = align_up(off + sizeof(int) * 2 * hd::kCostBuckets, 256);
    w.order = reinterpret_cast<int32_t*>(p + off);
    off = align_up(off + sizeof(int32_t) * (size_t)max_tiles, 256);
    w.boxes = nullptr;
    if (n_coords <= hd::kFilterDE) {
        w.boxes = reinterpret_cast<float4*>(p + off);
        off = align_up(off + 2 * sizeof(float4) * (size_t)(n / 32 + 1), 256);
    }
    w.bytes = off;
    return w;
}
}  // namespace

extern "C" int fg_knn_workspace_size(int64_t n, int32_t n_coords, int32_t n_splits, int32_t d_bin,
                                     int32_t n_bins, int32_t k, uint32_t flags, size_t* bytes) {
    if (!bytes) return FG_ERR_NULL;
    if (n < 0 || n_splits < 1 || n_bins < 1) return FG_ERR_BAD_SHAPE;
    *bytes = tile_path(n_coords, n_splits, d_bin, n_bins, k, flags)
                 ? tile_ws(nullptr, n, n_splits, d_bin, n_bins).bytes +
                       hd_ws(nullptr, n, n_coords, n_splits, d_bin, n_bins).bytes
                 : hd_path(n_coords, n_splits, d_bin, n_bins, k, flags)
                       ? hd_ws(nullptr, n, n_coords, n_splits, d_bin, n_bins).bytes
                       : 0;
    return 0;
}

extern "C" int fg_knn_fwd(const float* sorted_coords, const int32_t* sort_order,
                          const int64_t* bin_idx, const int32_t* bin_bounds,
                          const int64_t* row_splits, const double* dim_mins, const double* widths,
                          int64_t n, int32_t n_coords, int32_t n_splits, int32_t d_bin,
                          int32_t n_bins, int32_t k, const int8_t* dir_mask, double max_radius2,
                          uint32_t flags, int32_t* out_idx, void* out_d2, void* stream) {
    // convenience entry: stream-ordered scratch from the CUDA memory pool
    FG_TRY(check_args(sorted_coords, sort_order, bin_idx, bin_bounds, row_splits, dim_mins, widths,
                      n, n_coords, n_splits, d_bin, n_bins, k, dir_mask, max_radius2, flags,
                      out_idx, out_d2));
    if (n == 0) return 0;
    size_t bytes = 0;
    if (tile_path(n_coords, n_splits, d_bin, n_bins, k, flags))
        bytes = tile_ws(nullptr, n, n_splits, d_bin, n_bins).bytes +
                hd_ws(nullptr, n, n_coords, n_splits, d_bin, n_bins).bytes;
    else if (hd_path(n_coords, n_splits, d_bin, n_bins, k, flags))
        bytes = hd_ws(nullptr, n, n_coords, n_splits, d_bin, n_bins).bytes;
    void* ws = nullptr;
    cudaStream_t st = (cudaStream_t)stream;
    if (bytes) FG_CUDA(cudaMallocAsync(&ws, bytes, st));
    const int rc = fg_knn_fwd_ws(sorted_coords, sort_order, bin_idx, bin_bounds, row_splits,
                                 dim_mins, widths, n, n_coords, n_splits, d_bin, n_bins, k,
                                 dir_mask, max_radius2, flags, out_idx, out_d2, ws, bytes, stream);
    if (ws) FG_CUDA(cudaFreeAsync(ws, st));
    return rc;
}

extern "C" int fg_knn_fwd_ws(const float* sorted_coords, const int32_t* sort_order,
                             const int64_t* bin_idx, const int32_t* bin_bounds,
                             const int64_t* row_splits, const double* dim_mins,
                             const double* widths, int64_t n, int32_t n_coords, int32_t n_splits,
                             int32_t d_bin, int32_t n_bins, int32_t k, const int8_t* dir_mask,
                             double max_radius2, uint32_t flags, int32_t* out_idx, void* out_d2,
                             void* workspace, size_t workspace_bytes, void* stream) {
    FG_TRY(check_args(sorted_coords, sort_order, bin_idx, bin_bounds, row_splits, dim_mins, widths,
                      n, n_coords, n_splits, d_bin, n_bins, k, dir_mask, max_radius2, flags,
                      out_idx, out_d2));
    if (n == 0) return 0;
    int64_t total = 1;
    for (int i = 0; i < d_bin; ++i) total *= n_bins;
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
    a.qlist = nullptr;
    a.qcount = nullptr;
    a.qall = nullptr;
    a.x64 = nullptr;
    a.rnd = nullptr;
    if (flags & FG_KNN_STATS) {
        std::lock_guard<std::mutex> lk(g_stats_mu);
        if (!g_stats_dev) {
            FG_CUDA(cudaMalloc(&g_stats_dev, sizeof(unsigned long long) * kStatsTotal));
            FG_CUDA(cudaMemset(g_stats_dev, 0, sizeof(unsigned long long) * kStatsTotal));
        }
        a.stats = g_stats_dev;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (tile_path(n_coords, n_splits, d_bin, n_bins, k, flags)) {
        const TileWs w = tile_ws(workspace, n, n_splits, d_bin, n_bins);
        if (!workspace) return FG_ERR_NULL;
        const TileWs wh = hd_ws(static_cast<char*>(workspace) + w.bytes, n, n_coords, n_splits,
                                d_bin, n_bins);
        if (workspace_bytes < w.bytes + wh.bytes) return FG_ERR_WORKSPACE;
        tile::TileArgs t{};
        t.sc = a.sc;
        t.sid = sort_order;
        t.bounds = bin_bounds;
        t.mins = dim_mins;
        t.widths = widths;
        t.total = total;
        t.nb = n_bins;
        t.n = n;
        t.k = k;
        t.nblk = (n_bins + 1) / 2;
        t.bps = (int)(w.n_blocks / n_splits);
        t.n_blocks = (int)w.n_blocks;
        t.tiles = w.tiles;
        t.ctr = w.ctr;
        t.redo = w.redo;
        t.out_idx = out_idx;
        t.out_d2 = reinterpret_cast<float*>(out_d2);
        const bool split = !(flags & FG_KNN_FUSED_EPI);
        t.lists = split ? w.lists : nullptr;
        t.meta = split ? w.meta : nullptr;
        t.stats = a.stats ? a.stats + ST_COUNT : nullptr;
        // the clustered-data fallback (high-dimensional tile kernels, gated on
        // the tile kernels' decline rule on the device)
        tile::TileArgs th = t;
        th.tiles = wh.tiles;
        th.ctr = wh.ctr;
        th.redo = wh.redo;
        th.lists = nullptr;
        th.meta = nullptr;
        th.sc2 = wh.sc2;
        th.sid2 = wh.sid2;
        th.dense = wh.dense;
        th.boxes = wh.boxes;
        th.tcnt = wh.tcnt;
        th.tkey = wh.tkey;
        th.hist = wh.hist;
        th.order = wh.order;
        th.stats = nullptr;
        int* hint_dev = nullptr;
        bool last_clustered = true;
        FG_TRY(clustered_hint(&hint_dev, &last_clustered));
        t.hint = hint_dev;
        const bool fallback = !(flags & FG_KNN_NO_HD) && (last_clustered || !hint_dev);
        return tile::launch(t, a, d_bin, st, fallback ? &th : nullptr);
    }
    if (hd_path(n_coords, n_splits, d_bin, n_bins, k, flags)) {
        const TileWs w = hd_ws(workspace, n, n_coords, n_splits, d_bin, n_bins);
        if (!workspace) return FG_ERR_NULL;
        if (workspace_bytes < w.bytes) return FG_ERR_WORKSPACE;
        tile::TileArgs t{};
        t.sc = a.sc;
        t.sid = sort_order;
        t.bounds = bin_bounds;
        t.mins = dim_mins;
        t.widths = widths;
        t.total = total;
        t.nb = n_bins;
        t.n = n;
        t.k = k;
        t.nblk = (n_bins + 1) / 2;
        t.bps = (int)(w.n_blocks / n_splits);
        t.n_blocks = (int)w.n_blocks;
        t.tiles = w.tiles;
        t.ctr = w.ctr;
        t.redo = w.redo;
        t.out_idx = out_idx;
        t.stats = nullptr;
        t.sc2 = w.sc2;
        t.sid2 = w.sid2;
        t.dense = w.dense;
        t.boxes = w.boxes;
        t.tcnt = w.tcnt;
        t.tkey = w.tkey;
        t.hist = w.hist;
        t.order = w.order;
        switch ((n_coords + 3) / 4) {
            case 1: return hd::dispatch_hd_nv1(t, a, d_bin, st);
            case 2: return hd::dispatch_hd_nv2(t, a, d_bin, st);
            case 3: return hd::dispatch_hd_nv3(t, a, d_bin, st);
            default: return hd::dispatch_hd_nv4(t, a, d_bin, st);
        }
    }
    switch ((n_coords + 3) / 4) {
        case 1: return dispatch_nv1(a, d_bin, st);
        case 2: return dispatch_nv2(a, d_bin, st);
        case 3: return dispatch_nv3(a, d_bin, st);
        default: return dispatch_nv4(a, d_bin, st);
    }
}

extern "C" int fg_knn_f64_workspace_size(int64_t n, int32_t n_coords, int32_t n_splits,
                                         int32_t d_bin, int32_t n_bins, int32_t k, uint32_t flags,
                                         size_t* bytes) {
    (void)n_coords;
    (void)flags;
    if (!bytes) return FG_ERR_NULL;
    if (n < 0 || n_splits < 1 || n_bins < 1) return FG_ERR_BAD_SHAPE;
    *bytes = hd_ws(nullptr, n, n_coords, n_splits, d_bin, n_bins).bytes + 256;
    return 0;
}

extern "C" int fg_knn_fwd_f64_ws(const double* coords, const float* sorted_coords,
                                 const int32_t* sort_order, const int64_t* bin_idx,
                                 const int32_t* bin_bounds, const int64_t* row_splits,
                                 const double* dim_mins, const double* widths, int64_t n,
                                 int32_t n_coords, int32_t n_splits, int32_t d_bin, int32_t n_bins,
                                 int32_t k, const int8_t* dir_mask, double max_radius2,
                                 uint32_t flags, int32_t* out_idx, void* out_d2, void* workspace,
                                 size_t workspace_bytes, void* stream) {
    FG_TRY(check_args(sorted_coords, sort_order, bin_idx, bin_bounds, row_splits, dim_mins, widths,
                      n, n_coords, n_splits, d_bin, n_bins, k, dir_mask, max_radius2, flags,
                      out_idx, out_d2));
    if (n == 0) return 0;
    if (!coords || !workspace) return FG_ERR_NULL;
    if (!hd_shape(n_splits, d_bin, n_bins, k)) return FG_ERR_UNSUPPORTED;
    const TileWs w = hd_ws(workspace, n, n_coords, n_splits, d_bin, n_bins);
    if (workspace_bytes < w.bytes + 256) return FG_ERR_WORKSPACE;
    unsigned* rnd = reinterpret_cast<unsigned*>(static_cast<char*>(workspace) + w.bytes);
    cudaStream_t st = (cudaStream_t)stream;
    FG_CUDA(cudaMemsetAsync(rnd, 0, sizeof(unsigned), st));
    const int64_t m = n * n_coords;
    hd::k_abs_bound<<<(unsigned)std::min<int64_t>(ceil_div(m, 256), 148 * 8), 256, 0, st>>>(
        coords, m, n_coords, rnd);
    FG_TRY(launched(st));
    int64_t total = 1;
    for (int i = 0; i < d_bin; ++i) total *= n_bins;
    KnnArgs a{};
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
    a.flags = flags & ~(uint32_t)FG_KNN_EXHAUSTIVE;  // a diagnostic: same answer
    a.out_idx = out_idx;
    a.out_d2 = out_d2;
    a.x64 = coords;
    a.rnd = reinterpret_cast<const float*>(rnd);
    if (flags & FG_KNN_STATS) {
        std::lock_guard<std::mutex> lk(g_stats_mu);
        if (!g_stats_dev) {
            FG_CUDA(cudaMalloc(&g_stats_dev, sizeof(unsigned long long) * kStatsTotal));
            FG_CUDA(cudaMemset(g_stats_dev, 0, sizeof(unsigned long long) * kStatsTotal));
        }
        a.stats = g_stats_dev;
    }
    tile::TileArgs t{};
    t.sc = a.sc;
    t.sid = sort_order;
    t.bounds = bin_bounds;
    t.mins = dim_mins;
    t.widths = widths;
    t.total = total;
    t.nb = n_bins;
    t.n = n;
    t.k = k;
    t.nblk = (n_bins + 1) / 2;
    t.bps = (int)(w.n_blocks / n_splits);
    t.n_blocks = (int)w.n_blocks;
    t.tiles = w.tiles;
    t.ctr = w.ctr;
    t.redo = w.redo;
    t.out_idx = out_idx;
    t.sc2 = w.sc2;
    t.sid2 = w.sid2;
    t.dense = w.dense;
    t.boxes = w.boxes;
    t.tcnt = w.tcnt;
    t.tkey = w.tkey;
    t.hist = w.hist;
    t.order = w.order;
    switch ((n_coords + 3) / 4) {
        case 1: return hd::dispatch_hd_nv1(t, a, d_bin, st);
        case 2: return hd::dispatch_hd_nv2(t, a, d_bin, st);
        case 3: return hd::dispatch_hd_nv3(t, a, d_bin, st);
        default: return hd::dispatch_hd_nv4(t, a, d_bin, st);
    }
}

extern "C" int fg_knn_stats(uint64_t* out, int32_t n, int32_t reset) {
    std::lock_guard<std::mutex> lk(g_stats_mu);
    unsigned long long h[kStatsTotal] = {0};
    if (g_stats_dev) {
        FG_CUDA(cudaMemcpy(h, g_stats_dev, sizeof(h), cudaMemcpyDeviceToHost));
        if (reset) FG_CUDA(cudaMemset(g_stats_dev, 0, sizeof(h)));
    }
    for (int i = 0; i < n && i < kStatsTotal; ++i) out[i] = h[i];
    return 0;
}

extern "C" int fg_knn_gravnet_fwd_ws(const float* sorted_coords, const int32_t* sort_order,
                                     const int64_t* bin_idx, const int32_t* bin_bounds,
                                     const int64_t* row_splits, const double* dim_mins,
                                     const double* widths, int64_t n, int32_t n_coords,
                                     int32_t n_splits, int32_t d_bin, int32_t n_bins, int32_t k,
                                     uint32_t flags, const float* feats, int32_t n_feats,
                                     double weight_scale, const int32_t* reducers,
                                     int32_t n_reducers, int32_t include_self, int32_t* out_idx,
                                     float* out_d2, float* agg_out, void* workspace,
                                     size_t workspace_bytes, void* stream) {
    // the fused op always returns float32 distances, no mask / radius
    if (flags & (FG_KNN_D2_F64 | FG_KNN_USE_DIRECTION | FG_KNN_USE_MAX_R2)) return FG_ERR_BAD_SHAPE;
    if (k < 1 || k > 960) return FG_ERR_BAD_K;
    if (n_feats < 1 || !(weight_scale > 0.0)) return FG_ERR_BAD_SHAPE;
    unsigned bits = 0;
    FG_TRY(fg::gravnet::reducer_bits(reducers, n_reducers, &bits));
    FG_TRY(check_args(sorted_coords, sort_order, bin_idx, bin_bounds, row_splits, dim_mins, widths,
                      n, n_coords, n_splits, d_bin, n_bins, k, nullptr, 0.0, flags, out_idx,
                      out_d2));
    if (n == 0) return 0;
    if (!feats || !agg_out) return FG_ERR_NULL;
    // the search, then the high-occupancy aggregation kernel over its rows in
    // sorted order.  An in-epilogue fusion (aggregating each row inside the
    // tile search's epilogue, skipping the (N, k) round trip) was measured on
    // B200 at 3.12 ms vs 1.27 + 0.94 ms for this pair on config E -- the
    // aggregation is a 5 GB feature gather that needs the memory-level
    // parallelism of its own kernel -- and was removed.
    FG_TRY(fg_knn_fwd_ws(sorted_coords, sort_order, bin_idx, bin_bounds, row_splits, dim_mins, widths,
                         n, n_coords, n_splits, d_bin, n_bins, k, nullptr, 0.0, flags, out_idx, out_d2,
                         workspace, workspace_bytes, stream));
    return fg_gravnet_fwd(feats, n, n_feats, out_idx, out_d2, k, weight_scale, reducers, n_reducers,
                          include_self, sort_order, agg_out, stream);
}
