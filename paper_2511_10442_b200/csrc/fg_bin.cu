// fg_bin.cu -- bin_by_coordinates for sm_100a (replaces pyx:66-139).
//
// K1 k_bbox          per-split min/max over the first d_bin dims: block
//                    reduction per (block chunk, split segment), one ordered-
//                    uint atomicMin/Max per block and dim.
// K1b k_bbox_final   dim_mins / widths exactly as pyx:114-118 (float64).
// K2 k_assign        cell = floor((x - min) / w) in float64, clamped, row-major
//                    flat, global id; warp-aggregated (match_any) histogram
//                    whose returning atomics give every vertex a rank in its
//                    cell (arrival order).
// K3 k_scan          single-pass decoupled-look-back exclusive scan of the
//                    histogram -> bin_bounds (+ a cursor copy).  CUB-free.
// K4 k_place         vertex v goes to bin_bounds[cell] + rank (no second
//                    atomic pass), its coordinates read coalesced and stored
//                    to sorted_coords with 16-byte stores (float4 rows padded
//                    to 4*ceil(n_c/4)); then the stable fix-up that makes
//                    sort_order identical to the reference's stable counting
//                    sort: each cell segment is put in vertex-id order --
//                    k_fix_small (thread per cell, <= 32: only segments the
//                    arrival order left unsorted are rewritten), k_fix_medium
//                    (CTA bitonic in smem, <= 4096) and k_fix_big (cluster
//                    in-order compaction over the split) -- and re-gathered.
#include <cooperative_groups.h>

#include <algorithm>

#include "fg_common.cuh"
#include "fg_scan.cuh"

namespace fg {

std::atomic<uint64_t> g_launches{0};

namespace binning {

constexpr int kMaxBinDims = 5;
constexpr int kSmallCell = 32;
constexpr int kMediumCell = 8192;  // CTA bitonic in 32 KB of shared memory (B: its 6 cells of 4.6-6.3k points)

struct BinWs {
    unsigned long long* bbox;  // n_splits * d_bin * 2 (ordered-double min, max)
    double* inv_w;           // n_splits * d_bin: RN(1 / width), the cell fast path
    int32_t* cursor;         // n_cells (histogram, then scatter cursor)
    unsigned long long* st;  // scan tile status words
    unsigned* counters;      // [0] scan tile ticket, [1] medium count, [2] big count
    int32_t* medium;         // medium cell list
    int32_t* big;            // big cell list
    int32_t* rank;           // n: arrival rank of every vertex in its cell
    int64_t n_tiles;
    int64_t list_cap;
};

size_t carve(BinWs* w, void* base, int64_t n, int32_t n_splits, int32_t d_bin, int64_t n_cells) {
    size_t off = 0;
    char* b = (char*)base;
    auto take = [&](size_t bytes) {
        off = align_up(off, 256);
        char* p = b ? b + off : nullptr;
        off += bytes;
        return p;
    };
    w->n_tiles = ceil_div(n_cells, kScanTile);
    w->list_cap = n / (kSmallCell + 1) + 1;
    w->bbox = (unsigned long long*)take(sizeof(unsigned long long) * (size_t)n_splits * d_bin * 2);
    w->inv_w = (double*)take(sizeof(double) * (size_t)n_splits * d_bin);
    w->cursor = (int32_t*)take(sizeof(int32_t) * (size_t)n_cells);
    w->st = (unsigned long long*)take(sizeof(unsigned long long) * (size_t)w->n_tiles);
    w->counters = (unsigned*)take(sizeof(unsigned) * 4);
    w->medium = (int32_t*)take(sizeof(int32_t) * (size_t)w->list_cap);
    w->big = (int32_t*)take(sizeof(int32_t) * (size_t)w->list_cap);
    w->rank = (int32_t*)take(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    return align_up(off, 256);
}

// ---------------------------------------------------------------- K1
// Order-preserving double <-> uint64 map (the bbox atomics; float input is
// widened exactly, so one map serves both coordinate types).
__device__ __forceinline__ unsigned long long double_to_ordered(double f) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(f);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double ordered_to_double(unsigned long long u) {
    const unsigned long long b = (u & 0x8000000000000000ull) ? (u & 0x7fffffffffffffffull) : ~u;
    return __longlong_as_double((long long)b);
}

// One launch initialises the whole workspace: bbox slots (even = min, odd =
// max), the histogram, the scan's tile status words and the counters (three
// memsets and a kernel before: ~25 us of a 1M-point binning).
__global__ void k_bin_init(unsigned long long* __restrict__ bbox, int64_t m, int32_t* __restrict__ hist,
                           int64_t n_cells, unsigned long long* __restrict__ status, int64_t n_tiles,
                           unsigned* __restrict__ counters) {
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = t0; i < m; i += stride) bbox[i] = (i & 1) ? 0ull : ~0ull;
    for (int64_t i = t0; i < n_tiles; i += stride) status[i] = 0ull;
    if (t0 < 4) counters[t0] = 0u;
    const int64_t n4 = n_cells >> 2;  // hist is 256-byte aligned (carve)
    int4* h4 = reinterpret_cast<int4*>(hist);
    for (int64_t i = t0; i < n4; i += stride) h4[i] = make_int4(0, 0, 0, 0);
    for (int64_t i = 4 * n4 + t0; i < n_cells; i += stride) hist[i] = 0;
}

template <typename T, int DB>
__global__ void __launch_bounds__(256) k_bbox(const T* __restrict__ coords, int64_t n, int n_c,
                                              const int64_t* __restrict__ rs, int n_splits,
                                              int64_t chunk, unsigned long long* __restrict__ bbox) {
    __shared__ T s_mn[8][DB], s_mx[8][DB];
    int64_t lo = blockIdx.x * chunk;
    const int64_t hi = min(n, lo + chunk);
    if (lo >= hi) return;
    int s = split_of(rs, n_splits, lo);
    while (lo < hi) {
        const int64_t seg_end = min(hi, rs[s + 1]);
        if (seg_end <= lo) {  // empty split
            ++s;
            continue;
        }
        T mn[DB], mx[DB];
#pragma unroll
        for (int d = 0; d < DB; ++d) {
            mn[d] = (T)__builtin_huge_val();
            mx[d] = -(T)__builtin_huge_val();
        }
        for (int64_t v = lo + threadIdx.x; v < seg_end; v += blockDim.x) {
#pragma unroll
            for (int d = 0; d < DB; ++d) {
                const T x = coords[v * n_c + d];
                mn[d] = min(mn[d], x);
                mx[d] = max(mx[d], x);
            }
        }
#pragma unroll
        for (int d = 0; d < DB; ++d) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                mn[d] = min(mn[d], __shfl_xor_sync(FG_FULL_MASK, mn[d], o));
                mx[d] = max(mx[d], __shfl_xor_sync(FG_FULL_MASK, mx[d], o));
            }
        }
        const int w = threadIdx.x >> 5;
        if (lane_id() == 0) {
#pragma unroll
            for (int d = 0; d < DB; ++d) {
                s_mn[w][d] = mn[d];
                s_mx[w][d] = mx[d];
            }
        }
        __syncthreads();
        if (threadIdx.x < DB) {
            const int d = threadIdx.x;
            T a = s_mn[0][d], b = s_mx[0][d];
            for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
                a = min(a, s_mn[i][d]);
                b = max(b, s_mx[i][d]);
            }
            atomicMin(&bbox[((int64_t)s * DB + d) * 2 + 0], double_to_ordered((double)a));
            atomicMax(&bbox[((int64_t)s * DB + d) * 2 + 1], double_to_ordered((double)b));
        }
        __syncthreads();
        lo = seg_end;
        ++s;
    }
}

// pyx:99-118: empty split keeps min 0 / width 1; width = ext / n_bins or 1.0.
__global__ void k_bbox_final(const unsigned long long* __restrict__ bbox, const int64_t* __restrict__ rs,
                             int n_splits, int d_bin, int n_bins, double* __restrict__ mins,
                             double* __restrict__ widths, double* __restrict__ inv_w) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= (int64_t)n_splits * d_bin) return;
    const int64_t s = i / d_bin;
    if (rs[s + 1] <= rs[s]) {
        mins[i] = 0.0;
        widths[i] = 1.0;
        inv_w[i] = 1.0;
        return;
    }
    const double mn = ordered_to_double(bbox[i * 2 + 0]);
    const double mx = ordered_to_double(bbox[i * 2 + 1]);
    const double ext = __dsub_rn(mx, mn);
    const double w = ext > 0.0 ? __ddiv_rn(ext, (double)n_bins) : 1.0;
    mins[i] = mn;
    widths[i] = w;
    inv_w[i] = __drcp_rn(w);
}

// ---------------------------------------------------------------- K2
template <typename T, int DB>
__global__ void __launch_bounds__(256) k_assign(const T* __restrict__ coords, int64_t n, int n_c,
                                                const int64_t* __restrict__ rs, int n_splits,
                                                int n_bins, int64_t total,
                                                const double* __restrict__ mins,
                                                const double* __restrict__ widths,
                                                const double* __restrict__ inv_w,
                                                int64_t* __restrict__ bin_idx,
                                                int32_t* __restrict__ hist,
                                                int32_t* __restrict__ rank, bool vec4) {
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool live = v < n;
    unsigned long long g = ~0ull;
    if (live) {
        const int s = split_of(rs, n_splits, v);
        T x[DB];
        bool done = false;
        if constexpr (sizeof(T) == 4 && DB == 4) {
            if (vec4) {  // n_c == 4, 16-byte aligned rows: one load
                const float4 t = __ldg(reinterpret_cast<const float4*>(coords) + v);
                x[0] = t.x; x[1] = t.y; x[2] = t.z; x[3] = t.w;
                done = true;
            }
        }
        if (!done) {
#pragma unroll
            for (int d = 0; d < DB; ++d) x[d] = coords[v * n_c + d];
        }
        int64_t flat = 0;
#pragma unroll
        for (int d = 0; d < DB; ++d) {
            // floor(RN(a / w)) exactly as the reference, without the division in
            // the common case: q1 = RN(a * RN(1/w)) is within 3.02u|q1| of RN(a/w)
            // (u = 2^-53), so when no integer lies within 5e-16|q1| of q1 both
            // floor the same; otherwise (cell edges, q = 0, the top edge,
            // non-finite values) the exact division decides.
            const double a = __dsub_rn((double)x[d], mins[(int64_t)s * DB + d]);
            const double q1 = __dmul_rn(a, inv_w[(int64_t)s * DB + d]);
            const double f1 = floor(q1);
            const double eps = 5e-16 * fabs(q1);
            const double q = (q1 - f1 > eps && (f1 + 1.0) - q1 > eps)
                                 ? q1
                                 : __ddiv_rn(a, widths[(int64_t)s * DB + d]);
            int64_t c = (int64_t)floor(q);
            c = c < 0 ? 0 : (c >= n_bins ? n_bins - 1 : c);
            flat = flat * n_bins + c;
        }
        g = (unsigned long long)((int64_t)s * total + flat);
        bin_idx[v] = (int64_t)g;
    }
    // warp-aggregated histogram: one returning atomic per distinct cell in the
    // warp; the old count + the lane's rank among its peers = arrival rank
    const unsigned peers = __match_any_sync(FG_FULL_MASK, g);
    const int leader = __ffs(peers) - 1;
    int32_t base = 0;
    if (live && leader == lane_id()) base = atomicAdd(&hist[g], __popc(peers));
    base = __shfl_sync(FG_FULL_MASK, base, leader);
    if (live) rank[v] = base + __popc(peers & lanemask_lt());
}

// ---------------------------------------------------------------- K4
template <int NV, typename T>
__device__ __forceinline__ void gather_row(const T* __restrict__ coords, int n_c, int32_t v,
                                           float4* __restrict__ dst) {
    const T* src = coords + (int64_t)v * n_c;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        float t[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) t[e] = (4 * j + e < n_c) ? (float)src[4 * j + e] : 0.0f;
        dst[j] = make_float4(t[0], t[1], t[2], t[3]);
    }
}

// Vertex v -> slot bin_bounds[cell] + arrival rank: sort_order and the
// coordinates (read coalesced) land in one pass; cells whose arrival order is
// not the id order are fixed below.
constexpr int kPlacePer = 4;  // vertices per thread: their loads are in flight together
template <int NV, typename T>
__global__ void __launch_bounds__(256) k_place(const int64_t* __restrict__ bin_idx,
                                               const int32_t* __restrict__ rank,
                                               const int32_t* __restrict__ bounds, int64_t n,
                                               const T* __restrict__ coords, int n_c,
                                               int32_t* __restrict__ sort_order,
                                               float4* __restrict__ sorted) {
    const int64_t v0 = (int64_t)blockIdx.x * (256 * kPlacePer) + threadIdx.x;
    int64_t g[kPlacePer];
    int32_t r[kPlacePer], p[kPlacePer];
#pragma unroll
    for (int j = 0; j < kPlacePer; ++j) {
        const int64_t v = v0 + 256 * j;
        g[j] = v < n ? __ldcs(bin_idx + v) : -1;
        r[j] = v < n ? __ldcs(rank + v) : 0;
    }
#pragma unroll
    for (int j = 0; j < kPlacePer; ++j) p[j] = g[j] >= 0 ? __ldg(bounds + g[j]) + r[j] : -1;
#pragma unroll
    for (int j = 0; j < kPlacePer; ++j) {
        if (p[j] < 0) continue;
        const int64_t v = v0 + 256 * j;
        sort_order[p[j]] = (int32_t)v;
        gather_row<NV>(coords, n_c, (int32_t)v, sorted + (int64_t)p[j] * NV);
    }
}

// Thread per cell: sort segments of <= 32 ids (insertion sort) and re-gather
// the ones that were out of order;
// longer segments are queued for the CTA-level fix-ups.
template <int NV, typename T>
__global__ void __launch_bounds__(256) k_fix_small(const int32_t* __restrict__ bounds, int64_t n_cells,
                                                   int32_t* __restrict__ sort_order,
                                                   const T* __restrict__ coords, int n_c,
                                                   float4* __restrict__ sorted,
                                                   unsigned* __restrict__ counters,
                                                   int32_t* __restrict__ medium,
                                                   int32_t* __restrict__ big) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= n_cells) return;
    const int32_t lo = bounds[c], hi = bounds[c + 1];
    const int len = hi - lo;
    if (len == 0) return;
    if (len > kSmallCell) {
        if (len > kMediumCell)
            big[atomicAdd(&counters[2], 1u)] = (int32_t)c;
        else
            medium[atomicAdd(&counters[1], 1u)] = (int32_t)c;
        return;
    }
    if (len == 1) return;  // k_place wrote it
    int32_t ids[kSmallCell];
    bool sorted_in = true;
    for (int i = 0; i < len; ++i) {
        int32_t x = sort_order[lo + i];
        sorted_in &= i == 0 || ids[i - 1] < x;
        int j = i;
        while (j > 0 && ids[j - 1] > x) {
            ids[j] = ids[j - 1];
            --j;
        }
        ids[j] = x;
    }
    if (sorted_in) return;  // arrival order == id order: k_place wrote it
    for (int i = 0; i < len; ++i) {
        sort_order[lo + i] = ids[i];
        gather_row<NV>(coords, n_c, ids[i], sorted + (int64_t)(lo + i) * NV);
    }
}

template <int NV, typename T>
__global__ void __launch_bounds__(1024) k_fix_medium(const int32_t* __restrict__ bounds,
                                                     int32_t* __restrict__ sort_order,
                                                     const T* __restrict__ coords, int n_c,
                                                     float4* __restrict__ sorted,
                                                     const unsigned* __restrict__ counters,
                                                     const int32_t* __restrict__ medium) {
    __shared__ int32_t s[kMediumCell];
    const unsigned count = counters[1];
    for (unsigned it = blockIdx.x; it < count; it += gridDim.x) {
        const int32_t c = medium[it];
        const int32_t lo = bounds[c], len = bounds[c + 1] - lo;
        int p2 = 64;
        while (p2 < len) p2 <<= 1;
        for (int i = threadIdx.x; i < p2; i += blockDim.x)
            s[i] = i < len ? sort_order[lo + i] : 0x7fffffff;
        __syncthreads();
        for (int size = 2; size <= p2; size <<= 1)
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int i = threadIdx.x; i < p2 / 2; i += blockDim.x) {
                    const int a = ((i & ~(stride - 1)) << 1) | (i & (stride - 1)), b = a + stride;  // stride: a power of 2
                    const bool up = (a & size) == 0;
                    const int32_t x = s[a], y = s[b];
                    if ((x > y) == up) {
                        s[a] = y;
                        s[b] = x;
                    }
                }
                __syncthreads();
            }
        for (int i = threadIdx.x; i < len; i += blockDim.x) {
            sort_order[lo + i] = s[i];
            gather_row<NV>(coords, n_c, s[i], sorted + (int64_t)(lo + i) * NV);
        }
        __syncthreads();
    }
}

// Huge cells: the members of cell c in ascending id order are exactly the
// vertices v of its split with bin_idx[v] == c, in order.  A cluster of
// kBigCtas CTAs takes one big cell: each CTA owns 1/kBigCtas of the split
// range and each of its warps a contiguous slice of that; pass 1 counts the
// slice's members (ballots, no block barriers), one block scan + a scan over
// the cluster's CTAs through distributed shared memory give every warp its
// output offset, pass 2 writes the members in order (ballot ranks) and
// gathers their coordinates.  One CTA walking the whole split took 217 us at
// config B (200k points, ~15 big cells).
constexpr int kBigCtas = 8;
constexpr int kBigThreads = 512;

template <int NV, typename T>
__global__ void __cluster_dims__(kBigCtas, 1, 1) __launch_bounds__(kBigThreads)
k_fix_big(const int32_t* __restrict__ bounds, const int64_t* __restrict__ bin_idx,
          const int64_t* __restrict__ rs, int64_t total, int32_t* __restrict__ sort_order,
          const T* __restrict__ coords, int n_c, float4* __restrict__ sorted,
          const unsigned* __restrict__ counters, const int32_t* __restrict__ big) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    constexpr int kW = kBigThreads / 32;
    __shared__ int32_t s_warp[kW];
    __shared__ int32_t s_cta;  // this CTA's member count (read by the cluster)
    const unsigned count = counters[2];
    const int rank = (int)cluster.block_rank();
    const unsigned n_clusters = gridDim.x / kBigCtas;
    const int w = threadIdx.x >> 5, lane = lane_id();
    for (unsigned it = blockIdx.x / kBigCtas; it < count; it += n_clusters) {
        const int32_t c = big[it];
        const int64_t s = c / total;
        const int32_t lo = bounds[c];
        const int64_t v0 = rs[s], v1 = rs[s + 1];
        const int64_t per_cta = (v1 - v0 + kBigCtas - 1) / kBigCtas;
        const int64_t a0 = v0 + per_cta * rank, a1 = min(v1, a0 + per_cta);
        const int64_t per_w = (max(a1 - a0, (int64_t)0) + kW - 1) / kW;
        const int64_t b0 = a0 + per_w * w, b1 = min(a1, b0 + per_w);
        int cnt = 0;
        for (int64_t v = b0 + lane; v - lane < b1; v += 32)
            cnt += __popc(__ballot_sync(FG_FULL_MASK, v < b1 && bin_idx[v] == c));
        if (lane == 0) s_warp[w] = cnt;
        __syncthreads();
        if (w == 0) {
            const int x = lane < kW ? s_warp[lane] : 0;
            const int incl = warp_inclusive_scan(x);
            if (lane < kW) s_warp[lane] = incl - x;
            if (lane == kW - 1) s_cta = incl;
        }
        cluster.sync();  // every CTA's count visible cluster-wide
        int base = 0;
        for (int r = 0; r < rank; ++r) base += *cluster.map_shared_rank(&s_cta, r);
        int out = lo + base + s_warp[w];
        for (int64_t v = b0 + lane; v - lane < b1; v += 32) {
            const bool mem = v < b1 && bin_idx[v] == c;
            const unsigned bal = __ballot_sync(FG_FULL_MASK, mem);
            if (mem) {
                const int p = out + __popc(bal & lanemask_lt());
                sort_order[p] = (int32_t)v;
                gather_row<NV>(coords, n_c, (int32_t)v, sorted + (int64_t)p * NV);
            }
            out += __popc(bal);
        }
        cluster.sync();  // s_cta / s_warp are reused by the next cell
    }
}

template <int NV, typename T>
int launch_fixups(const int32_t* bounds, int64_t n, int64_t n_cells, int32_t* sort_order, const int64_t* bin_idx,
                  const int64_t* rs, int64_t total, const T* coords, int n_c, float* sorted,
                  const BinWs& w, cudaStream_t st) {
    float4* s4 = reinterpret_cast<float4*>(sorted);
    if (n > 0) {
        k_place<NV, T><<<(unsigned)ceil_div(n, 256 * kPlacePer), 256, 0, st>>>(bin_idx, w.rank, bounds, n, coords,
                                                                  n_c, sort_order, s4);
        FG_TRY(launched(st));
    }
    if (n_cells > 0) {
        k_fix_small<NV, T><<<(unsigned)ceil_div(n_cells, 256), 256, 0, st>>>(
            bounds, n_cells, sort_order, coords, n_c, s4, w.counters, w.medium, w.big);
        FG_TRY(launched(st));
    }
    k_fix_medium<NV, T><<<296, 1024, 0, st>>>(bounds, sort_order, coords, n_c, s4, w.counters,
                                           w.medium);
    FG_TRY(launched(st));
    k_fix_big<NV, T><<<kBigCtas * 37, kBigThreads, 0, st>>>(bounds, bin_idx, rs, total, sort_order,
                                                             coords, n_c, s4, w.counters, w.big);
    return launched(st);
}

template <typename T, int DB>
int launch_bin_core(const T* coords, int64_t n, int n_c, const int64_t* rs, int n_splits,
                    int n_bins, int64_t total, double* mins, double* widths, int64_t* bin_idx,
                    const BinWs& w, cudaStream_t st) {
    const int64_t m = (int64_t)n_splits * DB * 2;
    const int64_t n_cells = total * n_splits;
    const int64_t init_threads = std::max<int64_t>({m, w.n_tiles, (int64_t)4, ceil_div(n_cells, 4)});
    k_bin_init<<<(unsigned)std::min<int64_t>(ceil_div(init_threads, 256), 148 * 8), 256, 0, st>>>(
        w.bbox, m, w.cursor, n_cells, w.st, w.n_tiles, w.counters);
    FG_TRY(launched(st));
    if (n > 0) {
        const int64_t chunk = 2048;
        k_bbox<T, DB><<<(unsigned)ceil_div(n, chunk), 256, 0, st>>>(coords, n, n_c, rs, n_splits,
                                                                 chunk, w.bbox);
        FG_TRY(launched(st));
    }
    k_bbox_final<<<(unsigned)ceil_div((int64_t)n_splits * DB, 128), 128, 0, st>>>(
        w.bbox, rs, n_splits, DB, n_bins, mins, widths, w.inv_w);
    FG_TRY(launched(st));
    if (n > 0) {
        const bool vec4 = n_c == 4 && (reinterpret_cast<uintptr_t>(coords) & 15) == 0;
        k_assign<T, DB><<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(
            coords, n, n_c, rs, n_splits, n_bins, total, mins, widths, w.inv_w, bin_idx, w.cursor, w.rank,
            vec4);
        FG_TRY(launched(st));
    }
    return 0;
}

}  // namespace binning
}  // namespace fg

using namespace fg;
using namespace fg::binning;

extern "C" int fg_bin_workspace_size(int64_t n, int32_t n_splits, int32_t d_bin, int32_t n_bins,
                                     size_t* bytes) {
    if (!bytes) return FG_ERR_NULL;
    if (n < 0 || n_splits < 1 || n_bins < 1) return FG_ERR_BAD_SHAPE;
    if (d_bin < 1 || d_bin > kMaxBinDims) return FG_ERR_TOO_FEW_DIMS;
    int64_t total = 1;
    for (int i = 0; i < d_bin; ++i) total *= n_bins;
    BinWs w;
    *bytes = carve(&w, nullptr, n, n_splits, d_bin, total * n_splits);
    return 0;
}

namespace {
template <typename T>
int bin_entry(const T* coords, int64_t n, int32_t n_coords, const int64_t* row_splits,
              int32_t n_splits, int32_t d_bin, int32_t n_bins, int64_t* bin_idx,
              int32_t* sort_order, int32_t* bin_bounds, double* dim_mins, double* widths,
              float* sorted_coords, void* workspace, size_t workspace_bytes, void* stream) {
    if (n < 0 || n >= ((int64_t)1 << 31) || n_splits < 1 || n_bins < 1) return FG_ERR_BAD_SHAPE;
    if (n_coords > 16) return FG_ERR_TOO_MANY_DIMS;
    if (d_bin < 1 || d_bin > kMaxBinDims || d_bin > n_coords) return FG_ERR_TOO_FEW_DIMS;
    if (!row_splits || !bin_bounds || !dim_mins || !widths || !workspace) return FG_ERR_NULL;
    if (n > 0 && (!coords || !bin_idx || !sort_order || !sorted_coords)) return FG_ERR_NULL;
    int64_t total = 1;
    for (int i = 0; i < d_bin; ++i) total *= n_bins;
    const int64_t n_cells = total * n_splits;
    BinWs w;
    const size_t need = carve(&w, workspace, n, n_splits, d_bin, n_cells);
    if (workspace_bytes < need) return FG_ERR_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;

    switch (d_bin) {
        case 1: FG_TRY((launch_bin_core<T, 1>(coords, n, n_coords, row_splits, n_splits, n_bins, total, dim_mins, widths, bin_idx, w, st))); break;
        case 2: FG_TRY((launch_bin_core<T, 2>(coords, n, n_coords, row_splits, n_splits, n_bins, total, dim_mins, widths, bin_idx, w, st))); break;
        case 3: FG_TRY((launch_bin_core<T, 3>(coords, n, n_coords, row_splits, n_splits, n_bins, total, dim_mins, widths, bin_idx, w, st))); break;
        case 4: FG_TRY((launch_bin_core<T, 4>(coords, n, n_coords, row_splits, n_splits, n_bins, total, dim_mins, widths, bin_idx, w, st))); break;
        default: FG_TRY((launch_bin_core<T, 5>(coords, n, n_coords, row_splits, n_splits, n_bins, total, dim_mins, widths, bin_idx, w, st))); break;
    }
    fg::k_scan<<<(unsigned)w.n_tiles, kScanThreads, 0, st>>>(w.cursor, n_cells, bin_bounds, nullptr,
                                                        w.st, w.counters);
    FG_TRY(launched(st));
    if (n == 0) return 0;
    const int nv = (n_coords + 3) / 4;
    switch (nv) {
        case 1: return launch_fixups<1, T>(bin_bounds, n, n_cells, sort_order, bin_idx, row_splits, total, coords, n_coords, sorted_coords, w, st);
        case 2: return launch_fixups<2, T>(bin_bounds, n, n_cells, sort_order, bin_idx, row_splits, total, coords, n_coords, sorted_coords, w, st);
        case 3: return launch_fixups<3, T>(bin_bounds, n, n_cells, sort_order, bin_idx, row_splits, total, coords, n_coords, sorted_coords, w, st);
        default: return launch_fixups<4, T>(bin_bounds, n, n_cells, sort_order, bin_idx, row_splits, total, coords, n_coords, sorted_coords, w, st);
    }
}
}  // namespace

extern "C" int fg_bin_by_coordinates(const float* coords, int64_t n, int32_t n_coords,
                                     const int64_t* row_splits, int32_t n_splits, int32_t d_bin,
                                     int32_t n_bins, int64_t* bin_idx, int32_t* sort_order,
                                     int32_t* bin_bounds, double* dim_mins, double* widths,
                                     float* sorted_coords, void* workspace,
                                     size_t workspace_bytes, void* stream) {
    return bin_entry<float>(coords, n, n_coords, row_splits, n_splits, d_bin, n_bins, bin_idx,
                            sort_order, bin_bounds, dim_mins, widths, sorted_coords, workspace,
                            workspace_bytes, stream);
}

extern "C" int fg_bin_by_coordinates_f64(const double* coords, int64_t n, int32_t n_coords,
                                         const int64_t* row_splits, int32_t n_splits,
                                         int32_t d_bin, int32_t n_bins, int64_t* bin_idx,
                                         int32_t* sort_order, int32_t* bin_bounds,
                                         double* dim_mins, double* widths, float* sorted_coords,
                                         void* workspace, size_t workspace_bytes, void* stream) {
    return bin_entry<double>(coords, n, n_coords, row_splits, n_splits, d_bin, n_bins, bin_idx,
                             sort_order, bin_bounds, dim_mins, widths, sorted_coords, workspace,
                             workspace_bytes, stream);
}

namespace fg {
namespace binning {
__global__ void k_index_replace(int32_t* __restrict__ io, int64_t n, const int32_t* __restrict__ lut) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t x = io[i];
        if (x >= 0) io[i] = lut[x];
    }
}
}  // namespace binning
}  // namespace fg

extern "C" int fg_index_replacer(int32_t* io, int64_t n, const int32_t* lut, int64_t lut_n,
                                 void* stream) {
    if (n < 0 || lut_n < 0) return FG_ERR_BAD_SHAPE;
    if (n == 0) return 0;
    if (!io || !lut) return FG_ERR_NULL;
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(n, 256), 148 * 16);
    k_index_replace<<<grid, 256, 0, st>>>(io, n, lut);
    return launched(st);
}

extern "C" const char* fg_error_string(int code) {
    switch (code) {
        case FG_OK: return "ok";
        case FG_ERR_BAD_K: return "k must be a positive integer within the supported range";
        case FG_ERR_BAD_SHAPE: return "bad array sizes";
        case FG_ERR_TOO_FEW_DIMS: return "d_bin must be in [1, 5] and <= n_coords";
        case FG_ERR_WORKSPACE: return "workspace too small";
        case FG_ERR_NULL: return "required pointer is NULL";
        case FG_ERR_TOO_MANY_DIMS: return "n_coords must be <= 16";
        case FG_ERR_BAD_RADIUS: return "max_radius2 must be >= 0";
        case FG_ERR_BAD_CAPACITY: return "capacities must be >= 1";
        case FG_ERR_UNSUPPORTED: return "sizes outside the limits of the requested mode (deterministic backward: n <= 2^23, n*k < 2^32)";
        default: return code > 0 ? cudaGetErrorString((cudaError_t)code) : "unknown error";
    }
}

extern "C" int fg_abi_version(void) { return FG_ABI_VERSION; }

extern "C" uint64_t fg_launch_count(void) { return g_launches.load(); }
