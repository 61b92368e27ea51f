// fg_oc.cu -- object-condensation association matrices (replaces
// G/ocgraph.py:114-202: find_unique, max_same_count, oc_helper; the paper's
// CUDA Algorithm 3) for sm_100a.
//
// find_unique: one pass inserts every non-background vertex's (id, split) key
// into an open-addressing table with a 16-byte compare-and-swap (the key is
// two 64-bit words: ids are opaque int64 labels), recording the first vertex
// (atomicMin) and the member count per key.  A vertex is an object's first
// occurrence iff it is its key's minimum; the exclusive scan of those flags in
// vertex order is exactly the reference's object order (splits ascending,
// first occurrence inside a split).
//
// oc_helper: one block per (object, 2048-vertex window chunk), in ticket
// order.  Members of the chunk are ranked by ballots; the members before the
// chunk come from a decoupled look-back over the object's earlier chunks;
// members go to m[i, rank] (truncated to n_maxuq), non-members to
// m_not[i, offset - rank]; the object's last chunk fills the -1 suffixes.  The
// windows are re-read per object from L2 (every object of a split scans the
// same window).  Integer work throughout: bit-exact.
#include "fg_common.cuh"
#include "fg_scan.cuh"

namespace fg {
namespace oc {

struct __align__(16) Key {
    unsigned long long id, split;
};
constexpr unsigned long long kEmpty = ~0ull;
constexpr int kThreads = 256;
#ifndef FG_OC_ITEMS
#define FG_OC_ITEMS 8
#endif
constexpr int kItems = FG_OC_ITEMS;
constexpr int kChunk = kThreads * kItems;

__device__ __forceinline__ bool key_eq(const Key& a, const Key& b) { return a.id == b.id && a.split == b.split; }

__device__ __forceinline__ int split_of(const int64_t* __restrict__ rs, int S, int64_t v) {
    int lo = 0, hi = S;  // largest s with rs[s] <= v (empty splits skipped)
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (rs[mid] <= v) lo = mid; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

// Lanes holding the same key (consecutive vertices of one object) are merged
// first (match_any): one table operation per group, the group's lowest
// vertex and size.
__global__ void k_oc_insert(const int64_t* __restrict__ asso, int64_t n, const int64_t* __restrict__ rs,
                            int S, Key* __restrict__ table, uint64_t cap_mask,
                            unsigned long long* __restrict__ first, unsigned long long* __restrict__ count,
                            int64_t* __restrict__ slot_of) {
    const int lane = lane_id();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); b < n; b += stride) {
        const int64_t v = b + lane;  // b is warp-uniform: the match below sees the whole warp
        const int64_t a = v < n ? asso[v] : -1;
        const int s = a >= 0 ? split_of(rs, S, v) : -1;
        const unsigned grp = __match_any_sync(FG_FULL_MASK, (unsigned long long)a) &
                             __match_any_sync(FG_FULL_MASK, s);
        const int leader = __ffs(grp) - 1;
        int64_t h = -1;
        if (a >= 0 && lane == leader) {
            const Key key{(unsigned long long)a, (unsigned long long)s};
            const Key empty{kEmpty, kEmpty};
            uint64_t t = mix((uint64_t)a * 0x9e3779b97f4a7c15ull + (uint64_t)s) & cap_mask;
            for (;;) {
                const Key old = atomicCAS(&table[t], empty, key);
                if (key_eq(old, empty) || key_eq(old, key)) break;
                t = (t + 1) & cap_mask;
            }
            atomicMin(&first[t], (unsigned long long)v);  // lowest vertex of the group
            atomicAdd(&count[t], (unsigned long long)__popc(grp));
            h = (int64_t)t;
        }
        h = __shfl_sync(FG_FULL_MASK, h, leader);
        if (v < n) slot_of[v] = a >= 0 ? h : -1;
    }
}

__global__ void k_oc_flag(const int64_t* __restrict__ slot_of, int64_t n,
                          const unsigned long long* __restrict__ first, int32_t* __restrict__ flag) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t h = slot_of[v];
        flag[v] = (h >= 0 && first[h] == (unsigned long long)v) ? 1 : 0;
    }
}

// summary[0] = number of objects, summary[1] = largest member count
__global__ void k_oc_emit(const int64_t* __restrict__ asso, int64_t n, const int64_t* __restrict__ rs, int S,
                          const int64_t* __restrict__ slot_of, const int32_t* __restrict__ flag,
                          const int32_t* __restrict__ excl, const unsigned long long* __restrict__ count,
                          int64_t* __restrict__ unique_idx, int64_t* __restrict__ unique_rs,
                          int64_t* __restrict__ counts, int64_t* __restrict__ summary) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        if (v == 0) summary[0] = excl[n];
        if (!flag[v]) continue;
        const int64_t o = excl[v];
        const unsigned long long c = count[slot_of[v]];
        unique_idx[o] = asso[v];
        unique_rs[o] = split_of(rs, S, v);
        if (counts) counts[o] = (int64_t)c;
        atomicMax((unsigned long long*)&summary[1], c);
    }
}

// ---------------------------------------------------------------- matrices
struct MatArgs {
    const int64_t* asso;
    const int64_t* rs;
    const int64_t* uidx;
    const int64_t* urs;
    int64_t n_u, n_maxuq, n_maxrs;
    int n_chunks;                  // chunks of the largest window
    unsigned long long* status;    // [n_u][n_chunks] look-back words
    unsigned* ticket;
    int64_t* m;
    int64_t* m_not;
    unsigned long long* visits;
};

__device__ __forceinline__ void window_of(const MatArgs& a, int64_t i, int64_t& start, int64_t& len) {
    const int s = (int)a.urs[i];
    start = a.rs[s];
    len = min(a.rs[s + 1] - start, a.n_maxrs);
}

// One block per (object, window chunk), in ticket order so every block's
// predecessors have started: members of the chunk are ranked by ballots, the
// members before the chunk come from a decoupled look-back over the object's
// earlier chunks (flag 1 = chunk count, flag 2 = inclusive prefix), and the
// object's last chunk fills the -1 suffixes.
__global__ void __launch_bounds__(kThreads) k_oc_rows(const MatArgs a) {
    __shared__ int s_cnt[kItems * (kThreads / 32)];
    __shared__ int s_pre, s_tot;
    __shared__ unsigned s_tile;
    static_assert(kItems * (kThreads / 32) % 32 == 0, "scan layout");
    if (threadIdx.x == 0) s_tile = atomicAdd(a.ticket, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t i = tile / a.n_chunks;
    const int c = (int)(tile - i * a.n_chunks);
    int64_t start, len;
    window_of(a, i, start, len);
    const int n_ch = max(1, (int)((len + kChunk - 1) / kChunk));  // this object's chunks
    if (c >= n_ch) return;                                  // past its window (uniform)
    if (c == 0 && threadIdx.x == 0) atomicAdd(a.visits, (unsigned long long)len);
    const int64_t obj = a.uidx[i];
    const int lane = lane_id(), w = threadIdx.x >> 5;
    // item j of this thread = vertex c0 + j*kThreads + tid (coalesced loads and,
    // since ranks advance by at most one per lane, near-coalesced stores); the
    // rank of a vertex = members before it in (item, warp, lane) order
    const int o0 = c * kChunk + (int)threadIdx.x;  // window offsets fit in 32 bits
    const int len32 = (int)len;
    const int64_t* src = a.asso + start + o0;
    unsigned bal[kItems];
#pragma unroll
    for (int j = 0; j < kItems; ++j)
        bal[j] = __ballot_sync(FG_FULL_MASK, o0 + j * kThreads < len32 && src[j * kThreads] == obj);
    if (lane < kItems) {
        unsigned b = 0;
#pragma unroll
        for (int j = 0; j < kItems; ++j) b = lane == j ? bal[j] : b;
        s_cnt[lane * (kThreads / 32) + w] = __popc(b);
    }
    __syncthreads();
    if (w == 0) {  // exclusive scan of the kItems x warps counts, then the look-back
        constexpr int P = kItems * (kThreads / 32) / 32;
        int v[P], run = 0;
#pragma unroll
        for (int q = 0; q < P; ++q) {
            v[q] = s_cnt[lane * P + q];
            run += v[q];
        }
        const int incl = warp_inclusive_scan(run);
        int ex = incl - run;
#pragma unroll
        for (int q = 0; q < P; ++q) {
            s_cnt[lane * P + q] = ex;
            ex += v[q];
        }
        const int total = __shfl_sync(FG_FULL_MASK, incl, 31);
        unsigned long long* st = a.status + i * a.n_chunks;
        int prefix = 0;
        if (c == 0) {
            if (lane == 0) atomicExch(&st[0], (2ull << 62) | (unsigned)total);
        } else {
            if (lane == 0) atomicExch(&st[c], (1ull << 62) | (unsigned)total);
            int end = c - 1;
            for (;;) {
                const int idx = end - lane;
                unsigned long long word = 2ull << 62;  // before chunk 0: prefix 0
                if (idx >= 0) {
                    do {
                        word = *((volatile unsigned long long*)&st[idx]);
                    } while ((word >> 62) == 0);
                }
                const int val = idx >= 0 ? (int)(word & 0xffffffffu) : 0;
                const unsigned pm = __ballot_sync(FG_FULL_MASK, (word >> 62) == 2);
                if (pm) {
                    const int first = __ffs(pm) - 1;
                    prefix += __reduce_add_sync(FG_FULL_MASK, lane <= first ? val : 0);
                    break;
                }
                prefix += __reduce_add_sync(FG_FULL_MASK, val);
                end -= 32;
            }
            if (lane == 0) atomicExch(&st[c], (2ull << 62) | (unsigned)(prefix + total));
        }
        if (lane == 0) {
            s_pre = prefix;
            s_tot = prefix + total;
        }
    }
    __syncthreads();
    int64_t* mrow = a.m + i * a.n_maxuq;
    int64_t* nrow = a.m_not ? a.m_not + i * a.n_maxrs : nullptr;
    const int pre = s_pre;
    const int cap_uq = (int)min(a.n_maxuq, (int64_t)INT32_MAX);
    const unsigned below = lanemask_lt();
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        const int o = o0 + j * kThreads;
        if (o >= len32) break;
        const int r = pre + s_cnt[j * (kThreads / 32) + w] + __popc(bal[j] & below);
        if ((bal[j] >> lane) & 1u) {
            if (r < cap_uq) mrow[r] = start + o;
        } else if (nrow) {
            nrow[o - r] = start + o;  // o - r non-members precede it
        }
    }
    if (c == n_ch - 1) {  // -1 suffixes: this is the object's last chunk
        const int64_t tot = s_tot;
        for (int64_t x = min(tot, a.n_maxuq) + threadIdx.x; x < a.n_maxuq; x += kThreads) mrow[x] = -1;
        if (nrow)
            for (int64_t x = (len - tot) + threadIdx.x; x < a.n_maxrs; x += kThreads) nrow[x] = -1;
    }
}

}  // namespace oc
}  // namespace fg

using namespace fg;
using namespace fg::oc;

namespace {
uint64_t table_cap(int64_t n) {  // load factor <= 0.8 even if every vertex is its own object
    uint64_t c = 1024;
    while (c < (uint64_t)n + (uint64_t)n / 4) c <<= 1;
    return c;
}
size_t n_scan_tiles(int64_t n) { return (size_t)ceil_div(n, (int64_t)kScanTile); }

struct UniqueWs {
    Key* table;
    unsigned long long *first, *count;
    int64_t* slot_of;
    int32_t *flag, *excl, *cursor;
    unsigned long long* status;
    unsigned* ticket;
    size_t bytes;
};

UniqueWs carve_unique(void* base, int64_t n) {
    UniqueWs w{};
    const uint64_t cap = table_cap(n);
    char* p = (char*)base;
    size_t off = 0;
    auto take = [&](size_t b) {
        void* r = p ? p + off : nullptr;
        off += align_up(b, 256);
        return r;
    };
    w.table = (Key*)take(sizeof(Key) * cap);
    w.first = (unsigned long long*)take(8 * cap);
    w.count = (unsigned long long*)take(8 * cap);
    w.slot_of = (int64_t*)take(8 * (size_t)n);
    w.flag = (int32_t*)take(4 * (size_t)n);
    w.excl = (int32_t*)take(4 * ((size_t)n + 1));
    w.cursor = (int32_t*)take(4 * (size_t)n);
    w.status = (unsigned long long*)take(8 * (n_scan_tiles(n) + 1));
    w.ticket = (unsigned*)take(16);
    w.bytes = off;
    return w;
}
}  // namespace

extern "C" int fg_oc_unique_workspace_size(int64_t n, size_t* bytes) {
    if (!bytes) return FG_ERR_NULL;
    if (n < 0 || n > INT32_MAX - 1) return FG_ERR_BAD_SHAPE;
    *bytes = carve_unique(nullptr, n).bytes;
    return 0;
}

extern "C" int fg_oc_find_unique(const int64_t* asso, int64_t n, const int64_t* row_splits, int32_t n_splits,
                                 int64_t* unique_idx, int64_t* unique_rs, int64_t* counts, int64_t* summary,
                                 void* workspace, size_t workspace_bytes, void* stream) {
    if (n < 0 || n > INT32_MAX - 1 || n_splits < 1) return FG_ERR_BAD_SHAPE;
    if (!row_splits || !summary) return FG_ERR_NULL;
    cudaStream_t st = (cudaStream_t)stream;
    FG_CUDA(cudaMemsetAsync(summary, 0, 2 * sizeof(int64_t), st));
    if (n == 0) return 0;
    if (!asso || !unique_idx || !unique_rs || !workspace) return FG_ERR_NULL;
    UniqueWs w = carve_unique(workspace, n);
    if (workspace_bytes < w.bytes) return FG_ERR_WORKSPACE;
    const uint64_t cap = table_cap(n);
    FG_CUDA(cudaMemsetAsync(w.table, 0xff, sizeof(Key) * cap, st));
    FG_CUDA(cudaMemsetAsync(w.first, 0xff, 8 * cap, st));
    FG_CUDA(cudaMemsetAsync(w.count, 0, 8 * cap, st));
    FG_CUDA(cudaMemsetAsync(w.status, 0, 8 * (n_scan_tiles(n) + 1), st));
    FG_CUDA(cudaMemsetAsync(w.ticket, 0, 16, st));
    const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(n, (int64_t)256), 148 * 16);
    k_oc_insert<<<blocks, 256, 0, st>>>(asso, n, row_splits, n_splits, w.table, cap - 1, w.first, w.count,
                                        w.slot_of);
    FG_TRY(launched(st));
    k_oc_flag<<<blocks, 256, 0, st>>>(w.slot_of, n, w.first, w.flag);
    FG_TRY(launched(st));
    k_scan<<<(unsigned)n_scan_tiles(n), kScanThreads, 0, st>>>(w.flag, n, w.excl, w.cursor, w.status, w.ticket);
    FG_TRY(launched(st));
    k_oc_emit<<<blocks, 256, 0, st>>>(asso, n, row_splits, n_splits, w.slot_of, w.flag, w.excl, w.count,
                                      unique_idx, unique_rs, counts, summary);
    return launched(st);
}

extern "C" int fg_oc_matrices_workspace_size(int64_t n_unique, int64_t max_window, size_t* bytes) {
    if (!bytes) return FG_ERR_NULL;
    if (n_unique < 0 || max_window < 0) return FG_ERR_BAD_SHAPE;
    const int64_t chunks = std::max<int64_t>(1, ceil_div(max_window, (int64_t)kChunk));
    *bytes = align_up(sizeof(unsigned long long) * (size_t)(n_unique * chunks), 256) + 256;
    return 0;
}

extern "C" int fg_oc_matrices(const int64_t* asso, const int64_t* row_splits, int32_t n_splits,
                              const int64_t* unique_idx, const int64_t* unique_rs, int64_t n_unique,
                              int64_t n_maxuq, int64_t n_maxrs, int64_t max_window, int64_t* m, int64_t* m_not,
                              int64_t* visits, void* workspace, size_t workspace_bytes, void* stream) {
    if (n_maxuq < 1 || n_maxrs < 1) return FG_ERR_BAD_CAPACITY;
    if (n_unique < 0 || max_window < 0 || max_window > INT32_MAX - 2 * kChunk || n_splits < 1)
        return FG_ERR_BAD_SHAPE;
    if (!visits) return FG_ERR_NULL;
    cudaStream_t st = (cudaStream_t)stream;
    FG_CUDA(cudaMemsetAsync(visits, 0, sizeof(int64_t), st));
    if (n_unique == 0) return 0;
    if (!asso || !row_splits || !unique_idx || !unique_rs || !m || !workspace) return FG_ERR_NULL;
    size_t need = 0;
    FG_TRY(fg_oc_matrices_workspace_size(n_unique, max_window, &need));
    if (workspace_bytes < need) return FG_ERR_WORKSPACE;
    MatArgs a{};
    a.asso = asso;
    a.rs = row_splits;
    a.uidx = unique_idx;
    a.urs = unique_rs;
    a.n_u = n_unique;
    a.n_maxuq = n_maxuq;
    a.n_maxrs = n_maxrs;
    a.n_chunks = (int)std::max<int64_t>(1, ceil_div(std::min(max_window, n_maxrs), (int64_t)kChunk));
    const size_t n_status = (size_t)n_unique * a.n_chunks;
    a.status = (unsigned long long*)workspace;
    a.ticket = (unsigned*)((char*)workspace + align_up(sizeof(unsigned long long) * n_status, 256));
    a.m = m;
    a.m_not = m_not;
    a.visits = (unsigned long long*)visits;
    if (n_status > (size_t)INT32_MAX) return FG_ERR_BAD_SHAPE;
    FG_CUDA(cudaMemsetAsync(workspace, 0, need, st));
    k_oc_rows<<<(unsigned)n_status, kThreads, 0, st>>>(a);
    return launched(st);
}
