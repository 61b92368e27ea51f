// fg_gravnet.cu -- GravNet distance-weighted aggregation (replaces
// G/gravnet.py:64-150) for sm_100a.
//
// Semantics (G/gravnet.py): slot s of row v contributes when idx[v,s] >= 0 (and
// s > 0 unless include_self) with weight w = exp(-scale * d2[v,s]); reducers
// are applied in order, one F-wide block each: mean = sum / count over valid
// slots, max over valid slots (the backward routes it to the lowest arg-max
// slot, np.argmax), zeros for a row without valid slots.  Weights, products,
// sums and maxima are float64, outputs float32.
//
// Forward: warp per row (rows visited in `order` when given -- spatially sorted
// rows reuse each other's neighbour feature rows through L1/L2), lanes over
// features (FJ per lane), one pass over the slots.
// Backward, no floating-point atomics:
//   rows    warp per row v: valid count, per-feature arg-max slot (1 byte) and
//           grad_d2[v,s] = -scale * w_s * sum_f f[u_s,f] * coef[v,f,s];
//   reverse counting sort of the (v,s) pairs by neighbour u (int atomics +
//           the decoupled-look-back scan) -> for every u the list of (v,s)
//           that aggregated it;
//   columns warp per u gathers grad_feats[u,f] = sum over its list of
//           w_vs * (up_mean[v,f]/cnt_v + [argmax[v,f] == s] up_max[v,f])
//           in float64.
#include "fg_common.cuh"
#include "fg_scan.cuh"

namespace fg {
namespace gravnet {

constexpr int kRowWarps = 8;

struct GnArgs {
    const float* feats;
    int64_t n;
    int F;
    const int32_t* idx;
    const float* d2;
    int k;
    double scale;
    unsigned max_bits;  // bit b set: reducer block b is max (else mean)
    int n_red;
    int include_self;
    const int32_t* order;
};

__device__ __forceinline__ int64_t row_of(const GnArgs& g, int64_t p) {
    return g.order ? (int64_t)g.order[p] : p;
}

__device__ __forceinline__ bool is_max(const GnArgs& g, int b) { return (g.max_bits >> b) & 1u; }

__device__ __forceinline__ bool slot_valid(const GnArgs& g, int s, int32_t u) {
    return u >= 0 && (g.include_self || s > 0);
}

// ---------------------------------------------------------------- forward
template <int FJ>
__global__ void __launch_bounds__(kRowWarps * 32) k_gn_fwd(const GnArgs g, int f0, float* __restrict__ out) {
    const int lane = lane_id();
    const int64_t p = blockIdx.x * (int64_t)kRowWarps + (threadIdx.x >> 5);
    if (p >= g.n) return;
    const int64_t v = row_of(g, p);
    const int k = g.k, F = g.F, W = F * g.n_red;
    double sum[FJ], mx[FJ];
#pragma unroll
    for (int j = 0; j < FJ; ++j) {
        sum[j] = 0.0;
        mx[j] = -INFINITY;
    }
    int cnt = 0;
    for (int base = 0; base < k; base += 32) {
        const int s = base + lane;
        const int32_t u = s < k ? g.idx[v * k + s] : -1;
        const bool ok = s < k && slot_valid(g, s, u);
        const double w = ok ? exp(-g.scale * (double)g.d2[v * k + s]) : 0.0;
        unsigned okm = __ballot_sync(FG_FULL_MASK, ok);
        cnt += __popc(okm);
        while (okm) {
            const int j0 = __ffs(okm) - 1;
            okm &= okm - 1;
            const int32_t uj = __shfl_sync(FG_FULL_MASK, u, j0);
            const double wj = __shfl_sync(FG_FULL_MASK, w, j0);
#pragma unroll
            for (int j = 0; j < FJ; ++j) {
                const int f = f0 + lane + 32 * j;
                if (f < F) {
                    const double term = wj * (double)g.feats[(int64_t)uj * F + f];
                    sum[j] += term;
                    if (term > mx[j]) mx[j] = term;
                }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < FJ; ++j) {
        const int f = f0 + lane + 32 * j;
        if (f >= F) continue;
        for (int b = 0; b < g.n_red; ++b) {
            double val = 0.0;
            if (cnt > 0) val = is_max(g, b) ? mx[j] : sum[j] / (double)cnt;
            out[v * W + (int64_t)b * F + f] = (float)val;
        }
    }
}

// ---------------------------------------------------------------- backward
struct GnBwd {
    const float* up;      // (n, F * n_red)
    int32_t* cnt;         // (n) valid slots per row
    void* amax;           // (n, F) arg-max slot of the max blocks (AM, all-ones: none)
    float* grad_d2;       // (n, k)
    double* gd_acc;       // (n, k) float64 partials when F spans several chunks, else null
    int32_t* rev_cnt;     // (n) reverse-neighbour counts (scan input)
    int32_t* rev_off;     // (n + 1)
    int32_t* rev_cur;     // (n) fill cursor
    int32_t* rev;         // (n * k) entries v * k + s
    float* grad_feats;    // (n, F)
};

// Row pass: valid count, arg-max slots, grad_d2; counts reverse neighbours.
template <int FJ, typename AM>
__global__ void __launch_bounds__(kRowWarps * 32) k_gn_rows(const GnArgs g, const GnBwd bw, int f0,
                                                          int last_chunk) {
    const int lane = lane_id();
    const int64_t p = blockIdx.x * (int64_t)kRowWarps + (threadIdx.x >> 5);
    if (p >= g.n) return;
    const int64_t v = row_of(g, p);
    const int k = g.k, F = g.F, W = F * g.n_red;
    const bool has_max = g.max_bits != 0;
    // pass 1: count + arg-max (lowest slot on ties, np.argmax)
    int cnt = 0;
    double best[FJ];
    int bslot[FJ];
#pragma unroll
    for (int j = 0; j < FJ; ++j) {
        best[j] = -INFINITY;
        bslot[j] = -1;
    }
    for (int base = 0; base < k; base += 32) {
        const int s = base + lane;
        const int32_t u = s < k ? g.idx[v * k + s] : -1;
        const bool ok = s < k && slot_valid(g, s, u);
        if (ok && f0 == 0) atomicAdd(&bw.rev_cnt[u], 1);
        unsigned okm = __ballot_sync(FG_FULL_MASK, ok);
        cnt += __popc(okm);
        if (!has_max) continue;
        const double w = ok ? exp(-g.scale * (double)g.d2[v * k + s]) : 0.0;
        while (okm) {
            const int j0 = __ffs(okm) - 1;
            okm &= okm - 1;
            const int32_t uj = __shfl_sync(FG_FULL_MASK, u, j0);
            const double wj = __shfl_sync(FG_FULL_MASK, w, j0);
#pragma unroll
            for (int j = 0; j < FJ; ++j) {
                const int f = f0 + lane + 32 * j;
                if (f < F) {
                    const double term = wj * (double)g.feats[(int64_t)uj * F + f];
                    if (term > best[j]) {
                        best[j] = term;
                        bslot[j] = base + j0;
                    }
                }
            }
        }
    }
    if (lane == 0 && f0 == 0) bw.cnt[v] = cnt;
    // per-feature coefficients: mean blocks up/cnt, max blocks up at the arg-max
    double cmean[FJ], cmax[FJ];
#pragma unroll
    for (int j = 0; j < FJ; ++j) {
        cmean[j] = 0.0;
        cmax[j] = 0.0;
        const int f = f0 + lane + 32 * j;
        if (f >= F) continue;
        if (has_max) ((AM*)bw.amax)[v * F + f] = (AM)(cnt > 0 ? bslot[j] : -1);
        if (cnt == 0) continue;
        for (int b = 0; b < g.n_red; ++b) {
            const double ub = (double)bw.up[v * W + (int64_t)b * F + f];
            if (is_max(g, b))
                cmax[j] += ub;
            else
                cmean[j] += ub / (double)cnt;
        }
    }
    // pass 2: grad_d2[v,s] = -scale w_s sum_f f[u_s,f] (cmean_f + [amax_f == s] cmax_f)
    for (int base = 0; base < k; base += 32) {
        const int s = base + lane;
        const int32_t u = s < k ? g.idx[v * k + s] : -1;
        const bool ok = s < k && slot_valid(g, s, u) && cnt > 0;
        const unsigned okm = __ballot_sync(FG_FULL_MASK, ok);
        double mine = 0.0;  // this lane's slot total
        const int lim = min(32, k - base);
        for (int j0 = 0; j0 < lim; ++j0) {
            if (!((okm >> j0) & 1u)) continue;  // warp-uniform
            const int32_t uj = __shfl_sync(FG_FULL_MASK, u, j0);
            double part = 0.0;
#pragma unroll
            for (int j = 0; j < FJ; ++j) {
                const int f = f0 + lane + 32 * j;
                if (f < F) {
                    const double c = cmean[j] + (bslot[j] == base + j0 ? cmax[j] : 0.0);
                    part += (double)g.feats[(int64_t)uj * F + f] * c;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(FG_FULL_MASK, part, o);
            if (lane == j0) mine = part;
        }
        if (s < k) {
            const double w = ok ? exp(-g.scale * (double)g.d2[v * k + s]) : 0.0;
            double val = ok ? -g.scale * w * mine : 0.0;
            if (bw.gd_acc) {
                if (f0 > 0) val += bw.gd_acc[v * k + s];
                if (!last_chunk) bw.gd_acc[v * k + s] = val;
            }
            if (last_chunk) bw.grad_d2[v * k + s] = (float)val;
        }
    }
}

// Reverse fill: entry v*k + s goes to neighbour u's list.
__global__ void k_gn_fill(const GnArgs g, const GnBwd bw) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= g.n * g.k) return;
    const int64_t v = t / g.k;
    const int s = (int)(t - v * g.k);
    const int32_t u = g.idx[t];
    if (!slot_valid(g, s, u)) return;
    bw.rev[atomicAdd(&bw.rev_cur[u], 1)] = (int32_t)t;
}

// Column pass: grad_feats[u] from u's reverse list, float64.  The sum over the
// list is order-independent up to float64 rounding (the list order comes from
// the atomic fill), far inside the float32 output precision.
template <int FJ, typename AM>
__global__ void __launch_bounds__(kRowWarps * 32) k_gn_cols(const GnArgs g, const GnBwd bw, int f0) {
    const int lane = lane_id();
    const int64_t p = blockIdx.x * (int64_t)kRowWarps + (threadIdx.x >> 5);
    if (p >= g.n) return;
    const int64_t u = row_of(g, p);
    const int k = g.k, F = g.F, W = F * g.n_red;
    const int32_t lo = bw.rev_off[u], hi = bw.rev_off[u + 1];
    const AM* amax = (const AM*)bw.amax;
    double acc[FJ];
#pragma unroll
    for (int j = 0; j < FJ; ++j) acc[j] = 0.0;
    for (int32_t base = lo; base < hi; base += 32) {
        const int32_t e = base + lane;
        int32_t vv = 0, ss = 0;
        double w = 0.0, ic = 0.0;
        if (e < hi) {
            const int32_t t = bw.rev[e];
            vv = t / k;
            ss = t - vv * k;
            w = exp(-g.scale * (double)g.d2[t]);
            ic = 1.0 / (double)bw.cnt[vv];
        }
        const int nb = min(32, hi - base);
        for (int j0 = 0; j0 < nb; ++j0) {
            const int64_t v = __shfl_sync(FG_FULL_MASK, vv, j0);
            const int s = __shfl_sync(FG_FULL_MASK, ss, j0);
            const double wj = __shfl_sync(FG_FULL_MASK, w, j0);
            const double icj = __shfl_sync(FG_FULL_MASK, ic, j0);
#pragma unroll
            for (int j = 0; j < FJ; ++j) {
                const int f = f0 + lane + 32 * j;
                if (f >= F) continue;
                const bool at_max = amax && (int)amax[v * F + f] == s;
                double c = 0.0;
                for (int b = 0; b < g.n_red; ++b) {
                    const double ub = (double)bw.up[v * W + (int64_t)b * F + f];
                    if (!is_max(g, b))
                        c += ub * icj;
                    else if (at_max)
                        c += ub;
                }
                acc[j] += wj * c;
            }
        }
    }
#pragma unroll
    for (int j = 0; j < FJ; ++j) {
        const int f = f0 + lane + 32 * j;
        if (f < F) bw.grad_feats[u * F + f] = (float)acc[j];
    }
}

int check_reducers(const int32_t* reducers, int32_t n_red, GnArgs& g) {
    if (!reducers) return FG_ERR_NULL;
    if (n_red < 1 || n_red > 4) return FG_ERR_BAD_SHAPE;
    g.max_bits = 0;
    for (int i = 0; i < n_red; ++i) {
        if (reducers[i] != FG_REDUCE_MEAN && reducers[i] != FG_REDUCE_MAX) return FG_ERR_BAD_SHAPE;
        if (reducers[i] == FG_REDUCE_MAX) g.max_bits |= 1u << i;
    }
    g.n_red = n_red;
    return 0;
}

constexpr int kFChunk = 256;  // features per launch (FJ <= 8)

template <typename Launch>
int per_chunk(int F, Launch&& launch) {
    for (int f0 = 0; f0 < F; f0 += kFChunk) {
        const int left = F - f0;
        const int last = f0 + kFChunk >= F;
        int rc;
        if (left <= 32)
            rc = launch(std::integral_constant<int, 1>{}, f0, last);
        else if (left <= 64)
            rc = launch(std::integral_constant<int, 2>{}, f0, last);
        else if (left <= 128)
            rc = launch(std::integral_constant<int, 4>{}, f0, last);
        else
            rc = launch(std::integral_constant<int, 8>{}, f0, last);
        if (rc) return rc;
    }
    return 0;
}

struct BwdWs {
    int32_t* cnt;
    void* amax;
    double* gd_acc;
    int32_t* rev_cnt;
    int32_t* rev_off;
    int32_t* rev_cur;
    int32_t* rev;
    unsigned long long* status;
    unsigned* ticket;
    int64_t n_tiles;
};

inline size_t amax_bytes(int k) { return k <= 255 ? 1 : 2; }

size_t carve(BwdWs* w, void* base, int64_t n, int F, int k) {
    size_t off = 0;
    char* b = (char*)base;
    auto take = [&](size_t bytes) {
        off = align_up(off, 256);
        char* p = b ? b + off : nullptr;
        off += bytes;
        return p;
    };
    w->n_tiles = ceil_div(n, kScanTile);
    w->cnt = (int32_t*)take(sizeof(int32_t) * (size_t)n);
    w->amax = take((size_t)n * F * amax_bytes(k));
    w->gd_acc = F > kFChunk ? (double*)take(sizeof(double) * (size_t)n * k) : nullptr;
    w->rev_cnt = (int32_t*)take(sizeof(int32_t) * (size_t)n);
    w->rev_off = (int32_t*)take(sizeof(int32_t) * (size_t)(n + 1));
    w->rev_cur = (int32_t*)take(sizeof(int32_t) * (size_t)n);
    w->rev = (int32_t*)take(sizeof(int32_t) * (size_t)n * k);
    w->status = (unsigned long long*)take(sizeof(unsigned long long) * (size_t)(w->n_tiles + 1));
    w->ticket = (unsigned*)take(sizeof(unsigned) * 4);
    return align_up(off, 256);
}

template <typename AM>
int gn_backward(const GnArgs& g, const GnBwd& bw, const BwdWs& w, cudaStream_t st) {
    const unsigned blocks = (unsigned)ceil_div(g.n, kRowWarps);
    FG_TRY(per_chunk(g.F, [&](auto fj, int f0, int last) {
        k_gn_rows<decltype(fj)::value, AM><<<blocks, kRowWarps * 32, 0, st>>>(g, bw, f0, last);
        return launched(st);
    }));
    k_scan<<<(unsigned)w.n_tiles, kScanThreads, 0, st>>>(w.rev_cnt, g.n, w.rev_off, w.rev_cur, w.status,
                                                        w.ticket);
    FG_TRY(launched(st));
    k_gn_fill<<<(unsigned)ceil_div(g.n * g.k, 256), 256, 0, st>>>(g, bw);
    FG_TRY(launched(st));
    return per_chunk(g.F, [&](auto fj, int f0, int) {
        k_gn_cols<decltype(fj)::value, AM><<<blocks, kRowWarps * 32, 0, st>>>(g, bw, f0);
        return launched(st);
    });
}

}  // namespace gravnet
}  // namespace fg

using namespace fg;
using namespace fg::gravnet;

extern "C" int fg_gravnet_fwd(const float* feats, int64_t n, int32_t n_feats, const int32_t* idx,
                              const float* d2, int32_t k, double weight_scale,
                              const int32_t* reducers, int32_t n_reducers, int32_t include_self,
                              const int32_t* order, float* out, void* stream) {
    GnArgs g;
    FG_TRY(check_reducers(reducers, n_reducers, g));
    if (k < 1) return FG_ERR_BAD_K;
    if (n < 0 || n_feats < 1) return FG_ERR_BAD_SHAPE;
    if (!(weight_scale > 0.0)) return FG_ERR_BAD_SHAPE;
    if (n == 0) return 0;
    if (!feats || !idx || !d2 || !out) return FG_ERR_NULL;
    g.feats = feats; g.n = n; g.F = n_feats; g.idx = idx; g.d2 = d2; g.k = k;
    g.scale = weight_scale; g.include_self = include_self; g.order = order;
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned blocks = (unsigned)ceil_div(n, kRowWarps);
    return per_chunk(n_feats, [&](auto fj, int f0, int) {
        k_gn_fwd<decltype(fj)::value><<<blocks, kRowWarps * 32, 0, st>>>(g, f0, out);
        return launched(st);
    });
}

extern "C" int fg_gravnet_bwd_workspace_size(int64_t n, int32_t n_feats, int32_t k, size_t* bytes) {
    if (!bytes) return FG_ERR_NULL;
    if (k < 1 || k > 65535) return FG_ERR_BAD_K;
    if (n < 0 || n_feats < 1) return FG_ERR_BAD_SHAPE;
    BwdWs w;
    *bytes = carve(&w, nullptr, n, n_feats, k);
    return 0;
}

extern "C" int fg_gravnet_bwd(const float* feats, int64_t n, int32_t n_feats, const int32_t* idx,
                              const float* d2, int32_t k, double weight_scale,
                              const int32_t* reducers, int32_t n_reducers, int32_t include_self,
                              const int32_t* order, const float* upstream, float* grad_feats,
                              float* grad_d2, void* workspace, size_t workspace_bytes,
                              void* stream) {
    GnArgs g;
    FG_TRY(check_reducers(reducers, n_reducers, g));
    if (k < 1 || k > 65535) return FG_ERR_BAD_K;  // arg-max slots are stored in 1-2 bytes
    if (n < 0 || n_feats < 1) return FG_ERR_BAD_SHAPE;
    if (!(weight_scale > 0.0)) return FG_ERR_BAD_SHAPE;
    if ((int64_t)n * k >= (int64_t)INT32_MAX) return FG_ERR_BAD_SHAPE;  // 32-bit reverse entries
    if (n == 0) return 0;
    if (!feats || !idx || !d2 || !upstream || !grad_feats || !grad_d2 || !workspace) return FG_ERR_NULL;
    BwdWs w;
    const size_t need = carve(&w, workspace, n, n_feats, k);
    if (workspace_bytes < need) return FG_ERR_WORKSPACE;
    g.feats = feats; g.n = n; g.F = n_feats; g.idx = idx; g.d2 = d2; g.k = k;
    g.scale = weight_scale; g.include_self = include_self; g.order = order;
    const bool has_max = g.max_bits != 0;
    GnBwd bw;
    bw.up = upstream; bw.cnt = w.cnt; bw.amax = has_max ? w.amax : nullptr; bw.grad_d2 = grad_d2;
    bw.gd_acc = w.gd_acc; bw.rev_cnt = w.rev_cnt; bw.rev_off = w.rev_off; bw.rev_cur = w.rev_cur;
    bw.rev = w.rev; bw.grad_feats = grad_feats;
    cudaStream_t st = (cudaStream_t)stream;
    FG_CUDA(cudaMemsetAsync(w.rev_cnt, 0, sizeof(int32_t) * (size_t)n, st));
    FG_CUDA(cudaMemsetAsync(w.status, 0, sizeof(unsigned long long) * (size_t)(w.n_tiles + 1), st));
    FG_CUDA(cudaMemsetAsync(w.ticket, 0, sizeof(unsigned) * 4, st));
    return k <= 255 ? gn_backward<uint8_t>(g, bw, w, st) : gn_backward<uint16_t>(g, bw, w, st);
}
