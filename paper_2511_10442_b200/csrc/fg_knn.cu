// fg_knn.cu -- binned_select_knn forward for sm_100a (replaces pyx:188-329).
//
// One warp per query, queries visited in sorted (cell-major) order so the
// warps resident on an SM read overlapping candidate rows from L1/L2.
//
// Per query (query q at sorted position p, original id qid, cell c):
//   shell R = 0, 1, 2, ...: the in-grid rows of the Chebyshev cube of radius R
//   around c (a row = fixed leading d_bin-1 cells; along the last binned dim a
//   row of cells is ONE contiguous span of sorted points).  Lane r owns row r:
//   it prunes the row by the lead-dim box distance against the running bound
//   tau and trims the last-dim span to the cells the tau-ball can reach.  The
//   warp flattens the surviving spans (warp scan + shuffle search) so all 32
//   lanes evaluate one candidate each per step.
//   fp32 filter:  d2 = sum (q_i - x_i)^2 in fp32; a candidate enters the warp's
//   shared-memory buffer when d2 <= tau (self, hidden roles and max_radius2
//   applied here).  When the buffer fills, a 15-bit radix select finds an
//   upper bound T of the (k-1)-th smallest fp32 d2 and tau = T*(1+1e-5):
//   everything provably outside the final answer is dropped.
//   certificate: after shell R stop once the distance from q to the outside
//   of the scanned cube (computed per query from its own position, float64)
//   squared exceeds tau -- nothing unscanned can reach the answer.  This is
//   the reference's (w_min*r)^2 > maxd2 test (pyx:288-296) made per query.
//   exact epilogue: every buffered candidate gets its float64 d2 recomputed in
//   the reference's operation order (pyx:32-48, no FMA) and the buffer is
//   sorted by (d2_f64, original index); slots 1..k-1 take the first k-1
//   (lower index wins exact ties), slot 0 = self, padding (-1, 0).  Because
//   fp32 d2 is within ~1e-6 relative of the float64 value and every filter
//   keeps a 1e-5 relative margin, the result equals the float64 canonical
//   answer bit for bit, ties included.
#include <cfloat>

#include "fg_common.cuh"

namespace fg {
namespace search {

constexpr int kWarpsPerBlock = 4;
constexpr float kMargin = 1.0f + 1e-5f;
constexpr float kTiny = 1e-35f;

struct KnnArgs {
    const float4* sc;  // sorted coords, NV float4 per point
    const int32_t* sid;
    const int64_t* bin_idx;
    const int32_t* bounds;
    const int64_t* rs;
    const double* mins;
    const double* widths;
    int64_t n;
    int64_t total;
    int n_c, n_splits, d_bin, nb, k;
    const int8_t* dir;
    double max_r2;
    uint32_t flags;
    int32_t* out_idx;
    void* out_d2;
};

template <int CAP>
struct WarpBuf {
    float d[CAP];                 // fp32 d2 of buffered candidates
    int32_t p[CAP];               // their sorted positions
    unsigned long long key[CAP];  // exact epilogue: float64 d2 bits
    int32_t id[CAP];              // original ids
    int32_t cp[CAP];              // sorted positions (payload)
};

__device__ __forceinline__ void store_d2(const KnnArgs& a, int64_t off, double v) {
    if (a.flags & FG_KNN_D2_F64)
        reinterpret_cast<double*>(a.out_d2)[off] = v;
    else
        reinterpret_cast<float*>(a.out_d2)[off] = (float)v;
}

template <int NV>
__device__ __forceinline__ float fp32_d2(const float (&q)[4 * NV], const float4* c) {
    float acc = 0.0f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const float4 x = c[j];
        float t;
        t = q[4 * j + 0] - x.x; acc = fmaf(t, t, acc);
        t = q[4 * j + 1] - x.y; acc = fmaf(t, t, acc);
        t = q[4 * j + 2] - x.z; acc = fmaf(t, t, acc);
        t = q[4 * j + 3] - x.w; acc = fmaf(t, t, acc);
    }
    return acc;
}

template <int NV>
__device__ __forceinline__ double exact_pos_d2(const KnnArgs& a, const float (&q)[4 * NV],
                                               int32_t cpos) {
    float c[4 * NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const float4 x = a.sc[(int64_t)cpos * NV + j];
        c[4 * j] = x.x; c[4 * j + 1] = x.y; c[4 * j + 2] = x.z; c[4 * j + 3] = x.w;
    }
    return exact_d2<4 * NV>(q, c, a.n_c);
}

// Bitonic sort of buf.(key,id,cp)[0..len) by (key, id); len is a power of 2.
template <int CAP>
__device__ void warp_sort_exact(WarpBuf<CAP>& b, int len) {
    const int lane = lane_id();
    for (int size = 2; size <= len; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = lane; i < (len >> 1); i += 32) {
                const int x = 2 * stride * (i / stride) + (i % stride), y = x + stride;
                const bool up = (x & size) == 0;
                const unsigned long long kx = b.key[x], ky = b.key[y];
                const int32_t ix = b.id[x], iy = b.id[y];
                const bool gt = kx > ky || (kx == ky && ix > iy);
                if (gt == up) {
                    b.key[x] = ky; b.key[y] = kx;
                    b.id[x] = iy; b.id[y] = ix;
                    const int32_t t = b.cp[x]; b.cp[x] = b.cp[y]; b.cp[y] = t;
                }
            }
            __syncwarp();
        }
    }
}

// Exact keys for buffer entries [0, m); entries beyond max_radius2 get the
// sentinel key; then sort the first pow2 >= max(m, 32) entries.
template <int NV, int CAP>
__device__ int exact_keys_and_sort(const KnnArgs& a, WarpBuf<CAP>& b, int m,
                                   const float (&q)[4 * NV]) {
    const int lane = lane_id();
    int len = 32;
    while (len < m) len <<= 1;
    const bool use_r2 = a.flags & FG_KNN_USE_MAX_R2;
    for (int e = lane; e < len; e += 32) {
        if (e < m) {
            const int32_t cpos = b.p[e];
            const double d = exact_pos_d2<NV>(a, q, cpos);
            const bool ok = !use_r2 || d <= a.max_r2;
            b.key[e] = ok ? (unsigned long long)__double_as_longlong(d) : ~0ull;
            b.id[e] = ok ? a.sid[cpos] : 0x7fffffff;
            b.cp[e] = cpos;
        } else {
            b.key[e] = ~0ull;
            b.id[e] = 0x7fffffff;
            b.cp[e] = -1;
        }
    }
    __syncwarp();
    warp_sort_exact<CAP>(b, len);
    return len;
}

// Shrink the buffer.  Approximate: radix-select an upper bound of the need-th
// smallest fp32 d2 on its top 16 bits, keep everything within the margin.
// Exact (when that frees too little, e.g. massive ties): sort by exact key and
// keep exactly `need` entries.  Returns the new count, updates tau.
template <int NV, int CAP>
__device__ int compact(const KnnArgs& a, WarpBuf<CAP>& b, int m, int need, float& tau,
                       const float (&q)[4 * NV]) {
    const int lane = lane_id();
    constexpr int PER = CAP / 32;
    unsigned pref[PER];
    float dv[PER];
    int32_t pv[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = i * 32 + lane;
        dv[i] = e < m ? b.d[e] : __int_as_float(0x7f800000);
        pv[i] = e < m ? b.p[e] : 0;
        pref[i] = __float_as_uint(dv[i]) >> 16;
    }
    unsigned P = 0;
    for (int bit = 14; bit >= 0; --bit) {
        const unsigned t = P | ((1u << bit) - 1u);
        int c = 0;
#pragma unroll
        for (int i = 0; i < PER; ++i) c += pref[i] <= t ? 1 : 0;
        c = __reduce_add_sync(FG_FULL_MASK, c);
        if (c < need) P |= 1u << bit;
    }
    const float T = __uint_as_float((P << 16) | 0xffffu);
    const float nt = fminf(tau, T * kMargin + kTiny);
    __syncwarp();
    int w = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const bool keep = (i * 32 + lane) < m && dv[i] <= nt;
        const unsigned bal = __ballot_sync(FG_FULL_MASK, keep);
        if (keep) {
            const int pos = w + __popc(bal & lanemask_lt());
            b.d[pos] = dv[i];
            b.p[pos] = pv[i];
        }
        w += __popc(bal);
    }
    tau = nt;
    __syncwarp();
    if (w <= CAP - 32) return w;
    // exact compaction
    exact_keys_and_sort<NV, CAP>(a, b, w, q);
    // entries are sorted, so the valid ones form a prefix
    int kept = 0;
    float mx = 0.0f;
    for (int base = 0; base < need; base += 32) {
        const int e = base + lane;
        const unsigned long long key = e < need ? b.key[e] : ~0ull;
        const bool ok = key != ~0ull;
        if (ok) {
            const float df = __double2float_ru(__longlong_as_double((long long)key));
            b.d[e] = df;
            b.p[e] = b.cp[e];
            mx = fmaxf(mx, df);
        }
        kept += __popc(__ballot_sync(FG_FULL_MASK, ok));
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(FG_FULL_MASK, mx, o));
    if (kept >= need) tau = fminf(tau, mx * kMargin + kTiny);
    __syncwarp();
    return kept;
}

template <int NV, int CAP>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) k_knn_fwd(KnnArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpBuf<CAP>& buf = reinterpret_cast<WarpBuf<CAP>*>(smem_raw)[threadIdx.x >> 5];
    const int lane = lane_id();
    const int64_t warp_global = blockIdx.x * (int64_t)kWarpsPerBlock + (threadIdx.x >> 5);
    const int64_t warps_total = (int64_t)gridDim.x * kWarpsPerBlock;
    const int k = a.k, need = k - 1;
    const bool use_dir = a.flags & FG_KNN_USE_DIRECTION;
    const bool use_r2 = a.flags & FG_KNN_USE_MAX_R2;
    const bool exhaustive = a.flags & FG_KNN_EXHAUSTIVE;
    const int nb = a.nb, nl = a.d_bin - 1;
    const float r2_hi = use_r2 ? (float)(a.max_r2 * (1.0 + 1e-5)) + kTiny : 0.0f;
    const float r2_lo = use_r2 ? (float)(a.max_r2 * (1.0 - 1e-5)) : 0.0f;

    for (int64_t p = warp_global; p < a.n; p += warps_total) {
        const int32_t qid = a.sid[p];
        const int64_t row_out = (int64_t)qid * k;
        if (lane == 0) {
            a.out_idx[row_out] = qid;
            store_d2(a, row_out, 0.0);
        }
        const bool skip = need == 0 || (use_dir && (a.dir[qid] == 0 || a.dir[qid] == 2));
        if (skip) {
            for (int s = 1 + lane; s < k; s += 32) {
                a.out_idx[row_out + s] = -1;
                store_d2(a, row_out + s, 0.0);
            }
            continue;
        }
        float q[4 * NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const float4 x = a.sc[p * NV + j];
            q[4 * j] = x.x; q[4 * j + 1] = x.y; q[4 * j + 2] = x.z; q[4 * j + 3] = x.w;
        }
        // query cell and its split's grid
        const int64_t g = a.bin_idx[qid];
        const int64_t s = g / a.total;
        int64_t flat = g - s * a.total;
        int c[5];
        double mn[5], wd[5], qd[5], slack[5];
#pragma unroll
        for (int i = 4; i >= 0; --i) {
            if (i < a.d_bin) {
                c[i] = (int)(flat % nb);
                flat /= nb;
                mn[i] = a.mins[s * a.d_bin + i];
                wd[i] = a.widths[s * a.d_bin + i];
                qd[i] = (double)q[i];
                slack[i] = 1e-12 * (fabs(mn[i]) + fabs(qd[i]) + wd[i] * nb);
            } else {
                c[i] = 0; mn[i] = 0.0; wd[i] = 1.0; qd[i] = 0.0; slack[i] = 0.0;
            }
        }
        const int64_t cell_base = s * a.total;
        const int cl = c[nl];

        float tau = __int_as_float(0x7f800000);
        int m = 0;
        for (int R = 0;; ++R) {
            // clipped lead box of the cube
            int lo_d[4], len_d[4];
            int64_t rows = 1;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if (i < nl) {
                    const int lo = max(c[i] - R, 0), hi = min(c[i] + R, nb - 1);
                    lo_d[i] = lo;
                    len_d[i] = hi - lo + 1;
                    rows *= len_d[i];
                } else {
                    lo_d[i] = 0;
                    len_d[i] = 1;
                }
            }
            bool any_in_grid = false;
#pragma unroll
            for (int i = 0; i < 5; ++i)
                if (i < a.d_bin && (c[i] - R >= 0 || c[i] + R <= nb - 1)) any_in_grid = true;
            if (!any_in_grid) break;

            for (int64_t rb = 0; rb < rows; rb += 32) {
                const int64_t r = rb + lane;
                int32_t p0 = 0, n0 = 0, p1 = 0, n1 = 0;
                if (r < rows) {
                    int64_t rr = r;
                    int maxabs = 0;
                    int64_t rowflat = 0;
                    double bd2 = 0.0;
                    int jd[4];
#pragma unroll
                    for (int i = 3; i >= 0; --i) {
                        if (i < nl) {
                            jd[i] = lo_d[i] + (int)(rr % len_d[i]);
                            rr /= len_d[i];
                        } else {
                            jd[i] = 0;
                        }
                    }
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        if (i < nl) {
                            rowflat = rowflat * nb + jd[i];
                            maxabs = max(maxabs, abs(jd[i] - c[i]));
                            const double lo_e = mn[i] + jd[i] * wd[i];
                            const double hi_e = lo_e + wd[i];
                            double gap = fmax(fmax(lo_e - qd[i], qd[i] - hi_e), 0.0);
                            gap = fmax(gap - slack[i], 0.0);
                            bd2 += gap * gap;
                        }
                    }
                    // candidate cells along the last binned dim
                    int a0, b0, a1 = 1, b1 = 0;
                    if (maxabs == R) {
                        a0 = max(cl - R, 0);
                        b0 = min(cl + R, nb - 1);
                    } else {
                        a0 = cl - R; b0 = cl - R;   // may be out of grid
                        a1 = cl + R; b1 = cl + R;
                        if (a0 < 0) { a0 = 1; b0 = 0; }
                        if (a1 > nb - 1) { a1 = 1; b1 = 0; }
                    }
                    const bool prune = !exhaustive && tau < __int_as_float(0x7f800000);
                    if (prune) {
                        const double td = (double)tau;
                        if (bd2 > td) {
                            a0 = 1; b0 = 0; a1 = 1; b1 = 0;
                        } else {
                            const double rad = sqrt(td - bd2) * (1.0 + 1e-6) + slack[nl];
                            const double wa = floor((qd[nl] - rad - mn[nl]) / wd[nl]);
                            const double wb = floor((qd[nl] + rad - mn[nl]) / wd[nl]);
                            const int ia = (int)fmax(wa, -1.0), ib = (int)fmin(wb, (double)nb);
                            a0 = max(a0, ia); b0 = min(b0, ib);
                            a1 = max(a1, ia); b1 = min(b1, ib);
                        }
                    }
                    const int64_t rowcell = cell_base + rowflat * nb;
                    if (a0 <= b0) {
                        p0 = a.bounds[rowcell + a0];
                        n0 = a.bounds[rowcell + b0 + 1] - p0;
                    }
                    if (a1 <= b1) {
                        p1 = a.bounds[rowcell + a1];
                        n1 = a.bounds[rowcell + b1 + 1] - p1;
                    }
                }
                const int32_t mine = n0 + n1;
                const int32_t incl = warp_inclusive_scan(mine);
                const int32_t excl = incl - mine;
                const int32_t T = __shfl_sync(FG_FULL_MASK, incl, 31);
                for (int32_t j0 = 0; j0 < T; j0 += 32) {
                    const int32_t f = j0 + lane;
                    // owner lane: largest o with excl[o] <= f
                    int o = 0;
#pragma unroll
                    for (int step = 16; step > 0; step >>= 1) {
                        const int t = o + step;
                        const int32_t et = __shfl_sync(FG_FULL_MASK, excl, t);
                        if (et <= f) o = t;
                    }
                    const int32_t eo = __shfl_sync(FG_FULL_MASK, excl, o);
                    const int32_t po0 = __shfl_sync(FG_FULL_MASK, p0, o);
                    const int32_t no0 = __shfl_sync(FG_FULL_MASK, n0, o);
                    const int32_t po1 = __shfl_sync(FG_FULL_MASK, p1, o);
                    const int32_t loc = f - eo;
                    const int32_t cpos = loc < no0 ? po0 + loc : po1 + (loc - no0);
                    bool pass = false;
                    float d2 = 0.0f;
                    if (f < T) {
                        d2 = fp32_d2<NV>(q, a.sc + (int64_t)cpos * NV);
                        pass = d2 <= tau && cpos != (int32_t)p;
                        if (pass && use_dir) {
                            const int8_t role = a.dir[a.sid[cpos]];
                            pass = role == 0 || role == 3;
                        }
                        if (pass && use_r2) {
                            if (d2 > r2_hi)
                                pass = false;
                            else if (d2 >= r2_lo)
                                pass = exact_pos_d2<NV>(a, q, cpos) <= a.max_r2;
                        }
                    }
                    unsigned bal = __ballot_sync(FG_FULL_MASK, pass);
                    if (bal) {
                        if (m + __popc(bal) > CAP) {
                            m = compact<NV, CAP>(a, buf, m, need, tau, q);
                            pass = pass && d2 <= tau;
                            bal = __ballot_sync(FG_FULL_MASK, pass);
                        }
                        if (pass) {
                            const int pos = m + __popc(bal & lanemask_lt());
                            buf.d[pos] = d2;
                            buf.p[pos] = cpos;
                        }
                        m += __popc(bal);
                        __syncwarp();
                    }
                }
            }
            if (exhaustive) continue;
            // certificate
            double bmin = 1e300;
#pragma unroll
            for (int i = 0; i < 5; ++i) {
                if (i < a.d_bin) {
                    if (c[i] - R >= 1) bmin = fmin(bmin, qd[i] - (mn[i] + (c[i] - R) * wd[i]) - slack[i]);
                    if (c[i] + R <= nb - 2)
                        bmin = fmin(bmin, (mn[i] + (c[i] + R + 1) * wd[i]) - qd[i] - slack[i]);
                }
            }
            if (bmin >= 1e300) break;  // the cube covers the whole grid
            if (m >= need) {
                if (!(tau < __int_as_float(0x7f800000))) m = compact<NV, CAP>(a, buf, m, need, tau, q);
                if (bmin > 0.0 && bmin * bmin > (double)tau) break;
            } else if (use_r2) {
                if (bmin > 0.0 && bmin * bmin > a.max_r2 * (1.0 + 1e-5)) break;
            }
        }
        // exact epilogue
        exact_keys_and_sort<NV, CAP>(a, buf, m, q);
        for (int sl = 1 + lane; sl < k; sl += 32) {
            const int e = sl - 1;
            const unsigned long long key = e < m ? buf.key[e] : ~0ull;
            if (key != ~0ull) {
                a.out_idx[row_out + sl] = buf.id[e];
                store_d2(a, row_out + sl, __longlong_as_double((long long)key));
            } else {
                a.out_idx[row_out + sl] = -1;
                store_d2(a, row_out + sl, 0.0);
            }
        }
        __syncwarp();
    }
}

template <int NV, int CAP>
int launch_knn(const KnnArgs& a, cudaStream_t st) {
    const size_t smem = sizeof(WarpBuf<CAP>) * kWarpsPerBlock;
    auto kern = k_knn_fwd<NV, CAP>;
    if (smem > 48 * 1024) FG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t blocks = std::min<int64_t>(ceil_div(a.n, kWarpsPerBlock), (int64_t)1 << 30);
    kern<<<(unsigned)blocks, kWarpsPerBlock * 32, smem, st>>>(a);
    return launched(st);
}

template <int NV>
int dispatch_cap(const KnnArgs& a, cudaStream_t st) {
    const int need = a.k - 1;
    if (need + 64 <= 128) return launch_knn<NV, 128>(a, st);
    if (need + 64 <= 256) return launch_knn<NV, 256>(a, st);
    if (need + 64 <= 512) return launch_knn<NV, 512>(a, st);
    return launch_knn<NV, 1024>(a, st);
}

}  // namespace search
}  // namespace fg

using namespace fg;
using namespace fg::search;

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
    a.total = 1;
    for (int i = 0; i < d_bin; ++i) a.total *= n_bins;
    a.n_c = n_coords;
    a.n_splits = n_splits;
    a.d_bin = d_bin;
    a.nb = n_bins;
    a.k = k;
    a.dir = dir_mask;
    a.max_r2 = max_radius2;
    a.flags = flags;
    a.out_idx = out_idx;
    a.out_d2 = out_d2;
    cudaStream_t st = (cudaStream_t)stream;
    switch ((n_coords + 3) / 4) {
        case 1: return dispatch_cap<1>(a, st);
        case 2: return dispatch_cap<2>(a, st);
        case 3: return dispatch_cap<3>(a, st);
        default: return dispatch_cap<4>(a, st);
    }
}
