// fg_verify.cu -- brute-force exact kNN on the GPU (replaces brute_knn /
// _brute_one, _binned_cy.pyx:335-409; G/knn.py:118-132), written to share NO
// code with the binned search (fg_knn*.cu/cuh, fg_common.cuh): it is the
// independent GPU verifier of SURVEY 8(f)2, fast enough to check every row of
// the BASELINE configs (tests/test_gpu_verify.py).
//
// Deliberately simple: thread per query, the candidates of the block's splits
// streamed through shared memory in float64 tiles (every thread reads each
// candidate by broadcast), the reference's distance (float64 of the float32
// coordinates, sequential sum over ALL coordinates, no FMA: pyx:32-48), and a
// per-thread sorted list of the k-1 best (d2, index) pairs -- the canonical
// order: lower index wins exact ties.  Candidates arrive in ascending index, so
// a candidate tied with the current k-th never enters, and an insertion goes
// after every equal key.  Rows: slot 0 = the vertex itself (d2 0), then the
// k-1 nearest other vertices of its row split, (-1, 0.0) padding; DirectionMask
// roles and max_radius2 as pyx:351-372.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "../../include/fastgraph_b200.h"

namespace fg {
extern std::atomic<uint64_t> g_launches;
}

namespace {

constexpr int kThreads = 256;       // queries per block
constexpr int kTileDoubles = 4096;  // staged candidate coordinates (32 KB)
constexpr int kMaxK = 128;

template <int NC, typename TC>
__global__ void __launch_bounds__(kThreads) k_brute(const TC* __restrict__ coords, int n_c,
                                                    const int64_t* __restrict__ rs, int n_splits,
                                                    const int32_t* __restrict__ queries, int64_t n_q,
                                                    const int8_t* __restrict__ dir, double max_r2,
                                                    int use_r2, int k, int32_t* __restrict__ out_idx,
                                                    double* __restrict__ out_d2) {
    constexpr int T = kTileDoubles / NC;  // candidates per tile
    __shared__ double s_c[kTileDoubles];
    __shared__ int8_t s_ok[T];  // candidate role allows it (DirectionMask)
    __shared__ unsigned long long s_lo, s_hi;
    const int64_t qi = blockIdx.x * (int64_t)kThreads + threadIdx.x;
    const bool live = qi < n_q;
    const int64_t v = live ? (queries ? (int64_t)queries[qi] : qi) : 0;
    // split of v: the last s with rs[s] <= v (empty splits are skipped)
    int a = 0, b = n_splits;
    while (a < b) {
        const int m = (a + b + 1) >> 1;
        if (rs[m] <= v) a = m; else b = m - 1;
    }
    const int64_t lo = rs[a], hi = rs[a + 1];
    if (threadIdx.x == 0) {
        s_lo = ~0ull;
        s_hi = 0ull;
    }
    __syncthreads();
    if (live) {
        atomicMin(&s_lo, (unsigned long long)lo);
        atomicMax(&s_hi, (unsigned long long)hi);
    }
    const bool query = live && !(dir && (dir[v] == 0 || dir[v] == 2));
    double q[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) q[i] = (live && i < n_c) ? (double)coords[v * n_c + i] : 0.0;
    double key[kMaxK];
    int32_t id[kMaxK];
    const int need = k - 1;
    int filled = 0;
    double kth = 0.0;
    __syncthreads();
    const int64_t c_lo = (int64_t)s_lo, c_hi = (int64_t)s_hi;
    for (int64_t t0 = c_lo; t0 < c_hi; t0 += T) {
        const int64_t cnt = c_hi - t0 < T ? c_hi - t0 : T;
        __syncthreads();
        for (int64_t e = threadIdx.x; e < cnt * n_c; e += kThreads) {
            const int64_t j = e / n_c;
            s_c[j * NC + (e - j * n_c)] = (double)coords[t0 * n_c + e];
        }
        for (int64_t j = threadIdx.x; j < cnt; j += kThreads)
            s_ok[j] = !(dir && (dir[t0 + j] == 1 || dir[t0 + j] == 2));
        __syncthreads();
        if (!query) continue;
        const int64_t j0 = lo - t0 > 0 ? lo - t0 : 0, j1 = hi - t0 < cnt ? hi - t0 : cnt;
        for (int64_t j = j0; j < j1; ++j) {
            const int64_t u = t0 + j;
            if (u == v || !s_ok[j]) continue;
            double d2 = 0.0;
#pragma unroll
            for (int i = 0; i < NC; ++i) {
                if (i < n_c) {
                    const double t = __dsub_rn(q[i], s_c[j * NC + i]);
                    const double sq = __dmul_rn(t, t);
                    d2 = i == 0 ? sq : __dadd_rn(d2, sq);
                }
            }
            if (use_r2 && d2 > max_r2) continue;
            if (filled == need && !(d2 < kth)) continue;
            // insert after every key <= d2 (their indices are smaller)
            int p = filled < need ? filled++ : need - 1;
            while (p > 0 && key[p - 1] > d2) {
                key[p] = key[p - 1];
                id[p] = id[p - 1];
                --p;
            }
            key[p] = d2;
            id[p] = (int32_t)u;
            if (filled == need) kth = key[need - 1];
        }
    }
    if (!live) return;
    int32_t* oi = out_idx + qi * k;
    double* od = out_d2 + qi * k;
    oi[0] = (int32_t)v;
    od[0] = 0.0;
    for (int s = 1; s < k; ++s) {
        const bool f = query && s - 1 < filled;
        oi[s] = f ? id[s - 1] : -1;
        od[s] = f ? key[s - 1] : 0.0;
    }
}

}  // namespace

namespace {
template <typename TC>
int brute_entry(const TC* coords, int64_t n, int32_t n_coords, const int64_t* row_splits,
                int32_t n_splits, const int32_t* queries, int64_t n_queries, const int8_t* dir_mask,
                double max_radius2, uint32_t flags, int32_t k, int32_t* out_idx, double* out_d2,
                void* stream) {
    if (k < 1 || k > kMaxK) return FG_ERR_BAD_K;
    if (n < 0 || n >= ((int64_t)1 << 31) || n_splits < 1 || n_queries < 0) return FG_ERR_BAD_SHAPE;
    if (n_coords < 1) return FG_ERR_BAD_SHAPE;
    if (n_coords > 16) return FG_ERR_TOO_MANY_DIMS;
    if ((flags & FG_KNN_USE_MAX_R2) && !(max_radius2 >= 0.0)) return FG_ERR_BAD_RADIUS;
    const int64_t nq = queries ? n_queries : n;
    if (nq == 0) return 0;
    if (!coords || !row_splits || !out_idx || !out_d2) return FG_ERR_NULL;
    if ((flags & FG_KNN_USE_DIRECTION) && !dir_mask) return FG_ERR_NULL;
    const int8_t* dir = (flags & FG_KNN_USE_DIRECTION) ? dir_mask : nullptr;
    const int use_r2 = (flags & FG_KNN_USE_MAX_R2) ? 1 : 0;
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned blocks = (unsigned)((nq + kThreads - 1) / kThreads);
    switch ((n_coords + 3) / 4) {
        case 1: k_brute<4, TC><<<blocks, kThreads, 0, st>>>(coords, n_coords, row_splits, n_splits, queries, nq, dir, max_radius2, use_r2, k, out_idx, out_d2); break;
        case 2: k_brute<8, TC><<<blocks, kThreads, 0, st>>>(coords, n_coords, row_splits, n_splits, queries, nq, dir, max_radius2, use_r2, k, out_idx, out_d2); break;
        case 3: k_brute<12, TC><<<blocks, kThreads, 0, st>>>(coords, n_coords, row_splits, n_splits, queries, nq, dir, max_radius2, use_r2, k, out_idx, out_d2); break;
        default: k_brute<16, TC><<<blocks, kThreads, 0, st>>>(coords, n_coords, row_splits, n_splits, queries, nq, dir, max_radius2, use_r2, k, out_idx, out_d2); break;
    }
    fg::g_launches.fetch_add(1, std::memory_order_relaxed);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : (int)e;
}
}  // namespace

extern "C" int fg_brute_knn(const float* coords, int64_t n, int32_t n_coords, const int64_t* row_splits,
                            int32_t n_splits, const int32_t* queries, int64_t n_queries,
                            const int8_t* dir_mask, double max_radius2, uint32_t flags, int32_t k,
                            int32_t* out_idx, double* out_d2, void* stream) {
    return brute_entry<float>(coords, n, n_coords, row_splits, n_splits, queries, n_queries,
                              dir_mask, max_radius2, flags, k, out_idx, out_d2, stream);
}

extern "C" int fg_brute_knn_f64(const double* coords, int64_t n, int32_t n_coords,
                                const int64_t* row_splits, int32_t n_splits, const int32_t* queries,
                                int64_t n_queries, const int8_t* dir_mask, double max_radius2,
                                uint32_t flags, int32_t k, int32_t* out_idx, double* out_d2,
                                void* stream) {
    return brute_entry<double>(coords, n, n_coords, row_splits, n_splits, queries, n_queries,
                               dir_mask, max_radius2, flags, k, out_idx, out_d2, stream);
}
