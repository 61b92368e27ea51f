// fg_scan.cuh -- single-pass decoupled-look-back exclusive scan (CUB-free),
// shared by the binning (histogram -> bin_bounds) and the GravNet backward
// (reverse-neighbour counts -> offsets).
#pragma once
#include "fg_common.cuh"

namespace fg {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;
// shared-memory slot of tile item i: one pad word per 32 items, so the
// thread-contiguous reads (thread t, items 16t..16t+15) hit 32 distinct banks
// (unpadded they were 16-way conflicts) and the strided copies stay conflict-free
__device__ __forceinline__ int scan_slot(int i) { return i + (i >> 5); }

// Exclusive scan of hist[0..m) into out[0..m] (out[m] = grand total) and,
// when cursor is not null, a copy into cursor[0..m). Status word: bits 62-63 flag (0 invalid, 1 tile
// aggregate, 2 inclusive prefix), low 32 bits the value.
static __global__ void __launch_bounds__(kScanThreads) k_scan(const int32_t* __restrict__ hist, int64_t m,
                                                       int32_t* __restrict__ out,
                                                       int32_t* __restrict__ cursor,
                                                       unsigned long long* __restrict__ status,
                                                       unsigned* __restrict__ ticket) {
    __shared__ int32_t s_items[kScanTile + kScanTile / 32];
    __shared__ int32_t s_warp[kScanThreads / 32];
    __shared__ int32_t s_prefix;
    __shared__ unsigned s_tile;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t base = tile * kScanTile;
    for (int i = threadIdx.x; i < kScanTile; i += kScanThreads) {
        const int64_t g = base + i;
        s_items[scan_slot(i)] = g < m ? hist[g] : 0;
    }
    __syncthreads();
    int32_t local[kScanItems];
    int32_t run = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        local[j] = run;  // exclusive within the thread
        run += s_items[scan_slot(threadIdx.x * kScanItems + j)];
    }
    const int lane = lane_id(), w = threadIdx.x >> 5;
    const int32_t incl = warp_inclusive_scan(run);
    if (lane == 31) s_warp[w] = incl;
    __syncthreads();
    if (w == 0) {
        int32_t x = lane < kScanThreads / 32 ? s_warp[lane] : 0;
        x = warp_inclusive_scan(x);
        if (lane < kScanThreads / 32) s_warp[lane] = x;
    }
    __syncthreads();
    const int32_t thread_excl = (incl - run) + (w > 0 ? s_warp[w - 1] : 0);
    const int32_t tile_total = s_warp[kScanThreads / 32 - 1];
    // decoupled look-back (warp 0)
    if (w == 0) {
        int32_t prefix = 0;
        if (tile == 0) {
            if (lane == 0) {
                __threadfence();
                atomicExch(&status[0], (2ull << 62) | (unsigned)tile_total);
            }
        } else {
            if (lane == 0) {
                __threadfence();
                atomicExch(&status[tile], (1ull << 62) | (unsigned)tile_total);
            }
            int64_t end = tile - 1;  // closest predecessor examined by lane 0
            while (true) {
                const int64_t idx = end - lane;
                unsigned long long word = 2ull << 62;  // before tile 0: prefix 0
                if (idx >= 0) {
                    do {
                        word = *((volatile unsigned long long*)&status[idx]);
                    } while ((word >> 62) == 0);
                }
                const unsigned flag = (unsigned)(word >> 62);
                const int32_t val = idx >= 0 ? (int32_t)(word & 0xffffffffu) : 0;
                const unsigned pmask = __ballot_sync(FG_FULL_MASK, flag == 2);
                if (pmask) {
                    const int first = __ffs(pmask) - 1;
                    int32_t x = lane <= first ? val : 0;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FG_FULL_MASK, x, o);
                    prefix += x;
                    break;
                }
                int32_t x = val;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FG_FULL_MASK, x, o);
                prefix += x;
                end -= 32;
            }
            if (lane == 0) {
                __threadfence();
                atomicExch(&status[tile], (2ull << 62) | (unsigned)(prefix + tile_total));
            }
        }
        if (lane == 0) s_prefix = prefix;
    }
    __syncthreads();
    const int32_t pre = s_prefix + thread_excl;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) s_items[scan_slot(threadIdx.x * kScanItems + j)] = pre + local[j];
    __syncthreads();
    for (int i = threadIdx.x; i < kScanTile; i += kScanThreads) {
        const int64_t g = base + i;
        if (g < m) {
            const int32_t x = s_items[scan_slot(i)];
            out[g] = x;
            if (cursor) cursor[g] = x;
        }
    }
    if (base + kScanTile >= m && threadIdx.x == 0) out[m] = s_prefix + tile_total;
}

}  // namespace fg
