// Search kernels for coordinates of 1..4 dims (NV = 1 float4 per point):
// the warp-per-query kernel and the lane-per-query tile path.
#include "fg_knn_tile.cuh"

namespace fg {
namespace search {
int dispatch_nv1(const KnnArgs& a, int d_bin, cudaStream_t st) { return dispatch_db<1>(a, d_bin, st); }
}  // namespace search

namespace hd {
int dispatch_hd_nv1(tile::TileArgs& t, const search::KnnArgs& a, int d_bin, cudaStream_t st);
}

namespace tile {

template <int DB>
int launch_db(TileArgs& t, const search::KnnArgs& a, cudaStream_t st, TileArgs* clustered) {
    FG_CUDA(cudaMemsetAsync(t.ctr, 0, 8 * sizeof(int), st));
    k_tiles<DB><<<(unsigned)ceil_div(t.n_blocks, 4), 128, 0, st>>>(t);
    FG_TRY(launched(st));
    // per call (not cached in a static): the current device's SM count and the
    // shared-memory opt-ins are per device, and host threads may race on a cache
    int dev = 0, sms = 0;
    FG_CUDA(cudaGetDevice(&dev));
    FG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    FG_CUDA(cudaFuncSetAttribute(k_tile_search<DB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)tile_smem_bytes<false>()));
    FG_CUDA(cudaFuncSetAttribute(k_tile_search<DB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)tile_smem_bytes<true>()));
    if (t.lists)
        k_tile_search<DB, true><<<(unsigned)(sms * kScanCtasPerSm), kWarps * 32,
                                  tile_smem_bytes<true>(), st>>>(t);
    else
        k_tile_search<DB, false><<<(unsigned)(sms * kCtasPerSm), kWarps * 32,
                                   tile_smem_bytes<false>(), st>>>(t);
    FG_TRY(launched(st));
    if (t.lists) {  // split epilogue
        k_tile_finish<DB><<<(unsigned)(sms * 8), kFinishWarps * 32, 0, st>>>(t, a.n);
        FG_TRY(launched(st));
    }
    // whatever the tiles could not certify: the warp-per-query kernel
    search::KnnArgs r = a;
    r.qlist = t.redo;
    r.qcount = &t.ctr[2];
    r.qall = &t.ctr[4];
    if (clustered) {
        // data the tile kernels declined (clustered at the cell scale): the
        // high-dimensional tile kernels with dense cells in Morton order take
        // every query instead of the warp-per-query kernel (gated on the device)
        clustered->gate = &t.ctr[4];
        FG_TRY(hd::dispatch_hd_nv1(*clustered, a, DB, st));
        r.qall = nullptr;  // declined: the redo list is empty
    }
    return search::dispatch_db<1>(r, DB, st);
}

int launch(TileArgs& t, const search::KnnArgs& a, int d_bin, cudaStream_t st, TileArgs* clustered) {
    switch (d_bin) {
        case 1: return launch_db<1>(t, a, st, clustered);
        case 2: return launch_db<2>(t, a, st, clustered);
        case 3: return launch_db<3>(t, a, st, clustered);
        default: return launch_db<4>(t, a, st, clustered);
    }
}

}  // namespace tile
}  // namespace fg
