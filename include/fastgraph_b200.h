/*
 * fastgraph_b200.h -- C ABI of the B200-native bin-partitioned exact kNN.
 *
 * The drop-in boundary.  Every entry point takes plain device pointers and
 * sizes, enqueues its kernels on the given CUDA stream (`stream` is a
 * cudaStream_t / CUstream passed as void*; NULL = legacy default stream),
 * never synchronises the host and never allocates: outputs and scratch are
 * caller-owned (the Python layer uses torch's caching allocator).  Every
 * function returns 0 on success, a negative FG_ERR_* for a bad argument
 * (checked before any launch, nothing enqueued), or a positive cudaError_t
 * from the launch.  fg_error_string() describes a code.
 *
 * Each entry point names the reference interface it replaces; paths are
 * relative to /root/reference/pkg/src/gridknn ("pyx" = _kernels/_binned_cy.pyx).
 * The reference's backend protocol (pyx NAME/build_index/ring_cells/
 * binned_knn/brute_knn, selected by _kernels/__init__.py:23-38) is host numpy;
 * paper_2511_10442_b200/backend.py adapts it onto this ABI, and
 * paper_2511_10442_b200/ops.py registers the torch ops (fastgraph::*) on it.
 *
 * Conventions
 *  - coordinates are float32, row-major (n, n_coords), 1 <= n_coords <= 16;
 *  - row_splits are int64 offsets (n_splits + 1), starting at 0, non-decreasing,
 *    ending at n (G/core.py:49-98); empty splits are legal;
 *  - neighbour indices are int32 original vertex ids, n < 2^31 (G/knn.py:51);
 *  - distances are squared Euclidean over ALL n_coords dims (pyx:32-48).
 *  - parity contract: rows are sorted by (float64 d2 computed exactly as the
 *    reference does, original index) -- lower index wins ties; slot 0 is the
 *    vertex itself with d2 0; unfilled slots are (-1, 0).
 */
#ifndef FASTGRAPH_B200_H
#define FASTGRAPH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FG_ABI_VERSION 3

enum fg_status {
    FG_OK = 0,
    FG_ERR_BAD_K = -1,          /* k < 1 or too large (G/knn.py:48-50 BadKError)       */
    FG_ERR_BAD_SHAPE = -2,      /* bad sizes / dims (G/errors.py BadShapeError)         */
    FG_ERR_TOO_FEW_DIMS = -3,   /* d_bin outside [1,5] or > n_coords (TooFewDimsError) */
    FG_ERR_WORKSPACE = -4,      /* workspace smaller than fg_*_workspace_size()         */
    FG_ERR_NULL = -5,           /* required pointer is NULL                             */
    FG_ERR_TOO_MANY_DIMS = -6,  /* n_coords > 16                                        */
    FG_ERR_BAD_RADIUS = -7,     /* max_radius2 < 0 (G/knn.py:57-58 BadKError)          */
    FG_ERR_BAD_CAPACITY = -8,   /* n_maxuq / n_maxrs < 1 (G/ocgraph.py:176-179)         */
    FG_ERR_UNSUPPORTED = -9     /* sizes outside the requested mode's limits            */
};

/* Option bits for fg_knn_fwd (mirror KnnOptions, G/knn.py:34-45, and the
 * exhaustive_rings flag of binned_select_knn, G/knn.py:82-84). */
#define FG_KNN_USE_DIRECTION 0x1 /* dir_mask is read: roles 0/2 skip the query, 1/2 hide the
                                    candidate (pyx:210-211, 265-266; G/core.py:181-184)      */
#define FG_KNN_USE_MAX_R2 0x2    /* drop candidates with d2 > max_radius2 (boundary kept)  */
#define FG_KNN_EXHAUSTIVE 0x4    /* no early stop and no pruning (diagnostic, same result) */
#define FG_KNN_D2_F64 0x8        /* out_d2 is double (bit-exact reference float64 d2);
                                    otherwise float (= float32 of the reference d2)         */
#define FG_KNN_STATS 0x100       /* diagnostics: count search events (fg_knn_stats)        */
#define FG_KNN_NO_TILE 0x200     /* diagnostics: skip the lane-per-query tile path         */
#define FG_KNN_FUSED_EPI 0x800   /* diagnostics: tile epilogue inside the scan kernel      */
#define FG_KNN_NO_HD 0x1000      /* diagnostics: skip the high-dimensional tile path       */
#define FG_KNN_FORCE_HD 0x2000   /* diagnostics: high-dimensional tile path for any shape  */

/* Reducer codes for the GravNet aggregation (G/gravnet.py:26, order = blocks). */
#define FG_REDUCE_MEAN 0
#define FG_REDUCE_MAX 1

/* ---------------------------------------------------------------- binning */

/* Scratch bytes needed by fg_bin_by_coordinates for these sizes. */
int fg_bin_workspace_size(int64_t n, int32_t n_splits, int32_t d_bin, int32_t n_bins,
                          size_t *bytes);

/* bin_by_coordinates.  Replaces build_bin_index -> kb.build_index
 * (G/binning.py:136-170 -> pyx:66-139) and yields bit-identical arrays:
 *   bin_idx[n]        int64  global cell s*n_bins^d_bin + row-major flat cell
 *   sort_order[n]     int32  vertices cell by cell, ascending id within a cell
 *                            (the reference's stable counting sort)
 *   bin_bounds[S*n_bins^d_bin + 1] int32  sort_order range of every cell
 *   dim_mins[S*d_bin], widths[S*d_bin] float64 (empty split: 0 / 1.0)
 * plus the B200 layout the search reads:
 *   sorted_coords[n * coord_stride] float32, coords gathered in sort_order,
 *   zero padded to coord_stride = 4*ceil(n_coords/4) (16-byte vectors).
 * n_bins is the caller's (host) choice; the reference rule lives in the host
 * layer (G/binning.py:40-62,159-162). */
int fg_bin_by_coordinates(const float *coords, int64_t n, int32_t n_coords,
                          const int64_t *row_splits, int32_t n_splits, int32_t d_bin,
                          int32_t n_bins, int64_t *bin_idx, int32_t *sort_order,
                          int32_t *bin_bounds, double *dim_mins, double *widths,
                          float *sorted_coords, void *workspace, size_t workspace_bytes,
                          void *stream);

/* bin_by_coordinates on float64 coordinates (the reference's own dtype,
 * G/core.py:129): bounding boxes and cells from the float64 values, so every
 * array equals the reference's bit for bit for any finite input;
 * sorted_coords holds the float32 rounding (the search's filter stream). */
int fg_bin_by_coordinates_f64(const double *coords, int64_t n, int32_t n_coords,
                              const int64_t *row_splits, int32_t n_splits, int32_t d_bin,
                              int32_t n_bins, int64_t *bin_idx, int32_t *sort_order,
                              int32_t *bin_bounds, double *dim_mins, double *widths,
                              float *sorted_coords, void *workspace, size_t workspace_bytes,
                              void *stream);

/* index_replacer: io[i] = lut[io[i]] for io[i] >= 0, negatives kept.  The
 * reference does this implicitly (u = sort_order[p], pyx:262); fg_knn_fwd
 * already emits original ids, this is the standalone op. */
int fg_index_replacer(int32_t *io, int64_t n, const int32_t *lut, int64_t lut_n, void *stream);

/* ---------------------------------------------------------------- search */

/* binned_select_knn forward.  Replaces binned_select_knn -> kb.binned_knn
 * (G/knn.py:82-115 -> pyx:303-329, _search_one pyx:188-300).  Reads the
 * arrays of fg_bin_by_coordinates; writes out_idx[n*k] (int32) and
 * out_d2[n*k] (float or double, FG_KNN_D2_F64) at the ORIGINAL row of each
 * vertex.  dir_mask (int8, original order) is read only with
 * FG_KNN_USE_DIRECTION.  k counts the vertex itself (1 <= k <= 960). */
int fg_knn_fwd(const float *sorted_coords, const int32_t *sort_order, const int64_t *bin_idx,
               const int32_t *bin_bounds, const int64_t *row_splits, const double *dim_mins,
               const double *widths, int64_t n, int32_t n_coords, int32_t n_splits,
               int32_t d_bin, int32_t n_bins, int32_t k, const int8_t *dir_mask,
               double max_radius2, uint32_t flags, int32_t *out_idx, void *out_d2,
               void *stream);

/* Scratch bytes fg_knn_fwd_ws needs for this call (0 when only the
 * warp-per-query kernel runs: d_bin < n_coords, d > 4, k > 41, masks, ...). */
int fg_knn_workspace_size(int64_t n, int32_t n_coords, int32_t n_splits, int32_t d_bin,
                          int32_t n_bins, int32_t k, uint32_t flags, size_t *bytes);

/* fg_knn_fwd with caller-owned scratch (no allocation at all).  Same result:
 * the lane-per-query tile path certifies most rows, the warp-per-query kernel
 * finishes the rest on the same stream. */
int fg_knn_fwd_ws(const float *sorted_coords, const int32_t *sort_order, const int64_t *bin_idx,
                  const int32_t *bin_bounds, const int64_t *row_splits, const double *dim_mins,
                  const double *widths, int64_t n, int32_t n_coords, int32_t n_splits,
                  int32_t d_bin, int32_t n_bins, int32_t k, const int8_t *dir_mask,
                  double max_radius2, uint32_t flags, int32_t *out_idx, void *out_d2,
                  void *workspace, size_t workspace_bytes, void *stream);

/* binned_select_knn forward on float64 coordinates (the reference's dtype):
 * exact float64 keys from `coords` (n x n_coords, original order) in the
 * reference's operation order, so indices AND float64 distances equal the
 * reference's for any finite input; the float32 `sorted_coords` of
 * fg_bin_by_coordinates_f64 drive a filter whose error bound is derived from
 * max |coords| on the device.  Runs the lane-per-query tile kernel for every
 * shape; k <= 120 and n_bins <= 32 (FG_ERR_UNSUPPORTED otherwise).  Same flags,
 * outputs and canonical order as fg_knn_fwd_ws; FG_KNN_EXHAUSTIVE is accepted
 * and changes nothing (same answer). */
int fg_knn_f64_workspace_size(int64_t n, int32_t n_coords, int32_t n_splits, int32_t d_bin,
                              int32_t n_bins, int32_t k, uint32_t flags, size_t *bytes);
int fg_knn_fwd_f64_ws(const double *coords, const float *sorted_coords, const int32_t *sort_order,
                      const int64_t *bin_idx, const int32_t *bin_bounds,
                      const int64_t *row_splits, const double *dim_mins, const double *widths,
                      int64_t n, int32_t n_coords, int32_t n_splits, int32_t d_bin,
                      int32_t n_bins, int32_t k, const int8_t *dir_mask, double max_radius2,
                      uint32_t flags, int32_t *out_idx, void *out_d2, void *workspace,
                      size_t workspace_bytes, void *stream);

/* Diagnostics: copy (and optionally reset) the counters accumulated by
 * fg_knn_fwd launches made with FG_KNN_STATS: warp-per-query kernel [queries,
 * regions, chunks, appends, compactions, speculative-radius failures, exact
 * epilogues, rows], then the tile path [tiles, candidates, redo rows, failed tiles].
 * Synchronous; not for the hot path. */
int fg_knn_stats(uint64_t *out, int32_t n, int32_t reset);

/* Brute-force exact kNN (replaces brute_knn / _brute_one, _binned_cy.pyx:335-409;
 * G/knn.py:118-132) -- the independent GPU verifier: it shares
 * no code with the binned search.  Every vertex of the query's row split is a
 * candidate; distances in float64 in the reference's order (pyx:32-48); rows in
 * the canonical (d2, index) order: slot 0 = self, then the k-1 nearest other
 * vertices, (-1, 0.0) padding; FG_KNN_USE_DIRECTION / FG_KNN_USE_MAX_R2 as in
 * fg_knn_fwd.  `queries` (nullable): rows to compute (out rows follow it),
 * NULL = all n.  k <= 128. */
int fg_brute_knn(const float *coords, int64_t n, int32_t n_coords, const int64_t *row_splits,
                 int32_t n_splits, const int32_t *queries, int64_t n_queries,
                 const int8_t *dir_mask, double max_radius2, uint32_t flags, int32_t k,
                 int32_t *out_idx, double *out_d2, void *stream);
/* fg_brute_knn on float64 coordinates (the reference's dtype): same rows. */
int fg_brute_knn_f64(const double *coords, int64_t n, int32_t n_coords, const int64_t *row_splits,
                     int32_t n_splits, const int32_t *queries, int64_t n_queries,
                     const int8_t *dir_mask, double max_radius2, uint32_t flags, int32_t k,
                     int32_t *out_idx, double *out_d2, void *stream);

/* ---------------------------------------------------------------- backward */

int fg_knn_bwd_workspace_size(int64_t n, int32_t n_coords, int32_t k, size_t *bytes);

/* binned_select_knn backward.  Replaces knn_backward (G/knn.py:135-168):
 * for every valid non-self slot (v,s) -> u with upstream g = grad_d2[v,s],
 * grad[v] += 2g(x_v - x_u) and grad[u] -= 2g(x_v - x_u).  Terms are formed
 * exactly in float64 (fp32 g and x).  Two accumulation paths:
 *  - default: compensated fp32x4 atomics (hi + exact TwoSum error), ~2^-48 of
 *    the term magnitudes, fastest, not bitwise repeatable;
 *  - FG_BWD_DETERMINISTIC (up to 2^23 vertices and 2^32 slots): the slots are
 *    transposed into 512-position destination buckets (counting sorts, no
 *    floating-point atomics) and every destination sums its terms as int64
 *    fixed point (order-independent), ~2^-42 of the bucket's largest term:
 *    bitwise repeatable run to run like the reference's fixed-order np.add.at
 *    (pkg/tests/test_knn.py:302-309).
 * coords and grad_d2 are float32, or double with FG_BWD_X64 / FG_BWD_G64
 * (the reference's dtypes: terms 2g(x_v - x_u) in float64 exactly as numpy
 * forms them; default path only).  grad_coords is float32 (or double with
 * FG_BWD_F64).  `order` (nullable) is the row visiting order, e.g. the
 * sort_order of fg_bin_by_coordinates (spatial locality).
 * Workspace from fg_knn_bwd_workspace_size(n, n_coords, k). */
#define FG_BWD_F64 0x1
#define FG_BWD_DETERMINISTIC 0x2
#define FG_BWD_X64 0x4 /* coords is double */
#define FG_BWD_G64 0x8 /* grad_d2 is double */
int fg_knn_bwd(const void *coords, int64_t n, int32_t n_coords, const int32_t *idx, int32_t k,
               const void *grad_d2, const int32_t *order, void *grad_coords, int32_t grad_flags,
               void *workspace, size_t workspace_bytes, void *stream);

/* ---------------------------------------------------------------- GravNet */

/* gravnet_aggregate.  Replaces G/gravnet.py:64-97: per vertex, weights
 * w = exp(-scale*d2) over valid slots (idx >= 0, slot 0 only with
 * include_self), reducers applied in order (FG_REDUCE_*), one F-wide block
 * each: out[n, F*n_reducers] float32.  Arithmetic in float64.  `order`
 * (optional, may be NULL) is a permutation of the rows to visit them in --
 * the bin index's sort_order makes neighbouring warps share feature rows. */
int fg_gravnet_fwd(const float *feats, int64_t n, int32_t n_feats, const int32_t *idx,
                   const float *d2, int32_t k, double weight_scale, const int32_t *reducers,
                   int32_t n_reducers, int32_t include_self, const int32_t *order, float *out,
                   void *stream);

int fg_gravnet_bwd_workspace_size(int64_t n, int32_t n_feats, int32_t k, size_t *bytes);

/* Fused search + GravNet aggregation (the fusion the paper
 * describes): binned_select_knn (float32 distances, no mask /
 * radius) then gravnet_aggregate of its rows in sorted order, one call on one
 * stream.  Outputs are those of fg_knn_fwd_ws + fg_gravnet_fwd (scratch:
 * fg_knn_workspace_size with the same flags).  (An in-epilogue fusion was
 * slower on B200 and removed: DESIGN.md 5.) */
int fg_knn_gravnet_fwd_ws(const float *sorted_coords, const int32_t *sort_order,
                          const int64_t *bin_idx, const int32_t *bin_bounds,
                          const int64_t *row_splits, const double *dim_mins, const double *widths,
                          int64_t n, int32_t n_coords, int32_t n_splits, int32_t d_bin,
                          int32_t n_bins, int32_t k, uint32_t flags, const float *feats,
                          int32_t n_feats, double weight_scale, const int32_t *reducers,
                          int32_t n_reducers, int32_t include_self, int32_t *out_idx,
                          float *out_d2, float *agg_out, void *workspace, size_t workspace_bytes,
                          void *stream);

/* gravnet_aggregate_backward.  Replaces G/gravnet.py:100-150 ->
 * (grad_feats[n,F] float32, grad_d2[n,k] float32); max blocks route to the
 * lowest arg-max slot.  grad_d2 comes from a row pass, grad_feats from a pass
 * over each vertex's reverse-neighbour list (built in the workspace) plus the
 * max blocks' terms scattered to their arg-max neighbour; float64 inside.
 * n*k < 2^31. */
int fg_gravnet_bwd(const float *feats, int64_t n, int32_t n_feats, const int32_t *idx,
                   const float *d2, int32_t k, double weight_scale, const int32_t *reducers,
                   int32_t n_reducers, int32_t include_self, const int32_t *order,
                   const float *upstream, float *grad_feats, float *grad_d2, void *workspace,
                   size_t workspace_bytes, void *stream);

/* ---------------------------------------------------------------- association matrices */

/* Scratch for fg_oc_find_unique over n vertices (hash table + flags + scan). */
int fg_oc_unique_workspace_size(int64_t n, size_t *bytes);

/* find_unique + max_same_count.  Replaces G/ocgraph.py:114-149: objects are
 * the distinct non-negative ids per row split, in first-occurrence order.
 * asso int64[n] (negative = background), row_splits int64[n_splits+1] (device).
 * Writes unique_idx / unique_rs / counts (int64, capacity n; counts may be
 * NULL) and summary int64[2] = {n_unique, largest member count} on the device. */
int fg_oc_find_unique(const int64_t *asso, int64_t n, const int64_t *row_splits, int32_t n_splits,
                      int64_t *unique_idx, int64_t *unique_rs, int64_t *counts, int64_t *summary,
                      void *workspace, size_t workspace_bytes, void *stream);

/* Scratch for fg_oc_matrices (per-object chunk counts). */
int fg_oc_matrices_workspace_size(int64_t n_unique, int64_t max_window, size_t *bytes);

/* oc_helper.  Replaces G/ocgraph.py:152-202 (the paper's Algorithm 3): for
 * object i (unique_idx[i] in split unique_rs[i]) the window is the first
 * n_maxrs vertices of its split; m[i] (int64[n_unique, n_maxuq]) gets the
 * window's members ascending, truncated; m_not[i] (int64[n_unique, n_maxrs],
 * NULL = calc_m_not False) the rest of the window ascending; -1 suffixes.
 * visits (int64, device) = sum of window lengths.  max_window >= the largest
 * row split size (sizes the grid).  Errors: FG_ERR_BAD_CAPACITY. */
int fg_oc_matrices(const int64_t *asso, const int64_t *row_splits, int32_t n_splits,
                   const int64_t *unique_idx, const int64_t *unique_rs, int64_t n_unique,
                   int64_t n_maxuq, int64_t n_maxrs, int64_t max_window, int64_t *m, int64_t *m_not,
                   int64_t *visits, void *workspace, size_t workspace_bytes, void *stream);

/* ---------------------------------------------------------------- misc */

const char *fg_error_string(int code);
int fg_abi_version(void);
/* Kernels this library has launched since load (evidence for bench.py). */
uint64_t fg_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* FASTGRAPH_B200_H */
