/*
 * histobundle_b200.h -- C ABI of the B200-native bundling iteration.
 *
 * This is the drop-in boundary for the reference's operator layer: each entry
 * point replaces one numba kernel (or numpy routine) that
 * /root/reference/pkg/src/histobundle/bundler.py and raster.py call through
 * numba's native-call "FFI" (caller-allocated arrays + an edge range, kernels
 * write only their own rows, _kernels.py:1-6).  Here the arrays are device
 * pointers, the edge range is the whole shard, and every call is
 * stream-ordered on the caller's cudaStream_t (passed as void*).
 *
 * Conventions (all entry points):
 *   - return 0 on success, a negative HB_E* code on failure; the message is
 *     available from hb_last_error() (thread-local).
 *   - the library never allocates device memory; outputs and workspaces are
 *     caller-allocated (ownership as in bundler.py:112,119,145 / raster.py:86).
 *   - points are packed (N, 2) float64 grid coordinates, x then y;
 *     `starts` is (E+1) int64 with starts[0] == 0 (bundler.py:84-89).
 *   - histograms/fields are (B, V, U) row-major; counts are int32 per group,
 *     fields float32.
 *   - float64 arithmetic is bit-identical to the reference (no FMA
 *     contraction, float32 density differences, floor(x+0.5) cells).
 */
#ifndef HISTOBUNDLE_B200_H
#define HISTOBUNDLE_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define HB_API __attribute__((visibility("default")))
#else
#define HB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define HB_OK 0
#define HB_EINVAL (-1)   /* bad argument (sizes, null pointers)            */
#define HB_ECUDA (-2)    /* CUDA launch / runtime error                    */

/* status-flag bits written by device kernels (caller-owned int32) */
#define HB_STATUS_OUT_OF_BOUNDS 1 /* raster.py:57-67 "sample out of bounds" */
#define HB_STATUS_CAPACITY 4      /* a resample did not fit the output buffer */
#define HB_STATUS_INEXACT 8       /* integer fast path no longer equals float32 sums */

/* Tile-binned splatting state (all pointers caller-owned device memory).
 * The grid of every layer is cut into tile x tile cells; a segment is binned
 * to the tile holding its first cell and rasterised later into a
 * shared-memory window of (tile + 2*halo)^2 cells, so the histogram sees one
 * global atomic per touched cell per work chunk instead of one per
 * increment.  Records are 8 bytes: start cell (2 x u16), cell delta
 * (2 x s8), k0 (1 bit), integer weight (15 bits). */
typedef struct hb_tiles {
    int tile, halo;      /* cells */
    int ntx, nty;        /* tiles per row / per column of one layer */
    int nbins;           /* layers */
    int ntiles;          /* nbins * ntx * nty */
    int64_t *off;        /* (ntiles+1) bucket offsets into rec */
    int32_t *cap;        /* (ntiles) bucket capacities */
    int32_t *fill;       /* (ntiles) records claimed (demand, may exceed cap) */
    int32_t *work;       /* (ntiles+2) scratch: flush chunk prefix + counter */
    uint64_t *rec;       /* off[ntiles] records; NULL = census only */
    int64_t rec_capacity;
    /* Segment-key mode (mode == 1): segments of bundled edges are mostly
     * identical at the cell level, so instead of records every segment with
     * k0 == 1 and cell delta within +-halo adds its weight to one counter
     * keyed by (group, delta, start cell); hb_segtab_expand then rasterises
     * each non-zero key once with its multiplicity.  tab holds
     * nbins*(2*halo+1)^2*nv*nu uint32 counters, all zero between passes. */
    int mode;            /* 0 = tile records, 1 = segment-key table, 2 = census only */
    uint32_t *tab;
} hb_tiles;

HB_API int hb_abi_version(void);
HB_API const char *hb_last_error(void);
HB_API int hb_device_sm_count(void);
/* Total kernels this library has launched in the process (evidence counter). */
HB_API long long hb_launch_count(void);

/* Per-edge preparation of _sample_packed (bundler.py:77-85) on the device:
 * src/dst grid endpoints (p - origin) / cell of node_pos[sources[e]] and
 * node_pos[targets[e]] (model.py:214-216), and the point counts
 * max(ceil(|dst - src| / delta), 1) + 1 with numpy's norm
 * sqrt(dx*dx + dy*dy).  Scan counts with hb_scan_counts for `starts`. */
HB_API int hb_edge_prepare(const double *node_pos, const int64_t *sources,
                           const int64_t *targets, int64_t n_edges, double origin_x,
                           double origin_y, double cell, double delta, double *src,
                           double *dst, int64_t *counts, void *stream);

/* _materialize (bundler.py:152-163) with the endpoint pins gathered from the
 * node positions on the device. */
HB_API int hb_to_world_nodes(const double *pts, const int64_t *starts, int64_t n_edges,
                             double origin_x, double origin_y, double cell,
                             const double *node_pos, const int64_t *sources,
                             const int64_t *targets, double *out, void *stream);

/* _kernels.fill_samples (_kernels.py:22-43), called by _sample_packed
 * (bundler.py:77-89).  src/dst: (E,2) grid endpoints; starts from the host
 * count rule max(ceil(|d|/delta),1)+1; pts: (starts[E],2). */
HB_API int hb_sample_fill(const double *src, const double *dst, const int64_t *starts,
                   int64_t n_edges, double *pts, void *stream);

/* _offset_packed (bundler.py:92-106): interior points of edge e move by
 * disp[e] (per-edge (dx,dy) computed on the host with the reference's numpy
 * expression). */
HB_API int hb_offset(double *pts, const int64_t *starts, int64_t n_edges,
              const double *disp, void *stream);

/* _materialize (bundler.py:152-163): out = pts*cell + origin per point, the
 * first/last point of edge e replaced by src_world[e]/dst_world[e] (either
 * may be NULL to skip pinning). */
HB_API int hb_to_world(const double *pts, const int64_t *starts, int64_t n_edges,
                       double origin_x, double origin_y, double cell,
                       const double *src_world, const double *dst_world, double *out,
                       void *stream);

/* Tile geometry for a (nbins, nv, nu) grid whose segments span at most
 * max_seg_cells cells per axis (host only; fills tile/halo/ntx/nty/nbins/
 * ntiles, leaves the pointers alone).  Returns HB_EINVAL when binning does
 * not apply (grid wider than 65535, segments longer than 127 cells). */
HB_API int hb_tiles_geometry(int nbins, int nv, int nu, double max_seg_cells,
                             hb_tiles *t);

/* Bucket capacities for the next binned pass from the demand of the last
 * one: cap = fill + fill/4 + 64, off = exclusive prefix, fill := 0, and
 * *total (device int64) = off[ntiles], the records the pass may write. */
HB_API int hb_tiles_plan(const hb_tiles *t, int64_t *total, void *stream);

/* Rasterise every binned record into counts (int32 (B,V,U)). */
HB_API int hb_tiles_flush(const hb_tiles *t, int32_t *counts, int nv, int nu,
                          void *stream);

/* Segment-key geometry: fills halo/nbins and mode = 1; returns the number of
 * uint32 counters the caller must allocate (zeroed) in *entries. */
HB_API int hb_segtab_geometry(int nbins, int nv, int nu, double max_seg_cells,
                              hb_tiles *t, int64_t *entries);

/* Rasterise every non-zero segment key into counts and reset it to zero;
 * adds the number of non-zero keys to *nonzero (nullable). */
HB_API int hb_segtab_expand(const hb_tiles *t, int32_t *counts, int nv, int nu,
                            unsigned long long *nonzero, void *stream);

/* _kernels.accumulate (_kernels.py:46-77) via raster._accumulate_packed
 * (raster.py:70-94), per-group form: counts[group[e]] += weight[e] on every
 * rasterised cell of edge e.  weight may be NULL (all 1).  counts must be
 * zeroed by the caller.  Out-of-grid cells set HB_STATUS_OUT_OF_BOUNDS. */
HB_API int hb_splat(const double *pts, const int64_t *starts, int64_t n_edges,
             int64_t n_pts, const int32_t *group, const int32_t *weight,
             int32_t *counts, int nbins, int nv, int nu, int32_t *status,
             const hb_tiles *tiles, void *stream);
/* `tiles` (nullable): with tiles->rec == NULL the splat still adds straight
 * into counts but records each tile's demand in tiles->fill (census for the
 * next hb_tiles_plan) -- or, with mode == 2, ONLY records the demand and adds
 * nothing (a census pass before a binned splat of the same points); with
 * rec != NULL segments are binned and the caller finishes with
 * hb_tiles_flush.  hb_resample_emit takes the same argument. */

/* Workspace for hb_smooth / hb_smooth_counts: bytes of the float64 table, the
 * float32 staging plane and the fused fold's strip hand-off words. */
HB_API size_t hb_smooth_workspace_bytes(int nbins, int nv, int nu);

/* smooth_gaussian_approx (raster.py:203-219) of H = M * G, where G is the
 * per-group histogram (`counts` int32, or `hist` float32 when counts is
 * NULL): for each pass p a float64 integral image (column fold then row fold,
 * raster.py:133-139) and the 4-term box sum / (2r+1)^2 (raster.py:147-169).
 * matrix: (B,B) float32 row-major, NULL = identity; the mix is
 * H[l] = float32(sum_b M[l,b] G[b]) in float64, one rounding.
 * radii: npasses box radii (w-1)/2 from box_widths (raster.py:172-193).
 * layer_peak (B floats, nullable): max(rho_l, 0) of the final field, for
 * used_cell_count. */
HB_API int hb_smooth(const int32_t *counts, const float *hist, const float *matrix,
              int nbins, int nv, int nu, const int32_t *radii, int npasses,
              float *out, void *workspace, size_t workspace_bytes,
              float *layer_peak, void *stream);

/* hb_smooth of integer group counts whose mixed sums are exact
 * (H = scale * mix * G with an integer matrix `mix` (B,B) int32, NULL =
 * identity, and scale = 2^k).  The first pass is computed from exact
 * integer window sums -- the reference's float64 table is exact there, so
 * its box sum is the true window sum (no sequential fold needed); later
 * passes as in hb_smooth.  Also the exactness guard: HB_STATUS_INEXACT in
 * *status (nullable) when a cell has sum_b |mix[l,b]| * G[b] >= limit or a
 * negative count.  Needs radii[0] > 0 and nu <= 8192 (else use hb_smooth +
 * hb_exact_check); same workspace as hb_smooth. */
HB_API int hb_smooth_counts(const int32_t *counts, const int32_t *mix, double scale,
                            double limit, int nbins, int nv, int nu, const int32_t *radii,
                            int npasses, float *out, void *workspace, size_t workspace_bytes,
                            float *layer_peak, int32_t *status, void *stream);

/* The raw histogram H = M * G alone (raster.accumulate_edges, raster.py:108-130). */
HB_API int hb_mix_layers(const int32_t *counts, const float *hist, const float *matrix,
                         int nbins, int nv, int nu, float *out, void *stream);

/* raster.integral_image (raster.py:133-139) of B layers: table[b][v][u] =
 * T[b][v+1][u+1] (the zero first row/column is implicit). */
HB_API int hb_integral_image(const float *in, int nbins, int nv, int nu, double *table,
                             void *stream);

/* used_cell_count (bundler.py:292-305): adds to *count the number of cells
 * with rho > float32(rel * peak_l) over layers with peak_l > 0. */
HB_API int hb_used_cells(const float *rho, const float *layer_peak, int nbins, int nv,
                  int nu, double rel, unsigned long long *count, void *stream);

/* Quad advection field: B*V*U records {Q, GX, GY} of three float4 (48
 * bytes per cell, 16-byte aligned; size hb_grad_field_bytes): Q = rho at the
 * cell's 2x2 corners, GX/GY = the float32 central differences of
 * _cell_gradient (_kernels.py:101-114) at those corners.  Optional input of
 * hb_advect_points / hb_advect_laplacian (same results; three 16-byte loads
 * from one record per gradient sample and one 16-byte load per bilinear sample
 * instead of ~9 scattered ones). */
HB_API int64_t hb_grad_field_bytes(int nbins, int nv, int nu);
HB_API int hb_grad_field(const float *rho, int nbins, int nv, int nu, float *out,
                         void *stream);

/* Size (doubles) of the disp_partials buffer hb_advect_laplacian fills. */
HB_API int64_t hb_advect_partials(void);

/* _kernels.advect (_kernels.py:144-200) alone, in place: every interior
 * point of every polyline (endpoints are found from starts) moves to the
 * first step candidate m = h, h/2, ... >= min_step whose bilinear density is
 * >= its own (fixed_step: m = h, always taken).  Points are processed as one
 * flat stream (bit-identical positions to the per-edge form; see
 * hb_advect_flat.cu).  The points are [starts[0], starts[n_edges]) (so a
 * sub-range of edges is advected by offsetting starts and edge_layer);
 * n_pts bounds that range (the buffer size).  grad_field: nullable
 * hb_grad_field(rho).  Requires
 * nv, nu >= 3 and nbins*nv*nu < 2^31.  moved: u64 accumulator (added to);
 * disp_partials: hb_advect_partials() doubles (zeroed and filled here),
 * summed by hb_reduce_f64.  Follow with hb_advect_laplacian(h < 0) for the
 * Laplacian (and the fused resample count). */
HB_API int hb_advect_points(double *pts, const int64_t *starts, int64_t n_edges,
                            int64_t n_pts, const int32_t *edge_layer, const float *rho,
                            const float *grad_field, int nbins, int nv, int nu, double h,
                            double eps, double min_step, int fixed_step,
                            unsigned long long *moved, double *disp_partials, void *stream);

/* _kernels.advect (_kernels.py:144-200) -> _kernels.laplacian
 * (_kernels.py:275-296) -> _kernels.resample_count (_kernels.py:203-232) of
 * the NEXT iteration, fused in one streaming pass:
 *   pts_out = laplacian^lap_passes(advect(pts_in)),
 *   counts/pos = resample_count(pts_out, delta)   (when counts != NULL;
 *   same outputs as hb_resample_count).
 * h < 0 skips advection (Laplacian only, bundler.laplacian_smooth).
 * grad_field (nullable) is hb_grad_field(rho): same results, fewer gathers.
 * pts_out may alias pts_in.  edge_layer: (E) int32 layer of each edge (its
 * bin).  moved: u64 accumulator (added to).  disp_partials:
 * hb_advect_partials() doubles (zeroed and filled here), summed by
 * hb_reduce_f64 in fixed order. */
HB_API int hb_advect_laplacian(const double *pts_in, double *pts_out,
                        const int64_t *starts, int64_t n_edges, int64_t n_pts,
                        const int32_t *edge_layer, const float *rho,
                        const float *grad_field, int nbins,
                        int nv, int nu, double h, double eps, double min_step,
                        int fixed_step, double lap_factor, int lap_passes,
                        double delta, int64_t *counts, int32_t *pos,
                        unsigned long long *moved, double *disp_partials,
                        void *stream);

/* _kernels.laplacian (_kernels.py:275-296, lap_passes Jacobi sweeps) then
 * _kernels.resample_count (_kernels.py:203-232) on the result:
 *   pts_out = laplacian^lap_passes(pts_in)            (may alias pts_in)
 *   counts[e] = output points of polyline e, pos[j] = output index of kept
 *   point j or -1 (when counts != NULL; same outputs as hb_resample_count).
 * One lane-sequential pass (hb_lapcount.cu).  The points are [starts[0],
 * starts[n_edges]) (edge sub-ranges by offsetting starts/counts); n_pts
 * bounds that range (the buffer size) and must be < 2^31. */
HB_API int hb_laplacian_count(const double *pts_in, double *pts_out, const int64_t *starts,
                              int64_t n_edges, int64_t n_pts, double lap_factor,
                              int lap_passes, double delta, int64_t *counts, int32_t *pos,
                              void *stream);

/* Deterministic fixed-order sum of n doubles into *out (one block). */
/* hb_advect_points then hb_laplacian_count (lap_passes <= 1) in one pass:
 * each staged group of points is advected in shared memory (the flat
 * advect's arithmetic and deferral queue), then smoothed and counted; the
 * advected but unsmoothed points never go to memory.  In place.  Same
 * results as the two calls; `moved` / `disp_partials` as hb_advect_points. */
HB_API int hb_advect_laplacian_count(double *pts, const int64_t *starts, int64_t n_edges,
                                     int64_t n_pts, const int32_t *edge_layer, const float *rho,
                                     const float *grad_field, int nbins, int nv, int nu,
                                     double h, double eps, double min_step, int fixed_step,
                                     double lap_factor, int lap_passes, double delta,
                                     int64_t *counts, int32_t *pos, unsigned long long *moved,
                                     double *disp_partials, void *stream);
HB_API int hb_reduce_f64(const double *in, int64_t n, double *out, void *stream);

/* _kernels.resample_count (_kernels.py:203-232): counts[e] = output points
 * of edge e; pos[j] = local output index of kept point j, -1 if merged. */
HB_API int hb_resample_count(const double *pts, const int64_t *starts,
                      int64_t n_edges, double delta, int64_t *counts,
                      int32_t *pos, void *stream);

/* np.cumsum(counts) into new_starts[1..E], new_starts[0] = 0
 * (bundler.py:117-118). */
HB_API size_t hb_scan_workspace_bytes(int64_t n_edges);
HB_API int hb_scan_counts(const int64_t *counts, int64_t n_edges, int64_t *new_starts,
                   void *workspace, size_t workspace_bytes, void *stream);

/* _kernels.resample_emit (_kernels.py:235-272) fused with the next
 * iteration's accumulate: writes the resampled polylines into `out` at
 * new_starts and, when counts != NULL, rasterises every output segment into
 * counts (same contract as hb_splat; group may be NULL: every edge in
 * group 0).  Warps take work off one per-device
 * counter that the call zeroes on `stream` first, so emits on one device
 * must not run concurrently on different streams. */
HB_API int hb_resample_emit(const double *pts, const int64_t *starts,
                     int64_t n_edges, int64_t n_pts, const int32_t *pos,
                     const int64_t *new_starts, double *out,
                     const int32_t *group, const int32_t *weight,
                     int32_t *counts, int nv, int nu, int32_t *status,
                     const hb_tiles *tiles, void *stream);

/* hb_resample_emit for a caller that does not know the output total on the
 * host: out holds out_capacity points; if new_starts[n_edges] exceeds it the
 * kernel writes nothing and sets HB_STATUS_CAPACITY in *status. */
HB_API int hb_resample_emit_cap(const double *pts, const int64_t *starts, int64_t n_edges,
                                int64_t n_pts, const int32_t *pos, const int64_t *new_starts,
                                double *out, int64_t out_capacity, const int32_t *group,
                                const int32_t *weight, int32_t *counts, int nv, int nu,
                                int32_t *status, const hb_tiles *tiles, void *stream);

/* total_out (nullable) = starts[n_edges]; then starts[e] = min(starts[e],
 * cap) for every e when the total exceeds cap (keeps kernels that read the
 * point count from starts in bounds after an HB_STATUS_CAPACITY resample). */
HB_API int hb_clamp_starts(int64_t *starts, int64_t n_edges, int64_t cap, int64_t *total_out,
                           void *stream);

/* Per-point probes used by the single-point operator API
 * (bundler.density_at / gradient_at, bundler.py:203-217). */
HB_API int hb_probe(const float *rho_layer, int nv, int nu, const double *xy,
             int64_t n, double *value, double *grad, void *stream);

/* ---- edge binning (binning.py:81-177): best-of-restarts Lloyd K-means ----
 * features (n, d) float64 row-major, d <= 4; centroids (restarts, k, d);
 * assign (restarts, n) int8 cluster ids (k <= 64); restart lists are int32.
 * Arithmetic and order follow numpy's (einsum pairs d = 4 products as
 * (p0 + p2) + (p1 + p3); np.add.at folds in edge order; argmin / argmax take
 * the first extremum). */
/* KMeans._assign (binning.py:112-116) for the restarts in active[]: new
 * nearest centroid per edge; changed[r] |= 1 when any edge moved. */
HB_API int hb_kmeans_assign(const double *features, int64_t n, int d, int k,
                            const double *centroids, const int32_t *active, int n_active,
                            int8_t *assign, int32_t *changed, void *stream);
/* _update_centroids (binning.py:136-143) for restarts upd[]: sums in edge
 * order / counts; a cluster left empty keeps its centroid and sets empty[r]. */
HB_API int hb_kmeans_update(const double *features, int64_t n, int d, int k,
                            double *centroids, const int32_t *upd, int n_upd,
                            const int8_t *assign, int32_t *empty, void *stream);
/* The empty-cluster re-seed (binning.py:145-154) for restarts rs[]; the
 * workspace holds n_rs * n float64 distances. */
HB_API size_t hb_kmeans_reseed_workspace_bytes(int64_t n, int n_rs);
HB_API int hb_kmeans_reseed(const double *features, int64_t n, int d, int k,
                            double *centroids, const int32_t *rs, int n_rs,
                            const int8_t *assign, void *workspace, size_t workspace_bytes,
                            void *stream);
/* `iterations` Lloyd steps of every restart with the bookkeeping on the
 * device (no host round trip per step): flags = [live | changed | empty],
 * 3 * restarts int32, live = 1 and the rest 0 to start; a restart whose
 * assignment stopped changing drops out (binning.py:110-121).  The
 * workspace holds restarts * n float64 (hb_kmeans_reseed_workspace_bytes). */
HB_API int hb_kmeans_lloyd(const double *features, int64_t n, int d, int k, double *centroids,
                           int restarts, int8_t *assign, int32_t *flags, int iterations,
                           void *workspace, size_t workspace_bytes, void *stream);
/* Per-restart inertia partials (restarts x hb_kmeans_inertia_blocks()),
 * summed by the caller in order: picks the best restart (binning.py:124-130). */
HB_API int hb_kmeans_inertia_blocks(void);
HB_API int hb_kmeans_inertia(const double *features, int64_t n, int d, int k,
                             const double *centroids, int restarts, const int8_t *assign,
                             double *partial, void *stream);
/* Davies-Bouldin scatter sums and counts of one clustering (binning.py:
 * 165-171): scatter[c] = sum of norm(f_i - centroid_c) in edge order. */
HB_API int hb_kmeans_scatter(const double *features, int64_t n, int d, int k,
                             const double *centroids, const int8_t *assign, double *scatter,
                             int64_t *counts, void *stream);

/* ---- bounds, exactness guard, ordered accumulation (raster.py:57-94) ----
 * _check_bounds (raster.py:57-67): out4 = {xmin, ymin, xmax, ymax} of the
 * n_pts points; scratch32 is 32 bytes of device scratch. */
HB_API int hb_point_span(const double *pts, int64_t n_pts, void *scratch32, double *out4,
                         void *stream);
/* Guard of the integer fast path (per-group int32 counts mixed once): sets
 * HB_STATUS_INEXACT when some cell has sum_b |M[l,b]| * counts[b] >= limit
 * for a layer l (limit = 2^24 x the power-of-two quantum of every layer
 * weight: beyond it the reference's float32 sums round), or a negative
 * count.  abs_matrix: (B,B) float64 |M|, NULL = identity. */
HB_API int hb_exact_check(const int32_t *counts, const double *abs_matrix, int nbins, int nv,
                          int nu, double limit, int32_t *status, void *stream);
/* Hit offsets of _kernels.accumulate (_kernels.py:46-77) in the reference's
 * order: hoff[p] = number of cell increments of all segments before point
 * p (n_pts + 1 int64; hoff[n_pts] = the total).  Workspace:
 * hb_hits_workspace_bytes(n_pts). */
HB_API size_t hb_hits_workspace_bytes(int64_t n_pts);
HB_API int hb_hits_count(const double *pts, const int64_t *starts, int64_t n_edges,
                         int64_t n_pts, int64_t *hoff, void *workspace, size_t workspace_bytes,
                         void *stream);
/* The reference's float32 histogram (raster.py:70-94) bit for bit for any
 * layer weights: edges cut into `nparts` (= workers) partition_ranges
 * (_parallel.py:20-28, over edges_total global edges, this shard's first
 * global edge = edge_base), every cell of every partition folded in
 * (edge, segment, step) order with layer_w[e,l] = fl32(w[e]) * M[l, g[e]]
 * (bundler.py:345-346), partitions summed left to right.  w32 (NULL = 1)
 * and groups (NULL = 0) are indexed by GLOBAL edge; matrix (B,B) float32,
 * NULL = identity.  out: (B,V,U) float32.  Workspace:
 * hb_ordered_workspace_bytes(n_hits, nv, nu, nparts), n_hits = hoff[n_pts]. */
HB_API size_t hb_ordered_workspace_bytes(int64_t n_hits, int nv, int nu, int nparts);
HB_API int hb_accumulate_ordered(const double *pts, const int64_t *starts, int64_t n_edges,
                                 const int64_t *hoff, int64_t n_pts, int64_t n_hits, int nparts,
                                 int64_t edge_base, int64_t edges_total, const float *w32,
                                 const int32_t *groups, const float *matrix, int nbins, int nv,
                                 int nu, float *out, int32_t *status, void *workspace,
                                 size_t workspace_bytes, void *stream);

/* The two halves of hb_accumulate_ordered, for edge shards on several GPUs
 * (the records are exchanged by cell in between, so every cell's hits meet
 * on one rank in global order):
 * hb_hits_fill_sorted writes this shard's n_hits records (key = cell *
 * nparts + partition of the global edge, val = global edge), stably sorted
 * by key, into keys/vals; hb_ordered_fold folds records whose cells lie in
 * [cell_base, cell_base + n_cells) into out (B, n_cells) float32 -- first
 * stably sorting them by key when `sort` (rank-ordered concatenations). */
HB_API size_t hb_hits_sorted_workspace_bytes(int64_t n_hits);
HB_API int hb_hits_fill_sorted(const double *pts, const int64_t *starts, int64_t n_edges,
                               const int64_t *hoff, int64_t n_hits, int nparts,
                               int64_t edge_base, int64_t edges_total, int nv, int nu,
                               uint32_t *keys, int32_t *vals, int32_t *status, void *workspace,
                               size_t workspace_bytes, void *stream);
HB_API size_t hb_ordered_fold_workspace_bytes(int64_t n_hits, int64_t n_cells);
HB_API int hb_ordered_fold(uint32_t *keys, int32_t *vals, int64_t n_hits, int sort, int nparts,
                           int64_t cell_base, int64_t n_cells, const float *w32,
                           const int32_t *groups, const float *matrix, int nbins, float *out,
                           void *workspace, size_t workspace_bytes, void *stream);

/* ---- rendering (render.py:158-179) ----
 * Stroke width of every segment of every polyline (segments of edge e are
 * outputs starts[e]-e .. starts[e+1]-e-2): the mean of the layer's clamped
 * bilinear density at the segment's two ends over the layer peak, clipped to
 * [0, 1], mapped to w_min + (w_max - w_min) * ratio (want_ratio: the ratio
 * itself).  pts in grid coordinates; layer may be NULL (all layer 0). */
HB_API int hb_segment_widths(const double *pts, const int64_t *starts, int64_t n_edges,
                             const int32_t *layer, const float *rho, int nbins, int nv, int nu,
                             const float *peaks, double w_min, double w_max, int want_ratio,
                             double *out, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* HISTOBUNDLE_B200_H */
