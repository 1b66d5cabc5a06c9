// hb_ordered.cu -- histogram accumulation in the reference's float32
// summation order, for layer weights whose float32 sums are NOT exact
// (repulsive interaction matrices such as -alpha/(B-1), fractional edge
// weights), plus the bounds span and the exactness guard of the fast path.
//
// Reference semantics (raster.py:70-94, _kernels.py:46-77): the edges are cut
// into `workers` contiguous partitions (_parallel.py:20-28); each partition
// adds layer_w[e, l] = fl32(w_e) * M[l, b_e] (bundler.py:345-346) into a
// private zeroed float32 buffer, one hit at a time in (edge, segment, DDA
// step) order, and the buffers are summed left to right.  Per cell and layer
// that is a sequential float32 fold, so here:
//   1. hits_count : hits per point (segment) -> CUB scan -> hit offsets
//   2. hits_fill  : one (cell * P + partition, edge) record per hit, written
//                   at its position in the reference's global hit order
//   3. CUB stable radix sort by key: each cell's hits become contiguous,
//      partition-major, in reference order inside a partition
//   4. run-length encode by cell, then ordered_fold: one warp per cell, lane
//      = layer, folding the cell's hits in order (__fadd_rn on the
//      __fmul_rn layer weight) and combining partitions left to right.
// The result is the reference's float32 histogram bit for bit for the same
// `workers` value, whatever the weights.
#include <cub/cub.cuh>
#include <thrust/iterator/transform_iterator.h>

#include "hb_common.cuh"

namespace hb {

// ---- point span: _check_bounds (raster.py:57-67) ----------------------------
__device__ __forceinline__ unsigned long long ord_key(double x) {
    // order-preserving map of a double onto uint64 (min/max through atomics)
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_val(unsigned long long k) {
    const unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)b);
}

__global__ void __launch_bounds__(256)
span_kernel(const double2 *__restrict__ pts, int64_t n, unsigned long long *__restrict__ key4) {
    unsigned long long lo_x = ~0ull, lo_y = ~0ull, hi_x = 0, hi_y = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double2 p = pts[i];
        const unsigned long long kx = ord_key(p.x), ky = ord_key(p.y);
        lo_x = min(lo_x, kx); hi_x = max(hi_x, kx);
        lo_y = min(lo_y, ky); hi_y = max(hi_y, ky);
    }
    for (int d = 16; d; d >>= 1) {
        lo_x = min(lo_x, __shfl_xor_sync(0xffffffffu, lo_x, d));
        lo_y = min(lo_y, __shfl_xor_sync(0xffffffffu, lo_y, d));
        hi_x = max(hi_x, __shfl_xor_sync(0xffffffffu, hi_x, d));
        hi_y = max(hi_y, __shfl_xor_sync(0xffffffffu, hi_y, d));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(key4 + 0, lo_x);
        atomicMin(key4 + 1, lo_y);
        atomicMax(key4 + 2, hi_x);
        atomicMax(key4 + 3, hi_y);
    }
}

__global__ void span_init_kernel(unsigned long long *key4) {
    key4[0] = key4[1] = ~0ull;
    key4[2] = key4[3] = 0ull;
}
__global__ void span_final_kernel(const unsigned long long *key4, double *out4) {
    for (int k = 0; k < 4; ++k) out4[k] = ord_val(key4[k]);
}

// ---- exactness guard of the integer fast path ------------------------------
// The fast path sums integer per-group counts and mixes them once
// (hb_smooth), which equals the reference's float32 fold only while every
// partial sum is exact: |partial| <= sum_b |M[l,b]| * C[b] < limit (= 2^24
// times the common power-of-two quantum of all layer weights, computed on
// the host).  Flags HB_STATUS_INEXACT when any cell breaks it (or a count
// went negative, i.e. wrapped).
__global__ void __launch_bounds__(256)
exact_check_kernel(const int32_t *__restrict__ counts, const double *__restrict__ absm, int nb,
                   int64_t plane, double limit, int32_t *__restrict__ status) {
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < plane;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (!absm) {  // identity: every layer is its own count
            for (int b = 0; b < nb; ++b) {
                const int32_t c = counts[b * plane + i];
                bad |= c < 0 || (double)c >= limit;
            }
        } else {
            for (int l = 0; l < nb; ++l) {
                double a = 0.0;
                for (int b = 0; b < nb; ++b) {
                    const int32_t c = counts[b * plane + i];
                    bad |= c < 0;
                    a += absm[l * nb + b] * (double)c;
                }
                bad |= a >= limit;
            }
        }
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
        atomicOr(status, HB_STATUS_INEXACT);
}

// ---- ordered accumulation ---------------------------------------------------
// Hits of segment j of an edge (_kernels.py:56-77): steps + 1 - k0 cells, a
// zero-length segment only when it is the edge's first.
__device__ __forceinline__ int seg_hits(double2 a, double2 b, int j) {
    const int x0 = cell_round(a.x), y0 = cell_round(a.y);
    const int x1 = cell_round(b.x), y1 = cell_round(b.y);
    const int steps = max(abs(x1 - x0), abs(y1 - y0));
    const int k0 = j == 0 ? 0 : 1;
    return steps == 0 ? (k0 == 0 ? 1 : 0) : steps + 1 - k0;
}

// warp per edge (grid-stride); hcnt[p] = hits of the segment starting at p
// (0 for an edge's last point)
__global__ void __launch_bounds__(256)
hits_count_kernel(const double2 *__restrict__ pts, const int64_t *__restrict__ starts,
                  int64_t n_edges, int32_t *__restrict__ hcnt) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < n_edges; e += nw) {
        const int64_t s = starts[e], n = starts[e + 1] - s;
        for (int64_t j = lane; j < n; j += 32)
            hcnt[s + j] = j + 1 < n ? seg_hits(pts[s + j], pts[s + j + 1], (int)j) : 0;
    }
}

// Records of every hit at its global position hoff[p] + k.  key = cell * P +
// partition of the (global) edge; out-of-grid cells get the sentinel key
// 0xffffffff (and the status flag) and are skipped by the fold.
__global__ void __launch_bounds__(256)
hits_fill_kernel(const double2 *__restrict__ pts, const int64_t *__restrict__ starts,
                 int64_t n_edges, const int64_t *__restrict__ hoff, int nparts, int64_t edge_base,
                 int64_t edges_total, int nv, int nu, uint32_t *__restrict__ keys,
                 int32_t *__restrict__ vals, int32_t *__restrict__ status) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < n_edges; e += nw) {
        const int64_t ge = edge_base + e;
        // partition_ranges: part i = [i*E//w, (i+1)*E//w) -> i = ((e+1)*w - 1) // E
        const unsigned part = (unsigned)(((ge + 1) * nparts - 1) / edges_total);
        const int64_t s = starts[e], n = starts[e + 1] - s;
        for (int64_t j = lane; j + 1 < n; j += 32) {
            const double2 a = pts[s + j], b = pts[s + j + 1];
            const int x0 = cell_round(a.x), y0 = cell_round(a.y);
            const int x1 = cell_round(b.x), y1 = cell_round(b.y);
            const int dx = x1 - x0, dy = y1 - y0;
            const int steps = max(abs(dx), abs(dy));
            const int k0 = j == 0 ? 0 : 1;
            int64_t o = hoff[s + j];
            auto put = [&](int u, int v) {
                uint32_t key = 0xffffffffu;
                if ((unsigned)u < (unsigned)nu && (unsigned)v < (unsigned)nv)
                    key = (uint32_t)((int64_t)v * nu + u) * (uint32_t)nparts + part;
                else
                    atomicOr(status, HB_STATUS_OUT_OF_BOUNDS);
                keys[o] = key;
                vals[o] = (int32_t)ge;
                ++o;
            };
            if (steps == 0) {
                if (k0 == 0) put(x0, y0);
                continue;
            }
            const double inv = 1.0 / (double)steps;
            for (int k = k0; k <= steps; ++k)
                put(floor_i(dadd(dadd((double)x0, dmul((double)(k * dx), inv)), 0.5)),
                    floor_i(dadd(dadd((double)y0, dmul((double)(k * dy), inv)), 0.5)));
        }
    }
}

struct CellOf {
    uint32_t p;
    __host__ __device__ __forceinline__ uint32_t operator()(uint32_t k) const {
        return k == 0xffffffffu ? 0xffffffffu : k / p;
    }
};

// One warp per cell run (grid-stride over the runs): lane = layer (blocks of
// 32 layers), the cell's hits streamed 32 at a time and folded in order.
__global__ void __launch_bounds__(256)
ordered_fold_kernel(const uint32_t *__restrict__ keys, const int32_t *__restrict__ vals,
                    const uint32_t *__restrict__ run_cell, const int32_t *__restrict__ run_len,
                    const int64_t *__restrict__ run_off, const int *__restrict__ n_runs, int nparts,
                    const float *__restrict__ w32, const int32_t *__restrict__ groups,
                    const float *__restrict__ mat, int nb, int64_t cell_base, int64_t n_cells,
                    float *__restrict__ out) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int runs = *n_runs;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < runs; r += nw) {
        const uint32_t cell_key = run_cell[r];
        const int64_t cell = (int64_t)cell_key - cell_base;  // output column of this run
        if (cell_key == 0xffffffffu || cell < 0 || cell >= n_cells) continue;
        const int64_t off = run_off[r], len = run_len[r];
        for (int l0 = 0; l0 < nb; l0 += 32) {
            const int l = l0 + lane;
            float total = 0.0f, acc = 0.0f;
            bool first = true;
            int curp = -1;
            for (int64_t base = 0; base < len; base += 32) {
                const int64_t i = off + base + lane;
                const bool have = base + lane < len;
                const uint32_t key = have ? keys[i] : 0u;
                const int e = have ? vals[i] : 0;
                const int p = (int)(key % (uint32_t)nparts);
                const float w = (have && w32) ? w32[e] : 1.0f;
                const int b = (have && groups) ? groups[e] : 0;
                const int n = (int)min((int64_t)32, len - base);
                for (int k = 0; k < n; ++k) {
                    const int pk = __shfl_sync(full, p, k);
                    const float wk = __shfl_sync(full, w, k);
                    const int bk = __shfl_sync(full, b, k);
                    if (pk != curp) {  // next partition buffer (raster.py:91-94)
                        if (curp >= 0) {
                            total = first ? acc : __fadd_rn(total, acc);
                            first = false;
                        }
                        acc = 0.0f;
                        curp = pk;
                    }
                    if (l < nb) {
                        // layer_w[e, l] = fl32(w_e) * M.T[b_e][l] (bundler.py:345-346)
                        const float lw = mat ? __fmul_rn(wk, __ldg(mat + l * nb + bk))
                                             : (l == bk ? wk : 0.0f);
                        acc = __fadd_rn(acc, lw);
                    }
                }
            }
            if (curp >= 0) total = first ? acc : __fadd_rn(total, acc);
            if (l < nb) out[(int64_t)l * n_cells + cell] = total;
        }
    }
}

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

static int key_bits(int64_t plane, int nparts) {
    // valid keys are < maxkey; the sentinel 0xffffffff must sort after all
    // of them on the sorted bits, so its low `bits` bits (all ones) must
    // exceed maxkey - 1
    const uint64_t maxkey = (uint64_t)plane * (uint64_t)nparts;
    int bits = 1;
    while (bits < 32 && (1ull << bits) <= maxkey) ++bits;
    return bits;
}

static size_t sort_tmp_bytes(int64_t n) {
    size_t a = 0;
    cub::DoubleBuffer<uint32_t> k(nullptr, nullptr);
    cub::DoubleBuffer<int32_t> v(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, a, k, v, (int)n, 0, 32);
    return align_up(a);
}

static size_t fold_tmp_bytes(int64_t n, int64_t runs) {
    size_t b = 0, c = 0;
    thrust::transform_iterator<CellOf, const uint32_t *> it(nullptr, CellOf{1});
    cub::DeviceRunLengthEncode::Encode(nullptr, b, it, (uint32_t *)nullptr, (int32_t *)nullptr,
                                       (int *)nullptr, (int)n);
    cub::DeviceScan::ExclusiveSum(nullptr, c, (const int32_t *)nullptr, (int64_t *)nullptr,
                                  (int)runs);
    return align_up(b > c ? b : c);
}

// Stable sort of (key, val) pairs by key, in place (keys/vals on return),
// with a scratch double buffer and CUB temp from `ws`.
static int sort_pairs(uint32_t *keys, int32_t *vals, int64_t n, int end_bit, char *ws,
                      cudaStream_t st) {
    uint32_t *k2 = reinterpret_cast<uint32_t *>(ws); ws += align_up(4 * (size_t)n);
    int32_t *v2 = reinterpret_cast<int32_t *>(ws); ws += align_up(4 * (size_t)n);
    cub::DoubleBuffer<uint32_t> kb(keys, k2);
    cub::DoubleBuffer<int32_t> vb(vals, v2);
    size_t tb = sort_tmp_bytes(n);
    if (cub::DeviceRadixSort::SortPairs(ws, tb, kb, vb, (int)n, 0, end_bit, st) != cudaSuccess)
        return check_launch("hb_ordered(sort)", 0);
    if (kb.Current() != keys &&
        (cudaMemcpyAsync(keys, kb.Current(), 4 * (size_t)n, cudaMemcpyDeviceToDevice, st) !=
             cudaSuccess ||
         cudaMemcpyAsync(vals, vb.Current(), 4 * (size_t)n, cudaMemcpyDeviceToDevice, st) !=
             cudaSuccess))
        return check_launch("hb_ordered(sort copy)", 0);
    return HB_OK;
}
static size_t sort_ws_bytes(int64_t n) { return 2 * align_up(4 * (size_t)n) + sort_tmp_bytes(n); }

// Runs of equal cell over sorted records -> one warp per cell folds them.
static int fold_sorted(const uint32_t *keys, const int32_t *vals, int64_t n, int nparts,
                       int64_t cell_base, int64_t n_cells, const float *w32,
                       const int32_t *groups, const float *matrix, int nbins, float *out,
                       char *ws, cudaStream_t st) {
    const int64_t runs_cap = n < n_cells + 1 ? n : n_cells + 1;  // + the sentinel run
    uint32_t *run_cell = reinterpret_cast<uint32_t *>(ws); ws += align_up(4 * (size_t)(runs_cap + 1));
    int32_t *run_len = reinterpret_cast<int32_t *>(ws); ws += align_up(4 * (size_t)(runs_cap + 1));
    int64_t *run_off = reinterpret_cast<int64_t *>(ws); ws += align_up(8 * (size_t)(runs_cap + 1));
    int *n_runs = reinterpret_cast<int *>(ws); ws += 256;
    if (cudaMemsetAsync(run_len, 0, 4 * (size_t)(runs_cap + 1), st) != cudaSuccess)
        return check_launch("hb_ordered(memset)", 0);
    thrust::transform_iterator<CellOf, const uint32_t *> cells(keys, CellOf{(uint32_t)nparts});
    size_t tb = fold_tmp_bytes(n, runs_cap + 1);
    if (cub::DeviceRunLengthEncode::Encode(ws, tb, cells, run_cell, run_len, n_runs, (int)n,
                                           st) != cudaSuccess)
        return check_launch("hb_ordered(rle)", 0);
    // run offsets: exclusive scan of the run lengths (entries past n_runs
    // stay zero and are never read)
    tb = fold_tmp_bytes(n, runs_cap + 1);
    if (cub::DeviceScan::ExclusiveSum(ws, tb, run_len, run_off, (int)(runs_cap + 1), st) !=
        cudaSuccess)
        return check_launch("hb_ordered(scan)", 1);
    const int64_t fold_warps = runs_cap < (int64_t)device_sm_count() * 64
                                   ? runs_cap : (int64_t)device_sm_count() * 64;
    ordered_fold_kernel<<<(unsigned)((fold_warps * 32 + 255) / 256), 256, 0, st>>>(
        keys, vals, run_cell, run_len, run_off, n_runs, nparts, w32, groups, matrix, nbins,
        cell_base, n_cells, out);
    return check_launch("hb_ordered(fold)", 3);
}
static size_t fold_ws_bytes(int64_t n, int64_t n_cells) {
    const int64_t runs_cap = (n < n_cells + 1 ? n : n_cells + 1) + 1;
    return 2 * align_up(4 * (size_t)runs_cap) + align_up(8 * (size_t)runs_cap) + 256 +
           fold_tmp_bytes(n, runs_cap);
}

static void fill_launch(const double *pts, const int64_t *starts, int64_t n_edges,
                        const int64_t *hoff, int nparts, int64_t edge_base, int64_t edges_total,
                        int nv, int nu, uint32_t *keys, int32_t *vals, int32_t *status,
                        cudaStream_t st) {
    const int64_t warps = n_edges < (int64_t)device_sm_count() * 64 ? n_edges
                                                                 : (int64_t)device_sm_count() * 64;
    hits_fill_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<const double2 *>(pts), starts, n_edges, hoff, nparts, edge_base,
        edges_total, nv, nu, keys, vals, status);
}

}  // namespace hb

using namespace hb;

static inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

int hb_point_span(const double *pts, int64_t n_pts, void *scratch32, double *out4, void *stream) {
    if (n_pts < 0 || !scratch32 || !out4 || (n_pts > 0 && !pts))
        return set_error(HB_EINVAL, "hb_point_span: bad arguments");
    cudaStream_t st = as_stream(stream);
    auto *k4 = reinterpret_cast<unsigned long long *>(scratch32);
    span_init_kernel<<<1, 1, 0, st>>>(k4);
    int blocks = 4 * device_sm_count();
    if ((int64_t)blocks * 256 > n_pts) blocks = (int)((n_pts + 255) / 256);
    if (blocks > 0)
        span_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<const double2 *>(pts), n_pts, k4);
    span_final_kernel<<<1, 1, 0, st>>>(k4, out4);
    return check_launch("hb_point_span", blocks > 0 ? 3 : 2);
}

int hb_exact_check(const int32_t *counts, const double *abs_matrix, int nbins, int nv, int nu,
                   double limit, int32_t *status, void *stream) {
    if (!counts || !status || nbins < 1 || nv < 1 || nu < 1 || nv > kMaxDim || nu > kMaxDim)
        return set_error(HB_EINVAL, "hb_exact_check: bad arguments");
    const int64_t plane = (int64_t)nv * nu;
    int blocks = 4 * device_sm_count();
    if ((int64_t)blocks * 256 > plane) blocks = (int)((plane + 255) / 256);
    exact_check_kernel<<<blocks, 256, 0, as_stream(stream)>>>(counts, abs_matrix, nbins, plane,
                                                              limit, status);
    return check_launch("hb_exact_check");
}

size_t hb_hits_workspace_bytes(int64_t n_pts) {
    size_t a = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, a, (const int32_t *)nullptr, (int64_t *)nullptr,
                                  (int)(n_pts + 1));
    return align_up(4 * (size_t)(n_pts + 1)) + align_up(a) + 256;
}

int hb_hits_count(const double *pts, const int64_t *starts, int64_t n_edges, int64_t n_pts,
                  int64_t *hoff, void *workspace, size_t workspace_bytes, void *stream) {
    if (n_edges < 0 || n_pts < 0 || n_pts >= (1ll << 31) - 1 || !hoff ||
        (n_edges > 0 && (!pts || !starts)) || !workspace ||
        workspace_bytes < hb_hits_workspace_bytes(n_pts))
        return set_error(HB_EINVAL, "hb_hits_count: bad arguments");
    cudaStream_t st = as_stream(stream);
    int32_t *hcnt = reinterpret_cast<int32_t *>(workspace);
    void *tmp = reinterpret_cast<char *>(workspace) + align_up(4 * (size_t)(n_pts + 1));
    if (cudaMemsetAsync(hcnt, 0, 4 * (size_t)(n_pts + 1), st) != cudaSuccess)
        return check_launch("hb_hits_count(memset)", 0);
    int kernels = 0;
    if (n_edges > 0) {
        const int64_t warps = n_edges < (int64_t)device_sm_count() * 64 ? n_edges
                                                                     : (int64_t)device_sm_count() * 64;
        hits_count_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(
            reinterpret_cast<const double2 *>(pts), starts, n_edges, hcnt);
        ++kernels;
    }
    size_t a = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, a, hcnt, hoff, (int)(n_pts + 1), st);
    cub::DeviceScan::ExclusiveSum(tmp, a, hcnt, hoff, (int)(n_pts + 1), st);
    return check_launch("hb_hits_count", kernels + 1);
}

static bool ordered_args_ok(int64_t n_edges, int64_t n_hits, int nparts, int nv, int nu,
                            int64_t edge_base, int64_t edges_total) {
    const int64_t plane = (int64_t)nv * nu;
    return n_edges >= 0 && n_hits >= 0 && n_hits < (1ll << 31) && nparts >= 1 && nv >= 1 &&
           nu >= 1 && nv <= kMaxDim && nu <= kMaxDim && edge_base >= 0 &&
           edges_total >= edge_base + n_edges && edges_total < (1ll << 31) &&
           (uint64_t)plane * (uint64_t)nparts < 0xffffffffull;
}

size_t hb_ordered_workspace_bytes(int64_t n_hits, int nv, int nu, int nparts) {
    if (n_hits < 0 || nv < 1 || nu < 1 || nparts < 1) return 0;
    const int64_t plane = (int64_t)nv * nu;
    const size_t recs = 2 * align_up(4 * (size_t)n_hits);
    const size_t a = sort_ws_bytes(n_hits), b = fold_ws_bytes(n_hits, plane);
    return recs + (a > b ? a : b) + 256;
}

int hb_accumulate_ordered(const double *pts, const int64_t *starts, int64_t n_edges,
                          const int64_t *hoff, int64_t n_pts, int64_t n_hits, int nparts,
                          int64_t edge_base, int64_t edges_total, const float *w32,
                          const int32_t *groups, const float *matrix, int nbins, int nv, int nu,
                          float *out, int32_t *status, void *workspace, size_t workspace_bytes,
                          void *stream) {
    const int64_t plane = (int64_t)nv * nu;
    if (!ordered_args_ok(n_edges, n_hits, nparts, nv, nu, edge_base, edges_total) ||
        nbins < 1 || !out || !status || (n_edges > 0 && (!pts || !starts || !hoff)) ||
        !workspace || workspace_bytes < hb_ordered_workspace_bytes(n_hits, nv, nu, nparts))
        return set_error(HB_EINVAL, "hb_accumulate_ordered: bad arguments");
    (void)n_pts;
    cudaStream_t st = as_stream(stream);
    if (cudaMemsetAsync(out, 0, sizeof(float) * (size_t)nbins * plane, st) != cudaSuccess)
        return check_launch("hb_accumulate_ordered(memset)", 0);
    if (n_hits == 0 || n_edges == 0) return check_launch("hb_accumulate_ordered", 0);
    char *p = reinterpret_cast<char *>(workspace);
    uint32_t *keys = reinterpret_cast<uint32_t *>(p); p += align_up(4 * (size_t)n_hits);
    int32_t *vals = reinterpret_cast<int32_t *>(p); p += align_up(4 * (size_t)n_hits);
    fill_launch(pts, starts, n_edges, hoff, nparts, edge_base, edges_total, nv, nu, keys, vals,
                status, st);
    int rc = check_launch("hb_accumulate_ordered(fill)");
    if (rc) return rc;
    if ((rc = sort_pairs(keys, vals, n_hits, key_bits(plane, nparts), p, st))) return rc;
    return fold_sorted(keys, vals, n_hits, nparts, 0, plane, w32, groups, matrix, nbins, out, p,
                       st);
}

size_t hb_hits_sorted_workspace_bytes(int64_t n_hits) { return sort_ws_bytes(n_hits) + 256; }

int hb_hits_fill_sorted(const double *pts, const int64_t *starts, int64_t n_edges,
                        const int64_t *hoff, int64_t n_hits, int nparts, int64_t edge_base,
                        int64_t edges_total, int nv, int nu, uint32_t *keys, int32_t *vals,
                        int32_t *status, void *workspace, size_t workspace_bytes, void *stream) {
    if (!ordered_args_ok(n_edges, n_hits, nparts, nv, nu, edge_base, edges_total) || !status ||
        (n_hits > 0 && (!keys || !vals)) || (n_edges > 0 && (!pts || !starts || !hoff)) ||
        !workspace || workspace_bytes < hb_hits_sorted_workspace_bytes(n_hits))
        return set_error(HB_EINVAL, "hb_hits_fill_sorted: bad arguments");
    if (n_hits == 0 || n_edges == 0) return HB_OK;
    cudaStream_t st = as_stream(stream);
    fill_launch(pts, starts, n_edges, hoff, nparts, edge_base, edges_total, nv, nu, keys, vals,
                status, st);
    int rc = check_launch("hb_hits_fill_sorted(fill)");
    if (rc) return rc;
    return sort_pairs(keys, vals, n_hits, key_bits((int64_t)nv * nu, nparts),
                      reinterpret_cast<char *>(workspace), st);
}

size_t hb_ordered_fold_workspace_bytes(int64_t n_hits, int64_t n_cells) {
    const size_t a = sort_ws_bytes(n_hits), b = fold_ws_bytes(n_hits, n_cells);
    return (a > b ? a : b) + 256;
}

int hb_ordered_fold(uint32_t *keys, int32_t *vals, int64_t n_hits, int sort, int nparts,
                    int64_t cell_base, int64_t n_cells, const float *w32, const int32_t *groups,
                    const float *matrix, int nbins, float *out, void *workspace,
                    size_t workspace_bytes, void *stream) {
    if (n_hits < 0 || n_hits >= (1ll << 31) || nparts < 1 || nbins < 1 || cell_base < 0 ||
        n_cells < 1 || !out || (n_hits > 0 && (!keys || !vals)) || !workspace ||
        workspace_bytes < hb_ordered_fold_workspace_bytes(n_hits, n_cells) ||
        (uint64_t)(cell_base + n_cells) * (uint64_t)nparts >= 0xffffffffull)
        return set_error(HB_EINVAL, "hb_ordered_fold: bad arguments");
    cudaStream_t st = as_stream(stream);
    if (cudaMemsetAsync(out, 0, sizeof(float) * (size_t)nbins * n_cells, st) != cudaSuccess)
        return check_launch("hb_ordered_fold(memset)", 0);
    if (n_hits == 0) return HB_OK;
    char *p = reinterpret_cast<char *>(workspace);
    int rc;
    if (sort && (rc = sort_pairs(keys, vals, n_hits, 32, p, st))) return rc;
    return fold_sorted(keys, vals, n_hits, nparts, cell_base, n_cells, w32, groups, matrix, nbins,
                       out, p, st);
}

}  // extern "C"
