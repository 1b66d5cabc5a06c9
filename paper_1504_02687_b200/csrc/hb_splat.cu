// hb_splat.cu -- tile-binned histogram splatting (the accumulate of
// _kernels.py:46-77 / raster.py:70-94, reorganised for the B200 memory
// system).
//
// Why: a bundled iteration of config 4 adds ~1.3e9 increments into a 1M-cell
// int32 histogram (one cell takes 1.1e6 of them).  As L2 atomics that costs
// ~13 ms (~100 G RED/s).  Instead the streaming kernels append one 8-byte
// record per segment to the bucket of the tile holding its first cell
// (bin_or_splat, hb_common.cuh), and this file replays each bucket into a
// shared-memory window (tile + halo on every side) with shared atomics, then
// adds the window to the histogram with one global atomic per touched cell
// and work chunk.  Integer addition is associative: the result is the same
// int32 histogram bit for bit, whatever the binning.
#include <cub/block/block_scan.cuh>

#include "hb_common.cuh"

namespace hb {

constexpr int kPlanBlock = 1024;
constexpr int kFlushBlock = 512;
constexpr int kChunk = 16384;           // records per flush work item
constexpr int kMaxWindowBytes = 96 * 1024;

// cap = fill + fill/4 + 64 per tile, off = exclusive prefix, fill := 0
__global__ void __launch_bounds__(kPlanBlock)
tiles_plan_kernel(const __grid_constant__ hb_tiles t, int64_t *__restrict__ total) {
    using Scan = cub::BlockScan<int64_t, kPlanBlock>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < t.ntiles; base += kPlanBlock) {
        const int i = base + threadIdx.x;
        int64_t c = 0;
        if (i < t.ntiles) {
            const int64_t f = t.fill[i];
            c = f + f / 4 + 64;
            if (c > 0x7fffffff) c = 0x7fffffff;
            t.cap[i] = (int32_t)c;
            t.fill[i] = 0;
        }
        int64_t ex, agg;
        Scan(tmp).ExclusiveSum(c, ex, agg);
        if (i < t.ntiles) t.off[i] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry += agg;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        t.off[t.ntiles] = carry;
        *total = carry;
    }
}

// work[i] = exclusive prefix of flush chunks per tile, work[ntiles] = total,
// work[ntiles+1] = 0 (the flush kernel's work counter)
__global__ void __launch_bounds__(kPlanBlock)
tiles_worklist_kernel(const __grid_constant__ hb_tiles t) {
    using Scan = cub::BlockScan<int, kPlanBlock>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < t.ntiles; base += kPlanBlock) {
        const int i = base + threadIdx.x;
        int ch = 0;
        if (i < t.ntiles) {
            const int n = min(t.fill[i], t.cap[i]);
            ch = (n + kChunk - 1) / kChunk;
        }
        int ex, agg;
        Scan(tmp).ExclusiveSum(ch, ex, agg);
        if (i < t.ntiles) t.work[i] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry += agg;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        t.work[t.ntiles] = carry;
        t.work[t.ntiles + 1] = 0;
    }
}

// Persistent: CTAs pull (tile, chunk) items off a counter, rasterise the
// chunk's records into a shared window, flush the window.
__global__ void __launch_bounds__(kFlushBlock)
tiles_flush_kernel(const __grid_constant__ hb_tiles t, int32_t *__restrict__ counts, int nv,
                   int nu) {
    extern __shared__ int win[];
    __shared__ int s_item, s_tile;
    const int W = t.tile + 2 * t.halo;
    const int WW = W * W;
    const int64_t plane = (int64_t)nv * nu;
    const int per_layer = t.ntx * t.nty;
    for (;;) {
        if (threadIdx.x == 0) {
            const int item = atomicAdd(t.work + t.ntiles + 1, 1);
            int tile = -1;
            if (item < t.work[t.ntiles]) {
                int lo = 0, hi = t.ntiles;  // last tile with work[tile] <= item
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (t.work[mid] <= item) lo = mid; else hi = mid;
                }
                tile = lo;
            }
            s_item = item;
            s_tile = tile;
        }
        for (int i = threadIdx.x; i < WW; i += kFlushBlock) win[i] = 0;
        __syncthreads();
        const int tile = s_tile;
        if (tile < 0) break;
        const int item = s_item;
        const int g = tile / per_layer;
        const int r = tile - g * per_layer;
        const int ty = r / t.ntx, tx = r - ty * t.ntx;
        const int wx0 = tx * t.tile - t.halo, wy0 = ty * t.tile - t.halo;
        const int n = min(t.fill[tile], t.cap[tile]);
        const int c = item - t.work[tile];
        const int64_t lo = (int64_t)c * kChunk;
        const int64_t hi = lo + kChunk < (int64_t)n ? lo + kChunk : (int64_t)n;
        const uint64_t *rec = t.rec + t.off[tile];
        int32_t *layer = counts + (int64_t)g * plane;
        for (int64_t k = lo + threadIdx.x; k < hi; k += kFlushBlock) {
            const uint64_t rr = rec[k];
            const int x0 = (int)(rr & 0xffff), y0 = (int)((rr >> 16) & 0xffff);
            const int dx = (int)(int8_t)((rr >> 32) & 0xff), dy = (int)(int8_t)((rr >> 40) & 0xff);
            const int k0 = (int)((rr >> 48) & 1);
            const int w = (int)(rr >> 49);
            dda_walk(x0, y0, x0 + dx, y0 + dy, k0, [&](int u, int v) {
                const int lu = u - wx0, lv = v - wy0;
                if ((unsigned)lu < (unsigned)W && (unsigned)lv < (unsigned)W)
                    atomicAdd(win + lv * W + lu, w);
                else
                    atomicAdd(layer + (int64_t)v * nu + u, w);
            });
        }
        __syncthreads();
        for (int i = threadIdx.x; i < WW; i += kFlushBlock) {
            const int val = win[i];
            if (val) {
                const int v = wy0 + i / W, u = wx0 + i % W;
                atomicAdd(layer + (int64_t)v * nu + u, val);
            }
        }
        __syncthreads();
    }
}

}  // namespace hb

using namespace hb;

static inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

int hb_tiles_geometry(int nbins, int nv, int nu, double max_seg_cells, hb_tiles *t) {
    if (!t || nbins < 1 || nv < 1 || nu < 1 || !(max_seg_cells >= 0))
        return set_error(HB_EINVAL, "hb_tiles_geometry: bad arguments");
    if (nv > 65535 || nu > 65535 || max_seg_cells > 126.0)
        return set_error(HB_EINVAL, "hb_tiles_geometry: grid or segments too large to bin");
    const int halo = (int)ceil(max_seg_cells) + 1;
    const int wmax = (int)floor(sqrt((double)kMaxWindowBytes / sizeof(int)));
    int tile = wmax - 2 * halo;
    if (tile > 64) tile = 64;
    tile &= ~7;
    if (tile < 16) return set_error(HB_EINVAL, "hb_tiles_geometry: halo %d too large", halo);
    t->tile = tile;
    t->halo = halo;
    t->ntx = (nu + tile - 1) / tile;
    t->nty = (nv + tile - 1) / tile;
    t->nbins = nbins;
    const int64_t n = (int64_t)nbins * t->ntx * t->nty;
    if (n > 0x7fffffff) return set_error(HB_EINVAL, "hb_tiles_geometry: too many tiles");
    t->ntiles = (int)n;
    return HB_OK;
}

int hb_tiles_plan(const hb_tiles *t, int64_t *total, void *stream) {
    if (!t || !t->off || !t->cap || !t->fill || !total || t->ntiles < 1)
        return set_error(HB_EINVAL, "hb_tiles_plan: bad arguments");
    tiles_plan_kernel<<<1, kPlanBlock, 0, as_stream(stream)>>>(*t, total);
    return check_launch("hb_tiles_plan");
}

int hb_tiles_flush(const hb_tiles *t, int32_t *counts, int nv, int nu, void *stream) {
    if (!t || !t->off || !t->cap || !t->fill || !t->work || !t->rec || !counts || nv < 1 ||
        nu < 1 || nv > 65535 || nu > 65535)
        return set_error(HB_EINVAL, "hb_tiles_flush: bad arguments");
    cudaStream_t st = as_stream(stream);
    tiles_worklist_kernel<<<1, kPlanBlock, 0, st>>>(*t);
    const int W = t->tile + 2 * t->halo;
    const size_t smem = (size_t)W * W * sizeof(int);
    static size_t configured = 0;
    if (smem > configured) {
        if (cudaFuncSetAttribute(tiles_flush_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) != cudaSuccess)
            return check_launch("hb_tiles_flush(smem)", 0);
        configured = smem;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tiles_flush_kernel, kFlushBlock,
                                                      smem) != cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    tiles_flush_kernel<<<device_sm_count() * per_sm, kFlushBlock, smem, st>>>(*t, counts, nv, nu);
    return check_launch("hb_tiles_flush", 2);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Segment-key table (mode 1).  tab[((g*D*D + dir)*nv + y0)*nu + x0] holds the
// summed weight of every k0 == 1 segment of layer g that starts in cell
// (x0, y0) with cell delta dir = (dy+H)*D + (dx+H).  The expansion reads the
// table with 16-byte loads, rasterises each non-zero key once (weight x
// path is exactly the sum of the individual paths: integer addition) and
// resets it, so the table is zero again for the next pass.
namespace hb {

constexpr int kExpandBlock = 256;

__global__ void __launch_bounds__(kExpandBlock)
segtab_expand_kernel(const __grid_constant__ hb_tiles t, int32_t *__restrict__ counts, int nv,
                     int nu, int64_t n4, unsigned long long *__restrict__ nonzero) {
    const int H = t.halo, D = 2 * H + 1;
    unsigned keys = 0;
    const int64_t plane = (int64_t)nv * nu;
    uint4 *tab4 = reinterpret_cast<uint4 *>(t.tab);
    for (int64_t q = (int64_t)blockIdx.x * kExpandBlock + threadIdx.x; q < n4;
         q += (int64_t)gridDim.x * kExpandBlock) {
        const uint4 v4 = tab4[q];
        if ((v4.x | v4.y | v4.z | v4.w) == 0u) continue;
        tab4[q] = make_uint4(0u, 0u, 0u, 0u);
        const unsigned vals[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const unsigned val = vals[c];
            if (!val) continue;
            ++keys;
            const int64_t idx = q * 4 + c;
            const int64_t key = idx / plane;  // g*D*D + dir
            const int64_t cell = idx - key * plane;
            const int g = (int)(key / ((int64_t)D * D));
            const int dir = (int)(key - (int64_t)g * D * D);
            const int dy = dir / D - H, dx = dir % D - H;
            const int y0 = (int)(cell / nu), x0 = (int)(cell - (int64_t)y0 * nu);
            int32_t *layer = counts + (int64_t)g * plane;
            dda_walk(x0, y0, x0 + dx, y0 + dy, 1, [&](int u, int v) {
                atomicAdd(layer + (int64_t)v * nu + u, (int)val);
            });
        }
    }
    if (nonzero) {
        for (int o = 16; o; o >>= 1) keys += __shfl_down_sync(0xffffffffu, keys, o);
        if ((threadIdx.x & 31) == 0 && keys) atomicAdd(nonzero, (unsigned long long)keys);
    }
}

}  // namespace hb

extern "C" {

int hb_segtab_geometry(int nbins, int nv, int nu, double max_seg_cells, hb_tiles *t,
                       int64_t *entries) {
    if (!t || !entries || nbins < 1 || nv < 1 || nu < 1 || !(max_seg_cells >= 0))
        return set_error(HB_EINVAL, "hb_segtab_geometry: bad arguments");
    if (max_seg_cells > 60.0)
        return set_error(HB_EINVAL, "hb_segtab_geometry: segments too long for a key table");
    const int H = (int)ceil(max_seg_cells) + 1;
    const int64_t D = 2 * H + 1;
    t->mode = 1;
    t->halo = H;
    t->nbins = nbins;
    *entries = (int64_t)nbins * D * D * nv * nu;
    // whole uint4 loads in the expansion
    *entries = (*entries + 3) / 4 * 4;
    if (*entries >= ((int64_t)1 << 31))  // keys are 32-bit indices (bin_or_splat)
        return set_error(HB_EINVAL, "hb_segtab_geometry: key table above 2^31 entries");
    return HB_OK;
}

int hb_segtab_expand(const hb_tiles *t, int32_t *counts, int nv, int nu,
                     unsigned long long *nonzero, void *stream) {
    if (!t || t->mode != 1 || !t->tab || !counts || nv < 1 || nu < 1)
        return set_error(HB_EINVAL, "hb_segtab_expand: bad arguments");
    const int64_t D = 2 * t->halo + 1;
    const int64_t n = (int64_t)t->nbins * D * D * nv * nu;
    const int64_t n4 = (n + 3) / 4;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, segtab_expand_kernel,
                                                      kExpandBlock, 0) != cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    const int64_t want = (n4 + kExpandBlock - 1) / kExpandBlock;
    const int64_t cap = (int64_t)device_sm_count() * per_sm * 4;
    segtab_expand_kernel<<<(unsigned)(want < cap ? want : cap), kExpandBlock, 0,
                           as_stream(stream)>>>(*t, counts, nv, nu, n4, nonzero);
    return check_launch("hb_segtab_expand");
}

}  // extern "C"
