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

__device__ __forceinline__ void red_shared(unsigned addr, int v) {
    asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
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
        // Records have |dx|, |dy| <= halo (bin_or_splat_cells), so every cell
        // is inside the window: the walk is dda_walk's cell chain expressed as
        // a window index, idx = base + major_step * k + minor_mul * minor(k),
        // with minor(k) = floor(c + (k*d)*(1/steps) + 0.5) in float64 (k*d
        // carried as an exact double), and the adds go to shared memory by
        // address (red.shared) -- ~9 instructions per cell.
        const unsigned swin = (unsigned)__cvta_generic_to_shared(win);
        for (int64_t k = lo + threadIdx.x; k < hi; k += kFlushBlock) {
            const uint64_t rr = rec[k];
            const int x0 = (int)(rr & 0xffff), y0 = (int)((rr >> 16) & 0xffff);
            const int dx = (int)(int8_t)((rr >> 32) & 0xff), dy = (int)(int8_t)((rr >> 40) & 0xff);
            const int k0 = (int)((rr >> 48) & 1);
            const int w = (int)(rr >> 49);
            const int steps = max(abs(dx), abs(dy));
            if (steps == 0) {
                if (k0 == 0) red_shared(swin + 4u * (unsigned)((y0 - wy0) * W + (x0 - wx0)), w);
                continue;
            }
            const bool xdom = abs(dx) == steps;
            const int major_step = xdom ? (dx > 0 ? 1 : -1) : (dy > 0 ? W : -W);
            const int minor_mul = xdom ? W : 1;
            const int dmin = xdom ? dy : dx;
            const double c = (double)(xdom ? y0 : x0), inv = 1.0 / (double)steps;
            // window index of (major at k, minor = 0)
            int base = xdom ? (x0 - wx0) - wy0 * W : (y0 - wy0) * W - wx0;
            base += major_step * k0;
            double kd = (double)(k0 * dmin);
            const double dd = (double)dmin;
            for (int kk = k0; kk <= steps; ++kk) {
                const int minor = floor_i(dadd(dadd(c, dmul(kd, inv)), 0.5));
                red_shared(swin + 4u * (unsigned)(base + minor_mul * minor), w);
                base += major_step;
                kd = dadd(kd, dd);
            }
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
// Tile shape measured on config 4 (expansion ms/iteration): 64x32 0.665,
// 64x16 0.52, 64x8 0.40, 64x4 0.33, 64x2 / 32x4 / 16x8 0.33 -- small tiles
// give many blocks to hide the table scan's latency; the halo overhead of
// the shared histogram only costs flush atomics on touched cells.
#ifndef HB_EX_TY
#define HB_EX_TY 4
#endif
#ifndef HB_EX_UNROLL
#define HB_EX_UNROLL 2
#endif
#ifndef HB_EX_TX
#define HB_EX_TX 64
#endif
constexpr int kExTX = HB_EX_TX, kExTY = HB_EX_TY;  // start-cell tile of one expansion block
static_assert(kExTX <= 64 && kExTX % 4 == 0, "column field of the packed key is 6 bits");
static_assert(kExTY <= 128 && kExTY % 4 == 0, "tiles are whole 4x4 block rows; 7-bit row");
constexpr int kExUnroll = HB_EX_UNROLL;      // table loads in flight per thread per round
constexpr int kExRound = kExpandBlock * kExUnroll * 4;  // max keys found per round
constexpr int kExBuf = 2 * kExRound;                    // compacted key buffer
#ifdef HB_EX_STREAM
#define HB_EX_LOAD(p) __ldcs(p)
#else
#define HB_EX_LOAD(p) (*(p))
#endif

// One block per (start-cell tile, group).  The block scans every delta plane
// of the key table over its tile (aligned uint4 rows), zeroing what it reads
// and compacting the non-zero keys (plane, row, column, count) into a shared
// buffer; whenever the buffer could overflow, all threads rasterise buffered
// keys (_kernels.py:58-77, k0 = 1), one per thread, into a shared histogram
// covering the tile plus the H-cell halo its segments reach.  The shared
// histogram is added to the global one at the end: one atomic per touched
// cell instead of one per rasterised cell (bundled keys pile onto few cells).
__global__ void __launch_bounds__(kExpandBlock)
segtab_expand_kernel(const __grid_constant__ hb_tiles t, int32_t *__restrict__ counts, int nv,
                     int nu, unsigned long long *__restrict__ nonzero) {
    extern __shared__ int sh[];  // (kExTY + 2H) x (kExTX + 2H) cell counts
    __shared__ uint2 buf[kExBuf];
    __shared__ int nbuf;
    const int H = t.halo, D = 2 * H + 1, DD = D * D;
    const int SW = kExTX + 2 * H, SH = kExTY + 2 * H;
    const int nbx = segtab_nbx(nu), nby = segtab_nby(nv);
    const int ntx = (nu + kExTX - 1) / kExTX;
    const int tx0 = (blockIdx.x % ntx) * kExTX, ty0 = (blockIdx.x / ntx) * kExTY;
    const int g = blockIdx.y;
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < SW * SH; i += kExpandBlock) sh[i] = 0;
    if (threadIdx.x == 0) nbuf = 0;
    __syncthreads();
    // per plane the tile is (kExTY/4) block rows of kExTX/4 blocks of four
    // uint4 rows (one uint4 = 4 cells of one cell row): contiguous runs
    constexpr int c4 = kExTX / 4, per_plane = kExTY * c4;
    const int total = DD * per_plane;
    uint4 *tab4 = reinterpret_cast<uint4 *>(t.tab);
    // uint4 index of (plane, local block row br, local block bc, cell row ly)
    auto q4 = [&](int plane, int br, int bc, int ly) -> int64_t {
        return ((((int64_t)(g * DD + plane) * nby + (ty0 >> 2) + br) * nbx + (tx0 >> 2) + bc) << 2) +
               ly;
    };
    unsigned keys = 0;

    const unsigned ssh = (unsigned)__cvta_generic_to_shared(sh);
    auto rasterise = [&]() {  // all threads: drain the buffer into sh
        const int n = nbuf;
        for (int i = threadIdx.x; i < n; i += kExpandBlock) {
            const uint2 k = buf[i];
            const int plane = (int)(k.x >> 13), ly0 = (int)((k.x >> 6) & 127u),
                      lx0 = (int)(k.x & 63u);
            const int dy = plane / D - H, dx = plane % D - H;
            // dda_walk's chain from k0 = 1 as an index into sh (all cells are
            // within the H halo); a zero delta adds nothing at k0 = 1
            const int steps = max(abs(dx), abs(dy));
            if (steps == 0) continue;
            const bool xdom = abs(dx) == steps;
            const int major_step = xdom ? (dx > 0 ? 1 : -1) : (dy > 0 ? SW : -SW);
            const int minor_mul = xdom ? SW : 1;
            const int dmin = xdom ? dy : dx;
            // (global start cell: the float64 expression uses it)
            const double c = (double)(xdom ? ty0 + ly0 : tx0 + lx0), inv = 1.0 / (double)steps;
            // sh index of (major at k, minor 0): sh[(v - ty0 + H) * SW + (u - tx0 + H)]
            int base = xdom ? (lx0 + H) + (H - ty0) * SW : (ly0 + H) * SW + (H - tx0);
            base += major_step;
            double kd = (double)dmin;
            const double dd = (double)dmin;
            for (int kk = 1; kk <= steps; ++kk) {
                const int minor = floor_i(dadd(dadd(c, dmul(kd, inv)), 0.5));
                red_shared(ssh + 4u * (unsigned)(base + minor_mul * minor), (int)k.y);
                base += major_step;
                kd = dadd(kd, dd);
            }
        }
    };

    // Scan n table rows (uint4 = 4 cells of one cell row); decode(idx, plane,
    // br, bc, ly) names row idx.  Block-uniform trip count: the body has warp
    // shuffles and a barrier.
    auto consume = [&](int n, auto decode) {
        uint4 v[kExUnroll], vn[kExUnroll];
        int64_t at[kExUnroll], atn[kExUnroll];
        unsigned pkey[kExUnroll], pkn[kExUnroll];
        auto load = [&](int base) {  // rows of the round starting at base
#pragma unroll
            for (int k = 0; k < kExUnroll; ++k) {
                const int idx = base + k * kExpandBlock;
                int plane = 0, br = 0, bc = 0, ly = 0;
                vn[k] = make_uint4(0u, 0u, 0u, 0u);
                atn[k] = -1;
                pkn[k] = 0;
                if (idx < n && decode(idx, plane, br, bc, ly)) {
                    atn[k] = q4(plane, br, bc, ly);
                    vn[k] = HB_EX_LOAD(tab4 + atn[k]);
                    pkn[k] = ((unsigned)plane << 13) | ((unsigned)(br * 4 + ly) << 6) |
                             (unsigned)(bc * 4);
                }
            }
        };
        constexpr int kStep = kExpandBlock * kExUnroll;
        if (n > 0) load((int)threadIdx.x);
        for (int base0 = 0; base0 < n; base0 += kStep) {
#pragma unroll
            for (int k = 0; k < kExUnroll; ++k) v[k] = vn[k], at[k] = atn[k], pkey[k] = pkn[k];
            // the next round's rows are in flight while this round compacts
            if (base0 + kStep < n) load(base0 + kStep + (int)threadIdx.x);
            int mine = 0;
#pragma unroll
            for (int k = 0; k < kExUnroll; ++k)
                mine += (v[k].x != 0u) + (v[k].y != 0u) + (v[k].z != 0u) + (v[k].w != 0u);
            // warp-aggregated slot reservation
            int incl = mine;
            for (int d = 1; d < 32; d <<= 1) {
                const int o = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += o;
            }
            int slot = 0;
            if (lane == 31 && incl) slot = atomicAdd(&nbuf, incl);
            slot = __shfl_sync(0xffffffffu, slot, 31) + incl - mine;
            if (mine) {
                keys += mine;
#pragma unroll
                for (int k = 0; k < kExUnroll; ++k) {
                    if ((v[k].x | v[k].y | v[k].z | v[k].w) == 0u) continue;
                    tab4[at[k]] = make_uint4(0u, 0u, 0u, 0u);
                    const unsigned pk = pkey[k];
                    if (v[k].x) buf[slot++] = make_uint2(pk + 0u, v[k].x);
                    if (v[k].y) buf[slot++] = make_uint2(pk + 1u, v[k].y);
                    if (v[k].z) buf[slot++] = make_uint2(pk + 2u, v[k].z);
                    if (v[k].w) buf[slot++] = make_uint2(pk + 3u, v[k].w);
                }
            }
            __syncthreads();
            if (nbuf > kExBuf - kExRound) {  // (block-uniform) the next round could overflow
                rasterise();
                __syncthreads();
                if (threadIdx.x == 0) nbuf = 0;
                __syncthreads();
            }
        }
    };

    // every row of every plane over the tile
    consume(total, [&](int idx, int &plane, int &br, int &bc, int &ly) {
        plane = idx / per_plane;
        const int rem = idx - plane * per_plane;
        // rem -> (block row, block, cell row), cell row fastest
        ly = rem & 3, bc = (rem >> 2) % c4, br = (rem >> 2) / c4;
        return ty0 + br * 4 + ly < nv && tx0 + bc * 4 < nu;
    });
    rasterise();
    __syncthreads();
    int32_t *layer = counts + (int64_t)g * nv * nu;
    for (int i = threadIdx.x; i < SW * SH; i += kExpandBlock) {
        const int val = sh[i];
        if (val) {
            const int gy = ty0 - H + i / SW, gx = tx0 - H + i % SW;
            atomicAdd(layer + (int64_t)gy * nu + gx, val);
        }
    }
    if (nonzero) {
        for (int o = 16; o; o >>= 1) keys += __shfl_down_sync(0xffffffffu, keys, o);
        if (lane == 0 && keys) atomicAdd(nonzero, (unsigned long long)keys);
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
    // |round(x1) - round(x0)| <= ceil(|x1 - x0|): a segment no longer than
    // max_seg_cells moves at most ceil(max_seg_cells) cells per axis
    const int H = (int)ceil(max_seg_cells) < 1 ? 1 : (int)ceil(max_seg_cells);
    const int64_t D = 2 * H + 1;
    t->mode = 1;
    t->halo = H;
    t->nbins = nbins;
    // 4x4-cell blocks (segtab_index)
    *entries = (int64_t)nbins * D * D * segtab_nby(nv) * segtab_nbx(nu) * 16;
    if (*entries >= ((int64_t)1 << 31))  // keys are 32-bit indices (bin_or_splat)
        return set_error(HB_EINVAL, "hb_segtab_geometry: key table above 2^31 entries");
    return HB_OK;
}

int hb_segtab_expand(const hb_tiles *t, int32_t *counts, int nv, int nu,
                     unsigned long long *nonzero, void *stream) {
    if (!t || t->mode != 1 || !t->tab || !counts || nv < 1 || nu < 1 || t->halo < 1 ||
        t->nbins < 1)
        return set_error(HB_EINVAL, "hb_segtab_expand: bad arguments");
    const int H = t->halo;
    const size_t smem = sizeof(int) * (size_t)(kExTX + 2 * H) * (kExTY + 2 * H);
    // static (key buffer) + dynamic (histogram) can exceed the 48 KB default
    if (cudaFuncSetAttribute(segtab_expand_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return check_launch("hb_segtab_expand(smem)", 0);
    const unsigned ntiles = (unsigned)(((nu + kExTX - 1) / kExTX) * ((nv + kExTY - 1) / kExTY));
    segtab_expand_kernel<<<dim3(ntiles, t->nbins), kExpandBlock, smem, as_stream(stream)>>>(
        *t, counts, nv, nu, nonzero);
    return check_launch("hb_segtab_expand");
}

}  // extern "C"
