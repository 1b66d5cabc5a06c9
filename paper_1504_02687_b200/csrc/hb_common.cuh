// hb_common.cuh -- exact-arithmetic device helpers shared by the kernels.
//
// The float64 expressions below are written so nvcc emits exactly the
// operations numba emits for the reference kernels (no FMA: the library is
// compiled with --fmad=false and the critical products/sums additionally use
// __dmul_rn/__dadd_rn, which are never contracted).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/histobundle_b200.h"

namespace hb {

constexpr int kWarp = 32;

// ---- error reporting (hb_api.cu) ------------------------------------------
int set_error(int code, const char *fmt, ...);
// checks the last launch error and adds `kernels` to the library's launch
// counter (hb_launch_count, the bench's gpu_launches evidence)
int check_launch(const char *what, int kernels = 1);

// ---- exact float64 primitives ---------------------------------------------
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// Grid cell indices are 32-bit: every kernel entry checks nv, nu <= kMaxDim,
// so v*nu + u and k*dx never overflow.  int(math.floor(x)) of the reference
// becomes one F2I.FLOOR; CUDA's conversion saturates out-of-range values,
// which the clamps that always follow turn into the same clamped index the
// reference's int64 arithmetic produces.
constexpr int kMaxDim = 46340;  // kMaxDim^2 < 2^31

__device__ __forceinline__ int floor_i(double x) { return __double2int_rd(x); }

// int(math.floor(x + 0.5)) -- _kernels.py:59-62
__device__ __forceinline__ int cell_round(double x) { return floor_i(dadd(x, 0.5)); }

__device__ __forceinline__ int clampi(int v, int lo, int hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}

// sqrt((ax)^2 + (ay)^2) with the reference's association
__device__ __forceinline__ double hypot_ref(double ax, double ay) {
    return sqrt(dadd(dmul(ax, ax), dmul(ay, ay)));
}

// numba min(max(v, lo), hi) (_kernels.py:180-181).  v is never NaN and
// lo >= 1 > 0, so no signed zero can tie: the compare-select below returns
// the same double bit for bit, and compiles to 2 DSETP + 4 SEL where
// fmin/fmax carry NaN fix-ups (~12 instructions).
__device__ __forceinline__ double clamp_ref(double v, double lo, double hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}

// Exact sqrt-free comparisons.  sqrt() is correctly rounded and monotone, so
//   sqrt(d) <  lo  <=>  d <  sqrt_lt_bound(lo)   (smallest d with sqrt(d) >= lo)
//   sqrt(d) >  hi  <=>  d >  sqrt_gt_bound(hi)   (largest  d with sqrt(d) <= hi)
// and because scaling by 4^k scales sqrt by exactly 2^k,
//   sqrt(d) * 2^-k > hi  <=>  d > 4^k * sqrt_gt_bound(hi).
// neighbouring doubles of a finite positive t
__device__ __forceinline__ double next_up(double t) {
    return __longlong_as_double(__double_as_longlong(t) + 1);
}
__device__ __forceinline__ double next_down(double t) {
    return __longlong_as_double(__double_as_longlong(t) - 1);
}
__device__ __forceinline__ double sqrt_lt_bound(double lo) {
    double t = dmul(lo, lo);
    while (t > 0.0 && sqrt(next_down(t)) >= lo) t = next_down(t);
    while (sqrt(t) < lo) t = next_up(t);
    return t;
}
__device__ __forceinline__ double sqrt_gt_bound(double hi) {
    double t = dmul(hi, hi);
    while (sqrt(next_up(t)) <= hi) t = next_up(t);
    while (t > 0.0 && sqrt(t) > hi) t = next_down(t);
    return t;
}
// (x-ax)^2 + (y-ay)^2, the argument of the reference's sqrt (_kernels.py:222)
__device__ __forceinline__ double dist2_ref(double x, double y, double ax, double ay) {
    const double dx = dsub(x, ax), dy = dsub(y, ay);
    return dadd(dmul(dx, dx), dmul(dy, dy));
}

__device__ __forceinline__ float ldf(const float *p) { return __ldg(p); }

// a + f*(b - a) with the density difference taken in float32 and promoted
// afterwards (numba types rho[i] - rho[j] as float32)
__device__ __forceinline__ double lerp_f32diff(float a, float b, double f) {
    return dadd((double)a, dmul(f, (double)__fsub_rn(b, a)));
}

// _kernels.py:80-98 bilinear_value
__device__ __forceinline__ double bilinear_ref(const float *__restrict__ rho, int nv, int nu,
                                               double x, double y) {
    const int u0 = clampi(floor_i(x), 0, nu - 2);
    const int v0 = clampi(floor_i(y), 0, nv - 2);
    const double fx = dsub(x, (double)u0);
    const double fy = dsub(y, (double)v0);
    const float *r0 = rho + v0 * nu + u0;
    const float *r1 = r0 + nu;
    const double a = lerp_f32diff(ldf(r0), ldf(r0 + 1), fx);
    const double b = lerp_f32diff(ldf(r1), ldf(r1 + 1), fx);
    return dadd(a, dmul(fy, dsub(b, a)));
}

// _kernels.py:101-114 _cell_gradient (general, clamped), without its 0.5
// factor (see gradient2_value_ref)
__device__ __forceinline__ void cell_grad2_ref(const float *__restrict__ rho, int nv, int nu,
                                               int u, int v, double &gx, double &gy) {
    u = clampi(u, 1, nu - 2);
    v = clampi(v, 1, nv - 2);
    const float *c = rho + v * nu + u;
    gx = (double)__fsub_rn(ldf(c + 1), ldf(c - 1));
    gy = (double)__fsub_rn(ldf(c + nu), ldf(c - nu));
}

// _kernels.py:117-141 gradient_xy and, from the same 4x4 stencil, the
// bilinear value at (x, y) (both clamp u0/v0 to [0, dim-2] identically).
// Returns G = 2 * gradient_xy EXACTLY: the reference's 0.5 * (rho[+1] -
// rho[-1]) factors are power-of-two scalings, which commute with every IEEE
// rounding in the interpolation (values stay far from over/underflow), so
// they are applied once by the caller -- or never, where only the direction
// G/|G| is used.
// Interior fast path (u0 in [1, nu-3], v0 in [1, nv-3], i.e. no clamp can
// fire): 12 loads off one base pointer.  Otherwise the general clamped path.
__device__ __forceinline__ void gradient2_value_ref(const float *__restrict__ rho, int nv,
                                                    int nu, double x, double y, double &Gx,
                                                    double &Gy, double &val) {
    const int u0 = clampi(floor_i(x), 0, nu - 2);
    const int v0 = clampi(floor_i(y), 0, nv - 2);
    const double fx = dsub(x, (double)u0);
    const double fy = dsub(y, (double)v0);
    double g00x, g00y, g10x, g10y, g01x, g01y, g11x, g11y;
    float a00, a01, a10, a11;
    if (u0 >= 1 && u0 <= nu - 3 && v0 >= 1 && v0 <= nv - 3) {
        const float *c = rho + v0 * nu + u0;
        const float m0 = ldf(c - nu), m1 = ldf(c - nu + 1);
        const float r0 = ldf(c - 1), r3 = ldf(c + 2);
        a00 = ldf(c);
        a01 = ldf(c + 1);
        const float s0 = ldf(c + nu - 1), s3 = ldf(c + nu + 2);
        a10 = ldf(c + nu);
        a11 = ldf(c + nu + 1);
        const float t1 = ldf(c + 2 * nu), t2 = ldf(c + 2 * nu + 1);
        g00x = (double)__fsub_rn(a01, r0);
        g00y = (double)__fsub_rn(a10, m0);
        g10x = (double)__fsub_rn(r3, a00);
        g10y = (double)__fsub_rn(a11, m1);
        g01x = (double)__fsub_rn(a11, s0);
        g01y = (double)__fsub_rn(t1, a00);
        g11x = (double)__fsub_rn(s3, a10);
        g11y = (double)__fsub_rn(t2, a01);
    } else {
        cell_grad2_ref(rho, nv, nu, u0, v0, g00x, g00y);
        cell_grad2_ref(rho, nv, nu, u0 + 1, v0, g10x, g10y);
        cell_grad2_ref(rho, nv, nu, u0, v0 + 1, g01x, g01y);
        cell_grad2_ref(rho, nv, nu, u0 + 1, v0 + 1, g11x, g11y);
        const float *c = rho + v0 * nu + u0;
        a00 = ldf(c);
        a01 = ldf(c + 1);
        a10 = ldf(c + nu);
        a11 = ldf(c + nu + 1);
    }
    const double ax = dadd(g00x, dmul(fx, dsub(g10x, g00x)));
    const double bx = dadd(g01x, dmul(fx, dsub(g11x, g01x)));
    const double ay = dadd(g00y, dmul(fx, dsub(g10y, g00y)));
    const double by = dadd(g01y, dmul(fx, dsub(g11y, g01y)));
    Gx = dadd(ax, dmul(fy, dsub(bx, ax)));
    Gy = dadd(ay, dmul(fy, dsub(by, ay)));
    const double a = lerp_f32diff(a00, a01, fx);
    const double b = lerp_f32diff(a10, a11, fx);
    val = dadd(a, dmul(fy, dsub(b, a)));
}

// Same results from the quad field (hb_grad_field): q = rho at the 2x2
// corners of cell (u0, v0), qx/qy = the corners' float32 differences.
// q points at the WHOLE field (all layers, one {Q, GX, GY} record of three
// float4 per cell); `base` is the layer's first cell.  Offsets are 32-bit
// (the host checks 3 * layers*V*U < 2^32), which keeps the per-sample
// address math to a few integer ops.
struct QuadField {
    const float4 *q;
    unsigned base;
    const float4 *gy;  // split layout: the GY region (quad_gy)
};

// HB_QUAD_SPLIT=1 stores the field as two regions of the same buffer: {Q, GX}
// per cell (32 bytes, one 256-bit load for a gradient sample's first half,
// and the candidates' Q quads 32 bytes apart), then GY per cell (16 bytes).
// Same 48 bytes per cell as the interleaved {Q, GX, GY} record.
#ifndef HB_QUAD_SPLIT
#define HB_QUAD_SPLIT 0  // measured: advect 5.26 -> 5.32 ms (config 4), 33.4 -> 41.1 ms (config 5)
#endif
__host__ __device__ __forceinline__ const float4 *quad_gy(const float4 *gf, uint64_t total_cells) {
    return (HB_QUAD_SPLIT && gf) ? gf + 2 * total_cells : nullptr;
}

// float4s per quad record: {Q, GX, GY} (48 bytes).  4 pads the record to 64
// bytes (never straddles a 128-byte line; Q+GX is one 256-bit load) -- measured
// slower: advect 5.24 -> 5.31 ms on config 4, 33.5 -> 37.2 ms on config 5
#ifndef HB_QUAD_REC
#define HB_QUAD_REC 3
#endif
constexpr unsigned kQuadRec = HB_QUAD_REC;
static_assert(kQuadRec == 3 || kQuadRec == 4, "quad record: 48 or 64 bytes");

// 32 bytes (two float4) with one load; p 32-byte aligned
__device__ __forceinline__ void ldg_2x4(const float4 *p, float4 &a, float4 &b) {
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
        : "l"(p));
}

__device__ __forceinline__ void gradient2_value_quad(const QuadField &f, int nv, int nu, double x,
                                                     double y, double &Gx, double &Gy,
                                                     double &val) {
    const int u0 = clampi(floor_i(x), 0, nu - 2);
    const int v0 = clampi(floor_i(y), 0, nv - 2);
    const double fx = dsub(x, (double)u0);
    const double fy = dsub(y, (double)v0);
    const unsigned cell = f.base + (unsigned)(v0 * nu + u0);
    float4 q, dx, dy;
    if (HB_QUAD_SPLIT) {
        ldg_2x4(f.q + 2 * cell, q, dx);
        dy = __ldg(f.gy + cell);
    } else {
        const float4 *rec = f.q + kQuadRec * cell;
        if (kQuadRec == 4) {
            ldg_2x4(rec, q, dx);
        } else {
            q = __ldg(rec);
            dx = __ldg(rec + 1);
        }
        dy = __ldg(rec + 2);
    }
    // corners: .x (u0,v0)  .y (u0+1,v0)  .z (u0,v0+1)  .w (u0+1,v0+1)
    const double ax = dadd((double)dx.x, dmul(fx, dsub((double)dx.y, (double)dx.x)));
    const double bx = dadd((double)dx.z, dmul(fx, dsub((double)dx.w, (double)dx.z)));
    const double ay = dadd((double)dy.x, dmul(fx, dsub((double)dy.y, (double)dy.x)));
    const double by = dadd((double)dy.z, dmul(fx, dsub((double)dy.w, (double)dy.z)));
    Gx = dadd(ax, dmul(fy, dsub(bx, ax)));
    Gy = dadd(ay, dmul(fy, dsub(by, ay)));
    const double a = lerp_f32diff(q.x, q.y, fx);
    const double b = lerp_f32diff(q.z, q.w, fx);
    val = dadd(a, dmul(fy, dsub(b, a)));
}

// `inner`: the caller guarantees 1 <= x <= nu-2 and 1 <= y <= nv-2 (a
// clamped advection candidate), so floor() already lies in the clamp range.
template <bool inner = false>
__device__ __forceinline__ double bilinear_quad(const float4 *__restrict__ q, unsigned base,
                                                int nv, int nu, double x, double y) {
    const int u0 = inner ? floor_i(x) : clampi(floor_i(x), 0, nu - 2);
    const int v0 = inner ? floor_i(y) : clampi(floor_i(y), 0, nv - 2);
    const double fx = dsub(x, (double)u0);
    const double fy = dsub(y, (double)v0);
    const float4 c = __ldg(q + (HB_QUAD_SPLIT ? 2u : kQuadRec) * (base + (unsigned)(v0 * nu + u0)));
    const double a = lerp_f32diff(c.x, c.y, fx);
    const double b = lerp_f32diff(c.z, c.w, fx);
    return dadd(a, dmul(fy, dsub(b, a)));
}

// gradient_xy itself (bundler.gradient_at)
__device__ __forceinline__ void gradient_ref(const float *__restrict__ rho, int nv, int nu,
                                             double x, double y, double &gx, double &gy) {
    double v, Gx, Gy;
    gradient2_value_ref(rho, nv, nu, x, y, Gx, Gy, v);
    gx = dmul(0.5, Gx);
    gy = dmul(0.5, Gy);
}

// ---- DDA rasterisation of one segment (_kernels.py:58-77) ------------------
// Adds `w` to every cell of the segment's 8-connected chain; k starts at k0
// (0 for an edge's first segment, 1 otherwise: the junction cell belongs to
// the earlier segment).  A zero-length segment contributes only when k0 == 0.
// Cell = floor(x0 + (k*dx)*(1/steps) + 0.5) exactly as the reference.
// (endpoint cells already rounded: x = floor(px + 0.5))
template <typename T>
__device__ __forceinline__ void dda_splat_cells(int x0, int y0, int x1, int y1, int k0, T w,
                                                T *__restrict__ layer, int nv, int nu,
                                                int32_t *__restrict__ status) {
    const int dx = x1 - x0, dy = y1 - y0;
    const int steps = max(abs(dx), abs(dy));
    if (steps == 0) {
        if (k0 == 0) {
            if ((unsigned)x0 >= (unsigned)nu || (unsigned)y0 >= (unsigned)nv) {
                atomicOr(status, HB_STATUS_OUT_OF_BOUNDS);
                return;
            }
            atomicAdd(layer + y0 * nu + x0, w);
        }
        return;
    }
    const double inv = 1.0 / (double)steps;
    const double fx0 = (double)x0, fy0 = (double)y0;
    const bool inside = (unsigned)x0 < (unsigned)nu && (unsigned)y0 < (unsigned)nv &&
                        (unsigned)x1 < (unsigned)nu && (unsigned)y1 < (unsigned)nv;
    if (!inside) {  // error path: checked per cell, flag raised (raster.py:57-67)
        for (int k = k0; k <= steps; ++k) {
            const int u = floor_i(dadd(dadd(fx0, dmul((double)(k * dx), inv)), 0.5));
            const int v = floor_i(dadd(dadd(fy0, dmul((double)(k * dy), inv)), 0.5));
            if ((unsigned)u >= (unsigned)nu || (unsigned)v >= (unsigned)nv) {
                atomicOr(status, HB_STATUS_OUT_OF_BOUNDS);
                continue;
            }
            atomicAdd(layer + v * nu + u, w);
        }
        return;
    }
    // Every cell lies between the two (in-grid) endpoint cells, so no
    // per-cell check.  On an axis with |d| == steps the reference's
    // floor(x0 + (k*d)*(1/steps) + 0.5) is exactly x0 + sign(d)*k: (k*d)*inv
    // differs from +-k by at most k*2^-52 << 0.5.  Only the other axis needs
    // the float64 expression.  One loop for both orientations (the axes are
    // selected, not branched on), so lanes of a warp with x- and y-dominant
    // segments do not run two loops one after the other.
    const bool xdom = abs(dx) == steps;
    const int c_major = xdom ? x0 : y0;
    const int s_major = xdom ? (dx > 0 ? 1 : -1) : (dy > 0 ? 1 : -1);
    const int d_minor = xdom ? dy : dx;
    const double f_minor = xdom ? fy0 : fx0;
    (void)fx0;
    for (int k = k0; k <= steps; ++k) {
        const int major = c_major + s_major * k;
        const int minor = floor_i(dadd(dadd(f_minor, dmul((double)(k * d_minor), inv)), 0.5));
        const int u = xdom ? major : minor, v = xdom ? minor : major;
        atomicAdd(layer + v * nu + u, w);
    }
}

template <typename T>
__device__ __forceinline__ void dda_splat(double px0, double py0, double px1,
                                          double py1, int k0, T w,
                                          T *__restrict__ layer, int nv, int nu,
                                          int32_t *__restrict__ status) {
    dda_splat_cells<T>(cell_round(px0), cell_round(py0), cell_round(px1), cell_round(py1), k0, w,
                       layer, nv, nu, status);
}

// The same cell chain from integer endpoint cells already known to be inside
// the grid (the tile rasteriser replays binned records with it).
template <typename Visit>
__device__ __forceinline__ void dda_walk(int x0, int y0, int x1, int y1, int k0, Visit visit) {
    const int dx = x1 - x0, dy = y1 - y0;
    const int steps = max(abs(dx), abs(dy));
    if (steps == 0) {
        if (k0 == 0) visit(x0, y0);
        return;
    }
    const double inv = 1.0 / (double)steps;
    // one loop, axes selected (see dda_splat_cells)
    const bool xdom = abs(dx) == steps;
    const int c_major = xdom ? x0 : y0;
    const int s_major = xdom ? (dx > 0 ? 1 : -1) : (dy > 0 ? 1 : -1);
    const int d_minor = xdom ? dy : dx;
    const double f_minor = (double)(xdom ? y0 : x0);
    for (int k = k0; k <= steps; ++k) {
        const int major = c_major + s_major * k;
        const int minor = floor_i(dadd(dadd(f_minor, dmul((double)(k * d_minor), inv)), 0.5));
        visit(xdom ? major : minor, xdom ? minor : major);
    }
}

// ---- tile binning of segments (hb_splat.cu rasterises the buckets) ---------
__device__ __forceinline__ uint64_t encode_seg(int x0, int y0, int dx, int dy, int k0, int w) {
    return (uint64_t)(uint16_t)x0 | ((uint64_t)(uint16_t)y0 << 16) |
           ((uint64_t)(uint8_t)(int8_t)dx << 32) | ((uint64_t)(uint8_t)(int8_t)dy << 40) |
           ((uint64_t)(k0 & 1) << 48) | ((uint64_t)(w & 0x7fff) << 49);
}

// One segment per lane (has == false: none).  Every lane of the warp must
// call this (warp-aggregated bucket claims).  Binnable segments go to their
// tile's bucket; everything else -- census mode (no record storage), bucket
// overflow, non-unit float weights, long or out-of-grid segments -- is
// rasterised straight into the histogram exactly as before.
// first e in [0, n] with starts[e] >= v (starts is non-decreasing, starts[n] = N)
__device__ __forceinline__ int64_t lower_edge(const int64_t *__restrict__ starts, int64_t n,
                                              int64_t v) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (starts[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// Segment-key table layout: per (group, cell delta) plane, the start cells
// in 4x4 blocks of 16 consecutive entries (64 B), blocks row-major.  Keys of
// a bundle (parallel edges a few cells apart, same delta) share blocks, so
// the per-segment atomics touch far fewer L2 sectors than a row layout.
__host__ __device__ __forceinline__ int segtab_nbx(int nu) { return (nu + 3) >> 2; }
__host__ __device__ __forceinline__ int segtab_nby(int nv) { return (nv + 3) >> 2; }
__device__ __forceinline__ unsigned segtab_index(unsigned plane, int x0, int y0, int nv, int nu) {
    const unsigned nbx = (unsigned)segtab_nbx(nu), nby = (unsigned)segtab_nby(nv);
    return (((plane * nby + (unsigned)(y0 >> 2)) * nbx + (unsigned)(x0 >> 2)) << 4) +
           (unsigned)(((y0 & 3) << 2) | (x0 & 3));
}

template <typename T>
__device__ __forceinline__ void bin_or_splat_cells(bool has, int cx0, int cy0, int cx1, int cy1,
                                                   int k0, T w, int grp, T *__restrict__ hist,
                                                   int64_t plane, int nv, int nu,
                                                   int32_t *__restrict__ status,
                                                   const hb_tiles *__restrict__ tl) {
    bool direct = has;
    int tile = -1;
    uint64_t rec = 0;
    if (tl && tl->mode == 1) {  // segment-key table: one atomic per segment
        if (has) {
            const int x0 = cx0, y0 = cy0;
            const int dx = cx1 - x0, dy = cy1 - y0;
            const int H = tl->halo, iw = (int)w;
            if (k0 == 1 && dx == 0 && dy == 0) {
                direct = false;  // adds nothing (_kernels.py:67-71)
            } else if (k0 == 1 && abs(dx) <= H && abs(dy) <= H && (T)iw == w && iw >= 1 &&
                       (unsigned)x0 < (unsigned)nu && (unsigned)y0 < (unsigned)nv &&
                       (unsigned)(x0 + dx) < (unsigned)nu && (unsigned)(y0 + dy) < (unsigned)nv) {
                // delta-major key (a cell-major layout was measured slower: it
                // packs a hot cell's atomics into a few L2 slices)
                // (hb_segtab_geometry keeps the table below 2^31 entries,
                // so the index fits 32-bit arithmetic)
                const unsigned D = 2 * H + 1;
                const unsigned dir = (unsigned)grp * D * D + (unsigned)((dy + H) * D + (dx + H));
atomicAdd(tl->tab + segtab_index(dir, x0, y0, nv, nu), (unsigned)iw);
                direct = false;
            }
        }
        if (direct)
            dda_splat_cells<T>(cx0, cy0, cx1, cy1, k0, w, hist + (int64_t)grp * plane, nv, nu,
                               status);
        return;
    }
    if (has && tl) {
        const int x0 = cx0, y0 = cy0;
        const int dx = cx1 - x0, dy = cy1 - y0;
        const int iw = (int)w;
        if (dx == 0 && dy == 0 && k0 == 1) {
            direct = false;  // adds nothing (_kernels.py:67-71)
        } else if ((unsigned)x0 < (unsigned)nu && (unsigned)y0 < (unsigned)nv &&
                   (unsigned)(x0 + dx) < (unsigned)nu && (unsigned)(y0 + dy) < (unsigned)nv &&
                   abs(dx) <= tl->halo && abs(dy) <= tl->halo && (T)iw == w && iw >= 1 &&
                   iw <= 0x7fff) {
            // (|d| <= halo: every cell of the record lies in its tile's window,
            // so the flush needs no per-cell bounds check)
            tile = (grp * tl->nty + y0 / tl->tile) * tl->ntx + x0 / tl->tile;
            rec = encode_seg(x0, y0, dx, dy, k0, iw);
        }
    }
    if (tl) {
        const unsigned full = 0xffffffffu;
        const int lane = threadIdx.x & 31;
        const unsigned peers = __match_any_sync(full, tile);
        const int leader = __ffs(peers) - 1;
        int base = 0;
        if (tile >= 0 && lane == leader) base = atomicAdd(tl->fill + tile, __popc(peers));
        base = __shfl_sync(full, base, leader);
        if (tile >= 0) {
            const int slot = base + __popc(peers & ((1u << lane) - 1u));
            if (tl->rec && slot < tl->cap[tile]) {
                tl->rec[tl->off[tile] + slot] = rec;
                direct = false;
            }
        }
        if (tl->mode == 2) direct = false;  // census only: demand counted, nothing added
    }
    if (direct)
        dda_splat_cells<T>(cx0, cy0, cx1, cy1, k0, w, hist + (int64_t)grp * plane, nv, nu, status);
}

template <typename T>
__device__ __forceinline__ void bin_or_splat(bool has, double px0, double py0, double px1,
                                             double py1, int k0, T w, int grp,
                                             T *__restrict__ hist, int64_t plane, int nv, int nu,
                                             int32_t *__restrict__ status,
                                             const hb_tiles *__restrict__ tl) {
    bin_or_splat_cells<T>(has, cell_round(px0), cell_round(py0), cell_round(px1),
                          cell_round(py1), k0, w, grp, hist, plane, nv, nu, status, tl);
}

// ---- persistent warp-per-edge kernels ---------------------------------------
constexpr int kStreamBlock = 256;      // 8 warps
constexpr int kMaxStreamBlocks = 4096; // grid cap; also the metric-partials size

int device_sm_count();  // cached SM count of the current device (hb_api.cu)

// Grid for a persistent grid-stride kernel over n_edges warp work items:
// exactly the resident capacity (occupancy API, cached per kernel), never
// more blocks than there are warps' worth of edges.  For a given GPU model
// this is a pure function of n_edges, so per-block metric partials sum in a
// reproducible order.
// Resident blocks per SM, cached by (kernel address, block, dynamic smem):
// kernels sharing a signature must not share an entry.
inline int resident_blocks(const void *kernel, int block = kStreamBlock, size_t smem = 0) {
    struct Entry { const void *k; int block; size_t smem; int per_sm; };
    static Entry cache[64];
    static int n = 0;
    for (int i = 0; i < n; ++i)
        if (cache[i].k == kernel && cache[i].block == block && cache[i].smem == smem)
            return cache[i].per_sm;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem) !=
            cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    if (n < 64) cache[n++] = Entry{kernel, block, smem, per_sm};
    return per_sm;
}

template <typename Kernel>
inline unsigned persistent_grid(Kernel kernel, int64_t n_edges) {
    const int per_sm = resident_blocks(reinterpret_cast<const void *>(kernel));
    int64_t want = (n_edges + kStreamBlock / 32 - 1) / (kStreamBlock / 32);
    int64_t cap = (int64_t)device_sm_count() * per_sm;
    if (cap > kMaxStreamBlocks) cap = kMaxStreamBlocks;
    if (want > cap) want = cap;
    return (unsigned)(want < 1 ? 1 : want);
}

// One fused streaming pass over every polyline (hb_advect.cu):
//   advect (h >= 0) -> Laplacian (lap = 0 or 1 Jacobi sweep) -> write pout
//   (if non-null) -> resample count on the final points (if counts != null).
struct PolylinePass {
    const double2 *pin = nullptr;
    double2 *pout = nullptr;  // may alias pin (streaming reads run ahead of writes)
    const int64_t *starts = nullptr;
    int64_t n_edges = 0;
    const int32_t *edge_layer = nullptr;
    const float *rho = nullptr;
    const float4 *gf = nullptr;  // quad field (hb_grad_field), optional
    int nbins_field = 1;         // layers of the quad field (plane stride)
    int64_t plane = 0;
    int nv = 0, nu = 0;
    double xhi = 0.0, yhi = 0.0;  // nu - 1 - INTERIOR_MARGIN, nv - 1 - ... (exact)
    double h = -1.0, eps = 1e-8, min_step = 0.25;
    int fixed = 0;
    double factor = 0.5;
    int lap = 0;
    double delta = 1.0;
    int64_t *counts = nullptr;
    int32_t *pos = nullptr;
    unsigned long long *moved = nullptr;
    double *partials = nullptr;
};

int launch_polyline_pass(const PolylinePass &p, cudaStream_t st, const char *what);

}  // namespace hb
