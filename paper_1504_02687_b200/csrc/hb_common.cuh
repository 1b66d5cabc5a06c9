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

// int(math.floor(x + 0.5)) -- _kernels.py:59-62
__device__ __forceinline__ int64_t cell_round(double x) {
    return (int64_t)floor(dadd(x, 0.5));
}

// sqrt((ax)^2 + (ay)^2) with the reference's association
__device__ __forceinline__ double hypot_ref(double ax, double ay) {
    return sqrt(dadd(dmul(ax, ax), dmul(ay, ay)));
}

// numba min/max on non-NaN floats
__device__ __forceinline__ double fmin_ref(double a, double b) { return a < b ? a : b; }
__device__ __forceinline__ double fmax_ref(double a, double b) { return a > b ? a : b; }

__device__ __forceinline__ float ldf(const float *p) { return __ldg(p); }

// _kernels.py:80-98 bilinear_value.  The density difference is a float32
// subtraction, promoted afterwards.
__device__ __forceinline__ double bilinear_ref(const float *__restrict__ rho,
                                               int nv, int nu, double x, double y) {
    int64_t u0 = (int64_t)floor(x);
    int64_t v0 = (int64_t)floor(y);
    u0 = u0 < 0 ? 0 : (u0 > nu - 2 ? nu - 2 : u0);
    v0 = v0 < 0 ? 0 : (v0 > nv - 2 ? nv - 2 : v0);
    double fx = dsub(x, (double)u0);
    double fy = dsub(y, (double)v0);
    const float *r0 = rho + v0 * nu + u0;
    const float *r1 = r0 + nu;
    float a00 = ldf(r0), a01 = ldf(r0 + 1), a10 = ldf(r1), a11 = ldf(r1 + 1);
    float d0 = __fsub_rn(a01, a00);
    float d1 = __fsub_rn(a11, a10);
    double a = dadd((double)a00, dmul(fx, (double)d0));
    double b = dadd((double)a10, dmul(fx, (double)d1));
    return dadd(a, dmul(fy, dsub(b, a)));
}

// _kernels.py:101-114 _cell_gradient
__device__ __forceinline__ void cell_grad_ref(const float *__restrict__ rho, int nv,
                                              int nu, int64_t u, int64_t v,
                                              double &gx, double &gy) {
    u = u < 1 ? 1 : (u > nu - 2 ? nu - 2 : u);
    v = v < 1 ? 1 : (v > nv - 2 ? nv - 2 : v);
    const float *c = rho + v * nu + u;
    float dx = __fsub_rn(ldf(c + 1), ldf(c - 1));
    float dy = __fsub_rn(ldf(c + nu), ldf(c - nu));
    gx = dmul(0.5, (double)dx);
    gy = dmul(0.5, (double)dy);
}

// _kernels.py:117-141 gradient_xy
__device__ __forceinline__ void gradient_ref(const float *__restrict__ rho, int nv,
                                             int nu, double x, double y,
                                             double &gx, double &gy) {
    int64_t u0 = (int64_t)floor(x);
    int64_t v0 = (int64_t)floor(y);
    u0 = u0 < 0 ? 0 : (u0 > nu - 2 ? nu - 2 : u0);
    v0 = v0 < 0 ? 0 : (v0 > nv - 2 ? nv - 2 : v0);
    double fx = dsub(x, (double)u0);
    double fy = dsub(y, (double)v0);
    double g00x, g00y, g10x, g10y, g01x, g01y, g11x, g11y;
    cell_grad_ref(rho, nv, nu, u0, v0, g00x, g00y);
    cell_grad_ref(rho, nv, nu, u0 + 1, v0, g10x, g10y);
    cell_grad_ref(rho, nv, nu, u0, v0 + 1, g01x, g01y);
    cell_grad_ref(rho, nv, nu, u0 + 1, v0 + 1, g11x, g11y);
    double ax = dadd(g00x, dmul(fx, dsub(g10x, g00x)));
    double bx = dadd(g01x, dmul(fx, dsub(g11x, g01x)));
    double ay = dadd(g00y, dmul(fx, dsub(g10y, g00y)));
    double by = dadd(g01y, dmul(fx, dsub(g11y, g01y)));
    gx = dadd(ax, dmul(fy, dsub(bx, ax)));
    gy = dadd(ay, dmul(fy, dsub(by, ay)));
}

// ---- DDA rasterisation of one segment (_kernels.py:58-77) ------------------
// Adds `w` to every cell of the segment's 8-connected chain; k starts at k0
// (0 for an edge's first segment, 1 otherwise: the junction cell belongs to
// the earlier segment).  A zero-length segment contributes only when k0 == 0.
template <typename T>
__device__ __forceinline__ void dda_splat(double px0, double py0, double px1,
                                          double py1, int k0, T w,
                                          T *__restrict__ layer, int nv, int nu,
                                          int32_t *__restrict__ status) {
    const int64_t x0 = cell_round(px0), y0 = cell_round(py0);
    const int64_t x1 = cell_round(px1), y1 = cell_round(py1);
    const int64_t dx = x1 - x0, dy = y1 - y0;
    const int64_t adx = dx < 0 ? -dx : dx, ady = dy < 0 ? -dy : dy;
    const int64_t steps = adx > ady ? adx : ady;
    if (steps == 0) {
        if (k0 == 0) {
            if (x0 < 0 || x0 >= nu || y0 < 0 || y0 >= nv) {
                atomicOr(status, HB_STATUS_OUT_OF_BOUNDS);
                return;
            }
            atomicAdd(layer + y0 * nu + x0, w);
        }
        return;
    }
    const double inv = 1.0 / (double)steps;
    const double fx0 = (double)x0, fy0 = (double)y0;
    for (int64_t k = k0; k <= steps; ++k) {
        int64_t u = (int64_t)floor(dadd(dadd(fx0, dmul((double)(k * dx), inv)), 0.5));
        int64_t v = (int64_t)floor(dadd(dadd(fy0, dmul((double)(k * dy), inv)), 0.5));
        if (u < 0 || u >= nu || v < 0 || v >= nv) {
            atomicOr(status, HB_STATUS_OUT_OF_BOUNDS);
            continue;
        }
        atomicAdd(layer + v * nu + u, w);
    }
}

// ---- edge window: map a contiguous point range to its edges ---------------
// Largest e in [0, n_edges) with starts[e] <= p (p < starts[n_edges]).
// Warp-cooperative 32-ary search; all lanes return the same value.
__device__ __forceinline__ int64_t warp_find_edge(const int64_t *__restrict__ starts,
                                                  int64_t n_edges, int64_t p) {
    const int lane = threadIdx.x & 31;
    int64_t lo = 0, hi = n_edges;  // answer in [lo, hi)
    while (hi - lo > 32) {
        int64_t step = (hi - lo + 31) / 32;
        int64_t idx = lo + (int64_t)lane * step;
        bool ok = idx < hi && __ldg(starts + idx) <= p;
        unsigned m = __ballot_sync(0xffffffffu, ok);
        int last = 31 - __clz(m);  // lane 0 is always ok (starts[lo] <= p)
        lo = lo + (int64_t)last * step;
        int64_t nhi = lo + step;
        hi = nhi < hi ? nhi : hi;
    }
    int64_t idx = lo + lane;
    bool ok = idx < hi && __ldg(starts + idx) <= p;
    unsigned m = __ballot_sync(0xffffffffu, ok);
    return lo + (31 - __clz(m));
}

// A block's view of the edges overlapping points [lo, hi).  `st` holds
// starts[e0 .. e0+cnt] (cnt+1 entries).  Capacity: a range of L points meets
// at most L/2 + 1 edges because every polyline has >= 2 points.
template <int CAP>
struct EdgeWindow {
    int64_t e0;
    int cnt;
    int64_t st[CAP + 1];
};

template <int CAP>
__device__ void load_edge_window(EdgeWindow<CAP> &w, const int64_t *__restrict__ starts,
                                 int64_t n_edges, int64_t lo, int64_t hi) {
    if (threadIdx.x < 32) {
        int64_t e0 = warp_find_edge(starts, n_edges, lo);
        if (threadIdx.x == 0) w.e0 = e0;
    }
    __syncthreads();
    const int64_t e0 = w.e0;
    int64_t avail = n_edges - e0;  // edges e0..n_edges-1
    int cnt = (int)(avail < CAP ? avail : CAP);
    for (int i = threadIdx.x; i <= cnt; i += blockDim.x) w.st[i] = __ldg(starts + e0 + i);
    if (threadIdx.x == 0) w.cnt = cnt;
    __syncthreads();
    (void)hi;
}

// local edge index k with st[k] <= p < st[k+1]
template <int CAP>
__device__ __forceinline__ int window_edge(const EdgeWindow<CAP> &w, int64_t p) {
    int lo = 0, hi = w.cnt;  // st[lo] <= p, answer in [lo, hi)
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (w.st[mid] <= p) lo = mid; else hi = mid;
    }
    return lo;
}

}  // namespace hb
