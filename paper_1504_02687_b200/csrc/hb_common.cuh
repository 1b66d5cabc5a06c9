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

// ---- persistent warp-per-edge kernels ---------------------------------------
constexpr int kStreamBlock = 256;      // 8 warps
constexpr int kMaxStreamBlocks = 4096; // grid cap; also the metric-partials size

int device_sm_count();  // cached SM count of the current device (hb_api.cu)

// Grid for a persistent grid-stride kernel over n_edges warp work items:
// exactly the resident capacity (occupancy API, cached per kernel), never
// more blocks than there are warps' worth of edges.  For a given GPU model
// this is a pure function of n_edges, so per-block metric partials sum in a
// reproducible order.
template <typename Kernel>
inline unsigned persistent_grid(Kernel kernel, int64_t n_edges) {
    static int per_sm = 0;
    if (per_sm == 0) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kStreamBlock, 0) !=
                cudaSuccess ||
            per_sm < 1)
            per_sm = 1;
    }
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
    int64_t plane = 0;
    int nv = 0, nu = 0;
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
