// hb_advect_flat.cu -- density-monotone adaptive-step advection
// (_kernels.py:144-200) as a flat stream of points.
//
// Advection is independent per point; only "is this point an edge endpoint"
// and "which layer" depend on the polyline structure.  So instead of a warp
// per edge (partial last chunks, endpoint lanes idle), every warp owns a
// contiguous range of 32-point tiles of the packed array and walks `starts`
// with an edge cursor: one coalesced load of the next 32 edge starts per
// tile marks the endpoints (a start at position r makes r-1 an end).
//
// The step search tests m = h, h/2, h/4, ... >= min_step in order and takes
// the first candidate whose density is >= the point's own.  A point needs ~2
// candidates on average but a warp waits for its slowest lane (5-6), so each
// lane tests only kFirst candidates; points still searching are pushed,
// with their exact state (x, y, d, rho0, next m), onto a per-warp queue in
// shared memory, and whenever 32 are waiting all lanes pop one and continue
// its search for kMore candidates (re-queueing the rare long ones).  Every
// candidate is the reference's own expression evaluated in the reference's
// order, so the accepted position is bit-identical; only the order in which
// different points finish changes (and the summation order of the
// displacement metric, as with any change of worker count).
//
// Accepted points are written in place (a point is read only by its own
// lane, before any write).  The Jacobi Laplacian, which needs both
// neighbours' advected positions, runs afterwards as its own streaming pass
// fused with the resample count (hb_advect_laplacian with h < 0).
#include "hb_common.cuh"

namespace hb {

struct AdvectFlat {
    double2 *pts = nullptr;  // in place
    const int64_t *starts = nullptr;
    int64_t n_edges = 0, n_pts = 0;
    const int32_t *edge_layer = nullptr;
    const float *rho = nullptr;
    const float4 *gf = nullptr;  // quad field (hb_grad_field) or null
    int nbins = 1;
    unsigned plane = 0;  // cells per layer; layers * plane < 2^31 (checked)
    int nv = 0, nu = 0;
    double xhi = 0.0, yhi = 0.0, h = 0.0, eps = 1e-8, min_step = 0.25;
    int fixed = 0;
    unsigned long long *moved = nullptr;
    double *partials = nullptr;
};

// Measured on config 4 (advect ms/iteration): (first, more) = (1,1) 5.43,
// (1,2) 5.49, (2,1) 5.61, (2,2) 5.69, (2,3) 5.73, (3,2) 5.82.
#ifndef HB_FLAT_FIRST
#define HB_FLAT_FIRST 1
#endif
#ifndef HB_FLAT_MORE
#define HB_FLAT_MORE 1
#endif
constexpr int kFirst = HB_FLAT_FIRST;  // candidates per point before queueing
constexpr int kMore = HB_FLAT_MORE;    // candidates per queue round
constexpr int kQCap = 64;              // < 32 waiting + 32 pushed
constexpr int kFlatWarps = kStreamBlock / 32;

struct FlatQueue {  // per warp, structure of arrays
    double x[kQCap], y[kQCap], dx[kQCap], dy[kQCap], r0[kQCap], m[kQCap];
    int i[kQCap];  // point index relative to the launch's first point
    unsigned base[kQCap];
};

template <bool QUAD>
struct FlatField {
    const float4 *q;
    const float *rho;
    int nv, nu;
    double xhi, yhi;

    // _kernels.py:176-181: clamp the candidate, bilinear density >= rho0?
    __device__ __forceinline__ bool test(unsigned base, double x, double y, double dx, double dy,
                                         double m, double r0, double &nx, double &ny) const {
        nx = clamp_ref(dadd(x, dmul(m, dx)), 1.0, xhi);
        ny = clamp_ref(dadd(y, dmul(m, dy)), 1.0, yhi);
        // 1 <= nx <= nu-2 (nu >= 3): the candidate's cell needs no clamp
        const double v = QUAD ? bilinear_quad<true>(q, base, nv, nu, nx, ny)
                              : bilinear_ref(rho + base, nv, nu, nx, ny);
        return v >= r0;
    }
};

#ifndef HB_FLAT_MINB
#define HB_FLAT_MINB 4
#endif

template <bool QUAD>
__global__ void __launch_bounds__(kStreamBlock, HB_FLAT_MINB) advect_flat_kernel(const AdvectFlat p) {
    __shared__ FlatQueue s_queue[kFlatWarps];
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    FlatQueue &q = s_queue[threadIdx.x >> 5];
    const FlatField<QUAD> fld{p.gf, p.rho, p.nv, p.nu, p.xhi, p.yhi};
    const double min_step = p.min_step;

    const int64_t gw = ((int64_t)blockIdx.x * kStreamBlock + threadIdx.x) >> 5;
    const int64_t nw = (int64_t)gridDim.x * kFlatWarps;
    // the point count is read on the device (n_pts is the buffer bound), so
    // the launch needs no host copy of the current count
    // points [starts[0], starts[n_edges]) -- an edge sub-range may start
    // anywhere -- clamped to the buffer bound n_pts
    const int64_t P_lo = p.starts[0];
    const int64_t NP = p.starts[p.n_edges] < p.n_pts ? p.starts[p.n_edges] : p.n_pts;
    const int64_t tiles = NP > P_lo ? (NP - P_lo + 31) >> 5 : 0;
    const int64_t per = (tiles + nw - 1) / nw;
    int64_t t = gw * per;
    const int64_t t_end = t + per < tiles ? t + per : tiles;

    unsigned my_moved = 0;
    double my_disp = 0.0;
    int qn = 0;  // warp-uniform queue fill

    // indices below are 32-bit and relative to P_lo (point counts < 2^31,
    // checked on the host)
    double2 *const pts_r = p.pts + P_lo;
    const int NPr = (int)(NP - P_lo);
    auto accept = [&](int i, double x, double y, double nx, double ny) {
        if (nx != x || ny != y) {  // _kernels.py:187-190
            pts_r[i] = make_double2(nx, ny);
            ++my_moved;
            my_disp = dadd(my_disp, hypot_ref(dsub(nx, x), dsub(ny, y)));
        }
    };
    // one queue round: every lane pops one waiting point (if any) and tests
    // up to `rounds` more candidates; unfinished ones are pushed back
    auto queue_round = [&](int take, int rounds) {
        const bool have = lane < take;
        const int slot = qn - take + lane;
        double x = 0.0, y = 0.0, dx = 0.0, dy = 0.0, r0 = 0.0, m = -1.0;
        int i = 0;
        unsigned base = 0;
        if (have) {
            x = q.x[slot]; y = q.y[slot]; dx = q.dx[slot]; dy = q.dy[slot];
            r0 = q.r0[slot]; m = q.m[slot]; i = q.i[slot]; base = q.base[slot];
        }
        qn -= take;
        __syncwarp();
        for (int k = 0; have && (rounds < 0 || k < rounds) && m >= min_step; ++k) {
            double nx, ny;
            if (fld.test(base, x, y, dx, dy, m, r0, nx, ny)) {
                accept(i, x, y, nx, ny);
                m = -1.0;
                break;
            }
            m = dmul(m, 0.5);
        }
        const bool pend = have && m >= min_step;
        const unsigned pm = __ballot_sync(full, pend);
        if (pend) {
            const int s = qn + __popc(pm & lt_mask);
            q.x[s] = x; q.y[s] = y; q.dx[s] = dx; q.dy[s] = dy;
            q.r0[s] = r0; q.m[s] = m; q.i[s] = i; q.base[s] = base;
        }
        qn += __popc(pm);
        __syncwarp();
    };

    if (t < t_end) {
        // edge cursor: the edge containing point 32*t (last e: starts[e] <= i0)
        int e_cur = 0;
        if (lane == 0) {
            const int64_t i0 = P_lo + t * 32;
            int64_t lo = 0, hi = p.n_edges - 1;
            while (lo < hi) {
                const int64_t mid = (lo + hi + 1) >> 1;
                if (p.starts[mid] <= i0) lo = mid; else hi = mid - 1;
            }
            e_cur = (int)lo;
        }
        e_cur = __shfl_sync(full, e_cur, 0);
        const int n_edges = (int)p.n_edges;
        int s_cur = (int)(p.starts[e_cur] - P_lo);
        // one tile of loads in flight ahead of the math
        int i = (int)t * 32 + lane;
        double2 pt_nx = i < NPr ? pts_r[i] : make_double2(0.0, 0.0);
        for (; t < t_end; ++t) {
            const int i0 = (int)t * 32;
            i = i0 + lane;
            const bool valid = i < NPr;
            const double2 pt = pt_nx;
            if (t + 1 < t_end && i + 32 < NPr) pt_nx = pts_r[i + 32];
            // edge starts strictly after i0, up to i0 + 32
            const int ek = e_cur + 1 + lane;
            const int sv = ek <= n_edges ? (int)(p.starts[ek] - P_lo) : INT_MAX;
            const int rel = sv - i0;  // >= 1
            const unsigned in_win = __ballot_sync(full, rel <= 32);
            const unsigned smask = __reduce_or_sync(full, rel <= 31 ? (1u << rel) : 0u);
            const unsigned end31 = (in_win & ~__ballot_sync(full, rel <= 31)) ? 0x80000000u : 0u;
            const unsigned emask = smask | (smask >> 1) | (s_cur == i0 ? 1u : 0u) | end31;
            unsigned base = 0;
            if (p.nbins > 1 && valid) {
                const int e = e_cur + __popc(smask & (0xffffffffu >> (31 - lane)));
                base = (unsigned)p.edge_layer[e] * p.plane;
            }
            const int nst = __popc(in_win);
            if (nst) {
                e_cur += nst;
                s_cur = __shfl_sync(full, sv, nst - 1);
            }
            const bool interior = valid && !((emask >> lane) & 1u);

            bool pend = false;
            double x = pt.x, y = pt.y, dx = 0.0, dy = 0.0, r0 = 0.0, m = -1.0;
            if (interior) {
                // _kernels.py:163-175 (G = 2*gradient, see gradient2_value_ref)
                double Gx, Gy;
                if (QUAD) {
                    gradient2_value_quad(QuadField{p.gf, base, quad_gy(p.gf, (uint64_t)p.nbins * p.plane)},
                                         p.nv, p.nu, x, y, Gx, Gy, r0);
                } else {
                    gradient2_value_ref(p.rho + base, p.nv, p.nu, x, y, Gx, Gy, r0);
                }
                const double Gn = hypot_ref(Gx, Gy);
                if (Gn < 2.0 * p.eps) {
                    dx = dmul(0.5, Gx) / p.eps;
                    dy = dmul(0.5, Gy) / p.eps;
                } else {
                    dx = Gx / Gn;
                    dy = Gy / Gn;
                }
                m = p.h;
                if (p.fixed) {  // _kernels.py:177-185: one step, always taken
                    accept(i, x, y, clamp_ref(dadd(x, dmul(m, dx)), 1.0, p.xhi),
                           clamp_ref(dadd(y, dmul(m, dy)), 1.0, p.yhi));
                    m = -1.0;
                }
                for (int k = 0; k < kFirst && m >= min_step; ++k) {
                    double nx, ny;
                    if (fld.test(base, x, y, dx, dy, m, r0, nx, ny)) {
                        accept(i, x, y, nx, ny);
                        m = -1.0;
                        break;
                    }
                    m = dmul(m, 0.5);
                }
                pend = m >= min_step;
            }
            const unsigned pm = __ballot_sync(full, pend);
            if (pm) {
                if (pend) {
                    const int s = qn + __popc(pm & lt_mask);
                    q.x[s] = x; q.y[s] = y; q.dx[s] = dx; q.dy[s] = dy;
                    q.r0[s] = r0; q.m[s] = m; q.i[s] = i; q.base[s] = base;
                }
                qn += __popc(pm);
                __syncwarp();
                while (qn >= 32) queue_round(32, kMore);
            }
        }
        // drain: the last waiting points run to completion
        while (qn > 0) queue_round(qn < 32 ? qn : 32, -1);
    }

    // per-block metrics in a fixed order (deterministic for a fixed grid)
    __shared__ double red_d[kFlatWarps];
    __shared__ unsigned red_m[kFlatWarps];
    for (int o = 16; o; o >>= 1) {
        my_moved += __shfl_down_sync(full, my_moved, o);
        my_disp = dadd(my_disp, __shfl_down_sync(full, my_disp, o));
    }
    if (lane == 0) {
        red_d[threadIdx.x >> 5] = my_disp;
        red_m[threadIdx.x >> 5] = my_moved;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double sd = 0.0;
        unsigned long long sm = 0;
        for (int w = 0; w < kFlatWarps; ++w) {
            sd = dadd(sd, red_d[w]);
            sm += red_m[w];
        }
        p.partials[blockIdx.x] = sd;
        if (sm) atomicAdd(p.moved, sm);
    }
}

}  // namespace hb

using namespace hb;

extern "C" {

int hb_advect_points(double *pts, const int64_t *starts, int64_t n_edges, int64_t n_pts,
                     const int32_t *edge_layer, const float *rho, const float *grad_field,
                     int nbins, int nv, int nu, double h, double eps, double min_step,
                     int fixed_step, unsigned long long *moved, double *disp_partials,
                     void *stream) {
    if (n_edges < 0 || n_pts < 0 || nbins < 1 || nv < 3 || nu < 3 || nv > kMaxDim ||
        nu > kMaxDim || !moved || !disp_partials || !(h >= 0.0) ||
        (n_pts > 0 && n_edges > 0 && (!pts || !starts || !edge_layer || !rho)))
        return set_error(HB_EINVAL, "hb_advect_points: bad arguments");
    if ((int64_t)nbins * nv * nu >= ((int64_t)1 << 31) ||
        (grad_field && (int64_t)kQuadRec * nbins * nv * nu >= ((int64_t)1 << 32)))
        return set_error(HB_EINVAL, "hb_advect_points: field above 2^31 cells");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(disp_partials, 0, sizeof(double) * kMaxStreamBlocks, st) != cudaSuccess)
        return check_launch("hb_advect_points", 0);
    if (n_pts == 0 || n_edges == 0) return HB_OK;
    AdvectFlat p;
    p.pts = reinterpret_cast<double2 *>(pts);
    p.starts = starts;
    p.n_edges = n_edges;
    p.n_pts = n_pts;
    p.edge_layer = edge_layer;
    p.rho = rho;
    p.gf = reinterpret_cast<const float4 *>(grad_field);
    p.nbins = nbins;
    p.plane = (unsigned)((int64_t)nv * nu);
    p.nv = nv;
    p.nu = nu;
    p.xhi = (double)(nu - 2);  // == (nu - 1.0) - 1.0 exactly (_kernels.py:158-159)
    p.yhi = (double)(nv - 2);
    p.h = h;
    p.eps = eps;
    p.min_step = min_step;
    p.fixed = fixed_step;
    p.moved = moved;
    p.partials = disp_partials;
    const int64_t tiles = (n_pts + 31) / 32;
    if (p.gf) {
        advect_flat_kernel<true><<<persistent_grid(advect_flat_kernel<true>, tiles), kStreamBlock,
                                   0, st>>>(p);
    } else {
        advect_flat_kernel<false><<<persistent_grid(advect_flat_kernel<false>, tiles),
                                    kStreamBlock, 0, st>>>(p);
    }
    return check_launch("hb_advect_points");
}

}  // extern "C"
