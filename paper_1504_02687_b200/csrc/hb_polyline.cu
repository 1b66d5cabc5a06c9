// hb_polyline.cu -- polyline kernels: initial sampling, directed offset,
// histogram splat, resample count / scan / emit(+splat).
//
// Data layout: packed (N,2) float64 points (double2 per point, 16 B), edge
// offsets `starts` (E+1) int64.  Point-parallel kernels give each CTA a
// contiguous point range and recover the edges it touches with one warp
// search + a shared-memory window of `starts` (hb_common.cuh); the resample
// count, whose merge rule is a sequential walk, runs one warp per edge and
// resolves the walk with ballots (see resample_count_kernel).
#include <cub/device/device_scan.cuh>

#include "hb_common.cuh"

namespace hb {

// ---------------------------------------------------------------------------
// _kernels.fill_samples (_kernels.py:22-43): one warp per edge.
__global__ void sample_fill_kernel(const double2 *__restrict__ src,
                                   const double2 *__restrict__ dst,
                                   const int64_t *__restrict__ starts,
                                   int64_t n_edges, double2 *__restrict__ out) {
    const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
    const int lane = threadIdx.x & 31;
    if (e >= n_edges) return;
    const int64_t s = starts[e];
    const int64_t m = starts[e + 1] - s - 1;
    const double2 a = src[e], b = dst[e];
    const double dx = dsub(b.x, a.x), dy = dsub(b.y, a.y);
    for (int64_t k = 1 + lane; k < m; k += kWarp) {
        const double t = (double)k / (double)m;
        out[s + k] = make_double2(dadd(a.x, dmul(t, dx)), dadd(a.y, dmul(t, dy)));
    }
    if (lane == 0) {
        out[s] = a;
        out[s + m] = b;
    }
}

// bundler.py:92-106 (per-edge displacement precomputed on the host)
__global__ void offset_kernel(double2 *__restrict__ pts,
                              const int64_t *__restrict__ starts, int64_t n_edges,
                              const double2 *__restrict__ disp) {
    const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
    const int lane = threadIdx.x & 31;
    if (e >= n_edges) return;
    const int64_t s = starts[e], t = starts[e + 1] - 1;
    const double2 d = disp[e];
    for (int64_t j = s + 1 + lane; j < t; j += kWarp) {
        double2 p = pts[j];
        pts[j] = make_double2(dadd(p.x, d.x), dadd(p.y, d.y));
    }
}

// _materialize (bundler.py:152-163): world = p*cell + origin (multiply, then
// add), first/last point of each edge pinned to the node positions.
__global__ void to_world_kernel(const double2 *__restrict__ pts,
                                const int64_t *__restrict__ starts, int64_t n_edges,
                                double ox, double oy, double cell,
                                const double2 *__restrict__ src_world,
                                const double2 *__restrict__ dst_world,
                                double2 *__restrict__ out) {
    const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
    const int lane = threadIdx.x & 31;
    if (e >= n_edges) return;
    const int64_t s = starts[e], t = starts[e + 1] - 1;
    for (int64_t j = s + lane; j <= t; j += kWarp) {
        double2 w;
        if (j == s && src_world) {
            w = src_world[e];
        } else if (j == t && dst_world) {
            w = dst_world[e];
        } else {
            const double2 p = pts[j];
            w = make_double2(dadd(dmul(p.x, cell), ox), dadd(dmul(p.y, cell), oy));
        }
        out[j] = w;
    }
}

// ---------------------------------------------------------------------------
// accumulate (_kernels.py:46-77): thread per segment end point.  A CTA owns
// kSplatItems*kSplatBlock consecutive points; point j (not an edge's first)
// rasterises segment (j-1, j).
constexpr int kSplatBlock = 256;
constexpr int kSplatItems = 4;
constexpr int kSplatSpan = kSplatBlock * kSplatItems;

template <typename T>
__global__ void __launch_bounds__(kSplatBlock)
splat_kernel(const double2 *__restrict__ pts, const int64_t *__restrict__ starts,
             int64_t n_edges, int64_t n_pts, const int32_t *__restrict__ group,
             const T *__restrict__ weight, T *__restrict__ hist, int64_t plane,
             int nv, int nu, int32_t *__restrict__ status) {
    __shared__ EdgeWindow<kSplatSpan / 2 + 2> win;
    const int64_t lo = (int64_t)blockIdx.x * kSplatSpan;
    const int64_t hi = lo + kSplatSpan < n_pts ? lo + kSplatSpan : n_pts;
    load_edge_window(win, starts, n_edges, lo, hi);
#pragma unroll 1
    for (int it = 0; it < kSplatItems; ++it) {
        const int64_t j = lo + it * kSplatBlock + threadIdx.x;
        if (j >= hi) break;
        const int k = window_edge(win, j);
        const int64_t s = win.st[k];
        if (j == s) continue;
        const int64_t e = win.e0 + k;
        const double2 a = pts[j - 1], b = pts[j];
        const T w = weight ? weight[e] : T(1);
        dda_splat<T>(a.x, a.y, b.x, b.y, (j - 1 == s) ? 0 : 1, w,
                     hist + (int64_t)group[e] * plane, nv, nu, status);
    }
}

// ---------------------------------------------------------------------------
// resample_count (_kernels.py:203-232), one warp per edge.
//
// The reference walks the polyline keeping `a`, the last KEPT point; point j
// (not the last) is merged when |p_j - a| < 0.5*delta.  The warp takes 32
// points at a time and first assumes every predecessor is kept
// (g_j = |p_j - p_{j-1}|).  The first lane b whose test fails under that
// assumption really is merged (all lanes before it were kept, so their
// predecessors were right); lane b+1 is then re-tested against the true `a`
// and the process repeats from there.  Each repeat costs one ballot, so the
// common case (no merges) is fully parallel, and the arithmetic of every
// test is exactly the reference's sqrt((x-ax)^2 + (y-ay)^2).  Kept points get
// pieces = 2^k (halve g while g > 1.5*delta) and a warp prefix sum assigns
// their output positions.
__global__ void resample_count_kernel(const double2 *__restrict__ pts,
                                      const int64_t *__restrict__ starts,
                                      int64_t n_edges, double lo, double hi,
                                      int64_t *__restrict__ counts,
                                      int32_t *__restrict__ pos) {
    const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
    const int lane = threadIdx.x & 31;
    if (e >= n_edges) return;
    const unsigned full = 0xffffffffu;
    const int64_t s = starts[e];
    const int64_t n = starts[e + 1] - s;
    double2 a = pts[s];
    double2 prev = a;  // p_{c0-1}
    int64_t off = 0;   // output index of `a`
    if (lane == 0) pos[s] = 0;
    for (int64_t c0 = 1; c0 < n; c0 += kWarp) {
        const int64_t j = c0 + lane;
        const bool valid = j < n;
        const double2 p = valid ? pts[s + j] : make_double2(0.0, 0.0);
        double qx = __shfl_up_sync(full, p.x, 1);
        double qy = __shfl_up_sync(full, p.y, 1);
        if (lane == 0) { qx = prev.x; qy = prev.y; }
        const double gs = valid ? hypot_ref(dsub(p.x, qx), dsub(p.y, qy)) : 0.0;
        const bool last = (j == n - 1);
        bool kept = false;
        double gk = 0.0;
        int start = 0;
        while (start < kWarp) {
            double geff = gs;
            if (lane == start && valid) geff = hypot_ref(dsub(p.x, a.x), dsub(p.y, a.y));
            const bool act = valid && lane >= start;
            const unsigned m = __ballot_sync(full, act && !last && geff < lo);
            if (m == 0) {
                if (act) { kept = true; gk = geff; }
                break;
            }
            const int b = __ffs(m) - 1;
            if (act && lane < b) { kept = true; gk = geff; }
            if (b > start) {
                a.x = __shfl_sync(full, p.x, b - 1);
                a.y = __shfl_sync(full, p.y, b - 1);
            }
            start = b + 1;
        }
        int64_t pieces = 0;
        if (kept) {
            double g = gk;
            pieces = 1;
            while (g > hi) { g = dmul(g, 0.5); pieces *= 2; }
        }
        int64_t incl = pieces;
#pragma unroll
        for (int d = 1; d < kWarp; d <<= 1) {
            int64_t t = __shfl_up_sync(full, incl, d);
            if (lane >= d) incl += t;
        }
        if (valid) pos[s + j] = kept ? (int32_t)(off + incl) : -1;
        const unsigned km = __ballot_sync(full, kept);
        if (km) {
            const int lk = 31 - __clz(km);
            a.x = __shfl_sync(full, p.x, lk);
            a.y = __shfl_sync(full, p.y, lk);
        }
        off += __shfl_sync(full, incl, 31);
        prev.x = __shfl_sync(full, p.x, 31);
        prev.y = __shfl_sync(full, p.y, 31);
    }
    if (lane == 0) counts[e] = off + 1;
}

// ---------------------------------------------------------------------------
// resample_emit (_kernels.py:235-272) + accumulate of the new polylines.
// Thread per OLD point j: a kept point with output index pos[j] emits
// pieces-1 inserted points a + (k/pieces)(x - a) and itself, where a is the
// previous kept point (pieces = pos[j] - pos[a]), and rasterises the pieces
// output segments that end at them.
__global__ void __launch_bounds__(kSplatBlock)
emit_kernel(const double2 *__restrict__ pts, const int64_t *__restrict__ starts,
            int64_t n_edges, int64_t n_pts, const int32_t *__restrict__ pos,
            const int64_t *__restrict__ new_starts, double2 *__restrict__ out,
            const int32_t *__restrict__ group, const int32_t *__restrict__ weight,
            int32_t *__restrict__ hist, int64_t plane, int nv, int nu,
            int32_t *__restrict__ status) {
    __shared__ EdgeWindow<kSplatSpan / 2 + 2> win;
    const int64_t lo = (int64_t)blockIdx.x * kSplatSpan;
    const int64_t hi = lo + kSplatSpan < n_pts ? lo + kSplatSpan : n_pts;
    load_edge_window(win, starts, n_edges, lo, hi);
#pragma unroll 1
    for (int it = 0; it < kSplatItems; ++it) {
        const int64_t j = lo + it * kSplatBlock + threadIdx.x;
        if (j >= hi) break;
        const int pj = pos[j];
        if (pj < 0) continue;
        const int k = window_edge(win, j);
        const int64_t s = win.st[k];
        const int64_t e = win.e0 + k;
        const double2 x = pts[j];
        double2 *o = out + new_starts[e];
        if (j == s) {
            o[0] = x;
            continue;
        }
        int64_t i = j - 1;
        int pi;
        while ((pi = pos[i]) < 0) --i;
        const double2 a = pts[i];
        const int pieces = pj - pi;
        const double ddx = dsub(x.x, a.x), ddy = dsub(x.y, a.y);
        int32_t *layer = hist ? hist + (int64_t)group[e] * plane : nullptr;
        const int32_t w = weight ? weight[e] : 1;
        double2 q0 = a;
        for (int kk = 1; kk <= pieces; ++kk) {
            double2 q;
            if (kk < pieces) {
                const double t = (double)kk / (double)pieces;
                q = make_double2(dadd(a.x, dmul(t, ddx)), dadd(a.y, dmul(t, ddy)));
            } else {
                q = x;
            }
            o[pi + kk] = q;
            if (layer)
                dda_splat<int32_t>(q0.x, q0.y, q.x, q.y, (pi + kk - 1 == 0) ? 0 : 1, w,
                                   layer, nv, nu, status);
            q0 = q;
        }
    }
}

}  // namespace hb

using namespace hb;

static inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

static inline unsigned warp_blocks(int64_t n_items, int threads) {
    return (unsigned)((n_items * kWarp + threads - 1) / threads);
}

extern "C" {

int hb_sample_fill(const double *src, const double *dst, const int64_t *starts,
                   int64_t n_edges, double *pts, void *stream) {
    if (n_edges < 0 || (n_edges > 0 && (!src || !dst || !starts || !pts)))
        return set_error(HB_EINVAL, "hb_sample_fill: bad arguments");
    if (n_edges == 0) return HB_OK;
    sample_fill_kernel<<<warp_blocks(n_edges, 256), 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const double2 *>(src), reinterpret_cast<const double2 *>(dst),
        starts, n_edges, reinterpret_cast<double2 *>(pts));
    return check_launch("hb_sample_fill");
}

int hb_offset(double *pts, const int64_t *starts, int64_t n_edges, const double *disp,
              void *stream) {
    if (n_edges < 0 || (n_edges > 0 && (!pts || !starts || !disp)))
        return set_error(HB_EINVAL, "hb_offset: bad arguments");
    if (n_edges == 0) return HB_OK;
    offset_kernel<<<warp_blocks(n_edges, 256), 256, 0, as_stream(stream)>>>(
        reinterpret_cast<double2 *>(pts), starts, n_edges,
        reinterpret_cast<const double2 *>(disp));
    return check_launch("hb_offset");
}

int hb_to_world(const double *pts, const int64_t *starts, int64_t n_edges, double origin_x,
                double origin_y, double cell, const double *src_world,
                const double *dst_world, double *out, void *stream) {
    if (n_edges < 0 || (n_edges > 0 && (!pts || !starts || !out)))
        return set_error(HB_EINVAL, "hb_to_world: bad arguments");
    if (n_edges == 0) return HB_OK;
    to_world_kernel<<<warp_blocks(n_edges, 256), 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const double2 *>(pts), starts, n_edges, origin_x, origin_y, cell,
        reinterpret_cast<const double2 *>(src_world), reinterpret_cast<const double2 *>(dst_world),
        reinterpret_cast<double2 *>(out));
    return check_launch("hb_to_world");
}

int hb_splat(const double *pts, const int64_t *starts, int64_t n_edges, int64_t n_pts,
             const int32_t *group, const int32_t *weight, int32_t *counts, int nbins,
             int nv, int nu, int32_t *status, void *stream) {
    if (n_edges < 0 || n_pts < 0 || nbins < 1 || nv < 1 || nu < 1 || !counts || !status ||
        (n_edges > 0 && (!pts || !starts || !group)))
        return set_error(HB_EINVAL, "hb_splat: bad arguments");
    if (n_edges == 0 || n_pts == 0) return HB_OK;
    const unsigned blocks = (unsigned)((n_pts + kSplatSpan - 1) / kSplatSpan);
    splat_kernel<int32_t><<<blocks, kSplatBlock, 0, as_stream(stream)>>>(
        reinterpret_cast<const double2 *>(pts), starts, n_edges, n_pts, group, weight,
        counts, (int64_t)nv * nu, nv, nu, status);
    return check_launch("hb_splat");
}

int hb_splat_f32(const double *pts, const int64_t *starts, int64_t n_edges, int64_t n_pts,
                 const int32_t *group, const float *weight, float *hist, int nbins, int nv,
                 int nu, int32_t *status, void *stream) {
    if (n_edges < 0 || n_pts < 0 || nbins < 1 || nv < 1 || nu < 1 || !hist || !status ||
        (n_edges > 0 && (!pts || !starts || !group)))
        return set_error(HB_EINVAL, "hb_splat_f32: bad arguments");
    if (n_edges == 0 || n_pts == 0) return HB_OK;
    const unsigned blocks = (unsigned)((n_pts + kSplatSpan - 1) / kSplatSpan);
    splat_kernel<float><<<blocks, kSplatBlock, 0, as_stream(stream)>>>(
        reinterpret_cast<const double2 *>(pts), starts, n_edges, n_pts, group, weight, hist,
        (int64_t)nv * nu, nv, nu, status);
    return check_launch("hb_splat_f32");
}

int hb_resample_count(const double *pts, const int64_t *starts, int64_t n_edges,
                      double delta, int64_t *counts, int32_t *pos, void *stream) {
    if (n_edges < 0 || !(delta > 0) || (n_edges > 0 && (!pts || !starts || !counts || !pos)))
        return set_error(HB_EINVAL, "hb_resample_count: bad arguments");
    if (n_edges == 0) return HB_OK;
    // lo/hi exactly as _kernels.py:211-212
    const double lo = 0.5 * delta, hi = 1.5 * delta;
    resample_count_kernel<<<warp_blocks(n_edges, 256), 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const double2 *>(pts), starts, n_edges, lo, hi, counts, pos);
    return check_launch("hb_resample_count");
}

size_t hb_scan_workspace_bytes(int64_t n_edges) {
    size_t bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, bytes, (const int64_t *)nullptr,
                                  (int64_t *)nullptr, (int)(n_edges > 0 ? n_edges : 1));
    return bytes + 256;
}

int hb_scan_counts(const int64_t *counts, int64_t n_edges, int64_t *new_starts,
                   void *workspace, size_t workspace_bytes, void *stream) {
    if (n_edges < 0 || n_edges > 0x7fffffff || !new_starts || (n_edges > 0 && !counts))
        return set_error(HB_EINVAL, "hb_scan_counts: bad arguments");
    cudaStream_t st = as_stream(stream);
    if (cudaMemsetAsync(new_starts, 0, sizeof(int64_t), st) != cudaSuccess)
        return check_launch("hb_scan_counts(memset)", 0);
    if (n_edges == 0) return HB_OK;
    size_t need = 0;
    cub::DeviceScan::InclusiveSum(nullptr, need, counts, new_starts + 1, (int)n_edges, st);
    if (!workspace || workspace_bytes < need)
        return set_error(HB_EINVAL, "hb_scan_counts: workspace %zu < %zu bytes",
                         workspace_bytes, need);
    cub::DeviceScan::InclusiveSum(workspace, need, counts, new_starts + 1, (int)n_edges, st);
    return check_launch("hb_scan_counts", 2);
}

int hb_resample_emit(const double *pts, const int64_t *starts, int64_t n_edges,
                     int64_t n_pts, const int32_t *pos, const int64_t *new_starts,
                     double *out, const int32_t *group, const int32_t *weight,
                     int32_t *counts, int nv, int nu, int32_t *status, void *stream) {
    if (n_edges < 0 || n_pts < 0 || (n_edges > 0 && (!pts || !starts || !pos || !new_starts || !out)) ||
        (counts && (!group || !status || nv < 1 || nu < 1)))
        return set_error(HB_EINVAL, "hb_resample_emit: bad arguments");
    if (n_edges == 0 || n_pts == 0) return HB_OK;
    const unsigned blocks = (unsigned)((n_pts + kSplatSpan - 1) / kSplatSpan);
    emit_kernel<<<blocks, kSplatBlock, 0, as_stream(stream)>>>(
        reinterpret_cast<const double2 *>(pts), starts, n_edges, n_pts, pos, new_starts,
        reinterpret_cast<double2 *>(out), group, weight, counts, (int64_t)nv * nu, nv, nu,
        status);
    return check_launch("hb_resample_emit");
}

}  // extern "C"
