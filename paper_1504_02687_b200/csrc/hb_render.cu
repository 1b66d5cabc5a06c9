// hb_render.cu -- per-segment stroke widths of the renderer
// (/root/reference/pkg/src/histobundle/render.py:158-179, _segment_widths).
//
// For every point of every polyline: the layer's density at the point,
// bilinear with the reference's clamps (x into [0, nu - 1.000001], the cell
// into [0, nu - 2]), float32 corner differences promoted after the
// subtraction, clipped below at 0; a segment's width uses the mean of its two
// end densities relative to the layer peak, clipped to [0, 1], as
// w_min + (w_max - w_min) * ratio.  Linear scale only: the log scale's
// log1p stays with numpy on the host (its last-ulp behaviour is libm's).
// One thread per segment (edges are found from `starts` by binary search).
#include "hb_common.cuh"

namespace hb {

__device__ __forceinline__ double seg_density(const float *__restrict__ rho, int nv, int nu,
                                              double px, double py) {
    const double x = fmin(fmax(px, 0.0), (double)nu - 1.000001);
    const double y = fmin(fmax(py, 0.0), (double)nv - 1.000001);
    const int u0 = clampi((int)floor(x), 0, nu - 2);
    const int v0 = clampi((int)floor(y), 0, nv - 2);
    const double fx = dsub(x, (double)u0), fy = dsub(y, (double)v0);
    const float *r0 = rho + (int64_t)v0 * nu + u0, *r1 = r0 + nu;
    const double top = lerp_f32diff(r0[0], r0[1], fx);
    const double bot = lerp_f32diff(r1[0], r1[1], fx);
    const double d = dadd(top, dmul(fy, dsub(bot, top)));
    return d > 0.0 ? d : 0.0;  // np.maximum(d, 0.0)
}

__global__ void segment_widths_kernel(const double2 *__restrict__ pts,
                                      const int64_t *__restrict__ starts, int64_t n_edges,
                                      const int32_t *__restrict__ layer,
                                      const float *__restrict__ rho, int nv, int nu,
                                      const float *__restrict__ peaks, double w_min,
                                      double w_max, int want_ratio, double *__restrict__ out) {
    // segment s of edge e is output s - e (each edge has n_e - 1 segments)
    const int64_t n_seg = starts[n_edges] - n_edges;
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n_seg;
         s += (int64_t)gridDim.x * blockDim.x) {
        // edge e: the last e with starts[e] - e <= s
        int64_t lo = 0, hi = n_edges - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (starts[mid] - mid <= s) lo = mid; else hi = mid - 1;
        }
        const int64_t e = lo, j = s + e;  // point index of the segment's start
        const int b = layer ? layer[e] : 0;
        const float *rl = rho + (int64_t)b * nv * nu;
        const double peak = (double)peaks[b];
        double w;
        if (!(peak > 0.0)) {
            w = want_ratio ? 0.0 : w_min;  // render.py:162-163
        } else {
            const double2 a = pts[j], c = pts[j + 1];
            const double d = dmul(0.5, dadd(seg_density(rl, nv, nu, a.x, a.y),
                                             seg_density(rl, nv, nu, c.x, c.y)));
            double ratio = __ddiv_rn(d, peak);
            ratio = ratio < 0.0 ? 0.0 : (ratio > 1.0 ? 1.0 : ratio);  // np.clip
            w = want_ratio ? ratio : dadd(w_min, dmul(dsub(w_max, w_min), ratio));
        }
        out[s] = w;
    }
}

}  // namespace hb

using namespace hb;

extern "C" {

int hb_segment_widths(const double *pts, const int64_t *starts, int64_t n_edges,
                      const int32_t *layer, const float *rho, int nbins, int nv, int nu,
                      const float *peaks, double w_min, double w_max, int want_ratio,
                      double *out, void *stream) {
    if (n_edges < 0 || nbins < 1 || nv < 2 || nu < 2 || nv > kMaxDim || nu > kMaxDim ||
        (n_edges > 0 && (!pts || !starts || !rho || !peaks || !out)))
        return set_error(HB_EINVAL, "hb_segment_widths: bad arguments");
    if (n_edges == 0) return HB_OK;
    segment_widths_kernel<<<4 * device_sm_count(), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const double2 *>(pts), starts, n_edges, layer, rho, nv, nu, peaks, w_min,
        w_max, want_ratio, out);
    return check_launch("hb_segment_widths");
}

}  // extern "C"
