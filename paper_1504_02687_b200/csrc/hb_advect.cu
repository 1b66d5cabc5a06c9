// hb_advect.cu -- gradient advection with the density-monotone adaptive step
// (_kernels.py:144-200) fused with Jacobi Laplacian smoothing
// (_kernels.py:275-296).
//
// A CTA owns P = kAdvBlock - 2H consecutive points plus H halo points on
// each side (H = Laplacian passes).  Every thread advects its point (halo
// points are advected redundantly: advection is per point), the advected
// positions are staged in shared memory, and the `passes` Jacobi sweeps run
// there (each sweep shrinks the valid region by one point), so the fused
// kernel reads 16 B and writes 16 B per point and never re-reads the
// advected positions from HBM.  Density gathers hit the L2-resident field.
#include "hb_common.cuh"

namespace hb {

constexpr int kAdvBlock = 256;
constexpr int kAdvMaxHalo = 32;

__device__ __forceinline__ bool advect_point(const float *__restrict__ rho, int nv, int nu,
                                             double x, double y, double h, double eps,
                                             double min_step, int fixed, double &ox,
                                             double &oy, double &disp) {
    const double xlo = 1.0, ylo = 1.0;  // INTERIOR_MARGIN (_kernels.py:19)
    const double xhi = dsub(dsub((double)nu, 1.0), 1.0);
    const double yhi = dsub(dsub((double)nv, 1.0), 1.0);
    double gx, gy;
    gradient_ref(rho, nv, nu, x, y, gx, gy);
    double gn = hypot_ref(gx, gy);
    if (gn < eps) gn = eps;
    const double dx = gx / gn, dy = gy / gn;
    ox = x;
    oy = y;
    if (fixed) {
        const double nx = fmin_ref(fmax_ref(dadd(x, dmul(h, dx)), xlo), xhi);
        const double ny = fmin_ref(fmax_ref(dadd(y, dmul(h, dy)), ylo), yhi);
        ox = nx;
        oy = ny;
        if (nx != x || ny != y) {
            disp = hypot_ref(dsub(nx, x), dsub(ny, y));
            return true;
        }
        return false;
    }
    const double r0 = bilinear_ref(rho, nv, nu, x, y);
    for (double m = h; m >= min_step; m = dmul(m, 0.5)) {
        const double nx = fmin_ref(fmax_ref(dadd(x, dmul(m, dx)), xlo), xhi);
        const double ny = fmin_ref(fmax_ref(dadd(y, dmul(m, dy)), ylo), yhi);
        if (bilinear_ref(rho, nv, nu, nx, ny) >= r0) {
            ox = nx;
            oy = ny;
            if (nx != x || ny != y) {
                disp = hypot_ref(dsub(nx, x), dsub(ny, y));
                return true;
            }
            return false;
        }
    }
    return false;
}

__global__ void __launch_bounds__(kAdvBlock)
advect_laplacian_kernel(const double2 *__restrict__ pin, double2 *__restrict__ pout,
                        const int64_t *__restrict__ starts, int64_t n_edges, int64_t n_pts,
                        const int32_t *__restrict__ edge_layer, const float *__restrict__ rho,
                        int64_t plane, int nv, int nu, double h, double eps,
                        double min_step, int fixed, double factor, int passes,
                        unsigned long long *__restrict__ moved,
                        double *__restrict__ partials) {
    __shared__ EdgeWindow<kAdvBlock / 2 + 2> win;
    __shared__ double2 buf[2][kAdvBlock];
    __shared__ double red_d[kAdvBlock / 32];
    __shared__ unsigned red_m[kAdvBlock / 32];
    const int H = passes;
    const int P = kAdvBlock - 2 * H;
    const int t = threadIdx.x;
    const int64_t base = (int64_t)blockIdx.x * P - H;
    const int64_t j = base + t;
    const int64_t lo = base < 0 ? 0 : base;
    const int64_t hi = base + kAdvBlock < n_pts ? base + kAdvBlock : n_pts;
    load_edge_window(win, starts, n_edges, lo, hi);

    const bool valid = j >= 0 && j < n_pts;
    bool interior = false;
    double2 p = make_double2(0.0, 0.0);
    bool mv = false;
    double d = 0.0;
    const bool own = valid && t >= H && t < H + P;
    if (valid) {
        const int k = window_edge(win, j);
        const int64_t s = win.st[k], last = win.st[k + 1] - 1;
        interior = j > s && j < last;
        p = pin[j];
        if (interior && h >= 0.0) {  // h < 0: Laplacian only (laplacian_smooth)
            const float *layer = rho + (int64_t)edge_layer[win.e0 + k] * plane;
            double ox, oy, dd = 0.0;
            mv = advect_point(layer, nv, nu, p.x, p.y, h, eps, min_step, fixed, ox, oy, dd);
            p = make_double2(ox, oy);
            d = dd;
        }
    }
    buf[0][t] = p;
    __syncthreads();
    int cur = 0;
    for (int q = 1; q <= passes; ++q) {
        double2 nx = buf[cur][t];
        if (interior && t >= q && t < kAdvBlock - q) {
            const double2 l = buf[cur][t - 1], r = buf[cur][t + 1];
            const double mx = dmul(0.5, dadd(l.x, r.x));
            const double my = dmul(0.5, dadd(l.y, r.y));
            nx = make_double2(dadd(nx.x, dmul(factor, dsub(mx, nx.x))),
                              dadd(nx.y, dmul(factor, dsub(my, nx.y))));
        }
        buf[cur ^ 1][t] = nx;
        __syncthreads();
        cur ^= 1;
    }
    if (own) pout[j] = buf[cur][t];

    // per-block metrics in a fixed order (deterministic)
    unsigned cnt = (own && mv) ? 1u : 0u;
    double dd = (own && mv) ? d : 0.0;
    for (int o = 16; o; o >>= 1) {
        cnt += __shfl_down_sync(0xffffffffu, cnt, o);
        dd = dadd(dd, __shfl_down_sync(0xffffffffu, dd, o));
    }
    if ((t & 31) == 0) {
        red_d[t >> 5] = dd;
        red_m[t >> 5] = cnt;
    }
    __syncthreads();
    if (t == 0) {
        double s = 0.0;
        unsigned long long c = 0;
        for (int w = 0; w < kAdvBlock / 32; ++w) {
            s = dadd(s, red_d[w]);
            c += red_m[w];
        }
        partials[blockIdx.x] = s;
        if (c) atomicAdd(moved, c);
    }
}

// one block, fixed summation order
__global__ void reduce_f64_kernel(const double *__restrict__ in, int64_t n,
                                  double *__restrict__ out) {
    __shared__ double sh[1024];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = dadd(s, in[i]);
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) sh[threadIdx.x] = dadd(sh[threadIdx.x], sh[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

__global__ void probe_kernel(const float *__restrict__ rho, int nv, int nu,
                             const double2 *__restrict__ xy, int64_t n,
                             double *__restrict__ value, double2 *__restrict__ grad) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double2 p = xy[i];
    if (value) value[i] = bilinear_ref(rho, nv, nu, p.x, p.y);
    if (grad) {
        double gx, gy;
        gradient_ref(rho, nv, nu, p.x, p.y, gx, gy);
        grad[i] = make_double2(gx, gy);
    }
}

}  // namespace hb

using namespace hb;

static inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

int64_t hb_advect_partials(int64_t n_pts, int lap_passes) {
    if (lap_passes < 0 || lap_passes > kAdvMaxHalo) return -1;
    const int P = kAdvBlock - 2 * lap_passes;
    return n_pts > 0 ? (n_pts + P - 1) / P : 0;
}

int hb_advect_laplacian(const double *pts_in, double *pts_out, const int64_t *starts,
                        int64_t n_edges, int64_t n_pts, const int32_t *edge_layer,
                        const float *rho, int nbins, int nv, int nu, double h, double eps,
                        double min_step, int fixed_step, double lap_factor, int lap_passes,
                        unsigned long long *moved, double *disp_partials, void *stream) {
    if (n_edges < 0 || n_pts < 0 || nbins < 1 || nv < 3 || nu < 3 || lap_passes < 0 ||
        lap_passes > kAdvMaxHalo || !moved || !disp_partials ||
        (n_pts > 0 && (!pts_in || !pts_out || !starts || !edge_layer || !rho)))
        return set_error(HB_EINVAL, "hb_advect_laplacian: bad arguments");
    if (pts_in == pts_out && n_pts > 0)
        return set_error(HB_EINVAL, "hb_advect_laplacian: pts_in and pts_out alias");
    if (n_pts == 0) return HB_OK;
    const int64_t blocks = hb_advect_partials(n_pts, lap_passes);
    advect_laplacian_kernel<<<(unsigned)blocks, kAdvBlock, 0, as_stream(stream)>>>(
        reinterpret_cast<const double2 *>(pts_in), reinterpret_cast<double2 *>(pts_out),
        starts, n_edges, n_pts, edge_layer, rho, (int64_t)nv * nu, nv, nu, h, eps, min_step,
        fixed_step, lap_factor, lap_passes, moved, disp_partials);
    return check_launch("hb_advect_laplacian");
}

int hb_reduce_f64(const double *in, int64_t n, double *out, void *stream) {
    if (n < 0 || !out || (n > 0 && !in)) return set_error(HB_EINVAL, "hb_reduce_f64: bad arguments");
    reduce_f64_kernel<<<1, 1024, 0, as_stream(stream)>>>(in, n, out);
    return check_launch("hb_reduce_f64");
}

int hb_probe(const float *rho_layer, int nv, int nu, const double *xy, int64_t n,
             double *value, double *grad, void *stream) {
    if (!rho_layer || nv < 2 || nu < 2 || n < 0 || (n > 0 && !xy))
        return set_error(HB_EINVAL, "hb_probe: bad arguments");
    if (n == 0) return HB_OK;
    probe_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(
        rho_layer, nv, nu, reinterpret_cast<const double2 *>(xy), n, value,
        reinterpret_cast<double2 *>(grad));
    return check_launch("hb_probe");
}

}  // extern "C"
