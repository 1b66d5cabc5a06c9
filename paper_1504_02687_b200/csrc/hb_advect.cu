// hb_advect.cu -- the fused per-polyline pass: gradient advection with the
// density-monotone adaptive step (_kernels.py:144-200), Jacobi Laplacian
// smoothing (_kernels.py:275-296) and the next iteration's resample count
// (_kernels.py:203-232), in ONE streaming read of the points.
//
// Warp per edge, persistent grid-stride over edges.  The warp walks its edge
// in 32-point chunks with a one-chunk software pipeline:
//   A(c+1) = advect(chunk c+1)          (lanes in parallel, gathers from the
//                                        L2-resident density field)
//   F(c)   = A(c) + f*(0.5*(A(j-1)+A(j+1)) - A(c))   neighbours by shuffle;
//            A(j-1) of lane 0 is a carry, A(j+1) of lane 31 is lane 0 of A(c+1)
//   write F(c); resample-count F(c) (ballot walk, carries across chunks)
// so every point is read once (16 B) and written once (16 B) plus its 4 B
// resample code, and nothing waits on a CTA barrier.
//
// Resample count: the reference walks the polyline keeping `a`, the last
// KEPT point; point j (not the last) is merged when |p_j - a| < 0.5*delta.
// Lanes first assume every predecessor is kept (g_j = |p_j - p_{j-1}|); the
// first lane b whose test fails under that assumption really is merged (all
// lanes before it were kept), lane b+1 is re-tested against the true `a`, and
// so on -- one ballot per merge, fully parallel when nothing merges, and every
// test is the reference's exact sqrt((x-ax)^2 + (y-ay)^2).  Kept points get
// pieces = 2^k (halve g while g > 1.5*delta); a warp prefix sum places them.
#include "hb_common.cuh"

namespace hb {

struct Adv {
    double2 p;
    bool moved;
    double disp;
};

// _kernels.py:163-199 for one interior point.  (A warp-cooperative variant
// that tests the remaining candidates of pending points on idle lanes was
// measured slower on B200: the shuffles cost more than the divergence; so
// was gathering two or three step candidates at once -- the kernel is
// issue-bound, not latency-bound.)
template <bool quad>
__device__ __forceinline__ Adv advect_one(const float *__restrict__ rho, const QuadField &qf,
                                          int nv, int nu,
                                          double xhi, double yhi, double2 p, double h,
                                          double eps, double min_step, int fixed) {
    Adv r{p, false, 0.0};
    const double x = p.x, y = p.y;
    const double xlo = 1.0, ylo = 1.0;  // INTERIOR_MARGIN (_kernels.py:19)
    const bool inner_grid = nu >= 3 && nv >= 3;
    // G = 2*gradient exactly, so |G| = 2*gn and G/|G| == g/gn bit for bit;
    // only the eps clamp (gn < eps <=> |G| < 2*eps) needs the scaled values
    double Gx, Gy, r0;
    if (quad)
        gradient2_value_quad(qf, nv, nu, x, y, Gx, Gy, r0);
    else
        gradient2_value_ref(rho, nv, nu, x, y, Gx, Gy, r0);
    const double Gn = hypot_ref(Gx, Gy);
    double dx, dy;
    if (Gn < 2.0 * eps) {
        dx = dmul(0.5, Gx) / eps;
        dy = dmul(0.5, Gy) / eps;
    } else {
        dx = Gx / Gn;
        dy = Gy / Gn;
    }
    double m = h;
    while (fixed || m >= min_step) {
        const double nx = clamp_ref(dadd(x, dmul(m, dx)), xlo, xhi);
        const double ny = clamp_ref(dadd(y, dmul(m, dy)), ylo, yhi);
        // xhi = nu-2, yhi = nv-2: with nu, nv >= 3 the candidate's cell needs
        // no further clamp (inner_grid is warp-uniform)
        if (fixed ||
            (quad ? (inner_grid ? bilinear_quad<true>(qf.q, qf.base, nv, nu, nx, ny)
                                : bilinear_quad(qf.q, qf.base, nv, nu, nx, ny))
                  : bilinear_ref(rho, nv, nu, nx, ny)) >= r0) {
            r.p = make_double2(nx, ny);
            if (nx != x || ny != y) {
                r.moved = true;
                r.disp = hypot_ref(dsub(nx, x), dsub(ny, y));
            }
            break;
        }
        m = dmul(m, 0.5);
    }
    return r;
}

#ifndef HB_ADV_MINB
#define HB_ADV_MINB 4
#endif
#ifndef HB_CNT_MINB
#define HB_CNT_MINB 4
#endif

template <bool ADV, bool LAP, bool COUNT, bool QUAD>
__global__ void __launch_bounds__(kStreamBlock, (ADV && COUNT) ? 3 : (ADV ? HB_ADV_MINB : (COUNT ? HB_CNT_MINB : 4)))
polyline_pass_kernel(const PolylinePass p) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    constexpr bool do_adv = ADV;
    constexpr bool do_count = COUNT;
    const double lo = 0.5 * p.delta, hi = 1.5 * p.delta;  // _kernels.py:211-212
    const double lo2 = do_count ? sqrt_lt_bound(lo) : 0.0;
    const double hi2 = do_count ? sqrt_gt_bound(hi) : 0.0;
    // xhi = nu - 1 - INTERIOR_MARGIN (_kernels.py:158-159), set by the host
    const double xhi = p.xhi, yhi = p.yhi;
    const int64_t nwarps = (int64_t)gridDim.x * (kStreamBlock / 32);
    unsigned my_moved = 0;
    double my_disp = 0.0;
    __shared__ double2 s_row[COUNT ? kStreamBlock : 1];

    int64_t e = ((int64_t)blockIdx.x * kStreamBlock + threadIdx.x) / 32;
    // the next edge's bounds are fetched one edge ahead and every chunk's raw
    // points one chunk ahead, so each warp keeps a load in flight while it
    // runs the advection math
    int64_t s_nx = 0, t_nx = 0;
    if (e < p.n_edges) { s_nx = p.starts[e]; t_nx = p.starts[e + 1]; }
    for (; e < p.n_edges; e += nwarps) {
        const int64_t s = s_nx;
        const int n = (int)(t_nx - s);
        if (e + nwarps < p.n_edges) { s_nx = p.starts[e + nwarps]; t_nx = p.starts[e + nwarps + 1]; }
        const double2 *pin = p.pin + s;
        const int64_t lbase = do_adv ? (int64_t)p.edge_layer[e] * p.plane : 0;
        const float *rho = do_adv ? p.rho + lbase : nullptr;
        constexpr bool quad = ADV && QUAD;
        QuadField qf{nullptr, 0u, nullptr};
        if (quad)
            qf = QuadField{p.gf, (unsigned)lbase,
                           quad_gy(p.gf, (uint64_t)p.nbins_field * (uint64_t)p.plane)};

        double2 cur = make_double2(0.0, 0.0);   // A(chunk c), lane = local index - c0
        double2 left = make_double2(0.0, 0.0);  // A(c0 - 1)
        double2 ka = make_double2(0.0, 0.0);    // count: last kept final point
        double2 prevf = ka;                     // count: final point c0 - 1
        int off = 0;                            // count: output index of ka
        double2 raw = lane < n ? pin[lane] : make_double2(0.0, 0.0);

        // iteration c0 stages chunk c0+32 (advect) and finalises chunk c0
        for (int c0 = -kWarp; c0 < n; c0 += kWarp) {
            const int jn = c0 + kWarp + lane;
            double2 nxt = raw;
            if (jn + kWarp < n) raw = pin[jn + kWarp];
            if (jn < n) {
                if (do_adv && jn > 0 && jn < n - 1) {
                    const Adv a = advect_one<quad>(rho, qf, p.nv, p.nu, xhi, yhi, nxt, p.h,
                                             p.eps, p.min_step, p.fixed);
                    my_moved += a.moved;
                    if (a.moved) my_disp = dadd(my_disp, a.disp);
                    nxt = a.p;
                }
            } else {
                nxt = make_double2(0.0, 0.0);
            }
            if (c0 < 0) {  // prologue: chunk 0 staged
                cur = nxt;
                ka = make_double2(__shfl_sync(full, cur.x, 0), __shfl_sync(full, cur.y, 0));
                prevf = ka;
                if (do_count && lane == 0) p.pos[s] = 0;
                continue;
            }
            const int j = c0 + lane;
            const bool valid = j < n;
            double2 f = cur;
            if constexpr (LAP) {
                double lx = __shfl_up_sync(full, cur.x, 1), ly = __shfl_up_sync(full, cur.y, 1);
                double rx = __shfl_down_sync(full, cur.x, 1), ry = __shfl_down_sync(full, cur.y, 1);
                const double n0x = __shfl_sync(full, nxt.x, 0), n0y = __shfl_sync(full, nxt.y, 0);
                if (lane == 0) { lx = left.x; ly = left.y; }
                if (lane == 31) { rx = n0x; ry = n0y; }
                if (valid && j > 0 && j < n - 1) {
                    const double mx = dmul(0.5, dadd(lx, rx));
                    const double my = dmul(0.5, dadd(ly, ry));
                    f = make_double2(dadd(cur.x, dmul(p.factor, dsub(mx, cur.x))),
                                     dadd(cur.y, dmul(p.factor, dsub(my, cur.y))));
                }
                left.x = __shfl_sync(full, cur.x, 31);
                left.y = __shfl_sync(full, cur.y, 31);
            }
            if (p.pout && valid) p.pout[s + j] = f;

            if constexpr (COUNT) {
                // the chunk's final points in a per-warp shared row: every
                // anchor broadcast below is one LDS.128 instead of 4 SHFL
                double2 *row = s_row + (threadIdx.x & ~31);
                __syncwarp();
                row[lane] = f;
                __syncwarp();
                const double2 q = lane ? row[lane - 1] : prevf;  // predecessor
                const bool part = valid && j > 0;  // local point 0 is always kept at 0
                // squared gaps; g < lo <=> g2 < lo2 exactly (see sqrt_lt_bound).
                // (A bit-parallel resolution of isolated merges was measured
                // slower: in bundles merges come in long chains.)
                const double gs = part ? dist2_ref(f.x, f.y, q.x, q.y) : 0.0;
                const bool last = (j == n - 1);
                bool kept = false;
                double gk = 0.0;
                int start = (c0 == 0) ? 1 : 0;
                // Round 1: lane `start` measures against the carried anchor
                // `ka`.  Later rounds start right after a kept lane c, so
                // ka == f[start-1] and the speculative gap gs is already the
                // true one (same operands, same rounding).
                double geff = (lane == start && part) ? dist2_ref(f.x, f.y, ka.x, ka.y) : gs;
                while (start < kWarp) {
                    // speculate: every lane's predecessor is kept
                    const bool act = part && lane >= start;
                    const unsigned m = __ballot_sync(full, act && !last && geff < lo2);
                    if (m == 0) {
                        if (act) { kept = true; gk = geff; }
                        break;
                    }
                    const int b = __ffs(m) - 1;  // first merged lane
                    if (act && lane < b) { kept = true; gk = geff; }
                    if (b > start) ka = row[b - 1];
                    // resolve the whole merge chain at once: every later lane
                    // measures against the same anchor; the first one at
                    // >= lo (or the polyline's last point) is kept
                    const double ga = (part && lane > b) ? dist2_ref(f.x, f.y, ka.x, ka.y) : 0.0;
                    const unsigned mc =
                        __ballot_sync(full, part && lane > b && (last || !(ga < lo2)));
                    if (mc == 0) break;  // chain runs past this chunk; anchor carries
                    const int c = __ffs(mc) - 1;
                    if (lane == c) { kept = true; gk = ga; }
                    ka = row[c];
                    start = c + 1;
                    geff = gs;
                }
                // while (g > hi) { g *= 0.5; pieces *= 2; }  on squared gaps:
                // g * 2^-k > hi  <=>  g2 > 4^k * hi2 (exact power-of-two scaling)
                int pieces = kept ? 1 : 0;
                const unsigned km = __ballot_sync(full, kept);
                int incl, total;
                if (!__any_sync(full, kept && gk > hi2)) {
                    // every kept point is one piece: the prefix sum is a popcount
                    incl = __popc(km & (0xffffffffu >> (31 - lane)));
                    total = __popc(km);
                } else {
                    if (kept) {
                        double t = hi2;
                        while (gk > t) { t = dmul(t, 4.0); pieces *= 2; }
                    }
                    incl = pieces;
#pragma unroll
                    for (int d = 1; d < kWarp; d <<= 1) {
                        const int t = __shfl_up_sync(full, incl, d);
                        if (lane >= d) incl += t;
                    }
                    total = __shfl_sync(full, incl, 31);
                }
                if (part) p.pos[s + j] = kept ? off + incl : -1;
                if (km) ka = row[31 - __clz(km)];
                off += total;
                prevf = row[31];
            }
            cur = nxt;
        }
        if (do_count && lane == 0) p.counts[e] = (int64_t)off + 1;
    }

    if (p.partials) {
        // per-block metrics in a fixed order (deterministic for a fixed grid)
        __shared__ double red_d[kStreamBlock / 32];
        __shared__ unsigned red_m[kStreamBlock / 32];
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
            for (int w = 0; w < kStreamBlock / 32; ++w) {
                sd = dadd(sd, red_d[w]);
                sm += red_m[w];
            }
            p.partials[blockIdx.x] = sd;
            if (sm && p.moved) atomicAdd(p.moved, sm);
        }
    }
}

template <bool ADV, bool LAP, bool COUNT>
static int launch_variant(const PolylinePass &p, cudaStream_t st, const char *what) {
    if (p.partials &&
        cudaMemsetAsync(p.partials, 0, sizeof(double) * kMaxStreamBlocks, st) != cudaSuccess)
        return check_launch(what, 0);
    if constexpr (ADV) {
        if (p.gf != nullptr) {  // quad advection field (hb_grad_field)
            const unsigned grid =
                persistent_grid(polyline_pass_kernel<ADV, LAP, COUNT, true>, p.n_edges);
            polyline_pass_kernel<ADV, LAP, COUNT, true><<<grid, kStreamBlock, 0, st>>>(p);
            return check_launch(what);
        }
    }
    const unsigned grid = persistent_grid(polyline_pass_kernel<ADV, LAP, COUNT, false>, p.n_edges);
    polyline_pass_kernel<ADV, LAP, COUNT, false><<<grid, kStreamBlock, 0, st>>>(p);
    return check_launch(what);
}

int launch_polyline_pass(const PolylinePass &p, cudaStream_t st, const char *what) {
    if (p.n_edges == 0) return HB_OK;
    const bool adv = p.h >= 0.0, lap = p.lap != 0, cnt = p.counts != nullptr;
    const int v = (adv ? 4 : 0) | (lap ? 2 : 0) | (cnt ? 1 : 0);
    switch (v) {
        case 0: return launch_variant<false, false, false>(p, st, what);
        case 1: return launch_variant<false, false, true>(p, st, what);
        case 2: return launch_variant<false, true, false>(p, st, what);
        case 3: return launch_variant<false, true, true>(p, st, what);
        case 4: return launch_variant<true, false, false>(p, st, what);
        case 5: return launch_variant<true, false, true>(p, st, what);
        case 6: return launch_variant<true, true, false>(p, st, what);
        default: return launch_variant<true, true, true>(p, st, what);
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
    const double2 q = xy[i];
    if (value) value[i] = bilinear_ref(rho, nv, nu, q.x, q.y);
    if (grad) {
        double gx, gy;
        gradient_ref(rho, nv, nu, q.x, q.y, gx, gy);
        grad[i] = make_double2(gx, gy);
    }
}

}  // namespace hb

using namespace hb;

static inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

int64_t hb_advect_partials(void) { return kMaxStreamBlocks; }

int hb_advect_laplacian(const double *pts_in, double *pts_out, const int64_t *starts,
                        int64_t n_edges, int64_t n_pts, const int32_t *edge_layer,
                        const float *rho, const float *grad_field, int nbins, int nv, int nu,
                        double h, double eps,
                        double min_step, int fixed_step, double lap_factor, int lap_passes,
                        double delta, int64_t *counts, int32_t *pos,
                        unsigned long long *moved, double *disp_partials, void *stream) {
    const bool adv = h >= 0.0;
    if (n_edges < 0 || n_pts < 0 || lap_passes < 0 || (adv && (!moved || !disp_partials)) ||
        (adv && (nbins < 1 || nv < 3 || nu < 3 || nv > kMaxDim || nu > kMaxDim ||
                 (n_edges > 0 && !edge_layer) || !rho)) ||
        (counts && (!pos || !(delta > 0))) ||
        (n_pts > 0 && (!pts_in || !pts_out || !starts)))
        return set_error(HB_EINVAL, "hb_advect_laplacian: bad arguments");
    if (adv && grad_field && (int64_t)kQuadRec * nbins * nv * nu >= ((int64_t)1 << 32))
        return set_error(HB_EINVAL, "hb_advect_laplacian: quad field above 2^32/3 cells");
    if (n_pts == 0 || n_edges == 0) return HB_OK;
    cudaStream_t st = as_stream(stream);
    PolylinePass p{};
    p.pin = reinterpret_cast<const double2 *>(pts_in);
    p.pout = reinterpret_cast<double2 *>(pts_out);
    p.starts = starts;
    p.n_edges = n_edges;
    p.edge_layer = edge_layer;
    p.rho = rho;
    p.gf = reinterpret_cast<const float4 *>(grad_field);
    p.nbins_field = nbins;
    p.plane = (int64_t)nv * nu;
    p.nv = nv;
    p.nu = nu;
    p.xhi = (double)(nu - 2);  // == (nu - 1.0) - 1.0 exactly
    p.yhi = (double)(nv - 2);
    p.h = adv ? h : -1.0;
    p.eps = eps;
    p.min_step = min_step;
    p.fixed = fixed_step;
    p.factor = lap_factor;
    p.lap = lap_passes > 0 ? 1 : 0;
    p.delta = delta;
    p.moved = moved;
    p.partials = disp_partials;
    // passes 0/1: one fused launch.  More passes: the first launch fuses the
    // first sweep, every further Jacobi sweep is an in-place streaming launch
    // (identical results: each sweep only reads the previous one), and the
    // resample count rides on the last launch.
    p.counts = lap_passes <= 1 ? counts : nullptr;
    p.pos = lap_passes <= 1 ? pos : nullptr;
    int rc = launch_polyline_pass(p, st, "hb_advect_laplacian");
    for (int q = 1; rc == HB_OK && q < lap_passes; ++q) {
        PolylinePass sweep{};
        sweep.pin = reinterpret_cast<const double2 *>(pts_out);
        sweep.pout = reinterpret_cast<double2 *>(pts_out);
        sweep.starts = starts;
        sweep.n_edges = n_edges;
        sweep.h = -1.0;
        sweep.factor = lap_factor;
        sweep.lap = 1;
        sweep.delta = delta;
        if (q == lap_passes - 1) {
            sweep.counts = counts;
            sweep.pos = pos;
        }
        rc = launch_polyline_pass(sweep, st, "hb_advect_laplacian(sweep)");
    }
    return rc;
}

int hb_reduce_f64(const double *in, int64_t n, double *out, void *stream) {
    if (n < 0 || !out || (n > 0 && !in)) return set_error(HB_EINVAL, "hb_reduce_f64: bad arguments");
    reduce_f64_kernel<<<1, 1024, 0, as_stream(stream)>>>(in, n, out);
    return check_launch("hb_reduce_f64");
}

int hb_probe(const float *rho_layer, int nv, int nu, const double *xy, int64_t n,
             double *value, double *grad, void *stream) {
    if (!rho_layer || nv < 2 || nu < 2 || nv > kMaxDim || nu > kMaxDim || n < 0 || (n > 0 && !xy))
        return set_error(HB_EINVAL, "hb_probe: bad arguments");
    if (n == 0) return HB_OK;
    probe_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(
        rho_layer, nv, nu, reinterpret_cast<const double2 *>(xy), n, value,
        reinterpret_cast<double2 *>(grad));
    return check_launch("hb_probe");
}

}  // extern "C"
