/*
 * hb_oracle.c -- CPU ORACLE for the bundling iteration.  TEST INFRASTRUCTURE.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * the reported CPU baseline.  The product path (paper_1504_02687_b200) never
 * links or calls it.
 *
 * Each function restates one numba kernel / numpy routine of the reference
 * package (/root/reference/pkg/src/histobundle) operation for operation, so
 * the float64 results are bit-identical to the reference:
 *   - compiled with -ffp-contract=off (numba does not contract a*b+c into
 *     FMA, finding 3),
 *   - float32 differences of density values are taken in float32 before
 *     promotion (numba types rho[i]-rho[j] as float32),
 *   - rounding to a cell is floor(x + 0.5).
 * Parity of this file with the reference is pinned by tests/test_oracle.py
 * against the tests/golden fixtures, which tests/golden/make_golden.py produced by
 * running the reference itself (numba 0.65.0, numpy 2.3.5).
 *
 * Edge-range arguments (e_lo, e_hi) mirror the reference's partitioned
 * kernels (_kernels.py:1-6); the Python driver (oracle/oracle.py) runs them
 * on threads exactly like _parallel.map_partitions.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define HB_ORACLE_API __attribute__((visibility("default")))

/* _kernels.py:22-43 fill_samples */
HB_ORACLE_API void orc_fill_samples(const double *src, const double *dst,
                                    const int64_t *starts, int64_t n_edges,
                                    double *out) {
    for (int64_t e = 0; e < n_edges; ++e) {
        int64_t s = starts[e];
        int64_t m = starts[e + 1] - s - 1;
        double x0 = src[2 * e], y0 = src[2 * e + 1];
        double dx = dst[2 * e] - x0, dy = dst[2 * e + 1] - y0;
        for (int64_t k = 1; k < m; ++k) {
            double t = (double)k / (double)m;
            out[2 * (s + k)] = x0 + t * dx;
            out[2 * (s + k) + 1] = y0 + t * dy;
        }
        out[2 * s] = x0;
        out[2 * s + 1] = y0;
        out[2 * (s + m)] = dst[2 * e];
        out[2 * (s + m) + 1] = dst[2 * e + 1];
    }
}

static inline int64_t cell_of(double x) { return (int64_t)floor(x + 0.5); }

/* _kernels.py:46-77 accumulate: every rasterised cell of edge e gets
 * layer_w[e, l] on every layer l (float32 accumulation). */
HB_ORACLE_API void orc_accumulate(const double *pts, const int64_t *starts,
                                  const float *layer_w, int nbins, int nv,
                                  int nu, float *out, int64_t e_lo,
                                  int64_t e_hi) {
    const int64_t plane = (int64_t)nv * nu;
    for (int64_t e = e_lo; e < e_hi; ++e) {
        int64_t s = starts[e];
        int64_t n = starts[e + 1] - s;
        const float *w = layer_w + e * nbins;
        for (int64_t j = 0; j < n - 1; ++j) {
            int64_t x0 = cell_of(pts[2 * (s + j)]);
            int64_t y0 = cell_of(pts[2 * (s + j) + 1]);
            int64_t x1 = cell_of(pts[2 * (s + j + 1)]);
            int64_t y1 = cell_of(pts[2 * (s + j + 1) + 1]);
            int64_t dx = x1 - x0, dy = y1 - y0;
            int64_t adx = dx < 0 ? -dx : dx, ady = dy < 0 ? -dy : dy;
            int64_t steps = adx > ady ? adx : ady;
            int64_t k0 = (j == 0) ? 0 : 1;
            if (steps == 0) {
                if (k0 == 0)
                    for (int l = 0; l < nbins; ++l)
                        out[l * plane + y0 * nu + x0] += w[l];
                continue;
            }
            double inv = 1.0 / (double)steps;
            for (int64_t k = k0; k <= steps; ++k) {
                int64_t u = (int64_t)floor((double)x0 + (double)(k * dx) * inv + 0.5);
                int64_t v = (int64_t)floor((double)y0 + (double)(k * dy) * inv + 0.5);
                for (int l = 0; l < nbins; ++l)
                    out[l * plane + v * nu + u] += w[l];
            }
        }
    }
}

/* Same rasterisation, integer per-group counts: out[group[e]] += weight[e].
 * Equals orc_accumulate with an identity layer_w whenever the float sums are
 * exact. */
HB_ORACLE_API void orc_accumulate_counts(const double *pts,
                                         const int64_t *starts,
                                         const int64_t *group,
                                         const int32_t *weight, int nv, int nu,
                                         int32_t *out, int64_t e_lo,
                                         int64_t e_hi) {
    const int64_t plane = (int64_t)nv * nu;
    for (int64_t e = e_lo; e < e_hi; ++e) {
        int64_t s = starts[e];
        int64_t n = starts[e + 1] - s;
        int32_t *o = out + group[e] * plane;
        int32_t w = weight ? weight[e] : 1;
        for (int64_t j = 0; j < n - 1; ++j) {
            int64_t x0 = cell_of(pts[2 * (s + j)]);
            int64_t y0 = cell_of(pts[2 * (s + j) + 1]);
            int64_t x1 = cell_of(pts[2 * (s + j + 1)]);
            int64_t y1 = cell_of(pts[2 * (s + j + 1) + 1]);
            int64_t dx = x1 - x0, dy = y1 - y0;
            int64_t adx = dx < 0 ? -dx : dx, ady = dy < 0 ? -dy : dy;
            int64_t steps = adx > ady ? adx : ady;
            int64_t k0 = (j == 0) ? 0 : 1;
            if (steps == 0) {
                if (k0 == 0) o[y0 * nu + x0] += w;
                continue;
            }
            double inv = 1.0 / (double)steps;
            for (int64_t k = k0; k <= steps; ++k) {
                int64_t u = (int64_t)floor((double)x0 + (double)(k * dx) * inv + 0.5);
                int64_t v = (int64_t)floor((double)y0 + (double)(k * dy) * inv + 0.5);
                o[v * nu + u] += w;
            }
        }
    }
}

/* raster.py:133-169 box_filter on one layer via a float64 integral image.
 * Column cumsum first (numpy axis=0), then row cumsum (axis=1), both strict
 * sequential folds; box sum ((T11 - T01) - T10) + T00, divided by the full
 * window area, rounded to float32.  `table` is caller scratch of nv*nu
 * doubles (the zero first row/column of the reference table is implicit). */
HB_ORACLE_API void orc_box_filter(const float *in, float *out, int nv, int nu,
                                  int radius, double *table) {
    if (radius == 0) {
        memcpy(out, in, sizeof(float) * (size_t)nv * nu);
        return;
    }
    for (int u = 0; u < nu; ++u) table[u] = (double)in[u];
    for (int v = 1; v < nv; ++v)
        for (int u = 0; u < nu; ++u)
            table[(int64_t)v * nu + u] =
                table[(int64_t)(v - 1) * nu + u] + (double)in[(int64_t)v * nu + u];
    for (int v = 0; v < nv; ++v) {
        double *row = table + (int64_t)v * nu;
        for (int u = 1; u < nu; ++u) row[u] = row[u - 1] + row[u];
    }
    const double area = (double)((2 * radius + 1) * (2 * radius + 1));
#define TZ(r, c) (((r) == 0 || (c) == 0) ? 0.0 : table[(int64_t)((r)-1) * nu + ((c)-1)])
    for (int v = 0; v < nv; ++v) {
        int r0 = v - radius; r0 = r0 < 0 ? 0 : (r0 > nv ? nv : r0);
        int r1 = v + radius + 1; r1 = r1 < 0 ? 0 : (r1 > nv ? nv : r1);
        for (int u = 0; u < nu; ++u) {
            int c0 = u - radius; c0 = c0 < 0 ? 0 : (c0 > nu ? nu : c0);
            int c1 = u + radius + 1; c1 = c1 < 0 ? 0 : (c1 > nu ? nu : c1);
            double s = ((TZ(r1, c1) - TZ(r0, c1)) - TZ(r1, c0)) + TZ(r0, c0);
            out[(int64_t)v * nu + u] = (float)(s / area);
        }
    }
#undef TZ
}

/* raster.py:196-200 _smooth_layer for layers [b_lo, b_hi): successive box
 * filters of radius (w-1)/2.  `scratch` holds nv*nu floats, `table` nv*nu
 * doubles. */
HB_ORACLE_API void orc_smooth_layers(const float *in, float *out, int nv,
                                     int nu, const int *widths, int npasses,
                                     int b_lo, int b_hi, float *scratch,
                                     double *table) {
    const int64_t plane = (int64_t)nv * nu;
    for (int b = b_lo; b < b_hi; ++b) {
        const float *src = in + b * plane;
        float *dst = out + b * plane;
        for (int p = 0; p < npasses; ++p) {
            /* ping-pong so the final pass lands in dst */
            float *target = ((npasses - 1 - p) % 2 == 0) ? dst : scratch;
            orc_box_filter(src, target, nv, nu, (widths[p] - 1) / 2, table);
            src = target;
        }
    }
}

/* _kernels.py:80-98 bilinear_value */
static inline double bilinear(const float *rho, int nv, int nu, double x,
                              double y) {
    int64_t u0 = (int64_t)floor(x), v0 = (int64_t)floor(y);
    if (u0 < 0) u0 = 0; else if (u0 > nu - 2) u0 = nu - 2;
    if (v0 < 0) v0 = 0; else if (v0 > nv - 2) v0 = nv - 2;
    double fx = x - (double)u0, fy = y - (double)v0;
    const float *r0 = rho + v0 * nu + u0, *r1 = r0 + nu;
    float d0 = r0[1] - r0[0];
    float d1 = r1[1] - r1[0];
    double a = (double)r0[0] + fx * (double)d0;
    double b = (double)r1[0] + fx * (double)d1;
    return a + fy * (b - a);
}

/* _kernels.py:101-114 _cell_gradient */
static inline void cell_grad(const float *rho, int nv, int nu, int64_t u,
                             int64_t v, double *gx, double *gy) {
    if (u < 1) u = 1; else if (u > nu - 2) u = nu - 2;
    if (v < 1) v = 1; else if (v > nv - 2) v = nv - 2;
    float dxf = rho[v * nu + u + 1] - rho[v * nu + u - 1];
    float dyf = rho[(v + 1) * nu + u] - rho[(v - 1) * nu + u];
    *gx = 0.5 * (double)dxf;
    *gy = 0.5 * (double)dyf;
}

/* _kernels.py:117-141 gradient_xy */
static inline void gradient_xy(const float *rho, int nv, int nu, double x,
                               double y, double *gx, double *gy) {
    int64_t u0 = (int64_t)floor(x), v0 = (int64_t)floor(y);
    if (u0 < 0) u0 = 0; else if (u0 > nu - 2) u0 = nu - 2;
    if (v0 < 0) v0 = 0; else if (v0 > nv - 2) v0 = nv - 2;
    double fx = x - (double)u0, fy = y - (double)v0;
    double g00x, g00y, g10x, g10y, g01x, g01y, g11x, g11y;
    cell_grad(rho, nv, nu, u0, v0, &g00x, &g00y);
    cell_grad(rho, nv, nu, u0 + 1, v0, &g10x, &g10y);
    cell_grad(rho, nv, nu, u0, v0 + 1, &g01x, &g01y);
    cell_grad(rho, nv, nu, u0 + 1, v0 + 1, &g11x, &g11y);
    double ax = g00x + fx * (g10x - g00x);
    double bx = g01x + fx * (g11x - g01x);
    double ay = g00y + fx * (g10y - g00y);
    double by = g01y + fx * (g11y - g01y);
    *gx = ax + fy * (bx - ax);
    *gy = ay + fy * (by - ay);
}

HB_ORACLE_API double orc_bilinear(const float *rho, int nv, int nu, double x,
                                  double y) {
    return bilinear(rho, nv, nu, x, y);
}

HB_ORACLE_API void orc_gradient(const float *rho, int nv, int nu, double x,
                                double y, double *g) {
    gradient_xy(rho, nv, nu, x, y, &g[0], &g[1]);
}

static inline double dmin(double a, double b) { return a < b ? a : b; }
static inline double dmax(double a, double b) { return a > b ? a : b; }

/* _kernels.py:144-200 advect.  out3 = {interior, moved} and disp are
 * written to res_i[0..1], res_d[0]. */
HB_ORACLE_API void orc_advect(double *pts, const int64_t *starts,
                              const int64_t *edge_layer, const float *rho3,
                              int nbins, int nv, int nu, double h, double eps,
                              double min_step, int fixed_step, int64_t e_lo,
                              int64_t e_hi, int64_t *res_i, double *res_d) {
    (void)nbins;
    const double xlo = 1.0, ylo = 1.0;
    const double xhi = (double)nu - 1.0 - 1.0, yhi = (double)nv - 1.0 - 1.0;
    const int64_t plane = (int64_t)nv * nu;
    int64_t interior = 0, moved = 0;
    double disp = 0.0;
    for (int64_t e = e_lo; e < e_hi; ++e) {
        const float *rho = rho3 + edge_layer[e] * plane;
        int64_t s = starts[e];
        int64_t n = starts[e + 1] - s;
        for (int64_t j = 1; j < n - 1; ++j) {
            double x = pts[2 * (s + j)], y = pts[2 * (s + j) + 1];
            interior += 1;
            double gx, gy;
            gradient_xy(rho, nv, nu, x, y, &gx, &gy);
            double gn = sqrt(gx * gx + gy * gy);
            if (gn < eps) gn = eps;
            double dx = gx / gn, dy = gy / gn;
            if (fixed_step) {
                double nx = dmin(dmax(x + h * dx, xlo), xhi);
                double ny = dmin(dmax(y + h * dy, ylo), yhi);
                if (nx != x || ny != y) {
                    moved += 1;
                    disp += sqrt((nx - x) * (nx - x) + (ny - y) * (ny - y));
                }
                pts[2 * (s + j)] = nx;
                pts[2 * (s + j) + 1] = ny;
                continue;
            }
            double r0 = bilinear(rho, nv, nu, x, y);
            double m = h;
            while (m >= min_step) {
                double nx = dmin(dmax(x + m * dx, xlo), xhi);
                double ny = dmin(dmax(y + m * dy, ylo), yhi);
                if (bilinear(rho, nv, nu, nx, ny) >= r0) {
                    if (nx != x || ny != y) {
                        moved += 1;
                        disp += sqrt((nx - x) * (nx - x) + (ny - y) * (ny - y));
                    }
                    pts[2 * (s + j)] = nx;
                    pts[2 * (s + j) + 1] = ny;
                    break;
                }
                m *= 0.5;
            }
        }
    }
    res_i[0] = interior;
    res_i[1] = moved;
    res_d[0] = disp;
}

/* _kernels.py:203-232 resample_count */
HB_ORACLE_API void orc_resample_count(const double *pts, const int64_t *starts,
                                      double delta, int64_t *counts,
                                      int64_t e_lo, int64_t e_hi) {
    const double lo = 0.5 * delta, hi = 1.5 * delta;
    for (int64_t e = e_lo; e < e_hi; ++e) {
        int64_t s = starts[e];
        int64_t n = starts[e + 1] - s;
        double ax = pts[2 * s], ay = pts[2 * s + 1];
        int64_t total = 1;
        for (int64_t j = 1; j < n; ++j) {
            double x = pts[2 * (s + j)], y = pts[2 * (s + j) + 1];
            double g = sqrt((x - ax) * (x - ax) + (y - ay) * (y - ay));
            if (j < n - 1 && g < lo) continue;
            int64_t pieces = 1;
            while (g > hi) { g *= 0.5; pieces *= 2; }
            total += pieces;
            ax = x;
            ay = y;
        }
        counts[e] = total;
    }
}

/* _kernels.py:235-272 resample_emit */
HB_ORACLE_API void orc_resample_emit(const double *pts, const int64_t *starts,
                                     double delta, const int64_t *new_starts,
                                     double *out, int64_t e_lo, int64_t e_hi) {
    const double lo = 0.5 * delta, hi = 1.5 * delta;
    for (int64_t e = e_lo; e < e_hi; ++e) {
        int64_t s = starts[e];
        int64_t n = starts[e + 1] - s;
        int64_t w = new_starts[e];
        double ax = pts[2 * s], ay = pts[2 * s + 1];
        out[2 * w] = ax;
        out[2 * w + 1] = ay;
        w += 1;
        for (int64_t j = 1; j < n; ++j) {
            double x = pts[2 * (s + j)], y = pts[2 * (s + j) + 1];
            double g = sqrt((x - ax) * (x - ax) + (y - ay) * (y - ay));
            if (j < n - 1 && g < lo) continue;
            int64_t pieces = 1;
            while (g > hi) { g *= 0.5; pieces *= 2; }
            for (int64_t k = 1; k < pieces; ++k) {
                double t = (double)k / (double)pieces;
                out[2 * w] = ax + t * (x - ax);
                out[2 * w + 1] = ay + t * (y - ay);
                w += 1;
            }
            out[2 * w] = x;
            out[2 * w + 1] = y;
            w += 1;
            ax = x;
            ay = y;
        }
    }
}

/* _kernels.py:275-296 laplacian (Jacobi, endpoints fixed) */
HB_ORACLE_API void orc_laplacian(double *pts, const int64_t *starts,
                                 double factor, int passes, double *scratch,
                                 int64_t e_lo, int64_t e_hi) {
    for (int p = 0; p < passes; ++p) {
        for (int64_t e = e_lo; e < e_hi; ++e) {
            int64_t s = starts[e];
            int64_t n = starts[e + 1] - s;
            for (int64_t j = 1; j < n - 1; ++j) {
                const double *q = pts + 2 * (s + j);
                double mx = 0.5 * (q[-2] + q[2]);
                double my = 0.5 * (q[-1] + q[3]);
                scratch[2 * (s + j)] = q[0] + factor * (mx - q[0]);
                scratch[2 * (s + j) + 1] = q[1] + factor * (my - q[1]);
            }
        }
        for (int64_t e = e_lo; e < e_hi; ++e) {
            int64_t s = starts[e];
            int64_t n = starts[e + 1] - s;
            for (int64_t j = 1; j < n - 1; ++j) {
                pts[2 * (s + j)] = scratch[2 * (s + j)];
                pts[2 * (s + j) + 1] = scratch[2 * (s + j) + 1];
            }
        }
    }
}

/* bundler.py:292-305 used_cell_count: per layer, peak = max(rho, initial 0);
 * count rho > float32(rel * peak) (NumPy 2 / NEP 50 compares in float32). */
HB_ORACLE_API int64_t orc_used_cells(const float *rho, int nbins, int nv,
                                     int nu, double rel) {
    const int64_t plane = (int64_t)nv * nu;
    int64_t total = 0;
    for (int b = 0; b < nbins; ++b) {
        const float *r = rho + b * plane;
        float peak = 0.0f;
        for (int64_t i = 0; i < plane; ++i)
            if (r[i] > peak) peak = r[i];
        if (!((double)peak > 0.0)) continue;
        float thr = (float)(rel * (double)peak);
        for (int64_t i = 0; i < plane; ++i) total += r[i] > thr;
    }
    return total;
}

/* bundler.py:92-106 _offset_packed, per-edge displacement already computed
 * by the caller: interior points of edge e move by disp[e]. */
HB_ORACLE_API void orc_offset(double *pts, const int64_t *starts,
                              const double *disp, int64_t n_edges) {
    for (int64_t e = 0; e < n_edges; ++e)
        for (int64_t j = starts[e] + 1; j < starts[e + 1] - 1; ++j) {
            pts[2 * j] += disp[2 * e];
            pts[2 * j + 1] += disp[2 * e + 1];
        }
}
