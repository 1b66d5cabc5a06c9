// hb_binning.cu -- edge binning by best-of-restarts Lloyd K-means and the
// Davies-Bouldin index (/root/reference/pkg/src/histobundle/binning.py:81-177).
//
// Every restart is independent, so the device runs all active restarts of an
// iteration at once: one thread per (restart, edge) for the assignment step
// and one block per restart for the centroid update.  The
// arithmetic repeats numpy's, in numpy's order:
//   * squared distance einsum("rnkd,rnkd->rnk") (binning.py:114): for d = 4
//     numpy pairs the products as (p0 + p2) + (p1 + p3), for d <= 2 it adds
//     them in order (checked against numpy 2.3 in this container);
//   * argmin over clusters takes the first minimum (np.argmin);
//   * np.add.at(sums, assign, features) (binning.py:143) is a left fold in
//     edge order per (cluster, column): the update block stages the edges in
//     shared-memory tiles and a warp folds each cluster's hits in order;
//   * centroid = sums / counts (IEEE divide), empty clusters keep their
//     centroid until re-seeded with the farthest edges (binning.py:145-154):
//     dist = np.linalg.norm(axis=1) adds the squared columns in order, and
//     np.argmax takes the first maximum.
// Compiled with --fmad=false like the rest of the library: no contraction.
#include "hb_common.cuh"

namespace hb {

constexpr int kKmMaxK = 64;
constexpr int kKmMaxD = 4;

__device__ __forceinline__ double km_d2(const double *f, const double *c, int d) {
    // einsum's order (see the file comment)
    if (d == 4) {
        const double a0 = dsub(f[0], c[0]), a1 = dsub(f[1], c[1]);
        const double a2 = dsub(f[2], c[2]), a3 = dsub(f[3], c[3]);
        return dadd(dadd(dmul(a0, a0), dmul(a2, a2)), dadd(dmul(a1, a1), dmul(a3, a3)));
    }
    double s = 0.0;
    for (int j = 0; j < d; ++j) {
        const double a = dsub(f[j], c[j]);
        s = j == 0 ? dmul(a, a) : dadd(s, dmul(a, a));
    }
    return s;
}

// np.linalg.norm(x, axis=1): squares added in column order, then sqrt
__device__ __forceinline__ double km_norm(const double *f, const double *c, int d) {
    double s = 0.0;
    for (int j = 0; j < d; ++j) {
        const double a = dsub(f[j], c[j]);
        s = j == 0 ? dmul(a, a) : dadd(s, dmul(a, a));
    }
    return __dsqrt_rn(s);
}

// grid (edge blocks, active restarts); assign[r*n + i] int8 cluster
__global__ void __launch_bounds__(256)
km_assign_kernel(const double *__restrict__ f, int64_t n, int d, int k,
                 const double *__restrict__ cent, const int32_t *__restrict__ active,
                 int8_t *__restrict__ assign, int32_t *__restrict__ changed,
                 const int32_t *__restrict__ live) {
    __shared__ double s_c[kKmMaxK * kKmMaxD];
    const int r = active ? active[blockIdx.y] : (int)blockIdx.y;
    if (live && !live[r]) return;  // (device-driven loop: converged restart)
    for (int t = threadIdx.x; t < k * d; t += blockDim.x) s_c[t] = cent[(int64_t)r * k * d + t];
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool ch = false;
    if (i < n) {
        double fi[kKmMaxD];
        for (int j = 0; j < d; ++j) fi[j] = f[i * d + j];
        double best = km_d2(fi, s_c, d);
        int bc = 0;
        for (int c = 1; c < k; ++c) {
            const double v = km_d2(fi, s_c + c * d, d);
            if (v < best) { best = v; bc = c; }  // first minimum
        }
        int8_t *a = assign + (int64_t)r * n + i;
        ch = *a != (int8_t)bc;
        *a = (int8_t)bc;
    }
    if (__any_sync(0xffffffffu, ch) && (threadIdx.x & 31) == 0) atomicOr(changed + r, 1);
}

// One block per restart in `upd`.  The edges stream through shared memory in
// tiles of 1024 (assignments + feature rows); each tile is bucketed by
// cluster, stably (per 32-edge window: rank among same-cluster lanes by
// __match_any_sync, then window and cluster prefixes), and thread (c, j)
// folds column j of cluster c's rows in edge order -- one float64 chain per
// (cluster, column), as np.add.at orders it, with the next row read ahead.
// Then centroid = sums / count; an empty cluster raises empty[r].
constexpr int kUpdBlock = 256;
constexpr int kUpdTile = 1024;
constexpr int kUpdWin = kUpdTile / 32;
__global__ void __launch_bounds__(kUpdBlock)
km_update_kernel(const double *__restrict__ f, int64_t n, int d, int k,
                 double *__restrict__ cent, const int32_t *__restrict__ upd,
                 const int8_t *__restrict__ assign, int32_t *__restrict__ empty,
                 const int32_t *__restrict__ live, const int32_t *__restrict__ changed) {
    __shared__ int8_t s_a[kUpdTile];
    __shared__ short s_list[kUpdTile];
    __shared__ double s_f[kUpdTile * kKmMaxD];
    __shared__ short s_wc[kUpdWin][kKmMaxK];  // per (window, cluster): count, then offset
    __shared__ int s_base[kKmMaxK + 1];
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int r = upd ? upd[blockIdx.x] : (int)blockIdx.x;
    if (live && !(live[r] && changed[r])) return;
    const int8_t *a = assign + (int64_t)r * n;
    // thread t < k*d owns the chain of cluster t / d, column t % d
    const int my_c = threadIdx.x / d, my_j = threadIdx.x % d;
    const bool chain = threadIdx.x < k * d;
    double acc = 0.0;
    long long cnt = 0;
    for (int64_t t0 = 0; t0 < n; t0 += kUpdTile) {
        const int m = (int)(n - t0 < kUpdTile ? n - t0 : kUpdTile);
        __syncthreads();  // the previous tile is consumed
        for (int t = threadIdx.x; t < m; t += kUpdBlock) s_a[t] = a[t0 + t];
        for (int t = threadIdx.x; t < m * d; t += kUpdBlock) s_f[t] = f[t0 * d + t];
        for (int t = threadIdx.x; t < kUpdWin * k; t += kUpdBlock) s_wc[t / k][t % k] = 0;
        __syncthreads();
        // window counts and ranks
        int rank[kUpdWin / (kUpdBlock / 32)];
        for (int q = 0; q < kUpdWin / (kUpdBlock / 32); ++q) {
            const int wi = warp + q * (kUpdBlock / 32);
            const int e = wi * 32 + lane;
            const int c = e < m ? s_a[e] : -1;
            const unsigned peers = __match_any_sync(full, c);
            rank[q] = __popc(peers & ((1u << lane) - 1u));
            if (c >= 0 && rank[q] == 0) s_wc[wi][c] = (short)__popc(peers);
        }
        __syncthreads();
        // per cluster: window offsets (exclusive) and the tile count
        if (threadIdx.x < k) {
            int run = 0;
            for (int wi = 0; wi < kUpdWin; ++wi) {
                const int v = s_wc[wi][threadIdx.x];
                s_wc[wi][threadIdx.x] = (short)run;
                run += v;
            }
            s_base[threadIdx.x + 1] = run;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            s_base[0] = 0;
            for (int c = 0; c < k; ++c) s_base[c + 1] += s_base[c];
        }
        __syncthreads();
        for (int q = 0; q < kUpdWin / (kUpdBlock / 32); ++q) {
            const int wi = warp + q * (kUpdBlock / 32);
            const int e = wi * 32 + lane;
            if (e < m) {
                const int c = s_a[e];
                s_list[s_base[c] + s_wc[wi][c] + rank[q]] = (short)e;
            }
        }
        __syncthreads();
        if (chain) {
            const int lo = s_base[my_c], hi = s_base[my_c + 1];
            cnt += hi - lo;
            if (lo < hi) {
                double v = s_f[s_list[lo] * d + my_j];
                for (int q = lo + 1; q < hi; ++q) {  // np.add.at: edges in order
                    const double nv = s_f[s_list[q] * d + my_j];
                    acc = dadd(acc, v);
                    v = nv;
                }
                acc = dadd(acc, v);
            }
        }
    }
    if (chain) {
        double *cc = cent + ((int64_t)r * k + my_c) * d;
        if (cnt > 0) {
            cc[my_j] = __ddiv_rn(acc, (double)cnt);
        } else if (my_j == 0) {
            atomicOr(empty + r, 1);
        }
    }
}

// One block per restart in `rs` (restarts with emptied clusters, processed
// one after another): dist = norm(f - cent[assign]) into scratch, then for
// each empty cluster in ascending order the first farthest edge becomes its
// centroid and its distance -inf (binning.py:145-154).  counts are recounted
// here (an emptied cluster has none).
constexpr int kReseedBlock = 1024;
__global__ void __launch_bounds__(kReseedBlock)
km_reseed_kernel(const double *__restrict__ f, int64_t n, int d, int k, double *__restrict__ cent,
                 const int32_t *__restrict__ rs, const int8_t *__restrict__ assign,
                 double *__restrict__ dist, const int32_t *__restrict__ live,
                 const int32_t *__restrict__ changed, const int32_t *__restrict__ empty) {
    __shared__ int s_cnt[kKmMaxK];
    __shared__ double s_c[kKmMaxK * kKmMaxD];
    __shared__ double s_bv[kReseedBlock / 32];
    __shared__ long long s_bi[kReseedBlock / 32];
    const int r = rs ? rs[blockIdx.x] : (int)blockIdx.x;
    if (live && !(live[r] && changed[r] && empty[r])) return;
    double *dr = dist + (int64_t)blockIdx.x * n;
    const int8_t *a = assign + (int64_t)r * n;
    for (int t = threadIdx.x; t < k; t += blockDim.x) s_cnt[t] = 0;
    for (int t = threadIdx.x; t < k * d; t += blockDim.x) s_c[t] = cent[(int64_t)r * k * d + t];
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const int c = a[i];
        atomicAdd(&s_cnt[c], 1);
        dr[i] = km_norm(f + i * d, s_c + c * d, d);
    }
    __syncthreads();
    for (int c = 0; c < k; ++c) {
        if (s_cnt[c] != 0) continue;  // (block-uniform)
        // first maximum of dr
        double bv = -__longlong_as_double(0x7ff0000000000000LL);  // -inf
        long long bi = -1;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            const double v = dr[i];
            if (bi < 0 || v > bv) { bv = v; bi = i; }
        }
        for (int o = 16; o; o >>= 1) {
            const double ov = __shfl_down_sync(0xffffffffu, bv, o);
            const long long oi = __shfl_down_sync(0xffffffffu, bi, o);
            if (oi >= 0 && (bi < 0 || ov > bv || (ov == bv && oi < bi))) { bv = ov; bi = oi; }
        }
        if ((threadIdx.x & 31) == 0) {
            s_bv[threadIdx.x >> 5] = bv;
            s_bi[threadIdx.x >> 5] = bi;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int wv = 1; wv < kReseedBlock / 32; ++wv) {
                const double ov = s_bv[wv];
                const long long oi = s_bi[wv];
                if (oi >= 0 && (bi < 0 || ov > bv || (ov == bv && oi < bi))) { bv = ov; bi = oi; }
            }
            for (int j = 0; j < d; ++j) cent[((int64_t)r * k + c) * d + j] = f[bi * d + j];
            dr[bi] = -__longlong_as_double(0x7ff0000000000000LL);
        }
        __syncthreads();
    }
}

// end of a device-driven iteration: a restart stays live only if its
// assignment changed (binning.py:117-118); the per-iteration flags reset
__global__ void km_step_end_kernel(int restarts, int32_t *__restrict__ live,
                                   int32_t *__restrict__ changed, int32_t *__restrict__ empty) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < restarts) {
        live[r] = live[r] && changed[r];
        changed[r] = 0;
        empty[r] = 0;
    }
}

// per restart r: sum over edges of the squared distance to its centroid,
// per-block partials in a fixed order (used only to pick the best restart)
__global__ void __launch_bounds__(256)
km_inertia_kernel(const double *__restrict__ f, int64_t n, int d, int k,
                  const double *__restrict__ cent, const int8_t *__restrict__ assign,
                  double *__restrict__ partial) {
    __shared__ double s_c[kKmMaxK * kKmMaxD];
    __shared__ double s_w[8];
    const int r = blockIdx.y;
    for (int t = threadIdx.x; t < k * d; t += blockDim.x) s_c[t] = cent[(int64_t)r * k * d + t];
    __syncthreads();
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int c = assign[(int64_t)r * n + i];
        s = dadd(s, km_d2(f + i * d, s_c + c * d, d));
    }
    for (int o = 16; o; o >>= 1) s = dadd(s, __shfl_down_sync(0xffffffffu, s, o));
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int wv = 1; wv < 8; ++wv) s = dadd(s, s_w[wv]);
        partial[(int64_t)r * gridDim.x + blockIdx.x] = s;
    }
}

// Davies-Bouldin scatter (binning.py:167-171): one warp per cluster folds
// norm(f_i - centroid) over its edges in order; counts alongside
__global__ void __launch_bounds__(256)
km_scatter_kernel(const double *__restrict__ f, int64_t n, int d, int k,
                  const double *__restrict__ cent, const int8_t *__restrict__ assign,
                  double *__restrict__ scatter, int64_t *__restrict__ counts) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int c = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (c >= k) return;
    double cc[kKmMaxD];
    for (int j = 0; j < d; ++j) cc[j] = cent[c * d + j];
    double acc = 0.0;
    int64_t cnt = 0;
    for (int64_t i0 = 0; i0 < n; i0 += 32) {
        const int64_t i = i0 + lane;
        const bool hit = i < n && assign[i] == c;
        unsigned m = __ballot_sync(full, hit);
        if (!m) continue;
        const double v = hit ? km_norm(f + i * d, cc, d) : 0.0;
        cnt += __popc(m);
        while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            acc = dadd(acc, __shfl_sync(full, v, b));
        }
    }
    if (lane == 0) {
        scatter[c] = acc;
        counts[c] = cnt;
    }
}

}  // namespace hb

using namespace hb;

static inline cudaStream_t km_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

static bool km_shape_ok(int64_t n, int d, int k) {
    return n >= 1 && d >= 1 && d <= kKmMaxD && k >= 1 && k <= kKmMaxK && k <= 127;
}

extern "C" {

int hb_kmeans_assign(const double *features, int64_t n, int d, int k, const double *cent,
                     const int32_t *active, int n_active, int8_t *assign, int32_t *changed,
                     void *stream) {
    if (!km_shape_ok(n, d, k) || n_active < 0 || n_active > 65535 || !features || !cent ||
        (n_active > 0 && (!active || !assign || !changed)))
        return set_error(HB_EINVAL, "hb_kmeans_assign: bad arguments");
    if (n_active == 0) return HB_OK;
    dim3 g((unsigned)((n + 255) / 256), (unsigned)n_active);
    km_assign_kernel<<<g, 256, 0, km_stream(stream)>>>(features, n, d, k, cent, active, assign,
                                                      changed, nullptr);
    return check_launch("hb_kmeans_assign");
}

int hb_kmeans_update(const double *features, int64_t n, int d, int k, double *cent,
                     const int32_t *upd, int n_upd, const int8_t *assign, int32_t *empty,
                     void *stream) {
    if (!km_shape_ok(n, d, k) || n_upd < 0 || !features || !cent ||
        (n_upd > 0 && (!upd || !assign || !empty)))
        return set_error(HB_EINVAL, "hb_kmeans_update: bad arguments");
    if (n_upd == 0) return HB_OK;
    km_update_kernel<<<n_upd, kUpdBlock, 0, km_stream(stream)>>>(features, n, d, k, cent, upd,
                                                               assign, empty, nullptr, nullptr);
    return check_launch("hb_kmeans_update");
}

size_t hb_kmeans_reseed_workspace_bytes(int64_t n, int n_reseed) {
    return (size_t)(n > 0 ? n : 0) * (size_t)(n_reseed > 0 ? n_reseed : 0) * sizeof(double);
}

int hb_kmeans_reseed(const double *features, int64_t n, int d, int k, double *cent,
                     const int32_t *rs, int n_rs, const int8_t *assign, void *workspace,
                     size_t workspace_bytes, void *stream) {
    if (!km_shape_ok(n, d, k) || n_rs < 0 || !features || !cent ||
        (n_rs > 0 && (!rs || !assign || !workspace)))
        return set_error(HB_EINVAL, "hb_kmeans_reseed: bad arguments");
    if (n_rs == 0) return HB_OK;
    if (workspace_bytes < hb_kmeans_reseed_workspace_bytes(n, n_rs))
        return set_error(HB_EINVAL, "hb_kmeans_reseed: workspace too small");
    km_reseed_kernel<<<n_rs, kReseedBlock, 0, km_stream(stream)>>>(
        features, n, d, k, cent, rs, assign, reinterpret_cast<double *>(workspace), nullptr,
        nullptr, nullptr);
    return check_launch("hb_kmeans_reseed");
}

// `iterations` Lloyd steps of every restart with the restart bookkeeping on
// the device: flags = [live (restarts) | changed | empty] int32, live = 1 to
// start; a restart whose assignment stopped changing stays out.  The
// workspace holds restarts * n float64 re-seed distances.
int hb_kmeans_lloyd(const double *features, int64_t n, int d, int k, double *cent, int restarts,
                    int8_t *assign, int32_t *flags, int iterations, void *workspace,
                    size_t workspace_bytes, void *stream) {
    if (!km_shape_ok(n, d, k) || restarts < 1 || restarts > 65535 || iterations < 0 ||
        !features || !cent || !assign || !flags || !workspace)
        return set_error(HB_EINVAL, "hb_kmeans_lloyd: bad arguments");
    if (workspace_bytes < hb_kmeans_reseed_workspace_bytes(n, restarts))
        return set_error(HB_EINVAL, "hb_kmeans_lloyd: workspace too small");
    cudaStream_t st = km_stream(stream);
    int32_t *live = flags, *changed = flags + restarts, *empty = flags + 2 * restarts;
    dim3 g((unsigned)((n + 255) / 256), (unsigned)restarts);
    for (int it = 0; it < iterations; ++it) {
        km_assign_kernel<<<g, 256, 0, st>>>(features, n, d, k, cent, nullptr, assign, changed,
                                            live);
        km_update_kernel<<<restarts, kUpdBlock, 0, st>>>(features, n, d, k, cent, nullptr, assign,
                                                         empty, live, changed);
        km_reseed_kernel<<<restarts, kReseedBlock, 0, st>>>(
            features, n, d, k, cent, nullptr, assign, reinterpret_cast<double *>(workspace), live,
            changed, empty);
        km_step_end_kernel<<<(restarts + 255) / 256, 256, 0, st>>>(restarts, live, changed, empty);
    }
    return check_launch("hb_kmeans_lloyd", 4 * iterations);
}

int hb_kmeans_inertia_blocks(void) { return 64; }

int hb_kmeans_inertia(const double *features, int64_t n, int d, int k, const double *cent,
                      int restarts, const int8_t *assign, double *partial, void *stream) {
    if (!km_shape_ok(n, d, k) || restarts < 1 || restarts > 65535 || !features || !cent ||
        !assign || !partial)
        return set_error(HB_EINVAL, "hb_kmeans_inertia: bad arguments");
    dim3 g((unsigned)hb_kmeans_inertia_blocks(), (unsigned)restarts);
    km_inertia_kernel<<<g, 256, 0, km_stream(stream)>>>(features, n, d, k, cent, assign, partial);
    return check_launch("hb_kmeans_inertia");
}

int hb_kmeans_scatter(const double *features, int64_t n, int d, int k, const double *cent,
                      const int8_t *assign, double *scatter, int64_t *counts, void *stream) {
    if (!km_shape_ok(n, d, k) || !features || !cent || !assign || !scatter || !counts)
        return set_error(HB_EINVAL, "hb_kmeans_scatter: bad arguments");
    km_scatter_kernel<<<(unsigned)((k * 32 + 255) / 256), 256, 0, km_stream(stream)>>>(
        features, n, d, k, cent, assign, scatter, counts);
    return check_launch("hb_kmeans_scatter");
}

}  // extern "C"
