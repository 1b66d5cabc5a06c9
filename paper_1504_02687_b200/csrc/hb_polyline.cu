// hb_polyline.cu -- polyline kernels: initial sampling, directed offset,
// grid->world, histogram splat, resample count / scan / emit(+splat).
//
// Layout: packed (N,2) float64 points (one double2 = 16 B per point), edge
// offsets `starts` (E+1) int64.  The streaming kernels are warp-per-edge and
// persistent (grid-stride over edges): a warp walks its edge 32 points at a
// time with coalesced 512 B loads, and everything that depends on a
// neighbour (segment start, previous kept point) comes from a shuffle or from
// a carry kept in registers across chunks -- no searches, no CTA barriers.
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

// bundler.py:77-85 per edge: grid endpoints (p - origin) / cell and the
// point count max(ceil(|d| / delta), 1) + 1, |d| = sqrt(dx*dx + dy*dy) as
// np.linalg.norm computes it for a 2-vector.
__global__ void edge_prepare_kernel(const double2 *__restrict__ node_pos,
                                    const int64_t *__restrict__ sources,
                                    const int64_t *__restrict__ targets, int64_t n_edges,
                                    double ox, double oy, double cell, double delta,
                                    double2 *__restrict__ src, double2 *__restrict__ dst,
                                    int64_t *__restrict__ counts) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n_edges) return;
    const double2 a = node_pos[sources[e]], b = node_pos[targets[e]];
    const double2 sa = make_double2(dsub(a.x, ox) / cell, dsub(a.y, oy) / cell);
    const double2 sb = make_double2(dsub(b.x, ox) / cell, dsub(b.y, oy) / cell);
    src[e] = sa;
    dst[e] = sb;
    const double seg = hypot_ref(dsub(sb.x, sa.x), dsub(sb.y, sa.y));
    const double c = ceil(seg / delta);
    counts[e] = (c < 1.0 ? (int64_t)1 : (int64_t)c) + 1;
}

__global__ void to_world_nodes_kernel(const double2 *__restrict__ pts,
                                      const int64_t *__restrict__ starts, int64_t n_edges,
                                      double ox, double oy, double cell,
                                      const double2 *__restrict__ node_pos,
                                      const int64_t *__restrict__ sources,
                                      const int64_t *__restrict__ targets,
                                      double2 *__restrict__ out) {
    const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
    const int lane = threadIdx.x & 31;
    if (e >= n_edges) return;
    const int64_t s = starts[e], t = starts[e + 1] - 1;
    for (int64_t j = s + lane; j <= t; j += kWarp) {
        double2 w;
        if (j == s) {
            w = node_pos[sources[e]];
        } else if (j == t) {
            w = node_pos[targets[e]];
        } else {
            const double2 p = pts[j];
            w = make_double2(dadd(dmul(p.x, cell), ox), dadd(dmul(p.y, cell), oy));
        }
        out[j] = w;
    }
}

// ---------------------------------------------------------------------------
// accumulate (_kernels.py:46-77), warp per edge: lane j rasterises segment
// (j-1, j); its start point comes from the lane below (or the carry).
template <typename T>
__global__ void __launch_bounds__(kStreamBlock)
splat_kernel(const double2 *__restrict__ pts, const int64_t *__restrict__ starts,
             int64_t n_edges, const int32_t *__restrict__ group,
             const T *__restrict__ weight, T *__restrict__ hist, int64_t plane, int nv,
             int nu, int32_t *__restrict__ status, const __grid_constant__ hb_tiles tl,
             int use_tiles) {
    const hb_tiles *tiles = use_tiles ? &tl : nullptr;
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (kStreamBlock / 32);
    for (int64_t e = ((int64_t)blockIdx.x * kStreamBlock + threadIdx.x) / 32; e < n_edges;
         e += nwarps) {
        const int64_t s = starts[e];
        const int64_t n = starts[e + 1] - s;
        const int grp = group[e];
        const T w = weight ? weight[e] : T(1);
        double2 prev = pts[s];
        for (int64_t c0 = 1; c0 < n; c0 += kWarp) {
            const int64_t j = c0 + lane;
            const bool valid = j < n;
            const double2 p = valid ? pts[s + j] : make_double2(0.0, 0.0);
            double qx = __shfl_up_sync(full, p.x, 1), qy = __shfl_up_sync(full, p.y, 1);
            if (lane == 0) { qx = prev.x; qy = prev.y; }
            bin_or_splat<T>(valid, qx, qy, p.x, p.y, j == 1 ? 0 : 1, w, grp, hist, plane, nv, nu,
                            status, tiles);
            prev.x = __shfl_sync(full, p.x, 31);
            prev.y = __shfl_sync(full, p.y, 31);
        }
    }
}

// ---------------------------------------------------------------------------
// resample_emit (_kernels.py:235-272) + accumulate of the new polylines.
// pos[j] (from the count pass) is the output index of kept point j (-1 if
// merged).  A kept point x whose previous kept point is a (pieces = pos[x] -
// pos[a]) owns outputs pos[a]+1 .. pos[x]: k/pieces interpolants
// a + (k/pieces)(x - a), then x itself.
__device__ __forceinline__ double2 interp_piece(double2 a, double2 x, int k, int pieces) {
    if (k == pieces) return x;
    if (k == 0) return a;
    // t = k / pieces (_kernels.py:264); pieces = 2^s is a power of two, so
    // the quotient is exact and equals k * 2^-s (built from the exponent)
    const int sh = __ffs(pieces) - 1;
    const double t = dmul((double)k, __longlong_as_double((long long)(1023 - sh) << 52));
    return make_double2(dadd(a.x, dmul(t, dsub(x.x, a.x))), dadd(a.y, dmul(t, dsub(x.y, a.y))));
}

// Streaming point traffic is marked evict-first so the segment-key table's
// lines (hit by ~1 atomic per segment) stay resident in L2.
#ifndef HB_NO_STREAM_HINTS
#define HB_LD_STREAM(p) __ldcs(p)
#define HB_ST_STREAM(p, v) __stcs((p), (v))
#else
#define HB_LD_STREAM(p) (*(p))
#define HB_ST_STREAM(p, v) (*(p) = (v))
#endif

// ---------------------------------------------------------------------------
// Ring emit: input-major, each input read once.  A warp owns an edge-aligned
// range of whole polylines (balanced by input points, like the Laplacian +
// count pass) and walks it in 32-input chunks.  Kept input x (pos >= 0) with
// previous kept input a owns outputs G(a)+1 .. G(x): the interpolants
// a + (k/pieces)(x - a) (interp_piece, pieces = G(x) - G(a)) and x itself;
// an edge's first input owns only itself.  Every lane writes its outputs
// (usually one) into a per-warp ring of output slots in shared memory; as
// soon as 32 consecutive outputs are complete, the warp stores them
// (coalesced) and splats the segment ending at each, one output per lane.
// The previous output of a tile's lane 0 is carried in registers.  Output
// indices inside the range are 32-bit (a range holds < 2^31 outputs).
//
// (An output-tiled variant, which rescanned chunks and rebuilt a slot table
// per 32 outputs, issued ~2x the instructions per output; removed.)
constexpr int kRing = 128;  // slots per warp (power of two)
struct EmitRing {
    double2 q[kRing];
    int meta[kRing];  // (edge << 2) | min(local index, 2)
    // the next 32-input chunk, fetched by cp.async while the warp works on
    // the current one: points, pos, and starts / new_starts of the 32 edges
    // after the chunk's first edge
    double2 cpts[32];
    long long csv[32], cnsv[32];
    int cpos[32];
};

// cp.async with zero fill (src-size 0: nothing is read) for out-of-range lanes
__device__ __forceinline__ void emit_cp(void *smem, const void *gmem, int bytes, bool ok) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    if (bytes == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem),
                     "r"(ok ? 16 : 0));
    else if (bytes == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem),
                     "r"(ok ? 8 : 0));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem),
                     "r"(ok ? 4 : 0));
}

// Dynamic work for the ring emit: kEmitRangesPerWarp edge-aligned ranges
// per warp, taken off a counter (zeroed by the host before each launch), so
// warps that drew cheap ranges take more (a static range per warp left SMs
// idle for ~10 % of the kernel: sm__cycles_active avg 11.6 M vs max 12.9 M).
#ifndef HB_EMIT_RANGES_PER_WARP
#define HB_EMIT_RANGES_PER_WARP 16  // measured (emit ms, config 4): static 5.75, 4: 5.21, 8: 5.15, 16: 5.05, 32: 5.07
#endif
constexpr int kEmitRangesPerWarp = HB_EMIT_RANGES_PER_WARP;
__device__ unsigned long long g_emit_next;

// lower_edge (first e in [0, n] with starts[e] >= v, else n) as a 32-ary
// warp search: ~5 dependent loads instead of ~21
__device__ __forceinline__ int64_t warp_lower_edge(const int64_t *__restrict__ starts, int64_t n,
                                                   int64_t v) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    int64_t lo = 0, hi = n;  // answer in [lo, hi]
    while (hi - lo >= 32) {
        const int64_t step = (hi - lo) / 32;
        const unsigned b = __ballot_sync(full, starts[lo + (lane + 1) * step] >= v);
        if (b) {
            const int f = __ffs(b) - 1;
            hi = lo + (f + 1) * step;
            lo = lo + f * step;
        } else {
            lo = lo + 32 * step;
        }
    }
    const int64_t j = lo + lane;
    const unsigned b = __ballot_sync(full, j <= hi && starts[j] >= v);
    return b ? lo + __ffs(b) - 1 : hi;
}

#ifndef HB_EMIT_RING_MINB
#define HB_EMIT_RING_MINB 4
#endif
__global__ void __launch_bounds__(kStreamBlock, HB_EMIT_RING_MINB)
emit_ring_kernel(const double2 *__restrict__ pts, const int64_t *__restrict__ starts,
                 int64_t n_edges, const int32_t *__restrict__ pos,
                 const int64_t *__restrict__ new_starts, double2 *__restrict__ out,
                 const int32_t *__restrict__ group, const int32_t *__restrict__ weight,
                 int32_t *__restrict__ hist, int64_t plane, int nv, int nu,
                 int32_t *__restrict__ status, const __grid_constant__ hb_tiles tl, int use_tiles,
                 int64_t out_cap) {
    __shared__ __align__(16) EmitRing s_ring[kStreamBlock / 32];
    const hb_tiles *tiles = use_tiles ? &tl : nullptr;
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    if (new_starts[n_edges] > out_cap) {
        if (blockIdx.x == 0 && threadIdx.x == 0 && status) atomicOr(status, HB_STATUS_CAPACITY);
        return;
    }
    EmitRing &R = s_ring[threadIdx.x >> 5];
    const bool splat = hist != nullptr;

    // edge-aligned input ranges [J_a, J_b) = edges [e0, e1), taken dynamically
    const int64_t nw = (int64_t)gridDim.x * (kStreamBlock / 32);
    const int64_t n_ranges = nw * kEmitRangesPerWarp;
    const int64_t P_lo = starts[0], P_hi = starts[n_edges];
    const int64_t span = P_hi > P_lo ? P_hi - P_lo : 0;
    for (;;) {
    unsigned long long rg = 0;
    if (lane == 0) rg = atomicAdd(&g_emit_next, 1ull);
    const int64_t r = (int64_t)__shfl_sync(full, rg, 0);
    if (r >= n_ranges) break;  // (warp-uniform)
    const int64_t e0 = warp_lower_edge(starts, n_edges, P_lo + (span * r) / n_ranges);
    const int64_t e1 = warp_lower_edge(starts, n_edges, P_lo + (span * (r + 1)) / n_ranges);
    if (e0 >= e1) continue;
    const int64_t J_a = starts[e0], J_b = starts[e1];
    const int64_t O_a = new_starts[e0];
    const int O_n = (int)(new_starts[e1] - O_a);  // outputs of the range
    double2 *const outw = out + O_a;

    int F = 0;                              // first output not yet flushed
    int cqx = 0, cqy = 0;                   // cell of output F - 1 (previous tile's last)
    double2 ca = make_double2(0.0, 0.0);    // last kept input so far ...
    int cg = -1;                            // ... and its output index

    // store + splat outputs [F, F + cnt), cnt <= 32, all present in the ring
    auto flush = [&](int cnt) {
        __syncwarp();
        const int o = F + lane;
        const bool valid = lane < cnt;
        const int sl = o & (kRing - 1);
        const double2 q = valid ? R.q[sl] : make_double2(0.0, 0.0);
        const int meta = valid ? R.meta[sl] : 0;
        if (valid) HB_ST_STREAM(outw + o, q);
        if (splat) {
            // each output's cell is rounded once; segment m-1 -> m takes the
            // previous lane's (or the carried) cell
            const int cx = cell_round(q.x), cy = cell_round(q.y);
            int px = __shfl_up_sync(full, cx, 1), py = __shfl_up_sync(full, cy, 1);
            if (lane == 0) { px = cqx; py = cqy; }
            const int cls = meta & 3;
            const int e = meta >> 2;
            const bool seg = valid && cls >= 1;
            const int grp = seg && group ? group[e] : 0;
            const int32_t w = seg && weight ? weight[e] : 1;
            bin_or_splat_cells<int32_t>(seg, px, py, cx, cy, cls == 1 ? 0 : 1, w, grp, hist,
                                        plane, nv, nu, status, tiles);
            cqx = __shfl_sync(full, cx, cnt - 1);
            cqy = __shfl_sync(full, cy, cnt - 1);
        }
        F += cnt;
        __syncwarp();
    };

    // Inside the range everything is 32-bit and relative: inputs j - J_a,
    // edges e - e0, outputs G - O_a (point counts are below 2^31, checked on
    // the host by every pass that produces them).
    const double2 *pts_r = pts + J_a;
    const int32_t *pos_r = pos + J_a;
    const int64_t *st_r = starts + e0;
    const int64_t *ns_r = new_starts + e0;
    const int JN = (int)(J_b - J_a), EN = (int)(e1 - e0);
    // chunk [jn, jn + 32) of the range, jn's edge en -> R.c* (one cp.async group)
    auto prefetch = [&](int jn, int en) {
        const int j = jn + lane;
        const bool in = j < JN;
        emit_cp(&R.cpts[lane], pts_r + (in ? j : 0), 16, in);
        emit_cp(&R.cpos[lane], pos_r + (in ? j : 0), 4, in);
        const int ek = en + 1 + lane;
        const bool ev = ek <= EN;
        emit_cp(&R.csv[lane], st_r + (ev ? ek : 0), 8, ev);
        emit_cp(&R.cnsv[lane], ns_r + (ev ? ek : 0), 8, ev);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    int e_c = 0;   // edge of input jc
    int ns_c = 0;  // its new_starts (relative to O_a = new_starts[e0])
    prefetch(0, 0);
    for (int jc = 0; jc < JN; jc += 32) {
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncwarp();
        const bool in = jc + lane < JN;
        const double2 x = R.cpts[lane];
        const int pj = in ? R.cpos[lane] : -1;
        // edges starting in (jc, jc + 31] (every edge has >= 1 input)
        const int ek = e_c + 1 + lane;
        const int rel = ek <= EN ? (int)(R.csv[lane] - J_a) - jc : INT_MAX;  // >= 1
        const unsigned smask = __reduce_or_sync(full, rel <= 31 ? (1u << rel) : 0u);
        int d = __popc(smask & (0xffffffffu >> (31 - lane)));  // e - e_c
        if (e_c + d > EN - 1) d = EN - 1 - e_c;
        const int e = e_c + d;
        const int nsb = d > 0 ? (int)(R.cnsv[d - 1] - O_a) : ns_c;
        const int nst = __popc(__ballot_sync(full, rel <= 32));
        if (nst) ns_c = (int)(R.cnsv[nst - 1] - O_a);
        __syncwarp();  // R.c* is refilled below
        e_c += nst;
        if (jc + 32 < JN) prefetch(jc + 32, e_c);
        const bool kept = pj >= 0;
        int g = -1;
        if (kept) {
            g = nsb + pj;
            if ((unsigned)g >= (unsigned)O_n) g = -1;  // (inconsistent inputs: write nothing)
        }
        const unsigned kb = __ballot_sync(full, g >= 0);
        // previous kept input: nearest kept lane below, else the carry
        const unsigned lower = kb & lt_mask;
        const int pl = lower ? 31 - __clz(lower) : 0;
        double2 a = make_double2(__shfl_sync(full, x.x, pl), __shfl_sync(full, x.y, pl));
        int ga = __shfl_sync(full, g, pl);
        if (!lower) { a = ca; ga = cg; }
        if (kb) {
            const int L = 31 - __clz(kb);
            ca = make_double2(__shfl_sync(full, x.x, L), __shfl_sync(full, x.y, L));
            cg = __shfl_sync(full, g, L);
        }
        // this lane's outputs [nx, g]
        const bool own = g >= 0;
        int nx = own ? (pj == 0 ? g : ga + 1) : 1;
        const int last = own ? g : 0;
        const int pieces = g - ga;
        const int meta_hi = (int)(e0 + e) << 2;
        const int c_end = cg + 1;  // every output below is owned by a kept input seen so far
        for (;;) {
            const int limit = F + kRing;
            // write this lane's outputs below limit (warp-uniform trip count)
            int todo = (own && nx <= last) ? min(last, limit - 1) - nx + 1 : 0;
            for (int r = __reduce_max_sync(full, todo > 0 ? todo : 0); r > 0; --r) {
                if (todo > 0) {
                    const double2 q = nx == last ? x : interp_piece(a, x, nx - ga, pieces);
                    const int lm = pj - (last - nx);  // local index in the edge
                    R.q[nx & (kRing - 1)] = q;
                    R.meta[nx & (kRing - 1)] = meta_hi | (lm < 2 ? lm : 2);
                    ++nx;
                    --todo;
                }
            }
            // flush complete tiles
            const int done = min(c_end, limit);
            while (F + 32 <= done) flush(32);
            if (!__any_sync(full, own && nx <= last)) break;
        }
    }
    if (F < O_n) flush(O_n - F);
    }
}

// After a resample whose total exceeded the buffers (status bit set, nothing
// written), keep every later kernel in bounds: starts[e] = min(starts[e], cap).
// Two launches: entries below n_edges first (all read the untouched total),
// then the total itself (copied to total_out, nullable, before clamping).
__global__ void clamp_starts_kernel(int64_t *__restrict__ starts, int64_t n_edges, int64_t cap) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n_edges && starts[n_edges] > cap && starts[e] > cap) starts[e] = cap;
}
__global__ void clamp_total_kernel(int64_t *__restrict__ starts, int64_t n_edges, int64_t cap,
                                   int64_t *__restrict__ total_out) {
    const int64_t total = starts[n_edges];
    if (total_out) *total_out = total;
    if (total > cap) starts[n_edges] = cap;
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

int hb_edge_prepare(const double *node_pos, const int64_t *sources, const int64_t *targets,
                    int64_t n_edges, double origin_x, double origin_y, double cell, double delta,
                    double *src, double *dst, int64_t *counts, void *stream) {
    if (n_edges < 0 || !(cell > 0) || !(delta > 0) ||
        (n_edges > 0 && (!node_pos || !sources || !targets || !src || !dst || !counts)))
        return set_error(HB_EINVAL, "hb_edge_prepare: bad arguments");
    if (n_edges == 0) return HB_OK;
    edge_prepare_kernel<<<(unsigned)((n_edges + 255) / 256), 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const double2 *>(node_pos), sources, targets, n_edges, origin_x,
        origin_y, cell, delta, reinterpret_cast<double2 *>(src), reinterpret_cast<double2 *>(dst),
        counts);
    return check_launch("hb_edge_prepare");
}

int hb_to_world_nodes(const double *pts, const int64_t *starts, int64_t n_edges, double origin_x,
                      double origin_y, double cell, const double *node_pos,
                      const int64_t *sources, const int64_t *targets, double *out,
                      void *stream) {
    if (n_edges < 0 ||
        (n_edges > 0 && (!pts || !starts || !out || !node_pos || !sources || !targets)))
        return set_error(HB_EINVAL, "hb_to_world_nodes: bad arguments");
    if (n_edges == 0) return HB_OK;
    to_world_nodes_kernel<<<warp_blocks(n_edges, 256), 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const double2 *>(pts), starts, n_edges, origin_x, origin_y, cell,
        reinterpret_cast<const double2 *>(node_pos), sources, targets,
        reinterpret_cast<double2 *>(out));
    return check_launch("hb_to_world_nodes");
}

int hb_splat(const double *pts, const int64_t *starts, int64_t n_edges, int64_t n_pts,
             const int32_t *group, const int32_t *weight, int32_t *counts, int nbins,
             int nv, int nu, int32_t *status, const hb_tiles *tiles, void *stream) {
    if (n_edges < 0 || n_pts < 0 || nbins < 1 || nv < 1 || nu < 1 || nv > kMaxDim || nu > kMaxDim || !counts || !status ||
        (n_edges > 0 && (!pts || !starts || !group)))
        return set_error(HB_EINVAL, "hb_splat: bad arguments");
    if (n_edges == 0 || n_pts == 0) return HB_OK;
    splat_kernel<int32_t><<<persistent_grid(splat_kernel<int32_t>, n_edges), kStreamBlock, 0,
                            as_stream(stream)>>>(
        reinterpret_cast<const double2 *>(pts), starts, n_edges, group, weight, counts,
        (int64_t)nv * nu, nv, nu, status, tiles ? *tiles : hb_tiles{}, tiles != nullptr);
    return check_launch("hb_splat");
}

int hb_resample_count(const double *pts, const int64_t *starts, int64_t n_edges,
                      double delta, int64_t *counts, int32_t *pos, void *stream) {
    if (n_edges < 0 || !(delta > 0) || (n_edges > 0 && (!pts || !starts || !counts || !pos)))
        return set_error(HB_EINVAL, "hb_resample_count: bad arguments");
    if (n_edges == 0) return HB_OK;
    PolylinePass pp{};
    pp.pin = reinterpret_cast<const double2 *>(pts);
    pp.starts = starts;
    pp.n_edges = n_edges;
    pp.h = -1.0;  // no advection, no Laplacian: count only
    pp.delta = delta;
    pp.counts = counts;
    pp.pos = pos;
    return launch_polyline_pass(pp, as_stream(stream), "hb_resample_count");
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

int hb_resample_emit_cap(const double *pts, const int64_t *starts, int64_t n_edges,
                         int64_t n_pts, const int32_t *pos, const int64_t *new_starts,
                         double *out, int64_t out_capacity, const int32_t *group,
                         const int32_t *weight, int32_t *counts, int nv, int nu, int32_t *status,
                         const hb_tiles *tiles, void *stream) {
    if (n_edges < 0 || n_pts < 0 || out_capacity < 0 ||
        (n_edges > 0 && (!pts || !starts || !pos || !new_starts || !out)) ||
        ((counts || out_capacity < INT64_MAX) && !status) ||
        (counts && (nv < 1 || nu < 1 || nv > kMaxDim || nu > kMaxDim)))
        return set_error(HB_EINVAL, "hb_resample_emit: bad arguments");
    if (n_edges == 0 || n_pts == 0) return HB_OK;
    static void *work_of[64] = {};  // the counter's address per device
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64)
        return check_launch("hb_resample_emit(device)", 0);
    if (!work_of[dev] && cudaGetSymbolAddress(&work_of[dev], g_emit_next) != cudaSuccess)
        return check_launch("hb_resample_emit(symbol)", 0);
    if (cudaMemsetAsync(work_of[dev], 0, sizeof(unsigned long long), as_stream(stream)) !=
        cudaSuccess)
        return check_launch("hb_resample_emit(memset)", 0);
    emit_ring_kernel<<<persistent_grid(emit_ring_kernel, (n_pts + 31) / 32), kStreamBlock, 0,
                       as_stream(stream)>>>(
        reinterpret_cast<const double2 *>(pts), starts, n_edges, pos, new_starts,
        reinterpret_cast<double2 *>(out), group, weight, counts, (int64_t)nv * nu, nv, nu,
        status, tiles ? *tiles : hb_tiles{}, (counts && tiles) ? 1 : 0, out_capacity);
    return check_launch("hb_resample_emit");
}

int hb_resample_emit(const double *pts, const int64_t *starts, int64_t n_edges,
                     int64_t n_pts, const int32_t *pos, const int64_t *new_starts,
                     double *out, const int32_t *group, const int32_t *weight,
                     int32_t *counts, int nv, int nu, int32_t *status, const hb_tiles *tiles,
                     void *stream) {
    return hb_resample_emit_cap(pts, starts, n_edges, n_pts, pos, new_starts, out, INT64_MAX,
                                group, weight, counts, nv, nu, status, tiles, stream);
}

int hb_clamp_starts(int64_t *starts, int64_t n_edges, int64_t cap, int64_t *total_out,
                    void *stream) {
    if (n_edges < 0 || !starts || cap < 0) return set_error(HB_EINVAL, "hb_clamp_starts: bad arguments");
    if (n_edges > 0)
        clamp_starts_kernel<<<(unsigned)((n_edges + 255) / 256), 256, 0, as_stream(stream)>>>(
            starts, n_edges, cap);
    clamp_total_kernel<<<1, 1, 0, as_stream(stream)>>>(starts, n_edges, cap, total_out);
    return check_launch("hb_clamp_starts", n_edges > 0 ? 2 : 1);
}

}  // extern "C"
