// hb_lapcount.cu -- Jacobi Laplacian (_kernels.py:275-296) fused with the
// next iteration's resample count (_kernels.py:203-232), lane-sequential.
//
// resample_count walks each polyline keeping `a`, the last KEPT point:
// point j (not the last) merges when |p_j - a| < 0.5*delta, a kept point
// gets pieces = 2^k (halve g while g > 1.5*delta) and its output index is
// the running sum.  The walk is sequential, so instead of resolving it with
// warp ballots (one round per merge chain, ~400 warp instructions per 32
// points) every lane walks its own run of kRun consecutive points in order,
// like the reference, at ~20 instructions per point:
//
//   * Each warp owns a contiguous, edge-aligned range of the packed points
//     (balanced by point count) and takes it in groups of 32 runs x kRun,
//     staged through shared memory (coalesced global traffic; lanes walk
//     rows of a padded [run][point] table without bank conflicts).
//   * Edge starts of the group come from one window of `starts` per group;
//     run k's bits mark its starts and ends.
//   * Phase B: every lane walks its run: Laplacian from a sliding window of
//     the original points (run-boundary values are read before any lane
//     writes, so pts_out may alias pts_in), then the keep/merge step.  A
//     lane's run starts mid-edge with an unknown anchor: it SPECULATES that
//     the point just before its run was kept (anchor = that point's final
//     position, output offset 0 relative to it).  Lane 0 starts from the
//     exact state carried over from the previous group.
//   * Phase C: the speculation is right whenever that point was truly kept.
//     Otherwise the lane re-walks from the true anchor until its decision
//     sequence meets the speculative one at a point kept in both runs;
//     from there both walks are identical (same anchor), so only a constant
//     offset separates them.  Non-convergence inside a run (a merge chain
//     longer than the run) changes that lane's end state and is re-checked
//     for the next lane until stable.  A segmented scan over the lanes then
//     turns the relative output offsets into absolute ones.
//   * Final points and pos leave through the same shared tables, coalesced;
//     counts are written at each polyline's last point.
//
// Every comparison and every floating-point operation is the reference's,
// in its order (squared gaps against the exact sqrt thresholds, see
// sqrt_lt_bound), so pos/counts are bit-identical to a sequential walk.
#include "hb_common.cuh"

namespace hb {

struct LapCount {
    const double2 *pin = nullptr;
    double2 *pout = nullptr;  // may alias pin
    const int64_t *starts = nullptr;
    int64_t n_edges = 0, n_pts = 0;
    double factor = 0.5;
    int lap = 1;
    double delta = 1.0;
    int64_t *counts = nullptr;  // nullable: Laplacian only
    int32_t *pos = nullptr;
    // fused advection (hb_advect_laplacian_count): _kernels.advect on each
    // staged group before its Laplacian
    const int32_t *edge_layer = nullptr;
    const float *rho = nullptr;
    const float4 *gf = nullptr;
    int nbins = 1;
    unsigned plane = 0;
    int nv = 0, nu = 0;
    double xhi = 0.0, yhi = 0.0, h = 0.0, eps = 1e-8, min_step = 0.25;
    int fixed = 0;
    unsigned long long *moved = nullptr;
    double *partials = nullptr;
};

// Deferral queue of the fused advection, per warp (see hb_advect_flat.cu):
// points whose step search did not finish with the first candidate wait here
// with their exact state and are finished 32 at a time.
constexpr int kAQCap = 64;
struct AdvQueue {
    double dx[kAQCap], dy[kAQCap], r0[kAQCap], m[kAQCap];
    unsigned base[kAQCap];
    int slot[kAQCap];  // 0..255: row_pt[slot / kRun][slot % kRun]; 256: the halo point
};

constexpr int kLCBlock = 256;
constexpr int kLCWarps = kLCBlock / 32;
// Measured on config 4 (ms/iteration, run x min blocks): 32x1 4.91, 16x2
// 3.28, 8x3 2.77, 8x4 2.54, 6x4 2.91, 4x4 3.40 (the ballot walk: 3.99).
#ifndef HB_LC_RUN
#define HB_LC_RUN 8
#endif
constexpr int kRun = HB_LC_RUN;       // points per lane per group
constexpr int kGroup = 32 * kRun;     // points per warp per group
constexpr int kRowPad = kRun + 1;     // odd row stride: column walks are conflict-free
static_assert(kRun >= 2 && kRun <= 32, "run length");

#ifndef HB_LC_CPASYNC
#define HB_LC_CPASYNC 1
#endif

#ifndef HB_LC_MINB
#define HB_LC_MINB 4
#endif

__device__ __forceinline__ double2 lap_point(double2 l, double2 c, double2 r, double f) {
    // _kernels.py:290-293: mx = 0.5*(p[j-1]+p[j+1]); s = p + f*(mx - p)
    const double mx = dmul(0.5, dadd(l.x, r.x));
    const double my = dmul(0.5, dadd(l.y, r.y));
    return make_double2(dadd(c.x, dmul(f, dsub(mx, c.x))), dadd(c.y, dmul(f, dsub(my, c.y))));
}

__device__ __forceinline__ int pieces_of(double g2, double hi2) {
    // while (g > hi) { g *= 0.5; pieces *= 2; } on squared gaps (4^k scaling);
    // one compare for the common single piece
    if (!(g2 > hi2)) return 1;
    double t = dmul(hi2, 4.0);
    int pieces = 2;
    while (g2 > t) {
        t = dmul(t, 4.0);
        pieces *= 2;
    }
    return pieces;
}

// The advection of one staged group (_kernels.py:144-200), as the flat
// advect does it: round k gives lane l the point base + 1 + 32k + l (the last
// is the halo, base + kGroup); one step candidate per lane, unfinished
// searches wait in the queue with their exact state and are finished in
// full-warp rounds; the queue is drained before the Laplacian reads the group.
template <int ADV>
__device__ __forceinline__ void advect_group(const LapCount &p, double2 (*row_pt)[kRowPad],
                                             double2 *s_halo, AdvQueue *aq, int64_t base, int n,
                                             int64_t P1, unsigned mask, unsigned ends,
                                             int64_t e_first, bool start_next, bool end_next,
                                             unsigned &my_moved, double &my_disp) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const bool sn = __shfl_sync(full, start_next ? 1 : 0, 31) != 0;
    const bool en_ = __shfl_sync(full, end_next ? 1 : 0, 31) != 0;
    const double min_step = p.min_step;
    auto slot_ptr = [&](int sl) -> double2 * {
        return sl < kGroup ? &row_pt[sl / kRun][sl % kRun] : s_halo;
    };
    auto test = [&](unsigned lb, double x, double y, double dx, double dy, double m, double r0,
                    double &nx, double &ny) -> bool {
        nx = clamp_ref(dadd(x, dmul(m, dx)), 1.0, p.xhi);
        ny = clamp_ref(dadd(y, dmul(m, dy)), 1.0, p.yhi);
        const double v = ADV == 1 ? bilinear_quad<true>(p.gf, lb, p.nv, p.nu, nx, ny)
                                  : bilinear_ref(p.rho + lb, p.nv, p.nu, nx, ny);
        return v >= r0;
    };
    auto accept = [&](int sl, double x, double y, double nx, double ny) {
        if (nx != x || ny != y) {  // _kernels.py:187-190
            *slot_ptr(sl) = make_double2(nx, ny);
            ++my_moved;
            my_disp = dadd(my_disp, hypot_ref(dsub(nx, x), dsub(ny, y)));
        }
    };
    int qn = 0;
    auto queue_round = [&](int take, int rounds) {
        const bool have = lane < take;
        const int q = qn - take + lane;
        double dx = 0.0, dy = 0.0, r0 = 0.0, m = -1.0;
        unsigned lb = 0;
        int sl = 0;
        if (have) {
            dx = aq->dx[q]; dy = aq->dy[q]; r0 = aq->r0[q]; m = aq->m[q];
            lb = aq->base[q]; sl = aq->slot[q];
        }
        qn -= take;
        __syncwarp();
        double x = 0.0, y = 0.0;
        if (have) {
            const double2 pt = *slot_ptr(sl);
            x = pt.x;
            y = pt.y;
        }
        for (int k = 0; have && (rounds < 0 || k < rounds) && m >= min_step; ++k) {
            double nx, ny;
            if (test(lb, x, y, dx, dy, m, r0, nx, ny)) {
                accept(sl, x, y, nx, ny);
                m = -1.0;
                break;
            }
            m = dmul(m, 0.5);
        }
        const bool pend = have && m >= min_step;
        const unsigned pm = __ballot_sync(full, pend);
        if (pend) {
            const int w = qn + __popc(pm & lt_mask);
            aq->dx[w] = dx; aq->dy[w] = dy; aq->r0[w] = r0; aq->m[w] = m;
            aq->base[w] = lb; aq->slot[w] = sl;
        }
        qn += __popc(pm);
        __syncwarp();
    };
    for (int rd = 0; rd < kGroup / 32; ++rd) {
        const int i = 1 + rd * 32 + lane;  // group index of this lane's point
        const int r = i / kRun < 31 ? i / kRun : 31, t = i % kRun;
        const unsigned mr = __shfl_sync(full, mask, r), er = __shfl_sync(full, ends, r);
        const int64_t efr = __shfl_sync(full, e_first, r);
        bool inter;
        int64_t e;
        if (i < kGroup) {
            inter = i < n && !((mr >> t) & 1u) && !((er >> t) & 1u);
            e = efr + __popc(mr & ((2u << t) - 1u) & ~1u);
        } else {  // the halo point, base + kGroup
            inter = base + kGroup < P1 && !sn && !en_;
            e = efr + __popc(mr & ~1u) + (sn ? 1 : 0);
        }
        const unsigned lb = (p.nbins > 1 && inter) ? (unsigned)p.edge_layer[e] * p.plane : 0u;
        bool pend = false;
        double dx = 0.0, dy = 0.0, r0 = 0.0, m = -1.0;
        if (inter) {
            const double2 pt = *slot_ptr(i);
            const double x = pt.x, y = pt.y;
            double Gx, Gy;  // _kernels.py:163-175 (G = 2*gradient)
            if (ADV == 1)
                gradient2_value_quad(QuadField{p.gf, lb, quad_gy(p.gf, (uint64_t)p.nbins * p.plane)},
                                     p.nv, p.nu, x, y, Gx, Gy, r0);
            else
                gradient2_value_ref(p.rho + lb, p.nv, p.nu, x, y, Gx, Gy, r0);
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
            if (m >= min_step) {
                double nx, ny;
                if (test(lb, x, y, dx, dy, m, r0, nx, ny)) {
                    accept(i, x, y, nx, ny);
                    m = -1.0;
                } else {
                    m = dmul(m, 0.5);
                }
            }
            pend = m >= min_step;
        }
        const unsigned pm = __ballot_sync(full, pend);
        if (pm) {
            if (pend) {
                const int w = qn + __popc(pm & lt_mask);
                aq->dx[w] = dx; aq->dy[w] = dy; aq->r0[w] = r0; aq->m[w] = m;
                aq->base[w] = lb; aq->slot[w] = i;
            }
            qn += __popc(pm);
            __syncwarp();
            while (qn >= 32) queue_round(32, 1);
        }
    }
    while (qn > 0) queue_round(qn < 32 ? qn : 32, -1);  // the group must be final
}

// (the fused kernels' shared memory allows 3 blocks per SM: 85 registers)
template <bool COUNT, int ADV>  // ADV: 0 none, 1 quad field, 2 density gathers
__global__ void __launch_bounds__(kLCBlock, ADV ? 3 : HB_LC_MINB) lapcount_kernel(const LapCount p) {
    // per warp: the group's points as [run][point] (original, then final)
    // and its output codes; rows padded so lanes walking rows hit distinct banks
    extern __shared__ unsigned char lc_smem[];
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    double2 (*row_pt)[kRowPad] =
        reinterpret_cast<double2 (*)[kRowPad]>(lc_smem) + (size_t)wib * 32;
    int (*row_pos)[kRowPad] = reinterpret_cast<int (*)[kRowPad]>(
        lc_smem + sizeof(double2) * kLCWarps * 32 * kRowPad) + (size_t)wib * 32;
    // phase C's re-walk decisions (relative offsets, -1 = merged), so the
    // final write-out does not walk again
    int (*row_fix)[kRowPad] = reinterpret_cast<int (*)[kRowPad]>(
        lc_smem + (sizeof(double2) + sizeof(int)) * kLCWarps * 32 * kRowPad) + (size_t)wib * 32;
    // fused advection: the queue and the halo point (the next group's first
    // point, advected here because this group's Laplacian needs it)
    AdvQueue *aq = reinterpret_cast<AdvQueue *>(
        lc_smem + (sizeof(double2) + 2 * sizeof(int)) * kLCWarps * 32 * kRowPad) + wib;
    double2 *s_halo = reinterpret_cast<double2 *>(
        lc_smem + (sizeof(double2) + 2 * sizeof(int)) * kLCWarps * 32 * kRowPad +
        sizeof(AdvQueue) * kLCWarps) + wib;
    unsigned my_moved = 0;
    double my_disp = 0.0;
    const double lo2 = COUNT ? sqrt_lt_bound(0.5 * p.delta) : 0.0;  // _kernels.py:211-212
    const double hi2 = COUNT ? sqrt_gt_bound(1.5 * p.delta) : 0.0;
    constexpr unsigned run_bits = kRun == 32 ? 0xffffffffu : ((1u << kRun) - 1u);

    // edge-aligned point range of this warp
    const int64_t gw = ((int64_t)blockIdx.x * kLCBlock + threadIdx.x) >> 5;
    const int64_t nw = (int64_t)gridDim.x * kLCWarps;
    // the point count is read on the device (n_pts is the buffer bound)
    // points [starts[0], starts[n_edges]) (an edge sub-range may start anywhere)
    const int64_t P_lo = p.starts[0];
    const int64_t NP = p.starts[p.n_edges] < p.n_pts ? p.starts[p.n_edges] : p.n_pts;
    const int64_t span = NP > P_lo ? NP - P_lo : 0;
    int64_t e0 = 0, e1 = 0;
    if (lane == 0) {
        e0 = lower_edge(p.starts, p.n_edges, P_lo + (span * gw) / nw);
        e1 = lower_edge(p.starts, p.n_edges, P_lo + (span * (gw + 1)) / nw);
    }
    e0 = __shfl_sync(full, e0, 0);
    e1 = __shfl_sync(full, e1, 0);
    if (e0 < e1) {
    const int64_t P0 = p.starts[e0], P1 = p.starts[e1];

    int64_t e_g = e0;   // edge containing the group's first point
    int64_t s_g = P0;   // its start
    double2 carryA = make_double2(0.0, 0.0);  // original point base-1
    double2 c_anc = carryA;                   // exact count state after point base-1
    int c_off = 0;
    bool c_kept = true;

    for (int64_t base = P0; base < P1; base += kGroup) {
        const int n = (int)(P1 - base < kGroup ? P1 - base : kGroup);
        const double2 *pin = p.pin + base;
        // ---- stage the group coalesced: point i -> row i / kRun, column i % kRun
#if HB_LC_CPASYNC
        // global -> shared without a register round trip: all of the group's
        // loads are in flight at once (the starts scan below overlaps them)
        for (int i = lane; i < n; i += 32) {
            const unsigned sa = (unsigned)__cvta_generic_to_shared(&row_pt[i / kRun][i % kRun]);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(pin + i));
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
#else
        for (int i = lane; i < n; i += 32) row_pt[i / kRun][i % kRun] = pin[i];
#endif
        double2 next_first = make_double2(0.0, 0.0);  // original point base + kGroup
        if (lane == 31 && base + kGroup < P1) next_first = pin[kGroup];

        // ---- edge starts in (base, base + kGroup] -> per-run bit masks
        unsigned mask = 0u;       // starts at run positions 0..kRun-1
        bool start_next = false;  // (lane 31) point base + kGroup starts an edge
        bool end_next = false;    // point base + kGroup ends one
        int64_t e_scan = e_g + 1, s_last = s_g;
        int n_st = 0;
        for (;;) {
            const int64_t idx = e_scan + lane;
            const int64_t sv = idx <= e1 ? p.starts[idx] : INT64_MAX;
            const int64_t rel = sv - base;  // >= 1
            const unsigned in = __ballot_sync(full, rel <= kGroup);
            for (unsigned b = in; b; b &= b - 1) {
                const int i = __ffs(b) - 1;
                const int r = (int)__shfl_sync(full, rel, i);
                if (r < kGroup) {
                    if (r / kRun == lane) mask |= 1u << (r % kRun);
                } else if (lane == 31) {
                    start_next = true;
                }
            }
            const int c = __popc(in);
            n_st += c;
            if (c) s_last = __shfl_sync(full, sv, c - 1);
            if (in != full) {
                // (fused advection) does point base + kGroup end an edge?
                end_next = __shfl_sync(full, rel, c) == kGroup + 1;
                break;
            }
            e_scan += 32;
        }
        if (lane == 0 && s_g == base) mask |= 1u;
        // the run's last point ends an edge when the next run starts with one
        const unsigned nb0 = __shfl_down_sync(full, mask, 1) & 1u;
        const unsigned ends =
            ((mask >> 1) | ((lane == 31 ? (start_next ? 1u : 0u) : nb0) << (kRun - 1))) & run_bits;
        // edge of the run's first point: e_g + #starts in (0, kRun*lane]
        const unsigned mprime = lane == 0 ? (mask & ~1u) : mask;
        int incl = __popc(mprime);
        for (int d = 1; d < 32; d <<= 1) {
            const int o = __shfl_up_sync(full, incl, d);
            if (lane >= d) incl += o;
        }
        const int excl = incl - __popc(mprime);
        int64_t e_cur = e_g + excl + ((lane > 0 && (mask & 1u)) ? 1 : 0);
        const int64_t e_first = e_cur;
        const unsigned prev_mask = __shfl_up_sync(full, mask, 1);
#if HB_LC_CPASYNC
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
#endif
        __syncwarp();
        if (ADV) {
            // _kernels.advect (in place) on points base+1 .. base+kGroup; point
            // base was the previous group's halo (or starts the range: an
            // endpoint, never moved)
            if (lane == 0 && base != P0) row_pt[0][0] = *s_halo;
            if (lane == 31) *s_halo = next_first;
            __syncwarp();
            advect_group<ADV>(p, row_pt, s_halo, aq, base, n, P1, mask, ends, e_first,
                              start_next, end_next, my_moved, my_disp);
            __syncwarp();
            if (lane == 31) next_first = *s_halo;
        }

        // ---- run boundaries, read before any lane overwrites its row
        const int j0 = lane * kRun;
        const int len = n - j0 < 0 ? 0 : (n - j0 > kRun ? kRun : n - j0);
        double2 firstA = make_double2(0.0, 0.0), lastA = firstA, prevA = carryA,
                prev2 = firstA, nextA_end = next_first;
        if (len > 0) {
            firstA = row_pt[lane][0];
            lastA = row_pt[lane][len - 1];
            if (lane > 0) {
                prevA = row_pt[lane - 1][kRun - 1];
                prev2 = row_pt[lane - 1][kRun - 2];
            }
            if (lane < 31 && j0 + kRun < n) nextA_end = row_pt[lane + 1][0];
        }
        // speculative anchor: final position of point j0-1 (an endpoint when
        // it starts an edge or point j0 does)
        double2 spec_anc = prevA;
        if (COUNT && lane > 0 && len > 0 && p.lap && !((prev_mask >> (kRun - 1)) & 1u) &&
            !(mask & 1u))
            spec_anc = lap_point(prev2, prevA, firstA, p.factor);
        __syncwarp();

        // ---- phase B: Laplacian + speculative count, sequential per lane.
        // Offsets before the run's first edge start are relative to the
        // incoming anchor (0); from the first start on they are absolute.
        // Lane 0 starts from the exact carried state (absolute throughout).
        double2 anc = lane == 0 ? c_anc : spec_anc;
        int off = lane == 0 ? c_off : 0;
        bool seen_start = false, last_kept = lane == 0 ? c_kept : true;
        {
            double2 A = firstA, Al = prevA;
            // one point of the walk (full runs unroll it: no loop-carried select)
            auto walk = [&](int t, const double2 An) {
                const bool st = (mask >> t) & 1u, en = (ends >> t) & 1u;
                const double2 F = (p.lap && !st && !en) ? lap_point(Al, A, An, p.factor) : A;
                row_pt[lane][t] = F;
                if (COUNT) {
                    int pv = -1;
                    if (st) {
                        anc = F;
                        off = 0;
                        pv = 0;
                        last_kept = true;
                        if (t > 0) ++e_cur;
                        seen_start = true;
                    } else {
                        const double g2 = dist2_ref(F.x, F.y, anc.x, anc.y);
                        if (en || !(g2 < lo2)) {
                            off += pieces_of(g2, hi2);
                            anc = F;
                            pv = off;
                            last_kept = true;
                        } else {
                            last_kept = false;
                        }
                    }
                    if (en && (seen_start || lane == 0)) p.counts[e_cur] = (int64_t)off + 1;
                    row_pos[lane][t] = pv;
                }
                Al = A;
                A = An;
            };
            if (len == kRun) {
#pragma unroll
                for (int t = 0; t < kRun; ++t)
                    walk(t, t + 1 < kRun ? row_pt[lane][t + 1] : nextA_end);
            } else {
                for (int t = 0; t < len; ++t) walk(t, t + 1 < len ? row_pt[lane][t + 1] : nextA_end);
            }
        }
        const int lastlane = (n - 1) / kRun;
        int val = off;
        bool end_kept = last_kept;
        double2 end_anc = anc;
        if (COUNT) {
            // ---- phase C: lanes whose speculative anchor was wrong.
            // Exact: lane 0, empty runs, runs that begin with an edge start.
            const bool exact = (lane == 0) || len == 0 || (mask & 1u);
            const int t_fs = seen_start ? __ffs(mask) - 1 : len;  // first start in the run
            int end_rel = off;  // relative unless seen_start / lane 0
            bool fix = false;   // decisions before conv_t differ from phase B
            int conv_t = 0;     // first point after which the walks agree
            int shift = 0;      // true relative offset = phase-B offset + shift
            bool eval = !exact;
            for (int round = 0; round < 34; ++round) {
                const bool in_kept = __shfl_up_sync(full, end_kept ? 1 : 0, 1) != 0;
                const double2 in_anc = make_double2(__shfl_up_sync(full, end_anc.x, 1),
                                                    __shfl_up_sync(full, end_anc.y, 1));
                bool changed = false;
                if (eval) {
                    const double2 old_anc = end_anc;
                    const bool old_kept = end_kept;
                    if (in_kept) {  // point j0-1 truly kept: phase B was exact
                        fix = false;
                        conv_t = 0;
                        shift = 0;
                        end_anc = anc;
                        end_kept = last_kept;
                        end_rel = off;
                    } else {  // re-walk from the true anchor until the walks meet
                        fix = true;
                        double2 a2 = in_anc;
                        int o2 = 0, t = 0;
                        bool conv = false, k2 = false;
                        for (; t < t_fs; ++t) {
                            const double2 F = row_pt[lane][t];
                            const bool en = (ends >> t) & 1u;
                            const double g2 = dist2_ref(F.x, F.y, a2.x, a2.y);
                            k2 = en || !(g2 < lo2);
                            row_fix[lane][t] = -1;
                            if (k2) {
                                o2 += pieces_of(g2, hi2);
                                a2 = F;
                                row_fix[lane][t] = o2;
                                const int spv = row_pos[lane][t];
                                if (spv >= 0) {  // kept in both walks: identical from here
                                    conv = true;
                                    shift = o2 - spv;
                                    conv_t = t + 1;
                                    break;
                                }
                            }
                        }
                        if (!conv && t_fs < len) {  // the edge start resets the state
                            conv = true;
                            conv_t = t_fs;
                            shift = 0;
                        }
                        if (conv) {
                            end_anc = anc;
                            end_kept = last_kept;
                            end_rel = seen_start ? off : off + shift;
                        } else {  // one merge chain through the whole run
                            conv_t = len;
                            end_anc = a2;
                            end_kept = k2;
                            end_rel = o2;
                        }
                    }
                    changed = old_anc.x != end_anc.x || old_anc.y != end_anc.y ||
                              old_kept != end_kept;
                    eval = false;
                }
                const unsigned chg = __ballot_sync(full, changed);
                if (!chg) break;
                eval = !exact && (((chg << 1) >> lane) & 1u);  // predecessor changed
            }
            // absolute offsets: segmented scan, restarting at lanes whose end
            // offset is absolute (lane 0, or an edge start inside the run)
            val = end_rel;
            int flag = (lane == 0 || seen_start) ? 1 : 0;
            for (int d = 1; d < 32; d <<= 1) {
                const int ov = __shfl_up_sync(full, val, d);
                const int of = __shfl_up_sync(full, flag, d);
                if (lane >= d && !flag) {
                    val += ov;
                    flag = of;
                }
            }
            const int in_off = __shfl_up_sync(full, val, 1);  // offset of the incoming anchor
            if (!exact) {
                // before the first start: phase C's last re-walk (from the
                // final incoming anchor: a lane is re-evaluated whenever its
                // predecessor's end state changes) decides [0, conv_t);
                // phase B's values are shifted after it
                for (int t = 0; t < t_fs; ++t) {
                    int v = row_pos[lane][t];
                    if (fix && t < conv_t) {
                        v = row_fix[lane][t];
                    } else if (v >= 0) {
                        v += shift;
                    }
                    if (v >= 0) v += in_off;
                    row_pos[lane][t] = v;
                    if ((ends >> t) & 1u) p.counts[e_first] = (int64_t)v + 1;
                }
            }
        }
        __syncwarp();
        // ---- coalesced write-out of the final points (and output codes)
        for (int i = lane; i < n; i += 32) {
            p.pout[base + i] = row_pt[i / kRun][i % kRun];
            if (COUNT) p.pos[base + i] = row_pos[i / kRun][i % kRun];
        }
        __syncwarp();
        // ---- carry the exact state after the group's last point
        carryA = make_double2(__shfl_sync(full, lastA.x, lastlane), __shfl_sync(full, lastA.y, lastlane));
        if (COUNT) {
            c_anc = make_double2(__shfl_sync(full, end_anc.x, lastlane),
                                 __shfl_sync(full, end_anc.y, lastlane));
            c_off = __shfl_sync(full, val, lastlane);
            c_kept = __shfl_sync(full, end_kept ? 1 : 0, lastlane) != 0;
        }
        s_g = s_last;
        e_g += n_st;
    }
    }  // e0 < e1
    if (ADV) {
        // per-block metrics in a fixed order (deterministic for a fixed grid)
        __shared__ double red_d[kLCWarps];
        __shared__ unsigned red_m[kLCWarps];
        for (int o = 16; o; o >>= 1) {
            my_moved += __shfl_down_sync(full, my_moved, o);
            my_disp = dadd(my_disp, __shfl_down_sync(full, my_disp, o));
        }
        if (lane == 0) {
            red_d[wib] = my_disp;
            red_m[wib] = my_moved;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double sd = 0.0;
            unsigned long long sm = 0;
            for (int w = 0; w < kLCWarps; ++w) {
                sd = dadd(sd, red_d[w]);
                sm += red_m[w];
            }
            p.partials[blockIdx.x] = sd;
            if (sm) atomicAdd(p.moved, sm);
        }
    }
}

}  // namespace hb

using namespace hb;

// resident blocks (occupancy with this dynamic shared memory), never more
// warps than there are groups of points
template <typename K>
static unsigned lc_grid(K kernel, int64_t groups, size_t smem) {
    const int per_sm = resident_blocks(reinterpret_cast<const void *>(kernel), kLCBlock, smem);
    int64_t want = (groups + kLCWarps - 1) / kLCWarps;
    const int64_t cap = (int64_t)device_sm_count() * per_sm;
    if (want > cap) want = cap;
    return (unsigned)(want < 1 ? 1 : want);
}

template <bool COUNT, int ADV>
static int launch_lc(const LapCount &p, int64_t groups, size_t smem, cudaStream_t st) {
    if (cudaFuncSetAttribute(lapcount_kernel<COUNT, ADV>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return check_launch("hb_laplacian_count(smem)", 0);
    lapcount_kernel<COUNT, ADV>
        <<<lc_grid(lapcount_kernel<COUNT, ADV>, groups, smem), kLCBlock, smem, st>>>(p);
    return HB_OK;
}

extern "C" {

int hb_advect_laplacian_count(double *pts, const int64_t *starts, int64_t n_edges, int64_t n_pts,
                              const int32_t *edge_layer, const float *rho,
                              const float *grad_field, int nbins, int nv, int nu, double h,
                              double eps, double min_step, int fixed_step, double lap_factor,
                              int lap_passes, double delta, int64_t *counts, int32_t *pos,
                              unsigned long long *moved, double *disp_partials, void *stream) {
    if (n_edges < 0 || n_pts < 0 || lap_passes < 0 || lap_passes > 1 || nbins < 1 || nv < 3 ||
        nu < 3 || nv > kMaxDim || nu > kMaxDim || !moved || !disp_partials || !(h >= 0.0) ||
        (counts && (!pos || !(delta > 0))) ||
        (n_pts > 0 && n_edges > 0 && (!pts || !starts || !edge_layer || !rho)))
        return set_error(HB_EINVAL, "hb_advect_laplacian_count: bad arguments");
    if ((int64_t)nbins * nv * nu >= ((int64_t)1 << 31) ||
        (grad_field && (int64_t)kQuadRec * nbins * nv * nu >= ((int64_t)1 << 32)))
        return set_error(HB_EINVAL, "hb_advect_laplacian_count: field above 2^31 cells");
    if (n_pts >= ((int64_t)1 << 31))
        return set_error(HB_EINVAL, "hb_advect_laplacian_count: more than 2^31 points");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(disp_partials, 0, sizeof(double) * kMaxStreamBlocks, st) != cudaSuccess)
        return check_launch("hb_advect_laplacian_count(memset)", 0);
    if (n_pts == 0 || n_edges == 0) return HB_OK;
    LapCount p;
    p.pin = reinterpret_cast<const double2 *>(pts);
    p.pout = reinterpret_cast<double2 *>(pts);
    p.starts = starts;
    p.n_edges = n_edges;
    p.n_pts = n_pts;
    p.factor = lap_factor;
    p.lap = lap_passes;
    p.delta = delta;
    p.counts = counts;
    p.pos = pos;
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
    const int64_t groups = (n_pts + kGroup - 1) / kGroup;
    const size_t smem = (size_t)kLCWarps * 32 * kRowPad * (sizeof(double2) + 2 * sizeof(int)) +
                        (sizeof(AdvQueue) + sizeof(double2)) * kLCWarps;
    int rc;
    if (p.gf)
        rc = counts ? launch_lc<true, 1>(p, groups, smem, st) : launch_lc<false, 1>(p, groups, smem, st);
    else
        rc = counts ? launch_lc<true, 2>(p, groups, smem, st) : launch_lc<false, 2>(p, groups, smem, st);
    if (rc) return rc;
    return check_launch("hb_advect_laplacian_count");
}

int hb_laplacian_count(const double *pts_in, double *pts_out, const int64_t *starts,
                       int64_t n_edges, int64_t n_pts, double lap_factor, int lap_passes,
                       double delta, int64_t *counts, int32_t *pos, void *stream) {
    if (n_edges < 0 || n_pts < 0 || lap_passes < 0 || (counts && (!pos || !(delta > 0))) ||
        (n_pts > 0 && (!pts_in || !pts_out || !starts)))
        return set_error(HB_EINVAL, "hb_laplacian_count: bad arguments");
    if (n_pts == 0 || n_edges == 0) return HB_OK;
    if (n_pts >= ((int64_t)1 << 31))
        return set_error(HB_EINVAL, "hb_laplacian_count: more than 2^31 points");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const double *src = pts_in;
    // all but the last Jacobi sweep: in-place streaming sweeps
    for (int q = 0; q + 1 < lap_passes; ++q) {
        PolylinePass sweep{};
        sweep.pin = reinterpret_cast<const double2 *>(src);
        sweep.pout = reinterpret_cast<double2 *>(pts_out);
        sweep.starts = starts;
        sweep.n_edges = n_edges;
        sweep.h = -1.0;
        sweep.factor = lap_factor;
        sweep.lap = 1;
        sweep.delta = delta;
        const int rc = launch_polyline_pass(sweep, st, "hb_laplacian_count(sweep)");
        if (rc) return rc;
        src = pts_out;
    }
    if (!counts && lap_passes == 0) {
        if (src != pts_out &&
            cudaMemcpyAsync(pts_out, src, sizeof(double) * 2 * (size_t)n_pts,
                            cudaMemcpyDeviceToDevice, st) != cudaSuccess)
            return check_launch("hb_laplacian_count(copy)", 0);
        return HB_OK;
    }
    LapCount p;
    p.pin = reinterpret_cast<const double2 *>(src);
    p.pout = reinterpret_cast<double2 *>(pts_out);
    p.starts = starts;
    p.n_edges = n_edges;
    p.n_pts = n_pts;
    p.factor = lap_factor;
    p.lap = lap_passes > 0 ? 1 : 0;
    p.delta = delta;
    p.counts = counts;
    p.pos = pos;
    const int64_t groups = (n_pts + kGroup - 1) / kGroup;
    const size_t smem = (size_t)kLCWarps * 32 * kRowPad * (sizeof(double2) + 2 * sizeof(int));
    const int rc = counts ? launch_lc<true, 0>(p, groups, smem, st)
                          : launch_lc<false, 0>(p, groups, smem, st);
    if (rc) return rc;
    return check_launch("hb_laplacian_count");
}

}  // extern "C"
