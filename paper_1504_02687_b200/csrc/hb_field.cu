// hb_field.cu -- density-field kernels: layer mixing, the 3-pass box-filter
// Gaussian approximation, layer peaks and used-cell counting.
//
// Exactness: each box pass of the reference builds a
// float64 integral image with two strict left folds -- down every column,
// then along every row (np.cumsum axis 0 then axis 1, raster.py:133-139) --
// and takes ((T11 - T01) - T10) + T00 divided by the full window area
// (raster.py:147-169).  Pass inputs after the first are non-integer float32
// values, so the fold ORDER decides the last bits of the table; we keep the
// reference's order exactly:
//   fold     : both folds in one cooperative launch (fold_kernel: column
//              strips, C tiles handed from column lanes to row lanes in
//              shared memory, row carries handed between strips); the two
//              kernels below when the strips cannot all be co-resident:
//   col_fold : one lane per (layer, column), sequential in v; 32-row tiles
//              stream through a 4-deep cp.async ring, rows stored coalesced
//   row_scan : one lane per (layer, row), 32x32 tiles through a 4-deep
//              cp.async ring so global traffic stays coalesced, sequential in u
//   box      : one thread per cell, 4 table gathers, IEEE divide, f32 round
#include "hb_common.cuh"

namespace hb {

// Layer mixing of the per-group histograms (int32 counts or float32 sums):
// H[l] = float32(sum_b M[l,b] * G[b]) (float64 sum in ascending b, one
// rounding -- exact whenever the reference's float32 sums are exact,
// SURVEY §8a).  M == NULL means identity.
template <typename T>
__device__ __forceinline__ float mixed_value(const T *__restrict__ g, const float *__restrict__ mat,
                                             int nb, int l, int64_t plane, int64_t off) {
    if (!mat) return (float)g[l * plane + off];
    double acc = 0.0;
    for (int b = 0; b < nb; ++b)
        acc = dadd(acc, dmul((double)__ldg(mat + l * nb + b), (double)g[b * plane + off]));
    return __double2float_rn(acc);
}

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
// 16 / 4 bytes, zero-filled (nothing read) when !ok
__device__ __forceinline__ void cp_async16z(void *smem, const void *gmem, bool ok) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem),
                 "r"(ok ? 16 : 0));
}
__device__ __forceinline__ void cp_async4z(void *smem, const void *gmem, bool ok) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem),
                 "r"(ok ? 4 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Column fold, C[v][u] = C[v-1][u] + (double)L[v][u] strictly in v.  A warp
// owns 32*CPL columns (lane = column, CPL independent chains per lane so the
// float64 add latency of one chain hides behind the others) and streams them
// in 32-row tiles through a kColStages-deep cp.async ring in shared memory;
// every row of C leaves as coalesced 256-byte stores.
#ifndef HB_COL_STAGES
#define HB_COL_STAGES 4
#endif
constexpr int kColStages = HB_COL_STAGES;
// 1 column per lane measured best (config 4 column fold: 20.5 us vs 30.8 us
// with 2 -- more warps beat interleaved chains on this latency-bound fold)
#ifndef HB_COL_CPL
#define HB_COL_CPL 1
#endif
constexpr int kColCPL = HB_COL_CPL;
constexpr int kColW = 32 * kColCPL;                       // columns per warp
#ifndef HB_COL_WARPS
#define HB_COL_WARPS (kColCPL == 1 ? 2 : 1)
#endif
constexpr int kColWarps = HB_COL_WARPS;  // kColWarps * kColStages * 4 KB <= 48 KB static smem

__global__ void __launch_bounds__(kColWarps * 32)
col_fold_kernel(const float *__restrict__ in, int nbins, int nv, int nu,
                double *__restrict__ table) {
    __shared__ __align__(16) float ring[kColWarps][kColStages][32][kColW];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ncg = (nu + kColW - 1) / kColW;
    const int64_t g = (int64_t)blockIdx.x * kColWarps + warp;  // column group
    if (g >= (int64_t)nbins * ncg) return;
    const int l = (int)(g / ncg), u0 = (int)(g % ncg) * kColW;
    const int64_t plane = (int64_t)nv * nu;
    const float *src = in + l * plane + u0;
    double *dst = table + l * plane + u0;
    const int ncols = nu - u0 < kColW ? nu - u0 : kColW;
    const bool vec = (nu % 4) == 0;  // rows 16-byte aligned
    const int ntiles = (nv + 31) / 32;
    auto issue = [&](int t) {
        if (t < ntiles) {
            float (*tt)[kColW] = ring[warp][t % kColStages];
            const int r0 = t * 32;
            if (vec) {  // a row is kColW/4 chunks of 16 B
                constexpr int chunks = kColW / 4, rows_per = 32 / chunks;
                const int ch = lane % chunks;
#pragma unroll
                for (int k = 0; k < 32 / rows_per; ++k) {
                    const int r = lane / chunks + rows_per * k;
                    const bool ok = r0 + r < nv && ch * 4 < ncols;
                    cp_async16z(&tt[r][ch * 4], ok ? src + (int64_t)(r0 + r) * nu + ch * 4 : src,
                                ok);
                }
            } else {
                for (int r = 0; r < 32; ++r)
#pragma unroll
                    for (int k = 0; k < kColCPL; ++k) {
                        const int cc = lane + 32 * k;
                        const bool ok = r0 + r < nv && cc < ncols;
                        cp_async4z(&tt[r][cc], ok ? src + (int64_t)(r0 + r) * nu + cc : src, ok);
                    }
            }
        }
        cp_async_commit();  // one group per tile, possibly empty: uniform wait counts
    };
#pragma unroll
    for (int t = 0; t < kColStages - 1; ++t) issue(t);
    double c[kColCPL];
#pragma unroll
    for (int k = 0; k < kColCPL; ++k) c[k] = 0.0;
    for (int t = 0; t < ntiles; ++t) {
        issue(t + kColStages - 1);
        cp_async_wait<kColStages - 1>();
        __syncwarp();
        const float (*tt)[kColW] = ring[warp][t % kColStages];
        const int r0 = t * 32;
        const int nr = nv - r0 < 32 ? nv - r0 : 32;
        double *d = dst + (int64_t)r0 * nu;
        if (nr == 32 && t > 0) {
            // full tile, unrolled: the CPL chains interleave, so only the
            // float64 adds of each chain are dependent
#pragma unroll
            for (int r = 0; r < 32; ++r) {
#pragma unroll
                for (int k = 0; k < kColCPL; ++k) {
                    c[k] = dadd(c[k], (double)tt[r][lane + 32 * k]);
                    if (lane + 32 * k < ncols) d[lane + 32 * k] = c[k];
                }
                d += nu;
            }
        } else {
            for (int r = 0; r < nr; ++r) {
#pragma unroll
                for (int k = 0; k < kColCPL; ++k) {
                    const double x = (double)tt[r][lane + 32 * k];
                    c[k] = (r0 + r == 0) ? x : dadd(c[k], x);
                    if (lane + 32 * k < ncols) d[lane + 32 * k] = c[k];
                }
                d += nu;
            }
        }
        __syncwarp();
    }
}

// Row fold in place, T[v][u] = T[v][u-1] + C[v][u] strictly in u.  Rows are
// flattened over (layer, v).  A warp owns 32 rows and walks them in 32x32
// tiles through a kRowStages-deep cp.async ring (rows padded to 33 doubles:
// the lanes' column walks hit distinct banks); each lane folds its own row
// of a tile left to right, then the tile is stored back coalesced.
#ifndef HB_ROW_STAGES
#define HB_ROW_STAGES 4
#endif
constexpr int kRowStages = HB_ROW_STAGES;

__global__ void __launch_bounds__(32)
row_scan_kernel(double *__restrict__ table, int64_t n_rows, int nu) {
    __shared__ double ring[kRowStages][32][33];
    const int lane = threadIdx.x & 31;
    const int64_t r0 = (int64_t)blockIdx.x * 32;
    if (r0 >= n_rows) return;
    const int nr = (int)(n_rows - r0 < 32 ? n_rows - r0 : 32);
    const int ntiles = (nu + 31) / 32;
    auto issue = [&](int t) {
        if (t < ntiles) {
            const int c0 = t * 32;
            const int nc = nu - c0 < 32 ? nu - c0 : 32;
            if (lane < nc)
                for (int i = 0; i < nr; ++i)
                    cp_async8(&ring[t % kRowStages][i][lane], table + (r0 + i) * nu + c0 + lane);
        }
        cp_async_commit();
    };
#pragma unroll
    for (int t = 0; t < kRowStages - 1; ++t) issue(t);
    double carry = 0.0;
    for (int t = 0; t < ntiles; ++t) {
        issue(t + kRowStages - 1);
        cp_async_wait<kRowStages - 1>();
        __syncwarp();
        double (*tt)[33] = ring[t % kRowStages];
        const int c0 = t * 32;
        const int nc = nu - c0 < 32 ? nu - c0 : 32;
        if (lane < nr) {
            double c = carry;
            if (nc == 32 && t > 0) {  // full tile, unrolled
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    c = dadd(c, tt[lane][k]);
                    tt[lane][k] = c;
                }
            } else {
                for (int k = 0; k < nc; ++k) {
                    c = (c0 + k == 0) ? tt[lane][k] : dadd(c, tt[lane][k]);
                    tt[lane][k] = c;
                }
            }
            carry = c;
        }
        __syncwarp();
        if (lane < nc)
            for (int i = 0; i < nr; ++i) table[(r0 + i) * nu + c0 + lane] = tt[i][lane];
        __syncwarp();
    }
}

// Row fold for even nu (16-byte aligned rows): rows padded to 34 doubles so
// 16-byte cp.async / LDS.128 / STS.128 all stay aligned and, in 8-lane
// phases, bank-conflict free; each lane folds its row two values per shared
// load, and tiles leave as 16-byte coalesced stores (two rows per warp
// instruction).
constexpr int kRowPad2 = 34;
__global__ void __launch_bounds__(32)
row_scan2_kernel(double *__restrict__ table, int64_t n_rows, int nu) {
    __shared__ __align__(16) double ring[kRowStages][32][kRowPad2];
    const int lane = threadIdx.x & 31;
    const int64_t r0 = (int64_t)blockIdx.x * 32;
    if (r0 >= n_rows) return;
    const int nr = (int)(n_rows - r0 < 32 ? n_rows - r0 : 32);
    const int ntiles = (nu + 31) / 32;
    const int half = lane >> 4, q = lane & 15;  // two rows per instruction, 16 x 16 B each
    auto issue = [&](int t) {
        if (t < ntiles) {
            const int c0 = t * 32;
            const int nc = nu - c0 < 32 ? nu - c0 : 32;  // even
            double (*tt)[kRowPad2] = ring[t % kRowStages];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const int i = 2 * k + half;
                const bool ok = i < nr && 2 * q < nc;
                cp_async16z(&tt[i][2 * q], ok ? table + (r0 + i) * nu + c0 + 2 * q : table, ok);
            }
        }
        cp_async_commit();
    };
#pragma unroll
    for (int t = 0; t < kRowStages - 1; ++t) issue(t);
    double carry = 0.0;
    for (int t = 0; t < ntiles; ++t) {
        issue(t + kRowStages - 1);
        cp_async_wait<kRowStages - 1>();
        __syncwarp();
        double (*tt)[kRowPad2] = ring[t % kRowStages];
        const int c0 = t * 32;
        const int nc = nu - c0 < 32 ? nu - c0 : 32;
        if (lane < nr) {
            double c = carry;
            double2 *tr = reinterpret_cast<double2 *>(tt[lane]);
            if (nc == 32 && t > 0) {
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const double2 x = tr[k];
                    const double a = dadd(c, x.x);
                    c = dadd(a, x.y);
                    tr[k] = make_double2(a, c);
                }
            } else {
                for (int k = 0; k < nc; ++k) {
                    c = (c0 + k == 0) ? tt[lane][k] : dadd(c, tt[lane][k]);
                    tt[lane][k] = c;
                }
            }
            carry = c;
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const int i = 2 * k + half;
            if (i < nr && 2 * q < nc)
                *reinterpret_cast<double2 *>(table + (r0 + i) * nu + c0 + 2 * q) =
                    *reinterpret_cast<const double2 *>(&tt[i][2 * q]);
        }
        __syncwarp();
    }
}

// ---- fused integral table: one cooperative pass per box pass ----------------
// The two folds above are strict sequential float64 chains (H steps down every
// column, W steps along every row); the critical path of the whole table is
// (H + W) dependent DADDs (~8.3 cycles each), ~17 us on a 2048^2 layer.  The
// separate kernels also round-trip C and T through DRAM (config-5 map:
// 40 + 49 us) and, on small maps, run far below the chain floor for lack of
// memory-level parallelism (config 4: 20 + 22 us against ~4 us).
//
// fold_kernel<S> computes T with both folds in one launch.  CTA (l, k) owns
// the S columns [kS, kS+S) of layer l for the full height:
//   * column warps (S/32): lane = column, the column fold C[v][u] = C[v-1][u]
//     + x[v][u] kept in a register, written 32 rows at a time into a C tile
//     (shared, kFoldSlots-deep ring); the next 32 rows are loaded ahead.
//   * row warps (8 - S/32): lane = row, each takes whole tiles (block b goes
//     to row warp b mod kRowWarps); the row fold starts from the carry
//     T[v][kS] of strip k-1 and walks the tile's S columns in order (the
//     reference's order), in place; the tile then leaves as coalesced rows of
//     T, and T[v][kS+S] is handed to strip k+1.
// Hand-off between strips: carry[l][k][v] is pre-filled with kFoldSentinel
// (a NaN bit pattern no finite sum can take), so the 8-byte value is its own
// ready flag -- one relaxed store, one relaxed poll, no fence; the single
// consumer re-arms it.  Strips wait on one another, so the launch is
// cooperative (all CTAs co-resident).  Order of every float64 operation is
// the reference's; only who performs it changes.
constexpr int kFoldThreads = 256;
constexpr unsigned long long kFoldSentinel = ~0ull;

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

#ifdef HB_FOLD_TRACE  // diagnostic build: per (strip, block) event times of layer 0
__device__ unsigned long long g_fold_trace[64][128][4];
__device__ __forceinline__ void fold_trace(int l, int k, int b, int e) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (l == 0 && k < 64 && b < 128) g_fold_trace[k][b][e] = t;
}
#else
__device__ __forceinline__ void fold_trace(int, int, int, int) {}
#endif

// (double)f as a volatile conversion: left to itself the compiler keeps the
// float and converts right before each add, which puts the F2F latency
// (~18 cycles) on the column chain; pinned here, the conversion happens
// where it is written (a block ahead of its add)
__device__ __forceinline__ double f2d_pinned(float f) {
    double d;
    asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(f));
    return d;
}

template <int S>
struct FoldCfg {
    static constexpr int kColWarps = S / 32;
    static constexpr int kRowWarps = kFoldThreads / 32 - kColWarps;
    static constexpr int kPitch = S + 1;  // doubles; row-lane column walks: 2 wavefronts
    static constexpr int kSlots = S >= 128 ? 5 : 8;   // C tiles in flight
    static constexpr int kStages = S >= 128 ? 4 : 8;  // x blocks prefetched (cp.async)
    static constexpr size_t kSmem = sizeof(double) * (size_t)kSlots * 32 * kPitch +
                                    sizeof(float) * (size_t)kStages * 32 * S;
};

template <int S>
__global__ void __launch_bounds__(kFoldThreads, 1)
fold_kernel(const float *__restrict__ in, int nv, int nu, int nstrips,
            double *__restrict__ table, unsigned long long *__restrict__ carry) {
    using C = FoldCfg<S>;
    extern __shared__ __align__(16) double ftile[];
    __shared__ int s_prod;               // C tiles produced (blocks 0 .. s_prod-1)
    __shared__ int s_free[C::kSlots];    // slot i last released by block s_free[i]-1
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int l = blockIdx.x / nstrips, k = blockIdx.x % nstrips;
    const int u0 = k * S;
    const int ncols = min(S, nu - u0);
    const int64_t plane = (int64_t)nv * nu;
    const int nblk = (nv + 31) / 32;
    if (threadIdx.x == 0) s_prod = 0;
    if (threadIdx.x < C::kSlots) s_free[threadIdx.x] = 0;
    __syncthreads();
    volatile int *vprod = &s_prod;
    volatile int *vfree = s_free;

    if (warp < C::kColWarps) {
        // ---- column fold ----
        const int t = threadIdx.x;  // column within the strip
        float *xs = reinterpret_cast<float *>(ftile + (size_t)C::kSlots * 32 * C::kPitch);
        const bool vec = (nu % 4) == 0;  // 16-byte rows (u0 is a multiple of 64)
        // vec: thread t copies the 16-byte chunk ch of rows r0, r0+4, ..., r0+28
        constexpr int kCpr = S / 4;  // chunks per row
        const int ch = t % kCpr, r0 = t / kCpr;
        const bool chok = ch * 4 < ncols;
        const float *gsrc = in + l * plane + u0 + (vec ? (int64_t)r0 * nu + ch * 4 : t);
        const int soff = vec ? r0 * S + ch * 4 : t;
        // x rows of block bb -> staging stage bb % kStages (zero past the grid)
        auto issue = [&](int bb) {
            if (bb < nblk) {
                float *st = xs + (size_t)(bb % C::kStages) * 32 * S + soff;
                const float *g = gsrc + (int64_t)bb * 32 * nu;
                const int vb = bb * 32;
                if (vec) {
#pragma unroll
                    for (int m = 0; m < 8; ++m) {
                        const bool okq = chok && vb + r0 + 4 * m < nv;
                        cp_async16z(st + 4 * m * S, okq ? g + (int64_t)4 * m * nu : gsrc, okq);
                    }
                } else {
                    for (int r = 0; r < 32; ++r) {
                        const bool okq = vb + r < nv && t < ncols;
                        cp_async4z(st + r * S, okq ? g + (int64_t)r * nu : gsrc, okq);
                    }
                }
            }
            cp_async_commit();  // one group per block, possibly empty
        };
        // Per block: the DADD chain of block b interleaved with widening block
        // b+1 (LDS + F2F fill the chain's latency gaps), so the per-block
        // critical path is the 32 dependent DADDs plus two barriers.
        double xa[32], xc[32];
        auto widen = [&](int bb, double (&xd)[32]) {
            const float *xb = xs + (size_t)(bb % C::kStages) * 32 * S + t;
#pragma unroll
            for (int i = 0; i < 32; ++i) xd[i] = f2d_pinned(xb[i * S]);
        };
#pragma unroll
        for (int d = 0; d < C::kStages - 1; ++d) issue(d);
        cp_async_wait<C::kStages - 2>();  // block 0 landed
        asm volatile("bar.sync 1, %0;" ::"r"(S));
        widen(0, xa);
        double c = 0.0;
        auto step = [&](int b, double (&cur)[32], double (&nxt)[32]) {
            cp_async_wait<C::kStages - 3>();  // block b+1 landed (this thread's copies)
            asm volatile("bar.sync 1, %0;" ::"r"(S));  // ... and every thread's
            const int slot = b % C::kSlots;
            while (vfree[slot] < b - C::kSlots + 1) __nanosleep(32);
            double *tile = ftile + (size_t)slot * 32 * C::kPitch + t;
            const float *xn = xs + (size_t)((b + 1) % C::kStages) * 32 * S + t;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                // np.cumsum: the first element as is
                c = (b == 0 && i == 0) ? cur[0] : dadd(c, cur[i]);
                tile[i * C::kPitch] = c;
                nxt[i] = f2d_pinned(xn[i * S]);  // (unused after the last block)
            }
            asm volatile("bar.sync 1, %0;" ::"r"(S));  // C tile complete
            if (t == 0) {
                __threadfence_block();
                *vprod = b + 1;
                fold_trace(l, k, b, 0);
            }
            issue(b + C::kStages - 1);  // refills the stage block b-1 used
        };
        for (int b = 0; b < nblk; b += 2) {
            step(b, xa, xc);
            if (b + 1 < nblk) step(b + 1, xc, xa);
        }
    } else {
        // ---- row fold ----
        const int rw = warp - C::kColWarps;
        unsigned long long *cin = carry + ((int64_t)l * nstrips + k) * nv;
        unsigned long long *cout = carry + ((int64_t)l * nstrips + k + 1) * nv;
        double *dst = table + l * plane + u0;
        for (int b = rw; b < nblk; b += C::kRowWarps) {
            const int v = b * 32 + lane;
            const bool rok = v < nv;
            while (*vprod <= b) __nanosleep(32);
            __threadfence_block();
            double *tile = ftile + (size_t)(b % C::kSlots) * 32 * C::kPitch;
            double *row = tile + lane * C::kPitch;
            // the first 32 C values of the row are loaded before the carry
            // arrives; later chunks load while the previous one folds, so the
            // fold is a pure DADD chain
            double cur[32];
            const bool full = ncols == S;
            if (full) {
#pragma unroll
                for (int j = 0; j < 32; ++j) cur[j] = row[j];
            }
            double tv = 0.0;
            if (k > 0) {
                unsigned long long bits = kFoldSentinel;
                if (rok) {
                    while ((bits = ld_relaxed_u64(cin + v)) == kFoldSentinel) {
                    }
                    st_relaxed_u64(cin + v, kFoldSentinel);  // re-arm for the next pass
                }
                tv = __longlong_as_double((long long)bits);
            }
            if (lane == 0) fold_trace(l, k, b, 1);
            if (full) {
#pragma unroll
                for (int c = 0; c < S / 32; ++c) {
                    double nxt[32];
                    if (c + 1 < S / 32) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) nxt[j] = row[32 * (c + 1) + j];
                    }
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        // np.cumsum along the row: the first element as is
                        tv = (k == 0 && c == 0 && j == 0) ? cur[0] : dadd(tv, cur[j]);
                        cur[j] = tv;
                    }
#pragma unroll
                    for (int j = 0; j < 32; ++j) row[32 * c + j] = cur[j];
                    if (c + 1 < S / 32) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) cur[j] = nxt[j];
                    }
                }
            } else {
                for (int j = 0; j < ncols; ++j) {
                    tv = (k == 0 && j == 0) ? row[0] : dadd(tv, row[j]);
                    row[j] = tv;
                }
            }
            if (k + 1 < nstrips && rok) st_relaxed_u64(cout + v, (unsigned long long)__double_as_longlong(tv));
            if (lane == 0) fold_trace(l, k, b, 2);
            __syncwarp();
            // the tile's rows of T, coalesced
            const int nr = min(32, nv - b * 32);
            if (nr == 32 && full) {
                // full tile: 8 rows of loads in flight, then their stores.  A
                // lane takes columns lane, lane+32, ...: every shared load and
                // global store is a contiguous 256-byte warp access (a 16-byte
                // pair per lane would read each wavefront half-used)
                double *d = dst + (int64_t)(b * 32) * nu + lane;
                const double *s = tile + lane;
#pragma unroll
                for (int i0 = 0; i0 < 32; i0 += 8) {
                    double q[8][S / 32];
#pragma unroll
                    for (int ii = 0; ii < 8; ++ii)
#pragma unroll
                        for (int m = 0; m < S / 32; ++m)
                            q[ii][m] = s[(i0 + ii) * C::kPitch + 32 * m];
#pragma unroll
                    for (int ii = 0; ii < 8; ++ii)
#pragma unroll
                        for (int m = 0; m < S / 32; ++m)
                            d[(int64_t)(i0 + ii) * nu + 32 * m] = q[ii][m];
                }
            } else if ((nu & 1) == 0) {  // 16-byte stores: a lane writes 2 columns of a row
#pragma unroll 8
                for (int i = 0; i < nr; ++i) {
                    double *d = dst + (int64_t)(b * 32 + i) * nu;
                    const double *s = tile + i * C::kPitch;
#pragma unroll
                    for (int m = 0; m < S / 64; ++m) {
                        const int col = 2 * lane + 64 * m;
                        if (col < ncols)
                            *reinterpret_cast<double2 *>(d + col) = make_double2(s[col], s[col + 1]);
                    }
                }
            } else {
                for (int i = 0; i < nr; ++i) {
                    double *d = dst + (int64_t)(b * 32 + i) * nu;
                    const double *s = tile + i * C::kPitch;
#pragma unroll
                    for (int m = 0; m < S / 32; ++m) {
                        const int col = lane + 32 * m;
                        if (col < ncols) d[col] = s[col];
                    }
                }
            }
            __syncwarp();
            if (lane == 0) {
                vfree[b % C::kSlots] = b + 1;
                fold_trace(l, k, b, 3);
            }
        }
    }
}

// 4-term box sum with zero row/column 0 implicit (table holds T[1:,1:]).
__device__ __forceinline__ double tz(const double *__restrict__ t, int nu, int r, int c) {
    return (r == 0 || c == 0) ? 0.0 : t[(int64_t)(r - 1) * nu + (c - 1)];
}

constexpr int kBoxBlock = 256;
#ifndef HB_BOX_ROWS
#define HB_BOX_ROWS 4  // measured on the config-5 map: 1 0.595, 2 0.552, 4 0.545, 8 0.582 ms per hb_smooth
#endif
constexpr int kBoxRows = HB_BOX_ROWS;  // output rows per thread (4 independent table loads each)

// Layer peak, max(rho, initial=0): non-negative floats order like their int
// bits.  One atomic per block, and none when the block's maximum does not
// exceed the peak already stored (the peak only grows, so the final value is
// the true maximum whatever the order).  A warp-level atomic per 32 cells
// onto B addresses serialised in L2: 0.36 ms of the config-5 smoothing.
__device__ __forceinline__ void block_peak(float *__restrict__ peak, float m) {
    __shared__ float s_max[32];
    for (int d = 16; d; d >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, d));
    const int warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    if ((threadIdx.x & 31) == 0) s_max[warp] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < nw; ++w) m = fmaxf(m, s_max[w]);
        if (m > 0.0f && m > *reinterpret_cast<volatile float *>(peak))
            atomicMax(reinterpret_cast<int *>(peak), __float_as_int(m));
    }
}

// float32(s / area) with the float64 quotient correctly rounded, as the
// reference computes it (raster.py:169), without a float64 divide per cell:
// q = s * (1/area) is within 2 ulp of the true quotient s/area, and rounding
// to float32 can only differ between the two when a float32 rounding
// midpoint (low 29 bits of the float64 significand == 2^28) lies within
// those ulps -- then, and for results near float32's subnormal range, the
// IEEE divide decides.  The divide was 60 % of the box pass's instructions.
__device__ __forceinline__ float box_quotient_f32(double s, double area, double inv_area) {
    const double q = dmul(s, inv_area);
    const unsigned low = (unsigned)(__double_as_longlong(q) & 0x1fffffffull);
    if (low - (0x10000000u - 8u) <= 16u || (q != 0.0 && fabs(q) < 0x1p-120))
        return __double2float_rn(__ddiv_rn(s, area));
    return __double2float_rn(q);
}

// Each thread produces kBoxRows cells of one column; all 4*kBoxRows table
// reads are issued before the first quotient.  Indices are 32-bit (every
// plane is < 2^31 cells) and the zero row/column of the table is a select,
// so a cell costs ~4 address ops + 4 loads + 3 DADD + the quotient (the
// 64-bit index arithmetic of a generic gather was ~110 warp instructions per
// 32 cells, and issue-bound).
__global__ void __launch_bounds__(kBoxBlock)
box_kernel(const double *__restrict__ table, int nv, int nu, int radius,
           float *__restrict__ out, float *__restrict__ peak) {
    const int u = blockIdx.x * kBoxBlock + threadIdx.x;
    const int vb = blockIdx.y * kBoxRows;
    const int l = blockIdx.z;
    float m = 0.0f;
    if (u < nu) {
        const int64_t plane = (int64_t)nv * nu;
        // T[i][j] (i, j >= 1) at byte (i*nu + j) * 8 from tb; unsigned indices
        // so every address is one IMAD.WIDE.U32
        const char *tb = reinterpret_cast<const char *>(table + l * plane - nu - 1);
        auto T = [&](unsigned i, unsigned j) {
            return *reinterpret_cast<const double *>(tb + (size_t)(i * (unsigned)nu + j) * 8u);
        };
        const int c0 = min(max(u - radius, 0), nu), c1 = min(u + radius + 1, nu);  // c1 >= 1
        const double area = (double)((2 * radius + 1) * (2 * radius + 1));
        const double inv_area = __drcp_rn(area);
        double t11[kBoxRows], t01[kBoxRows], t10[kBoxRows], t00[kBoxRows];
#pragma unroll
        for (int k = 0; k < kBoxRows; ++k) {
            const int v = min(vb + k, nv - 1);
            const int r0 = max(v - radius, 0), r1 = min(v + radius + 1, nv);  // r1 >= 1
            t11[k] = T(r1, c1);
            t10[k] = c0 ? T(r1, c0) : 0.0;
            t01[k] = r0 ? T(r0, c1) : 0.0;
            t00[k] = (r0 && c0) ? T(r0, c0) : 0.0;
        }
        float *o = out + l * plane + u;
#pragma unroll
        for (int k = 0; k < kBoxRows; ++k) {
            if (vb + k < nv) {
                const double sum = dadd(dsub(dsub(t11[k], t01[k]), t10[k]), t00[k]);
                const float val = box_quotient_f32(sum, area, inv_area);
                o[(vb + k) * nu] = val;
                m = fmaxf(m, val > 0.0f ? val : 0.0f);
            }
        }
    }
    if (peak) block_peak(peak + l, m);
}

// ---- exact integer first pass ----------------------------------------------
// The first pass smooths H = M * G where G are integer group counts and every
// partial sum is exact (the caller's guard: |H| < 2^24 quanta).  Its float64
// integral table then holds exact multiples of the quantum (< 2^53 of them),
// so the reference's box sum ((T11 - T01) - T10) + T00 is the EXACT window
// sum -- computable in any order, with integers, and no float64 fold chain.
//
// box_int_kernel: one CTA per (TV x TU output tile, layer).  The input region
// (tile + radius halo on every side; zero outside the grid) is staged in
// shared memory (cp.async, or computed there as Hi = sum_b mix[l,b] * G[b]
// for a mixing matrix), then
//   vertical  : a thread per region column slides a (2r+1)-row window down
//               the tile's rows -> W (int32, shared)
//   horizontal: a thread per (row, 32-column chunk) slides a (2r+1)-column
//               window along W (int64) and writes float32(S * scale / area)
//               (the reference's quotient, box_quotient_f32).
// The guard -- any cell with sum_b |mix[l,b]| * G[b] >= limit, or a negative
// count -- sets HB_STATUS_INEXACT; each cell is checked by exactly one tile.
constexpr int kBoxIntTU = 128;   // output columns per CTA
constexpr int kBoxIntThreads = 256;
constexpr int kBoxIntMaxSmem = 220 * 1024;
#ifndef HB_BOX_INT_TILE_MAX_RADIUS
#define HB_BOX_INT_TILE_MAX_RADIUS 8  // larger radii take the separable vwin/hwin pair (config 3: 0.091 -> 0.081 ms; equal on config 4)
#endif
constexpr int kBoxIntTileMaxRadius = HB_BOX_INT_TILE_MAX_RADIUS;

__host__ __device__ __forceinline__ int box_int_pitch(int radius) {
    return (kBoxIntTU + 2 * radius) | 1;  // odd: conflict-free column walks
}
__host__ __device__ __forceinline__ size_t box_int_smem(int tv, int radius) {
    const int pitch = box_int_pitch(radius);
    return sizeof(int32_t) * ((size_t)(tv + 2 * radius) * pitch + (size_t)tv * pitch);
}

template <bool MIX>
__global__ void __launch_bounds__(kBoxIntThreads)
box_int_kernel(const int32_t *__restrict__ counts, const int32_t *__restrict__ mix, int nb,
               int nv, int nu, int radius, int tv, double scale, double limit,
               int32_t *__restrict__ status, float *__restrict__ out, float *__restrict__ peak) {
    extern __shared__ int32_t sm[];
    const int pitch = box_int_pitch(radius);
    const int rows_in = tv + 2 * radius, cols_in = kBoxIntTU + 2 * radius;
    int32_t *in = sm;                              // rows_in x pitch
    int32_t *wv = sm + (size_t)rows_in * pitch;    // tv x pitch
    const int u0 = blockIdx.x * kBoxIntTU, v0 = blockIdx.y * tv, l = blockIdx.z;
    const int ub = u0 - radius, vb = v0 - radius;  // region origin (may be < 0)
    const int64_t plane = (int64_t)nv * nu;
    bool bad = false;
    // 1. stage the region
    const int n_in = rows_in * cols_in;
    for (int k = threadIdx.x; k < n_in; k += kBoxIntThreads) {
        const int rr = k / cols_in, cc = k - rr * cols_in;
        const int v = vb + rr, u = ub + cc;
        const bool inside = (unsigned)v < (unsigned)nv && (unsigned)u < (unsigned)nu;
        const int64_t off = (int64_t)v * nu + u;
        if (!MIX) {
            const unsigned sa = (unsigned)__cvta_generic_to_shared(in + rr * pitch + cc);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa),
                         "l"(inside ? counts + l * plane + off : counts), "r"(inside ? 4 : 0));
        } else {
            long long acc = 0;
            double a = 0.0;
            if (inside)
                for (int b = 0; b < nb; ++b) {
                    const int32_t c = __ldg(counts + b * plane + off);
                    const int32_t m = __ldg(mix + l * nb + b);
                    acc += (long long)m * c;
                    a += fabs((double)m) * (double)c;
                    bad |= c < 0;
                }
            // own cells only: the guard sees each cell once
            if (rr >= radius && rr < radius + tv && cc >= radius && cc < radius + kBoxIntTU)
                bad |= a >= limit;
            in[rr * pitch + cc] = (int32_t)acc;
        }
    }
    if (!MIX) {
        asm volatile("cp.async.commit_group;\n" ::);
        asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();
    // 2. vertical window sums of every region column for the tile's rows
    for (int c = threadIdx.x; c < cols_in; c += kBoxIntThreads) {
        if (!MIX && c >= radius && c < radius + kBoxIntTU)  // the guard on own cells
            for (int t = 0; t < tv; ++t) {
                const int32_t x = in[(t + radius) * pitch + c];
                bad |= x < 0 || (double)x >= limit;
            }
        int32_t w = 0;
        for (int rr = 0; rr <= 2 * radius; ++rr) w += in[rr * pitch + c];
        wv[c] = w;
        for (int t = 1; t < tv; ++t) {
            w += in[(t + 2 * radius) * pitch + c] - in[(t - 1) * pitch + c];
            wv[t * pitch + c] = w;
        }
    }
    __syncthreads();
    // 3. horizontal window sums along W, quotient, store
    const double area = (double)((2 * radius + 1) * (2 * radius + 1));
    const double inv_area = __drcp_rn(area);
    float m = 0.0f;
    const int chunks = kBoxIntTU / 32;
    for (int job = threadIdx.x; job < tv * chunks; job += kBoxIntThreads) {
        // warps walk 32 different rows of the same chunk (odd pitch: no conflicts)
        const int t = (job / (32 * chunks)) * 32 + (job & 31);
        const int ch = (job >> 5) % chunks;
        if (t >= tv) continue;
        const int v = v0 + t;
        const int32_t *row = wv + t * pitch + ch * 32;  // region column of output ch*32 - r
        long long w = 0;
        for (int k = 0; k <= 2 * radius; ++k) w += row[k];
        float vals[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            if (j) w += (long long)row[j + 2 * radius] - row[j - 1];
            const float val = box_quotient_f32(dmul((double)w, scale), area, inv_area);
            vals[j] = val;
            m = fmaxf(m, val > 0.0f ? val : 0.0f);
        }
        const int u = u0 + ch * 32;
        if (v < nv) {
            float *o = out + l * plane + (int64_t)v * nu + u;
            if (u + 32 <= nu && (nu % 4) == 0) {
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                    *reinterpret_cast<float4 *>(o + j) =
                        make_float4(vals[j], vals[j + 1], vals[j + 2], vals[j + 3]);
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (u + j < nu) o[j] = vals[j];
            }
        }
    }
    if (status && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
        atomicOr(status, HB_STATUS_INEXACT);
    if (peak) block_peak(peak + l, m);
}

// Large radii: the tile's halo dominates (r = 50: a 64 x 128 tile stages
// 164 x 228 cells in 209 KB, one CTA per SM), so the same exact sums are
// taken separably through an int32 buffer in global memory (L2):
//   vwin_int : a thread per column slides a (2r+1)-row window down kVwinRows
//              rows (loads unrolled ahead, the outgoing row is an L1 hit)
//   hwin_int : a CTA takes kHwinRows rows of W (8 consecutive columns per
//              thread), scans each row into int64 prefixes in shared memory
//              and takes every window as a difference of two prefixes.
#ifndef HB_VWIN_ROWS
#define HB_VWIN_ROWS 128  // 64: 0.382, 128: 0.379, 256: 0.393 ms per config-5 hb_smooth_counts
#endif
constexpr int kVwinRows = HB_VWIN_ROWS;
constexpr int kVwinThreads = 128;
// Hi of one cell (MIX: sum_b mix[l,b] * G[b]; the guard's |.|-sum in `a`)
template <bool MIX>
__device__ __forceinline__ int32_t hi_cell(const int32_t *__restrict__ g, int64_t plane,
                                           const int32_t *__restrict__ mixrow, int nb,
                                           double &a, bool &neg) {
    if (!MIX) return __ldg(g);
    long long acc = 0;
    for (int b = 0; b < nb; ++b) {
        const int32_t c = __ldg(g + b * plane);
        const int32_t m = __ldg(mixrow + b);
        acc += (long long)m * c;
        a += fabs((double)m) * (double)c;
        neg |= c < 0;
    }
    return (int32_t)acc;
}

template <bool MIX>
__global__ void __launch_bounds__(kVwinThreads)
vwin_int_kernel(const int32_t *__restrict__ counts, const int32_t *__restrict__ mix, int nb,
                int nv, int nu, int radius, double limit, int32_t *__restrict__ status,
                int32_t *__restrict__ wout) {
    const int u = blockIdx.x * kVwinThreads + threadIdx.x;
    const int v0 = blockIdx.y * kVwinRows;
    const int l = blockIdx.z;
    const int64_t plane = (int64_t)nv * nu;
    bool bad = false;
    if (u < nu) {
        const int v1 = min(v0 + kVwinRows, nv);
        // groups of layer 0 at column u (MIX) or this layer's counts
        const int32_t *col = counts + (MIX ? 0 : l * plane) + u;
        const int32_t *mixrow = MIX ? mix + l * nb : nullptr;
        double a = 0.0;
        bool neg = false;
        // the guard, on this thread's own cells (each cell once)
        {
            const int32_t *p = col + (int64_t)v0 * nu;
            for (int v = v0; v < v1; ++v, p += nu) {
                double av = 0.0;
                const int32_t x = hi_cell<MIX>(p, plane, mixrow, nb, av, neg);
                bad |= MIX ? av >= limit : (x < 0 || (double)x >= limit);
            }
            bad |= neg;
        }
        int32_t w = 0;
        const int ra = max(v0 - radius, 0), rb = min(v0 + radius, nv - 1);
        const int32_t *p = col + (int64_t)ra * nu;
#pragma unroll 8
        for (int v = ra; v <= rb; ++v, p += nu) w += hi_cell<MIX>(p, plane, mixrow, nb, a, neg);
        int32_t *dst = wout + l * plane + (int64_t)v0 * nu + u;
        *dst = w;
        // slide: row v + radius enters, row v - radius - 1 leaves
        const int32_t *pin = col + (int64_t)(v0 + 1 + radius) * nu;
        const int32_t *pout = col + (int64_t)(v0 - radius) * nu;
#pragma unroll 8
        for (int v = v0 + 1; v < v1; ++v) {
            dst += nu;
            const int32_t xin = v + radius < nv ? hi_cell<MIX>(pin, plane, mixrow, nb, a, neg) : 0;
            const int32_t xout = v - radius - 1 >= 0 ? hi_cell<MIX>(pout, plane, mixrow, nb, a, neg)
                                                     : 0;
            w += xin - xout;
            *dst = w;
            pin += nu;
            pout += nu;
        }
    }
    if (status && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
        atomicOr(status, HB_STATUS_INEXACT);
}

constexpr int kHwinRows = 4;  // rows of W per CTA (the next row loads during a row's scan)
constexpr int kHwinCols = 8;  // consecutive columns per thread (nu <= 8 * 1024)
__host__ __device__ __forceinline__ int hwin_threads(int nu) {
    return ((nu + kHwinCols - 1) / kHwinCols + 31) / 32 * 32;
}
// prefix j lives at hwin_pad(j): a thread's 8 consecutive prefixes are 9
// words from the next thread's (conflict-free instead of 16-way)
__host__ __device__ __forceinline__ int hwin_pad(int j) { return j + (j >> 3); }
__host__ __device__ __forceinline__ size_t hwin_smem(int nu) {
    return sizeof(long long) * ((size_t)hwin_pad(nu) + 1 + 32);
}

// Each row of W is scanned across the CTA into exact int64 prefixes P
// (P[j] = sum of W[0..j), shared memory), and the horizontal window sum is
// P[min(u+r+1, nu)] - P[max(u-r, 0)] -- the same exact integer as a
// sliding window, at two shared loads per cell (the sliding window walked
// 2r+1 + 64 shared words per 32 cells and was issue-bound).
__global__ void __launch_bounds__(1024)
hwin_int_kernel(const int32_t *__restrict__ win, int nv, int nu, int radius, double scale,
                float *__restrict__ out, float *__restrict__ peak) {
    extern __shared__ long long hp[];  // P[0 .. nu] (padded), then 32 warp totals
    long long *wt = hp + hwin_pad(nu) + 1;
    const int vb = blockIdx.x * kHwinRows, l = blockIdx.y;
    const int64_t plane = (int64_t)nv * nu;
    const int nr = min(kHwinRows, nv - vb);
    const int c0 = threadIdx.x * kHwinCols;
    const bool vec = (nu % 4) == 0 && c0 + kHwinCols <= nu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int32_t *src = win + l * plane + (int64_t)vb * nu + c0;
    auto load_row = [&](int t, int32_t (&x)[kHwinCols]) {
        if (t < nr && vec) {
            const int4 a = __ldg(reinterpret_cast<const int4 *>(src + (int64_t)t * nu));
            const int4 b = __ldg(reinterpret_cast<const int4 *>(src + (int64_t)t * nu + 4));
            x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
            x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
        } else {
#pragma unroll
            for (int j = 0; j < kHwinCols; ++j)
                x[j] = (t < nr && c0 + j < nu) ? __ldg(src + (int64_t)t * nu + j) : 0;
        }
    };
    int32_t xc[kHwinCols], xn[kHwinCols];
    load_row(0, xc);
    const double area = (double)((2 * radius + 1) * (2 * radius + 1));
    const double inv_area = __drcp_rn(area);
    float m = 0.0f;
    for (int t = 0; t < nr; ++t) {
        load_row(t + 1, xn);  // the next row's loads overlap this row's scan
        long long inc[kHwinCols], run = 0;
#pragma unroll
        for (int j = 0; j < kHwinCols; ++j) {
            run += xc[j];
            inc[j] = run;
        }
        long long sc = run;  // inclusive warp scan of the thread totals
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, sc, d);
            if (lane >= d) sc += y;
        }
        if (lane == 31) wt[warp] = sc;
        __syncthreads();
        long long woff = lane < warp ? wt[lane] : 0;  // totals of the warps before this one
#pragma unroll
        for (int d = 16; d; d >>= 1) woff += __shfl_xor_sync(0xffffffffu, woff, d);
        const long long off = woff + sc - run;
        if (threadIdx.x == 0) hp[0] = 0;
#pragma unroll
        for (int j = 0; j < kHwinCols; ++j)
            if (c0 + j < nu) hp[hwin_pad(c0 + j + 1)] = off + inc[j];
        __syncthreads();  // (P and wt are rewritten only after the next row's first barrier)
        float vals[kHwinCols];
#pragma unroll
        for (int j = 0; j < kHwinCols; ++j) {
            const int u = c0 + j;
            const long long S =
                hp[hwin_pad(min(u + radius + 1, nu))] - hp[hwin_pad(min(max(u - radius, 0), nu))];
            vals[j] = box_quotient_f32(dmul((double)S, scale), area, inv_area);
            if (u < nu) m = fmaxf(m, vals[j] > 0.0f ? vals[j] : 0.0f);
        }
        float *o = out + l * plane + (int64_t)(vb + t) * nu + c0;
        if (vec) {
            *reinterpret_cast<float4 *>(o) = make_float4(vals[0], vals[1], vals[2], vals[3]);
            *reinterpret_cast<float4 *>(o + 4) = make_float4(vals[4], vals[5], vals[6], vals[7]);
        } else {
#pragma unroll
            for (int j = 0; j < kHwinCols; ++j)
                if (c0 + j < nu) o[j] = vals[j];
        }
#pragma unroll
        for (int j = 0; j < kHwinCols; ++j) xc[j] = xn[j];
    }
    if (peak) block_peak(peak + l, m);
}

// radius-0 pass (raster.py:157-158 returns a copy) and stand-alone layer
// mixing (the raw histogram H of raster.accumulate_edges).
template <typename T>
__global__ void mix_pass_kernel(const T *__restrict__ groups, const float *__restrict__ mat,
                                int nb, int64_t plane, float *__restrict__ out,
                                float *__restrict__ peak) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int l = blockIdx.y;
    float val = 0.0f;
    if (i < plane) {
        val = mixed_value<T>(groups, mat, nb, l, plane, i);
        out[l * plane + i] = val;
    }
    if (peak) block_peak(peak + l, val > 0.0f ? val : 0.0f);
}

// Quad advection field.  For every cell (u, v) of a layer, a 48-byte record
// of three float4 (interleaved, so a gradient sample reads 2 sectors, not 3):
//   Q  = rho at the 2x2 corners (u,v) (u+1,v) (u,v+1) (u+1,v+1)
//   GX = dX at the same corners,  GY = dY at the same corners,
// where dX/dY are _cell_gradient's float32 central differences
// (_kernels.py:101-114) at the clamped corner cell.  A bilinear sample
// (_kernels.py:80-98) is then one 16-byte load and the gradient+value of a
// point three.  Corners past the last row/column are never read (bilinear
// and gradient_xy clamp u0 <= nu-2, v0 <= nv-2) and are stored as 0.
__device__ __forceinline__ void cell_diff(const float *__restrict__ r, int nv, int nu, int u, int v,
                                          float &dx, float &dy) {
    const int uc = min(max(u, 1), nu - 2), vc = min(max(v, 1), nv - 2);
    const float *c = r + (int64_t)vc * nu + uc;
    dx = __fsub_rn(c[1], c[-1]);
    dy = __fsub_rn(c[nu], c[-nu]);
}

__global__ void grad_field_kernel(const float *__restrict__ rho, int nv, int nu,
                                  float4 *__restrict__ out) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    const int v = blockIdx.y;
    const int l = blockIdx.z;
    if (u >= nu) return;
    const int64_t plane = (int64_t)nv * nu;
    const float *r = rho + l * plane;
    const int64_t cell = l * plane + (int64_t)v * nu + u;
    // {Q, GX, GY} of the cell: interleaved, or {Q, GX} + GY in two regions
    float4 *rec = out + (HB_QUAD_SPLIT ? 2 : (int)kQuadRec) * cell;
    float4 *gyp = HB_QUAD_SPLIT ? out + 2 * (int64_t)gridDim.z * plane + cell : rec + 2;
    if (u > nu - 2 || v > nv - 2) {
        rec[0] = rec[1] = *gyp = make_float4(0.f, 0.f, 0.f, 0.f);
        return;
    }
    const float *c = r + (int64_t)v * nu + u;
    rec[0] = make_float4(c[0], c[1], c[nu], c[nu + 1]);
    float x00, y00, x10, y10, x01, y01, x11, y11;
    cell_diff(r, nv, nu, u, v, x00, y00);
    cell_diff(r, nv, nu, u + 1, v, x10, y10);
    cell_diff(r, nv, nu, u, v + 1, x01, y01);
    cell_diff(r, nv, nu, u + 1, v + 1, x11, y11);
    rec[1] = make_float4(x00, x10, x01, x11);
    *gyp = make_float4(y00, y10, y01, y11);
}

// used_cell_count (bundler.py:292-305): rho > float32(rel * peak_l) when
// peak_l > 0 (NEP 50 makes the comparison float32).
// kUsedPer cells per thread (strided by the block), one atomic per block.
constexpr int kUsedPer = 8;
__global__ void __launch_bounds__(256)
used_cells_kernel(const float *__restrict__ rho, const float *__restrict__ peak,
                  int64_t plane, double rel, unsigned long long *count) {
    __shared__ unsigned s_cnt[8];
    const int64_t i0 = (int64_t)blockIdx.x * (256 * kUsedPer) + threadIdx.x;
    const int l = blockIdx.y;
    const float pk = peak[l];
    unsigned c = 0;
    if ((double)pk > 0.0) {
        const float thr = __double2float_rn(dmul(rel, (double)pk));
        const float *r = rho + l * plane;
#pragma unroll
        for (int k = 0; k < kUsedPer; ++k) {
            const int64_t i = i0 + 256 * k;
            if (i < plane && r[i] > thr) ++c;
        }
    }
    for (int d = 16; d; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
    if ((threadIdx.x & 31) == 0) s_cnt[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) c += s_cnt[w];
        if (c) atomicAdd(count, (unsigned long long)c);
    }
}

}  // namespace hb

using namespace hb;

static void launch_row_fold(double *table, int64_t rows, int nu, cudaStream_t st) {
#ifndef HB_ROW_SCALAR
    if (nu % 2 == 0) {  // 16-byte aligned rows
        row_scan2_kernel<<<(unsigned)((rows + 31) / 32), 32, 0, st>>>(table, rows, nu);
        return;
    }
#endif
    row_scan_kernel<<<(unsigned)((rows + 31) / 32), 32, 0, st>>>(table, rows, nu);
}

static unsigned col_fold_blocks(int nbins, int nu) {
    const int64_t groups = (int64_t)nbins * ((nu + kColW - 1) / kColW);
    return (unsigned)((groups + kColWarps - 1) / kColWarps);
}

static inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Fused fold (fold_kernel<S>): strip width and whether it fits.  Every CTA
// must be co-resident (strips wait on one another): S = 64 when nbins *
// nstrips CTAs fit at one per SM, else S = 128; 0 = use the two fold kernels.
// HB_FOLD=0 in the environment selects the two fold kernels (A/B checks).
template <int S>
static int fold_blocks_per_sm() {
    static int per_sm = -1;  // a property of the kernel: computed once
    if (per_sm < 0) {
        const void *fn = (const void *)fold_kernel<S>;
        int n = 0;
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)FoldCfg<S>::kSmem) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, kFoldThreads,
                                                          FoldCfg<S>::kSmem) != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
        per_sm = n;
    }
    return per_sm;
}

static int fold_strip_width(int nbins, int nu) {
    const char *e = getenv("HB_FOLD");  // read per call: tests flip it in-process
    if (e && e[0] == '0') return 0;
    const int64_t sms = device_sm_count();
    if ((int64_t)nbins * ((nu + 63) / 64) <= fold_blocks_per_sm<64>() * sms) return 64;
    if ((int64_t)nbins * ((nu + 127) / 128) <= fold_blocks_per_sm<128>() * sms) return 128;
    return 0;
}

// carry hand-off words of fold_kernel: [nbins][nstrips][nv] (nstrips <= nu/64 + 1)
static size_t fold_carry_words(int nbins, int nv, int nu) {
    return (size_t)nbins * (size_t)(nu / 64 + 1) * (size_t)nv;
}

template <int S>
static cudaError_t launch_fold(const float *fin, int nbins, int nv, int nu, double *table,
                               unsigned long long *carry, cudaStream_t st) {
    int nstrips = (nu + S - 1) / S;
    void *args[] = {(void *)&fin, (void *)&nv, (void *)&nu, (void *)&nstrips, (void *)&table,
                    (void *)&carry};
    return cudaLaunchCooperativeKernel((const void *)fold_kernel<S>, dim3(nbins * nstrips),
                                       dim3(kFoldThreads), args, FoldCfg<S>::kSmem, st);
}

// One float box pass (raster.py:147-169) of every layer: column fold, row
// fold (float64 table), 4-term box / area -> dst (+ layer peaks).  carry:
// fold_kernel's hand-off words, all kFoldSentinel on entry and on exit.
// Returns the number of kernels launched.
static int float_box_pass(const float *fin, int nbins, int nv, int nu, int r, float *dst,
                          double *table, float *pk, unsigned long long *carry,
                          cudaStream_t st) {
    const int S = carry ? fold_strip_width(nbins, nu) : 0;
    int launched = 3;
    cudaError_t fe = cudaErrorNotReady;  // not launched
    if (S == 64) fe = launch_fold<64>(fin, nbins, nv, nu, table, carry, st);
    else if (S == 128) fe = launch_fold<128>(fin, nbins, nv, nu, table, carry, st);
    if (fe == cudaSuccess) {
        launched = 2;
    } else {
        // (a cooperative launch the device refuses -- e.g. too large beside
        // other work -- falls back to the two fold kernels; nothing ran)
        if (fe != cudaErrorNotReady) cudaGetLastError();
        col_fold_kernel<<<col_fold_blocks(nbins, nu), kColWarps * 32, 0, st>>>(fin, nbins, nv,
                                                                               nu, table);
        launch_row_fold(table, (int64_t)nbins * nv, nu, st);
    }
    dim3 gb((nu + kBoxBlock - 1) / kBoxBlock, (nv + kBoxRows - 1) / kBoxRows, nbins);
    box_kernel<<<gb, kBoxBlock, 0, st>>>(table, nv, nu, r, dst, pk);
    return launched;
}

// fold_kernel's carry words at the end of the smoothing workspace, armed
// (all kFoldSentinel) for this call; NULL when the fused fold is not used.
static unsigned long long *fold_carry(void *workspace, int nbins, int nv, int nu,
                                      cudaStream_t st) {
    if (!fold_strip_width(nbins, nu)) return nullptr;
    const size_t cells = (size_t)nbins * nv * nu;
    const size_t off = (cells * (sizeof(double) + sizeof(float)) + 255) & ~(size_t)255;
    auto *carry = reinterpret_cast<unsigned long long *>(static_cast<char *>(workspace) + off);
    if (cudaMemsetAsync(carry, 0xff, sizeof(unsigned long long) * fold_carry_words(nbins, nv, nu),
                        st) != cudaSuccess)
        return nullptr;
    return carry;
}

extern "C" {

size_t hb_smooth_workspace_bytes(int nbins, int nv, int nu) {
    const size_t cells = (size_t)nbins * nv * nu;
    return cells * sizeof(double) + cells * sizeof(float) + 256 +
           sizeof(unsigned long long) * fold_carry_words(nbins, nv, nu);
}

int hb_smooth(const int32_t *counts, const float *hist, const float *matrix, int nbins,
              int nv, int nu, const int32_t *radii, int npasses, float *out,
              void *workspace, size_t workspace_bytes, float *layer_peak, void *stream) {
    if (nbins < 1 || nv < 1 || nu < 1 || nv > kMaxDim || nu > kMaxDim || npasses < 1 || !radii || !out || (!counts && !hist))
        return set_error(HB_EINVAL, "hb_smooth: bad arguments");
    if (!workspace || workspace_bytes < hb_smooth_workspace_bytes(nbins, nv, nu))
        return set_error(HB_EINVAL, "hb_smooth: workspace too small");
    for (int p = 0; p < npasses; ++p)
        if (radii[p] < 0) return set_error(HB_EINVAL, "radius must be >= 0");
    cudaStream_t st = as_stream(stream);
    const int64_t plane = (int64_t)nv * nu;
    const size_t cells = (size_t)nbins * plane;
    double *table = reinterpret_cast<double *>(workspace);
    float *stage = reinterpret_cast<float *>(table + cells);
    unsigned long long *carry = fold_carry(workspace, nbins, nv, nu, st);
    if (layer_peak && cudaMemsetAsync(layer_peak, 0, sizeof(float) * nbins, st) != cudaSuccess)
        return check_launch("hb_smooth(memset)", 0);
    const float *src = nullptr;  // float32 input of passes after the first
    for (int p = 0; p < npasses; ++p) {
        const bool first = (p == 0);
        const bool mix_first = first && (counts || matrix);
        // passes alternate between stage and out so the last one lands in out
        float *dst = ((npasses - 1 - p) % 2 == 0) ? out : stage;
        float *pk = (p == npasses - 1) ? layer_peak : nullptr;
        const int r = radii[p];
        int launched = 1;
        if (r == 0) {
            dim3 g((unsigned)((plane + 255) / 256), nbins);
            if (first && counts)
                mix_pass_kernel<int32_t><<<g, 256, 0, st>>>(counts, matrix, nbins, plane, dst, pk);
            else
                mix_pass_kernel<float><<<g, 256, 0, st>>>(first ? hist : src,
                                                          first ? matrix : nullptr, nbins,
                                                          plane, dst, pk);
        } else {
            const float *fin = first ? hist : src;
            if (mix_first) {
                // H = float32(M * G) as its own elementwise pass into the stage
                // buffer (a fused mix in the sequential column fold was measured
                // 10x slower); the fold below consumes it before any pass
                // output can overwrite the stage buffer
                dim3 g((unsigned)((plane + 255) / 256), nbins);
                if (counts)
                    mix_pass_kernel<int32_t><<<g, 256, 0, st>>>(counts, matrix, nbins, plane,
                                                                stage, nullptr);
                else
                    mix_pass_kernel<float><<<g, 256, 0, st>>>(hist, matrix, nbins, plane, stage,
                                                              nullptr);
                fin = stage;
            } else {
                launched = 0;
            }
            launched += float_box_pass(fin, nbins, nv, nu, r, dst, table, pk, carry, st);
        }
        int rc = check_launch("hb_smooth", launched);
        if (rc) return rc;
        src = dst;
    }
    return HB_OK;
}

int hb_smooth_counts(const int32_t *counts, const int32_t *mix, double scale, double limit,
                     int nbins, int nv, int nu, const int32_t *radii, int npasses, float *out,
                     void *workspace, size_t workspace_bytes, float *layer_peak, int32_t *status,
                     void *stream) {
    if (!counts || nbins < 1 || nv < 1 || nu < 1 || nv > kMaxDim || nu > kMaxDim ||
        npasses < 1 || !radii || !out || !(scale > 0.0))
        return set_error(HB_EINVAL, "hb_smooth_counts: bad arguments");
    int sexp = 0;
    if (frexp(scale, &sexp) != 0.5) return set_error(HB_EINVAL, "hb_smooth_counts: scale must be 2^k");
    if (!workspace || workspace_bytes < hb_smooth_workspace_bytes(nbins, nv, nu))
        return set_error(HB_EINVAL, "hb_smooth_counts: workspace too small");
    for (int p = 0; p < npasses; ++p)
        if (radii[p] < 0) return set_error(HB_EINVAL, "radius must be >= 0");
    if (radii[0] == 0) return set_error(HB_EINVAL, "hb_smooth_counts: first radius must be > 0");
    cudaStream_t st = as_stream(stream);
    const int64_t plane = (int64_t)nv * nu;
    const size_t cells = (size_t)nbins * plane;
    double *table = reinterpret_cast<double *>(workspace);
    float *stage = reinterpret_cast<float *>(table + cells);
    unsigned long long *carry = fold_carry(workspace, nbins, nv, nu, st);
    if (layer_peak && cudaMemsetAsync(layer_peak, 0, sizeof(float) * nbins, st) != cudaSuccess)
        return check_launch("hb_smooth_counts(memset)", 0);
    // pass 0: exact integer window sums in shared-memory tiles
    {
        float *dst = ((npasses - 1) % 2 == 0) ? out : stage;
        float *pk = npasses == 1 ? layer_peak : nullptr;
        const int r = radii[0];
        int tv = 64;
        while (tv > 8 && box_int_smem(tv, r) > (size_t)kBoxIntMaxSmem) tv >>= 1;
        const size_t smem = box_int_smem(tv, r);
        const bool sums_fit = (double)(2 * r + 1) * limit < 2147483647.0;
        const size_t hsm = hwin_smem(nu);
        if (sums_fit && r > kBoxIntTileMaxRadius && hsm <= (size_t)kBoxIntMaxSmem &&
            hwin_threads(nu) <= 1024) {
            if (cudaFuncSetAttribute(hwin_int_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kBoxIntMaxSmem) != cudaSuccess)
                return check_launch("hb_smooth_counts(smem)", 0);
            int32_t *w = reinterpret_cast<int32_t *>(table);
            dim3 gv((nu + kVwinThreads - 1) / kVwinThreads, (nv + kVwinRows - 1) / kVwinRows,
                    nbins);
            if (mix)
                vwin_int_kernel<true><<<gv, kVwinThreads, 0, st>>>(counts, mix, nbins, nv, nu, r,
                                                                  limit, status, w);
            else
                vwin_int_kernel<false><<<gv, kVwinThreads, 0, st>>>(counts, mix, nbins, nv, nu, r,
                                                                   limit, status, w);
            hwin_int_kernel<<<dim3((nv + kHwinRows - 1) / kHwinRows, nbins), hwin_threads(nu),
                              hsm, st>>>(w, nv, nu, r, scale, dst, pk);
            int rc = check_launch("hb_smooth_counts", 2);
            if (rc) return rc;
        } else if (sums_fit && smem <= (size_t)kBoxIntMaxSmem) {
            if (cudaFuncSetAttribute(box_int_kernel<false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kBoxIntMaxSmem) != cudaSuccess ||
                cudaFuncSetAttribute(box_int_kernel<true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kBoxIntMaxSmem) != cudaSuccess)
                return check_launch("hb_smooth_counts(smem)", 0);
            dim3 g((nu + kBoxIntTU - 1) / kBoxIntTU, (nv + tv - 1) / tv, nbins);
            if (mix)
                box_int_kernel<true><<<g, kBoxIntThreads, smem, st>>>(
                    counts, mix, nbins, nv, nu, r, tv, scale, limit, status, dst, pk);
            else
                box_int_kernel<false><<<g, kBoxIntThreads, smem, st>>>(
                    counts, mix, nbins, nv, nu, r, tv, scale, limit, status, dst, pk);
            int rc = check_launch("hb_smooth_counts", 1);
            if (rc) return rc;
        } else {
            return set_error(HB_EINVAL, "hb_smooth_counts: radius too large for the integer pass");
        }
    }
    const float *src = ((npasses - 1) % 2 == 0) ? out : stage;
    for (int p = 1; p < npasses; ++p) {
        float *dst = ((npasses - 1 - p) % 2 == 0) ? out : stage;
        float *pk = (p == npasses - 1) ? layer_peak : nullptr;
        const int r = radii[p];
        int launched = 1;
        if (r == 0) {
            dim3 g((unsigned)((plane + 255) / 256), nbins);
            mix_pass_kernel<float><<<g, 256, 0, st>>>(src, nullptr, nbins, plane, dst, pk);
        } else {
            launched = float_box_pass(src, nbins, nv, nu, r, dst, table, pk, carry, st);
        }
        int rc = check_launch("hb_smooth_counts", launched);
        if (rc) return rc;
        src = dst;
    }
    return HB_OK;
}

#ifdef HB_FOLD_TRACE
HB_API int hb_debug_fold_trace(unsigned long long *out) {
    return cudaMemcpyFromSymbol(out, g_fold_trace, sizeof(g_fold_trace)) == cudaSuccess ? 0 : -1;
}
#endif

int hb_mix_layers(const int32_t *counts, const float *hist, const float *matrix, int nbins,
                  int nv, int nu, float *out, void *stream) {
    if (nbins < 1 || nv < 1 || nu < 1 || nv > kMaxDim || nu > kMaxDim || !out || (!counts && !hist))
        return set_error(HB_EINVAL, "hb_mix_layers: bad arguments");
    const int64_t plane = (int64_t)nv * nu;
    dim3 g((unsigned)((plane + 255) / 256), nbins);
    if (counts)
        mix_pass_kernel<int32_t><<<g, 256, 0, as_stream(stream)>>>(counts, matrix, nbins, plane,
                                                                   out, nullptr);
    else
        mix_pass_kernel<float><<<g, 256, 0, as_stream(stream)>>>(hist, matrix, nbins, plane,
                                                                 out, nullptr);
    return check_launch("hb_mix_layers");
}

int hb_integral_image(const float *in, int nbins, int nv, int nu, double *table,
                      void *stream) {
    if (!in || !table || nbins < 1 || nv < 1 || nu < 1 || nv > kMaxDim || nu > kMaxDim)
        return set_error(HB_EINVAL, "hb_integral_image: bad arguments");
    cudaStream_t st = as_stream(stream);
    col_fold_kernel<<<col_fold_blocks(nbins, nu), kColWarps * 32, 0, st>>>(in, nbins, nv, nu,
                                                                           table);
    const int64_t rows = (int64_t)nbins * nv;
    launch_row_fold(table, rows, nu, st);
    return check_launch("hb_integral_image", 2);
}

int64_t hb_grad_field_bytes(int nbins, int nv, int nu) {
    if (nbins < 1 || nv < 1 || nu < 1) {
        set_error(HB_EINVAL, "hb_grad_field_bytes: bad arguments");
        return -1;
    }
    return (int64_t)sizeof(float4) * kQuadRec * nbins * nv * nu;
}

int hb_grad_field(const float *rho, int nbins, int nv, int nu, float *out, void *stream) {
    if (!rho || !out || nbins < 1 || nv < 3 || nu < 3 || nv > kMaxDim || nu > kMaxDim)
        return set_error(HB_EINVAL, "hb_grad_field: bad arguments");
    dim3 g((nu + 255) / 256, nv, nbins);
    grad_field_kernel<<<g, 256, 0, as_stream(stream)>>>(rho, nv, nu, reinterpret_cast<float4 *>(out));
    return check_launch("hb_grad_field");
}

int hb_used_cells(const float *rho, const float *layer_peak, int nbins, int nv, int nu,
                  double rel, unsigned long long *count, void *stream) {
    if (!rho || !layer_peak || !count || nbins < 1 || nv < 1 || nu < 1 || nv > kMaxDim || nu > kMaxDim)
        return set_error(HB_EINVAL, "hb_used_cells: bad arguments");
    const int64_t plane = (int64_t)nv * nu;
    dim3 g((unsigned)((plane + 256 * kUsedPer - 1) / (256 * kUsedPer)), nbins);
    used_cells_kernel<<<g, 256, 0, as_stream(stream)>>>(rho, layer_peak, plane, rel, count);
    return check_launch("hb_used_cells");
}

}  // extern "C"
