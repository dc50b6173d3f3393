// bin_fast.cu -- k_bin_fast: the accumulate kernel (a4 + a5) for the common
// case of at most one binned attribute with 16-byte-aligned columns (C1, C3,
// C4, C5 and the paper's Fig. 1 sum-of-mass), same window layout and
// arithmetic as k_bin (bin_general.cu), written for few instructions per row:
//
//  * 32-bit pair indices, shared memory addressed as one u32 array through
//    32-bit shared-window addresses from one base register;
//  * one 16-byte pair per column prefetched one step ahead in registers;
//  * every row's work issued by its own lane: shared-memory count, 96-bit
//    fixed-point sum and min/max filter for rows in the CTA's window, and
//    predicated fire-and-forget L2 reductions for the rare work (rows outside
//    the window, min/max candidates, values outside the fixed-point range).
//    Round 1 batched that rare work through a per-warp queue drained 32 items
//    at a time; the pushes cost ~40 issue slots per row pair and the queue
//    ~24 KB of window, and the direct form measured 0.575 vs 0.591 ms on C3
//    (profiles/r02_kbin_ablation.txt).
#include <cuda_runtime.h>
#include <stdint.h>

#include "db_internal.h"
#include "dev_common.cuh"
#include "xsum.cuh"

#ifndef BIN_FAST_LD
#define BIN_FAST_LD __ldcg
#endif

namespace db {

extern __shared__ __align__(16) uint32_t f_dsm[];

#ifndef BIN_FAST_THREADS
#define BIN_FAST_THREADS 1024
#endif
constexpr int FAST_THREADS = BIN_FAST_THREADS;
// Shared memory past the window: BIN_SUM_EXACT keeps a per-warp queue of the
// sums that go to the digit rows (rows outside the window, values off the
// fixed-point grid): each is ~40 instructions of digit splitting plus three
// reductions, so they are batched and executed 32 at a time with every lane
// busy (one at a time from their own lanes, exact mode ran at 124 vs 143 G
// rows/s on C3).  Fast sums need none.
constexpr int XQ = 64;                 // >= 31 leftover + 32 new items
constexpr int XQ_WORDS = 3 * XQ;       // u32 bins[XQ] + f64 values[XQ]
int fast_queue_bytes(bool exact) { return exact ? (FAST_THREADS / 32) * XQ_WORDS * 4 + 16 : 16; }

// Window bytes per bin: count u32, fixed-point sum 3 x u32, min/max filter
// 2 x u32.  (Exact u64 min/max in the window instead of the filter -- 32 B per
// bin, an LDS.128 per row -- measured 0.637 vs 0.591 ms on C3: the smaller
// window sent more rows to L2.)
int fast_window_bytes_per_bin(const Accum &acc) { return 4 + 12 * acc.nsum + 8 * acc.nmm; }

__device__ __forceinline__ void s_red_add(uint32_t a, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ uint32_t s_atom_add(uint32_t a, uint32_t v) {
    uint32_t r;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(r) : "r"(a), "r"(v));
    return r;
}
__device__ __forceinline__ void s_red_min(uint32_t a, uint32_t v) {
    asm volatile("red.shared.min.u32 [%0], %1;" ::"r"(a), "r"(v));
}

// Hot-loop context: only the D used dimensions (so it stays in registers).
template <int D>
struct FastCtx {
    double lo[D], hi[D], scale[D];
    int resm1[D];
    int wo[D];
    unsigned we[D];
    uint32_t W;
    FxParam fx;
    uint32_t o_fx, o_cnt;  // word offsets (filters at 0)
    uint32_t sb;           // shared-window address of f_dsm[0]
    unsigned long long *mm;  // global {enc(min), ~enc(max)} slots
};

struct FastX {
    long long *xs;  // nullptr: BIN_SUM_FAST
    uint64_t B;
    int *sxr;       // this CTA's touched digit range (shared memory)
    uint32_t qb;    // BIN_SUM_EXACT: this warp's queue (word offset in the dynamic shared memory)
};

// BIN_SUM_EXACT: lanes with p append (bin, v) to the warp's queue; at 32 items
// the warp adds them to the digit rows with every lane busy.  Warp-uniform.
__device__ __forceinline__ void xs_push(bool p, uint32_t b, double v, const FastX &X, uint32_t &qn) {
    const unsigned m = __ballot_sync(0xffffffffu, p);
    if (m == 0) return;
    const unsigned lane = threadIdx.x & 31u;
    uint32_t *tags = f_dsm + X.qb;
    double *vals = (double *)(f_dsm + X.qb + XQ);
    if (p) {
        const unsigned pos = qn + __popc(m & ((1u << lane) - 1u));
        tags[pos] = b;
        vals[pos] = v;
    }
    qn += __popc(m);
    if (qn >= 32) {
        __syncwarp();
        const uint32_t tb = tags[lane];
        const double tv = vals[lane];
        const unsigned rest = qn - 32;
        uint32_t t2 = 0;
        double v2 = 0.0;
        if (lane < rest) t2 = tags[32 + lane], v2 = vals[32 + lane];
        __syncwarp();
        if (lane < rest) tags[lane] = t2, vals[lane] = v2;
        qn = rest;
        xsum_add_double(X.xs, X.B, 0, tb, tv, X.sxr);
        __syncwarp();
    }
}

// ---- predicated fire-and-forget reductions (no branch region per row) ----
__device__ __forceinline__ void ps_add(bool p, uint32_t a, uint32_t v) {
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %0, 0; @q red.shared.add.u32 [%1], %2; }" ::"r"((int)p), "r"(a), "r"(v)
                 : "memory");
}
__device__ __forceinline__ void ps_min(bool p, uint32_t a, uint32_t v) {
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %0, 0; @q red.shared.min.u32 [%1], %2; }" ::"r"((int)p), "r"(a), "r"(v)
                 : "memory");
}
__device__ __forceinline__ void pg_add_u64(bool p, unsigned long long *a, unsigned long long v) {
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %0, 0; @q red.relaxed.gpu.global.add.u64 [%1], %2; }" ::"r"((int)p),
                 "l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ void pg_add_f64(bool p, double *a, double v) {
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %0, 0; @q red.relaxed.gpu.global.add.f64 [%1], %2; }" ::"r"((int)p),
                 "l"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void pg_min_u64(bool p, unsigned long long *a, unsigned long long v) {
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %0, 0; @q red.relaxed.gpu.global.min.u64 [%1], %2; }" ::"r"((int)p),
                 "l"(a), "l"(v) : "memory");
}

// One row, all of its work issued by its own lane: in
// the window -> shared-memory count, 96-bit fixed-point sum and the min/max
// filter (an improving row also sends its exact value to the global slot);
// outside it -> L2 reductions of count, sum, min and max.  A value outside the
// fixed-point range sends its sum to L2 (its count and min/max stay in the
// window).  sm_100a ptxas wraps every predicated atomic in its own BSSY/BRA/
// BSYNC region; grouping the rare ones into fewer regions (with min-with-~0
// no-ops for the half not needed) was measured slower: 0.651 vs 0.583 ms on
// C3 -- the no-op reductions cost more than the regions.
template <int D, int A, int SM, int MM, bool XS>
__device__ __forceinline__ void lean_row(const FastCtx<D> &c, const double (&x)[D], double v, bool valid,
                                         uint32_t &n_in, unsigned long long *count, double *sum, const FastX &X,
                                         uint32_t &qn) {
    constexpr bool HS = A == 1 && SM == 1, HM = A == 1 && MM == 1;
    bool ok = valid;
    int k[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
        ok = ok && (c.lo[d] <= x[d]) && (x[d] <= c.hi[d]);
        k[d] = min(floor_nonneg(__dmul_rn(__dsub_rn(x[d], c.lo[d]), c.scale[d])), c.resm1[d]);
    }
    n_in += ok ? 1u : 0u;
    bool inw = ok;
    uint32_t l = 0;
#pragma unroll
    for (int d = D - 1; d >= 0; --d) {
        const unsigned r = (unsigned)(k[d] - c.wo[d]);
        inw = inw && (r < c.we[d]);
        l = l * c.we[d] + r;
    }
    uint32_t b = (uint32_t)k[0];
    if (D >= 2) b += (uint32_t)(c.resm1[0] + 1) * (uint32_t)k[1];
    if (D >= 3) b += (uint32_t)(c.resm1[0] + 1) * (uint32_t)(c.resm1[D > 2 ? 1 : 0] + 1) * (uint32_t)k[D > 2 ? 2 : 0];
    const bool glob = ok && !inw;
    const uint32_t W = c.W;
    DB_CHECK(!inw || l < W);
#pragma unroll
    for (int d = 0; d < D; ++d) DB_CHECK(!ok || (k[d] >= 0 && k[d] <= c.resm1[d]));
    ps_add(inw, c.sb + 4u * (c.o_cnt + l), 1u);
    bool sum_glob = glob;
    if (HS) {
        const uint32_t a0 = c.sb + 4u * (c.o_fx + l);
        unsigned long long q = 0;
        bool fx;
        if (XS) {
            fx = fx_quant_exact(c.fx, v, q);
        } else {
            fx = fx_path(c.fx, v);
            q = fx ? fx_quant(c.fx, v) : 0ull;
        }
        fx = fx && inw;
        sum_glob = glob || (inw && !fx);
        if (inw) {  // (almost every lane: a short region)
            if (!fx) q = (unsigned long long)FX_OFFSET;  // count-only offset: the sum goes to L2
            const unsigned qlo = (unsigned)q;
            unsigned qmid = (unsigned)(q >> 32);
            const unsigned old = s_atom_add(a0, qlo);
            qmid += (old + qlo < old) ? 1u : 0u;
            const unsigned old2 = s_atom_add(a0 + 4u * W, qmid);
            ps_add(old2 + qmid < old2, a0 + 8u * W, 1u);  // rare carry into the high word
        }
    }
    if (HM) {
        const unsigned long long e = enc_total(v);
        const unsigned eh = (unsigned)(e >> 32), neh = ~eh;
        uint2 f = make_uint2(0u, 0u);  // (a row outside the window: the filter does not apply)
        const uint32_t fa = c.sb + 8u * l;
        if (inw) asm volatile("ld.volatile.shared.v2.u32 {%0, %1}, [%2];" : "=r"(f.x), "=r"(f.y) : "r"(fa));
        ps_min(inw && eh < f.x, fa, eh);
        ps_min(inw && neh < f.y, fa + 4u, neh);
        unsigned long long *g = c.mm + 2ull * b;
        pg_min_u64(glob || (inw && eh <= f.x), g, e);
        pg_min_u64(glob || (inw && neh <= f.y), g + 1, ~e);
    }
    pg_add_u64(glob, count + b, 1ull);
    if (HS) {
        if (XS) xs_push(sum_glob, b, v, X, qn);
        else pg_add_f64(sum_glob, sum + b, v);
    }
}

constexpr int SAMPLE_PAIRS = 2;  // per thread, spread over the thread's range (the first is reused)

// The CTA's window: coarse histogram of 4 sample pairs per thread (spread over
// the thread's range) in the still-unused dynamic shared memory, then the best
// box (dev_common.cuh pick_box); also the largest exponent of the attribute.
// Everything indexed statically (D is a template parameter) so no scratch goes
// to local memory and the hot loop keeps the geometry in registers.
template <int D, int A>
__device__ __forceinline__ void fast_choose_window(const DGeom G, const WinPlan P, const double2 *cx0,
                                                   const double2 *cx1, const double2 *cx2,
                                                   const double2 *cv, uint32_t p0, uint32_t nthr, uint32_t npairs,
                                                bool want_exp, unsigned long long *s_best, int *s_origin,
                                                unsigned *s_exp) {
    if (threadIdx.x == 0) *s_exp = 0u;
    const bool hist = !P.full && !P.skip;
    if (hist)
        for (int i = threadIdx.x; i < WIN_CELLS; i += FAST_THREADS) f_dsm[i] = 0u;
    const uint32_t iters = p0 < npairs ? (npairs - 1 - p0) / nthr + 1 : 0u;
    const double2 *const cx[3] = {cx0, cx1, cx2};
    double2 sx[SAMPLE_PAIRS][D], sv[SAMPLE_PAIRS];
#pragma unroll
    for (int k = 0; k < SAMPLE_PAIRS; ++k) {
        const uint32_t it = (uint32_t)(((uint64_t)iters * k) / SAMPLE_PAIRS);
        const bool ok = it < iters;
        const uint32_t q = p0 + it * nthr;
#pragma unroll
        for (int d = 0; d < D; ++d) sx[k][d] = ok ? __ldcs(cx[d] + q) : make_double2(0.0, 0.0);
        sv[k] = (ok && A == 1) ? __ldcs(cv + q) : make_double2(0.0, 0.0);
    }
    __syncthreads();
    unsigned emax = 0u;
#pragma unroll
    for (int k = 0; k < SAMPLE_PAIRS; ++k) {
        const uint32_t it = (uint32_t)(((uint64_t)iters * k) / SAMPLE_PAIRS);
        if (it >= iters) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const double v = h ? sv[k].y : sv[k].x;
            const unsigned eb = ((unsigned)__double2hiint(v) >> 20) & 0x7ffu;
            if (A == 1 && eb != 0x7ffu && eb > emax) emax = eb;
            if (!hist) continue;
            bool inside = true;
            int cell = 0, mul = 1;
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const double x = h ? sx[k][d].y : sx[k][d].x;
                inside = inside && (G.lo[d] <= x) && (x <= G.hi[d]);
                const int kd = min(floor_nonneg(__dmul_rn(__dsub_rn(x, G.lo[d]), G.scale[d])), G.res[d] - 1);
                cell += (kd / P.cs[d]) * mul;
                mul *= P.nc[d];
            }
            DB_CHECK(!inside || (cell >= 0 && cell < WIN_CELLS));
            if (inside) atomicAdd(&f_dsm[cell], 1u);
        }
    }
    if (want_exp) {
        const unsigned m = __reduce_max_sync(0xffffffffu, emax);
        if ((threadIdx.x & 31) == 0 && m) atomicMax(s_exp, m);
    }
    __syncthreads();
    if (hist) {
        pick_box<D>(P, G.res[0], G.res[1], G.res[2], f_dsm, s_best, s_origin);
    } else if (threadIdx.x < 4) {
        s_origin[threadIdx.x] = threadIdx.x == 3 && P.skip ? 1 : 0;
    }
    __syncthreads();  // the histogram scratch becomes the window after this
}

template <int D, int A, int SM, int MM, bool XS>
__global__ void __launch_bounds__(FAST_THREADS, 1)
    k_bin_fast(Geom g, Inputs in, Accum acc, uint32_t npairs, int head, int wcap, int32_t *wcache, int reuse,
               unsigned long long *ktrace) {
    constexpr bool HS = A == 1 && SM == 1, HM = A == 1 && MM == 1;
    auto trace = [&](int k) {  // DATABIN_TRACE: per-CTA phase timestamps
        if (ktrace && threadIdx.x == 0) {
            unsigned long long ns;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
            ktrace[blockIdx.x * 4 + k] = ns;
        }
    };
    trace(0);
    __shared__ unsigned long long s_best[FAST_THREADS / 32];
    __shared__ int s_origin[6];
    __shared__ unsigned s_exp;
    __shared__ int s_xr[2 * BIN_MAX_ATTR];
    if (XS) xr_init(s_xr);
    FastCtx<D> c;
    unsigned long long *const count = acc.count;
    double *const sum = acc.sum;

    const double2 *cx[D];
#pragma unroll
    for (int d = 0; d < D; ++d) cx[d] = (const double2 *)(in.ax[d] + head);
    const double2 *cv = (const double2 *)((A == 1 ? in.at[0] : in.ax[0]) + head);
    const uint32_t nthr = gridDim.x * FAST_THREADS;
    const uint32_t p0 = blockIdx.x * FAST_THREADS + threadIdx.x;
    int res[3];
    {
        const DGeom G = load_geom<D>(g, acc.bounds);
        if (!G.ok) return;  // degenerate auto bounds: finalize reports it (uniform: every thread returns)
        // ---- this CTA's window, from a sample of its own rows
        const WinPlan P = window_plan(G, D, wcap);
        // (or the one this CTA chose at an earlier execute of the handle: only speed
        // depends on the window and the fixed-point scale, and sampling costs ~15 us)
        if (reuse) {
            if (threadIdx.x < 6) s_origin[threadIdx.x] = wcache[blockIdx.x * 8 + threadIdx.x];
            if (threadIdx.x == 6) s_exp = (unsigned)wcache[blockIdx.x * 8 + 6];
            __syncthreads();
        } else {
            fast_choose_window<D, A>(G, P, cx[0], cx[D > 1 ? 1 : 0], cx[D > 2 ? 2 : 0], cv, p0, nthr, npairs, HS,
                                     s_best, s_origin, &s_exp);
            if (threadIdx.x < 6) wcache[blockIdx.x * 8 + threadIdx.x] = s_origin[threadIdx.x];
            if (threadIdx.x == 6) wcache[blockIdx.x * 8 + 6] = (int32_t)s_exp;
        }
        c.W = 1;
#pragma unroll
        for (int d = 0; d < D; ++d) {
            c.lo[d] = G.lo[d];
            c.hi[d] = G.hi[d];
            c.scale[d] = G.scale[d];
            c.resm1[d] = G.res[d] - 1;
            c.wo[d] = s_origin[d];
            c.we[d] = P.skip ? 0u : (unsigned)P.e[d];
            c.W *= c.we[d];
        }
#pragma unroll
        for (int d = 0; d < 3; ++d) res[d] = G.res[d];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // reported window (CTA 0's); static indices only
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            acc.window[d] = d < D ? c.wo[d < D ? d : 0] : 0;
            acc.window[3 + d] = d < D ? (int)c.we[d < D ? d : 0] : 1;
        }
    }
    c.fx = XS ? fx_param_exact(s_exp) : fx_param(HS ? s_exp : 0u);
    c.mm = acc.mm;
    // rows: pairs [0, S) statically strided over the threads, then pairs [S,
    // npairs) claimed by warps in blocks of 32 x TAIL_Q pairs from a counter
    // (acc.window[7], zeroed by k_prep): equal static shares left the CTAs'
    // end times 30-50 us apart (DATABIN_TRACE), idling SMs at the end
    const uint32_t k1 = npairs / nthr - (npairs / nthr) / 8;
    const uint32_t S = k1 * nthr;
    double2 bx[D], bv = make_double2(0.0, 0.0);
    if (p0 < S) {
#pragma unroll
        for (int d = 0; d < D; ++d) bx[d] = BIN_FAST_LD(cx[d] + p0);
        if (A == 1) bv = BIN_FAST_LD(cv + p0);
    }
    const uint32_t W = c.W;
    c.o_fx = HM ? 2u * W : 0u;
    c.o_cnt = c.o_fx + (HS ? 3u * W : 0u);
    {  // opaque copy: keeps the base in a register instead of re-deriving it per row
        const uint32_t sb0 = (uint32_t)__cvta_generic_to_shared(f_dsm);
        asm volatile("mov.b32 %0, %1;" : "=r"(c.sb) : "r"(sb0));
    }

    for (uint32_t i = threadIdx.x; i < c.o_fx; i += FAST_THREADS) f_dsm[i] = ~0u;  // min/max filters
    const uint32_t o_end = c.o_cnt + W;
    for (uint32_t i = c.o_fx + threadIdx.x; i < o_end; i += FAST_THREADS) f_dsm[i] = 0u;
    const unsigned lane = threadIdx.x & 31u;
    const FastX X{XS ? acc.xs : nullptr, acc.nbins, s_xr, ((o_end + 1u) & ~1u) + (threadIdx.x >> 5) * XQ_WORDS};
    uint32_t qn = 0;  // (BIN_SUM_EXACT queue fill, warp-uniform)
    __syncthreads();

    trace(1);
    uint32_t n_in = 0, rows = 0;
    {
        for (uint32_t pb = p0 - lane; pb < S; pb += nthr) {  // warp-uniform trip count
            const uint32_t pc = pb + lane;
            const bool valid = pc < S;
            const uint32_t pn = pc + nthr;
            double2 nx[D], nv = make_double2(0.0, 0.0);
            if (pn < S) {
#pragma unroll
                for (int d = 0; d < D; ++d) nx[d] = BIN_FAST_LD(cx[d] + pn);
                if (A == 1) nv = BIN_FAST_LD(cv + pn);
            }
#ifdef BIN_FAST_LOADS_ONLY  // experiment: the streaming floor of this loop (rows consumed, nothing binned)
            {
                double acc_ = bv.x + bv.y;
#pragma unroll
                for (int d = 0; d < D; ++d) acc_ += bx[d].x + bx[d].y;
                n_in += (valid && acc_ == 12345.678) ? 1u : 0u;
                rows += valid ? 2u : 0u;
#pragma unroll
                for (int d = 0; d < D; ++d) bx[d] = nx[d];
                bv = nv;
                continue;
            }
#endif
            double x[D];
#pragma unroll
            for (int d = 0; d < D; ++d) x[d] = bx[d].x;
            lean_row<D, A, SM, MM, XS>(c, x, bv.x, valid, n_in, count, sum, X, qn);
#pragma unroll
            for (int d = 0; d < D; ++d) x[d] = bx[d].y;
            lean_row<D, A, SM, MM, XS>(c, x, bv.y, valid, n_in, count, sum, X, qn);
            rows += valid ? 2u : 0u;
#pragma unroll
            for (int d = 0; d < D; ++d) bx[d] = nx[d];
            bv = nv;
        }
    }
    {  // the tail: blocks of 32 x TAIL_Q consecutive pairs per claim (coalesced)
        constexpr uint32_t TAIL_Q = 16;
        uint32_t *ctr = (uint32_t *)acc.window + 7;
        for (;;) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(ctr, 32u * TAIL_Q);
            base = __shfl_sync(0xffffffffu, base, 0) + S;
            if (base >= npairs) break;
            uint32_t pc = base + lane;
            if (pc < npairs) {
#pragma unroll
                for (int d = 0; d < D; ++d) bx[d] = BIN_FAST_LD(cx[d] + pc);
                if (A == 1) bv = BIN_FAST_LD(cv + pc);
            }
            for (uint32_t i = 0; i < TAIL_Q; ++i, pc += 32) {
                const bool valid = pc < npairs;
                const uint32_t pn = pc + 32;
                double2 nx[D], nv = make_double2(0.0, 0.0);
                if (i + 1 < TAIL_Q && pn < npairs) {
#pragma unroll
                    for (int d = 0; d < D; ++d) nx[d] = BIN_FAST_LD(cx[d] + pn);
                    if (A == 1) nv = BIN_FAST_LD(cv + pn);
                }
                double x[D];
#pragma unroll
                for (int d = 0; d < D; ++d) x[d] = bx[d].x;
                lean_row<D, A, SM, MM, XS>(c, x, bv.x, valid, n_in, count, sum, X, qn);
#pragma unroll
                for (int d = 0; d < D; ++d) x[d] = bx[d].y;
                lean_row<D, A, SM, MM, XS>(c, x, bv.y, valid, n_in, count, sum, X, qn);
                rows += valid ? 2u : 0u;
#pragma unroll
                for (int d = 0; d < D; ++d) bx[d] = nx[d];
                bv = nv;
            }
        }
    }
    // the unpaired head row (lane 0) and tail row (lane 1) of the whole input, on warp 0 of CTA 0
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        const int64_t r = lane == 0 ? (head ? 0 : -1)
                                    : (lane == 1 && ((in.n - head) & 1) ? in.n - 1 : -1);
        double x[D], v = 0.0;
#pragma unroll
        for (int d = 0; d < D; ++d) x[d] = r >= 0 ? in.ax[d][r] : 0.0;
        if (A == 1 && r >= 0) v = in.at[0][r];
        lean_row<D, A, SM, MM, XS>(c, x, v, r >= 0, n_in, count, sum, X, qn);
        rows += r >= 0 ? 1u : 0u;
    }
    if (XS) {  // the exact-sum queue's remainder
        __syncwarp();
        if (lane < qn) xsum_add_double(X.xs, X.B, 0, f_dsm[X.qb + lane], ((const double *)(f_dsm + X.qb + XQ))[lane], X.sxr);
    }
    unsigned long long in_w = n_in, out_w = rows - n_in;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        in_w += __shfl_xor_sync(0xffffffffu, in_w, o);
        out_w += __shfl_xor_sync(0xffffffffu, out_w, o);
    }
    if (lane == 0) {
        if (in_w) atomicAdd(&count[acc.nbins], in_w);
        if (out_w) atomicAdd(&count[acc.nbins + 1], out_w);
    }
    __syncthreads();
    trace(2);

    // flush the window into the global accumulator (L2 reductions; with the
    // balanced tail all CTAs flush at once: ~25 us, vs ~10 us when their end
    // times were spread.  Rotating each CTA's flush order measured slower.)
    for (uint32_t l = threadIdx.x; l < W; l += FAST_THREADS) {
        const unsigned long long cnt = f_dsm[c.o_cnt + l];
        if (cnt == 0) continue;
        uint32_t rem = l, b = 0, mul = 1;
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const uint32_t kd = rem % c.we[d] + (uint32_t)c.wo[d];
            rem /= c.we[d];
            b += kd * mul;
            mul *= (uint32_t)res[d];
        }
        DB_CHECK(b < acc.nbins);
        atomicAdd(&count[b], cnt);
        if (HS) {
            const uint32_t w0 = c.o_fx + l;
            if (XS) {
                xsum_add_fixed(X.xs, X.B, 0, b, f_dsm[w0], f_dsm[w0 + W], f_dsm[w0 + 2 * W], cnt, FX_OFFSET, c.fx.F,
                               s_xr);
            } else {
                const double d = fx_to_double(f_dsm[w0], f_dsm[w0 + W], f_dsm[w0 + 2 * W], cnt, c.fx.inv_scale);
                if (d != 0.0) atomicAdd(&sum[b], d);
            }
        }
    }
    if (XS) {
        __syncthreads();
        xr_publish(s_xr, 1, acc.xrange);
    }
    if (ktrace) {
        __syncthreads();
        trace(3);
    }
}

// Eligible: <= 1 attribute, bins < 2^29, 16-byte pairs (all columns in the same
// 16-byte phase), fewer than 2^31 pairs.
bool fast_eligible(const Inputs &in, const Accum &acc, int ndim) {
    if (in.nattr > 1 || acc.nbins >= (1ull << 29)) return false;
    const uintptr_t ph = (uintptr_t)in.ax[0] & 15u;
    if (ph % 8) return false;
    for (int d = 0; d < ndim; ++d)
        if (((uintptr_t)in.ax[d] & 15u) != ph) return false;
    if (in.nattr == 1 && (acc.load_mask & 1u) && (((uintptr_t)in.at[0] & 15u) != ph)) return false;
    const int64_t head = ph ? 1 : 0;
    return in.n >= 2 + head && (in.n - head) / 2 < (1ll << 31);
}

template <int D, int A, int SM, int MM, bool XS>
static cudaError_t launch_fast_t(const Geom &g, const Inputs &in, const Accum &acc, const LaunchCfg &lc, int smem,
                                 int wcap, int32_t *wcache, int reuse, unsigned long long *ktrace, cudaStream_t s) {
    const int head = ((uintptr_t)in.ax[0] & 15u) ? 1 : 0;
    const uint32_t npairs = (uint32_t)((in.n - head) / 2);
    int blocks = lc.sms;  // one persistent CTA per SM: the whole shared memory holds the window
    const int64_t maxb = ((int64_t)npairs + FAST_THREADS - 1) / FAST_THREADS;
    if (maxb < blocks) blocks = (int)(maxb > 0 ? maxb : 1);
    auto kern = k_bin_fast<D, A, SM, MM, XS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<blocks, FAST_THREADS, smem, s>>>(g, in, acc, npairs, head, wcap, wcache, reuse, ktrace);
    return cudaGetLastError();
}

template <int D>
static cudaError_t launch_fast_d(const Geom &g, const Inputs &in, const Accum &acc, const LaunchCfg &lc, int smem,
                                 int wcap, int32_t *wc, int reuse, unsigned long long *kt, cudaStream_t s) {
    if (in.nattr == 0 || !(acc.load_mask & 1u))
        return launch_fast_t<D, 0, 0, 0, false>(g, in, acc, lc, smem, wcap, wc, reuse, kt, s);
    const bool sm = acc.sum_mask & 1u, mm = acc.mm_mask & 1u, xs = acc.xs != nullptr;
    if (sm && mm) {
        if (xs) return launch_fast_t<D, 1, 1, 1, true>(g, in, acc, lc, smem, wcap, wc, reuse, kt, s);
        return launch_fast_t<D, 1, 1, 1, false>(g, in, acc, lc, smem, wcap, wc, reuse, kt, s);
    }
    if (sm) {
        if (xs) return launch_fast_t<D, 1, 1, 0, true>(g, in, acc, lc, smem, wcap, wc, reuse, kt, s);
        return launch_fast_t<D, 1, 1, 0, false>(g, in, acc, lc, smem, wcap, wc, reuse, kt, s);
    }
    return launch_fast_t<D, 1, 0, 1, false>(g, in, acc, lc, smem, wcap, wc, reuse, kt, s);
}

cudaError_t launch_bin_fast(const Geom &g, const Inputs &in, const Accum &acc, const LaunchCfg &lc, int smem,
                            int wcap, int32_t *wcache, int reuse, unsigned long long *ktrace, cudaStream_t s) {
    switch (g.ndim) {
    case 1: return launch_fast_d<1>(g, in, acc, lc, smem, wcap, wcache, reuse, ktrace, s);
    case 2: return launch_fast_d<2>(g, in, acc, lc, smem, wcap, wcache, reuse, ktrace, s);
    default: return launch_fast_d<3>(g, in, acc, lc, smem, wcap, wcache, reuse, ktrace, s);
    }
}

}  // namespace db
