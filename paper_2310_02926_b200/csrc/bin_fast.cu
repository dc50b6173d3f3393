// bin_fast.cu -- k_bin_fast: the accumulate kernel (a4 + a5) for the common
// case of at most one binned attribute with 16-byte-aligned columns (C1, C3,
// C4, C5 and the paper's Fig. 1 sum-of-mass), same window layout and
// arithmetic as k_bin (bin_general.cu), written for few instructions per row:
//
//  * 32-bit pair indices, shared memory addressed as one u32 array with
//    warp-uniform word offsets (no generic-pointer round trips);
//  * one 16-byte pair per column prefetched one step ahead in registers;
//  * a per-warp queue of rare work.  Rows outside the window (~8% on C3) and
//    min/max candidates inside it (~12%: a CTA-bin sees only ~80 rows, so its
//    running extremes still move) would otherwise be divergent branches that
//    nearly every warp takes.  Lanes append (kind | bin, value) with a ballot
//    and the warp executes 32 queued items at a time with every lane busy,
//    as fire-and-forget L2 reductions (REDG.ADD / REDG.MIN, no loads).
#include <cuda_runtime.h>
#include <stdint.h>

#include "db_internal.h"
#include "dev_common.cuh"
#include "xsum.cuh"

namespace db {

extern __shared__ __align__(16) uint32_t f_dsm[];

#ifndef BIN_FAST_THREADS
#define BIN_FAST_THREADS 1024
#endif
constexpr int FAST_THREADS = BIN_FAST_THREADS;
constexpr int QCAP = 64;            // >= 31 leftover + 32 new items
constexpr int QWORDS = 3 * QCAP;    // u32 tags[QCAP] + f64 vals[QCAP]
constexpr uint32_t QBIN = (1u << 29) - 1;
enum : uint32_t { QK_GLOBAL = 1u, QK_MIN = 2u, QK_MAX = 4u };

int fast_queue_bytes() { return (FAST_THREADS / 32) * QWORDS * 4 + 16; }

// Shared-memory window accesses through 32-bit shared-window addresses from one
// base register (BIN_SADDR=1): generic atomics on the extern array made the
// compiler re-derive the window base (S2R SR_CgaCtaId + LEA) for every row.
#ifndef BIN_SADDR
#define BIN_SADDR 1
#endif
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
};

template <int D, int A, int SM, int MM, bool XS>
__device__ __forceinline__ uint32_t fast_row(const FastCtx<D> &c, const double (&x)[D], double v, bool valid,
                                             uint32_t &n_in) {
    constexpr bool HS = A == 1 && SM == 1, HM = A == 1 && MM == 1;
    bool ok = valid;
    int k[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
        ok = ok && (c.lo[d] <= x[d]) && (x[d] <= c.hi[d]);
        k[d] = min(floor_nonneg(__dmul_rn(__dsub_rn(x[d], c.lo[d]), c.scale[d])), c.resm1[d]);
    }
    if (!ok) return 0u;
    ++n_in;
    bool inw = true;
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
    if (!inw) return (QK_GLOBAL << 29) | b;
    if (BIN_SADDR) s_red_add(c.sb + 4u * (c.o_cnt + l), 1u);
    else atomicAdd(&f_dsm[c.o_cnt + l], 1u);
    const uint32_t W = c.W;
    uint32_t tag = 0;
    if (HS) {
        const uint32_t w0 = c.o_fx + l;
        unsigned qmid;
        unsigned long long q = 0;
        bool fx;
        if (XS) {
            fx = fx_quant_exact(c.fx, v, q);
        } else {
            fx = fx_path(c.fx, v);
            if (fx) q = fx_quant(c.fx, v);
        }
        if (fx) {
            const unsigned qlo = (unsigned)q;
            qmid = (unsigned)(q >> 32);
            const unsigned old = BIN_SADDR ? s_atom_add(c.sb + 4u * w0, qlo) : atomicAdd(&f_dsm[w0], qlo);
            qmid += (old + qlo < old) ? 1u : 0u;
        } else {  // rare: outside the fixed range -> sum (and min/max) go global; count stays here
            tag = ((QK_GLOBAL | QK_MIN) << 29) | b;
            qmid = FX_OFFSET_MID;
        }
        const unsigned old2 = BIN_SADDR ? s_atom_add(c.sb + 4u * (w0 + W), qmid) : atomicAdd(&f_dsm[w0 + W], qmid);
        if (old2 + qmid < old2) {
            if (BIN_SADDR) s_red_add(c.sb + 4u * (w0 + 2 * W), 1u);
            else atomicAdd(&f_dsm[w0 + 2 * W], 1u);
        }
    }
    if (HM && tag == 0) {
        const unsigned long long e = enc_total(v);
        const unsigned eh = (unsigned)(e >> 32), neh = ~eh;
        uint2 f;  // one LDS.64; stale values are safe (the words only decrease)
        const uint32_t fa = BIN_SADDR ? c.sb + 8u * l : (unsigned)__cvta_generic_to_shared(&f_dsm[2 * l]);
        asm volatile("ld.volatile.shared.v2.u32 {%0, %1}, [%2];" : "=r"(f.x), "=r"(f.y) : "r"(fa));
        uint32_t kind = 0;
        if (eh <= f.x) {
            kind |= QK_MIN;
            if (eh < f.x) {
                if (BIN_SADDR) s_red_min(fa, eh);
                else atomicMin(&f_dsm[2 * l], eh);
            }
        }
        if (neh <= f.y) {
            kind |= QK_MAX;
            if (neh < f.y) {
                if (BIN_SADDR) s_red_min(fa + 4u, neh);
                else atomicMin(&f_dsm[2 * l + 1], neh);
            }
        }
        if (kind) tag = (kind << 29) | b;
    }
    return tag;
}

// One queued item as fire-and-forget L2 reductions.  A QK_GLOBAL item from
// inside the window (value outside the fixed range) carries sum + min/max but
// its count is already in shared memory -> the low bit of `kind` picks count.
// `gf` (the CTA's window covers under half its rows, e.g. uniform data): the
// global rows' min/max first read the slot pair from L2 and reduce only when
// they improve it (stale reads are safe: the slots only decrease), which turns
// two L2 atomics per global row into one load for all but the first rows.
// Exact sums (BIN_SUM_EXACT): digit rows instead of the f64 reduction.
struct FastX {
    long long *xs;  // nullptr: BIN_SUM_FAST
    uint64_t B;
    int *sxr;       // this CTA's touched digit range (shared memory)
};

template <int A, int SM, int MM, bool XS>
__device__ __forceinline__ void fast_exec(uint32_t tag, double v, unsigned long long *count, double *sum,
                                          ulonglong2 *mm, bool gf, const FastX &X) {
    constexpr bool HS = A == 1 && SM == 1, HM = A == 1 && MM == 1;
    const uint32_t kind = tag >> 29, b = tag & QBIN;
    if (kind & QK_GLOBAL) {
        if (!(kind & QK_MIN)) atomicAdd(&count[b], 1ull);  // QK_GLOBAL|QK_MIN marks "count already counted"
        if (HS) {
            if (XS) xsum_add_double(X.xs, X.B, 0, b, v, X.sxr);
            else atomicAdd(&sum[b], v);
        }
        if (HM) {
            const unsigned long long e = enc_total(v);
            ulonglong2 cur = make_ulonglong2(~0ull, ~0ull);
            if (gf) cur = __ldcg(&mm[b]);
            if (e < cur.x) atomicMin(&mm[b].x, e);
            if (~e < cur.y) atomicMin(&mm[b].y, ~e);
        }
    } else if (HM) {
        const unsigned long long e = enc_total(v);
        if (kind & QK_MIN) atomicMin(&mm[b].x, e);
        if (kind & QK_MAX) atomicMin(&mm[b].y, ~e);
    }
}

template <int A, int SM, int MM, bool XS>
__device__ __forceinline__ void fast_push(uint32_t qb, uint32_t &qn, uint32_t tag, double v, unsigned lane,
                                          unsigned long long *count, double *sum, ulonglong2 *mm, bool gf,
                                          const FastX &X) {
    const unsigned m = __ballot_sync(0xffffffffu, tag != 0);
    if (m == 0) return;
    double *vals = (double *)&f_dsm[qb + QCAP];
    if (tag) {
        const unsigned pos = qn + __popc(m & ((1u << lane) - 1u));
        f_dsm[qb + pos] = tag;
        vals[pos] = v;
    }
    qn += __popc(m);
    if (qn >= 32) {
        __syncwarp();
        const uint32_t t = f_dsm[qb + lane];
        const double vv = vals[lane];
        const unsigned rest = qn - 32;
        uint32_t t2 = 0;
        double v2 = 0.0;
        if (lane < rest) {
            t2 = f_dsm[qb + 32 + lane];
            v2 = vals[32 + lane];
        }
        __syncwarp();
        if (lane < rest) {
            f_dsm[qb + lane] = t2;
            vals[lane] = v2;
        }
        qn = rest;
        fast_exec<A, SM, MM, XS>(t, vv, count, sum, mm, gf, X);
        __syncwarp();
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
    ulonglong2 *const mm = (ulonglong2 *)acc.mm;

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
#ifdef BIN_GF_OFF
    const bool gf = false;
#else
    const bool gf = s_origin[3] != 0;
#endif
    double2 bx[D], bv = make_double2(0.0, 0.0);
    if (p0 < npairs) {
#pragma unroll
        for (int d = 0; d < D; ++d) bx[d] = __ldcs(cx[d] + p0);
        if (A == 1) bv = __ldcs(cv + p0);
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
    const uint32_t qb = ((o_end + 3u) & ~3u) + (threadIdx.x >> 5) * QWORDS;
    const FastX X{XS ? acc.xs : nullptr, acc.nbins, s_xr};
    uint32_t qn = 0;
    __syncthreads();

    trace(1);
    uint32_t n_in = 0, rows = 0;
    for (uint32_t pb = p0 - lane; pb < npairs; pb += nthr) {  // warp-uniform trip count
        const uint32_t pc = pb + lane;
        const bool valid = pc < npairs;
        const uint32_t pn = pc + nthr;
        double2 nx[D], nv = make_double2(0.0, 0.0);
        if (pn < npairs) {
#pragma unroll
            for (int d = 0; d < D; ++d) nx[d] = __ldcs(cx[d] + pn);
            if (A == 1) nv = __ldcs(cv + pn);
        }
        double x[D];
#pragma unroll
        for (int d = 0; d < D; ++d) x[d] = bx[d].x;
        uint32_t t0 = fast_row<D, A, SM, MM, XS>(c, x, bv.x, valid, n_in);
        fast_push<A, SM, MM, XS>(qb, qn, t0, bv.x, lane, count, sum, mm, gf, X);
#pragma unroll
        for (int d = 0; d < D; ++d) x[d] = bx[d].y;
        uint32_t t1 = fast_row<D, A, SM, MM, XS>(c, x, bv.y, valid, n_in);
        fast_push<A, SM, MM, XS>(qb, qn, t1, bv.y, lane, count, sum, mm, gf, X);
        rows += valid ? 2u : 0u;
#pragma unroll
        for (int d = 0; d < D; ++d) bx[d] = nx[d];
        bv = nv;
    }
    // the unpaired head row (lane 0) and tail row (lane 1) of the whole input, on warp 0 of CTA 0
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        const int64_t r = lane == 0 ? (head ? 0 : -1)
                                    : (lane == 1 && ((in.n - head) & 1) ? in.n - 1 : -1);
        double x[D], v = 0.0;
#pragma unroll
        for (int d = 0; d < D; ++d) x[d] = r >= 0 ? in.ax[d][r] : 0.0;
        if (A == 1 && r >= 0) v = in.at[0][r];
        const uint32_t t = fast_row<D, A, SM, MM, XS>(c, x, v, r >= 0, n_in);
        rows += r >= 0 ? 1u : 0u;
        fast_push<A, SM, MM, XS>(qb, qn, t, v, lane, count, sum, mm, gf, X);
    }
    __syncwarp();
    if (lane < qn) fast_exec<A, SM, MM, XS>(f_dsm[qb + lane], ((double *)&f_dsm[qb + QCAP])[lane], count, sum, mm, gf, X);

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

    // flush the window into the global accumulator (L2 reductions)
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
