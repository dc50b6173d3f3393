// dev_common.cuh -- device helpers shared by the DataBin kernels (csrc/*.cu).
// Part of the product library; shares nothing with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "db_internal.h"

// Streaming column loads: L2-cached (ld.global.cg).  The evict-first hint
// (ld.global.cs) measured slower on every streaming kernel tried (C4 keys
// 7.05 vs 5.8 ms, C3 k_bin_fast 0.565 vs 0.559 ms).
#ifndef DB_LD_STREAM
#define DB_LD_STREAM __ldcg
#endif

namespace db {

// Checked build (-DDATABIN_CHECKED, tools/build_variants.py checked=DATABIN_CHECKED):
// device-side bounds checks on every computed shared-memory window index,
// global bin index and scatter position; a failing check prints its site and
// traps, so the execute fails loudly at bin_wait.  (compute-sanitizer is not
// available on the GPU pool: profiles/r02_compute_sanitizer_closed.txt.)
#ifdef DATABIN_CHECKED
#define DB_CHECK(c)                                                                             \
    do {                                                                                        \
        if (!(c)) {                                                                             \
            printf("DB_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c,  \
                   (int)blockIdx.x, (int)threadIdx.x);                                         \
            __trap();                                                                           \
        }                                                                                       \
    } while (0)
#else
#define DB_CHECK(c) \
    do {            \
    } while (0)
#endif

__device__ __forceinline__ unsigned long long enc_total(double x) {
    unsigned long long b = (unsigned long long)__double_as_longlong(x);
    unsigned long long m = (unsigned long long)((long long)b >> 63);
    return b ^ (m | 0x8000000000000000ull);
}
__device__ __forceinline__ double dec_total(unsigned long long e) {
    unsigned long long m = ~(unsigned long long)((long long)e >> 63);
    return __longlong_as_double((long long)(e ^ (m | 0x8000000000000000ull)));
}

// Shared-memory 2x64-bit read that the compiler may not cache in registers
// (other threads update these words atomically; see the monotone filter).
__device__ __forceinline__ ulonglong2 lds_volatile_u64x2(const ulonglong2 *p) {
    ulonglong2 r;
    unsigned a = (unsigned)__cvta_generic_to_shared(p);
    asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];" : "=l"(r.x), "=l"(r.y) : "r"(a));
    return r;
}

// floor(t) for 0 <= t < 2^31 without the (slow) F2I.F64 conversion pipe:
// t + 2^52 rounded toward -inf lands in [2^52, 2^53) where the ulp is 1, so
// its low mantissa word is exactly floor(t).  Out-of-range t (rows outside the
// mesh, NaN) give garbage that the caller masks.  Measured: the bin-index
// stage went from 0.14 ms to ... on C3 (profiles/r01_ablation.txt).
__device__ __forceinline__ int floor_nonneg(double t) {
    return __double2loint(__dadd_rd(t, 4503599627370496.0));
}

struct DGeom {
    double lo[3], hi[3], scale[3];
    int res[3];
    bool ok;
};

// Realised mesh bounds and scales; identical in every CTA of every kernel.
// ND = compile-time dimensionality (0 = take g.ndim at run time).
template <int ND = 0>
__device__ __forceinline__ DGeom load_geom(const Geom &g, const unsigned long long *bounds) {
    DGeom G;
    G.ok = true;
    const int ndim = ND > 0 ? ND : g.ndim;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        G.res[d] = d < ndim ? g.res[d] : 1;
        G.lo[d] = 0.0;
        G.hi[d] = 1.0;
        G.scale[d] = 1.0;
        if (d >= ndim) continue;
        double lo = g.lo[d], hi = g.hi[d];
        if (g.bounds_auto) {
            unsigned long long elo = bounds[d], nhi = bounds[ndim + d];
            if (elo == ~0ull || nhi == ~0ull) G.ok = false;  // no non-NaN row anywhere
            lo = dec_total(elo);
            hi = dec_total(~nhi);
            if (lo == hi) {  // reading R4
                lo = __dsub_rn(lo, 0.5);
                hi = __dadd_rn(hi, 0.5);
            }
        }
        G.lo[d] = lo;
        G.hi[d] = hi;
        G.scale[d] = __ddiv_rn((double)G.res[d], __dsub_rn(hi, lo));
        // reading R4: usable bounds are finite, lo < hi, with a finite width and
        // scale (manual bounds are checked the same way at bin_init)
        if (g.bounds_auto && (!(lo < hi) || isinf(lo) || isinf(hi) || isinf(__dsub_rn(hi, lo)) || isinf(G.scale[d])))
            G.ok = false;
    }
    return G;
}

// Bin coordinates of one row; returns false if outside the mesh.
template <int D>
__device__ __forceinline__ bool bin_coords(const DGeom &G, const double (&x)[D], int (&k)[D]) {
    bool in = true;
#pragma unroll
    for (int d = 0; d < D; ++d) {
        in = in && (G.lo[d] <= x[d]) && (x[d] <= G.hi[d]);
        double t = __dmul_rn(__dsub_rn(x[d], G.lo[d]), G.scale[d]);
        int kd = floor_nonneg(t);  // floor for in-bounds rows; garbage (masked by `in`) otherwise
        k[d] = min(kd, G.res[d] - 1);
    }
    return in;
}

// ---- fixed-point window sums (see bin_general.cu / bin_fast.cu headers) ----
// q' = round(v * 2^F) + 2^54 with |round(v * 2^F)| < 2^54, summed exactly in
// 96 bits; the flush subtracts count * 2^54.  (The count cannot be recovered
// from the sum alone: sum q / 2^55 is not bounded by 1/2 -- tried and
// rejected, WE4 catches it -- so windows keep an explicit count.)
// |q| < 2^54 keeps the middle word's per-row addend below 2^23, so it carries
// into the high word only every ~500 rows (a wider q made every ~4th row pay
// an extra shared atomic: +3.1M ATOMS on C3).
constexpr long long FX_OFFSET = 1ll << 54;
constexpr unsigned FX_OFFSET_MID = (unsigned)(FX_OFFSET >> 32);

struct FxParam {
    int F;
    double scale;      // 2^F
    double inv_scale;  // 2^-F
    unsigned lo;       // biased exponents [lo, lo + span) take the fixed path (plus exact 0)
    unsigned span;
};

// BIN_SUM_FAST: F from the sampled max exponent of the attribute: E_hi = e_max
// + 3 (biased eb_hi), F = 54 - E_hi; values in [2^(E_hi-9), 2^E_hi) ->
// quantisation <= 2^-46 |v| (within reading R8).
__device__ __forceinline__ FxParam fx_param(unsigned fxexp) {
    int eb_hi = (int)fxexp + 3;
    if (fxexp == 0) eb_hi = 1023 + 1;  // nothing sampled: assume |v| < 2
    const int F = 54 - (eb_hi - 1023);
    const bool usable = F > -900 && F < 900;
    const int eb_lo = max(eb_hi - 9, 1);
    FxParam P;
    P.F = F;
    P.lo = usable ? (unsigned)eb_lo : 1u;
    P.span = usable ? (unsigned)(eb_hi - eb_lo) : 0u;
    P.scale = usable ? ldexp(1.0, F) : 0.0;
    P.inv_scale = usable ? ldexp(1.0, -F) : 0.0;
    return P;
}

// BIN_SUM_EXACT: the grid's top binade is the sampled max one (E_hi = e_max
// + 1, F = 54 - E_hi), so every value of that binade and the next lies on the
// grid 2^-F exactly; a value takes the fixed path only if it is exactly on
// the grid and |q| < 2^54 (fx_quant_exact), else it goes to the digit rows.
__device__ __forceinline__ FxParam fx_param_exact(unsigned fxexp) {
    FxParam P = fx_param(fxexp == 0 ? 0u : (fxexp < 3u ? 1u : fxexp - 2u));
    P.lo = 1u;  // the exactness test decides
    P.span = P.scale != 0.0 ? 2046u : 0u;
    return P;
}

__device__ __forceinline__ bool fx_path(const FxParam &P, double v) {
    const unsigned eb = ((unsigned)__double2hiint(v) >> 20) & 0x7ffu;
    return eb - P.lo < P.span || v == 0.0;
}

// q' = round(v * 2^F) + 2^54 in (0, 2^55)
__device__ __forceinline__ unsigned long long fx_quant(const FxParam &P, double v) {
    return (unsigned long long)(__double2ll_rn(__dmul_rn(v, P.scale)) + FX_OFFSET);
}

// exact mode: q' as above when v * 2^F is an integer below 2^54 in magnitude
// (the multiply by a power of two is exact unless it leaves the normal range,
// which the round trip q * 2^-F == v also rules out); false -> digit rows.
__device__ __forceinline__ bool fx_quant_exact(const FxParam &P, double v, unsigned long long &qp) {
    const long long q = __double2ll_rn(__dmul_rn(v, P.scale));
    qp = (unsigned long long)(q + FX_OFFSET);
    return P.span != 0u && q > -FX_OFFSET && q < FX_OFFSET && __dmul_rn(__ll2double_rn(q), P.inv_scale) == v;
}

// Exact 96-bit fixed-point sum of cnt offset values -> f64 (one rounding when
// |q| < 2^62, else <= 1 ulp).
__device__ __forceinline__ double fx_to_double(uint32_t lo, uint32_t mid, uint32_t hi, unsigned long long cnt,
                                               double inv_scale) {
    unsigned __int128 qp = ((unsigned __int128)hi << 64) | ((unsigned __int128)mid << 32) | lo;
    __int128 q = (__int128)qp - (__int128)cnt * (__int128)FX_OFFSET;
    double d;
    if (q >= -(((__int128)1) << 62) && q < (((__int128)1) << 62)) {
        d = __ll2double_rn((long long)q);
    } else {
        long long qh = (long long)(q >> 32);
        unsigned long long ql = (unsigned long long)(q & 0xffffffffll);
        d = __dadd_rn(__dmul_rn(__ll2double_rn(qh), 4294967296.0), __ull2double_rn(ql));
    }
    return __dmul_rn(d, inv_scale);
}

// Compile-time op masks: for A == 1 the launchers instantiate SM/MM in {0,1}
// (sum requested, min/max requested); otherwise SM = MM = -1 (runtime masks).
template <int A, int SM, int MM>
struct OpMask {
    __device__ static __forceinline__ bool sum(uint32_t rt, int a) { return SM >= 0 ? (SM >> a) & 1 : (rt >> a) & 1u; }
    __device__ static __forceinline__ bool mm(uint32_t rt, int a) { return MM >= 0 ? (MM >> a) & 1 : (rt >> a) & 1u; }
    __device__ static __forceinline__ uint32_t sum_slot(uint32_t rt, int a) { return SM >= 0 ? 0u : __popc(rt & ((1u << a) - 1u)); }
    __device__ static __forceinline__ uint32_t mm_slot(uint32_t rt, int a) { return MM >= 0 ? 0u : __popc(rt & ((1u << a) - 1u)); }
};

// Window geometry of one CTA (from the window kernel) and derived constants.
struct WinGeom {
    int wo[3];
    unsigned we[3];
    int resm1[3];  // res - 1 per axis (upper clamp)
    uint32_t W;
};

__device__ __forceinline__ WinGeom load_window(const DGeom &G, const int32_t *window, int D) {
    WinGeom w;
    w.W = 1;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        w.wo[d] = d < D ? window[d] : 0;
        w.we[d] = d < D ? (unsigned)window[3 + d] : 1u;
        w.resm1[d] = G.res[d] - 1;
        w.W *= w.we[d];
    }
    return w;
}

// ---- window planning (shared by the window kernels and k_bin_fast) ----
constexpr int WIN_CELLS = 4096;

struct WinPlan {
    int e[3], cs[3], nc[3];
    bool full, skip;
};

__device__ __forceinline__ WinPlan window_plan(const DGeom &G, int D, int wcap) {
    WinPlan P;
    long long total = (long long)G.res[0] * G.res[1] * G.res[2];
    P.skip = !G.ok || wcap <= 0;
    P.full = !P.skip && total <= wcap;
    for (int d = 0; d < 3; ++d) P.e[d] = P.full ? G.res[d] : 1;
    if (!P.full && !P.skip) {
        const int *res = G.res;
        if (D == 1) {
            P.e[0] = min(res[0], wcap);
        } else if (D == 2) {
            int s = (int)floor(sqrt((double)wcap));
            P.e[0] = min(res[0], max(1, s));
            P.e[1] = min(res[1], wcap / P.e[0]);
            if (P.e[1] == res[1]) P.e[0] = min(res[0], wcap / res[1]);
        } else {
            int c = (int)floor(cbrt((double)wcap));
            P.e[0] = min(res[0], max(1, c));
            P.e[1] = min(res[1], max(1, c));
            P.e[2] = min(res[2], wcap / (P.e[0] * P.e[1]));
            if (P.e[2] == res[2]) {
                int s = (int)floor(sqrt((double)(wcap / res[2])));
                P.e[0] = min(res[0], max(1, s));
                P.e[1] = min(res[1], wcap / (res[2] * P.e[0]));
            }
        }
    }
    int ncmax = D == 1 ? WIN_CELLS : (D == 2 ? 64 : 16);
    for (int d = 0; d < 3; ++d) {
        P.cs[d] = (G.res[d] + ncmax - 1) / ncmax;
        P.nc[d] = (G.res[d] + P.cs[d] - 1) / P.cs[d];
    }
    return P;
}

// Inclusive scan of one line of <= 64 cells (stride `step`) by one warp.
__device__ __forceinline__ void warp_line_scan(unsigned *h, int base, int step, int len) {
    const int lane = threadIdx.x & 31;
    const int i0 = 2 * lane, i1 = 2 * lane + 1;
    unsigned a = i0 < len ? h[base + i0 * step] : 0u, b = i1 < len ? h[base + i1 * step] : 0u;
    unsigned s = a + b;
    for (int o = 1; o < 32; o <<= 1) {
        unsigned y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
    }
    const unsigned pre = s - a - b;
    if (i0 < len) h[base + i0 * step] = pre + a;
    if (i1 < len) h[base + i1 * step] = pre + a + b;
}


// Summed-area table of the coarse histogram `hist` (shared memory, nc cells),
// then the box of wc = e/cs coarse cells with the most samples (ties -> lowest
// index).  All threads of the CTA take part (blockDim >= 256); the box origin
// in bins is written to origin[0..2] (shared, int[6], see the end) and is
// valid after the return.
template <int D>
__device__ __forceinline__ void pick_box(const WinPlan P, const int res0, const int res1, const int res2,
                                         unsigned *hist, unsigned long long *best, int *origin) {
    const int res[3] = {res0, res1, res2};  // by value: no pointer into the caller's geometry
    const int *nc = P.nc;
    const int ncell = nc[0] * nc[1] * nc[2];
    const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
#pragma unroll
    for (int d = 0; d < D; ++d) {
        const int len = nc[d];
        const int lines = ncell / len;
        const int step = d == 0 ? 1 : (d == 1 ? nc[0] : nc[0] * nc[1]);
        if (len <= 64) {
            for (int ln = warp; ln < lines; ln += nwarps) {
                int base;
                if (d == 0) base = ln * nc[0];
                else if (d == 1) base = (ln % nc[0]) + (ln / nc[0]) * nc[0] * nc[1];
                else base = ln;
                warp_line_scan(hist, base, step, len);
            }
            __syncthreads();
        } else {  // 1D: Hillis-Steele over up to WIN_CELLS cells
            for (int off = 1; off < len; off <<= 1) {
                unsigned vv[16];
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    const int i = threadIdx.x + r * blockDim.x;
                    vv[r] = (i < len && i >= off) ? hist[i - off] : 0u;
                }
                __syncthreads();
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    const int i = threadIdx.x + r * blockDim.x;
                    if (i < len) hist[i] += vv[r];
                }
                __syncthreads();
            }
        }
    }
    int wc[3], np[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        wc[d] = d < D ? max(1, P.e[d] / P.cs[d]) : 1;
        np[d] = nc[d] - wc[d] + 1;
    }
    auto sat = [&](int i0, int i1, int i2) -> long long {
        if (i0 < 0 || i1 < 0 || i2 < 0) return 0;
        return hist[i0 + nc[0] * (i1 + nc[1] * i2)];
    };
    unsigned long long mybest = 0;  // (count << 32) | (0xffffffff - candidate)
    const int ncand = np[0] * np[1] * np[2];
    for (int c = threadIdx.x; c < ncand; c += blockDim.x) {
        const int o0 = c % np[0], o1 = (c / np[0]) % np[1], o2 = c / (np[0] * np[1]);
        const int a0 = o0 - 1, a1 = o1 - 1, a2 = o2 - 1;
        const int b0 = o0 + wc[0] - 1, b1 = o1 + wc[1] - 1, b2 = o2 + wc[2] - 1;
        const long long v = sat(b0, b1, b2) - sat(a0, b1, b2) - sat(b0, a1, b2) - sat(b0, b1, a2) + sat(a0, a1, b2) +
                            sat(a0, b1, a2) + sat(b0, a1, a2) - sat(a0, a1, a2);
        const unsigned long long key = ((unsigned long long)v << 32) | (0xffffffffull - (unsigned)c);
        mybest = key > mybest ? key : mybest;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, mybest, o);
        mybest = w > mybest ? w : mybest;
    }
    if ((threadIdx.x & 31) == 0) best[warp] = mybest;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long bb = 0;
        for (int i = 0; i < nwarps; ++i) bb = best[i] > bb ? best[i] : bb;
        const int c = (int)(0xffffffffull - (bb & 0xffffffffull));
        const int o[3] = {c % np[0], (c / np[0]) % np[1], c / (np[0] * np[1])};
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            int org = o[d] * P.cs[d];
            if (org + P.e[d] > res[d]) org = res[d] - P.e[d];
            origin[d] = org;
        }
        // origin[3]: the box holds under half of the sampled rows inside the
        // grid (spread-out data: most rows take the global path); origin[4],
        // origin[5]: sampled rows in the box / inside the grid
        origin[3] = (bb >> 32) * 2 < (unsigned long long)hist[ncell - 1] ? 1 : 0;
        origin[4] = (int)(bb >> 32);
        origin[5] = (int)hist[ncell - 1];
    }
    __syncthreads();
}

}  // namespace db
