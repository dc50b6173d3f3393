// kernels.cu -- sm_100a kernels of the DataBin hot path.
//
// Phases of one execute:
//   k_init      accumulator identities (reading R5)             [a3]
//   k_bounds    per-axis min/max, order-preserving u64 encoding [a2]
//   k_window    picks the shared-memory "hot window" of bins from a sample
//   k_bin       bin index (a4) + accumulate (a5): CTA-private window in
//               shared memory, global L2 reductions for the rest
//   k_finalize  avg = sum/count, decode min/max, sentinels        [a7]
// The cross-rank combine (a6) is NCCL, enqueued by handle.cpp.
//
// Arithmetic contract shared with the oracle by *definition* (not code):
//   scale_d = (double)res_d / (hi_d - lo_d)        (IEEE div, once per CTA)
//   inside  = lo_d <= x && x <= hi_d                (NaN -> outside)
//   k_d     = min(floor((x - lo_d) * scale_d), res_d - 1)   (RN sub, RN mul, no FMA)
//   b       = k_0 + res_0 * (k_1 + res_1 * k_2)     (x fastest)
// min/max use the u64 encoding enc(x) that orders like IEEE totalOrder, so
// -0.0 < +0.0 (reading R6); max is stored as ~enc(x) so every min/max slot
// is a u64 *min* (one NCCL Min allreduce covers both).
#include <cuda_runtime.h>
#include <stdint.h>

#include "db_internal.h"

namespace db {

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

struct DGeom {
    double lo[3], hi[3], scale[3];
    int res[3];
    bool ok;
};

// Realised mesh bounds and scales; identical in every CTA of every kernel.
__device__ __forceinline__ DGeom load_geom(const Geom &g, const unsigned long long *bounds) {
    DGeom G;
    G.ok = true;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        G.res[d] = d < g.ndim ? g.res[d] : 1;
        G.lo[d] = 0.0;
        G.hi[d] = 1.0;
        G.scale[d] = 1.0;
        if (d >= g.ndim) continue;
        double lo = g.lo[d], hi = g.hi[d];
        if (g.bounds_auto) {
            unsigned long long elo = bounds[d], nhi = bounds[g.ndim + d];
            if (elo == ~0ull || nhi == ~0ull) G.ok = false;  // no non-NaN row anywhere
            lo = dec_total(elo);
            hi = dec_total(~nhi);
            if (lo == hi) {  // reading R4
                lo = __dsub_rn(lo, 0.5);
                hi = __dadd_rn(hi, 0.5);
            }
            if (!(lo < hi) || isinf(lo) || isinf(hi)) G.ok = false;
        }
        G.lo[d] = lo;
        G.hi[d] = hi;
        G.scale[d] = __ddiv_rn((double)G.res[d], __dsub_rn(hi, lo));
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
        int kd = __double2int_rd(t);  // floor; saturates for out-of-range t (masked by `in`)
        k[d] = min(kd, G.res[d] - 1);
    }
    return in;
}

// ---------------------------------------------------------------- init [a3]
constexpr int WIN_CELLS_INIT = 4096;
__global__ void k_init(Accum acc, int ndim) {
    const uint64_t nb = acc.nbins;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t i = t0; i < (int64_t)nb + 2; i += stride) acc.count[i] = 0ull;
    for (int64_t i = t0; i < (int64_t)(nb * acc.nsum); i += stride) acc.sum[i] = 0.0;
    ulonglong2 ident = make_ulonglong2(~0ull, ~0ull);
    for (int64_t i = t0; i < (int64_t)(nb * acc.nmm); i += stride) ((ulonglong2 *)acc.mm)[i] = ident;
    if (t0 < 2 * ndim) acc.bounds[t0] = ~0ull;
    for (int64_t i = t0; i < WIN_CELLS_INIT; i += stride) acc.whist[i] = 0u;
    if (t0 < BIN_MAX_ATTR) acc.fxexp[t0] = 0u;
}

cudaError_t launch_init(const Accum &acc, int ndim, cudaStream_t s) {
    int64_t work = (int64_t)acc.nbins * (1 + acc.nsum + acc.nmm);
    int64_t blocks = (work / 4 + 255) / 256;
    if (blocks < 1) blocks = 1;
    if (blocks > 148 * 8) blocks = 148 * 8;
    k_init<<<(unsigned)blocks, 256, 0, s>>>(acc, ndim);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- bounds [a2]
__device__ __forceinline__ unsigned long long shfl_min_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}

template <int D>
__global__ void __launch_bounds__(512) k_bounds(Inputs in, unsigned long long *bounds) {
    unsigned long long mn[D], nmx[D];
#pragma unroll
    for (int d = 0; d < D; ++d) mn[d] = nmx[d] = ~0ull;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < in.n; i += stride) {
#pragma unroll
        for (int d = 0; d < D; ++d) {
            double x = __ldcs(in.ax[d] + i);
            if (x == x) {  // NaN rows do not define bounds
                unsigned long long e = enc_total(x);
                mn[d] = e < mn[d] ? e : mn[d];
                nmx[d] = ~e < nmx[d] ? ~e : nmx[d];
            }
        }
    }
    __shared__ unsigned long long red[2 * D][16];
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int d = 0; d < D; ++d) {
        unsigned long long a = shfl_min_u64(mn[d]), b = shfl_min_u64(nmx[d]);
        if (l == 0) { red[d][w] = a; red[D + d][w] = b; }
    }
    __syncthreads();
    if (threadIdx.x < 2 * D) {
        unsigned long long v = ~0ull;
        for (int j = 0; j < (int)(blockDim.x >> 5); ++j) v = red[threadIdx.x][j] < v ? red[threadIdx.x][j] : v;
        if (v != ~0ull) atomicMin(&bounds[threadIdx.x], v);
    }
}

cudaError_t launch_bounds(const Geom &g, const Inputs &in, const Accum &acc, const LaunchCfg &lc,
                          cudaStream_t s) {
    if (in.n == 0) return cudaSuccess;
    int64_t blocks = (in.n + 511) / 512;
    if (blocks > (int64_t)lc.sms * 4) blocks = (int64_t)lc.sms * 4;
    switch (g.ndim) {
    case 1: k_bounds<1><<<(unsigned)blocks, 512, 0, s>>>(in, acc.bounds); break;
    case 2: k_bounds<2><<<(unsigned)blocks, 512, 0, s>>>(in, acc.bounds); break;
    default: k_bounds<3><<<(unsigned)blocks, 512, 0, s>>>(in, acc.bounds); break;
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------- window
// Chooses the extents (product <= wcap) and the origin of the box of bins
// that each binning CTA privatises in shared memory.  The origin maximises
// the number of sampled rows inside the box (coarse histogram + summed-area
// table).  Only performance depends on this choice, never results.
//   k_window_sample  WIN_SAMPLE_CTAS CTAs: strided sample -> coarse histogram
//   k_window_pick    1 CTA: summed-area table, best box, writes acc.window
constexpr int WIN_THREADS = 1024;
constexpr int WIN_SAMPLE_CTAS = 64;
constexpr int WIN_SAMPLE_THREADS = 256;
constexpr int WIN_PER_THREAD = 4;
constexpr int WIN_SAMPLES = WIN_SAMPLE_CTAS * WIN_SAMPLE_THREADS * WIN_PER_THREAD;  // 65536
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

__global__ void __launch_bounds__(WIN_SAMPLE_THREADS) k_window_sample(Geom g, Inputs in, Accum acc, int wcap) {
    const int D = g.ndim;
    DGeom G = load_geom(g, acc.bounds);
    WinPlan P = window_plan(G, D, wcap);
    if (P.skip || in.n == 0) return;
    const int64_t S = in.n < WIN_SAMPLES ? in.n : WIN_SAMPLES;
    const int64_t stride = in.n / S;
    const int tid = blockIdx.x * WIN_SAMPLE_THREADS + threadIdx.x;
    // magnitude of the summed attributes: max biased exponent over the sample
    // (sets the fixed-point scale of the shared-memory sums; see k_bin)
    for (int a = 0; a < in.nattr; ++a) {
        if (!((acc.sum_mask >> a) & 1u)) continue;
        unsigned emax = 0;
#pragma unroll
        for (int k = 0; k < WIN_PER_THREAD; ++k) {
            int64_t j = tid + (int64_t)k * WIN_SAMPLE_CTAS * WIN_SAMPLE_THREADS;
            if (j < S) {
                double v = in.at[a][j * stride];
                unsigned eb = ((unsigned)__double2hiint(v) >> 20) & 0x7ffu;
                emax = (eb != 0x7ffu && eb > emax) ? eb : emax;
            }
        }
        for (int o = 16; o > 0; o >>= 1) emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
        if ((threadIdx.x & 31) == 0 && emax) atomicMax(&acc.fxexp[a], emax);
    }
    if (P.full) return;
    double x[WIN_PER_THREAD][3];
#pragma unroll
    for (int k = 0; k < WIN_PER_THREAD; ++k) {  // all loads first: one latency, not four
        int64_t j = tid + (int64_t)k * WIN_SAMPLE_CTAS * WIN_SAMPLE_THREADS;
        int64_t row = (j < S ? j : 0) * stride;
#pragma unroll
        for (int d = 0; d < 3; ++d) x[k][d] = d < D ? __ldcs(in.ax[d] + row) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < WIN_PER_THREAD; ++k) {
        int64_t j = tid + (int64_t)k * WIN_SAMPLE_CTAS * WIN_SAMPLE_THREADS;
        if (j >= S) continue;
        bool inside = true;
        int c = 0, mul = 1;
        for (int d = 0; d < D; ++d) {
            inside = inside && (G.lo[d] <= x[k][d]) && (x[k][d] <= G.hi[d]);
            int kd = min(__double2int_rd(__dmul_rn(__dsub_rn(x[k][d], G.lo[d]), G.scale[d])), G.res[d] - 1);
            c += (kd / P.cs[d]) * mul;
            mul *= P.nc[d];
        }
        if (inside) atomicAdd(&acc.whist[c], 1u);
    }
}

__global__ void __launch_bounds__(WIN_THREADS) k_window_pick(Geom g, Accum acc, int wcap) {
    __shared__ unsigned hist[WIN_CELLS];
    __shared__ unsigned long long best[WIN_THREADS / 32];
    const int D = g.ndim;
    DGeom G = load_geom(g, acc.bounds);
    WinPlan P = window_plan(G, D, wcap);
    if (P.skip) {
        if (threadIdx.x < 6) acc.window[threadIdx.x] = 0;
        return;
    }
    if (P.full) {
        if (threadIdx.x < 3) {
            acc.window[threadIdx.x] = 0;
            acc.window[3 + threadIdx.x] = G.res[threadIdx.x];
        }
        return;
    }
    const int *nc = P.nc;
    const int ncell = nc[0] * nc[1] * nc[2];
    for (int i = threadIdx.x; i < WIN_CELLS; i += blockDim.x) hist[i] = i < ncell ? acc.whist[i] : 0u;
    __syncthreads();
    // summed-area table, one axis at a time
    for (int d = 0; d < D; ++d) {
        int len = nc[d];
        int lines = ncell / len;
        int step = d == 0 ? 1 : (d == 1 ? nc[0] : nc[0] * nc[1]);
        if (D == 1) {  // Hillis-Steele over up to WIN_CELLS entries
            for (int off = 1; off < len; off <<= 1) {
                unsigned v[WIN_CELLS / WIN_THREADS];
                for (int r = 0; r < WIN_CELLS / WIN_THREADS; ++r) {
                    int i = threadIdx.x + r * WIN_THREADS;
                    v[r] = (i < len && i >= off) ? hist[i - off] : 0u;
                }
                __syncthreads();
                for (int r = 0; r < WIN_CELLS / WIN_THREADS; ++r) {
                    int i = threadIdx.x + r * WIN_THREADS;
                    if (i < len) hist[i] += v[r];
                }
                __syncthreads();
            }
        } else {
            for (int ln = threadIdx.x; ln < lines; ln += blockDim.x) {
                int base;
                if (d == 0) base = ln * nc[0];
                else if (d == 1) base = (ln % nc[0]) + (ln / nc[0]) * nc[0] * nc[1];
                else base = ln;
                unsigned acc_v = 0;
                for (int i = 0; i < len; ++i) {
                    acc_v += hist[base + i * step];
                    hist[base + i * step] = acc_v;
                }
            }
            __syncthreads();
        }
    }
    // candidate boxes on the coarse lattice
    int wc[3], np[3];
    for (int d = 0; d < 3; ++d) {
        wc[d] = d < D ? max(1, P.e[d] / P.cs[d]) : 1;
        np[d] = nc[d] - wc[d] + 1;
    }
    auto sat = [&](int i0, int i1, int i2) -> long long {
        if (i0 < 0 || i1 < 0 || i2 < 0) return 0;
        return hist[i0 + nc[0] * (i1 + nc[1] * i2)];
    };
    unsigned long long mybest = 0;  // (count << 32) | (0xffffffff - candidate): ties -> lowest index
    int ncand = np[0] * np[1] * np[2];
    for (int c = threadIdx.x; c < ncand; c += blockDim.x) {
        int o0 = c % np[0], o1 = (c / np[0]) % np[1], o2 = c / (np[0] * np[1]);
        int a0 = o0 - 1, a1 = o1 - 1, a2 = o2 - 1;
        int b0 = o0 + wc[0] - 1, b1 = o1 + wc[1] - 1, b2 = o2 + wc[2] - 1;
        long long v = sat(b0, b1, b2) - sat(a0, b1, b2) - sat(b0, a1, b2) - sat(b0, b1, a2) + sat(a0, a1, b2) +
                      sat(a0, b1, a2) + sat(b0, a1, a2) - sat(a0, a1, a2);
        unsigned long long key = ((unsigned long long)v << 32) | (0xffffffffull - (unsigned)c);
        mybest = key > mybest ? key : mybest;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long w = __shfl_xor_sync(0xffffffffu, mybest, o);
        mybest = w > mybest ? w : mybest;
    }
    if ((threadIdx.x & 31) == 0) best[threadIdx.x >> 5] = mybest;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long b = 0;
        for (int i = 0; i < WIN_THREADS / 32; ++i) b = best[i] > b ? best[i] : b;
        int c = (int)(0xffffffffull - (b & 0xffffffffull));
        int o[3] = {c % np[0], (c / np[0]) % np[1], c / (np[0] * np[1])};
        for (int d = 0; d < 3; ++d) {
            int org = o[d] * P.cs[d];
            if (org + P.e[d] > G.res[d]) org = G.res[d] - P.e[d];
            acc.window[d] = org;
            acc.window[3 + d] = P.e[d];
        }
    }
}

cudaError_t launch_window(const Geom &g, const Inputs &in, const Accum &acc, int wcap, cudaStream_t s) {
    k_window_sample<<<WIN_SAMPLE_CTAS, WIN_SAMPLE_THREADS, 0, s>>>(g, in, acc, wcap);
    k_window_pick<<<1, WIN_THREADS, 0, s>>>(g, acc, wcap);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- bin [a4 + a5]
// Shared-memory window layout (per CTA, W bins):
//   s_mm  [nmm][W]  ulonglong2 {enc(min), ~enc(max)}   u64 min via CAS, filtered
//   s_fx  [nsum][3][W] u32  96-bit fixed-point sum (lo, mid, hi words)
//   s_cnt [W]       u32 count
// On sm_100a the only native shared-memory atomics are 32-bit integer ones
// (ATOMS.ADD/MIN; f32/f64/u64 adds are ATOMS.CAST.SPIN loops that cost ~2 L1
// wavefronts per lane -- measured, profiles/r01_kbin_ncu_v1.txt).  The sum is
// therefore kept as an exact 96-bit integer of q' = round(v * 2^F) + 2^54,
// added with native u32 atomics and explicit carry propagation:
//   old = atomicAdd(lo, q'_lo); carry = old + q'_lo wrapped;
//   old = atomicAdd(mid, q'_mid + carry); if wrapped: atomicAdd(hi, 1)
// F is per attribute: values below 2^E_hi (E_hi = sampled max exponent + 3)
// and at least 2^(E_hi-9) (or exactly 0) take this path, so each value's
// quantisation error is <= 2^-46 |v|; any other value is added to the global
// f64 sum with a native L2 reduction instead.  At the flush the exact integer
// is converted to f64 once.
int window_bytes_per_bin(const Accum &acc) { return 4 + 12 * acc.nsum + 16 * acc.nmm; }

constexpr long long FX_OFFSET = 1ll << 54;  // makes every q' positive: q in (-2^54, 2^54)

template <int D, int A>
struct BinCtx {
    DGeom G;
    int wo[3], we[3];
    uint32_t W;
    ulonglong2 *s_mm;
    uint32_t *s_fx;
    unsigned *s_cnt;
    unsigned long long *count;
    double *sum;
    ulonglong2 *mm;
    uint64_t nbins;
    uint32_t sum_mask, mm_mask;
    double fx_scale[A > 0 ? A : 1];   // 2^F per attribute slot
    unsigned fx_lo[A > 0 ? A : 1];    // biased-exponent range [fx_lo, fx_hi) takes the fixed path
    unsigned fx_hi[A > 0 ? A : 1];
};

template <int D, int A>
__device__ __forceinline__ void accumulate_row(const BinCtx<D, A> &c, const double (&x)[D],
                                               const double (&v)[A > 0 ? A : 1], uint32_t &n_in) {
    int k[D];
    if (!bin_coords<D>(c.G, x, k)) return;
    ++n_in;
    bool inw = true;
    uint32_t l = 0, lm = 1;
#pragma unroll
    for (int d = 0; d < D; ++d) {
        unsigned r = (unsigned)(k[d] - c.wo[d]);
        inw = inw && (r < (unsigned)c.we[d]);
        l += r * lm;
        lm *= (unsigned)c.we[d];
    }
    uint64_t b = (uint64_t)k[0];
    if (D >= 2) b += (uint64_t)c.G.res[0] * (uint64_t)k[1];
    if (D >= 3) b += (uint64_t)c.G.res[0] * (uint64_t)c.G.res[1] * (uint64_t)k[2];
    if (inw) {
        atomicAdd(&c.s_cnt[l], 1u);
#pragma unroll
        for (int a = 0; a < A; ++a) {
            if ((c.sum_mask >> a) & 1u) {
                int slot = __popc(c.sum_mask & ((1u << a) - 1u));
                unsigned eb = ((unsigned)__double2hiint(v[a]) >> 20) & 0x7ffu;
                if ((eb >= c.fx_lo[a] && eb < c.fx_hi[a]) || v[a] == 0.0) {
                    long long q = __double2ll_rn(__dmul_rn(v[a], c.fx_scale[a])) + FX_OFFSET;
                    unsigned qlo = (unsigned)q, qmid = (unsigned)((unsigned long long)q >> 32);
                    uint32_t *w = c.s_fx + (size_t)slot * 3 * c.W + l;
                    unsigned old = atomicAdd(w, qlo);
                    qmid += (old + qlo < old) ? 1u : 0u;
                    unsigned old2 = atomicAdd(w + c.W, qmid);
                    if (old2 + qmid < old2) atomicAdd(w + 2 * c.W, 1u);
                } else {
                    // rare: outside the fixed range -> native f64 L2 reduction; the row still
                    // contributes the 2^54 offset so the flush can subtract count * 2^54
                    atomicAdd(&c.sum[(uint64_t)slot * c.nbins + b], v[a]);
                    uint32_t *w = c.s_fx + (size_t)slot * 3 * c.W + l;
                    const unsigned om = (unsigned)(FX_OFFSET >> 32);
                    unsigned old2 = atomicAdd(w + c.W, om);
                    if (old2 + om < old2) atomicAdd(w + 2 * c.W, 1u);
                }
            }
            if ((c.mm_mask >> a) & 1u) {
                int slot = __popc(c.mm_mask & ((1u << a) - 1u));
                ulonglong2 *p = &c.s_mm[(uint32_t)slot * c.W + l];
                unsigned long long e = enc_total(v[a]);
                ulonglong2 cur = lds_volatile_u64x2(p);  // monotone filter: stale is safe
                if (e < cur.x) atomicMin(&p->x, e);
                if (~e < cur.y) atomicMin(&p->y, ~e);
            }
        }
    } else {
        atomicAdd(&c.count[b], 1ull);
#pragma unroll
        for (int a = 0; a < A; ++a) {
            if ((c.sum_mask >> a) & 1u) {
                int slot = __popc(c.sum_mask & ((1u << a) - 1u));
                atomicAdd(&c.sum[(uint64_t)slot * c.nbins + b], v[a]);
            }
            if ((c.mm_mask >> a) & 1u) {
                int slot = __popc(c.mm_mask & ((1u << a) - 1u));
                ulonglong2 *p = &c.mm[(uint64_t)slot * c.nbins + b];
                unsigned long long e = enc_total(v[a]);
                ulonglong2 cur = __ldcg(p);
                if (e < cur.x) atomicMin(&p->x, e);
                if (~e < cur.y) atomicMin(&p->y, ~e);
            }
        }
    }
}

// Exact 96-bit fixed-point window sum -> f64 (one rounding when |q| < 2^63).
__device__ __forceinline__ double fx_to_double(uint32_t lo, uint32_t mid, uint32_t hi, unsigned cnt, double inv_scale) {
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

template <int A>
struct BinThreads { static constexpr int value = A <= 1 ? 1024 : 512; };

template <int D, int A, bool VEC>
__global__ void __launch_bounds__(BinThreads<A>::value, 1)
    k_bin(Geom g, Inputs in, Accum acc, int64_t head) {
    extern __shared__ __align__(16) unsigned char smem[];
    BinCtx<D, A> c;
    c.G = load_geom(g, acc.bounds);
    if (!c.G.ok) return;  // degenerate auto bounds: finalize reports it
    c.W = 1;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        c.wo[d] = d < D ? acc.window[d] : 0;
        c.we[d] = d < D ? acc.window[3 + d] : 1;
        c.W *= (uint32_t)c.we[d];
    }
    c.s_mm = (ulonglong2 *)smem;
    c.s_fx = (uint32_t *)(c.s_mm + (size_t)acc.nmm * c.W);
    c.s_cnt = c.s_fx + (size_t)acc.nsum * 3 * c.W;
    c.count = acc.count;
    c.sum = acc.sum;
    c.mm = (ulonglong2 *)acc.mm;
    c.nbins = acc.nbins;
    c.sum_mask = acc.sum_mask;
    c.mm_mask = acc.mm_mask;
    double inv_scale[A > 0 ? A : 1];
#pragma unroll
    for (int a = 0; a < A; ++a) {
        // E_hi = sampled max exponent + 3 (biased); F = 54 - E_hi (unbiased)
        int eb_hi = (int)acc.fxexp[a] + 3;
        if (acc.fxexp[a] == 0) eb_hi = 1023 + 1;  // nothing sampled: assume |v| < 2
        int F = 54 - (eb_hi - 1023);
        bool usable = F > -900 && F < 900;
        c.fx_hi[a] = usable ? (unsigned)eb_hi : 0u;
        c.fx_lo[a] = usable ? (unsigned)max(eb_hi - 9, 1) : 1u;
        c.fx_scale[a] = usable ? ldexp(1.0, F) : 0.0;
        inv_scale[a] = usable ? ldexp(1.0, -F) : 0.0;
    }
    const uint32_t load_mask = acc.load_mask;

    for (uint32_t i = threadIdx.x; i < (uint32_t)acc.nmm * c.W; i += blockDim.x)
        c.s_mm[i] = make_ulonglong2(~0ull, ~0ull);
    for (uint32_t i = threadIdx.x; i < (uint32_t)acc.nsum * 3 * c.W + c.W; i += blockDim.x) c.s_fx[i] = 0u;
    __syncthreads();

    uint32_t n_in = 0;
    const int64_t n = in.n;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    constexpr int AA = A > 0 ? A : 1;
    if (VEC) {
        // rows [head, head + 2*npairs) as 16-byte pairs; all columns share the
        // alignment.  Rolling prefetch: the next pair's loads are in flight while
        // the current pair is accumulated, so HBM latency overlaps the atomics.
        const int64_t npairs = (n - head) / 2;
        double2 cx[D], cv[AA];
        auto load_pair = [&](int64_t q, double2 (&xx)[D], double2 (&vv)[AA]) {
#pragma unroll
            for (int d = 0; d < D; ++d) xx[d] = __ldcs((const double2 *)(in.ax[d] + head) + q);
#pragma unroll
            for (int a = 0; a < A; ++a)
                vv[a] = ((load_mask >> a) & 1u) ? __ldcs((const double2 *)(in.at[a] + head) + q) : make_double2(0.0, 0.0);
        };
        if (tid < npairs) load_pair(tid, cx, cv);
        for (int64_t p = tid; p < npairs; p += nthr) {
            double2 nx[D], nv[AA];
            const int64_t pn = p + nthr;
            if (pn < npairs) load_pair(pn, nx, nv);
            double x[D], v[AA];
#pragma unroll
            for (int d = 0; d < D; ++d) x[d] = cx[d].x;
#pragma unroll
            for (int a = 0; a < A; ++a) v[a] = cv[a].x;
            accumulate_row<D, A>(c, x, v, n_in);
#pragma unroll
            for (int d = 0; d < D; ++d) x[d] = cx[d].y;
#pragma unroll
            for (int a = 0; a < A; ++a) v[a] = cv[a].y;
            accumulate_row<D, A>(c, x, v, n_in);
#pragma unroll
            for (int d = 0; d < D; ++d) cx[d] = nx[d];
#pragma unroll
            for (int a = 0; a < A; ++a) cv[a] = nv[a];
        }
        // the unpaired head row and tail row
        if (tid == 0 || tid == 1) {
            int64_t r = tid == 0 ? (head == 1 ? 0 : -1) : (((n - head) & 1) ? n - 1 : -1);
            if (r >= 0) {
                double x[D], v[AA];
#pragma unroll
                for (int d = 0; d < D; ++d) x[d] = in.ax[d][r];
#pragma unroll
                for (int a = 0; a < A; ++a) v[a] = ((load_mask >> a) & 1u) ? in.at[a][r] : 0.0;
                accumulate_row<D, A>(c, x, v, n_in);
            }
        }
    } else {
        for (int64_t r = tid; r < n; r += nthr) {
            double x[D], v[AA];
#pragma unroll
            for (int d = 0; d < D; ++d) x[d] = __ldcs(in.ax[d] + r);
#pragma unroll
            for (int a = 0; a < A; ++a) v[a] = ((load_mask >> a) & 1u) ? __ldcs(in.at[a] + r) : 0.0;
            accumulate_row<D, A>(c, x, v, n_in);
        }
    }

    // rows inside / outside: one reduction per warp
    uint32_t rows_mine = 0;
    if (VEC) {
        const int64_t npairs = (n - head) / 2;
        int64_t cnt = tid < npairs ? (npairs - 1 - tid) / nthr + 1 : 0;
        rows_mine = (uint32_t)(2 * cnt);
        if (tid == 0 && head == 1) rows_mine += 1;
        if (tid == 1 && ((n - head) & 1)) rows_mine += 1;
    } else {
        rows_mine = tid < n ? (uint32_t)((n - 1 - tid) / nthr + 1) : 0u;
    }
    unsigned long long in_w = n_in, out_w = rows_mine - n_in;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        in_w += __shfl_xor_sync(0xffffffffu, in_w, o);
        out_w += __shfl_xor_sync(0xffffffffu, out_w, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (in_w) atomicAdd(&acc.count[acc.nbins], in_w);
        if (out_w) atomicAdd(&acc.count[acc.nbins + 1], out_w);
    }
    __syncthreads();

    // flush the window into the global accumulator (L2 reductions)
    for (uint32_t l = threadIdx.x; l < c.W; l += blockDim.x) {
        unsigned cnt = c.s_cnt[l];
        if (cnt == 0) continue;
        uint32_t rem = l;
        uint64_t b = 0, mul = 1;
#pragma unroll
        for (int d = 0; d < D; ++d) {
            uint32_t kd = rem % (uint32_t)c.we[d] + (uint32_t)c.wo[d];
            rem /= (uint32_t)c.we[d];
            b += (uint64_t)kd * mul;
            mul *= (uint64_t)c.G.res[d];
        }
        atomicAdd(&c.count[b], (unsigned long long)cnt);
#pragma unroll
        for (int a = 0; a < A; ++a) {
            if ((c.sum_mask >> a) & 1u) {
                int s = __popc(c.sum_mask & ((1u << a) - 1u));
                const uint32_t *w = c.s_fx + (size_t)s * 3 * c.W + l;
                if (w[0] | w[c.W] | w[2 * c.W]) {
                    double d = fx_to_double(w[0], w[c.W], w[2 * c.W], cnt, inv_scale[a]);
                    atomicAdd(&c.sum[(uint64_t)s * c.nbins + b], d);
                }
            }
        }
        for (int s = 0; s < acc.nmm; ++s) {
            ulonglong2 m = c.s_mm[(uint32_t)s * c.W + l];
            ulonglong2 *p = &c.mm[(uint64_t)s * c.nbins + b];
            if (m.x != ~0ull) atomicMin(&p->x, m.x);
            if (m.y != ~0ull) atomicMin(&p->y, m.y);
        }
    }
}

template <int D, int A>
static cudaError_t launch_bin_da(const Geom &g, const Inputs &in, const Accum &acc, const LaunchCfg &lc,
                                 int smem, cudaStream_t s) {
    // 16-byte vector path when every column has the same 16-byte phase
    uintptr_t ph = (uintptr_t)in.ax[0] & 15u;
    bool vec = (ph % 8) == 0;
    for (int d = 0; d < g.ndim; ++d) vec = vec && (((uintptr_t)in.ax[d] & 15u) == ph);
    for (int a = 0; a < in.nattr; ++a)
        if ((acc.load_mask >> a) & 1u) vec = vec && (((uintptr_t)in.at[a] & 15u) == ph);
    int64_t head = ph ? 1 : 0;
    if (in.n < 2 + head) vec = false;
    constexpr int T = BinThreads<A>::value;
    int blocks = lc.sms;  // one persistent CTA per SM (the whole SM's shared memory holds the window)
    int64_t maxb = (in.n + T - 1) / T;
    if (maxb < blocks) blocks = (int)(maxb > 0 ? maxb : 1);
    if (vec) {
        auto kern = k_bin<D, A, true>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        kern<<<blocks, T, smem, s>>>(g, in, acc, head);
    } else {
        auto kern = k_bin<D, A, false>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        kern<<<blocks, T, smem, s>>>(g, in, acc, 0);
    }
    return cudaGetLastError();
}

template <int D>
static cudaError_t launch_bin_d(const Geom &g, const Inputs &in, const Accum &acc, const LaunchCfg &lc, int smem,
                                cudaStream_t s) {
    int na = in.nattr;
    if (na == 0) return launch_bin_da<D, 0>(g, in, acc, lc, smem, s);
    if (na == 1) return launch_bin_da<D, 1>(g, in, acc, lc, smem, s);
    if (na <= 4) return launch_bin_da<D, 4>(g, in, acc, lc, smem, s);
    return launch_bin_da<D, 16>(g, in, acc, lc, smem, s);
}

cudaError_t launch_bin(const Geom &g, const Inputs &in, const Accum &acc, const LaunchCfg &lc, int wcap,
                       int smem_bytes, cudaStream_t s) {
    (void)wcap;
    if (in.n == 0) return cudaSuccess;
    switch (g.ndim) {
    case 1: return launch_bin_d<1>(g, in, acc, lc, smem_bytes, s);
    case 2: return launch_bin_d<2>(g, in, acc, lc, smem_bytes, s);
    default: return launch_bin_d<3>(g, in, acc, lc, smem_bytes, s);
    }
}

// ---------------------------------------------------------------- finalize [a7]
__global__ void k_finalize(Geom g, Accum acc, Meta *meta, int variant) {
    DGeom G = load_geom(g, acc.bounds);
    const uint64_t nb = acc.nbins;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (G.ok) {
        for (int64_t b = t0; b < (int64_t)nb; b += stride) {
            unsigned long long cnt = acc.count[b];
            double dc = (double)cnt;
            for (int s = 0; s < acc.nsum; ++s) {
                double sm = acc.sum[(uint64_t)s * nb + b];
                acc.oavg[(uint64_t)s * nb + b] = cnt ? __ddiv_rn(sm, dc) : __longlong_as_double(0x7ff8000000000000ll);
            }
            for (int s = 0; s < acc.nmm; ++s) {
                ulonglong2 m = ((const ulonglong2 *)acc.mm)[(uint64_t)s * nb + b];
                acc.omin[(uint64_t)s * nb + b] = cnt ? dec_total(m.x) : __longlong_as_double(0x7ff0000000000000ll);
                acc.omax[(uint64_t)s * nb + b] = cnt ? dec_total(~m.y) : __longlong_as_double((long long)0xfff0000000000000ull);
            }
        }
    }
    if (t0 == 0) {
        meta->status = G.ok ? 0 : BIN_EDEGENERATE;
        meta->variant = variant;
        meta->n_in = acc.count[nb];
        meta->n_out = acc.count[nb + 1];
        for (int d = 0; d < 3; ++d) {
            meta->lo[d] = G.lo[d];
            meta->hi[d] = G.hi[d];
            meta->window[d] = acc.window[d];
            meta->window[3 + d] = acc.window[3 + d];
        }
        __threadfence_system();
        meta->done = 1;
    }
}

cudaError_t launch_finalize(const Geom &g, const Accum &acc, Meta *meta_dev, int64_t n_rows_local, int variant,
                            cudaStream_t s) {
    (void)n_rows_local;
    int64_t blocks = ((int64_t)acc.nbins + 255) / 256;
    if (blocks < 1) blocks = 1;
    if (blocks > 148 * 8) blocks = 148 * 8;
    k_finalize<<<(unsigned)blocks, 256, 0, s>>>(g, acc, meta_dev, variant);
    return cudaGetLastError();
}

}  // namespace db
