// multi.cu -- fused multi-operator binning.
//
// The paper's in situ step runs the DataBin operator on 10 variables over 9
// coordinate systems, "each coordinate system ... in a separate data binning
// operator instance" one after another.  Here K instances
// share one column list and run as ONE launch sequence:
//
//   k_multi_init      identities of all K accumulators (grid.y = instance)   [a3]
//   k_multi_bounds    min/max of every auto-bounded axis column, once per
//                     column, scattered into each instance's bounds         [a2]
//   k_multi_bin       one pass over the rows per L2-sized group of instances
//                     (usually one group): each row's used columns are read
//                     once per pass (staged in shared memory), then every
//                     instance of the group bins it (index a4, reductions a5 as
//                     native L2 reductions: RED.ADD.64 count, RED.ADD.F64 sum,
//                     REDG.MIN.64 on {enc(min), ~enc(max)})
//   k_multi_finalize  avg, decode, sentinels, meta for all K (grid.y)        [a7]
//
// The per-instance arithmetic is the single-instance definition (kernels.cu
// header; readings R1-R17): the same floor/clamp index, the same u64
// totalOrder encoding for min/max, the same finalize body (tail.cuh).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "db_internal.h"
#include "dev_common.cuh"
#include "tail.cuh"
#include "xsum.cuh"

#ifndef MULTI_LD
#define MULTI_LD __ldcg
#endif

namespace db {

constexpr int MULTI_THREADS = 256;
constexpr int MULTI_INIT_THREADS = 512;

// ---------------------------------------------------------------- init [a3]
__global__ void __launch_bounds__(MULTI_INIT_THREADS) k_multi_init(MultiArgs a) {
    const MultiOp &o = a.ops[blockIdx.y];
    const Accum acc = o.acc;
    const uint64_t nb = acc.nbins;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t i = t0; i < (int64_t)nb + 2; i += stride) acc.count[i] = 0ull;
    for (int64_t i = t0; i < (int64_t)(nb * acc.nsum); i += stride) acc.sum[i] = 0.0;
    const ulonglong2 ident = make_ulonglong2(~0ull, ~0ull);
    for (int64_t i = t0; i < (int64_t)(nb * acc.nmm); i += stride) ((ulonglong2 *)acc.mm)[i] = ident;
    if (t0 < 2 * o.g.ndim) acc.bounds[t0] = ~0ull;
    if (o.flt && a.use_flt)
        for (int64_t i = t0; i < (int64_t)(nb * o.nfc * 16); i += stride) o.flt[i] = ~0u;
    if (acc.xs) {  // exact sums: clear the digits of the slot's previous execute (range reset after)
        for (int s = 0; s < acc.nsum; ++s) {
            const int klo = acc.xrange[2 * s], khi = -acc.xrange[2 * s + 1];
            if (klo == XR_EMPTY || klo > khi) continue;
            long long *d = acc.xs + ((uint64_t)s * XD + klo) * nb;
            const int64_t m = (int64_t)(khi - klo + 1) * (int64_t)nb;
            for (int64_t i = t0; i < m; i += stride) d[i] = 0ll;
        }
    }
}

cudaError_t launch_multi_init(const MultiArgs &a, uint64_t max_work, cudaStream_t s) {
    int64_t bx = ((int64_t)(max_work / 2) + MULTI_INIT_THREADS - 1) / MULTI_INIT_THREADS;
    if (bx < 1) bx = 1;
    if (bx > 148 * 4) bx = 148 * 4;
    k_multi_init<<<dim3((unsigned)bx, (unsigned)a.nops), MULTI_INIT_THREADS, 0, s>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- bounds [a2]
// Each bound column's min / ~max (NaN rows skipped, reading R4) is reduced
// once and min-reduced into the bounds words of every auto-bounded instance
// that takes that column as an axis.
__global__ void __launch_bounds__(512) k_multi_bounds(MultiArgs a) {
    unsigned long long mn[MULTI_MAX_COLS], nmx[MULTI_MAX_COLS];
#pragma unroll
    for (int c = 0; c < MULTI_MAX_COLS; ++c) mn[c] = nmx[c] = ~0ull;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
#pragma unroll
        for (int c = 0; c < MULTI_MAX_COLS; ++c) {
            if (!((a.bound_cols >> c) & 1u)) continue;
            const double x = DB_LD_STREAM(a.col[c] + i);
            if (x == x) {
                const unsigned long long e = enc_total(x);
                mn[c] = e < mn[c] ? e : mn[c];
                nmx[c] = ~e < nmx[c] ? ~e : nmx[c];
            }
        }
    }
    __shared__ unsigned long long red[2 * MULTI_MAX_COLS][16];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int c = 0; c < MULTI_MAX_COLS; ++c) {
        if (!((a.bound_cols >> c) & 1u)) continue;
        unsigned long long x = mn[c], y = nmx[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long x2 = __shfl_xor_sync(0xffffffffu, x, o), y2 = __shfl_xor_sync(0xffffffffu, y, o);
            x = x2 < x ? x2 : x;
            y = y2 < y ? y2 : y;
        }
        if (l == 0) {
            red[c][w] = x;
            red[MULTI_MAX_COLS + c][w] = y;
        }
    }
    __syncthreads();
    if (threadIdx.x < 2 * MULTI_MAX_COLS) {
        const int c = threadIdx.x % MULTI_MAX_COLS, hi = threadIdx.x / MULTI_MAX_COLS;
        if (!((a.bound_cols >> c) & 1u)) return;
        unsigned long long v = ~0ull;
        for (int j = 0; j < (int)(blockDim.x >> 5); ++j) v = red[threadIdx.x][j] < v ? red[threadIdx.x][j] : v;
        if (v == ~0ull) return;
        for (int k = 0; k < a.nops; ++k) {
            const MultiOp &o = a.ops[k];
            if (!o.g.bounds_auto) continue;
            for (int d = 0; d < o.g.ndim; ++d)
                if (o.axc[d] == c) atomicMin(&o.acc.bounds[hi ? o.g.ndim + d : d], v);
        }
    }
}

cudaError_t launch_multi_bounds(const MultiArgs &a, const LaunchCfg &lc, cudaStream_t s) {
    if (a.n == 0 || !a.bound_cols) return cudaSuccess;
    int64_t blocks = (a.n + 511) / 512;
    if (blocks > (int64_t)lc.sms * 4) blocks = (int64_t)lc.sms * 4;
    k_multi_bounds<<<(unsigned)blocks, 512, 0, s>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- bin [a4 + a5]
// The accumulator pointers come from the shared-memory instance table, so the
// compiler cannot prove they are global and atomicAdd/atomicMin become generic
// returning ATOMs (one L2 round trip each; measured 2x slower than k_bin's
// global path).  Explicit fire-and-forget global reductions instead:
__device__ __forceinline__ void red_add_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(__cvta_generic_to_global(p)), "l"(v) : "memory");
}
__device__ __forceinline__ void red_add_f64(double *p, double v) {
    asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(__cvta_generic_to_global(p)), "d"(v) : "memory");
}
__device__ __forceinline__ void red_min_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.min.u64 [%0], %1;" ::"l"(__cvta_generic_to_global(p)), "l"(v) : "memory");
}
__device__ __forceinline__ void red_min_u32(uint32_t *p, uint32_t v) {
    asm volatile("red.relaxed.gpu.global.min.u32 [%0], %1;" ::"l"(__cvta_generic_to_global(p)), "r"(v) : "memory");
}
// 32 bytes of filter words in one L2 request (LDG.256, sm_100)
__device__ __forceinline__ void ld_flt8(const uint32_t *p, uint32_t (&f)[8]) {
    asm volatile("ld.relaxed.gpu.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(f[0]), "=r"(f[1]), "=r"(f[2]), "=r"(f[3]), "=r"(f[4]), "=r"(f[5]), "=r"(f[6]), "=r"(f[7])
                 : "l"(__cvta_generic_to_global(p)));
}

// Instance table as the hot loop reads it (shared memory, warp-uniform reads).
struct MOpS {
    double lo[3], hi[3], scale[3];
    unsigned long long *count;
    double *sum;
    ulonglong2 *mm;
    uint32_t *flt;     // min/max filter lines (MultiOp::flt)
    long long *xs;     // BIN_SUM_EXACT digit rows (nullptr: fast sums)
    int32_t *xrange;
    uint64_t nbins;
    int32_t res[3];
    int32_t axc[3];
    int32_t atc[BIN_MAX_ATTR];
    int8_t sslot[BIN_MAX_ATTR], mslot[BIN_MAX_ATTR];  // sum / min-max slot of each attribute, -1 none
    uint32_t desc[BIN_MAX_ATTR];  // packed: column | (sslot + 1) << 8 | (mslot + 1) << 16 (one shared load)
    int32_t ndim, nattr, ok, nfc;
};

#ifndef BIN_MULTI_MINB
#define BIN_MULTI_MINB 2
#endif
__global__ void __launch_bounds__(MULTI_THREADS, BIN_MULTI_MINB) k_multi_bin(MultiArgs a) {
    __shared__ MOpS so[MULTI_MAX_OPS];
    __shared__ double sv[MULTI_MAX_COLS][MULTI_THREADS];  // this CTA's rows, one column per line
    __shared__ unsigned s_in[MULTI_MAX_OPS], s_out[MULTI_MAX_OPS];
    __shared__ int s_xr[MULTI_MAX_OPS][2 * BIN_MAX_ATTR];  // exact sums: digits touched per instance
    const int K = a.k1 - a.k0;  // this launch's group of instances
    if (threadIdx.x < K) {
        const MultiOp &o = a.ops[a.k0 + threadIdx.x];
        const DGeom G = load_geom(o.g, o.acc.bounds);
        MOpS &t = so[threadIdx.x];
        for (int d = 0; d < 3; ++d) {
            t.lo[d] = G.lo[d];
            t.hi[d] = G.hi[d];
            t.scale[d] = G.scale[d];
            t.res[d] = G.res[d];
            t.axc[d] = o.axc[d];
        }
        for (int j = 0; j < BIN_MAX_ATTR; ++j) t.atc[j] = o.atc[j];
        t.count = o.acc.count;
        t.sum = o.acc.sum;
        t.mm = (ulonglong2 *)o.acc.mm;
        t.flt = o.flt;
        t.nfc = o.nfc;
        t.xs = o.acc.xs;
        t.xrange = o.acc.xrange;
        t.nbins = o.acc.nbins;
        t.ndim = o.g.ndim;
        t.nattr = o.nattr;
        t.ok = G.ok ? 1 : 0;  // degenerate auto bounds: nothing is binned, finalize reports it
        for (int j = 0, ss = 0, ms = 0; j < BIN_MAX_ATTR; ++j) {
            const bool in = j < o.nattr;
            t.sslot[j] = (int8_t)(in && ((o.acc.sum_mask >> j) & 1u) ? ss++ : -1);
            t.mslot[j] = (int8_t)(in && ((o.acc.mm_mask >> j) & 1u) ? ms++ : -1);
            t.desc[j] = (uint32_t)(o.atc[j] & 0xff) | ((uint32_t)(t.sslot[j] + 1) << 8) | ((uint32_t)(t.mslot[j] + 1) << 16);
        }
        s_in[threadIdx.x] = 0u;
        s_out[threadIdx.x] = 0u;
    }
    for (int i = threadIdx.x; i < MULTI_MAX_OPS * 2 * BIN_MAX_ATTR; i += MULTI_THREADS) (&s_xr[0][0])[i] = XR_EMPTY;
    __syncthreads();
    const unsigned lane = threadIdx.x & 31u;
    const int64_t stride = (int64_t)gridDim.x * MULTI_THREADS;
    for (int64_t base = (int64_t)blockIdx.x * MULTI_THREADS; base < a.n; base += stride) {
        const int64_t i = base + threadIdx.x;
        const bool valid = i < a.n;
        // each used column of this row read once from HBM (only this thread reads its line)
#pragma unroll
        for (int c = 0; c < MULTI_MAX_COLS; ++c)
            if ((a.used_cols >> c) & 1u) sv[c][threadIdx.x] = valid ? MULTI_LD(a.col[c] + i) : 0.0;
        for (int k = blockIdx.y; k < K; k += gridDim.y) {  // (grid.y > 1: instances spread over CTAs, few rows)
            const MOpS &o = so[k];
            if (!o.ok) continue;
            bool in = valid;
            uint32_t b = 0, mul = 1;
            for (int d = 0; d < o.ndim; ++d) {
                const double x = sv[o.axc[d]][threadIdx.x];
                in = in && (o.lo[d] <= x) && (x <= o.hi[d]);
                const int kd = min(floor_nonneg(__dmul_rn(__dsub_rn(x, o.lo[d]), o.scale[d])), o.res[d] - 1);
                b += (uint32_t)kd * mul;
                mul *= (uint32_t)o.res[d];
            }
            const unsigned bi = __ballot_sync(0xffffffffu, in), bo = __ballot_sync(0xffffffffu, valid && !in);
            if (lane == 0) {
                if (bi) atomicAdd(&s_in[k], (unsigned)__popc(bi));
                if (bo) atomicAdd(&s_out[k], (unsigned)__popc(bo));
            }
            if (!in) continue;
            DB_CHECK(b < o.nbins);
            red_add_u64(&o.count[b], 1ull);
            const uint64_t B = o.nbins;
            // attributes in chunks of 8.  Min/max: a filter line per bin and chunk
            // holds hi32(enc(min)) and hi32(~enc(max)) of every attribute (64 B,
            // two LDG.256 = two L2 requests instead of one 16-B slot load per
            // attribute); it is loaded first, the count / sum reductions are
            // fired while the load is in flight, and a min or max reduction (plus
            // the filter word's) is sent only when the row's hi32 is <= the loaded
            // word.  Slots and filter words only decrease and a word is the hi32
            // of a value already sent to its slot, so a skipped row's value is >
            // a value the slot will hold: skipping never loses the extremum.
            // Launches with MultiArgs::use_flt = 0 send every min/max reduction.
            // (each attribute's value and descriptor read from shared memory once)
            ulonglong2 *const mmb = o.mm;
            double *const sumb = o.sum;
            long long *const xsb = o.xs;
            const int na = o.nattr;
            for (int j0 = 0; j0 < na; j0 += 8) {
                uint32_t f[16];
                double v[8];
                uint32_t ds[8];
                uint32_t *const fl = o.flt && a.use_flt ? o.flt + ((uint64_t)b * o.nfc + (j0 >> 3)) * 16 : nullptr;
#pragma unroll
                for (int u = 0; u < 16; ++u) f[u] = ~0u;
                if (fl) {
                    ld_flt8(fl, *reinterpret_cast<uint32_t(*)[8]>(&f[0]));
                    if (na - j0 > 4) ld_flt8(fl + 8, *reinterpret_cast<uint32_t(*)[8]>(&f[8]));
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int j = j0 + u;
                    ds[u] = j < na ? o.desc[j] : 0u;
                    v[u] = j < na ? sv[ds[u] & 0xffu][threadIdx.x] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t sl = (ds[u] >> 8) & 0xffu;
                    if (!sl) continue;
                    if (xsb) xsum_add_double(xsb, B, (int)sl - 1, b, v[u], s_xr[k]);
                    else red_add_f64(&sumb[(uint64_t)(sl - 1u) * B + b], v[u]);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t ml = ds[u] >> 16;
                    if (!ml) continue;
                    ulonglong2 *p = mmb + (uint64_t)(ml - 1u) * B + b;
                    const unsigned long long e = enc_total(v[u]);
                    const uint32_t hn = (uint32_t)(e >> 32), hx = ~hn;
                    if (hn <= f[2 * u]) {
                        red_min_u64(&p->x, e);
                        if (fl && hn < f[2 * u]) red_min_u32(fl + 2 * u, hn);
                    }
                    if (hx <= f[2 * u + 1]) {
                        red_min_u64(&p->y, ~e);
                        if (fl && hx < f[2 * u + 1]) red_min_u32(fl + 2 * u + 1, hx);
                    }
                }
            }
        }
    }
    __syncthreads();
    if (threadIdx.x < K) {
        const MOpS &o = so[threadIdx.x];
        if (s_in[threadIdx.x]) red_add_u64(&o.count[o.nbins], (unsigned long long)s_in[threadIdx.x]);
        if (s_out[threadIdx.x]) red_add_u64(&o.count[o.nbins + 1], (unsigned long long)s_out[threadIdx.x]);
    }
    for (int i = threadIdx.x; i < K * 2 * BIN_MAX_ATTR; i += MULTI_THREADS) {  // publish the digit ranges
        const int k = i / (2 * BIN_MAX_ATTR), t = i % (2 * BIN_MAX_ATTR);
        if (so[k].xs && s_xr[k][t] != XR_EMPTY) atomicMin(&so[k].xrange[t], s_xr[k][t]);
    }
}

cudaError_t launch_multi_bin(const MultiArgs &a, const LaunchCfg &lc, cudaStream_t s) {
    if (a.n == 0 || a.k1 <= a.k0) return cudaSuccess;
    int64_t blocks = (a.n + MULTI_THREADS - 1) / MULTI_THREADS;
    static const int per_sm = getenv("DATABIN_MULTI_CTAS_PER_SM") ? atoi(getenv("DATABIN_MULTI_CTAS_PER_SM")) : 4;
    const int64_t cap = (int64_t)lc.sms * per_sm;  // grid-stride CTAs (2 resident per SM at 94 registers)
    if (blocks > cap) blocks = cap;
    // too few rows to fill the machine: the group's instances go to separate
    // CTAs (grid.y), each re-reading its rows' columns (from L2)
    static const int ymax = getenv("DATABIN_MULTI_YMAX") ? atoi(getenv("DATABIN_MULTI_YMAX")) : 32;
    int64_t y = (cap + blocks - 1) / blocks;
    const int K = a.k1 - a.k0;
    if (y > K) y = K;
    if (y > ymax) y = ymax;
    if (y < 1) y = 1;
    k_multi_bin<<<dim3((unsigned)blocks, (unsigned)y), MULTI_THREADS, 0, s>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- finalize [a7]
__global__ void k_multi_finalize(MultiArgs a) {
    const MultiOp &o = a.ops[blockIdx.y];
    const Geom g = o.g;
    const Accum acc = o.acc;
    finalize_body(g, acc, o.meta, 64);
}

cudaError_t launch_multi_finalize(const MultiArgs &a, uint64_t max_bins, cudaStream_t s) {
    int64_t bx = ((int64_t)max_bins + 255) / 256;
    if (bx < 1) bx = 1;
    if (bx > 148 * 4) bx = 148 * 4;
    k_multi_finalize<<<dim3((unsigned)bx, (unsigned)a.nops), 256, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace db
