// bin_general.cu -- the general accumulate kernel k_bin (a4 + a5): any number
// of attributes (0..16), any column alignment, any row count.  The common
// single-attribute, 16-byte-aligned case runs the leaner k_bin_fast
// (bin_fast.cu); both share the window layout and the arithmetic below.
//
// Shared-memory window (per CTA, W bins; word offsets):
//   [0, 2*nmm*W)            u32x2  min/max filter {hi32(enc(min)), hi32(~enc(max))}
//   [.., + 3*nsum*W)        u32    96-bit fixed-point sums (lo, mid, hi words per slot)
//   [.., + W)               u32    count
// On sm_100a the only native shared-memory atomics are 32-bit integer ones
// (ATOMS.ADD/MIN); f32/f64/u64 adds and u64 min are ATOMS.CAST.SPIN CAS loops
// (~2 L1 wavefronts per lane; profiles/r01_kbin_ncu_v1_cas.txt).  Hence:
//  * sums: exact 96-bit integer of q' = round(v*2^F) + 2^62 with native u32
//    atomics and carry propagation from the returned old value
//      old = atomicAdd(lo, q'_lo); carry = (old + q'_lo wrapped)
//      old = atomicAdd(mid, q'_mid + carry); if wrapped: atomicAdd(hi, 1)
//    F per attribute from the sampled max exponent (dev_common.cuh fx_param);
//    values outside the fixed range take a native f64 L2 reduction and add
//    only the offset.  The flush converts the exact integer to f64 once.
//  * min/max: a conservative 32-bit filter per bin (native ATOMS.MIN); rows
//    that may improve it send the exact value to the global u64 min slot with
//    REDG.MIN.64 (values only move one way, so stale filter reads are safe).
//  * rows outside the window: native L2 reductions on the global accumulator.
#include <cuda_runtime.h>
#include <stdint.h>

#include "db_internal.h"
#include "dev_common.cuh"
#include "xsum.cuh"

namespace db {

extern __shared__ __align__(16) uint32_t g_dsm[];

// This file is compiled twice: as itself (BIN_SUM_FAST instances + the
// dispatching launcher) and through bin_general_x.cu with BIN_GENERAL_XS = 1
// (the BIN_SUM_EXACT instances), so the two sets build in parallel.
#ifndef BIN_GENERAL_XS
#define BIN_GENERAL_XS 0
#endif
#if !BIN_GENERAL_XS
int window_bytes_per_bin(const Accum &acc) { return 4 + 12 * acc.nsum + 8 * acc.nmm; }
#endif

struct GenCtx {
    DGeom G;
    WinGeom w;
    uint32_t o_fx, o_cnt;  // word offsets in shared memory (o_mm = 0)
    unsigned long long *count;
    double *sum;
    ulonglong2 *mm;
    uint64_t nbins;
    uint32_t sum_mask, mm_mask;
    long long *xs;  // BIN_SUM_EXACT digit rows (xsum.cuh), nullptr for BIN_SUM_FAST
    int *sxr;       // this CTA's touched digit ranges (shared memory)
};

template <int D>
__device__ __forceinline__ uint64_t global_bin(const GenCtx &c, const int (&k)[D]) {
    uint64_t b = (uint64_t)k[0];
    if (D >= 2) b += (uint64_t)(c.w.resm1[0] + 1) * (uint64_t)k[1];
    if (D >= 3) b += (uint64_t)(c.w.resm1[0] + 1) * (uint64_t)(c.w.resm1[1] + 1) * (uint64_t)k[2];
    return b;
}

template <int D, int A, bool XS>
__device__ __forceinline__ void accumulate_row(const GenCtx &c, const FxParam (&fx)[A > 0 ? A : 1],
                                               const double (&x)[D], const double (&v)[A > 0 ? A : 1],
                                               uint32_t &n_in) {
    bool in = true;
    int k[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
        in = in && (c.G.lo[d] <= x[d]) && (x[d] <= c.G.hi[d]);
        k[d] = min(floor_nonneg(__dmul_rn(__dsub_rn(x[d], c.G.lo[d]), c.G.scale[d])), c.w.resm1[d]);
    }
    if (!in) return;
    ++n_in;
    bool inw = true;
    uint32_t l = 0;
#pragma unroll
    for (int d = D - 1; d >= 0; --d) {
        const unsigned r = (unsigned)(k[d] - c.w.wo[d]);
        inw = inw && (r < c.w.we[d]);
        l = l * c.w.we[d] + r;
    }
    const uint32_t W = c.w.W;
    DB_CHECK(!inw || l < W);
#pragma unroll
    for (int d = 0; d < D; ++d) DB_CHECK(k[d] >= 0 && k[d] <= c.w.resm1[d]);
    if (inw) {
        atomicAdd(&g_dsm[c.o_cnt + l], 1u);
#pragma unroll
        for (int a = 0; a < A; ++a) {
            if ((c.sum_mask >> a) & 1u) {
                const uint32_t s = __popc(c.sum_mask & ((1u << a) - 1u));
                const uint32_t w0 = c.o_fx + s * 3 * W + l;
                unsigned qmid;
                unsigned long long q = 0;
                bool fxp;
                if (XS) {
                    fxp = fx_quant_exact(fx[a], v[a], q);
                } else {
                    fxp = fx_path(fx[a], v[a]);
                    if (fxp) q = fx_quant(fx[a], v[a]);
                }
                if (fxp) {
                    const unsigned qlo = (unsigned)q;
                    qmid = (unsigned)(q >> 32);
                    const unsigned old = atomicAdd(&g_dsm[w0], qlo);
                    qmid += (old + qlo < old) ? 1u : 0u;
                } else {  // rare: outside the fixed range -> f64 L2 reduction, offset only here
                    if (XS) xsum_add_double(c.xs, c.nbins, (int)s, global_bin<D>(c, k), v[a], c.sxr);
                    else atomicAdd(&c.sum[(uint64_t)s * c.nbins + global_bin<D>(c, k)], v[a]);
                    qmid = FX_OFFSET_MID;
                }
                const unsigned old2 = atomicAdd(&g_dsm[w0 + W], qmid);
                if (old2 + qmid < old2) atomicAdd(&g_dsm[w0 + 2 * W], 1u);
            }
            if ((c.mm_mask >> a) & 1u) {
                const uint32_t s = __popc(c.mm_mask & ((1u << a) - 1u));
                const uint32_t ra = 2 * (s * W + l);
                const unsigned long long e = enc_total(v[a]);
                const unsigned eh = (unsigned)(e >> 32), neh = ~eh;
                uint2 f;  // one LDS.64; stale values are safe (the words only decrease)
                asm volatile("ld.volatile.shared.v2.u32 {%0, %1}, [%2];" : "=r"(f.x), "=r"(f.y) : "r"((unsigned)__cvta_generic_to_shared(&g_dsm[ra])));
                if (eh <= f.x || neh <= f.y) {
                    ulonglong2 *p = &c.mm[(uint64_t)s * c.nbins + global_bin<D>(c, k)];
                    if (eh <= f.x) {
                        if (eh < f.x) atomicMin(&g_dsm[ra], eh);
                        atomicMin(&p->x, e);
                    }
                    if (neh <= f.y) {
                        if (neh < f.y) atomicMin(&g_dsm[ra + 1], neh);
                        atomicMin(&p->y, ~e);
                    }
                }
            }
        }
    } else {
        const uint64_t b = global_bin<D>(c, k);
        atomicAdd(&c.count[b], 1ull);
#pragma unroll
        for (int a = 0; a < A; ++a) {
            if ((c.sum_mask >> a) & 1u) {
                const uint32_t s = __popc(c.sum_mask & ((1u << a) - 1u));
                if (XS) xsum_add_double(c.xs, c.nbins, (int)s, b, v[a], c.sxr);
                else atomicAdd(&c.sum[(uint64_t)s * c.nbins + b], v[a]);
            }
            if ((c.mm_mask >> a) & 1u) {
                ulonglong2 *p = &c.mm[(uint64_t)__popc(c.mm_mask & ((1u << a) - 1u)) * c.nbins + b];
                const unsigned long long e = enc_total(v[a]);
                atomicMin(&p->x, e);
                atomicMin(&p->y, ~e);
            }
        }
    }
}

template <int A>
struct GenThreads { static constexpr int value = A <= 1 ? 1024 : 512; };

template <int D, int A, bool VEC, bool XS>
__global__ void __launch_bounds__(GenThreads<A>::value, 1)
    k_bin(Geom g, Inputs in, Accum acc, int64_t head) {
    __shared__ int s_xr[2 * BIN_MAX_ATTR];
    if (XS) xr_init(s_xr);
    GenCtx c;
    c.xs = XS ? acc.xs : nullptr;
    c.sxr = s_xr;
    c.G = load_geom<D>(g, acc.bounds);
    if (!c.G.ok) return;  // degenerate auto bounds: finalize reports it
    c.w = load_window(c.G, acc.window, D);
    const uint32_t W = c.w.W;
    c.o_fx = 2u * acc.nmm * W;
    c.o_cnt = c.o_fx + 3u * acc.nsum * W;
    c.count = acc.count;
    c.sum = acc.sum;
    c.mm = (ulonglong2 *)acc.mm;
    c.nbins = acc.nbins;
    c.sum_mask = acc.sum_mask;
    c.mm_mask = acc.mm_mask;
    constexpr int AA = A > 0 ? A : 1;
    FxParam fx[AA];
#pragma unroll
    for (int a = 0; a < A; ++a) fx[a] = XS ? fx_param_exact(acc.fxexp[a]) : fx_param(acc.fxexp[a]);
    const uint32_t load_mask = acc.load_mask;

    for (uint32_t i = threadIdx.x; i < c.o_fx; i += blockDim.x) g_dsm[i] = ~0u;  // filters
    const uint32_t o_end = c.o_cnt + W;
    for (uint32_t i = c.o_fx + threadIdx.x; i < o_end; i += blockDim.x) g_dsm[i] = 0u;
    __syncthreads();

    uint32_t n_in = 0;
    const int64_t n = in.n;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    uint64_t rows_mine = 0;
    auto row = [&](int64_t r) {
        double x[D], v[AA];
#pragma unroll
        for (int d = 0; d < D; ++d) x[d] = DB_LD_STREAM(in.ax[d] + r);
#pragma unroll
        for (int a = 0; a < A; ++a) v[a] = ((load_mask >> a) & 1u) ? DB_LD_STREAM(in.at[a] + r) : 0.0;
        accumulate_row<D, A, XS>(c, fx, x, v, n_in);
        ++rows_mine;
    };
    if (VEC) {
        // rows [head, head + 2*npairs) as 16-byte pairs, one pair prefetched ahead
        const int64_t npairs = (n - head) / 2;
        double2 cx[D], cv[AA];
        auto load_pair = [&](int64_t q, double2 (&xx)[D], double2 (&vv)[AA]) {
#pragma unroll
            for (int d = 0; d < D; ++d) xx[d] = DB_LD_STREAM((const double2 *)(in.ax[d] + head) + q);
#pragma unroll
            for (int a = 0; a < A; ++a)
                vv[a] = ((load_mask >> a) & 1u) ? DB_LD_STREAM((const double2 *)(in.at[a] + head) + q) : make_double2(0.0, 0.0);
        };
        if (tid < npairs) load_pair(tid, cx, cv);
        for (int64_t p = tid; p < npairs; p += nthr) {
            double2 nx[D], nv[AA];
            if (p + nthr < npairs) load_pair(p + nthr, nx, nv);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double x[D], v[AA];
#pragma unroll
                for (int d = 0; d < D; ++d) x[d] = h ? cx[d].y : cx[d].x;
#pragma unroll
                for (int a = 0; a < A; ++a) v[a] = h ? cv[a].y : cv[a].x;
                accumulate_row<D, A, XS>(c, fx, x, v, n_in);
            }
            rows_mine += 2;
#pragma unroll
            for (int d = 0; d < D; ++d) cx[d] = nx[d];
#pragma unroll
            for (int a = 0; a < A; ++a) cv[a] = nv[a];
        }
        if (tid == 0 && head == 1) row(0);                   // unpaired head row
        if (tid == 1 && ((n - head) & 1)) row(n - 1);         // unpaired tail row
    } else {
        for (int64_t r = tid; r < n; r += nthr) row(r);
    }

    // rows inside / outside: one reduction per warp
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
    for (uint32_t l = threadIdx.x; l < W; l += blockDim.x) {
        const unsigned long long cnt = g_dsm[c.o_cnt + l];
        if (cnt == 0) continue;
        uint32_t rem = l;
        uint64_t b = 0, mul = 1;
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const uint32_t kd = rem % c.w.we[d] + (uint32_t)c.w.wo[d];
            rem /= c.w.we[d];
            b += (uint64_t)kd * mul;
            mul *= (uint64_t)c.G.res[d];
        }
        atomicAdd(&c.count[b], cnt);
#pragma unroll
        for (int a = 0; a < A; ++a) {
            if ((c.sum_mask >> a) & 1u) {
                const uint32_t s = __popc(c.sum_mask & ((1u << a) - 1u));
                const uint32_t w0 = c.o_fx + s * 3 * W + l;
                if (XS) {
                    xsum_add_fixed(c.xs, c.nbins, (int)s, b, g_dsm[w0], g_dsm[w0 + W], g_dsm[w0 + 2 * W], cnt,
                                   FX_OFFSET, fx[a].F, s_xr);
                } else {
                    const double d = fx_to_double(g_dsm[w0], g_dsm[w0 + W], g_dsm[w0 + 2 * W], cnt, fx[a].inv_scale);
                    if (d != 0.0) atomicAdd(&c.sum[(uint64_t)s * c.nbins + b], d);
                }
            }
        }
    }
    if (XS) {
        __syncthreads();
        xr_publish(s_xr, acc.nsum, acc.xrange);
    }
}

template <int D, int A>
static cudaError_t launch_general(const Geom &g, const Inputs &in, const Accum &acc, const LaunchCfg &lc, int smem,
                                  cudaStream_t s) {
    // 16-byte vector path when every loaded column has the same 16-byte phase
    uintptr_t ph = (uintptr_t)in.ax[0] & 15u;
    bool vec = (ph % 8) == 0;
    for (int d = 0; d < g.ndim; ++d) vec = vec && (((uintptr_t)in.ax[d] & 15u) == ph);
    for (int a = 0; a < in.nattr; ++a)
        if ((acc.load_mask >> a) & 1u) vec = vec && (((uintptr_t)in.at[a] & 15u) == ph);
    const int64_t head = ph ? 1 : 0;
    if (in.n < 2 + head) vec = false;
    constexpr int T = GenThreads<A>::value;
    int blocks = lc.sms;  // one persistent CTA per SM: the whole shared memory holds the window
    const int64_t maxb = (in.n + T - 1) / T;
    if (maxb < blocks) blocks = (int)(maxb > 0 ? maxb : 1);
    constexpr bool XS = BIN_GENERAL_XS != 0;
    auto kern = vec ? k_bin<D, A, true, XS> : k_bin<D, A, false, XS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<blocks, T, smem, s>>>(g, in, acc, vec ? head : 0);
    return cudaGetLastError();
}

template <int D>
static cudaError_t launch_general_d(const Geom &g, const Inputs &in, const Accum &acc, const LaunchCfg &lc, int smem,
                                    cudaStream_t s) {
    const int na = in.nattr;
    if (na == 0) return launch_general<D, 0>(g, in, acc, lc, smem, s);
    if (na == 1) return launch_general<D, 1>(g, in, acc, lc, smem, s);
    if (na <= 4) return launch_general<D, 4>(g, in, acc, lc, smem, s);
    if (na <= 8) return launch_general<D, 8>(g, in, acc, lc, smem, s);  // (the A = 16 instance spills)
    return launch_general<D, 16>(g, in, acc, lc, smem, s);
}

#if BIN_GENERAL_XS
cudaError_t launch_bin_general_exact(const Geom &g, const Inputs &in, const Accum &acc, const LaunchCfg &lc, int smem,
                                     cudaStream_t s) {
#else
cudaError_t launch_bin_general_exact(const Geom &g, const Inputs &in, const Accum &acc, const LaunchCfg &lc, int smem,
                                     cudaStream_t s);
cudaError_t launch_bin_general(const Geom &g, const Inputs &in, const Accum &acc, const LaunchCfg &lc, int smem,
                               cudaStream_t s) {
    if (acc.xs) return launch_bin_general_exact(g, in, acc, lc, smem, s);
#endif
    switch (g.ndim) {
    case 1: return launch_general_d<1>(g, in, acc, lc, smem, s);
    case 2: return launch_general_d<2>(g, in, acc, lc, smem, s);
    default: return launch_general_d<3>(g, in, acc, lc, smem, s);
    }
}

}  // namespace db
