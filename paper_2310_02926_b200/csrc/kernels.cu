// kernels.cu -- sm_100a kernels of the DataBin hot path.
//
// Phases of one execute:
//   k_init      accumulator identities (reading R5)             [a3]
//   k_bounds    per-axis min/max, order-preserving u64 encoding [a2]
//   k_window    picks the shared-memory "hot window" of bins from a sample
//   k_bin       bin index (a4) + accumulate (a5): CTA-private window in
//               shared memory, global L2 reductions for the rest
//   k_finalize  avg = sum/count, decode min/max, sentinels        [a7]
// The cross-rank combine (a6) is the fused NVLink peer kernel of
// combine_peer.cu by default (NCCL allreduce + k_finalize as the fallback,
// DATABIN_COMBINE=nccl), enqueued by handle.cpp.
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
#include "dev_common.cuh"
#include "xsum.cuh"
#include "tail.cuh"

namespace db {
// ---------------------------------------------------------------- init [a3] + window
// k_prep: accumulator identities (reading R5) in CTAs 1..; with manual bounds
// CTA 0 meanwhile chooses the window.  k_window does the window choice after
// the automatic bounds are known.  The window -- the box of bins each binning
// CTA privatises in shared memory; only speed depends on it -- is the box
// position holding the most of 16,384 strided sample rows (coarse histogram +
// summed-area table).  The sample also records the largest exponent of each
// summed attribute (fixed-point scale, dev_common.cuh fx_param); fxexp is
// cleared by the finalize kernel for the next execute on the slot.
constexpr int WIN_SAMPLES = 16384;
constexpr int PREP_THREADS = 512;
constexpr int WIN_BATCH = 8;  // sample rows per thread in flight

// Best box from the coarse histogram in shared memory -> win[0..5] (origin,
// extent); win[6], win[7] = sampled rows in the box / inside the grid.
__device__ void window_pick(const Geom &g, const DGeom &G, const WinPlan &P, int32_t *win, unsigned *hist,
                            unsigned long long *best) {
    __shared__ int origin[6];
    if (P.skip || P.full) {
        if (threadIdx.x < 3) {
            win[threadIdx.x] = 0;
            win[3 + threadIdx.x] = P.skip ? 0 : G.res[threadIdx.x];
        }
        if (threadIdx.x == 0) {
            win[6] = P.full ? 1 : 0;
            win[7] = 1;
        }
        return;
    }
    switch (g.ndim) {
    case 1: pick_box<1>(P, G.res[0], G.res[1], G.res[2], hist, best, origin); break;
    case 2: pick_box<2>(P, G.res[0], G.res[1], G.res[2], hist, best, origin); break;
    default: pick_box<3>(P, G.res[0], G.res[1], G.res[2], hist, best, origin); break;
    }
    if (threadIdx.x < 3) {
        win[threadIdx.x] = origin[threadIdx.x];
        win[3 + threadIdx.x] = P.e[threadIdx.x];
    }
    if (threadIdx.x == 0) {
        win[6] = origin[4];
        win[7] = origin[5];
    }
}

// One CTA: sample, coarse histogram in shared memory, pick -> win[0..7];
// with `exps` also the sampled exponent maxima -> acc.fxexp.
__device__ __forceinline__ void window_choose(const Geom &g, const Inputs &in, const Accum &acc, int wcap, int32_t *win,
                                              bool exps) {
    __shared__ unsigned hist[WIN_CELLS];
    __shared__ unsigned long long best[PREP_THREADS / 32];
    const DGeom G = load_geom(g, acc.bounds);
    const WinPlan P = window_plan(G, g.ndim, wcap);
    const int D = g.ndim;
    for (int i = threadIdx.x; i < WIN_CELLS; i += blockDim.x) hist[i] = 0u;
    __syncthreads();
    const bool work = !P.skip && in.n > 0;
    const int64_t S = in.n < WIN_SAMPLES ? in.n : WIN_SAMPLES;
    const int64_t stride = work ? in.n / S : 1;
    // largest exponent of each summed attribute over the sample
    for (int a = 0; exps && work && a < in.nattr; ++a) {
        if (!((acc.sum_mask >> a) & 1u)) continue;
        unsigned emax = 0u;
        for (int64_t j0 = threadIdx.x; j0 < S; j0 += (int64_t)blockDim.x * WIN_BATCH) {
            double v[WIN_BATCH];
#pragma unroll
            for (int k = 0; k < WIN_BATCH; ++k) {
                const int64_t j = j0 + (int64_t)k * blockDim.x;
                v[k] = j < S ? __ldcs(in.at[a] + j * stride) : 0.0;
            }
#pragma unroll
            for (int k = 0; k < WIN_BATCH; ++k) {
                const unsigned eb = ((unsigned)__double2hiint(v[k]) >> 20) & 0x7ffu;
                if (eb != 0x7ffu && eb > emax) emax = eb;
            }
        }
        const unsigned m = __reduce_max_sync(0xffffffffu, emax);
        if ((threadIdx.x & 31) == 0 && m) atomicMax(&acc.fxexp[a], m);
    }
    // coarse histogram of the sampled rows
    if (work && !P.full) {
        for (int64_t j0 = threadIdx.x; j0 < S; j0 += (int64_t)blockDim.x * WIN_BATCH) {
            double x[WIN_BATCH][3];
#pragma unroll
            for (int k = 0; k < WIN_BATCH; ++k) {
                const int64_t j = j0 + (int64_t)k * blockDim.x;
#pragma unroll
                for (int d = 0; d < 3; ++d) x[k][d] = (d < D && j < S) ? __ldcs(in.ax[d] + j * stride) : 0.0;
            }
#pragma unroll
            for (int k = 0; k < WIN_BATCH; ++k) {
                const int64_t j = j0 + (int64_t)k * blockDim.x;
                bool inside = j < S;
                int c = 0, mul = 1;
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    if (d >= D) break;
                    inside = inside && (G.lo[d] <= x[k][d]) && (x[k][d] <= G.hi[d]);
                    const int kd = min(floor_nonneg(__dmul_rn(__dsub_rn(x[k][d], G.lo[d]), G.scale[d])), G.res[d] - 1);
                    c += (kd / P.cs[d]) * mul;
                    mul *= P.nc[d];
                }
                if (inside) atomicAdd(&hist[c], 1u);
            }
        }
    }
    __syncthreads();
    window_pick(g, G, P, win, hist, best);
}

// Route probe (handle.cpp): the window a CTA would get for wcap bins, and how
// many of 16,384 sampled rows it would hold -> out[0..7] (device memory).
__global__ void __launch_bounds__(PREP_THREADS) k_probe(Geom g, Inputs in, Accum acc, int wcap, int32_t *out) {
    window_choose(g, in, acc, wcap, out, false);
}

cudaError_t launch_probe(const Geom &g, const Inputs &in, const Accum &acc, int wcap, int32_t *out, cudaStream_t s) {
    k_probe<<<1, PREP_THREADS, 0, s>>>(g, in, acc, wcap, out);
    return cudaGetLastError();
}

__global__ void __launch_bounds__(PREP_THREADS) k_prep(Geom g, Inputs in, Accum acc, int wcap, int choose) {
    if (choose && blockIdx.x == 0) {  // manual bounds: the window needs no other input
        window_choose(g, in, acc, wcap, acc.window, true);
        return;
    }
    const int zb = choose ? (int)blockIdx.x - 1 : (int)blockIdx.x, nzb = choose ? gridDim.x - 1 : gridDim.x;
    const uint64_t nb = acc.nbins;
    const int64_t stride = (int64_t)nzb * blockDim.x;
    const int64_t t0 = (int64_t)zb * blockDim.x + threadIdx.x;
    for (int64_t i = t0; i < (int64_t)nb + 2; i += stride) acc.count[i] = 0ull;
    for (int64_t i = t0; i < (int64_t)(nb * acc.nsum); i += stride) acc.sum[i] = 0.0;
    const ulonglong2 ident = make_ulonglong2(~0ull, ~0ull);
    for (int64_t i = t0; i < (int64_t)(nb * acc.nmm); i += stride) ((ulonglong2 *)acc.mm)[i] = ident;
    if (t0 < 2 * g.ndim) acc.bounds[t0] = ~0ull;
    if (t0 == 0) acc.window[7] = 0;  // k_bin_fast's tail work counter
    if (acc.xs) {  // exact sums: clear the digits the slot's previous execute touched (the
                   // range itself is reset by a stream-ordered memset after this kernel)
        for (int s = 0; s < acc.nsum; ++s) {
            const int klo = acc.xrange[2 * s], khi = -acc.xrange[2 * s + 1];
            if (klo == XR_EMPTY || klo > khi) continue;
            long long *d = acc.xs + ((uint64_t)s * XD + klo) * nb;
            const int64_t m = (int64_t)(khi - klo + 1) * (int64_t)nb;
            for (int64_t i = t0; i < m; i += stride) d[i] = 0ll;
        }
    }
}

__global__ void __launch_bounds__(PREP_THREADS) k_window(Geom g, Inputs in, Accum acc, int wcap) {
    window_choose(g, in, acc, wcap, acc.window, true);
}

cudaError_t launch_init(const Geom &g, const Inputs &in, const Accum &acc, int wcap, bool choose_window,
                        cudaStream_t s) {
    const int64_t work = (int64_t)acc.nbins * (1 + acc.nsum + acc.nmm);
    int64_t blocks = (work / 2 + PREP_THREADS - 1) / PREP_THREADS;
    if (blocks < 16) blocks = 16;
    if (blocks > 148 * 4) blocks = 148 * 4;
    k_prep<<<(unsigned)blocks + (choose_window ? 1 : 0), PREP_THREADS, 0, s>>>(g, in, acc, wcap, choose_window ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_window(const Geom &g, const Inputs &in, const Accum &acc, int wcap, cudaStream_t s) {
    k_window<<<1, PREP_THREADS, 0, s>>>(g, in, acc, wcap);
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
            double x = DB_LD_STREAM(in.ax[d] + i);
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

// ---------------------------------------------------------------- finalize [a7]
// (body in tail.cuh)
__global__ void k_finalize(Geom g, Accum acc, Meta *meta, int variant) { finalize_body(g, acc, meta, variant); }

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
