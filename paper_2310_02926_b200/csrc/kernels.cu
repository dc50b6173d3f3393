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
#include "dev_common.cuh"

namespace db {
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
            int kd = min(floor_nonneg(__dmul_rn(__dsub_rn(x[k][d], G.lo[d]), G.scale[d])), G.res[d] - 1);
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
