// det.cu -- deterministic DataBin (bin_spec_t.deterministic = 1).
//
// Atomic accumulation makes fp64 sums depend on update order (PAPER.md:533
// "requires the use of atomic memory updates").  This mode reproduces the
// sequential definition exactly: every bin's sum is folded from +0.0 in
// ascending row order, so results are bit-identical to the oracle (and, with
// nranks > 1, to the oracle's partition mode P = nranks after the
// rank-ordered fold done in handle.cpp).
//
//   k_det_keys      bin index per row (nbins for rows outside the mesh) and
//                   the payload: the attribute value itself when exactly one
//                   attribute is binned (the sort carries it, so the fold
//                   reads it sequentially), else the row index (gathered)
//   radix passes    stable LSD sort of (key, payload) by key, digits of
//                   <= 8 bits (as many bits as B needs, split evenly):
//                   k_rs_hist -> exclusive scan -> k_rs_scatter.  The
//                   scatter ranks each tile of 4096 keys stably without a
//                   block barrier per item: warps rank 32 keys at a time by
//                   ballots over the digit bits against warp-private digit
//                   counters, one block scan turns them into tile offsets,
//                   and the tile is reordered in shared memory so the global
//                   writes go out as contiguous runs per digit
//   k_det_segments  first/last position of every bin in the sorted order
//   k_det_fold      one thread per bin folds its segment in row order
//                   (k_det_fold_long: one warp per bin of > 256 rows)
#include <cuda_runtime.h>
#include <stdint.h>

#include "db_internal.h"
#include "dev_common.cuh"

namespace db {

// payload: VALS ? the value of attribute `va` : the row index (as u32 in the low word)
template <bool VALS>
__global__ void __launch_bounds__(256) k_det_keys(Geom g, Inputs in, Accum acc, uint32_t *keys, void *payload, int va) {
    const DGeom G = load_geom(g, acc.bounds);
    const uint32_t B = (uint32_t)acc.nbins;
    uint32_t n_in = 0, n_seen = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    constexpr int U = 4;  // rows per thread in flight
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < in.n; i0 += U * stride) {
        double x[U][3], v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + u * stride;
#pragma unroll
            for (int d = 0; d < 3; ++d) x[u][d] = (d < g.ndim && i < in.n) ? DB_LD_STREAM(in.ax[d] + i) : 0.0;
            v[u] = (VALS && i < in.n) ? DB_LD_STREAM(in.at[va] + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + u * stride;
            if (i >= in.n) continue;
            bool inside = G.ok;
            uint32_t b = 0, mul = 1;
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                if (d >= g.ndim) break;
                inside = inside && (G.lo[d] <= x[u][d]) && (x[u][d] <= G.hi[d]);
                int kd = min(floor_nonneg(__dmul_rn(__dsub_rn(x[u][d], G.lo[d]), G.scale[d])), G.res[d] - 1);
                b += (uint32_t)kd * mul;
                mul *= (uint32_t)G.res[d];
            }
            keys[i] = inside ? b : B;
            if (VALS) ((double *)payload)[i] = v[u];
            else ((uint32_t *)payload)[i] = (uint32_t)i;
            n_in += inside;
            n_seen++;
        }
    }
    unsigned long long a = n_in, o = n_seen - n_in;
    for (int s = 16; s > 0; s >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, s);
        o += __shfl_xor_sync(0xffffffffu, o, s);
    }
    if ((threadIdx.x & 31) == 0) {
        if (a) atomicAdd(&acc.count[acc.nbins], a);
        if (o) atomicAdd(&acc.count[acc.nbins + 1], o);
    }
}

// ---- stable LSD radix sort, 8-bit digits, striped tiles of 4096 ----
constexpr int RS_THREADS = 256;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;

__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const uint32_t *keys, int64_t n, int shift, uint32_t mask,
                                                        uint32_t *hist, int64_t nblk) {
    constexpr int NW = RS_THREADS / 32;
    __shared__ uint32_t h[NW][256];  // per-warp counters: skewed digits (Plummer core) do not serialise the CTA
    const int w = threadIdx.x >> 5;
    for (int k = 0; k < NW; ++k) h[k][threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
    uint32_t kk[RS_ITEMS];
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) {
        const int64_t i = base + j * RS_THREADS + threadIdx.x;
        kk[j] = i < n ? DB_LD_STREAM(keys + i) : ~0u;
    }
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j)
        if (base + j * RS_THREADS + threadIdx.x < n) atomicAdd(&h[w][(kk[j] >> shift) & mask], 1u);
    __syncthreads();
    uint32_t s = 0;
    for (int k = 0; k < NW; ++k) s += h[k][threadIdx.x];
    hist[(int64_t)threadIdx.x * nblk + blockIdx.x] = s;  // digit-major
}

template <typename P>
__global__ void __launch_bounds__(RS_THREADS, 3) k_rs_scatter(const uint32_t *keys, const P *pay, int64_t n, int shift,
                                                           int dbits, const uint32_t *offs, int64_t nblk,
                                                           uint32_t *keys_out, P *pay_out) {
    constexpr int NW = RS_THREADS / 32;
    __shared__ uint32_t wcnt[NW][256];  // per warp and digit: count, then warp prefix
    __shared__ uint32_t dstart[256];    // tile-local start of each digit
    __shared__ uint32_t goff[256];      // this tile's global offset of each digit
    __shared__ uint32_t wtot[NW];
    extern __shared__ __align__(16) unsigned char rs_dsm[];  // the tile, reordered by digit
    P *spay = (P *)rs_dsm;
    uint32_t *skey = (uint32_t *)(rs_dsm + (size_t)RS_TILE * sizeof(P));
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t mask = (1u << dbits) - 1u;
    for (int k = 0; k < NW; ++k) wcnt[k][threadIdx.x] = 0u;
    goff[threadIdx.x] = offs[(int64_t)threadIdx.x * nblk + blockIdx.x];
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
    const unsigned lt = (1u << lane) - 1u;
    uint32_t key[RS_ITEMS], lr[RS_ITEMS];  // (the payload is read at placement: fewer registers, more CTAs)
    // warp w owns keys [base + w*512, base + (w+1)*512) in 16 rounds of 32: stable order
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        const int64_t i = base + w * (32 * RS_ITEMS) + r * 32 + lane;
        key[r] = i < n ? DB_LD_STREAM(keys + i) : 0u;
    }
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        const int64_t i = base + w * (32 * RS_ITEMS) + r * 32 + lane;
        const bool valid = i < n;
        const uint32_t d = (key[r] >> shift) & mask;
        unsigned peers = __ballot_sync(0xffffffffu, valid);
        for (int b = 0; b < dbits; ++b) {
            const unsigned bb = __ballot_sync(0xffffffffu, (d >> b) & 1u);
            peers &= ((d >> b) & 1u) ? bb : ~bb;
        }
        const uint32_t before = valid ? wcnt[w][d] : 0u;
        const uint32_t rank = __popc(peers & lt);
        __syncwarp();
        if (valid && rank == 0) wcnt[w][d] = before + __popc(peers);
        __syncwarp();
        lr[r] = before + rank;
    }
    __syncthreads();
    {  // thread t = digit t: warp prefixes, tile total, then the exclusive scan over digits
        uint32_t run = 0;
        for (int k = 0; k < NW; ++k) {
            const uint32_t c = wcnt[k][threadIdx.x];
            wcnt[k][threadIdx.x] = run;
            run += c;
        }
        uint32_t inc = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) wtot[w] = inc;
        __syncthreads();
        uint32_t pre = 0;
        for (int k = 0; k < w; ++k) pre += wtot[k];
        dstart[threadIdx.x] = pre + inc - run;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
        const int64_t i = base + w * (32 * RS_ITEMS) + r * 32 + lane;
        if (i >= n) continue;
        const uint32_t d = (key[r] >> shift) & mask;
        const uint32_t idx = dstart[d] + wcnt[w][d] + lr[r];
        DB_CHECK(idx < (uint32_t)RS_TILE);
        skey[idx] = key[r];
        spay[idx] = DB_LD_STREAM(pay + i);
    }
    __syncthreads();
    const int64_t cnt = n - base < RS_TILE ? n - base : RS_TILE;
    for (int64_t i = threadIdx.x; i < cnt; i += RS_THREADS) {  // contiguous runs per digit
        const uint32_t k = skey[i], d = (k >> shift) & mask;
        const uint64_t gp = (uint64_t)goff[d] + (uint64_t)(i - dstart[d]);
        DB_CHECK(gp < (uint64_t)n);
        keys_out[gp] = k;
        pay_out[gp] = spay[i];
    }
}

// ---- exclusive scan of u32 (totals < 2^32) ----
constexpr int SC_THREADS = 1024;
constexpr int SC_ITEMS = 4;
constexpr int SC_TILE = SC_THREADS * SC_ITEMS;

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *total) {
    __shared__ uint32_t ws[SC_THREADS / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t s = lane < SC_THREADS / 32 ? ws[lane] : 0u;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        ws[lane] = s;
    }
    __syncthreads();
    uint32_t pre = (w ? ws[w - 1] : 0u) + x - v;
    *total = ws[SC_THREADS / 32 - 1];
    __syncthreads();
    return pre;
}

__global__ void __launch_bounds__(SC_THREADS) k_scan_reduce(const uint32_t *d, int64_t len, uint32_t *part) {
    int64_t base = (int64_t)blockIdx.x * SC_TILE;
    uint32_t s = 0;
    for (int k = 0; k < SC_ITEMS; ++k) {
        int64_t i = base + (int64_t)threadIdx.x * SC_ITEMS + k;
        if (i < len) s += d[i];
    }
    uint32_t tot;
    block_excl_scan(s, &tot);
    if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(SC_THREADS) k_scan_part(uint32_t *part, int64_t np) {
    uint32_t carry = 0;
    for (int64_t c = 0; c < np; c += SC_THREADS) {
        int64_t i = c + threadIdx.x;
        uint32_t v = i < np ? part[i] : 0u, tot;
        uint32_t pre = block_excl_scan(v, &tot);
        if (i < np) part[i] = carry + pre;
        carry += tot;
    }
}

__global__ void __launch_bounds__(SC_THREADS) k_scan_down(uint32_t *d, int64_t len, const uint32_t *part) {
    int64_t base = (int64_t)blockIdx.x * SC_TILE;
    uint32_t v[SC_ITEMS], s = 0;
    for (int k = 0; k < SC_ITEMS; ++k) {
        int64_t i = base + (int64_t)threadIdx.x * SC_ITEMS + k;
        v[k] = i < len ? d[i] : 0u;
        s += v[k];
    }
    uint32_t tot;
    uint32_t pre = block_excl_scan(s, &tot) + part[blockIdx.x];
    for (int k = 0; k < SC_ITEMS; ++k) {
        int64_t i = base + (int64_t)threadIdx.x * SC_ITEMS + k;
        if (i < len) d[i] = pre;
        pre += v[k];
    }
}

static cudaError_t scan_excl(uint32_t *d, int64_t len, uint32_t *part, cudaStream_t s, int *launches) {
    int64_t np = (len + SC_TILE - 1) / SC_TILE;
    if (np == 0) return cudaSuccess;
    k_scan_reduce<<<(unsigned)np, SC_THREADS, 0, s>>>(d, len, part);
    k_scan_part<<<1, SC_THREADS, 0, s>>>(part, np);
    k_scan_down<<<(unsigned)np, SC_THREADS, 0, s>>>(d, len, part);
    *launches += 3;
    return cudaGetLastError();
}

// ---- segments and the in-order fold ----
__global__ void k_det_clear(uint32_t *seg, uint64_t len) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (uint64_t)gridDim.x * blockDim.x)
        seg[i] = 0u;
}

__global__ void k_det_segments(const uint32_t *keys, int64_t n, uint32_t B, uint32_t *seg_start, uint32_t *seg_end) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
    for (int64_t j0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; j0 < n; j0 += stride) {
        uint32_t k[5];
        if (j0 + 4 <= n && (((uintptr_t)(keys + j0)) & 15u) == 0) {
            const uint4 q = DB_LD_STREAM((const uint4 *)(keys + j0));
            k[0] = q.x, k[1] = q.y, k[2] = q.z, k[3] = q.w;
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) k[u] = j0 + u < n ? keys[j0 + u] : ~0u;
        }
        k[4] = j0 + 4 < n ? keys[j0 + 4] : ~0u;
        uint32_t prev = j0 > 0 ? keys[j0 - 1] : ~0u;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t j = j0 + u;
            if (j >= n) break;
            if (k[u] < B) {
                if (prev != k[u]) seg_start[k[u]] = (uint32_t)j;
                if (k[u + 1] != k[u]) seg_end[k[u]] = (uint32_t)(j + 1);
            }
            prev = k[u];
        }
    }
}

// The fold of a bin is a chain of dependent adds in row order (the stable
// sort keeps row order within a bin), so its length -- not bandwidth -- is
// the critical path: the hottest C3 bin holds ~1.2e5 rows.
//   k_det_fold        one thread per bin with <= DET_LONG rows
//   k_det_fold_long   one warp per longer bin: lanes load a step of rows
//                     (256 rows, coalesced, one step ahead) into shared memory and do
//                     min/max; lane 0 runs the add chain from shared memory
// VALS: payload = the values of the one binned attribute in sorted order;
// else row indices into the attribute columns.
constexpr uint32_t DET_LONG = 256;

template <bool VALS>
__device__ __forceinline__ double det_val(const Inputs &in, const void *payload, int a, uint32_t j) {
    if (VALS) return DB_LD_STREAM((const double *)payload + j);
    return in.at[a][((const uint32_t *)payload)[j]];
}

__device__ __forceinline__ void det_store(const Accum &acc, uint64_t b, int a, bool want_sum, bool want_mm, double s,
                                          unsigned long long emin, unsigned long long nemax) {
    const uint64_t B = acc.nbins;
    if (want_sum) acc.sum[(uint64_t)__popc(acc.sum_mask & ((1u << a) - 1u)) * B + b] = s;
    if (want_mm)
        ((ulonglong2 *)acc.mm)[(uint64_t)__popc(acc.mm_mask & ((1u << a) - 1u)) * B + b] = make_ulonglong2(emin, nemax);
}

template <bool VALS>
__global__ void __launch_bounds__(256) k_det_fold(Inputs in, Accum acc, const void *payload, const uint32_t *seg_start,
                                                  const uint32_t *seg_end, uint32_t *long_list, uint32_t *long_cnt) {
    const uint64_t B = acc.nbins;
    constexpr int K = 8;
    for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < B; b += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t j0 = seg_start[b], j1 = seg_end[b];
        acc.count[b] = (unsigned long long)(j1 - j0);
        if (j1 - j0 > DET_LONG) long_list[atomicAdd(long_cnt, 1u)] = (uint32_t)b;  // k_det_fold_long's work
        if (j1 == j0 || j1 - j0 > DET_LONG) continue;
        for (int a = 0; a < in.nattr; ++a) {
            const bool want_sum = (acc.sum_mask >> a) & 1u, want_mm = (acc.mm_mask >> a) & 1u;
            if (!want_sum && !want_mm) continue;
            double s = 0.0;  // the sequential fold starts at +0.0
            unsigned long long emin = ~0ull, nemax = ~0ull;
            for (uint32_t j = j0; j < j1; j += K) {
                double v[K];
#pragma unroll
                for (int k = 0; k < K; ++k) v[k] = j + k < j1 ? det_val<VALS>(in, payload, a, j + k) : 0.0;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    if (j + k >= j1) break;
                    if (want_sum) s = __dadd_rn(s, v[k]);
                    if (want_mm) {
                        const unsigned long long e = enc_total(v[k]);
                        emin = e < emin ? e : emin;
                        nemax = ~e < nemax ? ~e : nemax;
                    }
                }
            }
            det_store(acc, b, a, want_sum, want_mm, s, emin, nemax);
        }
    }
}

// Resident warps take the long bins one at a time from the list (one atomic
// per bin), so every chain starts as soon as a warp is free: the step costs
// about the longest chain, not a sum over launch waves.
template <bool VALS>
__global__ void __launch_bounds__(256) k_det_fold_long(Inputs in, Accum acc, const void *payload,
                                                       const uint32_t *seg_start, const uint32_t *seg_end,
                                                       const uint32_t *long_list, uint32_t *long_ctr) {
    constexpr int CH = 256, PER = CH / 32;  // a step's add chain (~2k cycles) covers the next step's loads
    __shared__ __align__(16) double buf[8][2][CH];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t nlong = long_ctr[0];
    for (;;) {
        uint32_t i = 0;
        if (lane == 0) i = atomicAdd(&long_ctr[1], 1u);
        i = __shfl_sync(0xffffffffu, i, 0);
        if (i >= nlong) break;
        const uint64_t b = long_list[i];
        const uint32_t j0 = seg_start[b], j1 = seg_end[b];
        for (int a = 0; a < in.nattr; ++a) {
            const bool want_sum = (acc.sum_mask >> a) & 1u, want_mm = (acc.mm_mask >> a) & 1u;
            if (!want_sum && !want_mm) continue;
            double s = 0.0;
            unsigned long long emin = ~0ull, nemax = ~0ull;
            const uint32_t nch = (j1 - j0 + CH - 1) / CH;
            double r[PER];
            auto load = [&](uint32_t c) {  // issue only: nothing here waits for the data
#pragma unroll
                for (int u = 0; u < PER; ++u) {
                    const uint32_t j = j0 + c * CH + u * 32 + lane;
                    r[u] = j < j1 ? det_val<VALS>(in, payload, a, j) : 0.0;
                }
            };
            auto stash = [&](uint32_t c) {  // (the data has arrived by now) min/max, then shared memory
#pragma unroll
                for (int u = 0; u < PER; ++u) {
                    const uint32_t j = j0 + c * CH + u * 32 + lane;
                    if (want_mm && j < j1) {
                        const unsigned long long e = enc_total(r[u]);
                        emin = e < emin ? e : emin;
                        nemax = ~e < nemax ? ~e : nemax;
                    }
                    buf[w][c & 1][u * 32 + lane] = r[u];
                }
            };
            load(0);
            stash(0);
            __syncwarp();
            for (uint32_t c = 0; c < nch; ++c) {
                if (c + 1 < nch) load(c + 1);  // next step in flight while lane 0 adds this one
                if (want_sum && lane == 0) {
                    const uint32_t m = min((uint32_t)CH, j1 - j0 - c * CH);
                    const double2 *q = (const double2 *)buf[w][c & 1];
                    if (m == (uint32_t)CH) {  // 16 values in registers ahead of their 16 dependent adds
                        double2 v[8], nv[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) v[u] = q[u];
#pragma unroll
                        for (int k = 0; k < CH / 16; ++k) {
                            if (k + 1 < CH / 16) {
#pragma unroll
                                for (int u = 0; u < 8; ++u) nv[u] = q[(k + 1) * 8 + u];
                            }
#pragma unroll
                            for (int u = 0; u < 8; ++u) {
                                s = __dadd_rn(s, v[u].x);
                                s = __dadd_rn(s, v[u].y);
                            }
#pragma unroll
                            for (int u = 0; u < 8; ++u) v[u] = nv[u];
                        }
                    } else {
                        const double *q1 = buf[w][c & 1];
                        for (uint32_t k = 0; k < m; ++k) s = __dadd_rn(s, q1[k]);
                    }
                }
                __syncwarp();
                if (c + 1 < nch) stash(c + 1);
                __syncwarp();
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long x = __shfl_xor_sync(0xffffffffu, emin, o);
                const unsigned long long y = __shfl_xor_sync(0xffffffffu, nemax, o);
                emin = x < emin ? x : emin;
                nemax = y < nemax ? y : nemax;
            }
            if (lane == 0) det_store(acc, b, a, want_sum, want_mm, s, emin, nemax);
        }
    }
}

// ---- multi-rank deterministic combine: rank-ordered fold of gathered sums
// (oracle partition mode): s = ((+0.0 + s_0) + s_1) + ...
__global__ void k_det_rank_fold(const double *gathered, int nranks, uint64_t len, double *sum) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (uint64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < nranks; ++r) s = __dadd_rn(s, gathered[(uint64_t)r * len + i]);
        sum[i] = s;
    }
}

cudaError_t launch_rank_fold(const double *gathered, int nranks, uint64_t len, double *sum, int sms, cudaStream_t s) {
    uint64_t blocks = (len + 255) / 256;
    if (blocks > (uint64_t)sms * 8) blocks = (uint64_t)sms * 8;
    if (blocks == 0) return cudaSuccess;
    k_det_rank_fold<<<(unsigned)blocks, 256, 0, s>>>(gathered, nranks, len, sum);
    return cudaGetLastError();
}

// ---- scratch ----
void free_det_scratch(DetScratch &ds) {
    if (ds.device < 0) return;
    DeviceGuard g(ds.device);
    uint32_t *ps[] = {ds.keys, ds.keys_alt, ds.rows, ds.rows_alt, ds.hist, ds.offsets};
    for (uint32_t *p : ps)
        if (p) cudaFree(p);
    if (ds.keys) count_free(ds.cap_rows * 24 + ds.cap_hist * 4 + (int64_t)ds.cap_bins * 12 + 64);
    ds = DetScratch{};
}

int ensure_det_scratch(DetScratch &ds, int64_t n, uint64_t nbins, int device, int sms) {
    (void)sms;
    if (n >= (int64_t)0xffffffffLL) return set_error(BIN_EINVAL, "deterministic mode: %lld rows >= 2^32", (long long)n);
    int64_t nblk = (n + RS_TILE - 1) / RS_TILE;
    int64_t hist_len = 256 * nblk;
    int64_t part_len = (hist_len > (int64_t)nbins + 1 ? hist_len : (int64_t)nbins + 1) / SC_TILE + 2;
    if (ds.keys && ds.device == device && ds.cap_rows >= n && ds.cap_hist >= hist_len + part_len &&
        ds.cap_bins >= nbins)
        return BIN_OK;
    free_det_scratch(ds);
    DeviceGuard g(device);
    int64_t rows = n > 0 ? n : 1;
    ds.device = device;
    ds.cap_rows = rows;
    ds.cap_hist = hist_len + part_len;
    ds.cap_bins = nbins;
    // payload arrays hold 8 bytes per row (a value, or a row index in the low word)
    bool ok = cudaMalloc(&ds.keys, rows * 4) == cudaSuccess && cudaMalloc(&ds.keys_alt, rows * 4) == cudaSuccess &&
              cudaMalloc(&ds.rows, rows * 8) == cudaSuccess && cudaMalloc(&ds.rows_alt, rows * 8) == cudaSuccess &&
              cudaMalloc(&ds.hist, ds.cap_hist * 4) == cudaSuccess &&
              cudaMalloc(&ds.offsets, nbins * 12 + 64) == cudaSuccess;  // seg_start, seg_end, long list, 2 counters
    count_alloc(ds.cap_rows * 24 + ds.cap_hist * 4 + (int64_t)ds.cap_bins * 12 + 64);
    if (!ok) {
        cudaGetLastError();
        free_det_scratch(ds);
        return set_error(BIN_ENOMEM, "deterministic scratch for %lld rows", (long long)n);
    }
    return BIN_OK;
}

cudaError_t launch_deterministic(const Geom &g, const Inputs &in, const Accum &acc, DetScratch &ds,
                                 const LaunchCfg &lc, cudaStream_t s, int *launches) {
    const int64_t n = in.n;
    const uint32_t B = (uint32_t)acc.nbins;
    uint32_t *seg_start = ds.offsets, *seg_end = ds.offsets + acc.nbins;
    int64_t fill_blocks = (int64_t)lc.sms * 8;
    // carry the values through the sort when exactly one attribute is binned
    int nl = 0, va = 0;
    for (int a = 0; a < in.nattr; ++a)
        if ((acc.load_mask >> a) & 1u) ++nl, va = a;
    const bool vals = nl == 1;
    k_det_clear<<<(unsigned)fill_blocks, 256, 0, s>>>(ds.offsets, 2 * acc.nbins);
    k_det_clear<<<1, 32, 0, s>>>(ds.offsets + 3 * acc.nbins, 2);  // long-bin counters
    (*launches)++;
    (*launches)++;
    void *pay = ds.rows;
    if (n > 0) {
        if (vals) k_det_keys<true><<<(unsigned)fill_blocks, 256, 0, s>>>(g, in, acc, ds.keys, ds.rows, va);
        else k_det_keys<false><<<(unsigned)fill_blocks, 256, 0, s>>>(g, in, acc, ds.keys, ds.rows, va);
        (*launches)++;
        int bits = 0;
        while (bits < 32 && ((uint64_t)B >> bits) != 0) ++bits;  // keys are in [0, B]
        const int passes = (bits + 7) / 8;
        int64_t nblk = (n + RS_TILE - 1) / RS_TILE;
        uint32_t *hist = ds.hist, *part = ds.hist + 256 * nblk;
        uint32_t *k0 = ds.keys, *k1 = ds.keys_alt;
        void *r0 = ds.rows, *r1 = ds.rows_alt;
        for (int ps = 0, shift = 0; ps < passes; ++ps) {
            const int dbits = (bits - shift + (passes - ps) - 1) / (passes - ps);  // even split
            const uint32_t mask = (1u << dbits) - 1u;
            k_rs_hist<<<(unsigned)nblk, RS_THREADS, 0, s>>>(k0, n, shift, mask, hist, nblk);
            (*launches)++;
            cudaError_t e = scan_excl(hist, 256 * nblk, part, s, launches);
            if (e != cudaSuccess) return e;
            if (vals) {
                const size_t sm = (size_t)RS_TILE * 12;
                cudaFuncSetAttribute(k_rs_scatter<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                k_rs_scatter<double><<<(unsigned)nblk, RS_THREADS, sm, s>>>(k0, (const double *)r0, n, shift, dbits,
                                                                         hist, nblk, k1, (double *)r1);
            } else {
                const size_t sm = (size_t)RS_TILE * 8;
                cudaFuncSetAttribute(k_rs_scatter<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                k_rs_scatter<uint32_t><<<(unsigned)nblk, RS_THREADS, sm, s>>>(k0, (const uint32_t *)r0, n, shift,
                                                                           dbits, hist, nblk, k1, (uint32_t *)r1);
            }
            (*launches)++;
            uint32_t *t = k0; k0 = k1; k1 = t;
            void *tp = r0; r0 = r1; r1 = tp;
            shift += dbits;
        }
        k_det_segments<<<(unsigned)fill_blocks, 256, 0, s>>>(k0, n, B, seg_start, seg_end);
        (*launches)++;
        pay = r0;
    }
    int64_t fold_blocks = ((int64_t)acc.nbins + 255) / 256;  // one thread per bin
    if (fold_blocks < 1) fold_blocks = 1;
    // long bins: all warps resident at once, taking bins from the list (a warp per
    // bin in launch order ran the core bins' chains wave after wave: 5x slower)
    const int64_t long_blocks = (int64_t)lc.sms * 8;
    uint32_t *long_list = ds.offsets + 2 * acc.nbins, *long_ctr = long_list + acc.nbins;
    if (vals && n > 0) {
        k_det_fold<true><<<(unsigned)fold_blocks, 256, 0, s>>>(in, acc, pay, seg_start, seg_end, long_list, long_ctr);
        k_det_fold_long<true><<<(unsigned)long_blocks, 256, 0, s>>>(in, acc, pay, seg_start, seg_end, long_list,
                                                                     long_ctr);
    } else {
        k_det_fold<false><<<(unsigned)fold_blocks, 256, 0, s>>>(in, acc, pay, seg_start, seg_end, long_list, long_ctr);
        k_det_fold_long<false><<<(unsigned)long_blocks, 256, 0, s>>>(in, acc, pay, seg_start, seg_end, long_list,
                                                                      long_ctr);
    }
    (*launches) += 2;
    return cudaGetLastError();
}

}  // namespace db
