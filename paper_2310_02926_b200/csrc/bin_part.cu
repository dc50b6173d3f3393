// bin_part.cu -- the partition route of a4 + a5 for spread-out data
// (uniform particles, big 3D meshes: C2, C4, C5), where no shared-memory
// window holds most rows and the window route pays 2-13 L2 reductions per row.
//
// The mesh's bins are cut into T "tiles" of Wt consecutive linear bin indices,
// Wt chosen so one tile's accumulators fit in one CTA's shared memory.  Then
//   P1 k_part_keys     read the axes, write each row's bin index (u32, ~0 when
//                      outside), count rows per tile (shared memory, then one
//                      L2 add per tile and CTA)
//   P2 k_part_scan1/2  per-tile prefix over chunks, tile starts and the
//                      per-(group, chunk) write offsets: every output position
//                      is known before the scatter (no L2 atomic claims)
//   P3 k_part_scatter  read keys + attributes (TMA bulk copies, double buffer),
//                      counting-sort each batch of rows by group in shared
//                      memory, write the rows out as contiguous runs at the
//                      offsets of P2 (coalesced).
//                      Group = tile when T <= 64; else a super-tile of G1
//                      consecutive tiles (<= 64 of them), and
//   P3' k_part_refine  regroups each super-tile's rows by tile the same way, so
//                      every batch writes long runs (a one-level scatter into
//                      thousands of tiles wrote 1-2 rows per run: partial
//                      sectors, 2x DRAM write traffic, read-modify-write);
//   P4 k_part_reduce   each CTA takes an equal slice of the grouped rows and,
//                      tile by tile, accumulates them in shared memory: every
//                      row hits the window.  count: u32 ATOMS.ADD; sums: the
//                      96-bit fixed point of bin_general.cu with the exponent
//                      window holding most of the CTA's sampled values; min/
//                      max: exact u64 slots updated only when a read shows
//                      improvement.  Each tile is flushed into the global
//                      accumulator with one L2 reduction per bin and statistic.
// Algorithmic bytes stay 8(D+A)/row; this route streams 8D+4 + 2(8A+4) + 8A+4
// (+ 2(8A+4) with P3') bytes per row (D = 2, A = 1: 56 B vs 24) with no
// per-row global atomics.  Row order inside a tile is not kept (atomic mode).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "db_internal.h"
#include "dev_common.cuh"
#include "xsum.cuh"

namespace db {

extern __shared__ __align__(16) uint32_t p_dsm[];

constexpr int PART_THREADS = 1024;

// Exclusive scan of a[0..n) in shared memory by the whole CTA (blockDim a
// multiple of 32, <= 1024); returns the total.  wsum: 33 words of scratch.
__device__ __forceinline__ uint32_t block_scan_excl(uint32_t *a, uint32_t n, uint32_t *wsum) {
    const uint32_t nt = blockDim.x, per = (n + nt - 1) / nt;
    const uint32_t s0 = min(n, threadIdx.x * per), s1 = min(n, s0 + per);
    uint32_t sum = 0;
    for (uint32_t i = s0; i < s1; ++i) sum += a[i];
    const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= (unsigned)o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const uint32_t nw = nt >> 5;
        uint32_t w = lane < nw ? wsum[lane] : 0u, wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= (unsigned)o) wi += y;
        }
        if (lane < nw) wsum[lane] = wi - w;  // exclusive warp offsets
        if (lane == 31) wsum[32] = wi;       // total
    }
    __syncthreads();
    uint32_t run = wsum[warp] + inc - sum;
    const uint32_t total = wsum[32];
    for (uint32_t i = s0; i < s1; ++i) {
        const uint32_t v = a[i];
        a[i] = run;
        run += v;
    }
    __syncthreads();
    return total;
}

__device__ __forceinline__ uint32_t udiv(uint32_t x, const UDiv &p) {
    const uint32_t t = __umulhi(x, p.m);
    return (t + ((x - t) >> p.s1)) >> p.s2;
}

// Bin index of one row (a4), or ~0u outside the mesh.
template <int D>
__device__ __forceinline__ uint32_t part_key(const DGeom &G, const double (&x)[D]) {
    bool in = G.ok;
    uint32_t b = 0, mul = 1;
#pragma unroll
    for (int d = 0; d < D; ++d) {
        in = in && (G.lo[d] <= x[d]) && (x[d] <= G.hi[d]);
        const int k = min(floor_nonneg(__dmul_rn(__dsub_rn(x[d], G.lo[d]), G.scale[d])), G.res[d] - 1);
        b += (uint32_t)k * mul;
        mul *= (uint32_t)G.res[d];
    }
    return in ? b : ~0u;
}

// ---------------------------------------------------------------- P1
#ifndef PART_KEYS_LD
#define PART_KEYS_LD __ldcg
#endif
#ifndef PART_RED_LD
#define PART_RED_LD __ldcg
#endif
// Key slots: pair p (rows head+2p, head+2p+1) -> slots 2p, 2p+1; the
// unpaired head row -> slot 2*npairs, the unpaired tail row -> 2*npairs+1.
// Both belong to the last chunk.  Chunk c = pairs [npairs*c/C, npairs*(c+1)/C),
// the same in P1 and P3.  Writes cnt[t*C + c] = rows of chunk c in tile t.
// PART_KEYS_TMA: the chunk's axis columns are staged into shared memory by
// TMA bulk copies (cp.async.bulk, one mbarrier per buffer, two buffers of
// KEYS_SP pairs per column), so the loads in flight cost no registers.
#ifndef PART_KEYS_TMA
#define PART_KEYS_TMA 1
#endif
constexpr uint32_t KEYS_SP = 1024;  // pairs per stage and column (16 KB)
__device__ __forceinline__ void keys_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
                 "r"((unsigned)__cvta_generic_to_shared(bar))
                 : "memory");
}
size_t keys_smem(int D, uint32_t T) { return (PART_KEYS_TMA ? 2ull * D * KEYS_SP * 16 : 0ull) + (size_t)T * 4; }

template <int D, int NT>
__global__ void __launch_bounds__(NT, 2) k_part_keys(Geom g, Inputs in, Accum acc, PartArgs pa) {
#if PART_KEYS_TMA
    const double2 *stage = (const double2 *)p_dsm;         // [2][D][KEYS_SP]
    uint32_t *hist = p_dsm + (2u * D * KEYS_SP * 16u) / 4u;  // [T]
    __shared__ __align__(8) uint64_t kbar[2];
#else
    uint32_t *hist = p_dsm;  // [T]
#endif
    const DGeom G = load_geom<D>(g, acc.bounds);
    const uint32_t T = pa.T, C = pa.C, c = blockIdx.x;
    for (uint32_t i = threadIdx.x; i < T; i += NT) hist[i] = 0u;
    const uint32_t p0 = (uint32_t)(((uint64_t)pa.npairs * c) / C), p1 = (uint32_t)(((uint64_t)pa.npairs * (c + 1)) / C);
    const double2 *cx[D];
#pragma unroll
    for (int d = 0; d < D; ++d) cx[d] = (const double2 *)(in.ax[d] + pa.head);
    uint2 *kout = (uint2 *)pa.keys;
    const uint32_t Wt = pa.Wt;
    uint32_t n_in = 0, rows = 0;
    auto one = [&](const double (&x)[D]) -> uint32_t {
        const uint32_t b = part_key<D>(G, x);
        if (b != ~0u) {
            DB_CHECK(udiv(b, pa.wt_div) == b / Wt && b / Wt < T && b < acc.nbins);
            atomicAdd(&hist[udiv(b, pa.wt_div)], 1u);
            ++n_in;
        }
        return b;
    };
#if PART_KEYS_TMA
    const uint32_t nst = (p1 - p0 + KEYS_SP - 1) / KEYS_SP;
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&kbar[b]))
                         : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();  // (also: hist zeroed)
    auto issue = [&](uint32_t k) {  // thread 0: stage k into buffer k & 1
        const uint32_t ps = p0 + k * KEYS_SP, np = min(KEYS_SP, p1 - ps);
        uint64_t *bar = &kbar[k & 1u];
        unsigned long long st;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 %0, [%1], %2;"
                     : "=l"(st) : "r"((unsigned)__cvta_generic_to_shared(bar)), "r"((unsigned)(D * np * 16u)) : "memory");
        (void)st;
#pragma unroll
        for (int d = 0; d < D; ++d)
            keys_g2s((void *)(stage + ((k & 1u) * D + d) * KEYS_SP), cx[d] + ps, np * 16u, bar);
    };
    if (threadIdx.x == 0) {
        if (nst > 0) issue(0);
        if (nst > 1) issue(1);
    }
    for (uint32_t k = 0; k < nst; ++k) {
        {
            const unsigned bar = (unsigned)__cvta_generic_to_shared(&kbar[k & 1u]), par = (k >> 1) & 1u;
            unsigned done = 0;
            while (!done)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(done) : "r"(bar), "r"(par) : "memory");
        }
        const uint32_t ps = p0 + k * KEYS_SP, np = min(KEYS_SP, p1 - ps);
        const double2 *sb = stage + (k & 1u) * D * KEYS_SP;
        for (uint32_t li = threadIdx.x; li < np; li += NT) {
            double2 a[D];
#pragma unroll
            for (int d = 0; d < D; ++d) a[d] = sb[d * KEYS_SP + li];
            double x[D];
#pragma unroll
            for (int d = 0; d < D; ++d) x[d] = a[d].x;
            const uint32_t k0 = one(x);
#pragma unroll
            for (int d = 0; d < D; ++d) x[d] = a[d].y;
            const uint32_t k1 = one(x);
            __stcg(kout + ps + li, make_uint2(k0, k1));
            rows += 2;
        }
        __syncthreads();  // buffer k & 1 read by every thread
        if (threadIdx.x == 0 && k + 2 < nst) issue(k + 2);
    }
#else
    __syncthreads();
    for (uint32_t p = p0 + threadIdx.x; p < p1; p += 2 * NT) {
        const uint32_t q = p + NT;
        const bool has2 = q < p1;
        double2 a[D], b[D];
#pragma unroll
        for (int d = 0; d < D; ++d) {
            a[d] = PART_KEYS_LD(cx[d] + p);
            b[d] = has2 ? PART_KEYS_LD(cx[d] + q) : make_double2(0.0, 0.0);
        }
        double x[D];
#pragma unroll
        for (int d = 0; d < D; ++d) x[d] = a[d].x;
        const uint32_t k0 = one(x);
#pragma unroll
        for (int d = 0; d < D; ++d) x[d] = a[d].y;
        const uint32_t k1 = one(x);
        __stcg(kout + p, make_uint2(k0, k1));
        rows += 2;
        if (has2) {
#pragma unroll
            for (int d = 0; d < D; ++d) x[d] = b[d].x;
            const uint32_t k2 = one(x);
#pragma unroll
            for (int d = 0; d < D; ++d) x[d] = b[d].y;
            const uint32_t k3 = one(x);
            __stcg(kout + q, make_uint2(k2, k3));
            rows += 2;
        }
    }
#endif
    if (c == C - 1 && threadIdx.x < 2) {  // unpaired head / tail row
        const int64_t r = threadIdx.x == 0 ? (pa.head ? 0 : -1) : (pa.tail ? in.n - 1 : -1);
        if (r >= 0) {
            double x[D];
#pragma unroll
            for (int d = 0; d < D; ++d) x[d] = in.ax[d][r];
            pa.keys[2 * (uint64_t)pa.npairs + threadIdx.x] = one(x);
            rows += 1;
        }
    }
    unsigned long long in_w = n_in, out_w = rows - n_in;
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
    for (uint32_t t = threadIdx.x; t < T; t += NT) pa.cnt[(uint64_t)t * C + c] = hist[t];
}

// ---------------------------------------------------------------- P2
// k_part_scan1, one CTA per super-tile s (tiles [s*G1, s*G1 + G1)): each tile
// row of cnt becomes its exclusive prefix over chunks (rows of tile t from
// chunks < c), tot[t] = its total; off1[s*(C+1) + c] = rows of super-tile s
// from chunks < c (off1[.. + C] = the super-tile's total).
__global__ void __launch_bounds__(1024) k_part_scan1(PartArgs pa) {
    uint32_t *c1 = p_dsm, *wsum = p_dsm + pa.C + 1;
    const uint32_t C = pa.C, s = blockIdx.x, lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t tb = s * pa.G1, te = min(pa.T, tb + pa.G1);
    for (uint32_t i = threadIdx.x; i <= C; i += blockDim.x) c1[i] = 0u;
    __syncthreads();
    for (uint32_t t = tb + warp; t < te; t += blockDim.x >> 5) {
        uint32_t *row = pa.cnt + (uint64_t)t * C;
        uint32_t run = 0;
        for (uint32_t base = 0; base < C; base += 32) {
            const uint32_t i = base + lane;
            const uint32_t v = i < C ? row[i] : 0u;
            uint32_t inc = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= (unsigned)o) inc += y;
            }
            if (i < C) {
                row[i] = run + inc - v;
                if (v) atomicAdd(&c1[i], v);
            }
            run += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) pa.tot[t] = run;
    }
    __syncthreads();
    const uint32_t total = block_scan_excl(c1, C, wsum);
    for (uint32_t i = threadIdx.x; i < C; i += blockDim.x) pa.off1[(uint64_t)s * (C + 1) + i] = c1[i];
    if (threadIdx.x == 0) pa.off1[(uint64_t)s * (C + 1) + C] = total;
}

// k_part_scan2, one CTA: tstart[t] = first grouped row of tile t, tstart[T] =
// rows inside the mesh.
__global__ void __launch_bounds__(1024) k_part_scan2(PartArgs pa) {
    uint32_t *a = p_dsm, *wsum = p_dsm + pa.T;
    const uint32_t T = pa.T;
    for (uint32_t t = threadIdx.x; t < T; t += blockDim.x) a[t] = pa.tot[t];
    __syncthreads();
    const uint32_t total = block_scan_excl(a, T, wsum);
    for (uint32_t t = threadIdx.x; t < T; t += blockDim.x) pa.tstart[t] = a[t];
    if (threadIdx.x == 0) pa.tstart[T] = total;
}


// Warp 0: exclusive scan of bcnt[0..ng) (ng <= 128) -> boff, hand out each
// group's output range from the CTA's cursors (gbase = cur; cur += count),
// clear bcnt; *nst = batch total.  No global atomics: the cursors start at
// the positions P2 computed for this chunk / work item.
__device__ __forceinline__ void claim_ranges(uint32_t *bcnt, uint32_t *boff, uint32_t *gbase, uint32_t *cur,
                                             uint32_t ng, uint32_t *nst) {
    const unsigned lane = threadIdx.x & 31u;
    uint32_t c[4], s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t g = 4 * lane + k;
        c[k] = g < ng ? bcnt[g] : 0u;
        s += c[k];
    }
    uint32_t inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= (unsigned)o) inc += y;
    }
    uint32_t run = inc - s;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t g = 4 * lane + k;
        if (g < ng) {
            boff[g] = run;
            gbase[g] = cur[g];
            cur[g] += c[k];
            bcnt[g] = 0u;
        }
        run += c[k];
    }
    if (lane == 31) *nst = inc;
}

// ---------------------------------------------------------------- P3
// Chunk c's rows grouped by tile (T <= 64: straight into skey/sval) or by
// super-tile (into xkey/xval).  Shared memory: in[2] {keys uint2 [NP] | vals
// double2 [A][NP]} | st_val f64 [A][R] | st_key u32 [R] | st_g u8 [R] |
// bcnt, boff, gbase, cur [128] | nst
template <int A, int PPT, int NT>
__global__ void __launch_bounds__(NT, 2) k_part_scatter(Inputs in, PartArgs pa) {
    constexpr int NP = PPT * NT, R = 2 * NP;
    // input buffers: keys uint2 [NP + 2] (bulk copy from the batch's first pair
    // rounded down to even, so source and size are 16-byte multiples) | vals double2 [A][NP]
    constexpr size_t KB = (size_t)(NP + 2) * 8;
    constexpr size_t IN_BYTES = KB + (size_t)NP * 16 * A;
    __shared__ __align__(8) uint64_t sbar[2];
    unsigned char *sm = (unsigned char *)p_dsm;
    double *st_val = (double *)(sm + 2 * IN_BYTES);
    uint32_t *st_key = (uint32_t *)(st_val + A * R);
    uint8_t *st_g = (uint8_t *)(st_key + R);
    uint32_t *bcnt = (uint32_t *)(st_g + R), *boff = bcnt + 128, *gbase = boff + 128, *cur = gbase + 128,
             *nstp = cur + 128;
    const bool two = pa.G1 > 1;
    uint32_t *okey = two ? pa.xkey : pa.skey;
    double *oval = two ? pa.xval : pa.sval;
    const uint32_t ng = pa.T1;
    const uint32_t C = pa.C, c = blockIdx.x;
    const uint32_t p0 = (uint32_t)(((uint64_t)pa.npairs * c) / C), p1 = (uint32_t)(((uint64_t)pa.npairs * (c + 1)) / C);
    const uint2 *kin = (const uint2 *)pa.keys;
    const int nl = pa.nl;
    const double2 *cv[A > 0 ? A : 1];
#pragma unroll
    for (int j = 0; j < A; ++j) cv[j] = (const double2 *)(in.at[pa.lattr[j < nl ? j : 0]] + pa.head);
    const uint64_t cap = pa.cap;
    const uint32_t nb = (p1 - p0 + NP - 1) / NP;
    // TMA bulk copies of batch k into buffer k & 1 (thread 0; one mbarrier per buffer)
    auto issue = [&](uint32_t k) {
        unsigned char *ib = sm + (k & 1) * IN_BYTES;
        const uint32_t ps = p0 + k * NP, np = min((uint32_t)NP, p1 - ps);
        const uint32_t kbase = ps & ~1u, nkp = (ps + np - kbase + 1u) & ~1u;  // <= npairs + 1 slots: in bounds
        uint64_t *bar = &sbar[k & 1];
        unsigned long long st;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 %0, [%1], %2;"
                     : "=l"(st) : "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(nkp * 8u + (uint32_t)nl * np * 16u)
                     : "memory");
        (void)st;
        keys_g2s(ib, kin + kbase, nkp * 8u, bar);
#pragma unroll
        for (int j = 0; j < A; ++j)
            if (j < nl) keys_g2s(ib + KB + (size_t)j * NP * 16, cv[j] + ps, np * 16u, bar);
    };
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&sbar[b]))
                         : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (nb > 0) issue(0);
    }
    if (threadIdx.x < 128) {
        bcnt[threadIdx.x] = 0u;
        const uint32_t gi = threadIdx.x;
        if (gi < ng)
            cur[gi] = two ? pa.tstart[gi * pa.G1] + pa.off1[(uint64_t)gi * (C + 1) + c]
                          : pa.tstart[gi] + pa.cnt[(uint64_t)gi * C + c];
    }
    __syncthreads();
    for (uint32_t k = 0; k < nb; ++k) {
        if (threadIdx.x == 0 && k + 1 < nb) issue(k + 1);  // (buffer (k+1)&1 was last read before this
                                                            //  iteration's barriers of batch k-1)
        {
            const unsigned bar = (unsigned)__cvta_generic_to_shared(&sbar[k & 1]), par = (k >> 1) & 1u;
            unsigned done = 0;
            while (!done)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(done) : "r"(bar), "r"(par) : "memory");
        }
        const unsigned char *ib = sm + (k & 1) * IN_BYTES;
        const uint32_t koff = (p0 + k * NP) & 1u;
        uint32_t key[2 * PPT], g[2 * PPT], rk[2 * PPT];
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
            const uint32_t li = q * NT + threadIdx.x;
            const uint2 kk = (p0 + k * NP + li < p1) ? ((const uint2 *)ib)[koff + li] : make_uint2(~0u, ~0u);
            key[2 * q] = kk.x;
            key[2 * q + 1] = kk.y;
        }
#pragma unroll
        for (int r = 0; r < 2 * PPT; ++r) {
            g[r] = key[r] != ~0u ? udiv(key[r], pa.wg_div) : 0u;
            rk[r] = key[r] != ~0u ? atomicAdd(&bcnt[g[r]], 1u) : 0u;
        }
        __syncthreads();
        if (threadIdx.x < 32) claim_ranges(bcnt, boff, gbase, cur, ng, nstp);
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 2 * PPT; ++r) {
            if (key[r] == ~0u) continue;
            const uint32_t pos = boff[g[r]] + rk[r], li = (r >> 1) * NT + threadIdx.x;
            DB_CHECK(g[r] < ng && pos < (uint32_t)R);
            st_key[pos] = key[r];
            st_g[pos] = (uint8_t)g[r];
#pragma unroll
            for (int j = 0; j < A; ++j) {
                const double2 v = ((const double2 *)(ib + KB))[(size_t)j * NP + li];
                st_val[j * R + pos] = (r & 1) ? v.y : v.x;
            }
        }
        __syncthreads();
        const uint32_t nst = *nstp;
#pragma unroll 2
        for (uint32_t i = threadIdx.x; i < nst; i += NT) {
            const uint32_t gg = st_g[i];
            const uint64_t gp = (uint64_t)gbase[gg] + (i - boff[gg]);
            DB_CHECK(gg < ng && gp < cap && gp >= pa.tstart[gg * pa.G1] && gp < pa.tstart[min(pa.T, (gg + 1) * pa.G1)]);
            __stcg(okey + gp, st_key[i]);
#pragma unroll
            for (int j = 0; j < A; ++j)
                if (j < nl) __stcg(oval + j * cap + gp, st_val[j * R + i]);
        }
    }
    __syncthreads();
    if (c == C - 1 && threadIdx.x < 2) {  // unpaired head / tail row (slots 2*npairs, 2*npairs+1)
        const int64_t r = threadIdx.x == 0 ? (pa.head ? 0 : -1) : (pa.tail ? in.n - 1 : -1);
        if (r >= 0) {
            const uint32_t key = pa.keys[2 * (uint64_t)pa.npairs + threadIdx.x];
            if (key != ~0u) {
                const uint64_t gp = atomicAdd(&cur[udiv(key, pa.wg_div)], 1u);
                okey[gp] = key;
#pragma unroll
                for (int j = 0; j < A; ++j)
                    if (j < nl) oval[j * cap + gp] = in.at[pa.lattr[j]][r];
            }
        }
    }
}

// ---------------------------------------------------------------- P3'
// Regroups the super-tile-grouped rows (xkey/xval) by tile.  Work item (s, c)
// = the rows of super-tile s that came from chunk c: contiguous in xkey at
// tstart[s*G1] + off1[s][c], and their tiles' output ranges are known from
// P2 (tstart[t] + cnt[t][c]), so no atomics.  CTA b takes the items whose
// first row lies in [ns*b/G, ns*(b+1)/G) (items are at most one chunk).
// Shared memory: in[2] {keys u32 [R] | vals f64 [A][R]} | st_val f64 [A][R] |
// st_key u32 [R] | st_g u8 [R] | bcnt, boff, gbase, cur [128] | nst
template <int A, int RPT, int NT>
__global__ void __launch_bounds__(NT, 2) k_part_refine(PartArgs pa) {
    constexpr int R = RPT * NT;
    constexpr int RS = R + 4;  // input slots: the batch from its row rounded down to a multiple of 4
    constexpr size_t IN_BYTES = (size_t)RS * (4 + 8 * A);
    unsigned char *sm = (unsigned char *)p_dsm;
    double *st_val = (double *)(sm + 2 * IN_BYTES);
    uint32_t *st_key = (uint32_t *)(st_val + A * R);
    uint8_t *st_g = (uint8_t *)(st_key + R);
    uint32_t *bcnt = (uint32_t *)(st_g + R), *boff = bcnt + 128, *gbase = boff + 128, *cur = gbase + 128,
             *nstp = cur + 128;
    const uint32_t T = pa.T, G1 = pa.G1, T1 = pa.T1, Wt = pa.Wt, C = pa.C;
    const uint32_t ns = pa.tstart[T];
    const uint32_t lo = (uint32_t)(((uint64_t)ns * blockIdx.x) / gridDim.x);
    const uint32_t hi = (uint32_t)(((uint64_t)ns * (blockIdx.x + 1)) / gridDim.x);
    const int nl = pa.nl;
    const uint64_t cap = pa.cap;
    const uint32_t NI = T1 * C;
    auto istart = [&](uint32_t it) -> uint32_t {
        if (it >= NI) return ns;
        const uint32_t s = it / C, c = it - s * C;
        return pa.tstart[s * G1] + pa.off1[(uint64_t)s * (C + 1) + c];
    };
    // first item starting at or after lo; items [i0, i1)
    auto lower = [&](uint32_t x) -> uint32_t {
        uint32_t a = 0, b = NI;
        while (a < b) {
            const uint32_t m = (a + b) >> 1;
            if (istart(m) < x) a = m + 1;
            else b = m;
        }
        return a;
    };
    const uint32_t i0 = lower(lo), i1 = blockIdx.x + 1 == gridDim.x ? NI : lower(hi);
    // batch descriptors (uniform across the CTA): rows [b0, b1) of item it
    uint32_t n_it = i0, n_b0 = i0 < NI ? istart(i0) : ns;
    auto next_batch = [&](uint32_t &b0, uint32_t &b1, uint32_t &it) -> bool {
        while (n_it < i1 && n_b0 >= istart(n_it + 1)) {
            ++n_it;
            n_b0 = istart(n_it);
        }
        if (n_it >= i1) return false;
        it = n_it;
        b0 = n_b0;
        b1 = min(b0 + (uint32_t)R, istart(n_it + 1));
        n_b0 = b1;
        return true;
    };
    // TMA bulk copies of rows [b0 & ~3, round4(b1)) into buffer buf (thread 0;
    // slot s = row - (b0 & ~3); the scratch arrays are padded so the rounded
    // range stays inside them, and the value planes are 4-row aligned)
    __shared__ __align__(8) uint64_t rbar[2];
    auto issue = [&](int buf, uint32_t b0, uint32_t b1) {
        unsigned char *ib = sm + buf * IN_BYTES;
        const uint32_t base = b0 & ~3u, nr = (b1 - base + 3u) & ~3u;
        uint64_t *bar = &rbar[buf];
        unsigned long long st;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 %0, [%1], %2;"
                     : "=l"(st) : "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(nr * 4u + (uint32_t)nl * nr * 8u)
                     : "memory");
        (void)st;
        keys_g2s(ib, pa.xkey + base, nr * 4u, bar);
#pragma unroll
        for (int j = 0; j < A; ++j)
            if (j < nl) keys_g2s(ib + (size_t)RS * 4 + (size_t)j * RS * 8, pa.xval + j * cap + base, nr * 8u, bar);
    };
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&rbar[b]))
                         : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    uint32_t rphase = 0;  // parity bits of rbar[0], rbar[1]
    if (threadIdx.x < 128) bcnt[threadIdx.x] = 0u;
    uint32_t cb0 = 0, cb1 = 0, cit = 0, loaded_it = ~0u;
    bool have = next_batch(cb0, cb1, cit);
    if (have && threadIdx.x == 0) issue(0, cb0, cb1);
    __syncthreads();
    for (int k = 0; have; ++k) {
        uint32_t nb0_ = 0, nb1_ = 0, nit_ = 0;
        const bool more = next_batch(nb0_, nb1_, nit_);
        if (more && threadIdx.x == 0) issue((k + 1) & 1, nb0_, nb1_);
        const uint32_t s = cit / C, tb = s * G1, ngt = min(G1, T - tb);
        if (cit != loaded_it) {  // new work item: its tiles' output cursors
            const uint32_t c = cit - s * C;
            if (threadIdx.x < ngt) cur[threadIdx.x] = pa.tstart[tb + threadIdx.x] + pa.cnt[(uint64_t)(tb + threadIdx.x) * C + c];
            loaded_it = cit;
        }
        {
            const unsigned bar = (unsigned)__cvta_generic_to_shared(&rbar[k & 1]), par = (rphase >> (k & 1)) & 1u;
            unsigned done = 0;
            while (!done)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(done) : "r"(bar), "r"(par) : "memory");
            rphase ^= 1u << (k & 1);
        }
        const unsigned char *ib = sm + (k & 1) * IN_BYTES;
        const uint32_t off = cb0 & 3u;
        uint32_t key[RPT], g[RPT], rk[RPT];
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const uint32_t li = q * NT + threadIdx.x;
            key[q] = cb0 + li < cb1 ? ((const uint32_t *)ib)[off + li] : ~0u;
            g[q] = key[q] != ~0u ? udiv(key[q], pa.wt_div) - tb : 0u;
            rk[q] = key[q] != ~0u ? atomicAdd(&bcnt[g[q]], 1u) : 0u;
        }
        __syncthreads();
        if (threadIdx.x < 32) claim_ranges(bcnt, boff, gbase, cur, ngt, nstp);
        __syncthreads();
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            if (key[q] == ~0u) continue;
            const uint32_t pos = boff[g[q]] + rk[q], li = q * NT + threadIdx.x;
            DB_CHECK(g[q] < ngt && pos < (uint32_t)R);
            st_key[pos] = key[q];
            st_g[pos] = (uint8_t)g[q];
#pragma unroll
            for (int j = 0; j < A; ++j) st_val[j * R + pos] = ((const double *)(ib + (size_t)RS * 4))[(size_t)j * RS + off + li];
        }
        __syncthreads();
        const uint32_t nst = *nstp;
#pragma unroll 2
        for (uint32_t i = threadIdx.x; i < nst; i += NT) {
            const uint32_t gg = st_g[i];
            const uint64_t gp = (uint64_t)gbase[gg] + (i - boff[gg]);
            DB_CHECK(gp >= pa.tstart[tb + gg] && gp < pa.tstart[tb + gg + 1]);
            __stcg(pa.skey + gp, st_key[i]);
#pragma unroll
            for (int j = 0; j < A; ++j)
                if (j < nl) __stcg(pa.sval + j * cap + gp, st_val[j * R + i]);
        }
        have = more;
        cb0 = nb0_, cb1 = nb1_, cit = nit_;
    }
}

// ---------------------------------------------------------------- P4
// Window words: mm u64 {enc(min), ~enc(max)} [nmm][W] (exact) | fixed-point
// sums u32 [nsum][3][W] | count u32 [W].  Before the first tile the same
// memory holds the exponent histograms [A][2048] of the CTA's sampled values.
template <int A, bool XS>
__global__ void __launch_bounds__(PART_THREADS, 1) k_part_reduce(Accum acc, PartArgs pa) {
    constexpr int AA = A > 0 ? A : 1;
    constexpr int U = A <= 1 ? 4 : 2;  // rows per thread per stage (two stages in flight)
    const uint32_t T = pa.T, Wt = pa.Wt;
    const uint64_t B = acc.nbins, cap = pa.cap;
    const uint32_t ns = pa.tstart[T];
    const uint32_t lo = (uint32_t)(((uint64_t)ns * blockIdx.x) / gridDim.x);
    const uint32_t hi = (uint32_t)(((uint64_t)ns * (blockIdx.x + 1)) / gridDim.x);
    if (lo >= hi) return;
    __shared__ int s_xr[2 * BIN_MAX_ATTR];  // BIN_SUM_EXACT: digits this CTA touched (xsum.cuh)
    if (XS) xr_init(s_xr);
    const int nl = pa.nl;
    const uint32_t sum_mask = acc.sum_mask, mm_mask = acc.mm_mask;
    int ss[AA], ms[AA];  // sum / min-max slot of load slot j, -1 if none
#pragma unroll
    for (int j = 0; j < AA; ++j) {
        const int a = j < nl ? pa.lattr[j] : 0;
        ss[j] = (j < nl && ((sum_mask >> a) & 1u)) ? (int)__popc(sum_mask & ((1u << a) - 1u)) : -1;
        ms[j] = (j < nl && ((mm_mask >> a) & 1u)) ? (int)__popc(mm_mask & ((1u << a) - 1u)) : -1;
    }
    // ---- fixed-point exponent window per summed attribute: the 9 consecutive
    // exponents holding the most of 2048 sampled values of this CTA's rows
    // (a max-based choice lets one outlier, e.g. the central body of mass
    // 1000, push every ordinary value out of range into f64 L2 reductions)
    FxParam fx[AA];
    {
        uint32_t *eh = p_dsm;  // [A][2048]
        __shared__ uint32_t s_best[AA][32];
        for (uint32_t i = threadIdx.x; i < AA * 2048; i += PART_THREADS) eh[i] = 0u;
        __syncthreads();
        const uint32_t m = hi - lo, K = min(m, 2048u);
#pragma unroll
        for (int j = 0; j < A; ++j) {
            if (ss[j] < 0) continue;
            for (uint32_t k = threadIdx.x; k < K; k += PART_THREADS) {
                const double v = __ldcs(pa.sval + j * cap + lo + (uint32_t)(((uint64_t)k * m) / K));
                const unsigned eb = ((unsigned)__double2hiint(v) >> 20) & 0x7ffu;
                if (eb != 0u && eb != 0x7ffu) atomicAdd(&eh[j * 2048 + eb], 1u);
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < AA; ++j) {
            uint32_t best = 0;
            for (uint32_t e = threadIdx.x; e < 2048; e += PART_THREADS) {
                uint32_t cnt = 0;
                for (uint32_t k = 0; k < 9 && e + k < 2047; ++k) cnt += eh[j * 2048 + e + k];
                const uint32_t key = (cnt << 11) | e;  // most values, ties -> larger exponents
                best = cnt && key > best ? key : best;
            }
            best = __reduce_max_sync(0xffffffffu, best);
            if ((threadIdx.x & 31) == 0) s_best[j][threadIdx.x >> 5] = best;
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < AA; ++j) {
            uint32_t best = 0;
            for (int w = 0; w < PART_THREADS / 32; ++w) best = max(best, s_best[j][w]);
            // exponents [e, e + 9) -> fx_param(fxexp = e + 6) (eb_hi = fxexp + 3)
            fx[j] = fx_param(best ? (best & 2047u) + 6u : 0u);
            if (XS) {  // exact sums: grid topped by the window's highest sampled binade
                unsigned top = 0;
                if (best)
                    for (unsigned k = 0; k < 9; ++k)
                        if (eh[j * 2048 + (best & 2047u) + k]) top = (best & 2047u) + k;
                fx[j] = fx_param_exact(top);
            }
        }
        __syncthreads();
    }
    const uint32_t nsum = acc.nsum, nmm = acc.nmm;
    ulonglong2 *wmm = (ulonglong2 *)p_dsm;
    // first tile: the last t with tstart[t] <= lo
    uint32_t t0 = 0, t1 = T;
    while (t1 - t0 > 1) {
        const uint32_t mid = (t0 + t1) >> 1;
        if (pa.tstart[mid] <= lo) t0 = mid;
        else t1 = mid;
    }
    for (uint32_t t = t0; t < T; ++t) {
        const uint32_t ts = pa.tstart[t], te = pa.tstart[t + 1];
        if (ts >= hi) break;
        const uint32_t r0 = max(lo, ts), r1 = min(hi, te);
        if (r0 >= r1) continue;
        const uint64_t base = (uint64_t)t * Wt;
        const uint32_t W = (uint32_t)min((uint64_t)Wt, B - base);
        const uint32_t o_fx = 4u * nmm * W, o_cnt = o_fx + 3u * nsum * W;
        for (uint32_t i = threadIdx.x; i < nmm * W; i += PART_THREADS) wmm[i] = make_ulonglong2(~0ull, ~0ull);
        for (uint32_t i = o_fx + threadIdx.x; i < o_cnt + W; i += PART_THREADS) p_dsm[i] = 0u;
        __syncthreads();
        const uint32_t bl = (uint32_t)base;
        uint32_t key[U];
        double v[AA][U];
        auto load = [&](uint32_t i0) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t i = i0 + u * PART_THREADS;
                const bool ok = i < r1;
                key[u] = ok ? PART_RED_LD(pa.skey + i) : ~0u;
#pragma unroll
                for (int j = 0; j < A; ++j) v[j][u] = (ok && j < nl) ? PART_RED_LD(pa.sval + j * cap + i) : 0.0;
            }
        };
        load(r0 + threadIdx.x);
        for (uint32_t i0 = r0 + threadIdx.x; i0 < r1; i0 += U * PART_THREADS) {
            uint32_t ck[U];
            double cvv[AA][U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                ck[u] = key[u];
#pragma unroll
                for (int j = 0; j < A; ++j) cvv[j][u] = v[j][u];
            }
            load(i0 + U * PART_THREADS);  // next stage in flight while this one is accumulated
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (ck[u] == ~0u) continue;
                const uint32_t l = ck[u] - bl;
                DB_CHECK(l < W);
                atomicAdd(&p_dsm[o_cnt + l], 1u);
#pragma unroll
                for (int j = 0; j < A; ++j) {
                    const double x = cvv[j][u];
                    if (ss[j] >= 0) {
                        const uint32_t w0 = o_fx + (uint32_t)ss[j] * 3u * W + l;
                        unsigned qmid;
                        unsigned long long q = 0;
                        bool fxp;
                        if (XS) {
                            fxp = fx_quant_exact(fx[j], x, q);
                        } else {
                            fxp = fx_path(fx[j], x);
                            if (fxp) q = fx_quant(fx[j], x);
                        }
                        if (fxp) {
                            const unsigned qlo = (unsigned)q;
                            qmid = (unsigned)(q >> 32);
                            const unsigned old = atomicAdd(&p_dsm[w0], qlo);
                            qmid += (old + qlo < old) ? 1u : 0u;
                        } else {  // outside the fixed range: f64 L2 reduction, offset only here
                            if (XS) xsum_add_double(acc.xs, B, ss[j], base + l, x, s_xr);
                            else atomicAdd(&acc.sum[(uint64_t)ss[j] * B + base + l], x);
                            qmid = FX_OFFSET_MID;
                        }
                        const unsigned old2 = atomicAdd(&p_dsm[w0 + W], qmid);
                        if (old2 + qmid < old2) atomicAdd(&p_dsm[w0 + 2 * W], 1u);
                    }
                    if (ms[j] >= 0) {
                        const unsigned long long e = enc_total(x);
                        ulonglong2 *slot = &wmm[(uint32_t)ms[j] * W + l];
                        const ulonglong2 f = lds_volatile_u64x2(slot);  // stale is safe: slots only decrease
                        if (e < f.x) atomicMin(&slot->x, e);
                        if (~e < f.y) atomicMin(&slot->y, ~e);
                    }
                }
            }
        }
        __syncthreads();
        // a tile whose rows are all this CTA's (C4: ~16 whole tiles per CTA)
        // is written with plain stores: no other CTA touches its bins, and
        // k_prep left them at the identities (sums: load + add, since values
        // outside the fixed range were already reduced into them above)
        const bool owned = !XS && r0 == ts && r1 == te;
        for (uint32_t l = threadIdx.x; l < W; l += PART_THREADS) {
            const unsigned long long cnt = p_dsm[o_cnt + l];
            if (cnt == 0) continue;
            const uint64_t b = base + l;
            if (owned) {
                __stcg(&acc.count[b], cnt);
#pragma unroll
                for (int j = 0; j < A; ++j) {
                    if (ss[j] >= 0) {
                        const uint32_t w0 = o_fx + (uint32_t)ss[j] * 3u * W + l;
                        const double d = fx_to_double(p_dsm[w0], p_dsm[w0 + W], p_dsm[w0 + 2 * W], cnt, fx[j].inv_scale);
                        double *ps = &acc.sum[(uint64_t)ss[j] * B + b];
                        if (d != 0.0) __stcg(ps, __ldcg(ps) + d);
                    }
                    if (ms[j] >= 0)
                        __stcg((ulonglong2 *)acc.mm + (uint64_t)ms[j] * B + b, wmm[(uint32_t)ms[j] * W + l]);
                }
                continue;
            }
            atomicAdd(&acc.count[b], cnt);
#pragma unroll
            for (int j = 0; j < A; ++j) {
                if (ss[j] >= 0) {
                    const uint32_t w0 = o_fx + (uint32_t)ss[j] * 3u * W + l;
                    if (XS) {
                        xsum_add_fixed(acc.xs, B, ss[j], b, p_dsm[w0], p_dsm[w0 + W], p_dsm[w0 + 2 * W], cnt,
                                       FX_OFFSET, fx[j].F, s_xr);
                    } else {
                        const double d =
                            fx_to_double(p_dsm[w0], p_dsm[w0 + W], p_dsm[w0 + 2 * W], cnt, fx[j].inv_scale);
                        if (d != 0.0) atomicAdd(&acc.sum[(uint64_t)ss[j] * B + b], d);
                    }
                }
                if (ms[j] >= 0) {
                    const ulonglong2 m = wmm[(uint32_t)ms[j] * W + l];
                    ulonglong2 *g = (ulonglong2 *)acc.mm + (uint64_t)ms[j] * B + b;
                    if (m.x != ~0ull) atomicMin(&g->x, m.x);
                    if (m.y != ~0ull) atomicMin(&g->y, m.y);
                }
            }
        }
        __syncthreads();
    }
    if (XS) xr_publish(s_xr, acc.nsum, acc.xrange);  // (after the last tile's barrier)
}


// DATABIN_PART_TIMING=1 (diagnosis): CUDA events between the partition-route
// kernels of every execute; averages printed at exit.
namespace {
struct PartTiming {
    bool on = getenv("DATABIN_PART_TIMING") != nullptr;
    cudaEvent_t ev[8] = {};
    double ms[8] = {};
    int n = 0, k = 0;
    void mark(cudaStream_t s) {
        if (!on) return;
        if (!ev[k]) cudaEventCreate(&ev[k]);
        cudaEventRecord(ev[k++], s);
    }
    void collect() {
        if (!on || k < 2) return;
        cudaEventSynchronize(ev[k - 1]);
        for (int i = 1; i < k; ++i) {
            float m = 0;
            cudaEventElapsedTime(&m, ev[i - 1], ev[i]);
            ms[i] += m;
        }
        ++n;
        k = 0;
    }
    ~PartTiming() {
        if (!on || !n) return;
        fprintf(stderr, "[databin part timing] %d executes, ms per execute:", n);
        for (int i = 1; i < 8; ++i) fprintf(stderr, " %.4f", ms[i] / n);
        fprintf(stderr, "\n");
    }
};
PartTiming g_pt;
}  // namespace

// ---------------------------------------------------------------- host side
int part_bytes_per_bin(const Accum &acc) { return 4 + 12 * acc.nsum + 16 * acc.nmm; }

// scatter / refine: 512-thread CTAs, two per SM, so one CTA's barrier phases
// overlap the other's copies (one 1024-thread CTA per SM ran at ~2.6 TB/s)
constexpr int SC_THREADS = 512;
template <int A> struct PartCfg {
    static constexpr int PPT = A <= 1 ? 2 : 1;  // scatter: pairs per thread per batch
#ifndef PART_RPT1
#define PART_RPT1 5
#endif
    static constexpr int RPT = A <= 1 ? PART_RPT1 : 2;  // refine: rows per thread per batch
};
static size_t scatter_smem(int A, int ppt) {
    const size_t NP = (size_t)ppt * SC_THREADS, R = 2 * NP;
    return 2 * ((NP + 2) * 8 + NP * 16 * (size_t)A) + R * (8 * (size_t)A + 4 + 1) + (4 * 128 + 4) * 4;
}
static size_t refine_smem(int A, int rpt) {
    const size_t R = (size_t)rpt * SC_THREADS;
    return 2 * (R + 4) * (4 + 8 * (size_t)A) + R * (8 * (size_t)A + 4 + 1) + (4 * 128 + 4) * 4;
}
static size_t reduce_smem(const Accum &acc, const PartArgs &pa) {
    const size_t win = (size_t)pa.Wt * part_bytes_per_bin(acc), eh = (size_t)(pa.nl > 0 ? pa.nl : 1) * 2048 * 4;
    return win > eh ? win : eh;
}
static int a_class(int nl) { return nl == 0 ? 0 : (nl == 1 ? 1 : 4); }

// The partition route applies when: every loaded column shares the 16-byte
// phase, at most 4 attributes are read, n < 2^32 and the tiles fit.
bool part_plan(const Inputs &in, const Accum &acc, int ndim, int smem_optin, int sms, PartArgs *pa) {
    int nl = 0;
    for (int a = 0; a < in.nattr; ++a)
        if ((acc.load_mask >> a) & 1u) {
            if (nl == 4) return false;
            pa->lattr[nl++] = a;
        }
    pa->nl = nl;
    const uintptr_t ph = (uintptr_t)in.ax[0] & 15u;
    if (ph % 8) return false;
    for (int d = 0; d < ndim; ++d)
        if (((uintptr_t)in.ax[d] & 15u) != ph) return false;
    for (int j = 0; j < nl; ++j)
        if (((uintptr_t)in.at[pa->lattr[j]] & 15u) != ph) return false;
    const int64_t head = ph ? 1 : 0;
    if (in.n < 2 + head || in.n >= (1ll << 32) - 4) return false;
    const int64_t avail = (int64_t)smem_optin - 1024;
    const int64_t wmax = avail / part_bytes_per_bin(acc);
    if (wmax < 64) return false;
    const uint64_t B = acc.nbins;
    const uint64_t T = (B + wmax - 1) / wmax;
    if (T > 8192) return false;
    pa->T = (uint32_t)T;
    pa->Wt = (uint32_t)((B + T - 1) / T);
    pa->G1 = T <= 64 ? 1u : (uint32_t)((T + 63) / 64);
    pa->T1 = (uint32_t)((T + pa->G1 - 1) / pa->G1);
    pa->wt_div = udiv_make(pa->Wt);
    pa->wg_div = udiv_make(pa->Wt * pa->G1);
    pa->head = (int)head;
    pa->npairs = (uint32_t)((in.n - head) / 2);
    pa->tail = ((in.n - head) & 1) ? 1 : 0;
    pa->C = 2 * (uint32_t)sms;  // chunks: two 512-thread CTAs per SM in P1 and P3
    const int A = a_class(nl);
    if ((int64_t)scatter_smem(A, A <= 1 ? 2 : 1) > avail || (int64_t)refine_smem(A, A <= 1 ? PART_RPT1 : 2) > avail ||
        (int64_t)reduce_smem(acc, *pa) > avail || (int64_t)keys_smem(ndim, (uint32_t)T) + 33 * 4 > avail ||
        (int64_t)(pa->C + 1 + 33) * 4 > avail)
        return false;
    return true;
}

template <int D>
static cudaError_t launch_keys_d(const Geom &g, const Inputs &in, const Accum &acc, const PartArgs &pa, cudaStream_t s) {
    const size_t smem = keys_smem(D, pa.T);
    auto k = k_part_keys<D, SC_THREADS>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<pa.C, SC_THREADS, smem, s>>>(g, in, acc, pa);
    return cudaGetLastError();
}

template <int A>
static cudaError_t launch_part_tail(const Inputs &in, const Accum &acc, const PartArgs &pa, cudaStream_t s,
                                   int *launches) {
    cudaError_t e;
    const size_t sm0 = ((size_t)pa.C + 1 + 33) * 4;
    if ((e = cudaFuncSetAttribute(k_part_scan1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm0)) != cudaSuccess)
        return e;
    g_pt.mark(s);
    k_part_scan1<<<pa.T1, 1024, sm0, s>>>(pa);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const size_t sm1 = ((size_t)pa.T + 33) * 4;
    if ((e = cudaFuncSetAttribute(k_part_scan2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1)) != cudaSuccess)
        return e;
    k_part_scan2<<<1, 1024, sm1, s>>>(pa);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    constexpr int PPT = PartCfg<A>::PPT, RPT = PartCfg<A>::RPT;
    const size_t sm2 = scatter_smem(A, PPT);
    auto k2 = k_part_scatter<A, PPT, SC_THREADS>;
    if ((e = cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2)) != cudaSuccess) return e;
    g_pt.mark(s);
    k2<<<pa.C, SC_THREADS, sm2, s>>>(in, pa);
    g_pt.mark(s);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    *launches = 5;
    if (pa.G1 > 1) {
        const size_t smr = refine_smem(A, RPT);
        auto kr = k_part_refine<A, RPT, SC_THREADS>;
        if ((e = cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smr)) != cudaSuccess)
            return e;
        kr<<<pa.C, SC_THREADS, smr, s>>>(pa);
        g_pt.mark(s);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        *launches = 6;
    }
    const size_t sm3 = reduce_smem(acc, pa);
    auto k3 = acc.xs ? k_part_reduce<A, true> : k_part_reduce<A, false>;
    if ((e = cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm3)) != cudaSuccess) return e;
    k3<<<pa.C / 2, PART_THREADS, sm3, s>>>(acc, pa);  // one 1024-thread CTA per SM (C = 2 x SMs)
    g_pt.mark(s);
    g_pt.collect();
    return cudaGetLastError();
}

cudaError_t launch_partition(const Geom &g, const Inputs &in, const Accum &acc, const PartArgs &pa, cudaStream_t s,
                             int *launches) {
    cudaError_t e;
    g_pt.mark(s);
    switch (g.ndim) {
    case 1: e = launch_keys_d<1>(g, in, acc, pa, s); break;
    case 2: e = launch_keys_d<2>(g, in, acc, pa, s); break;
    default: e = launch_keys_d<3>(g, in, acc, pa, s); break;
    }
    if (e != cudaSuccess) return e;
    switch (a_class(pa.nl)) {
    case 0: return launch_part_tail<0>(in, acc, pa, s, launches);
    case 1: return launch_part_tail<1>(in, acc, pa, s, launches);
    default: return launch_part_tail<4>(in, acc, pa, s, launches);
    }
}

}  // namespace db
