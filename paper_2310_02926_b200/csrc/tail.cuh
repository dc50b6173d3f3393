// tail.cuh -- the last phase of an execute as device functions: finalize
// (a7) and the fused NVLink peer combine + finalize (a6 + a7), used by
// k_finalize (kernels.cu) and k_combine_peer (combine_peer.cu).  Grid-stride
// loops: any grid / block shape.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "db_internal.h"
#include "dev_common.cuh"
#include "xsum.cuh"

namespace db {

// ---------------------------------------------------------------- finalize [a7]
// BIN_SUM_EXACT: a bin's sum is its digit row rounded once (xsum.cuh), written
// into the sum output, then divided for the average.
__device__ __forceinline__ double exact_sum_of(const Accum &acc, int s, uint64_t b, unsigned long long cnt) {
    if (!cnt) return 0.0;
    const int klo = __ldcg(acc.xrange + 2 * s), nkhi = __ldcg(acc.xrange + 2 * s + 1);
    if (klo == XR_EMPTY) return 0.0;
    return xsum_round(acc.xs, acc.nbins, s, b, klo, -nkhi);
}

__device__ __forceinline__ void finalize_body(const Geom &g, const Accum &acc, Meta *meta, int variant) {
    DGeom G = load_geom(g, acc.bounds);
    const uint64_t nb = acc.nbins;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (G.ok && acc.xs) {
        for (int64_t b = t0; b < (int64_t)nb; b += stride) {
            const unsigned long long cnt = __ldcg(acc.count + b);
            for (int s = 0; s < acc.nsum; ++s) {
                const double sm = exact_sum_of(acc, s, (uint64_t)b, cnt);
                acc.sum[(uint64_t)s * nb + b] = sm;
                acc.oavg[(uint64_t)s * nb + b] = cnt ? __ddiv_rn(sm, (double)cnt) : __longlong_as_double(0x7ff8000000000000ll);
            }
            for (int s = 0; s < acc.nmm; ++s) {
                const ulonglong2 m = __ldcg((const ulonglong2 *)acc.mm + (uint64_t)s * nb + b);
                acc.omin[(uint64_t)s * nb + b] = cnt ? dec_total(m.x) : __longlong_as_double(0x7ff0000000000000ll);
                acc.omax[(uint64_t)s * nb + b] = cnt ? dec_total(~m.y) : __longlong_as_double((long long)0xfff0000000000000ull);
            }
        }
    } else if (G.ok && acc.nsum <= 1 && acc.nmm <= 1) {
        // common case: issue the bin's loads together (one latency, not three)
        for (int64_t b = t0; b < (int64_t)nb; b += stride) {
            const unsigned long long cnt = __ldcg(acc.count + b);
            const double sm = acc.nsum ? __ldcg(acc.sum + b) : 0.0;
            const ulonglong2 m = acc.nmm ? __ldcg((const ulonglong2 *)acc.mm + b) : make_ulonglong2(0ull, 0ull);
            if (acc.nsum) acc.oavg[b] = cnt ? __ddiv_rn(sm, (double)cnt) : __longlong_as_double(0x7ff8000000000000ll);
            if (acc.nmm) {
                acc.omin[b] = cnt ? dec_total(m.x) : __longlong_as_double(0x7ff0000000000000ll);
                acc.omax[b] = cnt ? dec_total(~m.y) : __longlong_as_double((long long)0xfff0000000000000ull);
            }
        }
    } else if (G.ok) {
        // several attributes: a chunk's loads are all issued before its stores
        // (the stores may alias the loaded arrays as far as the compiler knows,
        // so a load-divide-store loop waited for every load in turn)
        constexpr int FC = 8;
        for (int64_t b = t0; b < (int64_t)nb; b += stride) {
            const unsigned long long cnt = __ldcg(acc.count + b);
            const double dc = (double)cnt;
            for (int s0 = 0; s0 < acc.nsum; s0 += FC) {
                double sv[FC];
#pragma unroll
                for (int u = 0; u < FC; ++u)
                    sv[u] = s0 + u < acc.nsum ? __ldcg(acc.sum + (uint64_t)(s0 + u) * nb + b) : 0.0;
#pragma unroll
                for (int u = 0; u < FC; ++u)
                    if (s0 + u < acc.nsum)
                        acc.oavg[(uint64_t)(s0 + u) * nb + b] =
                            cnt ? __ddiv_rn(sv[u], dc) : __longlong_as_double(0x7ff8000000000000ll);
            }
            for (int s0 = 0; s0 < acc.nmm; s0 += FC) {
                ulonglong2 mv[FC];
#pragma unroll
                for (int u = 0; u < FC; ++u)
                    mv[u] = s0 + u < acc.nmm ? __ldcg((const ulonglong2 *)acc.mm + (uint64_t)(s0 + u) * nb + b)
                                             : make_ulonglong2(0ull, 0ull);
#pragma unroll
                for (int u = 0; u < FC; ++u)
                    if (s0 + u < acc.nmm) {
                        acc.omin[(uint64_t)(s0 + u) * nb + b] =
                            cnt ? dec_total(mv[u].x) : __longlong_as_double(0x7ff0000000000000ll);
                        acc.omax[(uint64_t)(s0 + u) * nb + b] =
                            cnt ? dec_total(~mv[u].y) : __longlong_as_double((long long)0xfff0000000000000ull);
                    }
            }
        }
    }
    if (t0 == 0) {
        meta->status = G.ok ? 0 : BIN_EDEGENERATE;
        meta->variant = variant;
        meta->n_in = __ldcg(acc.count + nb);
        meta->n_out = __ldcg(acc.count + nb + 1);
        for (int d = 0; d < 3; ++d) {
            meta->lo[d] = G.lo[d];
            meta->hi[d] = G.hi[d];
            meta->window[d] = acc.window[d];
            meta->window[3 + d] = acc.window[3 + d];
        }
        meta->done = 1;  // device memory; the host copies it on demand (bin_wait)
    }
    if (t0 < BIN_MAX_ATTR) acc.fxexp[t0] = 0u;  // for the next execute's sample on this slot
}

// ---------------------------------------------------------------- peer combine [a6 + a7]
constexpr long long SPIN_LIMIT_CYCLES = 4000000000ll;  // ~2 s

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    return ns;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Barrier words hold the execute's epoch; barrier B's word also carries
// PEER_FAIL when the publishing rank's combine did not complete (a CTA timed
// out at barrier A and skipped its bins), so every rank reports BIN_ENCCL.
constexpr unsigned long long PEER_FAIL = 1ull << 63;

// thread 0 of the calling CTA: wait until (flags[p] & ~PEER_FAIL) >= epoch for
// all p; false on timeout, *failed |= a peer published PEER_FAIL for `epoch`
__device__ __forceinline__ bool wait_all(const unsigned long long *flags, int nranks, unsigned long long epoch,
                                         bool *failed = nullptr) {
    const long long t0 = clock64();
    for (int p = 0; p < nranks; ++p) {
        unsigned long long v;
        while (((v = ld_acquire_sys(flags + p)) & ~PEER_FAIL) < epoch) {
            if (clock64() - t0 > SPIN_LIMIT_CYCLES) return false;
            __nanosleep(64);
        }
        if (failed && (v & PEER_FAIL) && (v & ~PEER_FAIL) == epoch) *failed = true;
    }
    return true;
}

// Common case (<= 1 summed and <= 1 min/max attribute, NR ranks): NR lanes
// per bin -- lane p loads rank p's partials, the group combines them with
// shuffles (sum folded in rank order), and lane q stores the results into
// rank q -- so a slice has NR x more requests in flight than a thread per bin
// (the combine is bound by outstanding NVLink requests, not link bandwidth:
// tools/microbench/peer_bench.cu).
template <int NR>
__device__ __forceinline__ void combine_slice_fast(const PeerSet &ps, uint64_t s0, uint64_t s1, bool hs, bool hm) {
    const double qnan = __longlong_as_double(0x7ff8000000000000ll);
    const double pinf = __longlong_as_double(0x7ff0000000000000ll);
    const double ninf = __longlong_as_double((long long)0xfff0000000000000ull);
    const unsigned lane = threadIdx.x & 31u, p = lane % NR;
    const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t span = (s1 - s0) * NR;
    for (uint64_t t = t0; t - lane < span; t += nt) {  // warp-uniform trip count (shuffles below)
        const bool valid = t < span;
        const uint64_t b = s0 + (valid ? t / NR : 0);
        const unsigned long long c = valid ? __ldcg(ps.count[p] + b) : 0ull;
        const double sv = (valid && hs) ? __ldcg(ps.sum[p] + b) : 0.0;
        const ulonglong2 m = (valid && hm) ? __ldcg((const ulonglong2 *)ps.mm[p] + b) : make_ulonglong2(~0ull, ~0ull);
        unsigned long long cnt = c, mn = m.x, nx = m.y;
        double sm = 0.0;  // rank-order fold from +0.0 (oracle partition mode)
        const unsigned g0 = lane - p;
#pragma unroll
        for (int q = 0; q < NR; ++q) sm = __dadd_rn(sm, __shfl_sync(0xffffffffu, sv, g0 + q));
#pragma unroll
        for (int o = 1; o < NR; o <<= 1) {
            cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
            const unsigned long long x = __shfl_xor_sync(0xffffffffu, mn, o);
            const unsigned long long y = __shfl_xor_sync(0xffffffffu, nx, o);
            mn = x < mn ? x : mn;
            nx = y < nx ? y : nx;
        }
        if (!valid) continue;
        const unsigned q = p;  // this lane stores into rank q
        ps.count[q][b] = cnt;
        if (hs) {
            ps.sum[q][b] = sm;
            ps.oavg[q][b] = cnt ? __ddiv_rn(sm, (double)cnt) : qnan;
        }
        if (hm) {
            ps.omin[q][b] = cnt ? dec_total(mn) : pinf;
            ps.omax[q][b] = cnt ? dec_total(~nx) : ninf;
        }
    }
}

// ---- TMA bulk-copy slice (cp.async.bulk): each CTA takes chunks of CB bins of
// the slice; one thread pulls every rank's count/sum/min-max chunk into
// shared memory (one mbarrier), the CTA reduces and finalizes there, and one
// thread pushes the five output chunks to every rank with bulk stores.  Bulk
// copies move 4-8 KB per request instead of 8-16 B per lane, so the slice is
// no longer bound by SM-issued NVLink requests.  Shared memory (u64 words):
// in [NR][count CB | sum CB | mm 2CB], out [count | sum | avg | min | max][CB].
#ifndef BIN_COMB_CB
#define BIN_COMB_CB 256
#endif
constexpr uint32_t COMB_CB = BIN_COMB_CB;  // bins per chunk (2 x 256 B per array per rank)

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
                 "r"((unsigned)__cvta_generic_to_shared(bar))
                 : "memory");
}
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(dst), "r"((unsigned)__cvta_generic_to_shared(src)), "r"(bytes)
                 : "memory");
}

template <int NR>
__device__ void combine_slice_bulk(const PeerSet &ps, uint64_t e0, uint64_t e1, bool hs, bool hm) {
    extern __shared__ __align__(128) unsigned long long cb_smem[];
    __shared__ __align__(8) uint64_t bar;
    constexpr uint32_t CB = COMB_CB, IN = 4 * CB;  // u64 words per rank
    unsigned long long *in = cb_smem, *out = cb_smem + NR * IN;
    const double qnan = __longlong_as_double(0x7ff8000000000000ll);
    const double pinf = __longlong_as_double(0x7ff0000000000000ll);
    const double ninf = __longlong_as_double((long long)0xfff0000000000000ull);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t parity = 0;
    const uint64_t nch = (e1 - e0 + CB - 1) / CB;
    for (uint64_t ch = blockIdx.x; ch < nch; ch += gridDim.x) {
        const uint64_t b0 = e0 + ch * CB;
        const uint32_t nb = (uint32_t)min((uint64_t)CB, e1 - b0);  // even
        if (threadIdx.x == 0) {
            const uint32_t bytes = NR * nb * 8u * (1u + (hs ? 1u : 0u) + (hm ? 2u : 0u));
            unsigned long long st;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 %0, [%1], %2;"
                         : "=l"(st) : "r"((unsigned)__cvta_generic_to_shared(&bar)), "r"(bytes) : "memory");
            (void)st;
#pragma unroll
            for (int p = 0; p < NR; ++p) {
                bulk_g2s(in + p * IN, ps.count[p] + b0, nb * 8u, &bar);
                if (hs) bulk_g2s(in + p * IN + CB, ps.sum[p] + b0, nb * 8u, &bar);
                if (hm) bulk_g2s(in + p * IN + 2 * CB, ps.mm[p] + 2 * b0, nb * 16u, &bar);
            }
        }
        {  // wait for the chunk (all threads)
            unsigned done = 0;
            while (!done) {
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(done) : "r"((unsigned)__cvta_generic_to_shared(&bar)), "r"(parity) : "memory");
            }
            parity ^= 1u;
        }
        for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) {
            unsigned long long cnt = 0, mn = ~0ull, nx = ~0ull;
            double sm = 0.0;  // rank-order fold from +0.0 (oracle partition mode)
#pragma unroll
            for (int p = 0; p < NR; ++p) {
                const unsigned long long *q = in + p * IN;
                cnt += q[i];
                if (hs) sm = __dadd_rn(sm, __longlong_as_double((long long)q[CB + i]));
                if (hm) {
                    const unsigned long long a = q[2 * CB + 2 * i], b = q[2 * CB + 2 * i + 1];
                    mn = a < mn ? a : mn;
                    nx = b < nx ? b : nx;
                }
            }
            out[i] = cnt;
            if (hs) {
                out[CB + i] = (unsigned long long)__double_as_longlong(sm);
                out[2 * CB + i] = (unsigned long long)__double_as_longlong(cnt ? __ddiv_rn(sm, (double)cnt) : qnan);
            }
            if (hm) {
                out[3 * CB + i] = (unsigned long long)__double_as_longlong(cnt ? dec_total(mn) : pinf);
                out[4 * CB + i] = (unsigned long long)__double_as_longlong(cnt ? dec_total(~nx) : ninf);
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy writes -> bulk copies
        __syncthreads();
        if (threadIdx.x == 0) {
#pragma unroll
            for (int q = 0; q < NR; ++q) {
                bulk_s2g(ps.count[q] + b0, out, nb * 8u);
                if (hs) {
                    bulk_s2g(ps.sum[q] + b0, out + CB, nb * 8u);
                    bulk_s2g(ps.oavg[q] + b0, out + 2 * CB, nb * 8u);
                }
                if (hm) {
                    bulk_s2g(ps.omin[q] + b0, out + 3 * CB, nb * 8u);
                    bulk_s2g(ps.omax[q] + b0, out + 4 * CB, nb * 8u);
                }
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem reusable
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {  // writes performed, and ordered before the generic-proxy flag stores
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        asm volatile("fence.proxy.async.global;" ::: "memory");
    }
}

// bulk: the slice uses TMA bulk copies (the kernel was launched with
// combine_bulk_smem(nranks) bytes of dynamic shared memory)
template <bool EXACT>
__device__ __forceinline__ void combine_peer_body(const Geom &g, const PeerSet &ps, int rank, int nranks,
                                                  unsigned long long epoch, Meta *meta, int variant, bool bulk) {
    __shared__ bool ok_s, last_s;
    const Accum &me = ps.me;
    const uint64_t B = me.nbins;
    // ---- barrier A: all partial accumulators complete
    if (threadIdx.x == 0) {
        if (blockIdx.x == 0) {
            meta->trace[0] = globaltimer();
            __threadfence_system();
            for (int p = 0; p < nranks; ++p) st_release_sys(ps.flags[p] + rank, epoch);  // flagsA[rank] on peer p
        }
        ok_s = wait_all(ps.flags[rank], nranks, epoch);
        if (!ok_s) atomicOr(ps.ctas_failed, 1u);  // this CTA skips its bins: the rank's combine failed
        if (blockIdx.x == 0) {
            meta->trace[1] = globaltimer();
            if (ok_s) {
                // n_in / n_out summed over the ranks now, while every rank's words are
                // final: after barrier B a peer may already re-zero them for its next
                // execute on this slot
                unsigned long long nin = 0, nout = 0;
                for (int p = 0; p < nranks; ++p) {
                    nin += __ldcg(ps.count[p] + B);
                    nout += __ldcg(ps.count[p] + B + 1);
                }
                meta->n_in = nin;
                meta->n_out = nout;
            }
        }
    }
    __syncthreads();
    const bool ok = ok_s;
    // ---- my slice: reduce over ranks, finalize, store into every rank
    const uint64_t s0 = (B * (uint64_t)rank) / nranks, s1 = (B * (uint64_t)(rank + 1)) / nranks;
    const int nsum = me.nsum, nmm = me.nmm;
    const double qnan = __longlong_as_double(0x7ff8000000000000ll);
    const double pinf = __longlong_as_double(0x7ff0000000000000ll);
    const double ninf = __longlong_as_double((long long)0xfff0000000000000ull);
    // exact sums: the union of the ranks' touched digit ranges, per summed attribute
    __shared__ int s_klo[BIN_MAX_ATTR], s_khi[BIN_MAX_ATTR];
    constexpr bool exact = EXACT;  // (a separate instance: the fast combine carries no digit code)
    if (exact && threadIdx.x < nsum) {
        int lo = XR_EMPTY, nhi = XR_EMPTY;
        for (int p = 0; p < nranks; ++p) {
            lo = min(lo, __ldcg(ps.xrange[p] + 2 * threadIdx.x));
            nhi = min(nhi, __ldcg(ps.xrange[p] + 2 * threadIdx.x + 1));
        }
        s_klo[threadIdx.x] = lo == XR_EMPTY ? 1 : lo;
        s_khi[threadIdx.x] = lo == XR_EMPTY ? 0 : -nhi;
    }
    if (exact) __syncthreads();
    auto generic = [&](uint64_t b) {
        unsigned long long cnt = 0;
        for (int p = 0; p < nranks; ++p) cnt += __ldcg(ps.count[p] + b);
        for (int q = 0; q < nranks; ++q) ps.count[q][b] = cnt;
        for (int s = 0; s < nsum; ++s) {
            double sm = 0.0;  // rank-order fold from +0.0 (oracle partition mode)
            if constexpr (EXACT) {  // digits add as integers over the ranks, then one rounding
                long long d[XD];
                const int klo = s_klo[s], khi = s_khi[s];
                for (int k = klo; k <= khi; ++k) {
                    long long a = 0;
                    for (int p = 0; p < nranks; ++p) a += __ldcg(ps.xs[p] + ((uint64_t)s * XD + k) * B + b);
                    d[k - klo] = a;
                }
                sm = cnt ? xsum_round_digits(d, klo, khi) : 0.0;
            } else
            for (int p = 0; p < nranks; ++p) sm = __dadd_rn(sm, __ldcg(ps.sum[p] + (uint64_t)s * B + b));
            const double avg = cnt ? __ddiv_rn(sm, (double)cnt) : qnan;
            for (int q = 0; q < nranks; ++q) {
                ps.sum[q][(uint64_t)s * B + b] = sm;
                ps.oavg[q][(uint64_t)s * B + b] = avg;
            }
        }
        for (int s = 0; s < nmm; ++s) {
            unsigned long long m = ~0ull, nx = ~0ull;
            for (int p = 0; p < nranks; ++p) {
                const ulonglong2 v = __ldcg((const ulonglong2 *)ps.mm[p] + (uint64_t)s * B + b);
                m = v.x < m ? v.x : m;
                nx = v.y < nx ? v.y : nx;
            }
            const double mn = cnt ? dec_total(m) : pinf, mx = cnt ? dec_total(~nx) : ninf;
            for (int q = 0; q < nranks; ++q) {
                ps.omin[q][(uint64_t)s * B + b] = mn;
                ps.omax[q][(uint64_t)s * B + b] = mx;
            }
        }
    };
    // fast path (common case): NR lanes per bin; else the generic per-bin loop
    const bool fastp = ok && !exact && nsum <= 1 && nmm <= 1 && (nranks == 2 || nranks == 4 || nranks == 8);
    if (bulk && fastp) {  // TMA bulk copies for the even-aligned body; the <= 2 edge bins below
        const uint64_t e0 = (s0 + 1) & ~1ull, e1 = s1 & ~1ull;
        if (e0 < e1) {
            if (nranks == 2) combine_slice_bulk<2>(ps, e0, e1, nsum == 1, nmm == 1);
            else if (nranks == 4) combine_slice_bulk<4>(ps, e0, e1, nsum == 1, nmm == 1);
            else combine_slice_bulk<8>(ps, e0, e1, nsum == 1, nmm == 1);
        }
        if (blockIdx.x == 0 && threadIdx.x < 2) {
            const uint64_t b = threadIdx.x == 0 ? s0 : e1;
            const bool edge = threadIdx.x == 0 ? (e0 < e1 ? s0 < e0 : false) : (e0 < e1 ? e1 < s1 : false);
            if (edge) generic(b);
            if (threadIdx.x == 0 && !(e0 < e1))
                for (uint64_t bb = s0; bb < s1; ++bb) generic(bb);
        }
    } else if (fastp && nranks == 2) combine_slice_fast<2>(ps, s0, s1, nsum == 1, nmm == 1);
    else if (fastp && nranks == 4) combine_slice_fast<4>(ps, s0, s1, nsum == 1, nmm == 1);
    else if (fastp && nranks == 8) combine_slice_fast<8>(ps, s0, s1, nsum == 1, nmm == 1);
    if (!fastp)
        for (uint64_t b = s0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; ok && b < s1;
             b += (uint64_t)gridDim.x * blockDim.x)
            generic(b);
    // ---- barrier B: every slice written everywhere
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) last_s = atomicAdd(ps.ctas_done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last_s) return;
    if (threadIdx.x == 0) {
        meta->trace[2] = globaltimer();
        *ps.ctas_done = 0u;  // reset for the next execute (stream-ordered)
        const bool failed = atomicExch(ps.ctas_failed, 0u) != 0u;  // some CTA of this rank timed out
        __threadfence_system();
        const unsigned long long fb = epoch | (failed ? PEER_FAIL : 0ull);
        for (int p = 0; p < nranks; ++p) st_release_sys(ps.flags[p] + 64 + rank, fb);  // flagsB
        bool peer_failed = false;
        const bool ok2 = !failed && wait_all(ps.flags[rank] + 64, nranks, epoch, &peer_failed) && !peer_failed;
        const DGeom G = load_geom(g, me.bounds);
        meta->status = !ok2 ? BIN_ENCCL : (G.ok ? 0 : BIN_EDEGENERATE);
        meta->variant = variant;
        for (int d = 0; d < 3; ++d) {
            meta->lo[d] = G.lo[d];
            meta->hi[d] = G.hi[d];
            meta->window[d] = me.window[d];
            meta->window[3 + d] = me.window[3 + d];
        }
        meta->done = 1;
        meta->trace[3] = globaltimer();
        for (int a = 0; a < BIN_MAX_ATTR; ++a) me.fxexp[a] = 0u;
    }
}

// ---------------------------------------------------------------- NVLS combine [a6 + a7]
// The same barriers and slice ownership as combine_peer_body, but the slice
// is reduced IN THE SWITCH: multimem.ld_reduce on the multicast address reads
// every rank's copy of a word and returns their sum / min (count Sum u64, sum
// Sum f64 -- order unspecified, reading R8 --, min/max Min u64, exact-sum digits
// Sum u64), and multimem.st writes the finalized values into every rank's
// arrays with one store.  Per rank and bin of its slice that is 8 B x words
// read and written once over NVLink instead of nranks times.
__device__ __forceinline__ unsigned long long mc_add_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double mc_add_f64(const double *p) {
    double v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ unsigned long long mc_min_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.min.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ int mc_min_s32(const int *p) {
    int v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.min.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void mc_st_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("multimem.st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void mc_st_f64(double *p, double v) {
    asm volatile("multimem.st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
// 16 bytes (two 64-bit words, bit patterns kept) to every rank in one request
__device__ __forceinline__ void mc_st_2x64(void *p, unsigned long long a, unsigned long long b) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p),
                 "f"(__uint_as_float((unsigned)a)), "f"(__uint_as_float((unsigned)(a >> 32))),
                 "f"(__uint_as_float((unsigned)b)), "f"(__uint_as_float((unsigned)(b >> 32)))
                 : "memory");
}

template <bool EXACT>
__device__ __forceinline__ void combine_nvls_body(const Geom &g, const PeerSet &ps, int rank, int nranks,
                                                  unsigned long long epoch, Meta *meta, int variant) {
    __shared__ bool ok_s, last_s;
    const Accum &me = ps.me;
    const uint64_t B = me.nbins;
    // ---- barrier A: all partial accumulators complete
    if (threadIdx.x == 0) {
        if (blockIdx.x == 0) {
            meta->trace[0] = globaltimer();
            __threadfence_system();
            for (int p = 0; p < nranks; ++p) st_release_sys(ps.flags[p] + rank, epoch);
        }
        ok_s = wait_all(ps.flags[rank], nranks, epoch);
        if (!ok_s) atomicOr(ps.ctas_failed, 1u);
        if (blockIdx.x == 0) {
            meta->trace[1] = globaltimer();
            if (ok_s) {  // summed over the ranks now (after barrier B a peer may re-zero them)
                meta->n_in = mc_add_u64(ps.mc_count + B);
                meta->n_out = mc_add_u64(ps.mc_count + B + 1);
            }
        }
    }
    __syncthreads();
    const bool ok = ok_s;
    const uint64_t s0 = (B * (uint64_t)rank) / nranks, s1 = (B * (uint64_t)(rank + 1)) / nranks;
    const int nsum = me.nsum, nmm = me.nmm;
    const double qnan = __longlong_as_double(0x7ff8000000000000ll);
    const double pinf = __longlong_as_double(0x7ff0000000000000ll);
    const double ninf = __longlong_as_double((long long)0xfff0000000000000ull);
    __shared__ int s_klo[BIN_MAX_ATTR], s_khi[BIN_MAX_ATTR];
    if (EXACT && threadIdx.x < nsum) {  // the union of the ranks' touched digit ranges
        const int lo = mc_min_s32(ps.mc_xrange + 2 * threadIdx.x), nhi = mc_min_s32(ps.mc_xrange + 2 * threadIdx.x + 1);
        s_klo[threadIdx.x] = lo == XR_EMPTY ? 1 : lo;
        s_khi[threadIdx.x] = lo == XR_EMPTY ? 0 : -nhi;
    }
    if (EXACT) __syncthreads();
    // bins in pairs (16-byte multimem stores: the switch's small-request rate,
    // not link bandwidth, bounds this loop); an unpaired edge bin on each side
    const uint64_t e0 = (s0 + 1) & ~1ull, e1 = s1 & ~1ull;
    auto one_pair = [&](uint64_t b, bool two) {
        const int H = two ? 2 : 1;
        if (!EXACT && nsum <= 1 && nmm <= 1) {  // common case: every load in flight before any store
            unsigned long long cnt[2] = {0ull, 0ull}, mn[2] = {~0ull, ~0ull}, nx[2] = {~0ull, ~0ull};
            double sm[2] = {0.0, 0.0};
            for (int h = 0; h < H; ++h) {
                cnt[h] = mc_add_u64(ps.mc_count + b + h);
                if (nsum) sm[h] = mc_add_f64(ps.mc_sum + b + h);
                if (nmm) {
                    mn[h] = mc_min_u64(ps.mc_mm + 2 * (b + h));
                    nx[h] = mc_min_u64(ps.mc_mm + 2 * (b + h) + 1);
                }
            }
            double av[2], lo[2], hi[2];
            for (int h = 0; h < 2; ++h) {
                av[h] = cnt[h] ? __ddiv_rn(sm[h], (double)cnt[h]) : qnan;
                lo[h] = cnt[h] ? dec_total(mn[h]) : pinf;
                hi[h] = cnt[h] ? dec_total(~nx[h]) : ninf;
            }
            if (two) {
                mc_st_2x64(ps.mc_count + b, cnt[0], cnt[1]);
                if (nsum) {
                    mc_st_2x64(ps.mc_sum + b, __double_as_longlong(sm[0]), __double_as_longlong(sm[1]));
                    mc_st_2x64(ps.mc_oavg + b, __double_as_longlong(av[0]), __double_as_longlong(av[1]));
                }
                if (nmm) {
                    mc_st_2x64(ps.mc_omin + b, __double_as_longlong(lo[0]), __double_as_longlong(lo[1]));
                    mc_st_2x64(ps.mc_omax + b, __double_as_longlong(hi[0]), __double_as_longlong(hi[1]));
                }
            } else {
                mc_st_u64(ps.mc_count + b, cnt[0]);
                if (nsum) mc_st_f64(ps.mc_sum + b, sm[0]), mc_st_f64(ps.mc_oavg + b, av[0]);
                if (nmm) mc_st_f64(ps.mc_omin + b, lo[0]), mc_st_f64(ps.mc_omax + b, hi[0]);
            }
            return;
        }
        unsigned long long cnt[2];
        cnt[0] = mc_add_u64(ps.mc_count + b);
        cnt[1] = two ? mc_add_u64(ps.mc_count + b + 1) : 0ull;
        if (two) mc_st_2x64(ps.mc_count + b, cnt[0], cnt[1]);
        else mc_st_u64(ps.mc_count + b, cnt[0]);
        for (int s = 0; s < nsum; ++s) {
            double sm[2], av[2];
            for (int h = 0; h < H; ++h) {
                if constexpr (EXACT) {  // digits add as integers in the switch, then one rounding
                    long long d[XD];
                    const int klo = s_klo[s], khi = s_khi[s];
                    for (int k = klo; k <= khi; ++k)
                        d[k - klo] = (long long)mc_add_u64((const unsigned long long *)ps.mc_xs +
                                                           ((uint64_t)s * XD + k) * B + b + h);
                    sm[h] = cnt[h] ? xsum_round_digits(d, klo, khi) : 0.0;
                } else {
                    sm[h] = mc_add_f64(ps.mc_sum + (uint64_t)s * B + b + h);
                }
                av[h] = cnt[h] ? __ddiv_rn(sm[h], (double)cnt[h]) : qnan;
            }
            double *ds = ps.mc_sum + (uint64_t)s * B + b, *da = ps.mc_oavg + (uint64_t)s * B + b;
            if (two) {
                mc_st_2x64(ds, __double_as_longlong(sm[0]), __double_as_longlong(sm[1]));
                mc_st_2x64(da, __double_as_longlong(av[0]), __double_as_longlong(av[1]));
            } else {
                mc_st_f64(ds, sm[0]);
                mc_st_f64(da, av[0]);
            }
        }
        for (int s = 0; s < nmm; ++s) {
            double mn[2], mx[2];
            for (int h = 0; h < (two ? 2 : 1); ++h) {
                const uint64_t w = 2 * ((uint64_t)s * B + b + h);
                const unsigned long long m = mc_min_u64(ps.mc_mm + w), nx = mc_min_u64(ps.mc_mm + w + 1);
                mn[h] = cnt[h] ? dec_total(m) : pinf;
                mx[h] = cnt[h] ? dec_total(~nx) : ninf;
            }
            double *dn = ps.mc_omin + (uint64_t)s * B + b, *dx = ps.mc_omax + (uint64_t)s * B + b;
            if (two) {
                mc_st_2x64(dn, __double_as_longlong(mn[0]), __double_as_longlong(mn[1]));
                mc_st_2x64(dx, __double_as_longlong(mx[0]), __double_as_longlong(mx[1]));
            } else {
                mc_st_f64(dn, mn[0]);
                mc_st_f64(dx, mx[0]);
            }
        }
    };
    if (ok && e0 < e1) {
        for (uint64_t j = e0 / 2 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < e1 / 2;
             j += (uint64_t)gridDim.x * blockDim.x)
            one_pair(2 * j, true);
    }
    if (ok && blockIdx.x == 0 && threadIdx.x < 2) {  // edge bins
        if (e0 < e1) {
            if (threadIdx.x == 0 && s0 < e0) one_pair(s0, false);
            if (threadIdx.x == 1 && e1 < s1) one_pair(e1, false);
        } else if (threadIdx.x == 0) {
            for (uint64_t b = s0; b < s1; ++b) one_pair(b, false);
        }
    }
    // ---- barrier B: every slice written everywhere
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) last_s = atomicAdd(ps.ctas_done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last_s) return;
    if (threadIdx.x == 0) {
        meta->trace[2] = globaltimer();
        *ps.ctas_done = 0u;
        const bool failed = atomicExch(ps.ctas_failed, 0u) != 0u;
        __threadfence_system();
        const unsigned long long fb = epoch | (failed ? PEER_FAIL : 0ull);
        for (int p = 0; p < nranks; ++p) st_release_sys(ps.flags[p] + 64 + rank, fb);
        bool peer_failed = false;
        const bool ok2 = !failed && wait_all(ps.flags[rank] + 64, nranks, epoch, &peer_failed) && !peer_failed;
        const DGeom G = load_geom(g, me.bounds);
        meta->status = !ok2 ? BIN_ENCCL : (G.ok ? 0 : BIN_EDEGENERATE);
        meta->variant = variant;
        for (int d = 0; d < 3; ++d) {
            meta->lo[d] = G.lo[d];
            meta->hi[d] = G.hi[d];
            meta->window[d] = me.window[d];
            meta->window[3 + d] = me.window[3 + d];
        }
        meta->done = 1;
        meta->trace[3] = globaltimer();
        for (int a = 0; a < BIN_MAX_ATTR; ++a) me.fxexp[a] = 0u;
    }
}

}  // namespace db
