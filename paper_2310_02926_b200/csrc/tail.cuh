// tail.cuh -- the last phase of an execute as device functions: finalize
// (a7) and the fused NVLink peer combine + finalize (a6 + a7), used by
// k_finalize (kernels.cu) and k_combine_peer (combine_peer.cu).  Grid-stride
// loops: any grid / block shape.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "db_internal.h"
#include "dev_common.cuh"

namespace db {

// ---------------------------------------------------------------- finalize [a7]
__device__ __forceinline__ void finalize_body(const Geom &g, const Accum &acc, Meta *meta, int variant) {
    DGeom G = load_geom(g, acc.bounds);
    const uint64_t nb = acc.nbins;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (G.ok && acc.nsum <= 1 && acc.nmm <= 1) {
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
        for (int64_t b = t0; b < (int64_t)nb; b += stride) {
            const unsigned long long cnt = __ldcg(acc.count + b);
            const double dc = (double)cnt;
            for (int s = 0; s < acc.nsum; ++s) {
                const double sm = __ldcg(acc.sum + (uint64_t)s * nb + b);
                acc.oavg[(uint64_t)s * nb + b] = cnt ? __ddiv_rn(sm, dc) : __longlong_as_double(0x7ff8000000000000ll);
            }
            for (int s = 0; s < acc.nmm; ++s) {
                const ulonglong2 m = __ldcg((const ulonglong2 *)acc.mm + (uint64_t)s * nb + b);
                acc.omin[(uint64_t)s * nb + b] = cnt ? dec_total(m.x) : __longlong_as_double(0x7ff0000000000000ll);
                acc.omax[(uint64_t)s * nb + b] = cnt ? dec_total(~m.y) : __longlong_as_double((long long)0xfff0000000000000ull);
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
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// thread 0 of the calling CTA: wait until flags[p*stride] >= epoch for all p
__device__ __forceinline__ bool wait_all(const unsigned long long *flags, int nranks, unsigned long long epoch) {
    const long long t0 = clock64();
    for (int p = 0; p < nranks; ++p) {
        while (ld_acquire_sys(flags + p) < epoch) {
            if (clock64() - t0 > SPIN_LIMIT_CYCLES) return false;
            __nanosleep(64);
        }
    }
    return true;
}

__device__ __forceinline__ void combine_peer_body(const Geom &g, const PeerSet &ps, int rank, int nranks,
                                                  unsigned long long epoch, Meta *meta, int variant) {
    __shared__ bool ok_s, last_s;
    const Accum &me = ps.me;
    const uint64_t B = me.nbins;
    // ---- barrier A: all partial accumulators complete
    if (threadIdx.x == 0) {
        if (blockIdx.x == 0) {
            __threadfence_system();
            for (int p = 0; p < nranks; ++p) st_release_sys(ps.flags[p] + rank, epoch);  // flagsA[rank] on peer p
        }
        ok_s = wait_all(ps.flags[rank], nranks, epoch);
    }
    __syncthreads();
    const bool ok = ok_s;
    // ---- my slice: reduce over ranks, finalize, store into every rank
    const uint64_t s0 = (B * (uint64_t)rank) / nranks, s1 = (B * (uint64_t)(rank + 1)) / nranks;
    const int nsum = me.nsum, nmm = me.nmm;
    const double qnan = __longlong_as_double(0x7ff8000000000000ll);
    const double pinf = __longlong_as_double(0x7ff0000000000000ll);
    const double ninf = __longlong_as_double((long long)0xfff0000000000000ull);
    for (uint64_t b = s0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; ok && b < s1;
         b += (uint64_t)gridDim.x * blockDim.x) {
        unsigned long long cnt = 0;
        for (int p = 0; p < nranks; ++p) cnt += __ldcg(ps.count[p] + b);
        for (int q = 0; q < nranks; ++q) ps.count[q][b] = cnt;
        for (int s = 0; s < nsum; ++s) {
            double sm = 0.0;  // rank-order fold from +0.0 (oracle partition mode)
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
    }
    // ---- barrier B: every slice written everywhere
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) last_s = atomicAdd(ps.ctas_done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last_s) return;
    if (threadIdx.x == 0) {
        *ps.ctas_done = 0u;  // reset for the next execute (stream-ordered)
        __threadfence_system();
        for (int p = 0; p < nranks; ++p) st_release_sys(ps.flags[p] + 64 + rank, epoch);  // flagsB
        const bool ok2 = ok && wait_all(ps.flags[rank] + 64, nranks, epoch);
        // n_in / n_out (summed over ranks) and the result meta
        unsigned long long nin = 0, nout = 0;
        for (int p = 0; p < nranks; ++p) {
            nin += __ldcg(ps.count[p] + B);
            nout += __ldcg(ps.count[p] + B + 1);
        }
        const DGeom G = load_geom(g, me.bounds);
        meta->status = !ok2 ? BIN_ENCCL : (G.ok ? 0 : BIN_EDEGENERATE);
        meta->variant = variant;
        meta->n_in = nin;
        meta->n_out = nout;
        for (int d = 0; d < 3; ++d) {
            meta->lo[d] = G.lo[d];
            meta->hi[d] = G.hi[d];
            meta->window[d] = me.window[d];
            meta->window[3 + d] = me.window[3 + d];
        }
        meta->done = 1;
        for (int a = 0; a < BIN_MAX_ATTR; ++a) me.fxexp[a] = 0u;
    }
}

}  // namespace db
