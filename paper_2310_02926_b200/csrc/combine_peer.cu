// combine_peer.cu -- the cross-rank combine (a6) fused with
// finalize (a7) into ONE kernel over NVLink peer memory.
//
// Every rank's slot accumulators (count, sum, min/max slots) and outputs are
// mapped into every other rank's address space with CUDA IPC at bin_init.
// k_combine_peer on rank r:
//   1. barrier A: publishes "my accumulator is complete" (system-scope release
//      store of the execute's epoch into each peer's flag word) and waits for
//      every peer's flag (acquire loads, bounded spin);
//   2. reduces its slice [r*B/N, (r+1)*B/N) of bins by loading all N ranks'
//      partial accumulators over NVLink (16-byte loads, coalesced), computes
//      count, sum (folded in rank order: bit-identical to the oracle's
//      partition mode when the partials are), min, max, avg, and stores the
//      final values of its slice into EVERY rank's output arrays -- a
//      reduce-scatter, the finalize and an all-gather in one pass;
//   3. barrier B (last CTA of the grid): completes only when every peer has
//      written its slice into this rank's outputs, so results are final when
//      the kernel is.
// Each bin's entries on all ranks are read and written only by its slice
// owner, so no two ranks race on a word.  The barriers spin on flags written
// by kernels on OTHER GPUs (one rank per GPU, checked at bin_init); a spin
// that exceeds ~2 s reports BIN_ENCCL instead of hanging.
#include <cuda_runtime.h>
#include <stdint.h>

#include "db_internal.h"
#include "dev_common.cuh"

namespace db {

constexpr int COMB_THREADS = 256;
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
__device__ bool wait_all(const unsigned long long *flags, int nranks, unsigned long long epoch) {
    const long long t0 = clock64();
    for (int p = 0; p < nranks; ++p) {
        while (ld_acquire_sys(flags + p) < epoch) {
            if (clock64() - t0 > SPIN_LIMIT_CYCLES) return false;
            __nanosleep(64);
        }
    }
    return true;
}

__global__ void __launch_bounds__(COMB_THREADS) k_combine_peer(Geom g, PeerSet ps, int rank, int nranks,
                                                               unsigned long long epoch, Meta *meta, int variant,
                                                               int deterministic) {
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
    (void)deterministic;
}

cudaError_t launch_combine_peer(const Geom &g, const PeerSet &ps, int rank, int nranks, unsigned long long epoch,
                                Meta *meta, int variant, int deterministic, int sms, cudaStream_t s) {
    const uint64_t B = ps.me.nbins;
    const uint64_t slice = (B + nranks - 1) / nranks;
    uint64_t blocks = (slice + COMB_THREADS - 1) / COMB_THREADS;
    if (blocks > (uint64_t)sms * 4) blocks = (uint64_t)sms * 4;
    if (blocks < 1) blocks = 1;
    k_combine_peer<<<(unsigned)blocks, COMB_THREADS, 0, s>>>(g, ps, rank, nranks, epoch, meta, variant, deterministic);
    return cudaGetLastError();
}

}  // namespace db
