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
#include <stdlib.h>

#include "db_internal.h"
#include "dev_common.cuh"
#include "tail.cuh"

namespace db {

constexpr int COMB_THREADS = 256;

template <bool EXACT>
__global__ void __launch_bounds__(COMB_THREADS) k_combine_peer(Geom g, PeerSet ps, int rank, int nranks,
                                                               unsigned long long epoch, Meta *meta, int variant,
                                                               int bulk) {
    combine_peer_body<EXACT>(g, ps, rank, nranks, epoch, meta, variant, bulk != 0);
}

template <bool EXACT>
__global__ void __launch_bounds__(COMB_THREADS) k_combine_nvls(Geom g, PeerSet ps, int rank, int nranks,
                                                               unsigned long long epoch, Meta *meta, int variant) {
    combine_nvls_body<EXACT>(g, ps, rank, nranks, epoch, meta, variant);
}

// One-device rank group (bin_execute_group): rank blockIdx.y runs the same
// body over its own peer set; the group's ranks all live in this launch.
template <bool EXACT>
__global__ void __launch_bounds__(COMB_THREADS) k_combine_group(Geom g, const GroupRank *gr, int nranks,
                                                                unsigned long long epoch, int variant, int bulk) {
    const GroupRank &r = gr[blockIdx.y];
    combine_peer_body<EXACT>(g, r.ps, (int)blockIdx.y, nranks, epoch, r.meta, variant, bulk != 0);
}

// dynamic shared memory of the bulk slice: NR ranks x 4 words + 5 output words per bin
static size_t combine_bulk_smem(int nranks) { return ((size_t)nranks * 4 + 5) * COMB_CB * 8; }

cudaError_t launch_combine_peer(const Geom &g, const PeerSet &ps, int rank, int nranks, unsigned long long epoch,
                                Meta *meta, int variant, int deterministic, int sms, cudaStream_t s) {
    const uint64_t B = ps.me.nbins;
    const uint64_t slice = (B + nranks - 1) / nranks;
    (void)deterministic;
    if (ps.mc_count) {  // NVLS: in-switch reduction, one thread per bin of the slice
        uint64_t blocks = (slice / 2 + COMB_THREADS - 1) / COMB_THREADS;  // a thread per bin pair
        if (blocks > (uint64_t)sms * 8) blocks = (uint64_t)sms * 8;
        if (blocks < 1) blocks = 1;
        if (ps.me.xs)
            k_combine_nvls<true><<<(unsigned)blocks, COMB_THREADS, 0, s>>>(g, ps, rank, nranks, epoch, meta, variant | 64);
        else
            k_combine_nvls<false><<<(unsigned)blocks, COMB_THREADS, 0, s>>>(g, ps, rank, nranks, epoch, meta, variant | 64);
        return cudaGetLastError();
    }
    static const bool no_bulk = getenv("DATABIN_COMBINE_BULK") && getenv("DATABIN_COMBINE_BULK")[0] == '0';
    const bool bulk = !no_bulk && !ps.me.xs && ps.me.nsum <= 1 && ps.me.nmm <= 1 &&
                      (nranks == 2 || nranks == 4 || nranks == 8);
    uint64_t blocks;
    size_t smem = 0;
    if (bulk) {
        smem = combine_bulk_smem(nranks);
        cudaError_t e = cudaFuncSetAttribute(k_combine_peer<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        blocks = (slice + COMB_CB - 1) / COMB_CB;  // one chunk of COMB_CB bins per CTA and step
        if (blocks > (uint64_t)sms * 4) blocks = (uint64_t)sms * 4;
    } else {
        blocks = (slice * nranks + COMB_THREADS - 1) / COMB_THREADS;  // up to nranks lanes per bin
        if (blocks > (uint64_t)sms * 8) blocks = (uint64_t)sms * 8;
    }
    if (blocks < 1) blocks = 1;
    if (ps.me.xs)
        k_combine_peer<true><<<(unsigned)blocks, COMB_THREADS, smem, s>>>(g, ps, rank, nranks, epoch, meta, variant, 0);
    else
        k_combine_peer<false><<<(unsigned)blocks, COMB_THREADS, smem, s>>>(g, ps, rank, nranks, epoch, meta, variant,
                                                                           bulk ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_combine_group(const Geom &g, const GroupRank *dev_ranks, const Accum &acc0, int nranks,
                                 unsigned long long epoch, int variant, int sms, cudaStream_t s) {
    const uint64_t B = acc0.nbins;
    const uint64_t slice = (B + nranks - 1) / nranks;
    static const bool no_bulk = getenv("DATABIN_COMBINE_BULK") && getenv("DATABIN_COMBINE_BULK")[0] == '0';
    const bool bulk = !no_bulk && !acc0.xs && acc0.nsum <= 1 && acc0.nmm <= 1 &&
                      (nranks == 2 || nranks == 4 || nranks == 8);
    // the barriers spin inside this launch: every CTA of every rank must be
    // resident at once, so at most one CTA per SM in total (<= 75 KB of shared
    // memory and 256 threads each: any CTA fits an SM on its own)
    uint64_t per_rank = (uint64_t)(sms / nranks);
    if (per_rank < 1) per_rank = 1;
    uint64_t want = bulk ? (slice + COMB_CB - 1) / COMB_CB : (slice * nranks + COMB_THREADS - 1) / COMB_THREADS;
    const uint64_t blocks = want < 1 ? 1 : (want < per_rank ? want : per_rank);
    size_t smem = 0;
    if (bulk) {
        smem = combine_bulk_smem(nranks);
        cudaError_t e = cudaFuncSetAttribute(k_combine_group<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const dim3 grid((unsigned)blocks, (unsigned)nranks);
    if (acc0.xs)
        k_combine_group<true><<<grid, COMB_THREADS, 0, s>>>(g, dev_ranks, nranks, epoch, variant, 0);
    else
        k_combine_group<false><<<grid, COMB_THREADS, smem, s>>>(g, dev_ranks, nranks, epoch, variant, bulk ? 1 : 0);
    return cudaGetLastError();
}

}  // namespace db
