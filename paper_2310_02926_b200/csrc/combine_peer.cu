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
#include "tail.cuh"

namespace db {

constexpr int COMB_THREADS = 256;

__global__ void __launch_bounds__(COMB_THREADS) k_combine_peer(Geom g, PeerSet ps, int rank, int nranks,
                                                               unsigned long long epoch, Meta *meta, int variant) {
    combine_peer_body(g, ps, rank, nranks, epoch, meta, variant);
}

cudaError_t launch_combine_peer(const Geom &g, const PeerSet &ps, int rank, int nranks, unsigned long long epoch,
                                Meta *meta, int variant, int deterministic, int sms, cudaStream_t s) {
    const uint64_t B = ps.me.nbins;
    const uint64_t slice = (B + nranks - 1) / nranks;
    uint64_t blocks = (slice * nranks + COMB_THREADS - 1) / COMB_THREADS;  // up to nranks lanes per bin
    if (blocks > (uint64_t)sms * 8) blocks = (uint64_t)sms * 8;
    if (blocks < 1) blocks = 1;
    (void)deterministic;
    k_combine_peer<<<(unsigned)blocks, COMB_THREADS, 0, s>>>(g, ps, rank, nranks, epoch, meta, variant);
    return cudaGetLastError();
}

}  // namespace db
