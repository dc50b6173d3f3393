// db_internal.h -- internal declarations of libdatabin (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include <nccl.h>

#include "../../include/databin.h"

namespace db {

// ---------------------------------------------------------------- errors
int set_error(int code, const char *fmt, ...);
int cuda_error(cudaError_t e, const char *what);
#define DB_CUDA(expr)                                         \
    do {                                                      \
        cudaError_t e_ = (expr);                              \
        if (e_ != cudaSuccess) return ::db::cuda_error(e_, #expr); \
    } while (0)

// checks one bin_spec_t (BIN_EINVAL / BIN_ENOTSUP with a message), *nbins = prod(res)
int validate_spec(const bin_spec_t *sp, uint64_t *nbins);

// ---------------------------------------------------------------- allocator
void *dev_alloc(size_t bytes, int device, cudaStream_t stream, bool async);
void dev_free(void *p, int device, cudaStream_t stream, bool async);
void *host_alloc(size_t bytes, bool pinned);
void host_free(void *p, bool pinned);
void *uva_alloc(size_t bytes);
void uva_free(void *p);
void count_alloc(int64_t bytes);
void count_free(int64_t bytes);

// RAII device switch
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (dev >= 0 && dev != prev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

}  // namespace db

// ---------------------------------------------------------------- array handle
struct bin_array {
    std::atomic<int> refs{1};
    void *ptr = nullptr;
    int64_t n = 0;
    int32_t dtype = BIN_F64;
    int32_t device = -1;  // -1 host
    bin_allocator_t alloc = BIN_ALLOC_EXTERNAL;
    cudaStream_t stream = nullptr;
    bin_stream_mode_t mode = BIN_SYNC;
    bool owned = false;  // library frees ptr with `alloc`
    void (*release)(void *, void *) = nullptr;
    void *release_ctx = nullptr;
    bin_array *source = nullptr;  // views keep their source alive
    // library work reading/writing this memory: the last event recorded on each
    // (device, stream) that used it -- release/synchronize wait for all of them
    // (one event per array would cover only the most recent user)
    struct Use {
        int device;
        cudaStream_t stream;
        cudaEvent_t ev;
    };
    std::vector<Use> uses;
    std::mutex mu;
};

namespace db {
// records an event on `s` (on device `dev`) marking library work that reads `a`
int array_mark_use(bin_array *a, cudaStream_t s, int dev);
bool is_device_memory(const bin_array *a);
}  // namespace db

// ---------------------------------------------------------------- kernels
namespace db {

constexpr int XD_DIGITS = 66;  // exact-sum digits per (summed attribute, bin): xsum.cuh XD

struct Geom {
    int32_t ndim;
    int32_t res[3];
    int32_t bounds_auto;
    double lo[3], hi[3];
};

// Meta block written by the finalize kernel into mapped pinned host memory.
struct Meta {
    int32_t status;  // 0 ok, BIN_EDEGENERATE
    int32_t variant;
    uint64_t n_in, n_out;
    double lo[3], hi[3];
    int32_t window[6];  // origin[3], extent[3]
    int32_t done;
    int32_t pad;
    uint64_t trace[4];  // peer combine: %globaltimer at entry, after barrier A, last CTA done, after barrier B
};

struct Accum {
    unsigned long long *count;  // nbins + 2 (n_in, n_out)
    double *sum;                // nsum * nbins
    unsigned long long *mm;     // nmm * nbins * 2: {enc(min), ~enc(max)}
    unsigned long long *bounds; // 2*ndim: {enc(lo_d)..., ~enc(hi_d)...}
    int32_t *window;            // 6 ints: origin[3], extent[3]
    uint32_t *fxexp;            // 16: max biased exponent of each summed attribute over the sample
    double *omin, *omax, *oavg; // outputs
    long long *xs;              // BIN_SUM_EXACT: nsum x XD x nbins carry-save digits (xsum.cuh), else nullptr
    int32_t *xrange;            // BIN_SUM_EXACT: 2 * nsum {min digit, -max digit} touched by the slot's
                                // last execute (init zeroes them, then resets the range)
    uint64_t nbins;
    int32_t nsum, nmm;
    uint32_t sum_mask, mm_mask, load_mask;
};

struct Inputs {
    const double *ax[3];
    const double *at[BIN_MAX_ATTR];
    int64_t n;
    int32_t nattr;
};

struct LaunchCfg {
    int sms;
    int smem_optin;  // bytes per block
};

// Each returns cudaError_t of the launch.
cudaError_t launch_init(const Geom &g, const Inputs &in, const Accum &acc, int wcap, bool choose_window,
                        cudaStream_t s);
cudaError_t launch_bounds(const Geom &g, const Inputs &in, const Accum &acc, const LaunchCfg &lc,
                          cudaStream_t s);
cudaError_t launch_window(const Geom &g, const Inputs &in, const Accum &acc, int wcap, cudaStream_t s);
cudaError_t launch_bin_general(const Geom &g, const Inputs &in, const Accum &acc, const LaunchCfg &lc, int smem,
                               cudaStream_t s);
// wcache: per-CTA window + fixed-point exponent (8 ints per CTA) written when
// reuse == 0, read instead of sampling when reuse != 0
// ktrace (DATABIN_TRACE, else nullptr): per-CTA %globaltimer at start, loop
// start, loop end, flush end (4 u64 per CTA)
cudaError_t launch_bin_fast(const Geom &g, const Inputs &in, const Accum &acc, const LaunchCfg &lc, int smem,
                            int wcap, int32_t *wcache, int reuse, unsigned long long *ktrace, cudaStream_t s);
bool fast_eligible(const Inputs &in, const Accum &acc, int ndim);
int fast_queue_bytes(bool exact);  // k_bin_fast shared memory past the window
cudaError_t launch_finalize(const Geom &g, const Accum &acc, Meta *meta_dev, int64_t n_rows_local,
                            int variant, cudaStream_t s);
// bytes of shared memory per window bin
int window_bytes_per_bin(const Accum &acc);
int fast_window_bytes_per_bin(const Accum &acc);  // k_bin_fast's window (bin_fast.cu)


// partition route (bin_part.cu): rows grouped by tile of Wt bins, then
// accumulated tile by tile in shared memory
// x / d for a divisor fixed per launch: t = umulhi(x, m), q = (t + ((x - t) >> s1)) >> s2
// (the branch-free round-up method; exact for every 32-bit x and d >= 1)
struct UDiv {
    uint32_t m, s1, s2;
};
inline UDiv udiv_make(uint32_t d) {
    uint32_t l = 0;
    while (l < 32 && (1ull << l) < d) ++l;  // ceil(log2 d)
    UDiv u;
    u.m = (uint32_t)((((1ull << 32) * ((1ull << l) - d)) / d) + 1);
    u.s1 = l < 1 ? l : 1;
    u.s2 = l > 1 ? l - 1 : 0;
    return u;
}
struct PartArgs {
    uint32_t *keys;    // [2*npairs + 2] bin index per row slot, ~0u outside
    uint32_t *cnt;     // [T][C] rows of chunk c in tile t -> exclusive prefix over c
    uint32_t *tot;     // [T] rows per tile
    uint32_t *tstart;  // [T + 1] first grouped row of each tile
    uint32_t *off1;    // [T1][C + 1] rows of super-tile s from chunks < c
    uint32_t *skey;    // [cap] bin index of the rows grouped by tile
    double *sval;      // [nl][cap] their attribute values
    uint32_t *xkey;    // [cap] rows grouped by super-tile (G1 > 1 only)
    double *xval;      // [nl][cap]
    uint64_t cap;
    uint32_t npairs;
    int32_t head, tail;
    uint32_t Wt, T, C;  // bins per tile, tiles, chunks (CTAs of P1 and P3)
    uint32_t G1, T1;    // tiles per super-tile (1: one level), super-tiles
    UDiv wt_div, wg_div;  // / Wt and / (Wt * G1)
    int32_t nl;         // attributes read (<= 4) and which
    int32_t lattr[4];
};
bool part_plan(const Inputs &in, const Accum &acc, int ndim, int smem_optin, int sms, PartArgs *pa);
cudaError_t launch_partition(const Geom &g, const Inputs &in, const Accum &acc, const PartArgs &pa, cudaStream_t s,
                             int *launches);
cudaError_t launch_probe(const Geom &g, const Inputs &in, const Accum &acc, int wcap, int32_t *out, cudaStream_t s);

// fused NVLink combine + finalize (combine_peer.cu)
constexpr int PEER_MAX = 16;  // ranks on the node (barrier words hold up to 64)
struct PeerSet {
    Accum me;  // this rank's slot (local pointers)
    unsigned long long *count[PEER_MAX];  // every rank's slot arrays, mapped here (CUDA IPC)
    double *sum[PEER_MAX];
    unsigned long long *mm[PEER_MAX];
    double *omin[PEER_MAX], *omax[PEER_MAX], *oavg[PEER_MAX];
    long long *xs[PEER_MAX];              // BIN_SUM_EXACT: every rank's digit rows and ranges
    int32_t *xrange[PEER_MAX];
    unsigned long long *flags[PEER_MAX];  // every rank's barrier words [A: 0..63][B: 64..127]
    unsigned *ctas_done;                  // this rank's last-CTA counter
    unsigned *ctas_failed;                // nonzero: a CTA of this rank timed out at barrier A
    // NVLS: multicast addresses of this slot's arrays (the same offsets on every
    // rank); mc_count == nullptr when the handle has no NVLS region
    unsigned long long *mc_count;
    double *mc_sum;
    unsigned long long *mc_mm;
    double *mc_omin, *mc_omax, *mc_oavg;
    long long *mc_xs;
    int32_t *mc_xrange;
};
cudaError_t launch_combine_peer(const Geom &g, const PeerSet &ps, int rank, int nranks, unsigned long long epoch,
                                Meta *meta, int variant, int deterministic, int sms, cudaStream_t s);

// NVLS multicast memory (nvls.cpp): unicast + multicast mappings of one region
struct NvlsRegion {
    void *uc = nullptr, *mc = nullptr;
    size_t size = 0;
    unsigned long long mem = 0, mch = 0;  // CUmemGenericAllocationHandle
    int device = -1;
    bool bound = false;
};
bool nvls_available(int device);
bool nvls_setup(size_t bytes, int rank, int nranks, int device, ncclComm_t comm, cudaStream_t s,
                const void *nccl_id128, NvlsRegion *out);
void nvls_free(NvlsRegion &r);
// a rank group on one device: the same combine body for all ranks in one launch
// (blockIdx.y = rank); every CTA co-resides (<= sms CTAs in total)
struct GroupRank {
    PeerSet ps;
    Meta *meta;
};
cudaError_t launch_combine_group(const Geom &g, const GroupRank *dev_ranks, const Accum &acc0, int nranks,
                                 unsigned long long epoch, int variant, int sms, cudaStream_t s);

// deterministic mode (sort-based, bit-exact vs the sequential oracle)
struct DetScratch {
    uint32_t *keys = nullptr, *keys_alt = nullptr;   // bin index per row (or ~0 for outside)
    uint32_t *rows = nullptr, *rows_alt = nullptr;   // row index permutation
    uint32_t *hist = nullptr;                        // digit histograms
    uint32_t *offsets = nullptr;                     // bin segment starts (nbins + 1)
    int64_t cap_rows = 0;
    int64_t cap_hist = 0;
    uint64_t cap_bins = 0;
    int device = -1;
};
cudaError_t launch_deterministic(const Geom &g, const Inputs &in, const Accum &acc, DetScratch &ds,
                                 const LaunchCfg &lc, cudaStream_t s, int *launches);
void free_det_scratch(DetScratch &ds);
cudaError_t launch_rank_fold(const double *gathered, int nranks, uint64_t len, double *sum, int sms, cudaStream_t s);
int ensure_det_scratch(DetScratch &ds, int64_t n, uint64_t nbins, int device, int sms);


// fused multi-operator binning (multi.cu): K instances over one column list
constexpr int MULTI_MAX_OPS = BIN_MULTI_MAX_OPS;
constexpr int MULTI_MAX_COLS = BIN_MULTI_MAX_COLS;
struct MultiOp {
    Geom g;
    Accum acc;   // count/sum/mm/bounds/outputs of this instance inside the slot allocation
    Meta *meta;  // device
    int32_t axc[3];
    int32_t atc[BIN_MAX_ATTR];
    int32_t nattr;
    uint32_t *flt;  // min/max filter: [bin][chunk of 8 attributes][hi32(enc min), hi32(~enc max)] (64 B), or nullptr
    int32_t nfc;    // filter chunks per bin (ceil(nattr / 8) when the instance has min/max, else 0)
};
struct MultiArgs {
    const double *col[MULTI_MAX_COLS];
    int64_t n;
    int32_t ncols, nops;
    int32_t k0, k1;         // instances [k0, k1) of this accumulate launch (L2-sized group)
    uint32_t used_cols;     // columns any instance reads
    uint32_t bound_cols;    // columns some auto-bounded instance takes bounds of
    int32_t use_flt;        // min/max filter lines on (off while rows are few per bin: nearly every row is a first touch)
    const MultiOp *ops;     // device array [nops]
};
cudaError_t launch_multi_init(const MultiArgs &a, uint64_t max_work, cudaStream_t s);
cudaError_t launch_multi_bounds(const MultiArgs &a, const LaunchCfg &lc, cudaStream_t s);
cudaError_t launch_multi_bin(const MultiArgs &a, const LaunchCfg &lc, cudaStream_t s);
cudaError_t launch_multi_finalize(const MultiArgs &a, uint64_t max_bins, cudaStream_t s);
}  // namespace db
