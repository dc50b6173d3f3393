// handle.cpp -- the DataBin operator instance: placement and execution
// method (Sec. 3), input view resolution (a1), the phase
// sequence of one execute, the NCCL cross-rank combine (a6)
// and results.
#include <cuda_runtime.h>
#include <math.h>
#include <nccl.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "db_internal.h"

using namespace db;

namespace {

enum { EV_STAGE = 0, EV_INIT0, EV_INIT1, EV_BOUNDS1, EV_WINDOW1, EV_BIN1, EV_COMBINE1, EV_FINAL1, EV_N };

struct Slot {
    Accum acc{};
    unsigned char *base = nullptr;  // the slot's single device allocation (IPC-exported in peer mode)
    bool external = false;          // base lies in the handle's NVLS region (not cudaMalloc'ed)
    PeerSet peers{};
    Meta *meta_h = nullptr, *meta_d = nullptr;
    cudaEvent_t done = nullptr, released = nullptr, zeroed = nullptr;
    cudaEvent_t binned = nullptr;  // rank group: this rank's accumulate is complete (bin_execute_group)
    bool staged_any = false;       // rank group: the execute staged inputs (tail deferred to the group)
    bool used_before = false;  // a previous execute used this slot (its done event is valid)
    cudaEvent_t ev[EV_N] = {};
    bool recd[EV_N] = {};  // which events this execute recorded (profiling)
    bool prof_pending = false;
    bool meta_valid = false;
    uint64_t ticket = 0;
    bool used = false;
    cudaStream_t stream = nullptr;
    int launches = 0;
    int bin_launches = 0;
    int variant = 0;
    size_t dev_bytes = 0;
};

struct Stage {
    void *p = nullptr;
    size_t bytes = 0;
};

}  // namespace

// A rank group on one device (bin_init_group): P handles whose combine is the
// fused peer combine + finalize over the group's slot arrays, launched once
// for all P ranks (grid.y = rank) after every rank has binned.
struct bin_group {
    int nranks = 0;
    int device = 0;
    std::vector<bin_handle *> member;  // rank -> handle (nullptr once finalized)
    GroupRank *dev = nullptr;          // [2 slots][nranks] peer sets + metas (device)
    cudaStream_t stream = nullptr;     // the combine's stream
    cudaEvent_t done[2] = {};
    int alive = 0;
};

struct bin_handle {
    bin_spec_t spec{};
    bin_placement_t place{};
    int rank = 0, nranks = 1;
    int device = 0;
    ncclComm_t comm = nullptr;
    cudaStream_t side = nullptr;
    cudaStream_t meta_stream = nullptr;
    cudaStream_t copy = nullptr;  // staging copies (host, peer, snapshot)
    cudaStream_t prep = nullptr;  // accumulator identities of the next slot (off the critical path)
    Slot slot[2];
    uint64_t next_ticket = 1;
    Stage stage[2][BIN_MAX_DIM + BIN_MAX_ATTR];
    cudaEvent_t producer_ev[BIN_MAX_DIM + BIN_MAX_ATTR] = {};
    LaunchCfg lc{};
    int wcap = 0, smem_bytes = 0;
    uint64_t nbins = 1;
    int nsum = 0, nmm = 0;
    uint32_t sum_mask = 0, mm_mask = 0, load_mask = 0;
    bool prof = false;
    bin_profile_t pacc{};
    cudaStream_t last = nullptr;
    DetScratch det;
    bool peer = false;                       // fused NVLink combine (combine_peer.cu) instead of NCCL
    unsigned long long *flags = nullptr;     // this rank's barrier words (IPC-exported)
    unsigned *ctas_done = nullptr;
    std::vector<void *> opened;              // peer mappings to close at finalize
    double *gather = nullptr;  // deterministic multi-rank: nranks x nsum x nbins partial sums
    size_t gather_bytes = 0;
    // accumulate route (BIN_ROUTE_*): auto = chosen by the k_probe sample
    int route = 0;                  // 0 not yet chosen, else BIN_ROUTE_WINDOW / BIN_ROUTE_PARTITION
    int32_t *probe_d = nullptr;     // k_probe output: window[6] + rows in box, rows inside
    int32_t *probe_h = nullptr;     // pinned mirror
    cudaEvent_t probe_ev = nullptr;
    bool probe_inflight = false;
    int since_probe = 0;
    int32_t *wcache = nullptr;  // k_bin_fast per-CTA windows [sms][8] (reused across executes)
    unsigned long long *ktrace = nullptr;  // DATABIN_TRACE: k_bin_fast per-CTA phase timestamps [sms][4]
    int64_t wcache_n = -1;
    int64_t wcache_age = 0;
    unsigned char *part_base = nullptr;  // partition-route scratch (grown on demand)
    size_t part_bytes = 0;
    bin_group *group = nullptr;  // member of a one-device rank group (bin_init_group)
    NvlsRegion nvls;             // multicast-bound memory holding both slots (NVLS combine)
    bool finalized = false;
};

// The window route holds a row in shared memory only if it falls in the CTA's
// hot window; with less than this fraction of the sampled rows in the best
// window the partition route (bin_part.cu) moves fewer L2 reductions per row.
static double route_coverage() {
    const char *e = getenv("DATABIN_ROUTE_COVERAGE");
    return e ? atof(e) : 0.5;
}
constexpr int ROUTE_REPROBE = 64;  // executes between asynchronous re-checks
constexpr int WINDOW_RESAMPLE = 16;  // k_bin_fast executes between per-CTA window samples

static int probe_route(const int32_t *p) {
    return (p[7] > 0 && (double)p[6] < route_coverage() * (double)p[7]) ? BIN_ROUTE_PARTITION : BIN_ROUTE_WINDOW;
}

// Carves the partition scratch (256-byte aligned pieces): keys [n+2] |
// cnt [T*C] | tot [T] | tstart [T+1] | off1 [T1*(C+1)] | skey [n] |
// sval [nl][cap] | (two-level) xkey [n] | xval [nl][cap], cap = n rounded up to 4.
static int ensure_part_scratch(bin_handle *h, int64_t n, PartArgs &pa) {
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t nv = (size_t)(pa.nl > 0 ? pa.nl : 1);
    const uint64_t capn = ((uint64_t)n + 3) & ~(uint64_t)3;  // value planes 32-byte aligned (refine's 16-byte copies)
    size_t o = 0;
    const size_t o_keys = o; o += al(((size_t)n + 2) * 4);
    const size_t o_cnt = o; o += al((size_t)pa.T * pa.C * 4);
    const size_t o_tot = o; o += al((size_t)pa.T * 4);
    const size_t o_ts = o; o += al(((size_t)pa.T + 1) * 4);
    const size_t o_off1 = o; o += al((size_t)pa.T1 * (pa.C + 1) * 4);
    const size_t o_skey = o; o += al((size_t)n * 4);
    const size_t o_sval = o; o += al((size_t)capn * 8 * nv);
    const size_t o_xkey = o; if (pa.G1 > 1) o += al(((size_t)capn + 4) * 4);     // (refine's bulk copies read whole
    const size_t o_xval = o; if (pa.G1 > 1) o += al(((size_t)capn * nv + 4) * 8);  //  4-row groups)
    const size_t total = o;
    if (total > h->part_bytes) {
        if (h->part_base) {
            cudaFree(h->part_base);  // synchronises the device: no execute still uses it
            count_free((int64_t)h->part_bytes);
            h->part_base = nullptr;
            h->part_bytes = 0;
        }
        const size_t want = total + total / 8;  // headroom for slowly growing n
        cudaError_t e = cudaMalloc(&h->part_base, want);
        if (e != cudaSuccess) {
            cudaGetLastError();
            h->part_base = nullptr;
            return set_error(BIN_ENOMEM, "partition route: %zu bytes of scratch on device %d", want, h->device);
        }
        count_alloc((int64_t)want);
        h->part_bytes = want;
    }
    pa.keys = (uint32_t *)(h->part_base + o_keys);
    pa.cnt = (uint32_t *)(h->part_base + o_cnt);
    pa.tot = (uint32_t *)(h->part_base + o_tot);
    pa.tstart = (uint32_t *)(h->part_base + o_ts);
    pa.off1 = (uint32_t *)(h->part_base + o_off1);
    pa.skey = (uint32_t *)(h->part_base + o_skey);
    pa.sval = (double *)(h->part_base + o_sval);
    pa.xkey = (uint32_t *)(h->part_base + o_xkey);
    pa.xval = (double *)(h->part_base + o_xval);
    pa.cap = capn;
    return BIN_OK;
}

static int nccl_error(ncclResult_t r, const char *what) {
    return set_error(BIN_ENCCL, "%s: %s", what, ncclGetErrorString(r));
}

static void free_slot(bin_handle *h, Slot &s) {
    DeviceGuard g(h->device);
    if (s.acc.count) {
        if (!s.external) cudaFree(s.acc.count);
        count_free((int64_t)s.dev_bytes);
    }
    s.acc = Accum{};
    if (s.meta_h) { cudaFreeHost(s.meta_h); count_free((int64_t)sizeof(Meta)); }
    s.meta_h = s.meta_d = nullptr;
    if (s.done) cudaEventDestroy(s.done);
    if (s.released) cudaEventDestroy(s.released);
    if (s.zeroed) cudaEventDestroy(s.zeroed);
    s.zeroed = nullptr;
    if (s.binned) cudaEventDestroy(s.binned);
    s.binned = nullptr;
    for (auto &e : s.ev)
        if (e) cudaEventDestroy(e), e = nullptr;
    s.done = s.released = nullptr;
}

// One slot allocation's layout (all pieces 256-byte aligned).
struct SlotLayout {
    size_t count, sum, mm, bounds, window, fxexp, omin, omax, oavg, meta, xrange, xs, total;
};
static SlotLayout slot_layout(const bin_handle *h) {
    const uint64_t B = h->nbins;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    SlotLayout L;
    L.count = 0;
    L.sum = L.count + al((B + 2) * 8);
    L.mm = L.sum + al(B * 8 * h->nsum);
    L.bounds = L.mm + al(B * 16 * h->nmm);
    L.window = L.bounds + al(6 * 8);
    L.fxexp = L.window + al(8 * 4);
    L.omin = L.fxexp + al(16 * 4);
    L.omax = L.omin + al(B * 8 * h->nmm);
    L.oavg = L.omax + al(B * 8 * h->nmm);
    L.meta = L.oavg + al(B * 8 * h->nsum);
    const bool exact = h->spec.sum_mode == BIN_SUM_EXACT && h->nsum > 0;
    L.xrange = L.meta + al(sizeof(Meta));
    L.xs = L.xrange + al(2 * BIN_MAX_ATTR * 4);
    L.total = exact ? L.xs + al(B * 8 * XD_DIGITS * h->nsum) : L.xrange;
    return L;
}

// ext: carve the slot from this memory (the NVLS region), else cudaMalloc it.
static int alloc_slot(bin_handle *h, Slot &s, unsigned char *ext = nullptr) {
    const uint64_t B = h->nbins;
    const SlotLayout L = slot_layout(h);
    const bool exact = h->spec.sum_mode == BIN_SUM_EXACT && h->nsum > 0;
    const size_t total = L.total;
    unsigned char *base = ext;
    cudaError_t e = ext ? cudaSuccess : cudaMalloc(&base, total);
    s.base = base;
    s.external = ext != nullptr;
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_error(BIN_ENOMEM, "bin_init: %zu bytes of bin arrays on device %d", total, h->device);
    }
    count_alloc((int64_t)total);
    s.dev_bytes = total;
    if ((e = cudaMemset(base, 0, total)) != cudaSuccess) return cuda_error(e, "bin_init memset");
    s.acc.count = (unsigned long long *)(base + L.count);
    s.acc.sum = (double *)(base + L.sum);
    s.acc.mm = (unsigned long long *)(base + L.mm);
    s.acc.bounds = (unsigned long long *)(base + L.bounds);
    s.acc.window = (int32_t *)(base + L.window);
    s.acc.fxexp = (uint32_t *)(base + L.fxexp);
    s.acc.omin = (double *)(base + L.omin);
    s.acc.omax = (double *)(base + L.omax);
    s.acc.oavg = (double *)(base + L.oavg);
    if (exact) {
        s.acc.xrange = (int32_t *)(base + L.xrange);
        s.acc.xs = (long long *)(base + L.xs);
        if ((e = cudaMemset(s.acc.xrange, 0x7f, 2 * BIN_MAX_ATTR * 4)) != cudaSuccess)
            return cuda_error(e, "bin_init memset(xrange)");
    }
    s.acc.nbins = B;
    s.acc.nsum = h->nsum;
    s.acc.nmm = h->nmm;
    s.acc.sum_mask = h->sum_mask;
    s.acc.mm_mask = h->mm_mask;
    s.acc.load_mask = h->load_mask;
    // result meta: written by the finalize kernel in device memory, copied to this
    // pinned mirror only when the host asks (bin_wait) -- no PCIe writes in the step
    DB_CUDA(cudaHostAlloc((void **)&s.meta_h, sizeof(Meta), cudaHostAllocPortable));
    count_alloc((int64_t)sizeof(Meta));
    memset(s.meta_h, 0, sizeof(Meta));
    s.meta_d = (Meta *)(base + L.meta);
    DB_CUDA(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
    DB_CUDA(cudaEventCreateWithFlags(&s.released, cudaEventDisableTiming));
    DB_CUDA(cudaEventCreateWithFlags(&s.zeroed, cudaEventDisableTiming));
    DB_CUDA(cudaEventCreateWithFlags(&s.binned, cudaEventDisableTiming));
    for (auto &ev : s.ev) DB_CUDA(cudaEventCreate(&ev));
    return BIN_OK;
}

int db::validate_spec(const bin_spec_t *sp, uint64_t *nbins) {
    if (sp->ndim < 1 || sp->ndim > BIN_MAX_DIM) return set_error(BIN_ENOTSUP, "ndim %d not in 1..3", sp->ndim);
    if (sp->nattr < 0 || sp->nattr > BIN_MAX_ATTR) return set_error(BIN_ENOTSUP, "nattr %d not in 0..16", sp->nattr);
    uint64_t B = 1;
    for (int d = 0; d < sp->ndim; ++d) {
        if (sp->res[d] < 1) return set_error(BIN_EINVAL, "res[%d] = %d < 1", d, sp->res[d]);
        B *= (uint64_t)sp->res[d];
        if (B >= (1ull << 32)) return set_error(BIN_EINVAL, "prod(res) >= 2^32");
        if (!sp->bounds_auto) {
            if (!(sp->lo[d] < sp->hi[d]) || !isfinite(sp->lo[d]) || !isfinite(sp->hi[d]))
                return set_error(BIN_EINVAL, "axis %d: need finite lo < hi (got %g, %g)", d, sp->lo[d], sp->hi[d]);
            if (!isfinite((double)sp->res[d] / (sp->hi[d] - sp->lo[d])) || sp->hi[d] - sp->lo[d] == INFINITY)
                return set_error(BIN_EINVAL, "axis %d: hi - lo overflows", d);
        }
    }
    if (sp->sum_mode != BIN_SUM_FAST && sp->sum_mode != BIN_SUM_EXACT)
        return set_error(BIN_EINVAL, "sum_mode %d is not a BIN_SUM_* value", sp->sum_mode);
    if (sp->sum_mode == BIN_SUM_EXACT && sp->deterministic)
        return set_error(BIN_EINVAL, "BIN_SUM_EXACT and deterministic are exclusive (exact sums are order-free)");
    if (sp->route < BIN_ROUTE_AUTO || sp->route > BIN_ROUTE_PARTITION)
        return set_error(BIN_EINVAL, "route %d is not a BIN_ROUTE_* value", sp->route);
    for (int a = 0; a < sp->nattr; ++a)
        if (sp->ops[a] & ~(uint32_t)(BIN_OP_SUM | BIN_OP_MIN | BIN_OP_MAX | BIN_OP_AVG))
            return set_error(BIN_EINVAL, "ops[%d] = 0x%x has unknown bits", a, sp->ops[a]);
    *nbins = B;
    return BIN_OK;
}

extern "C" {

void bin_placement_default(bin_placement_t *p) {
    if (!p) return;
    p->device_id = BIN_DEVICE_AUTO;
    p->device_start = 0;
    p->device_stride = 1;
    p->devices_to_use = 0;
    p->exec = BIN_EXEC_SYNC;
    p->async_snapshot = 1;
}

int bin_resolve_device(const bin_placement_t *p, int32_t rank, int32_t n_avail, int32_t *device) {
    if (!p || !device) return set_error(BIN_EINVAL, "bin_resolve_device: NULL argument");
    if (n_avail < 1) return set_error(BIN_EDEVICE, "no devices available (n_a = %d)", n_avail);
    if (p->device_id == BIN_DEVICE_HOST)
        return set_error(BIN_ENOTSUP, "host placement (device_id = -1): this library has no CPU path");
    if (p->device_id >= 0) {
        *device = p->device_id % n_avail;  // explicit ids wrap like Eq. (1) (reading R14b)
        return BIN_OK;
    }
    if (p->device_id != BIN_DEVICE_AUTO) return set_error(BIN_EDEVICE, "device_id %d", p->device_id);
    if (rank < 0) return set_error(BIN_EINVAL, "rank %d < 0", rank);
    if (p->device_stride < 1) return set_error(BIN_EINVAL, "device_stride %d < 1", p->device_stride);
    if (p->device_start < 0) return set_error(BIN_EINVAL, "device_start %d < 0", p->device_start);
    int n_u = p->devices_to_use > 0 ? p->devices_to_use : n_avail;  // default n_u = n_a
    // Eq. (1): d = ((r mod n_u) * s + d_0) mod n_a  (reading R14)
    long long d = ((long long)(rank % n_u) * p->device_stride + p->device_start) % n_avail;
    *device = (int32_t)d;
    return BIN_OK;
}

int bin_nccl_unique_id(void *out128) {
    if (!out128) return set_error(BIN_EINVAL, "bin_nccl_unique_id: NULL");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return nccl_error(r, "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    memcpy(out128, &id, 128);
    return BIN_OK;
}

// Peer mode: map every rank's slot allocations and barrier words into this
// process with CUDA IPC (handles exchanged through an NCCL all-gather), so the
// combine + finalize can run as one kernel over NVLink.  All ranks must be on
// distinct GPUs of one node; every rank must succeed, else all use NCCL.
static bool setup_peer(bin_handle *h) {
    const int R = h->nranks, r = h->rank;
    if (R > PEER_MAX) return false;
    const char *env = getenv("DATABIN_COMBINE");
    if (env && strcmp(env, "nccl") == 0) return false;
    struct Rec {
        cudaIpcMemHandle_t slot[2], flags;
        char uuid[16];
        int ok;
    };
    Rec mine;
    memset(&mine, 0, sizeof mine);
    mine.ok = 1;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, h->device) != cudaSuccess) mine.ok = 0;
    else memcpy(mine.uuid, &prop.uuid, 16);
    if (cudaMalloc(&h->flags, 128 * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMemset(h->flags, 0, 128 * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc(&h->ctas_done, 64) != cudaSuccess || cudaMemset(h->ctas_done, 0, 64) != cudaSuccess)
        mine.ok = 0;
    const bool nvls = h->nvls.mc != nullptr;  // slots in multicast memory: no unicast peer mappings needed
    for (int k = 0; k < 2 && mine.ok && !nvls; ++k)
        if (cudaIpcGetMemHandle(&mine.slot[k], h->slot[k].base) != cudaSuccess) mine.ok = 0;
    if (mine.ok && cudaIpcGetMemHandle(&mine.flags, h->flags) != cudaSuccess) mine.ok = 0;
    cudaGetLastError();
    // all-gather the records through NCCL (device buffers)
    const size_t rb = (sizeof(Rec) + 15) & ~(size_t)15;
    unsigned char *dbuf = nullptr;
    std::vector<unsigned char> all(rb * R);
    bool ok = cudaMalloc(&dbuf, rb * (R + 1)) == cudaSuccess;
    if (ok) ok = cudaMemcpy(dbuf + rb * R, &mine, sizeof mine, cudaMemcpyHostToDevice) == cudaSuccess;
    if (ok) ok = ncclAllGather(dbuf + rb * R, dbuf, rb, ncclUint8, h->comm, h->side) == ncclSuccess;
    if (ok) ok = cudaStreamSynchronize(h->side) == cudaSuccess;
    if (ok) ok = cudaMemcpy(all.data(), dbuf, rb * R, cudaMemcpyDeviceToHost) == cudaSuccess;
    if (dbuf) cudaFree(dbuf);
    cudaGetLastError();
    if (!ok) return false;  // NCCL itself is broken; bin_init reports it on first use
    std::vector<Rec> rec(R);
    for (int p = 0; p < R; ++p) memcpy(&rec[p], all.data() + rb * p, sizeof(Rec));
    bool good = true;
    for (int p = 0; p < R; ++p) {
        good = good && rec[p].ok;
        for (int q = 0; q < p; ++q) good = good && memcmp(rec[p].uuid, rec[q].uuid, 16) != 0;  // one rank per GPU
    }
    // open the peers' allocations
    unsigned char *slot_base[PEER_MAX][2] = {};
    unsigned long long *flags[PEER_MAX] = {};
    for (int p = 0; p < R && good; ++p) {
        if (p == r) {
            slot_base[p][0] = h->slot[0].base;
            slot_base[p][1] = h->slot[1].base;
            flags[p] = h->flags;
            continue;
        }
        void *ptr = nullptr;
        for (int k = 0; k < 2 && good && !nvls; ++k) {
            if (cudaIpcOpenMemHandle(&ptr, rec[p].slot[k], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) good = false;
            else h->opened.push_back(ptr), slot_base[p][k] = (unsigned char *)ptr;
        }
        if (good && cudaIpcOpenMemHandle(&ptr, rec[p].flags, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) good = false;
        else if (good) h->opened.push_back(ptr), flags[p] = (unsigned long long *)ptr;
    }
    cudaGetLastError();
    // every rank must agree
    int *dflag = nullptr;
    int agree = good ? 1 : 0;
    if (cudaMalloc(&dflag, sizeof(int)) == cudaSuccess &&
        cudaMemcpy(dflag, &agree, sizeof(int), cudaMemcpyHostToDevice) == cudaSuccess &&
        ncclAllReduce(dflag, dflag, 1, ncclInt32, ncclMin, h->comm, h->side) == ncclSuccess &&
        cudaStreamSynchronize(h->side) == cudaSuccess)
        cudaMemcpy(&agree, dflag, sizeof(int), cudaMemcpyDeviceToHost);
    else
        agree = 0;
    if (dflag) cudaFree(dflag);
    cudaGetLastError();
    if (!agree) return false;
    for (int k = 0; k < 2; ++k) {
        Slot &S = h->slot[k];
        PeerSet &ps = S.peers;
        ps.me = S.acc;
        ps.ctas_done = h->ctas_done + k;
        ps.ctas_failed = h->ctas_done + 4 + k;
        auto rel = [&](const void *local, int p) {
            return slot_base[p][k] + ((const unsigned char *)local - S.base);
        };
        if (nvls) {  // the combine reads and writes every rank through the multicast mapping
            auto mc = [&](const void *local) {
                return (unsigned char *)h->nvls.mc + ((const unsigned char *)local - (const unsigned char *)h->nvls.uc);
            };
            ps.mc_count = (unsigned long long *)mc(S.acc.count);
            ps.mc_sum = (double *)mc(S.acc.sum);
            ps.mc_mm = (unsigned long long *)mc(S.acc.mm);
            ps.mc_omin = (double *)mc(S.acc.omin);
            ps.mc_omax = (double *)mc(S.acc.omax);
            ps.mc_oavg = (double *)mc(S.acc.oavg);
            ps.mc_xs = S.acc.xs ? (long long *)mc(S.acc.xs) : nullptr;
            ps.mc_xrange = S.acc.xrange ? (int32_t *)mc(S.acc.xrange) : nullptr;
            for (int p = 0; p < R; ++p) ps.flags[p] = flags[p];
            continue;
        }
        for (int p = 0; p < R; ++p) {
            ps.count[p] = (unsigned long long *)rel(S.acc.count, p);
            ps.sum[p] = (double *)rel(S.acc.sum, p);
            ps.mm[p] = (unsigned long long *)rel(S.acc.mm, p);
            ps.omin[p] = (double *)rel(S.acc.omin, p);
            ps.omax[p] = (double *)rel(S.acc.omax, p);
            ps.oavg[p] = (double *)rel(S.acc.oavg, p);
            ps.xs[p] = S.acc.xs ? (long long *)rel(S.acc.xs, p) : nullptr;
            ps.xrange[p] = S.acc.xrange ? (int32_t *)rel(S.acc.xrange, p) : nullptr;
            ps.flags[p] = flags[p];
        }
    }
    return true;
}

int bin_init(const bin_spec_t *spec, const bin_placement_t *place, const bin_comm_t *comm, bin_handle_t **out) {
    if (!spec || !out) return set_error(BIN_EINVAL, "bin_init: NULL spec/out");
    *out = nullptr;
    uint64_t B = 0;
    int rc = validate_spec(spec, &B);
    if (rc) return rc;
    bin_placement_t pl;
    if (place) pl = *place;
    else bin_placement_default(&pl);
    if (pl.exec < BIN_EXEC_SYNC || pl.exec > BIN_EXEC_PEER) return set_error(BIN_EINVAL, "exec %d", pl.exec);
    int rank = comm ? comm->rank : 0, nranks = comm ? comm->nranks : 1;
    if (nranks < 1 || rank < 0 || rank >= nranks) return set_error(BIN_EINVAL, "rank %d of %d", rank, nranks);
    if (nranks > 1 && (!comm || !comm->nccl_unique_id))
        return set_error(BIN_EINVAL, "nranks > 1 needs an NCCL unique id");
    int n_a = 0;
    cudaError_t ce = cudaGetDeviceCount(&n_a);
    if (ce != cudaSuccess) {
        cudaGetLastError();
        if (pl.device_id == BIN_DEVICE_HOST) return bin_resolve_device(&pl, rank, 1, &n_a);
        return set_error(BIN_EDEVICE, "no CUDA device: %s", cudaGetErrorString(ce));
    }
    int dev = 0;
    rc = bin_resolve_device(&pl, rank, n_a, &dev);
    if (rc) return rc;

    bin_handle *h = new bin_handle;
    h->spec = *spec;
    h->place = pl;
    h->rank = rank;
    h->nranks = nranks;
    h->device = dev;
    h->nbins = B;
    for (int a = 0; a < spec->nattr; ++a) {
        uint32_t o = spec->ops[a];
        if (o & (BIN_OP_SUM | BIN_OP_AVG)) h->sum_mask |= 1u << a;
        if (o & (BIN_OP_MIN | BIN_OP_MAX)) h->mm_mask |= 1u << a;
    }
    h->load_mask = h->sum_mask | h->mm_mask;
    h->nsum = __builtin_popcount(h->sum_mask);
    h->nmm = __builtin_popcount(h->mm_mask);
    DeviceGuard g(dev);
    auto fail = [&](int code) {
        bin_finalize(h);
        return code;
    };
    if ((ce = cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking)) != cudaSuccess)
        return fail(cuda_error(ce, "cudaStreamCreate"));
    if ((ce = cudaStreamCreateWithFlags(&h->meta_stream, cudaStreamNonBlocking)) != cudaSuccess)
        return fail(cuda_error(ce, "cudaStreamCreate"));
    if ((ce = cudaStreamCreateWithFlags(&h->copy, cudaStreamNonBlocking)) != cudaSuccess)
        return fail(cuda_error(ce, "cudaStreamCreate"));
    if ((ce = cudaStreamCreateWithFlags(&h->prep, cudaStreamNonBlocking)) != cudaSuccess)
        return fail(cuda_error(ce, "cudaStreamCreate"));
    if (!h->spec.deterministic && h->spec.route == BIN_ROUTE_AUTO) {  // route probe buffers (executes allocate nothing)
        if ((ce = cudaMalloc(&h->probe_d, 64)) != cudaSuccess) return fail(cuda_error(ce, "cudaMalloc(probe)"));
        count_alloc(64);
        if ((ce = cudaHostAlloc((void **)&h->probe_h, 64, cudaHostAllocPortable)) != cudaSuccess)
            return fail(cuda_error(ce, "cudaHostAlloc(probe)"));
        count_alloc(64);
        if ((ce = cudaEventCreateWithFlags(&h->probe_ev, cudaEventDisableTiming)) != cudaSuccess)
            return fail(cuda_error(ce, "cudaEventCreate(probe)"));
    }
    // direct NVLink access to every other GPU this one can reach (peer copies and
    // the peer combine); without it cudaMemcpyPeerAsync stages through the host
    for (int d = 0; d < n_a; ++d) {
        int can = 0;
        if (d != dev && cudaDeviceCanAccessPeer(&can, dev, d) == cudaSuccess && can) cudaDeviceEnablePeerAccess(d, 0);
        cudaGetLastError();  // "already enabled" is fine
    }
    cudaDeviceGetAttribute(&h->lc.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&h->lc.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    Accum probe{};
    probe.nsum = h->nsum;
    probe.nmm = h->nmm;
    probe.nbins = B;
    // k_bin_fast (<= 1 attribute) keeps exact min/max in its window; the general kernel a filter
    const int bpb = spec->nattr <= 1 ? fast_window_bytes_per_bin(probe) : window_bytes_per_bin(probe);
    const int qbytes = (spec->nattr <= 1 && B < (1ull << 29)) ? fast_queue_bytes(spec->sum_mode == BIN_SUM_EXACT)
                                                                : 0;  // k_bin_fast's exact-sum queues
    const int static_smem = 1024;  // kernels' static __shared__ (k_bin_fast: window-pick scratch)
    h->wcap = (h->lc.smem_optin - static_smem - qbytes) / bpb;
    h->smem_bytes = (int)((uint64_t)h->wcap >= B ? B * bpb : (uint64_t)h->wcap * bpb);
    h->smem_bytes = ((h->smem_bytes + 15) & ~15) + qbytes;
    if (nranks > 1) {  // the communicator first: the NVLS region is a collective allocation
        ncclUniqueId id;
        memcpy(&id, comm->nccl_unique_id, sizeof id);
        ncclResult_t r = ncclCommInitRank(&h->comm, nranks, id, rank);
        if (r != ncclSuccess) {
            h->comm = nullptr;
            return fail(nccl_error(r, "ncclCommInitRank"));
        }
    }
    // NVLS combine (DATABIN_COMBINE=nvls, every GPU supporting multicast): both
    // slots in one multicast-bound region, reduced in the switch.  Measured
    // slower than the IPC peer combine's TMA bulk copies at 2 and 4 ranks on
    // C3 (slice 52-62 us vs 20-40 us: 8-byte multimem requests are rate-bound),
    // so the peer combine stays the default (DATABIN_COMBINE=nccl: NCCL).
    // Deterministic sums need the rank-ordered fold, which the switch does not keep.
    const size_t slot_sz = (slot_layout(h).total + 4095) & ~(size_t)4095;
    {
        const char *env = getenv("DATABIN_COMBINE");
        const bool want = nranks > 1 && nranks <= PEER_MAX && !spec->deterministic && env && strcmp(env, "nvls") == 0;
        if (want && !nvls_setup(2 * slot_sz, rank, nranks, dev, h->comm, h->side, comm->nccl_unique_id, &h->nvls))
            h->nvls = NvlsRegion{};
    }
    for (int k = 0; k < 2; ++k)
        if ((rc = alloc_slot(h, h->slot[k], h->nvls.uc ? (unsigned char *)h->nvls.uc + k * slot_sz : nullptr)))
            return fail(rc);
    if ((ce = cudaMalloc(&h->wcache, (size_t)h->lc.sms * 8 * sizeof(int32_t))) != cudaSuccess)
        return fail(cuda_error(ce, "cudaMalloc(window cache)"));
    count_alloc((int64_t)h->lc.sms * 32);
    if (getenv("DATABIN_TRACE")) {
        if ((ce = cudaMalloc(&h->ktrace, (size_t)h->lc.sms * 32)) != cudaSuccess)
            return fail(cuda_error(ce, "cudaMalloc(trace)"));
        cudaMemset(h->ktrace, 0, (size_t)h->lc.sms * 32);
    }
    for (auto &e : h->producer_ev)
        if ((ce = cudaEventCreateWithFlags(&e, cudaEventDisableTiming)) != cudaSuccess)
            return fail(cuda_error(ce, "cudaEventCreate"));
    if (nranks > 1 && spec->deterministic && h->nsum) {
        h->gather_bytes = (size_t)nranks * h->nsum * B * 8;
        h->gather = (double *)dev_alloc(h->gather_bytes, dev, nullptr, false);
        if (!h->gather) return fail(set_error(BIN_ENOMEM, "deterministic gather buffer"));
    }
    if (nranks > 1) h->peer = setup_peer(h);
    *out = h;
    return BIN_OK;
}

static void accumulate_profile(bin_handle *h, Slot &S);

static int stage_buffer(bin_handle *h, int sl, int col, size_t bytes, void **p) {
    Stage &st = h->stage[sl][col];
    if (st.bytes < bytes) {
        if (st.p) {
            cudaFree(st.p);
            count_free((int64_t)st.bytes);
        }
        st.p = nullptr;
        st.bytes = 0;
        st.p = dev_alloc(bytes, h->device, nullptr, false);
        if (!st.p) return set_error(BIN_ENOMEM, "staging buffer of %zu bytes", bytes);
        st.bytes = bytes;
    }
    *p = st.p;
    return BIN_OK;
}

// k_probe + D2H of its 8 ints; `wait`: block until the route is known (first
// execute), else leave it in flight (read back by a later execute).
static int run_probe(bin_handle *h, const Geom &geom, const Inputs &in, Slot &S, cudaStream_t s, bool wait) {
    cudaError_t e;
    if ((e = launch_probe(geom, in, S.acc, h->wcap, h->probe_d, s)) != cudaSuccess)
        return cuda_error(e, "route probe kernel");
    S.launches++;
    DB_CUDA(cudaMemcpyAsync(h->probe_h, h->probe_d, 8 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    DB_CUDA(cudaEventRecord(h->probe_ev, s));
    h->probe_inflight = true;
    h->since_probe = 0;
    if (wait) {
        DB_CUDA(cudaEventSynchronize(h->probe_ev));
        h->route = probe_route(h->probe_h);
        h->probe_inflight = false;
    }
    return BIN_OK;
}

// The end of an execute on its work stream S.stream: completion / release
// events, input-use tracking, and the lockstep wait.
static int finish_execute(bin_handle *h, Slot &S, bool staged_any, bin_array_t *const *axes, int32_t naxes,
                          bin_array_t *const *attrs, int32_t nattr, int32_t nshards) {
    cudaStream_t s = S.stream;
    DB_CUDA(cudaEventRecord(S.done, s));
    if (!staged_any) DB_CUDA(cudaEventRecord(S.released, s));
    S.prof_pending = h->prof;
    int rc;
    for (int sh = 0; sh < nshards; ++sh)
        for (int i = 0; i < naxes + nattr; ++i) {
            bin_array *a = i < naxes ? axes[sh * naxes + i] : attrs[sh * nattr + i - naxes];
            if ((rc = array_mark_use(a, s, h->device))) return rc;
        }
    if (h->place.exec == BIN_EXEC_SYNC && axes[0]->mode == BIN_SYNC) {
        cudaError_t e = cudaEventSynchronize(S.done);
        if (e != cudaSuccess) return cuda_error(e, "bin_execute (lockstep) synchronize");
    }
    return BIN_OK;
}

// One execute over nshards row blocks (nshards == 1: bin_execute).  Shard s's
// columns are axes[s * ndim + d] and attrs[s * nattr + a].  With several shards
// every column is staged into one buffer, shard after shard (host: H2D; other
// GPU: NVLink peer copy; this GPU: D2D), and binned as one batch.
static int execute_impl(bin_handle *h, bin_array_t *const *axes, int32_t naxes, bin_array_t *const *attrs,
                        int32_t nattr, int32_t nshards, uint64_t *ticket) {
    if (!h || h->finalized) return set_error(BIN_ESTATE, "bin_execute: handle is NULL or finalized");
    if (naxes != h->spec.ndim) return set_error(BIN_ESHAPE, "%d axis columns for a %dD mesh", naxes, h->spec.ndim);
    if (nattr != h->spec.nattr) return set_error(BIN_ESHAPE, "%d attribute columns, spec has %d", nattr, h->spec.nattr);
    if (nshards < 1 || nshards > BIN_MAX_SHARDS)
        return set_error(BIN_EINVAL, "%d shards (1..%d)", nshards, BIN_MAX_SHARDS);
    bin_array *cols[BIN_MAX_DIM + BIN_MAX_ATTR];
    const int ncols = naxes + nattr;
    int64_t shard_n[BIN_MAX_SHARDS];
    int64_t n = 0;
    for (int sh = 0; sh < nshards; ++sh) {
        bin_array *c0 = nullptr;
        for (int i = 0; i < ncols; ++i) {
            bin_array *c = i < naxes ? axes[sh * naxes + i] : attrs[sh * nattr + i - naxes];
            if (!c) return set_error(BIN_EINVAL, "shard %d column %d is NULL", sh, i);
            if (c->dtype != BIN_F64) return set_error(BIN_EDTYPE, "shard %d column %d is not BIN_F64", sh, i);
            if (!c0) c0 = c;
            if (c->n != c0->n)
                return set_error(BIN_ESHAPE, "shard %d: column %d has %lld rows, column 0 has %lld", sh, i,
                                 (long long)c->n, (long long)c0->n);
        }
        shard_n[sh] = c0->n;
        n += c0->n;
    }
    for (int i = 0; i < ncols; ++i) cols[i] = i < naxes ? axes[i] : attrs[i - naxes];  // shard 0 (ordering, mode)
    DeviceGuard g(h->device);
    const uint64_t t = h->next_ticket++;
    const int sl = (int)(t & 1);
    Slot &S = h->slot[sl];

    // ---- work stream (execution method)
    cudaStream_t s = h->side;
    if (h->place.exec == BIN_EXEC_SYNC && is_device_memory(cols[0]) && cols[0]->device == h->device)
        s = cols[0]->stream;  // lockstep: ordered on the producer's stream
    if (S.used && S.prof_pending) {  // keep per-phase times of every execute while profiling
        DB_CUDA(cudaEventSynchronize(S.done));
        accumulate_profile(h, S);
    }
    if (S.used && S.stream != s) DB_CUDA(cudaStreamWaitEvent(s, S.done, 0));
    {  // the previous execute may run on another stream: scratch (det, partition) is shared
        Slot &P = h->slot[sl ^ 1];
        if (P.used && P.stream != s) DB_CUDA(cudaStreamWaitEvent(s, P.done, 0));
    }
    S.ticket = t;
    S.used_before = S.used;
    S.used = true;
    S.meta_valid = false;
    S.stream = s;
    S.launches = 0;
    S.bin_launches = 0;
    h->last = s;
    for (bool &r : S.recd) r = false;
    if (h->prof) {
        DB_CUDA(cudaEventRecord(S.ev[EV_STAGE], s));
        S.recd[EV_STAGE] = true;
    }

    // ---- a1: resolve input views on the analysis device.  Columns already on
    // it are read in place (zero copy); the others -- host memory, another GPU
    // (peer copy over NVLink), or an asynchronous snapshot --
    // are copied into this slot's staging buffers on the handle's copy stream,
    // so a snapshot/peer copy overlaps the previous execute's binning.
    Inputs in{};
    in.n = n;
    in.nattr = nattr;
    bool staged_any = false;
    const bool snapshot = h->place.exec == BIN_EXEC_ASYNC && h->place.async_snapshot;
    bool stage[BIN_MAX_DIM + BIN_MAX_ATTR];
    for (int i = 0; i < ncols; ++i) {
        bin_array *a = cols[i];
        const bool local = a->alloc == BIN_ALLOC_CUDA_UVA || (is_device_memory(a) && a->device == h->device);
        stage[i] = n > 0 && (!local || snapshot || nshards > 1);
        staged_any = staged_any || stage[i];
    }
    if (staged_any && S.used) DB_CUDA(cudaStreamWaitEvent(h->copy, S.done, 0));  // staging buffers free again
    if (nshards > 1) {  // fan-in: every column concatenated shard after shard into one staging buffer
        for (int i = 0; i < ncols && n > 0; ++i) {
            void *dst = nullptr;
            int rc0 = stage_buffer(h, sl, i, (size_t)n * 8, &dst);
            if (rc0) return rc0;
            int64_t off = 0;
            for (int sh = 0; sh < nshards; ++sh) {
                bin_array *a = i < naxes ? axes[sh * naxes + i] : attrs[sh * nattr + i - naxes];
                const size_t bytes = (size_t)shard_n[sh] * 8;
                if (a->device >= 0 || a->alloc == BIN_ALLOC_HOST_PINNED) {  // after the producer's pending work
                    const int pd = a->device >= 0 ? a->device : h->device;
                    DeviceGuard g2(pd);
                    cudaEvent_t tmp;
                    DB_CUDA(cudaEventCreateWithFlags(&tmp, cudaEventDisableTiming));
                    DB_CUDA(cudaEventRecord(tmp, a->stream));
                    DeviceGuard g3(h->device);
                    DB_CUDA(cudaStreamWaitEvent(h->copy, tmp, 0));
                    cudaEventDestroy(tmp);
                }
                unsigned char *d = (unsigned char *)dst + (size_t)off * 8;
                if (bytes) {
                    if (a->device == -1 || a->alloc == BIN_ALLOC_HOST || a->alloc == BIN_ALLOC_HOST_PINNED)
                        DB_CUDA(cudaMemcpyAsync(d, a->ptr, bytes, cudaMemcpyHostToDevice, h->copy));
                    else if (a->device != h->device && a->alloc != BIN_ALLOC_CUDA_UVA)
                        DB_CUDA(cudaMemcpyPeerAsync(d, h->device, a->ptr, a->device, bytes, h->copy));
                    else
                        DB_CUDA(cudaMemcpyAsync(d, a->ptr, bytes, cudaMemcpyDeviceToDevice, h->copy));
                }
                off += shard_n[sh];
            }
            if (i < naxes) in.ax[i] = (const double *)dst;
            else in.at[i - naxes] = (const double *)dst;
        }
    }
    for (int i = 0; i < ncols && nshards == 1; ++i) {
        bin_array *a = cols[i];
        const double *p = (const double *)a->ptr;
        cudaStream_t consumer = stage[i] ? h->copy : s;
        // order after the producer's pending work on its own stream
        if (a->stream != consumer && (a->device >= 0 || a->alloc == BIN_ALLOC_HOST_PINNED)) {
            const int pd = a->device >= 0 ? a->device : h->device;
            DeviceGuard g2(pd);
            if (pd != h->device) {
                // events are per device: a temporary on the producer's device
                cudaEvent_t tmp;
                DB_CUDA(cudaEventCreateWithFlags(&tmp, cudaEventDisableTiming));
                DB_CUDA(cudaEventRecord(tmp, a->stream));
                DeviceGuard g3(h->device);
                DB_CUDA(cudaStreamWaitEvent(consumer, tmp, 0));
                cudaEventDestroy(tmp);
            } else {
                DB_CUDA(cudaEventRecord(h->producer_ev[i], a->stream));
                DB_CUDA(cudaStreamWaitEvent(consumer, h->producer_ev[i], 0));
            }
        }
        if (stage[i]) {
            void *dst = nullptr;
            int rc = stage_buffer(h, sl, i, (size_t)n * 8, &dst);
            if (rc) return rc;
            if (a->device == -1 || a->alloc == BIN_ALLOC_HOST || a->alloc == BIN_ALLOC_HOST_PINNED)
                DB_CUDA(cudaMemcpyAsync(dst, a->ptr, (size_t)n * 8, cudaMemcpyHostToDevice, h->copy));
            else if (a->device != h->device && a->alloc != BIN_ALLOC_CUDA_UVA)
                DB_CUDA(cudaMemcpyPeerAsync(dst, h->device, a->ptr, a->device, (size_t)n * 8, h->copy));
            else
                DB_CUDA(cudaMemcpyAsync(dst, a->ptr, (size_t)n * 8, cudaMemcpyDeviceToDevice, h->copy));
            p = (const double *)dst;
        }
        if (i < naxes) in.ax[i] = p;
        else in.at[i - naxes] = p;
    }
    if (staged_any) {  // inputs copied: the producer may overwrite; the analysis may start
        DB_CUDA(cudaEventRecord(S.released, h->copy));
        DB_CUDA(cudaStreamWaitEvent(s, S.released, 0));
    }

    Geom geom{};
    geom.ndim = h->spec.ndim;
    geom.bounds_auto = h->spec.bounds_auto;
    for (int d = 0; d < 3; ++d) {
        geom.res[d] = d < geom.ndim ? h->spec.res[d] : 1;
        geom.lo[d] = d < geom.ndim ? h->spec.lo[d] : 0.0;
        geom.hi[d] = d < geom.ndim ? h->spec.hi[d] : 1.0;
    }
    cudaError_t e;
    // profiling: an event only after a phase that enqueued work (an event costs
    // ~2-3 us of stream time; empty phases get none and read as 0)
    auto rec = [&](int k, bool work) -> int {
        if (h->prof && work) {
            DB_CUDA(cudaEventRecord(S.ev[k], s));
            S.recd[k] = true;
        }
        return BIN_OK;
    };
    int rc;
    if ((rc = rec(EV_INIT0, staged_any))) return rc;
    // exact sums: every digit stays below 2^62 in magnitude only while the rows of
    // ALL ranks together stay below 2^30 (the cross-rank combine adds the ranks'
    // digits before it normalises the carries), so each rank takes < 2^30 / nranks
    if (S.acc.xs && n >= (1ll << 30) / h->nranks)
        return set_error(BIN_EINVAL, "BIN_SUM_EXACT: %lld rows per execute and rank (limit 2^30 / %d ranks: digit headroom)",
                         (long long)n, h->nranks);
    // ---- route: partition (bin_part.cu) or window; auto follows the last probe
    PartArgs pa{};
    const bool part_ok = n > 0 && !h->spec.deterministic && h->spec.route != BIN_ROUTE_WINDOW &&
                         part_plan(in, S.acc, geom.ndim, h->lc.smem_optin, h->lc.sms, &pa);
    if (part_ok && h->spec.route == BIN_ROUTE_AUTO && h->probe_inflight) {
        cudaError_t q = cudaEventQuery(h->probe_ev);
        if (q == cudaSuccess) {
            h->route = probe_route(h->probe_h);
            h->probe_inflight = false;
        } else if (q == cudaErrorNotReady) {
            cudaGetLastError();
        } else {
            return cuda_error(q, "route probe");
        }
    }
    // first execute with manual bounds: the synchronous probe runs before the
    // init so that the route (and the one-launch step) is known from the start
    bool probed = false;
    if (part_ok && h->spec.route == BIN_ROUTE_AUTO && h->route == 0 && !geom.bounds_auto) {
        if ((rc = run_probe(h, geom, in, S, s, true))) return rc;
        probed = true;
    }
    bool part = part_ok && (h->spec.route == BIN_ROUTE_PARTITION || h->route == BIN_ROUTE_PARTITION);
    // ---- a3: accumulator identities (+ the window choice when the bounds are manual
    // and the general kernel will run; k_bin_fast chooses its windows per CTA)
    bool fast = n > 0 && !h->spec.deterministic && !part && fast_eligible(in, S.acc, geom.ndim);
    // a3 on the handle's prep stream: the slot's identities are written as soon
    // as its previous execute is done (typically while the previous execute on
    // the other slot is still binning), off the critical path; the work stream
    // waits for them before its first kernel that touches the slot
    if (S.used_before) DB_CUDA(cudaStreamWaitEvent(h->prep, S.done, 0));
    if ((e = launch_init(geom, in, S.acc, h->wcap, false, h->prep)) != cudaSuccess)
        return cuda_error(e, "init kernel");
    S.launches++;
    if (S.acc.xs)  // exact sums: the digits of the last execute are clear; reset their range
        DB_CUDA(cudaMemsetAsync(S.acc.xrange, 0x7f, 2 * BIN_MAX_ATTR * 4, h->prep));
    DB_CUDA(cudaEventRecord(S.zeroed, h->prep));
    DB_CUDA(cudaStreamWaitEvent(s, S.zeroed, 0));
    const bool window_in_prep = !geom.bounds_auto && !h->spec.deterministic && !fast && !part;
    // ---- a2: automatic bounds (+ cross-rank Min, reading R3)
    if (geom.bounds_auto) {
        if ((e = launch_bounds(geom, in, S.acc, h->lc, s)) != cudaSuccess) return cuda_error(e, "bounds kernel");
        if (n > 0) S.launches++;
        if (h->comm) {
            ncclResult_t r = ncclAllReduce(S.acc.bounds, S.acc.bounds, 2 * geom.ndim, ncclUint64, ncclMin, h->comm, s);
            if (r != ncclSuccess) return nccl_error(r, "ncclAllReduce(bounds)");
        }
    }
    // ---- route probe (auto): first execute synchronously, then every ROUTE_REPROBE
    // executes in the background (read back at a later execute, never waited for)
    if ((rc = rec(EV_BOUNDS1, geom.bounds_auto))) return rc;
    if (part_ok && h->spec.route == BIN_ROUTE_AUTO && !h->probe_inflight && !probed &&
        (h->route == 0 || ++h->since_probe >= ROUTE_REPROBE)) {
        const bool first = h->route == 0;
        if ((rc = run_probe(h, geom, in, S, s, first))) return rc;
        probed = true;
        if (first) {
            part = h->route == BIN_ROUTE_PARTITION;
            fast = fast && !part;
        }
    }
    int variant;
    if (h->spec.deterministic) {
        if ((rc = rec(EV_WINDOW1, probed))) return rc;
        int launches = 0;
        if ((rc = ensure_det_scratch(h->det, n, h->nbins, h->device, h->lc.sms))) return rc;
        if ((e = launch_deterministic(geom, in, S.acc, h->det, h->lc, s, &launches)) != cudaSuccess)
            return cuda_error(e, "deterministic binning");
        S.launches += launches;
        S.bin_launches += 1;
        variant = 3;
    } else {
        // ---- hot-window choice, then a4 + a5
        const bool win_kernel = !fast && !part && n > 0;  // (window_in_prep: manual bounds, chosen here too)
        if (win_kernel) {
            if ((e = launch_window(geom, in, S.acc, h->wcap, s)) != cudaSuccess) return cuda_error(e, "window kernel");
            S.launches += 1;
        }
        if ((rc = rec(EV_WINDOW1, win_kernel || probed))) return rc;
        if (n / h->lc.sms >= (int64_t)0xffffffffLL)
            return set_error(BIN_EINVAL, "%lld rows per call exceed the per-CTA u32 window counters", (long long)n);
        if (part) {
            if ((rc = ensure_part_scratch(h, n, pa))) return rc;
            int pl = 0;
            if ((e = launch_partition(geom, in, S.acc, pa, s, &pl)) != cudaSuccess)
                return cuda_error(e, "partition route kernels");
            S.launches += pl, S.bin_launches += pl;
            variant = 4;
        } else {
            variant = ((uint64_t)h->wcap >= h->nbins ? 2 : 1) | (fast ? 16 : 0);
            if (n > 0) {
                // per-CTA windows: sampled at the first fast execute and every
                // WINDOW_RESAMPLE-th after it (and whenever the row count changes)
                const bool reuse = fast && h->wcache_n == n && h->wcache_age % WINDOW_RESAMPLE != 0;
                if (fast) {
                    h->wcache_n = n;
                    h->wcache_age = reuse ? h->wcache_age + 1 : 1;
                }
                e = fast ? launch_bin_fast(geom, in, S.acc, h->lc, h->smem_bytes, h->wcap, h->wcache, reuse ? 1 : 0,
                                           h->ktrace, s)
                         : launch_bin_general(geom, in, S.acc, h->lc, h->smem_bytes, s);
                if (e != cudaSuccess) return cuda_error(e, "bin kernel");
                S.launches++, S.bin_launches++;
            }
        }
    }
    if ((rc = rec(EV_BIN1, n > 0))) return rc;
    if (h->group) {  // rank group: bin_execute_group launches the combine once for all ranks
        DB_CUDA(cudaEventRecord(S.binned, s));
        S.variant = variant | 32;
        S.staged_any = staged_any;
        if (ticket) *ticket = t;
        return BIN_OK;
    }
    // ---- a6 + a7 fused over NVLink peer memory (one kernel), or NCCL + finalize
    if (h->peer) {
        if ((e = launch_combine_peer(geom, S.peers, h->rank, h->nranks, t, S.meta_d, variant | 32,
                                     h->spec.deterministic, h->lc.sms, s)) != cudaSuccess)
            return cuda_error(e, "peer combine kernel");
        S.launches++;
        S.variant = variant | 32 | (S.peers.mc_count ? 64 : 0);
        if ((rc = rec(EV_FINAL1, true))) return rc;
    } else {
    // ---- a6: cross-rank combine over NVLink (one NCCL group)
    if (h->comm) {
        const uint64_t B = h->nbins;
        ncclResult_t r = ncclGroupStart();
        if (r == ncclSuccess) r = ncclAllReduce(S.acc.count, S.acc.count, B + 2, ncclUint64, ncclSum, h->comm, s);
        if (r == ncclSuccess && h->nsum && !h->gather && !S.acc.xs)
            r = ncclAllReduce(S.acc.sum, S.acc.sum, B * h->nsum, ncclFloat64, ncclSum, h->comm, s);
        if (r == ncclSuccess && S.acc.xs) {  // exact sums: digits add as integers (order-free), ranges unite
            r = ncclAllReduce(S.acc.xs, S.acc.xs, B * h->nsum * XD_DIGITS, ncclInt64, ncclSum, h->comm, s);
            if (r == ncclSuccess)
                r = ncclAllReduce(S.acc.xrange, S.acc.xrange, 2 * h->nsum, ncclInt32, ncclMin, h->comm, s);
        }
        if (r == ncclSuccess && h->nsum && h->gather)  // deterministic: gather partials, fold in rank order
            r = ncclAllGather(S.acc.sum, h->gather, B * h->nsum, ncclFloat64, h->comm, s);
        if (r == ncclSuccess && h->nmm)
            r = ncclAllReduce(S.acc.mm, S.acc.mm, B * h->nmm * 2, ncclUint64, ncclMin, h->comm, s);
        ncclResult_t r2 = ncclGroupEnd();
        if (r != ncclSuccess) return nccl_error(r, "ncclAllReduce(bins)");
        if (r2 != ncclSuccess) return nccl_error(r2, "ncclGroupEnd");
        if (h->gather) {
            if ((e = launch_rank_fold(h->gather, h->nranks, B * h->nsum, S.acc.sum, h->lc.sms, s)) != cudaSuccess)
                return cuda_error(e, "rank-ordered fold");
            S.launches++;
        }
    }
    if ((rc = rec(EV_COMBINE1, h->comm != nullptr))) return rc;
    // ---- a7: finalize
    if ((e = launch_finalize(geom, S.acc, S.meta_d, n, variant, s)) != cudaSuccess) return cuda_error(e, "finalize kernel");
    S.launches++;
    S.variant = variant;
    if ((rc = rec(EV_FINAL1, true))) return rc;
    }
    if (ticket) *ticket = t;
    return finish_execute(h, S, staged_any, axes, naxes, attrs, nattr, nshards);
}

int bin_execute(bin_handle_t *h, bin_array_t *const *axes, int32_t naxes, bin_array_t *const *attrs,
                int32_t nattr, uint64_t *ticket) {
    if (h && h->group) return set_error(BIN_ESTATE, "bin_execute: handle belongs to a rank group (bin_execute_group)");
    return execute_impl(h, axes, naxes, attrs, nattr, 1, ticket);
}

int bin_execute_shards(bin_handle_t *h, bin_array_t *const *axes, int32_t naxes, bin_array_t *const *attrs,
                       int32_t nattr, int32_t nshards, uint64_t *ticket) {
    if (h && h->group) return set_error(BIN_ESTATE, "bin_execute_shards: handle belongs to a rank group");
    return execute_impl(h, axes, naxes, attrs, nattr, nshards, ticket);
}

static Slot *find_slot(bin_handle *h, uint64_t t) {
    Slot &S = h->slot[t & 1];
    return (S.used && S.ticket == t) ? &S : nullptr;
}

int bin_inputs_released(bin_handle_t *h, uint64_t ticket, bin_event_t *ev) {
    if (!h || !ev) return set_error(BIN_EINVAL, "bin_inputs_released: NULL argument");
    Slot *S = find_slot(h, ticket);
    if (!S) return set_error(BIN_ESTATE, "unknown or recycled ticket %llu", (unsigned long long)ticket);
    *ev = (bin_event_t)S->released;
    return BIN_OK;
}

// Copies a completed slot's result meta (device) to its pinned mirror on the
// handle's meta stream (non-blocking: it does not serialise with the work).
static int fetch_meta(bin_handle *h, Slot &S) {
    if (S.meta_valid) return BIN_OK;
    DB_CUDA(cudaMemcpyAsync(S.meta_h, S.meta_d, sizeof(Meta), cudaMemcpyDeviceToHost, h->meta_stream));
    DB_CUDA(cudaStreamSynchronize(h->meta_stream));
    S.meta_valid = true;
    static const bool tr = getenv("DATABIN_TRACE") != nullptr;
    if (tr && h->ktrace && (S.meta_h->variant & 16)) {  // k_bin_fast per-CTA phases (us)
        std::vector<unsigned long long> x((size_t)h->lc.sms * 4);
        if (cudaMemcpy(x.data(), h->ktrace, x.size() * 8, cudaMemcpyDeviceToHost) == cudaSuccess) {
            double t0 = 1e30, w = 0, lmin = 1e30, lmax = 0, f = 0, emin = 1e30, emax = 0;
            for (int c = 0; c < h->lc.sms; ++c) {
                const unsigned long long *q = &x[(size_t)c * 4];
                if (!q[3]) continue;
                t0 = fmin(t0, (double)q[0]);
                w = fmax(w, (double)(q[1] - q[0]));
                lmin = fmin(lmin, (double)(q[2] - q[1]));
                lmax = fmax(lmax, (double)(q[2] - q[1]));
                f = fmax(f, (double)(q[3] - q[2]));
                emin = fmin(emin, (double)q[3]);
                emax = fmax(emax, (double)q[3]);
            }
            fprintf(stderr, "[databin trace] rank %d ticket %llu k_bin_fast: prologue <= %.1f, loop %.1f..%.1f, "
                            "flush <= %.1f, CTA end spread %.1f, total %.1f us\n", h->rank,
                    (unsigned long long)S.ticket, w * 1e-3, lmin * 1e-3, lmax * 1e-3, f * 1e-3, (emax - emin) * 1e-3,
                    (emax - t0) * 1e-3);
        }
    }
    if (tr && (S.meta_h->variant & 32)) {  // peer combine phase times on this rank (us)
        const uint64_t *x = S.meta_h->trace;
        fprintf(stderr, "[databin trace] rank %d ticket %llu: barrier A %.1f, slice %.1f, barrier B %.1f us\n",
                h->rank, (unsigned long long)S.ticket, (x[1] - x[0]) * 1e-3, ((double)x[2] - (double)x[1]) * 1e-3,
                ((double)x[3] - (double)x[2]) * 1e-3);
    }
    return BIN_OK;
}

static void accumulate_profile(bin_handle *h, Slot &S) {
    if (!S.prof_pending) return;
    S.prof_pending = false;
    fetch_meta(h, S);
    float ms[EV_N] = {};
    for (int k = 1, last = EV_STAGE; k < EV_N; ++k)
        if (S.recd[k]) {  // a phase's time runs from the previous recorded event
            cudaEventElapsedTime(&ms[k], S.ev[last], S.ev[k]);
            last = k;
        }
    cudaGetLastError();
    bin_profile_t &p = h->pacc;
    p.ms_stage += ms[EV_INIT0];
    p.ms_init += ms[EV_INIT1];
    p.ms_bounds += ms[EV_BOUNDS1];
    p.ms_window += ms[EV_WINDOW1];
    p.ms_bin += ms[EV_BIN1];
    p.ms_combine += ms[EV_COMBINE1];
    p.ms_finalize += ms[EV_FINAL1];
    p.executes += 1;
    p.kernel_launches += S.launches;
    p.bin_launches += S.bin_launches;
    p.variant = S.variant;
    for (int d = 0; d < 3; ++d) p.window[d] = S.meta_h->window[3 + d];
}

int bin_wait(bin_handle_t *h, uint64_t ticket) {
    if (!h || h->finalized) return set_error(BIN_ESTATE, "bin_wait: handle is NULL or finalized");
    Slot *S = find_slot(h, ticket);
    if (!S) return set_error(BIN_ESTATE, "unknown or recycled ticket %llu", (unsigned long long)ticket);
    DeviceGuard g(h->device);
    cudaError_t e = cudaEventSynchronize(S->done);
    if (e != cudaSuccess) return cuda_error(e, "bin_wait");
    int rc = fetch_meta(h, *S);
    if (rc) return rc;
    accumulate_profile(h, *S);
    if (S->meta_h->status == BIN_ENCCL)
        return set_error(BIN_ENCCL, "peer combine: a rank did not reach the NVLink barrier within ~2 s");
    if (S->meta_h->status == BIN_EDEGENERATE)
        return set_error(BIN_EDEGENERATE, "auto bounds: no finite rows in total, or an infinite/unrecoverable axis");
    return BIN_OK;
}

int bin_result(bin_handle_t *h, uint64_t ticket, bin_result_t *out) {
    if (!out) return set_error(BIN_EINVAL, "bin_result: NULL out");
    int rc = bin_wait(h, ticket);
    if (rc) return rc;
    Slot &S = *find_slot(h, ticket);
    memset(out, 0, sizeof *out);
    const uint64_t B = h->nbins;
    out->count = (const uint64_t *)S.acc.count;
    for (int a = 0; a < h->spec.nattr; ++a) {
        uint32_t o = h->spec.ops[a];
        if ((h->sum_mask >> a) & 1u) {
            int slot = __builtin_popcount(h->sum_mask & ((1u << a) - 1u));
            if (o & BIN_OP_SUM) out->sum[a] = S.acc.sum + (uint64_t)slot * B;
            if (o & BIN_OP_AVG) out->avg[a] = S.acc.oavg + (uint64_t)slot * B;
        }
        if ((h->mm_mask >> a) & 1u) {
            int slot = __builtin_popcount(h->mm_mask & ((1u << a) - 1u));
            if (o & BIN_OP_MIN) out->min[a] = S.acc.omin + (uint64_t)slot * B;
            if (o & BIN_OP_MAX) out->max[a] = S.acc.omax + (uint64_t)slot * B;
        }
    }
    out->nbins = B;
    out->n_in = S.meta_h->n_in;
    out->n_out = S.meta_h->n_out;
    out->device = h->device;
    for (int d = 0; d < 3; ++d) {
        out->lo[d] = d < h->spec.ndim ? S.meta_h->lo[d] : 0.0;
        out->hi[d] = d < h->spec.ndim ? S.meta_h->hi[d] : 0.0;
    }
    return BIN_OK;
}

// ---------------------------------------------------------------- one-device rank group
static void group_drop(bin_handle *h) {
    bin_group *G = h->group;
    if (!G) return;
    h->group = nullptr;
    if (h->rank >= 0 && h->rank < (int)G->member.size() && G->member[h->rank] == h) G->member[h->rank] = nullptr;
    if (--G->alive > 0) return;
    DeviceGuard g(G->device);
    if (G->stream) cudaStreamSynchronize(G->stream), cudaStreamDestroy(G->stream);
    for (auto &e : G->done)
        if (e) cudaEventDestroy(e);
    if (G->dev) cudaFree(G->dev);
    delete G;
}

int bin_init_group(const bin_spec_t *spec, const bin_placement_t *place, int32_t nranks, bin_handle_t **out) {
    if (!spec || !out) return set_error(BIN_EINVAL, "bin_init_group: NULL spec/out");
    if (nranks < 1 || nranks > PEER_MAX) return set_error(BIN_EINVAL, "bin_init_group: %d ranks (1..%d)", nranks, PEER_MAX);
    if (spec->bounds_auto)
        return set_error(BIN_ENOTSUP, "bin_init_group: automatic bounds need the cross-rank Min (NCCL); give manual bounds");
    for (int r = 0; r < nranks; ++r) out[r] = nullptr;
    bin_group *G = new bin_group;
    G->nranks = nranks;
    G->member.assign(nranks, nullptr);
    auto fail = [&](int code) {
        for (int r = 0; r < nranks; ++r)
            if (out[r]) bin_finalize(out[r]), out[r] = nullptr;
        if (G->alive == 0) {  // no member took ownership yet
            if (G->stream) cudaStreamDestroy(G->stream);
            for (auto &e : G->done)
                if (e) cudaEventDestroy(e);
            if (G->dev) cudaFree(G->dev);
            delete G;
        }
        return code;
    };
    for (int r = 0; r < nranks; ++r) {
        int rc = bin_init(spec, place, nullptr, &out[r]);  // one rank each, all on the same device
        if (rc) return fail(rc);
    }
    G->device = out[0]->device;
    DeviceGuard g(G->device);
    cudaError_t ce;
    if ((ce = cudaStreamCreateWithFlags(&G->stream, cudaStreamNonBlocking)) != cudaSuccess)
        return fail(cuda_error(ce, "bin_init_group: stream"));
    for (auto &e : G->done)
        if ((ce = cudaEventCreateWithFlags(&e, cudaEventDisableTiming)) != cudaSuccess)
            return fail(cuda_error(ce, "bin_init_group: event"));
    for (int r = 0; r < nranks; ++r) {
        bin_handle *h = out[r];
        if ((ce = cudaMalloc(&h->flags, 128 * sizeof(unsigned long long))) != cudaSuccess ||
            (ce = cudaMemset(h->flags, 0, 128 * sizeof(unsigned long long))) != cudaSuccess ||
            (ce = cudaMalloc(&h->ctas_done, 64)) != cudaSuccess || (ce = cudaMemset(h->ctas_done, 0, 64)) != cudaSuccess)
            return fail(cuda_error(ce, "bin_init_group: barrier words"));
    }
    std::vector<GroupRank> host((size_t)2 * nranks);
    for (int k = 0; k < 2; ++k)
        for (int r = 0; r < nranks; ++r) {
            bin_handle *h = out[r];
            PeerSet &ps = h->slot[k].peers;
            ps = PeerSet{};
            ps.me = h->slot[k].acc;
            ps.ctas_done = h->ctas_done + k;
            ps.ctas_failed = h->ctas_done + 4 + k;
            for (int p = 0; p < nranks; ++p) {  // same address space: the peers' slot arrays directly
                const Accum &a = out[p]->slot[k].acc;
                ps.count[p] = a.count;
                ps.sum[p] = a.sum;
                ps.mm[p] = a.mm;
                ps.omin[p] = a.omin;
                ps.omax[p] = a.omax;
                ps.oavg[p] = a.oavg;
                ps.xs[p] = a.xs;
                ps.xrange[p] = a.xrange;
                ps.flags[p] = out[p]->flags;
            }
            host[(size_t)k * nranks + r] = GroupRank{ps, h->slot[k].meta_d};
        }
    if ((ce = cudaMalloc(&G->dev, host.size() * sizeof(GroupRank))) != cudaSuccess)
        return fail(cuda_error(ce, "bin_init_group: peer sets"));
    if ((ce = cudaMemcpy(G->dev, host.data(), host.size() * sizeof(GroupRank), cudaMemcpyHostToDevice)) != cudaSuccess)
        return fail(cuda_error(ce, "bin_init_group: peer sets"));
    for (int r = 0; r < nranks; ++r) {
        out[r]->rank = r;
        out[r]->nranks = nranks;
        out[r]->peer = true;
        out[r]->group = G;
        G->member[r] = out[r];
        G->alive++;
    }
    return BIN_OK;
}

int bin_execute_group(bin_handle_t *const *hs, int32_t nranks, bin_array_t *const *axes, int32_t naxes,
                      bin_array_t *const *attrs, int32_t nattr, uint64_t *ticket) {
    if (!hs || nranks < 1 || !hs[0] || !hs[0]->group) return set_error(BIN_EINVAL, "bin_execute_group: not a rank group");
    bin_group *G = hs[0]->group;
    if (nranks != G->nranks) return set_error(BIN_EINVAL, "bin_execute_group: %d handles for a group of %d", nranks, G->nranks);
    for (int r = 0; r < nranks; ++r)
        if (!hs[r] || hs[r]->finalized || hs[r]->group != G || hs[r]->rank != r || G->member[r] != hs[r])
            return set_error(BIN_ESTATE, "bin_execute_group: handle %d is not rank %d of this group (or finalized)", r, r);
    if (!axes || (nattr && !attrs)) return set_error(BIN_EINVAL, "bin_execute_group: NULL columns");
    const uint64_t t = hs[0]->next_ticket;
    for (int r = 0; r < nranks; ++r)
        if (hs[r]->next_ticket != t) return set_error(BIN_ESTATE, "bin_execute_group: ranks out of step");
    // a1-a5 of every rank on its own work stream
    for (int r = 0; r < nranks; ++r) {
        uint64_t tr = 0;
        int rc = execute_impl(hs[r], axes + (size_t)r * naxes, naxes, attrs + (size_t)r * nattr, nattr, 1, &tr);
        if (rc) return rc;
    }
    // a6 + a7: one launch over all ranks once every rank has binned
    const int sl = (int)(t & 1);
    DeviceGuard g(G->device);
    for (int r = 0; r < nranks; ++r) DB_CUDA(cudaStreamWaitEvent(G->stream, hs[r]->slot[sl].binned, 0));
    bin_handle *h0 = hs[0];
    Geom geom{};
    geom.ndim = h0->spec.ndim;
    geom.bounds_auto = 0;
    for (int d = 0; d < 3; ++d) {
        geom.res[d] = d < geom.ndim ? h0->spec.res[d] : 1;
        geom.lo[d] = d < geom.ndim ? h0->spec.lo[d] : 0.0;
        geom.hi[d] = d < geom.ndim ? h0->spec.hi[d] : 1.0;
    }
    cudaError_t e = launch_combine_group(geom, G->dev + (size_t)sl * nranks, h0->slot[sl].acc, nranks, t,
                                         h0->slot[sl].variant, h0->lc.sms, G->stream);
    if (e != cudaSuccess) return cuda_error(e, "group combine kernel");
    DB_CUDA(cudaEventRecord(G->done[sl], G->stream));
    for (int r = 0; r < nranks; ++r) {
        bin_handle *h = hs[r];
        Slot &S = h->slot[sl];
        DB_CUDA(cudaStreamWaitEvent(S.stream, G->done[sl], 0));
        S.launches++;
        if (h->prof) {
            DB_CUDA(cudaEventRecord(S.ev[EV_FINAL1], S.stream));
            S.recd[EV_FINAL1] = true;
        }
        int rc = finish_execute(h, S, S.staged_any, axes + (size_t)r * naxes, naxes, attrs + (size_t)r * nattr, nattr, 1);
        if (rc) return rc;
    }
    if (ticket) *ticket = t;
    return BIN_OK;
}

int bin_stream(bin_handle_t *h, bin_stream_t *stream) {
    if (!h || !stream) return set_error(BIN_EINVAL, "bin_stream: NULL argument");
    *stream = (bin_stream_t)(h->last ? h->last : h->side);
    return BIN_OK;
}

int bin_profile_enable(bin_handle_t *h, int32_t on) {
    if (!h) return set_error(BIN_EINVAL, "bin_profile_enable: NULL handle");
    h->prof = on != 0;
    memset(&h->pacc, 0, sizeof h->pacc);
    return BIN_OK;
}

int bin_profile_read(bin_handle_t *h, bin_profile_t *out) {
    if (!h || !out) return set_error(BIN_EINVAL, "bin_profile_read: NULL argument");
    DeviceGuard g(h->device);
    for (auto &S : h->slot)
        if (S.prof_pending && cudaEventQuery(S.done) == cudaSuccess) accumulate_profile(h, S);
    *out = h->pacc;
    return BIN_OK;
}

int bin_finalize(bin_handle_t *h) {
    if (!h) return BIN_OK;
    int rc = BIN_OK;
    {
        DeviceGuard g(h->device);
        for (auto &S : h->slot)
            if (S.done) {
                cudaError_t e = cudaEventSynchronize(S.done);
                if (e != cudaSuccess && rc == BIN_OK) rc = cuda_error(e, "bin_finalize");
            }
        if (h->side) cudaStreamSynchronize(h->side);
        if (h->prep) cudaStreamSynchronize(h->prep);
        if (h->copy) cudaStreamSynchronize(h->copy);
        for (void *p : h->opened) cudaIpcCloseMemHandle(p);
        h->opened.clear();
        if (h->flags) cudaFree(h->flags);
        if (h->ctas_done) cudaFree(h->ctas_done);
        h->flags = nullptr;
        h->ctas_done = nullptr;
        if (h->comm) {
            ncclCommDestroy(h->comm);
            h->comm = nullptr;
        }
        group_drop(h);
        for (auto &S : h->slot) free_slot(h, S);
        nvls_free(h->nvls);
        for (auto &row : h->stage)
            for (auto &st : row)
                if (st.p) {
                    cudaFree(st.p);
                    count_free((int64_t)st.bytes);
                    st.p = nullptr;
                }
        for (auto &e : h->producer_ev)
            if (e) cudaEventDestroy(e), e = nullptr;
        free_det_scratch(h->det);
        if (h->part_base) {
            cudaFree(h->part_base);
            count_free((int64_t)h->part_bytes);
            h->part_base = nullptr;
        }
        if (h->probe_d) {
            cudaFree(h->probe_d);
            count_free(64);
            h->probe_d = nullptr;
        }
        if (h->probe_h) {
            cudaFreeHost(h->probe_h);
            count_free(64);
            h->probe_h = nullptr;
        }
        if (h->probe_ev) cudaEventDestroy(h->probe_ev), h->probe_ev = nullptr;
        if (h->ktrace) cudaFree(h->ktrace), h->ktrace = nullptr;
        if (h->wcache) {
            cudaFree(h->wcache);
            count_free((int64_t)h->lc.sms * 32);
            h->wcache = nullptr;
        }
        if (h->gather) {
            cudaFree(h->gather);
            count_free((int64_t)h->gather_bytes);
            h->gather = nullptr;
        }
        if (h->side) cudaStreamDestroy(h->side);
        if (h->meta_stream) cudaStreamDestroy(h->meta_stream);
        if (h->copy) {
            cudaStreamSynchronize(h->copy);
            cudaStreamDestroy(h->copy);
        }
        h->copy = nullptr;
        if (h->prep) {
            cudaStreamSynchronize(h->prep);
            cudaStreamDestroy(h->prep);
        }
        h->prep = nullptr;
        h->side = nullptr;
        h->meta_stream = nullptr;
    }
    h->finalized = true;
    delete h;
    return rc;
}

}  // extern "C"
