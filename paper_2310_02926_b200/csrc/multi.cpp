// multi.cpp -- bin_multi_*: K DataBin instances over one shared column list,
// executed as one fused launch sequence (multi.cu; SURVEY.md 8(f) row 1,
// PAPER.md:511-514).  Placement, staging and stream ordering follow the
// single-instance operator (handle.cpp, Sec. 3 / PAPER.md:406-435); the
// cross-rank combine is three NCCL allreduces over the
// type-major slot layout: all counts (Sum u64), all sums (Sum f64), all
// min/max words (Min u64).
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdlib.h>
#include <string.h>

#include <string>
#include <vector>

#include "db_internal.h"

using namespace db;

namespace {

enum { MEV_START = 0, MEV_INIT, MEV_BOUNDS, MEV_BIN, MEV_COMBINE, MEV_FINAL, MEV_N };

struct MSlot {
    unsigned char *base = nullptr;
    size_t bytes = 0;
    MultiOp *ops_d = nullptr;          // device instance table (pointers into base)
    std::vector<MultiOp> ops_h;        // host copy of the same table
    unsigned long long *count = nullptr;  // type-major regions (for the NCCL combine)
    double *sum = nullptr;
    unsigned long long *mm = nullptr;
    unsigned long long *bounds = nullptr;
    long long *xs = nullptr;      // exact-sum digits of all exact instances (type-major)
    int32_t *xrange = nullptr;    // 2 * BIN_MAX_ATTR per instance
    uint64_t n_count = 0, n_sum = 0, n_mm = 0, n_bounds = 0, n_xs = 0;
    Meta *meta_d = nullptr;            // [K]
    Meta *meta_h = nullptr;            // pinned mirror
    bool meta_valid = false;
    cudaEvent_t done = nullptr, released = nullptr, zeroed = nullptr;
    cudaEvent_t ev[MEV_N] = {};
    bool recd[MEV_N] = {};
    bool prof_pending = false;
    bool used = false;
    uint64_t ticket = 0;
    cudaStream_t stream = nullptr;
    int launches = 0;
    int variant = 64;
};

}  // namespace

struct bin_multi {
    std::vector<bin_multi_op_t> ops;
    int K = 0, ncols = 0;
    bin_placement_t place{};
    int rank = 0, nranks = 1, device = 0;
    ncclComm_t comm = nullptr;
    cudaStream_t side = nullptr, copy = nullptr, meta_stream = nullptr;
    cudaStream_t prep = nullptr;  // accumulator identities of the next slot, off the critical path
    MSlot slot[2];
    uint64_t next_ticket = 1;
    void *stage[2][BIN_MULTI_MAX_COLS] = {};
    size_t stage_bytes[2][BIN_MULTI_MAX_COLS] = {};
    cudaEvent_t producer_ev[BIN_MULTI_MAX_COLS] = {};
    LaunchCfg lc{};
    uint32_t used_cols = 0, bound_cols = 0;
    uint64_t max_work = 0, max_bins = 0;
    std::vector<int> groups;  // accumulate launches: instances [groups[g], groups[g+1])
    bool prof = false;
    bin_profile_t pacc{};
    cudaStream_t last = nullptr;
    bool finalized = false;
};

static int m_nccl_error(ncclResult_t r, const char *what) {
    return set_error(BIN_ENCCL, "%s: %s", what, ncclGetErrorString(r));
}

// One device allocation per slot: counts of all K | sums of all K | min/max of
// all K | bounds of all K | outputs (min, max, avg) | metas | instance table |
// a zeroed scratch line (window/fxexp words the shared finalize body touches).
static int alloc_mslot(bin_multi *m, MSlot &S) {
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const int K = m->K;
    std::vector<uint64_t> B(K);
    std::vector<int> ns(K), nm(K);
    std::vector<int> nfc(K);
    uint64_t nc = 0, nsu = 0, nmm = 0, nout_mm = 0, nout_avg = 0, nxs = 0, nflt = 0;
    for (int k = 0; k < K; ++k) {
        const bin_spec_t &sp = m->ops[k].spec;
        uint64_t b = 1;
        for (int d = 0; d < sp.ndim; ++d) b *= (uint64_t)sp.res[d];
        B[k] = b;
        ns[k] = nm[k] = 0;
        for (int a = 0; a < sp.nattr; ++a) {
            if (sp.ops[a] & (BIN_OP_SUM | BIN_OP_AVG)) ns[k]++;
            if (sp.ops[a] & (BIN_OP_MIN | BIN_OP_MAX)) nm[k]++;
        }
        if (sp.sum_mode == BIN_SUM_EXACT) nxs += b * ns[k] * XD_DIGITS;
        nfc[k] = nm[k] ? (sp.nattr + 7) / 8 : 0;
        nflt += b * nfc[k] * 16;
        nc += b + 2;
        nsu += b * ns[k];
        nmm += 2 * b * nm[k];
        nout_mm += b * nm[k];
        nout_avg += b * ns[k];
    }
    size_t o = 0;
    const size_t o_count = o; o += al(nc * 8);
    const size_t o_sum = o; o += al(nsu * 8);
    const size_t o_mm = o; o += al(nmm * 8);
    const size_t o_bounds = o; o += al((size_t)K * 6 * 8);
    const size_t o_omin = o; o += al(nout_mm * 8);
    const size_t o_omax = o; o += al(nout_mm * 8);
    const size_t o_oavg = o; o += al(nout_avg * 8);
    const size_t o_meta = o; o += al((size_t)K * sizeof(Meta));
    const size_t o_ops = o; o += al((size_t)K * sizeof(MultiOp));
    const size_t o_scratch = o; o += al(256);
    const size_t o_xrange = o; o += al((size_t)K * 2 * BIN_MAX_ATTR * 4);
    const size_t o_xs = o; o += al(nxs * 8);
    const size_t o_flt = o; o += al(nflt * 4);
    const size_t total = o;
    cudaError_t e = cudaMalloc(&S.base, total);
    if (e != cudaSuccess) {
        cudaGetLastError();
        S.base = nullptr;
        return set_error(BIN_ENOMEM, "bin_multi_init: %zu bytes of bin arrays on device %d", total, m->device);
    }
    S.bytes = total;
    count_alloc((int64_t)total);
    DB_CUDA(cudaMemset(S.base, 0, total));
    unsigned char *b0 = S.base;
    S.count = (unsigned long long *)(b0 + o_count);
    S.sum = (double *)(b0 + o_sum);
    S.mm = (unsigned long long *)(b0 + o_mm);
    S.bounds = (unsigned long long *)(b0 + o_bounds);
    S.n_count = nc, S.n_sum = nsu, S.n_mm = nmm, S.n_bounds = (uint64_t)K * 6;
    S.xrange = (int32_t *)(b0 + o_xrange);
    S.xs = nxs ? (long long *)(b0 + o_xs) : nullptr;
    S.n_xs = nxs;
    DB_CUDA(cudaMemset(S.xrange, 0x7f, (size_t)K * 2 * BIN_MAX_ATTR * 4));
    S.meta_d = (Meta *)(b0 + o_meta);
    S.ops_d = (MultiOp *)(b0 + o_ops);
    S.ops_h.assign(K, MultiOp{});
    uint64_t pc = 0, ps = 0, pm = 0, pomm = 0, poavg = 0, px = 0, pf = 0;
    for (int k = 0; k < K; ++k) {
        const bin_multi_op_t &op = m->ops[k];
        MultiOp &t = S.ops_h[k];
        t.g.ndim = op.spec.ndim;
        t.g.bounds_auto = op.spec.bounds_auto;
        for (int d = 0; d < 3; ++d) {
            t.g.res[d] = d < op.spec.ndim ? op.spec.res[d] : 1;
            t.g.lo[d] = d < op.spec.ndim ? op.spec.lo[d] : 0.0;
            t.g.hi[d] = d < op.spec.ndim ? op.spec.hi[d] : 1.0;
            t.axc[d] = d < op.spec.ndim ? op.axis_col[d] : 0;
        }
        for (int a = 0; a < BIN_MAX_ATTR; ++a) t.atc[a] = a < op.spec.nattr ? op.attr_col[a] : 0;
        t.nattr = op.spec.nattr;
        Accum &acc = t.acc;
        acc.count = S.count + pc;
        acc.sum = S.sum + ps;
        acc.mm = S.mm + pm;
        acc.bounds = S.bounds + (uint64_t)k * 6;
        acc.window = (int32_t *)(b0 + o_scratch);
        acc.fxexp = (uint32_t *)(b0 + o_scratch + 64);
        acc.omin = (double *)(b0 + o_omin) + pomm;
        acc.omax = (double *)(b0 + o_omax) + pomm;
        acc.oavg = (double *)(b0 + o_oavg) + poavg;
        acc.nbins = B[k];
        acc.nsum = ns[k];
        acc.nmm = nm[k];
        for (int a = 0; a < op.spec.nattr; ++a) {
            if (op.spec.ops[a] & (BIN_OP_SUM | BIN_OP_AVG)) acc.sum_mask |= 1u << a;
            if (op.spec.ops[a] & (BIN_OP_MIN | BIN_OP_MAX)) acc.mm_mask |= 1u << a;
        }
        acc.load_mask = acc.sum_mask | acc.mm_mask;
        if (op.spec.sum_mode == BIN_SUM_EXACT && ns[k] > 0) {
            acc.xs = S.xs + px;
            acc.xrange = S.xrange + (size_t)k * 2 * BIN_MAX_ATTR;
            px += B[k] * ns[k] * XD_DIGITS;
        }
        t.flt = nfc[k] ? (uint32_t *)(b0 + o_flt) + pf : nullptr;
        t.nfc = nfc[k];
        pf += B[k] * nfc[k] * 16;
        t.meta = S.meta_d + k;
        pc += B[k] + 2;
        ps += B[k] * ns[k];
        pm += 2 * B[k] * nm[k];
        pomm += B[k] * nm[k];
        poavg += B[k] * ns[k];
    }
    DB_CUDA(cudaMemcpy(S.ops_d, S.ops_h.data(), (size_t)K * sizeof(MultiOp), cudaMemcpyHostToDevice));
    DB_CUDA(cudaHostAlloc((void **)&S.meta_h, (size_t)K * sizeof(Meta), cudaHostAllocPortable));
    count_alloc((int64_t)(K * sizeof(Meta)));
    memset(S.meta_h, 0, (size_t)K * sizeof(Meta));
    DB_CUDA(cudaEventCreateWithFlags(&S.done, cudaEventDisableTiming));
    DB_CUDA(cudaEventCreateWithFlags(&S.released, cudaEventDisableTiming));
    DB_CUDA(cudaEventCreateWithFlags(&S.zeroed, cudaEventDisableTiming));
    for (auto &ev : S.ev) DB_CUDA(cudaEventCreate(&ev));
    return BIN_OK;
}

static void free_mslot(bin_multi *m, MSlot &S) {
    if (S.base) {
        cudaFree(S.base);
        count_free((int64_t)S.bytes);
    }
    S.base = nullptr;
    if (S.meta_h) {
        cudaFreeHost(S.meta_h);
        count_free((int64_t)(m->K * sizeof(Meta)));
    }
    S.meta_h = nullptr;
    if (S.done) cudaEventDestroy(S.done);
    if (S.released) cudaEventDestroy(S.released);
    if (S.zeroed) cudaEventDestroy(S.zeroed);
    S.done = S.released = S.zeroed = nullptr;
    for (auto &e : S.ev)
        if (e) cudaEventDestroy(e), e = nullptr;
}

extern "C" {

int bin_multi_finalize(bin_multi_t *m);

int bin_multi_init(const bin_multi_op_t *ops, int32_t nops, int32_t ncols, const bin_placement_t *place,
                   const bin_comm_t *comm, bin_multi_t **out) {
    if (!ops || !out) return set_error(BIN_EINVAL, "bin_multi_init: NULL ops/out");
    *out = nullptr;
    if (nops < 1 || nops > BIN_MULTI_MAX_OPS)
        return set_error(BIN_EINVAL, "bin_multi_init: %d instances (1..%d)", nops, BIN_MULTI_MAX_OPS);
    if (ncols < 1 || ncols > BIN_MULTI_MAX_COLS)
        return set_error(BIN_EINVAL, "bin_multi_init: %d columns (1..%d)", ncols, BIN_MULTI_MAX_COLS);
    uint32_t used = 0, bound = 0;
    uint64_t max_work = 0, max_bins = 0;
    for (int k = 0; k < nops; ++k) {
        uint64_t B = 0;
        int rc = validate_spec(&ops[k].spec, &B);
        if (rc) {
            const std::string msg = bin_last_error();
            return set_error(rc, "instance %d: %s", k, msg.c_str());
        }
        if (ops[k].spec.deterministic)
            return set_error(BIN_ENOTSUP, "instance %d: deterministic mode is not fused (use bin_init)", k);
        int ns = 0, nm = 0;
        for (int d = 0; d < ops[k].spec.ndim; ++d) {
            const int c = ops[k].axis_col[d];
            if (c < 0 || c >= ncols) return set_error(BIN_EINVAL, "instance %d: axis_col[%d] = %d", k, d, c);
            used |= 1u << c;
            if (ops[k].spec.bounds_auto) bound |= 1u << c;
        }
        for (int a = 0; a < ops[k].spec.nattr; ++a) {
            const uint32_t o = ops[k].spec.ops[a];
            if (o & (BIN_OP_SUM | BIN_OP_AVG)) ns++;
            if (o & (BIN_OP_MIN | BIN_OP_MAX)) nm++;
            if (!o) continue;
            const int c = ops[k].attr_col[a];
            if (c < 0 || c >= ncols) return set_error(BIN_EINVAL, "instance %d: attr_col[%d] = %d", k, a, c);
            used |= 1u << c;
        }
        const uint64_t w = B * (1 + ns + nm);
        if (w > max_work) max_work = w;
        if (B > max_bins) max_bins = B;
    }
    bin_placement_t pl;
    if (place) pl = *place;
    else bin_placement_default(&pl);
    if (pl.exec < BIN_EXEC_SYNC || pl.exec > BIN_EXEC_PEER) return set_error(BIN_EINVAL, "exec %d", pl.exec);
    const int rank = comm ? comm->rank : 0, nranks = comm ? comm->nranks : 1;
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
    int rc = bin_resolve_device(&pl, rank, n_a, &dev);
    if (rc) return rc;

    bin_multi *m = new bin_multi;
    m->ops.assign(ops, ops + nops);
    m->K = nops;
    m->ncols = ncols;
    m->place = pl;
    m->rank = rank;
    m->nranks = nranks;
    m->device = dev;
    m->used_cols = used;
    m->bound_cols = bound;
    m->max_work = max_work;
    m->max_bins = max_bins;
    // Instances are accumulated in groups whose hot lines (count, sums, min/max
    // filter line) together fit an L2 budget: the reductions of one pass land
    // in L2 only while the pass's working set stays resident (C6: 3 instances
    // of 8 MiB per pass measured best).  Each extra group costs
    // one more read of the columns.
    {
        const char *env = getenv("DATABIN_MULTI_L2_MB");
        const double budget = (env ? atof(env) : 24.0) * 1048576.0;
        double acc = 0;
        m->groups.push_back(0);
        for (int k = 0; k < nops; ++k) {
            const bin_spec_t &sp = ops[k].spec;
            double B = 1;
            for (int d = 0; d < sp.ndim; ++d) B *= sp.res[d];
            int ns = 0, nm = 0;
            for (int a2 = 0; a2 < sp.nattr; ++a2) {
                if (sp.ops[a2] & (BIN_OP_SUM | BIN_OP_AVG)) ns++;
                if (sp.ops[a2] & (BIN_OP_MIN | BIN_OP_MAX)) nm++;
            }
            // hot per bin: count, sums and the min/max filter line (the min/max
            // slots themselves are only touched by the rare improving rows)
            const double bytes = B * (8.0 + 8.0 * ns + (nm ? 64.0 * ((sp.nattr + 7) / 8) : 0.0));
            if (k > m->groups.back() && acc + bytes > budget) {
                m->groups.push_back(k);
                acc = 0;
            }
            acc += bytes;
        }
        m->groups.push_back(nops);
    }
    DeviceGuard g(dev);
    auto fail = [&](int code) {
        bin_multi_finalize(m);
        return code;
    };
    if ((ce = cudaStreamCreateWithFlags(&m->side, cudaStreamNonBlocking)) != cudaSuccess)
        return fail(cuda_error(ce, "cudaStreamCreate"));
    if ((ce = cudaStreamCreateWithFlags(&m->copy, cudaStreamNonBlocking)) != cudaSuccess)
        return fail(cuda_error(ce, "cudaStreamCreate"));
    if ((ce = cudaStreamCreateWithFlags(&m->prep, cudaStreamNonBlocking)) != cudaSuccess)
        return fail(cuda_error(ce, "cudaStreamCreate"));
    if ((ce = cudaStreamCreateWithFlags(&m->meta_stream, cudaStreamNonBlocking)) != cudaSuccess)
        return fail(cuda_error(ce, "cudaStreamCreate"));
    for (int d = 0; d < n_a; ++d) {  // NVLink peer copies of columns that live on another GPU
        int can = 0;
        if (d != dev && cudaDeviceCanAccessPeer(&can, dev, d) == cudaSuccess && can) cudaDeviceEnablePeerAccess(d, 0);
        cudaGetLastError();
    }
    cudaDeviceGetAttribute(&m->lc.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&m->lc.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    for (auto &S : m->slot)
        if ((rc = alloc_mslot(m, S))) return fail(rc);
    for (auto &e : m->producer_ev)
        if ((ce = cudaEventCreateWithFlags(&e, cudaEventDisableTiming)) != cudaSuccess)
            return fail(cuda_error(ce, "cudaEventCreate"));
    if (nranks > 1) {
        ncclUniqueId id;
        memcpy(&id, comm->nccl_unique_id, sizeof id);
        ncclResult_t r = ncclCommInitRank(&m->comm, nranks, id, rank);
        if (r != ncclSuccess) {
            m->comm = nullptr;
            return fail(m_nccl_error(r, "ncclCommInitRank"));
        }
    }
    *out = m;
    return BIN_OK;
}

static void m_accumulate_profile(bin_multi *m, MSlot &S);

int bin_multi_execute(bin_multi_t *m, bin_array_t *const *cols, int32_t ncols, uint64_t *ticket) {
    if (!m || m->finalized) return set_error(BIN_ESTATE, "bin_multi_execute: NULL or finalized");
    if (!cols) return set_error(BIN_EINVAL, "bin_multi_execute: NULL cols");
    if (ncols != m->ncols) return set_error(BIN_ESHAPE, "%d columns, the instance set has %d", ncols, m->ncols);
    for (int i = 0; i < ncols; ++i) {
        if (!cols[i]) return set_error(BIN_EINVAL, "column %d is NULL", i);
        if (cols[i]->dtype != BIN_F64) return set_error(BIN_EDTYPE, "column %d is not BIN_F64", i);
        if (cols[i]->n != cols[0]->n)
            return set_error(BIN_ESHAPE, "column %d has %lld rows, column 0 has %lld", i, (long long)cols[i]->n,
                             (long long)cols[0]->n);
    }
    const int64_t n = cols[0]->n;
    DeviceGuard g(m->device);
    const uint64_t t = m->next_ticket++;
    const int sl = (int)(t & 1);
    MSlot &S = m->slot[sl];
    cudaStream_t s = m->side;
    if (m->place.exec == BIN_EXEC_SYNC && is_device_memory(cols[0]) && cols[0]->device == m->device)
        s = cols[0]->stream;  // lockstep: ordered on the producer's stream
    if (S.used && S.prof_pending) {
        DB_CUDA(cudaEventSynchronize(S.done));
        m_accumulate_profile(m, S);
    }
    if (S.used && S.stream != s) DB_CUDA(cudaStreamWaitEvent(s, S.done, 0));
    {
        MSlot &P = m->slot[sl ^ 1];
        if (P.used && P.stream != s) DB_CUDA(cudaStreamWaitEvent(s, P.done, 0));
    }
    const bool had = S.used;
    S.ticket = t;
    S.used = true;
    S.meta_valid = false;
    S.stream = s;
    S.launches = 0;
    m->last = s;
    for (bool &r : S.recd) r = false;
    // ---- a3 for all K on the prep stream, as soon as the slot's previous
    // execute is done (typically while the other slot's execute still runs)
    if (S.xs && n >= (1ll << 30) / m->nranks)  // all ranks' rows < 2^30: digit headroom of the cross-rank add
        return set_error(BIN_EINVAL, "BIN_SUM_EXACT: %lld rows per execute and rank (limit 2^30 / %d ranks)",
                         (long long)n, m->nranks);
    // min/max filter lines pay only once bins see several rows each: below
    // that nearly every row is the first of its bin, passes the filter and
    // would add the filter's own reductions to the slot's (then the lines are
    // neither cleared nor read; measured crossover 4-15 rows per bin)
    static const double flt_rpb = getenv("DATABIN_MULTI_FILTER_RPB") ? atof(getenv("DATABIN_MULTI_FILTER_RPB")) : 8.0;
    const int use_flt = (double)n >= flt_rpb * (double)m->max_bins ? 1 : 0;
    {
        MultiArgs ai{};
        ai.nops = m->K;
        ai.ops = S.ops_d;
        ai.use_flt = use_flt;
        if (had) DB_CUDA(cudaStreamWaitEvent(m->prep, S.done, 0));
        cudaError_t e0 = launch_multi_init(ai, m->max_work, m->prep);
        if (e0 != cudaSuccess) return cuda_error(e0, "multi init kernel");
        S.launches++;
        if (S.xs)  // exact sums: digits cleared; reset every instance's touched range
            DB_CUDA(cudaMemsetAsync(S.xrange, 0x7f, (size_t)m->K * 2 * BIN_MAX_ATTR * 4, m->prep));
        DB_CUDA(cudaEventRecord(S.zeroed, m->prep));
    }
    // ---- a1: view resolution (zero copy on the analysis device, else staged)
    MultiArgs a{};
    a.n = n;
    a.ncols = ncols;
    a.nops = m->K;
    a.used_cols = m->used_cols;
    a.bound_cols = m->bound_cols;
    a.ops = S.ops_d;
    const bool snapshot = m->place.exec == BIN_EXEC_ASYNC && m->place.async_snapshot;
    bool stage[BIN_MULTI_MAX_COLS] = {};
    bool staged_any = false;
    for (int i = 0; i < ncols; ++i) {
        bin_array *c = cols[i];
        const bool local = c->alloc == BIN_ALLOC_CUDA_UVA || (is_device_memory(c) && c->device == m->device);
        stage[i] = n > 0 && ((m->used_cols >> i) & 1u) && (!local || snapshot);
        staged_any = staged_any || stage[i];
    }
    if (staged_any && had) DB_CUDA(cudaStreamWaitEvent(m->copy, S.done, 0));
    for (int i = 0; i < ncols; ++i) {
        bin_array *c = cols[i];
        const double *p = (const double *)c->ptr;
        if (!((m->used_cols >> i) & 1u)) {
            a.col[i] = p;
            continue;
        }
        cudaStream_t consumer = stage[i] ? m->copy : s;
        if (c->stream != consumer && (c->device >= 0 || c->alloc == BIN_ALLOC_HOST_PINNED)) {
            const int pd = c->device >= 0 ? c->device : m->device;
            if (pd != m->device) {
                DeviceGuard g2(pd);
                cudaEvent_t tmp;
                DB_CUDA(cudaEventCreateWithFlags(&tmp, cudaEventDisableTiming));
                DB_CUDA(cudaEventRecord(tmp, c->stream));
                DeviceGuard g3(m->device);
                DB_CUDA(cudaStreamWaitEvent(consumer, tmp, 0));
                cudaEventDestroy(tmp);
            } else {
                DB_CUDA(cudaEventRecord(m->producer_ev[i], c->stream));
                DB_CUDA(cudaStreamWaitEvent(consumer, m->producer_ev[i], 0));
            }
        }
        if (stage[i]) {
            const size_t bytes = (size_t)n * 8;
            if (m->stage_bytes[sl][i] < bytes) {
                if (m->stage[sl][i]) {
                    cudaFree(m->stage[sl][i]);
                    count_free((int64_t)m->stage_bytes[sl][i]);
                }
                m->stage_bytes[sl][i] = 0;
                m->stage[sl][i] = dev_alloc(bytes, m->device, nullptr, false);
                if (!m->stage[sl][i]) return set_error(BIN_ENOMEM, "staging buffer of %zu bytes", bytes);
                m->stage_bytes[sl][i] = bytes;
            }
            void *dst = m->stage[sl][i];
            if (c->device == -1 || c->alloc == BIN_ALLOC_HOST || c->alloc == BIN_ALLOC_HOST_PINNED)
                DB_CUDA(cudaMemcpyAsync(dst, c->ptr, bytes, cudaMemcpyHostToDevice, m->copy));
            else if (c->device != m->device && c->alloc != BIN_ALLOC_CUDA_UVA)
                DB_CUDA(cudaMemcpyPeerAsync(dst, m->device, c->ptr, c->device, bytes, m->copy));
            else
                DB_CUDA(cudaMemcpyAsync(dst, c->ptr, bytes, cudaMemcpyDeviceToDevice, m->copy));
            p = (const double *)dst;
        }
        a.col[i] = p;
    }
    if (staged_any) {
        DB_CUDA(cudaEventRecord(S.released, m->copy));
        DB_CUDA(cudaStreamWaitEvent(s, S.released, 0));
    }
    auto rec = [&](int k, bool work) -> int {
        if (m->prof && work) {
            DB_CUDA(cudaEventRecord(S.ev[k], s));
            S.recd[k] = true;
        }
        return BIN_OK;
    };
    // profiled phases start once the inputs are ready (after the producer /
    // staging waits): the phase times are the analysis' own device time
    int rc;
    if ((rc = rec(MEV_START, true))) return rc;
    cudaError_t e;
    DB_CUDA(cudaStreamWaitEvent(s, S.zeroed, 0));  // identities (enqueued on the prep stream above)
    if ((rc = rec(MEV_INIT, true))) return rc;
    // ---- a2 for every auto-bounded axis column (+ cross-rank Min)
    if (m->bound_cols) {
        if ((e = launch_multi_bounds(a, m->lc, s)) != cudaSuccess) return cuda_error(e, "multi bounds kernel");
        if (n > 0) S.launches++;
        if (m->comm) {
            ncclResult_t r = ncclAllReduce(S.bounds, S.bounds, S.n_bounds, ncclUint64, ncclMin, m->comm, s);
            if (r != ncclSuccess) return m_nccl_error(r, "ncclAllReduce(bounds)");
        }
    }
    if ((rc = rec(MEV_BOUNDS, m->bound_cols != 0))) return rc;
    a.use_flt = use_flt;
    // ---- a4 + a5 for all K: one pass over the rows per L2-sized group; with
    // under ~3 rows per bin all K go in one pass (the lines are touched about
    // once each, residency buys little, and the launch spreads the instances
    // over grid.y: C6 at 46,875 rows 0.183 -> 0.160 ms, 131,072 0.275 -> 0.261)
    static const double one_pass_rpb = getenv("DATABIN_MULTI_ONEPASS_RPB") ? atof(getenv("DATABIN_MULTI_ONEPASS_RPB")) : 3.0;
    const bool one_pass = (double)n < one_pass_rpb * (double)m->max_bins;
    const size_t ngroups = one_pass ? 1 : m->groups.size() - 1;
    for (size_t gi = 0; gi < ngroups; ++gi) {
        a.k0 = one_pass ? 0 : m->groups[gi];
        a.k1 = one_pass ? m->K : m->groups[gi + 1];
        if ((e = launch_multi_bin(a, m->lc, s)) != cudaSuccess) return cuda_error(e, "multi bin kernel");
        if (n > 0) S.launches++;
    }
    if ((rc = rec(MEV_BIN, n > 0))) return rc;
    // ---- a6: one NCCL group over the type-major regions of all K
    if (m->comm) {
        ncclResult_t r = ncclGroupStart();
        if (r == ncclSuccess) r = ncclAllReduce(S.count, S.count, S.n_count, ncclUint64, ncclSum, m->comm, s);
        if (r == ncclSuccess && S.n_sum) r = ncclAllReduce(S.sum, S.sum, S.n_sum, ncclFloat64, ncclSum, m->comm, s);
        if (r == ncclSuccess && S.n_mm) r = ncclAllReduce(S.mm, S.mm, S.n_mm, ncclUint64, ncclMin, m->comm, s);
        if (r == ncclSuccess && S.n_xs) {  // exact sums: integer digits add exactly; ranges unite
            r = ncclAllReduce(S.xs, S.xs, S.n_xs, ncclInt64, ncclSum, m->comm, s);
            if (r == ncclSuccess)
                r = ncclAllReduce(S.xrange, S.xrange, (size_t)m->K * 2 * BIN_MAX_ATTR, ncclInt32, ncclMin, m->comm, s);
        }
        ncclResult_t r2 = ncclGroupEnd();
        if (r != ncclSuccess) return m_nccl_error(r, "ncclAllReduce(multi bins)");
        if (r2 != ncclSuccess) return m_nccl_error(r2, "ncclGroupEnd");
    }
    if ((rc = rec(MEV_COMBINE, m->comm != nullptr))) return rc;
    // ---- a7 for all K
    if ((e = launch_multi_finalize(a, m->max_bins, s)) != cudaSuccess) return cuda_error(e, "multi finalize kernel");
    S.launches++;
    if ((rc = rec(MEV_FINAL, true))) return rc;
    DB_CUDA(cudaEventRecord(S.done, s));
    if (!staged_any) DB_CUDA(cudaEventRecord(S.released, s));
    S.prof_pending = m->prof;
    for (int i = 0; i < ncols; ++i)
        if ((m->used_cols >> i) & 1u)
            if ((rc = array_mark_use(cols[i], s, m->device))) return rc;
    if (ticket) *ticket = t;
    if (m->place.exec == BIN_EXEC_SYNC && cols[0]->mode == BIN_SYNC) {
        e = cudaEventSynchronize(S.done);
        if (e != cudaSuccess) return cuda_error(e, "bin_multi_execute (lockstep) synchronize");
    }
    return BIN_OK;
}

static MSlot *m_find(bin_multi *m, uint64_t t) {
    MSlot &S = m->slot[t & 1];
    return (S.used && S.ticket == t) ? &S : nullptr;
}

static int m_fetch_meta(bin_multi *m, MSlot &S) {
    if (S.meta_valid) return BIN_OK;
    DB_CUDA(cudaMemcpyAsync(S.meta_h, S.meta_d, (size_t)m->K * sizeof(Meta), cudaMemcpyDeviceToHost, m->meta_stream));
    DB_CUDA(cudaStreamSynchronize(m->meta_stream));
    S.meta_valid = true;
    return BIN_OK;
}

static void m_accumulate_profile(bin_multi *m, MSlot &S) {
    if (!S.prof_pending) return;
    S.prof_pending = false;
    float ms[MEV_N] = {};
    for (int k = 1, last = MEV_START; k < MEV_N; ++k)
        if (S.recd[k]) {
            cudaEventElapsedTime(&ms[k], S.ev[last], S.ev[k]);
            last = k;
        }
    cudaGetLastError();
    bin_profile_t &p = m->pacc;
    p.ms_init += ms[MEV_INIT];
    p.ms_bounds += ms[MEV_BOUNDS];
    p.ms_bin += ms[MEV_BIN];
    p.ms_combine += ms[MEV_COMBINE];
    p.ms_finalize += ms[MEV_FINAL];
    p.executes += 1;
    p.kernel_launches += S.launches;
    p.bin_launches += 1;
    p.variant = S.variant;
}

int bin_multi_inputs_released(bin_multi_t *m, uint64_t ticket, bin_event_t *ev) {
    if (!m || !ev) return set_error(BIN_EINVAL, "bin_multi_inputs_released: NULL argument");
    MSlot *S = m_find(m, ticket);
    if (!S) return set_error(BIN_ESTATE, "unknown or recycled ticket %llu", (unsigned long long)ticket);
    *ev = (bin_event_t)S->released;
    return BIN_OK;
}

int bin_multi_wait(bin_multi_t *m, uint64_t ticket) {
    if (!m || m->finalized) return set_error(BIN_ESTATE, "bin_multi_wait: NULL or finalized");
    MSlot *S = m_find(m, ticket);
    if (!S) return set_error(BIN_ESTATE, "unknown or recycled ticket %llu", (unsigned long long)ticket);
    DeviceGuard g(m->device);
    cudaError_t e = cudaEventSynchronize(S->done);
    if (e != cudaSuccess) return cuda_error(e, "bin_multi_wait");
    int rc = m_fetch_meta(m, *S);
    if (rc) return rc;
    m_accumulate_profile(m, *S);
    for (int k = 0; k < m->K; ++k)
        if (S->meta_h[k].status == BIN_EDEGENERATE)
            return set_error(BIN_EDEGENERATE, "instance %d: auto bounds with no finite rows in total", k);
    return BIN_OK;
}

int bin_multi_result(bin_multi_t *m, uint64_t ticket, int32_t op, bin_result_t *out) {
    if (!out) return set_error(BIN_EINVAL, "bin_multi_result: NULL out");
    if (!m || op < 0 || op >= m->K) return set_error(BIN_EINVAL, "bin_multi_result: instance %d", op);
    int rc = bin_multi_wait(m, ticket);
    if (rc) return rc;
    MSlot &S = *m_find(m, ticket);
    const MultiOp &t = S.ops_h[op];
    const bin_spec_t &sp = m->ops[op].spec;
    memset(out, 0, sizeof *out);
    const uint64_t B = t.acc.nbins;
    out->count = (const uint64_t *)t.acc.count;
    for (int a = 0; a < sp.nattr; ++a) {
        const uint32_t o = sp.ops[a];
        if ((t.acc.sum_mask >> a) & 1u) {
            const int slot = __builtin_popcount(t.acc.sum_mask & ((1u << a) - 1u));
            if (o & BIN_OP_SUM) out->sum[a] = t.acc.sum + (uint64_t)slot * B;
            if (o & BIN_OP_AVG) out->avg[a] = t.acc.oavg + (uint64_t)slot * B;
        }
        if ((t.acc.mm_mask >> a) & 1u) {
            const int slot = __builtin_popcount(t.acc.mm_mask & ((1u << a) - 1u));
            if (o & BIN_OP_MIN) out->min[a] = t.acc.omin + (uint64_t)slot * B;
            if (o & BIN_OP_MAX) out->max[a] = t.acc.omax + (uint64_t)slot * B;
        }
    }
    out->nbins = B;
    out->n_in = S.meta_h[op].n_in;
    out->n_out = S.meta_h[op].n_out;
    out->device = m->device;
    for (int d = 0; d < 3; ++d) {
        out->lo[d] = d < sp.ndim ? S.meta_h[op].lo[d] : 0.0;
        out->hi[d] = d < sp.ndim ? S.meta_h[op].hi[d] : 0.0;
    }
    return BIN_OK;
}

int bin_multi_profile_enable(bin_multi_t *m, int32_t on) {
    if (!m) return set_error(BIN_EINVAL, "bin_multi_profile_enable: NULL");
    m->prof = on != 0;
    memset(&m->pacc, 0, sizeof m->pacc);
    return BIN_OK;
}

int bin_multi_profile_read(bin_multi_t *m, bin_profile_t *out) {
    if (!m || !out) return set_error(BIN_EINVAL, "bin_multi_profile_read: NULL");
    DeviceGuard g(m->device);
    for (auto &S : m->slot)
        if (S.used && S.prof_pending) {
            DB_CUDA(cudaEventSynchronize(S.done));
            m_accumulate_profile(m, S);
        }
    *out = m->pacc;
    return BIN_OK;
}

int bin_multi_stream(bin_multi_t *m, bin_stream_t *stream) {
    if (!m || !stream) return set_error(BIN_EINVAL, "bin_multi_stream: NULL");
    *stream = (bin_stream_t)(m->last ? m->last : m->side);
    return BIN_OK;
}

int bin_multi_finalize(bin_multi_t *m) {
    if (!m) return BIN_OK;
    int rc = BIN_OK;
    {
        DeviceGuard g(m->device);
        for (auto &S : m->slot)
            if (S.done) {
                cudaError_t e = cudaEventSynchronize(S.done);
                if (e != cudaSuccess && rc == BIN_OK) rc = cuda_error(e, "bin_multi_finalize");
            }
        if (m->side) cudaStreamSynchronize(m->side);
        if (m->copy) cudaStreamSynchronize(m->copy);
        if (m->comm) {
            ncclCommDestroy(m->comm);
            m->comm = nullptr;
        }
        for (auto &S : m->slot) free_mslot(m, S);
        for (int s = 0; s < 2; ++s)
            for (int i = 0; i < BIN_MULTI_MAX_COLS; ++i)
                if (m->stage[s][i]) {
                    cudaFree(m->stage[s][i]);
                    count_free((int64_t)m->stage_bytes[s][i]);
                    m->stage[s][i] = nullptr;
                }
        for (auto &e : m->producer_ev)
            if (e) cudaEventDestroy(e), e = nullptr;
        if (m->side) cudaStreamDestroy(m->side);
        if (m->copy) cudaStreamDestroy(m->copy);
        if (m->meta_stream) cudaStreamDestroy(m->meta_stream);
        if (m->prep) {
            cudaStreamSynchronize(m->prep);
            cudaStreamDestroy(m->prep);
        }
        m->side = m->copy = m->meta_stream = m->prep = nullptr;
    }
    m->finalized = true;
    delete m;
    return rc;
}

}  // extern "C"
