/*
 * databin.h -- C ABI of the B200-native in situ DataBin library
 * (libdatabin.so, built from paper_2310_02926_b200/csrc/).
 *
 * The library implements the data-parallel hot path of arXiv 2310.02926
 * ("Extensions to the SENSEI In situ Framework for Heterogeneous
 * Architectures"): the DataBin analysis of Sec. 4.2,
 * fed through a HAMR-like zero-copy array handle (Sec. 2)
 * and placed/executed per the execution-model extensions of Sec. 3
 * (PAPER.md:406-435).
 *
 * Conventions for every function below
 *   - Return value: BIN_OK (0) or one of the BIN_E* codes.  A thread-local
 *     message for the last failure is available from bin_last_error().
 *   - Pointers are plain host or device addresses; sizes are element counts
 *     unless stated.  No function takes or returns a torch type.
 *   - Streams/events are CUDA runtime handles passed as opaque pointers
 *     (bin_stream_t == cudaStream_t, bin_event_t == cudaEvent_t); NULL means
 *     the legacy default stream.
 *   - Asynchronous CUDA faults are sticky: they surface as BIN_ECUDA from the
 *     next bin_wait / bin_result / bin_finalize / bin_array_synchronize.
 *   - No CPU fallback exists: every binning step runs in the library's CUDA
 *     kernels (sm_100a).  Host placement (device_id == -1) is BIN_ENOTSUP.
 */
#ifndef DATABIN_H
#define DATABIN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *bin_stream_t; /* == cudaStream_t */
typedef struct CUevent_st *bin_event_t;   /* == cudaEvent_t  */

/* ---- error codes ---- */
enum {
    BIN_OK = 0,
    BIN_EINVAL = 1,      /* bad argument or spec (lo >= hi, res <= 0, prod(res) >= 2^32, ...) */
    BIN_ESHAPE = 2,      /* column lengths differ or wrong column count */
    BIN_EDTYPE = 3,      /* element type is not BIN_F64 */
    BIN_EDEVICE = 4,     /* bad device id, or peer access impossible */
    BIN_EDEGENERATE = 5, /* auto bounds over zero rows in total, or unrecoverable lo == hi */
    BIN_ENOMEM = 6,      /* an allocation failed */
    BIN_ENOTSUP = 7,     /* host placement, ndim outside 1..3, nattr > 16 */
    BIN_ECUDA = 8,       /* CUDA runtime error (message has the CUDA string) */
    BIN_ENCCL = 9,       /* NCCL error */
    BIN_ESTATE = 10      /* call out of order (unknown ticket, handle finalized, ...) */
};

/* ---- element types ---- */
enum { BIN_F64 = 0 }; /* the HDA examples are svtkHAMRDoubleArray */

/* ---- array handle: the paper's svtkHAMRDataArray (HDA), Sec. 2 ----
 * Allocators mirror svtkAllocator: host malloc, page-locked
 * host, CUDA synchronous / stream-ordered asynchronous / universally
 * addressable (managed), and EXTERNAL for memory the library did not
 * allocate and will never free itself. */
typedef enum {
    BIN_ALLOC_HOST = 0,
    BIN_ALLOC_HOST_PINNED = 1,
    BIN_ALLOC_CUDA = 2,
    BIN_ALLOC_CUDA_ASYNC = 3,
    BIN_ALLOC_CUDA_UVA = 4,
    BIN_ALLOC_EXTERNAL = 5
} bin_allocator_t;

/* svtkStreamMode: SYNC = every operation issued for the
 * array has completed before the issuing call returns; ASYNC = the call may
 * return while the operation is in flight; the user synchronizes. */
typedef enum { BIN_SYNC = 0, BIN_ASYNC = 1 } bin_stream_mode_t;

typedef struct bin_array bin_array_t; /* opaque, reference counted */

/* Zero-copy wrap of externally allocated memory (PAPER.md:346-360,
 * Listing 1).  Captures: ptr, length n (elements), dtype, the device the
 * memory lives on (-1 = host), the allocator that manages it, the stream
 * that orders operations on it, and the stream mode.
 * Ownership: if release != NULL it is called exactly once as
 * release(release_ctx, ptr) when the last reference (the array and every
 * accessible view of it) is released AND all library work reading it has
 * drained -- the shared_ptr-with-deleter contract of Listing 1.  With
 * release == NULL the pointer is borrowed and the caller manages its life
 * (PAPER.md:359-360).  Performs no allocation of any kind.
 * Errors: BIN_EINVAL (ptr NULL with n > 0, n < 0), BIN_EDTYPE, BIN_EDEVICE. */
int bin_array_wrap(const void *ptr, int64_t n, int32_t dtype, int32_t device,
                   bin_allocator_t alloc, bin_stream_t stream,
                   bin_stream_mode_t mode,
                   void (*release)(void *release_ctx, void *ptr),
                   void *release_ctx, bin_array_t **out);

/* Allocating constructor (Listing 2).  Memory is allocated
 * with `alloc` on `device` (ignored for host allocators); for
 * BIN_ALLOC_CUDA_ASYNC the allocation is stream-ordered on `stream`.
 * If fill != NULL every element is set to *fill (on `stream`; complete on
 * return when mode == BIN_SYNC).  The library frees the memory on release.
 * Errors: BIN_EINVAL, BIN_EDTYPE, BIN_EDEVICE, BIN_ENOMEM, BIN_ECUDA. */
int bin_array_alloc(int64_t n, int32_t dtype, int32_t device,
                    bin_allocator_t alloc, bin_stream_t stream,
                    bin_stream_mode_t mode, const double *fill,
                    bin_array_t **out);

/* Direct access (GetData): the raw pointer in the
 * array's own location.  No allocation, no transfer. */
int bin_array_data(bin_array_t *a, void **ptr);

/* Metadata query: length, device (-1 host), allocator, stream. */
int bin_array_info(const bin_array_t *a, int64_t *n, int32_t *device,
                   int32_t *alloc, bin_stream_t *stream);

/* Location-agnostic read-only access (GetCUDAAccessible / GetHostAccessible,
 * PAPER.md:381-389).  device >= 0 requests device memory on that GPU,
 * device == -1 requests host memory.  If the data is already accessible
 * there (same device; managed memory from anywhere; host memory for a host
 * request) *ptr is the array's own pointer and no work is done.  Otherwise a
 * temporary is allocated at the requested location and an asynchronous copy
 * (H2D, D2H or peer over NVLink) is enqueued on `stream` (NULL = the array's
 * stream); call bin_array_synchronize(*view) before reading when the array's
 * mode is BIN_ASYNC.  *view is a new reference that keeps the temporary (or
 * the source) alive; release it with bin_array_release.
 * Errors: BIN_EDEVICE, BIN_ENOMEM, BIN_ECUDA. */
int bin_array_get_accessible(bin_array_t *a, int32_t device,
                             bin_stream_t stream, const void **ptr,
                             bin_array_t **view);

/* Waits for every operation enqueued for this array (fills, moves) to
 * complete (Synchronize()). */
int bin_array_synchronize(bin_array_t *a);

/* Drops one reference.  At the last reference: waits for in-flight library
 * work that reads the array, frees library-owned memory, or calls the
 * wrap's release callback exactly once. NULL is a no-op. */
void bin_array_release(bin_array_t *a);

/* Allocation counters of the library's allocator (zero-copy discipline
 * tests): live allocations, allocations ever made, live bytes. */
void bin_alloc_stats(int64_t *live, int64_t *total, int64_t *live_bytes);

/* ---- the DataBin operator, Sec. 4.2 ---- */
enum { BIN_OP_SUM = 1, BIN_OP_MIN = 2, BIN_OP_MAX = 4, BIN_OP_AVG = 8 };
#define BIN_MAX_DIM 3
#define BIN_MAX_ATTR 16

typedef struct {
    int32_t ndim;               /* 1..3 coordinate axes */
    int32_t res[BIN_MAX_DIM];   /* cells per axis; prod(res) < 2^32 */
    int32_t bounds_auto;        /* 0: lo/hi below; 1: global min/max of each axis */
    double lo[BIN_MAX_DIM];     /* manual bounds, lo < hi, finite */
    double hi[BIN_MAX_DIM];
    int32_t nattr;              /* 0..16 binned (non-coordinate) variables */
    uint32_t ops[BIN_MAX_ATTR]; /* per attribute: OR of BIN_OP_* (AVG implies SUM) */
    int32_t deterministic;      /* 1: sums bit-identical to the sequential oracle
                                   in partition mode P = nranks (slow; correctness mode) */
    int32_t route;              /* accumulate route (speed only; results agree within the sum
                                   tolerance): BIN_ROUTE_AUTO (0, default) picks from a 16,384-row
                                   sample at the first execute (one host wait) and re-checks it
                                   asynchronously every 64 executes; BIN_ROUTE_WINDOW: shared-memory
                                   hot window + L2 reductions (clustered data); BIN_ROUTE_PARTITION:
                                   rows grouped by bin tile, then accumulated tile by tile in shared
                                   memory (spread-out data, large meshes).  Ignored when
                                   deterministic; falls back to the window route when the
                                   partition plan does not apply (> 4 attributes read, n >= 2^32,
                                   unaligned columns, > 8192 tiles). */
    int32_t sum_mode;           /* BIN_SUM_FAST (0, default): sums accumulated in an unspecified order
                                   (within 1e-12 * sum|v| of the row-order sum, R8);
                                   BIN_SUM_EXACT: every bin's sum is its exact real sum rounded once
                                   to nearest-even (R20; zero -> +0.0, beyond DBL_MAX ->
                                   +-inf), avg = that sum / count -- identical across runs, routes and
                                   rank counts.  Needs finite attribute values (R7), fewer than
                                   2^30 / nranks rows per execute and rank (all ranks' rows < 2^30:
                                   digit headroom of the cross-rank add), and deterministic == 0
                                   (else BIN_EINVAL);
                                   costs 66 x 8 bytes per bin and summed attribute of device memory. */
} bin_spec_t;
enum { BIN_ROUTE_AUTO = 0, BIN_ROUTE_WINDOW = 1, BIN_ROUTE_PARTITION = 2 };
enum { BIN_SUM_FAST = 0, BIN_SUM_EXACT = 1 };

/* Execution method + placement (Sec. 3; XML attributes at PAPER.md:426-433). */
enum { BIN_EXEC_SYNC = 0, BIN_EXEC_ASYNC = 1, BIN_EXEC_PEER = 2 };
enum { BIN_DEVICE_HOST = -1, BIN_DEVICE_AUTO = -2 };
typedef struct {
    int32_t device_id;      /* -2 auto by Eq. (1) (default), >= 0 explicit, -1 host -> BIN_ENOTSUP */
    int32_t device_start;   /* d_0 in Eq. (1), default 0 */
    int32_t device_stride;  /* s in Eq. (1), default 1 */
    int32_t devices_to_use; /* n_u in Eq. (1); <= 0 means n_a (default) */
    int32_t exec;           /* BIN_EXEC_SYNC: lockstep, ordered on the data's stream
                               BIN_EXEC_ASYNC: side stream concurrent with the producer
                               BIN_EXEC_PEER: analysis on another GPU, inputs moved over NVLink */
    int32_t async_snapshot; /* ASYNC only: 1 = deep-copy the inputs first (the paper's method),
                               0 = read in place; bin_inputs_released tells when the producer may overwrite */
} bin_placement_t;

/* Multi-rank combine: ranks bin their own rows and every rank
 * receives the combined grid (reading R21).  nccl_unique_id points at a
 * 128-byte ncclUniqueId created by bin_nccl_unique_id on rank 0 and broadcast
 * by the caller (NULL when nranks == 1).  The combine is chosen at bin_init
 * (environment variable DATABIN_COMBINE, which must be the same on every
 * rank): default -- one kernel that reduces the rank's bin slice from every
 * rank's accumulators over NVLink peer memory (CUDA IPC), finalizes it and
 * writes it into every rank, when all ranks are on distinct GPUs of one node;
 * "nvls" -- the same, reduced in the NVSwitch (multicast memory); "nccl" --
 * NCCL allreduces + a finalize kernel (also the fallback when peer mapping
 * fails).  Deterministic handles fold the ranks' sums in rank order. */
typedef struct {
    int32_t rank, nranks;
    const void *nccl_unique_id;
} bin_comm_t;

typedef struct bin_handle bin_handle_t; /* opaque */

/* Output of one execute (device pointers on result.device, library-owned,
 * valid until the second following bin_execute on the handle, or
 * bin_finalize).  Bins are linearised x fastest: b = k0 + res0*(k1 + res1*k2).
 * Empty bins: count 0, sum +0.0, min +inf, max -inf, avg NaN.  Arrays for
 * ops not requested are NULL. */
typedef struct {
    const uint64_t *count;
    const double *sum[BIN_MAX_ATTR];
    const double *min[BIN_MAX_ATTR];
    const double *max[BIN_MAX_ATTR];
    const double *avg[BIN_MAX_ATTR];
    uint64_t nbins;
    uint64_t n_in, n_out;     /* rows inside / outside the mesh, summed over ranks */
    int32_t device;
    double lo[BIN_MAX_DIM], hi[BIN_MAX_DIM]; /* realised bounds (auto: global min/max, widened if lo == hi) */
} bin_result_t;

/* Per-phase device time accumulated over executes while profiling is on,
 * measured with CUDA events on the stream each phase is launched on. */
typedef struct {
    double ms_bounds, ms_init, ms_window, ms_bin, ms_combine, ms_finalize, ms_stage;
    int64_t executes;
    int64_t kernel_launches;  /* library kernels launched (all phases) */
    int64_t bin_launches;     /* launches of the accumulate kernel */
    int32_t variant;          /* last accumulate variant (low 4 bits): 1 smem window + L2, 2 smem full grid,
                                 3 deterministic, 4 partition route; +16 when the single-attribute
                                 k_bin_fast kernel ran, +32 when the NVLink peer combine ran,
                                 +64 when it ran in the switch (NVLS, DATABIN_COMBINE=nvls) */
    int32_t window[BIN_MAX_DIM]; /* last window extents (bins), 0 = no window */
} bin_profile_t;

/* Fills *p with the defaults of PAPER.md:422 / :428 (device_id = -2,
 * d_0 = 0, s = 1, n_u = n_a, lockstep, snapshot on). */
void bin_placement_default(bin_placement_t *p);

/* Eq. (1): d = ((r mod n_u) * s + d_0) mod n_a  (reading R14),
 * or the explicit device, wrapped modulo n_a like Eq. (1) itself (reading
 * R14b).  Host-only, needs no GPU.  n_avail = n_a.
 * Errors: BIN_ENOTSUP (device_id == -1), BIN_EDEVICE (device_id < -2 or
 * n_avail < 1), BIN_EINVAL (stride < 1, device_start < 0). */
int bin_resolve_device(const bin_placement_t *p, int32_t rank, int32_t n_avail,
                       int32_t *device);

/* Creates an operator instance: validates the spec, resolves the analysis
 * device (Eq. 1 with rank = comm->rank), creates streams and, for
 * nranks > 1, the NCCL communicator.  comm may be NULL (single rank).
 * Errors: BIN_EINVAL, BIN_ENOTSUP, BIN_EDEVICE, BIN_ENCCL, BIN_ECUDA. */
int bin_init(const bin_spec_t *spec, const bin_placement_t *place,
             const bin_comm_t *comm, bin_handle_t **out);

/* Bins one batch of rows: axes[0..ndim) and attrs[0..nattr) are equal-length
 * f64 columns (any location; moved as needed per the placement).  Enqueues
 * the whole path -- view resolution, [auto bounds + allreduce], accumulator
 * init, binning, cross-rank combine, finalize -- and returns a ticket.
 * SYNC exec returns after enqueue on the data's stream (lockstep in stream
 * order); it blocks until completion only if the first axis array's mode is
 * BIN_SYNC.  ASYNC/PEER return after enqueue.
 * Errors: BIN_ESHAPE, BIN_EDTYPE, BIN_EDEVICE, BIN_ENOMEM, BIN_ECUDA, BIN_ENCCL. */
int bin_execute(bin_handle_t *h, bin_array_t *const *axes, int32_t naxes,
                bin_array_t *const *attrs, int32_t nattr, uint64_t *ticket);

/* Fan-in execute (the paper's "dedicated device" placement, PAPER.md:496-497:
 * "Data is moved from the three simulation GPUs ... to the one in situ GPU"):
 * bins nshards row blocks -- e.g. the arrays of several producer GPUs -- as ONE
 * batch into one result.  Shard s's columns are axes[s*naxes + d] and
 * attrs[s*nattr + a]; columns agree in length within a shard, shards may
 * differ in length and live anywhere (host, this GPU, other GPUs).  Every
 * column is staged on the handle's copy stream into one buffer, shard after
 * shard (NVLink peer copies from other GPUs run concurrently with the
 * previous execute), each copy ordered after its producer stream's pending
 * work; then the execute proceeds as bin_execute over the concatenated rows
 * (deterministic mode folds them in shard order).  nshards == 1 is
 * bin_execute.  Errors: as bin_execute; BIN_EINVAL for nshards outside
 * 1..BIN_MAX_SHARDS. */
#define BIN_MAX_SHARDS 64
int bin_execute_shards(bin_handle_t *h, bin_array_t *const *axes, int32_t naxes,
                       bin_array_t *const *attrs, int32_t nattr, int32_t nshards, uint64_t *ticket);

/* One-device rank group (PAPER.md:479 with Eq. (1): when there are
 * more ranks than devices, several ranks bin on one GPU).  bin_init_group
 * creates nranks (1..16) handles out[0..nranks) on ONE device (resolved from
 * `place` for rank 0), rank r = out[r]; each bins only its own rows into its
 * own accumulators, exactly as one process per GPU does, and the group's
 * combine is the fused peer combine + finalize kernel of the multi-GPU path
 * (same device code: barrier words, rank-order sum fold, exact-digit add,
 * min/max, finalize, all-gather of the results into every rank) launched once
 * for all ranks.  Results of rank r equal a multi-process run with nranks
 * ranks -- in deterministic / exact mode the oracle's partition mode P = nranks
 * bit for bit.  Manual bounds only (auto bounds: BIN_ENOTSUP).  Each handle
 * is finalized with bin_finalize; bin_execute on a member is BIN_ESTATE.
 * Errors: as bin_init; BIN_EINVAL for nranks outside 1..16 or NULL pointers. */
int bin_init_group(const bin_spec_t *spec, const bin_placement_t *place, int32_t nranks, bin_handle_t **out);

/* Collective execute of a rank group: h[r] (rank r, all nranks members in
 * order) bins rank r's columns axes[r*naxes + d], attrs[r*nattr + a] on its
 * own work stream (placement as bin_execute), then one launch combines and
 * finalizes all ranks after every rank has binned; each rank's result is then
 * available through bin_wait / bin_result on its own handle with the shared
 * *ticket.  The combine launch spins on barrier words inside the kernel, so it
 * uses at most one CTA per SM in total and needs them co-resident: other work
 * that fills every SM of the device at the same time can delay it past its
 * ~2 s barrier timeout (reported as BIN_ENCCL at bin_wait, never a hang).
 * Errors: as bin_execute; BIN_ESTATE when a handle is not rank r of the group,
 * was finalized, or the ranks' tickets differ (e.g. after a failed group
 * execute: the group must then be finalized and re-created). */
int bin_execute_group(bin_handle_t *const *h, int32_t nranks, bin_array_t *const *axes, int32_t naxes,
                      bin_array_t *const *attrs, int32_t nattr, uint64_t *ticket);

/* Event after which the producer may overwrite the inputs of `ticket`
 * (snapshot copy done, or binning done when reading in place). */
int bin_inputs_released(bin_handle_t *h, uint64_t ticket, bin_event_t *ev);

/* Blocks until `ticket` is complete; surfaces async CUDA/NCCL faults and
 * BIN_EDEGENERATE (auto bounds over zero rows). */
int bin_wait(bin_handle_t *h, uint64_t ticket);

/* Waits like bin_wait, then fills *out. */
int bin_result(bin_handle_t *h, uint64_t ticket, bin_result_t *out);

/* The stream the handle enqueues its work on for the last execute. */
int bin_stream(bin_handle_t *h, bin_stream_t *stream);

/* Profiling: on != 0 starts accumulating per-phase event times (resets). */
int bin_profile_enable(bin_handle_t *h, int32_t on);
int bin_profile_read(bin_handle_t *h, bin_profile_t *out);

/* Drains all streams, frees every library buffer, destroys the NCCL
 * communicator and the handle.  NULL is a no-op returning BIN_OK. */
int bin_finalize(bin_handle_t *h);

/* Writes a fresh 128-byte ncclUniqueId to out (rank 0 calls it). */
int bin_nccl_unique_id(void *out128);

/* Utility for bindings: stream-ordered copy between any two addresses
 * (host or device; cudaMemcpyDefault).  stream NULL = synchronous copy. */
int bin_copy(void *dst, const void *src, uint64_t bytes, bin_stream_t stream);

/* Thread-local message of the last failing call ("" if none). */
const char *bin_last_error(void);

/* Library version string. */
const char *bin_version(void);

/* ---- fused multi-operator binning ----
 * The paper's in situ step applies the DataBin operator "to 10 variables over
 * 9 coordinate systems for a total of 90 binning operations", each coordinate
 * system "done sequentially in a separate data binning operator instance"
 * (PAPER.md:511-514).  A bin_multi_t runs K such instances over ONE shared
 * list of columns as a single fused launch sequence: one identity kernel for
 * all K accumulators, one bounds kernel for every auto-bounded axis column,
 * one accumulate kernel that reads each row's columns once and updates all K
 * meshes, [the cross-rank combine of all K: three NCCL allreduces], one
 * finalize kernel for all K.  Per instance the result is the one a separate
 * bin_init/bin_execute of the same spec gives (same definition, same
 * readings R1-R17; counts/min/max bit-identical, sums within reading R8).
 *
 * bin_multi_op_t: spec = the instance's mesh, bounds and reductions
 *   (deterministic must be 0 -> else BIN_ENOTSUP; route is ignored;
 *   sum_mode BIN_SUM_EXACT gives that instance once-rounded exact sums);
 *   axis_col[d] / attr_col[a] = indices into the column list given to
 *   bin_multi_execute (0 <= index < ncols; a column may serve any number of
 *   instances, as axis or attribute).
 * Limits: 1 <= nops <= BIN_MULTI_MAX_OPS, 1 <= ncols <= BIN_MULTI_MAX_COLS. */
#define BIN_MULTI_MAX_OPS 32
#define BIN_MULTI_MAX_COLS 16
typedef struct {
    bin_spec_t spec;
    int32_t axis_col[BIN_MAX_DIM];
    int32_t attr_col[BIN_MAX_ATTR];
} bin_multi_op_t;
typedef struct bin_multi bin_multi_t; /* opaque */

/* Creates the fused instance set: validates every spec and column index
 * (BIN_EINVAL / BIN_ENOTSUP as bin_init), resolves the device by Eq. (1),
 * allocates two result slots holding all K accumulators (type-major: all
 * counts, all sums, all min/max, so a multi-rank combine is three NCCL
 * allreduces), creates the NCCL communicator when comm->nranks > 1.
 * ops is copied; the caller keeps ownership. */
int bin_multi_init(const bin_multi_op_t *ops, int32_t nops, int32_t ncols, const bin_placement_t *place,
                   const bin_comm_t *comm, bin_multi_t **out);

/* Bins one batch of rows through all K instances.  cols[0..ncols) are
 * equal-length f64 columns; device-resident columns on the analysis device
 * are read in place (zero copy), others are staged on the copy stream (host
 * memory: H2D; another GPU: NVLink peer copy).  Work is stream-ordered after
 * each column's producer stream.  Returns after enqueue (lockstep SYNC with a
 * BIN_SYNC first column blocks until done, as bin_execute).  Results of a
 * ticket stay valid until the second following execute.
 * Errors: BIN_ESHAPE (ncols or lengths), BIN_EDTYPE, BIN_ENOMEM, BIN_ECUDA, BIN_ENCCL. */
int bin_multi_execute(bin_multi_t *m, bin_array_t *const *cols, int32_t ncols, uint64_t *ticket);

/* Blocks until `ticket` is done; BIN_EDEGENERATE if any auto-bounded
 * instance saw no finite rows. */
int bin_multi_wait(bin_multi_t *m, uint64_t ticket);

/* Event after which the producer may overwrite the columns of `ticket`
 * (their snapshot/staging copies done, or the accumulate done when read in
 * place); as bin_inputs_released. */
int bin_multi_inputs_released(bin_multi_t *m, uint64_t ticket, bin_event_t *ev);

/* Waits, then fills *out with instance `op`'s result (library-owned device
 * pointers, same layout and sentinels as bin_result).  BIN_EINVAL for op out
 * of range. */
int bin_multi_result(bin_multi_t *m, uint64_t ticket, int32_t op, bin_result_t *out);

/* Profiling of the fused sequence (ms_init, ms_bounds, ms_bin, ms_combine,
 * ms_finalize, executes, kernel_launches; variant = 64). */
int bin_multi_profile_enable(bin_multi_t *m, int32_t on);
int bin_multi_profile_read(bin_multi_t *m, bin_profile_t *out);

/* The stream the last execute was enqueued on. */
int bin_multi_stream(bin_multi_t *m, bin_stream_t *stream);

/* Drains, frees everything, destroys the communicator.  NULL is a no-op. */
int bin_multi_finalize(bin_multi_t *m);

#ifdef __cplusplus
}
#endif
#endif /* DATABIN_H */
