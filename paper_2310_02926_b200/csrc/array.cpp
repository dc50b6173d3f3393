// array.cpp -- the HAMR-like array handle (svtkHAMRDataArray analog),
// zero-copy wrap with coordinated lifetime (Listing 1),
// allocating constructors over the svtkAllocator kinds,
// location-agnostic read-only access with automatic temporaries
// (PAPER.md:381-389), direct access and Synchronize (Listing 3).
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>

#include "db_internal.h"

namespace db {

// ---------------------------------------------------------------- errors
static thread_local char g_err[1024] = "";

int set_error(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

int cuda_error(cudaError_t e, const char *what) {
    return set_error(BIN_ECUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

// ---------------------------------------------------------------- allocator
static std::atomic<int64_t> g_live{0}, g_total{0}, g_live_bytes{0};

void count_alloc(int64_t bytes) {
    g_live++;
    g_total++;
    g_live_bytes += bytes;
}
void count_free(int64_t bytes) {
    g_live--;
    g_live_bytes -= bytes;
}

void *dev_alloc(size_t bytes, int device, cudaStream_t stream, bool async) {
    DeviceGuard g(device);
    void *p = nullptr;
    size_t b = bytes ? bytes : 16;
    cudaError_t e = async ? cudaMallocAsync(&p, b, stream) : cudaMalloc(&p, b);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    count_alloc((int64_t)b);
    return p;
}

void dev_free(void *p, int device, cudaStream_t stream, bool async) {
    if (!p) return;
    DeviceGuard g(device);
    size_t sz = 0;
    cudaPointerAttributes at;
    (void)at;
    if (async) cudaFreeAsync(p, stream);
    else cudaFree(p);
    (void)sz;
}

void *host_alloc(size_t bytes, bool pinned) {
    void *p = nullptr;
    size_t b = bytes ? bytes : 16;
    if (pinned) {
        if (cudaHostAlloc(&p, b, cudaHostAllocPortable) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
    } else {
        p = malloc(b);
    }
    if (p) count_alloc((int64_t)b);
    return p;
}

void host_free(void *p, bool pinned) {
    if (!p) return;
    if (pinned) cudaFreeHost(p);
    else free(p);
}

void *uva_alloc(size_t bytes) {
    void *p = nullptr;
    if (cudaMallocManaged(&p, bytes ? bytes : 16) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    count_alloc((int64_t)(bytes ? bytes : 16));
    return p;
}
void uva_free(void *p) {
    if (p) cudaFree(p);
}

bool is_device_memory(const bin_array *a) {
    return a->device >= 0 && a->alloc != BIN_ALLOC_HOST && a->alloc != BIN_ALLOC_HOST_PINNED;
}

int array_mark_use(bin_array *a, cudaStream_t s, int dev) {
    for (bin_array *x = a; x; x = x->source) {
        std::lock_guard<std::mutex> lk(x->mu);
        DeviceGuard g(dev);
        bin_array::Use *u = nullptr;
        for (auto &r : x->uses)
            if (r.device == dev && r.stream == s) u = &r;
        if (!u) {
            cudaEvent_t ev;
            DB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            x->uses.push_back({dev, s, ev});
            u = &x->uses.back();
        }
        DB_CUDA(cudaEventRecord(u->ev, s));  // supersedes only this stream's earlier use
    }
    return BIN_OK;
}

// waits for every recorded use; destroy: also drop the events
static cudaError_t drain_uses(bin_array *x, bool destroy) {
    cudaError_t rc = cudaSuccess;
    for (auto &u : x->uses) {
        DeviceGuard g(u.device);
        cudaError_t e = cudaEventSynchronize(u.ev);
        if (e != cudaSuccess && rc == cudaSuccess) rc = e;
        if (destroy) cudaEventDestroy(u.ev);
    }
    if (destroy) x->uses.clear();
    return rc;
}

static size_t elem_size(int32_t dtype) { return dtype == BIN_F64 ? 8 : 0; }

static void free_storage(bin_array *a) {
    size_t bytes = (size_t)a->n * elem_size(a->dtype);
    if (a->owned) {
        switch (a->alloc) {
        case BIN_ALLOC_HOST: host_free(a->ptr, false); break;
        case BIN_ALLOC_HOST_PINNED: host_free(a->ptr, true); break;
        case BIN_ALLOC_CUDA: dev_free(a->ptr, a->device, nullptr, false); break;
        case BIN_ALLOC_CUDA_ASYNC: dev_free(a->ptr, a->device, a->stream, true); break;
        case BIN_ALLOC_CUDA_UVA: uva_free(a->ptr); break;
        default: break;
        }
        count_free((int64_t)(bytes ? bytes : 16));
    } else if (a->release) {
        a->release(a->release_ctx, a->ptr);  // exactly once: the last reference is gone
    }
    a->ptr = nullptr;
}

}  // namespace db

using namespace db;

extern "C" {

void bin_alloc_stats(int64_t *live, int64_t *total, int64_t *live_bytes) {
    if (live) *live = g_live.load();
    if (total) *total = g_total.load();
    if (live_bytes) *live_bytes = g_live_bytes.load();
}

int bin_array_wrap(const void *ptr, int64_t n, int32_t dtype, int32_t device, bin_allocator_t alloc,
                   bin_stream_t stream, bin_stream_mode_t mode, void (*release)(void *, void *),
                   void *release_ctx, bin_array_t **out) {
    if (!out) return set_error(BIN_EINVAL, "bin_array_wrap: out is NULL");
    *out = nullptr;
    if (n < 0 || (n > 0 && !ptr)) return set_error(BIN_EINVAL, "bin_array_wrap: bad ptr/length (n=%lld)", (long long)n);
    if (dtype != BIN_F64) return set_error(BIN_EDTYPE, "bin_array_wrap: dtype %d is not BIN_F64", dtype);
    if (device < -1) return set_error(BIN_EDEVICE, "bin_array_wrap: device %d", device);
    if ((int)alloc < 0 || (int)alloc > BIN_ALLOC_EXTERNAL) return set_error(BIN_EINVAL, "bin_array_wrap: allocator %d", alloc);
    if (device >= 0) {
        int nd = 0;
        if (cudaGetDeviceCount(&nd) != cudaSuccess) { cudaGetLastError(); nd = 0; }
        if (device >= nd) return set_error(BIN_EDEVICE, "bin_array_wrap: device %d of %d", device, nd);
    }
    bin_array *a = new bin_array;
    a->ptr = const_cast<void *>(ptr);
    a->n = n;
    a->dtype = dtype;
    a->device = (alloc == BIN_ALLOC_HOST || alloc == BIN_ALLOC_HOST_PINNED) ? -1 : device;
    a->alloc = alloc;
    a->stream = (cudaStream_t)stream;
    a->mode = mode;
    a->owned = false;
    a->release = release;
    a->release_ctx = release_ctx;
    *out = a;
    return BIN_OK;
}

int bin_array_alloc(int64_t n, int32_t dtype, int32_t device, bin_allocator_t alloc, bin_stream_t stream,
                    bin_stream_mode_t mode, const double *fill, bin_array_t **out) {
    if (!out) return set_error(BIN_EINVAL, "bin_array_alloc: out is NULL");
    *out = nullptr;
    if (n < 0) return set_error(BIN_EINVAL, "bin_array_alloc: n < 0");
    if (dtype != BIN_F64) return set_error(BIN_EDTYPE, "bin_array_alloc: dtype %d is not BIN_F64", dtype);
    if (alloc == BIN_ALLOC_EXTERNAL) return set_error(BIN_EINVAL, "bin_array_alloc: EXTERNAL cannot allocate");
    bool host = alloc == BIN_ALLOC_HOST || alloc == BIN_ALLOC_HOST_PINNED;
    if (!host) {
        int nd = 0;
        if (cudaGetDeviceCount(&nd) != cudaSuccess) { cudaGetLastError(); nd = 0; }
        if (device < 0 || device >= nd) return set_error(BIN_EDEVICE, "bin_array_alloc: device %d of %d", device, nd);
    }
    size_t bytes = (size_t)n * 8;
    void *p = nullptr;
    switch (alloc) {
    case BIN_ALLOC_HOST: p = host_alloc(bytes, false); break;
    case BIN_ALLOC_HOST_PINNED: p = host_alloc(bytes, true); break;
    case BIN_ALLOC_CUDA: p = dev_alloc(bytes, device, nullptr, false); break;
    case BIN_ALLOC_CUDA_ASYNC: p = dev_alloc(bytes, device, (cudaStream_t)stream, true); break;
    case BIN_ALLOC_CUDA_UVA: p = uva_alloc(bytes); break;
    default: break;
    }
    if (!p) return set_error(BIN_ENOMEM, "bin_array_alloc: %zu bytes with allocator %d failed", bytes, alloc);
    bin_array *a = new bin_array;
    a->ptr = p;
    a->n = n;
    a->dtype = dtype;
    a->device = host ? -1 : device;
    a->alloc = alloc;
    a->stream = (cudaStream_t)stream;
    a->mode = mode;
    a->owned = true;
    *out = a;
    if (fill && n > 0) {
        if (host) {
            double *d = (double *)p;
            for (int64_t i = 0; i < n; ++i) d[i] = *fill;
        } else {
            DeviceGuard g(device);
            // fill on the array's stream: host pattern then device-side doubling copies
            double v = *fill;
            cudaError_t e = cudaMemcpyAsync(p, &v, 8, cudaMemcpyHostToDevice, (cudaStream_t)stream);
            for (int64_t have = 1; e == cudaSuccess && have < n; have *= 2) {
                int64_t c = have < n - have ? have : n - have;
                e = cudaMemcpyAsync((double *)p + have, p, (size_t)c * 8, cudaMemcpyDeviceToDevice,
                                    (cudaStream_t)stream);
            }
            if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);  // v lives on this stack
            if (e != cudaSuccess) {
                bin_array_release(a);
                *out = nullptr;
                return cuda_error(e, "bin_array_alloc fill");
            }
        }
    }
    return BIN_OK;
}

int bin_array_data(bin_array_t *a, void **ptr) {
    if (!a || !ptr) return set_error(BIN_EINVAL, "bin_array_data: NULL argument");
    *ptr = a->ptr;
    return BIN_OK;
}

int bin_array_info(const bin_array_t *a, int64_t *n, int32_t *device, int32_t *alloc, bin_stream_t *stream) {
    if (!a) return set_error(BIN_EINVAL, "bin_array_info: NULL array");
    if (n) *n = a->n;
    if (device) *device = a->device;
    if (alloc) *alloc = (int32_t)a->alloc;
    if (stream) *stream = (bin_stream_t)a->stream;
    return BIN_OK;
}

int bin_array_get_accessible(bin_array_t *a, int32_t device, bin_stream_t stream, const void **ptr,
                             bin_array_t **view) {
    if (!a || !ptr || !view) return set_error(BIN_EINVAL, "bin_array_get_accessible: NULL argument");
    *ptr = nullptr;
    *view = nullptr;
    if (device < -1) return set_error(BIN_EDEVICE, "bin_array_get_accessible: device %d", device);
    cudaStream_t s = stream ? (cudaStream_t)stream : a->stream;
    bool direct = false;
    if (a->alloc == BIN_ALLOC_CUDA_UVA) direct = true;            // universally addressable
    else if (device == -1) direct = (a->device == -1);              // host request
    else direct = is_device_memory(a) && a->device == device;       // same GPU
    a->refs++;  // the view references its source
    bin_array *v = new bin_array;
    v->source = a;
    v->n = a->n;
    v->dtype = a->dtype;
    v->stream = s;
    v->mode = a->mode;
    if (direct) {
        v->ptr = a->ptr;
        v->device = a->device;
        v->alloc = BIN_ALLOC_EXTERNAL;
        v->owned = false;
        *view = v;
        *ptr = v->ptr;
        return BIN_OK;
    }
    size_t bytes = (size_t)a->n * 8;
    int rc = BIN_OK;
    if (device == -1) {  // device -> host temporary
        v->device = -1;
        v->alloc = BIN_ALLOC_HOST_PINNED;
        v->ptr = host_alloc(bytes, true);
        if (!v->ptr) rc = set_error(BIN_ENOMEM, "get_accessible: host temporary of %zu bytes", bytes);
        else {
            DeviceGuard g(a->device);
            cudaError_t e = cudaMemcpyAsync(v->ptr, a->ptr, bytes, cudaMemcpyDeviceToHost, s);
            if (e != cudaSuccess) rc = cuda_error(e, "get_accessible D2H");
        }
    } else {
        v->device = device;
        v->alloc = BIN_ALLOC_CUDA;
        v->ptr = dev_alloc(bytes, device, nullptr, false);
        if (!v->ptr) rc = set_error(BIN_ENOMEM, "get_accessible: device temporary of %zu bytes", bytes);
        else if (a->device == -1) {
            DeviceGuard g(device);
            cudaError_t e = cudaMemcpyAsync(v->ptr, a->ptr, bytes, cudaMemcpyHostToDevice, s);
            if (e != cudaSuccess) rc = cuda_error(e, "get_accessible H2D");
        } else {
            DeviceGuard g(device);
            int can = 0;  // NVLink direct access (else the copy stages through the host)
            if (cudaDeviceCanAccessPeer(&can, device, a->device) == cudaSuccess && can)
                cudaDeviceEnablePeerAccess(a->device, 0);
            cudaGetLastError();
            cudaError_t e = cudaMemcpyPeerAsync(v->ptr, device, a->ptr, a->device, bytes, s);
            if (e != cudaSuccess) rc = cuda_error(e, "get_accessible peer copy");
        }
    }
    v->owned = v->ptr != nullptr;
    if (rc != BIN_OK) {
        bin_array_release(v);
        return rc;
    }
    if (v->mode == BIN_SYNC) {
        cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
            bin_array_release(v);
            return cuda_error(e, "get_accessible synchronize");
        }
    } else {
        array_mark_use(v, s, device >= 0 ? device : (a->device >= 0 ? a->device : 0));
    }
    *view = v;
    *ptr = v->ptr;
    return BIN_OK;
}

int bin_array_synchronize(bin_array_t *a) {
    if (!a) return set_error(BIN_EINVAL, "bin_array_synchronize: NULL array");
    for (bin_array *x = a; x; x = x->source) {
        std::lock_guard<std::mutex> lk(x->mu);
        cudaError_t e0 = drain_uses(x, false);
        if (e0 != cudaSuccess) return cuda_error(e0, "bin_array_synchronize");
        if (x->stream && (x->device >= 0 || x->alloc == BIN_ALLOC_HOST_PINNED)) {
            DeviceGuard g(x->device);
            cudaError_t e = cudaStreamSynchronize(x->stream);
            if (e != cudaSuccess) return cuda_error(e, "bin_array_synchronize stream");
        }
    }
    return BIN_OK;
}

void bin_array_release(bin_array_t *a) {
    while (a) {
        if (--a->refs > 0) return;
        drain_uses(a, true);  // library work on any stream/GPU that reads/writes this memory
        free_storage(a);
        bin_array *src = a->source;
        delete a;
        a = src;  // a view drops its reference on the source
    }
}

int bin_copy(void *dst, const void *src, uint64_t bytes, bin_stream_t stream) {
    if (bytes == 0) return BIN_OK;
    if (!dst || !src) return set_error(BIN_EINVAL, "bin_copy: NULL pointer");
    cudaError_t e = stream ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream)
                           : cudaMemcpy(dst, src, bytes, cudaMemcpyDefault);
    if (e != cudaSuccess) return cuda_error(e, "bin_copy");
    return BIN_OK;
}

const char *bin_last_error(void) { return g_err; }

const char *bin_version(void) { return "databin-b200 0.1 (sm_100a)"; }

}  // extern "C"
