// nvls.cpp -- NVLink SHARP (NVLS) multicast memory for the cross-rank combine
// (a6).
//
// One region per handle, identical in size on every rank: physical memory on
// the rank's own GPU (cuMemCreate) bound into a multicast object that spans
// the ranks' GPUs, mapped twice -- at a unicast address (the slots' ordinary
// device pointer, used by every kernel as before) and at the multicast address
// (multimem.ld_reduce / multimem.st in the combine kernel: the NVSwitch reads
// every rank's copy and reduces in the switch, or writes every rank's copy).
//
// Rank 0 creates the multicast object and hands its POSIX file descriptor to
// the other ranks over abstract-namespace Unix datagram sockets (SCM_RIGHTS);
// NCCL all-reduces serve as the barriers of the setup and as the agreement
// that every rank succeeded (else every rank falls back to the IPC peer or NCCL
// combine).  Driver entry points come from cudaGetDriverEntryPoint, so the
// library still loads on hosts without a driver.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <poll.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include "db_internal.h"

namespace db {

namespace {

struct Drv {
    decltype(&cuDeviceGet) DeviceGet = nullptr;
    decltype(&cuDeviceGetAttribute) DeviceGetAttribute = nullptr;
    decltype(&cuMulticastGetGranularity) MulticastGetGranularity = nullptr;
    decltype(&cuMulticastCreate) MulticastCreate = nullptr;
    decltype(&cuMulticastAddDevice) MulticastAddDevice = nullptr;
    decltype(&cuMulticastBindMem) MulticastBindMem = nullptr;
    decltype(&cuMulticastUnbind) MulticastUnbind = nullptr;
    decltype(&cuMemExportToShareableHandle) MemExportToShareableHandle = nullptr;
    decltype(&cuMemImportFromShareableHandle) MemImportFromShareableHandle = nullptr;
    decltype(&cuMemCreate) MemCreate = nullptr;
    decltype(&cuMemRelease) MemRelease = nullptr;
    decltype(&cuMemGetAllocationGranularity) MemGetAllocationGranularity = nullptr;
    decltype(&cuMemAddressReserve) MemAddressReserve = nullptr;
    decltype(&cuMemAddressFree) MemAddressFree = nullptr;
    decltype(&cuMemMap) MemMap = nullptr;
    decltype(&cuMemUnmap) MemUnmap = nullptr;
    decltype(&cuMemSetAccess) MemSetAccess = nullptr;
    bool ok = false;
};

template <class F>
bool entry(const char *name, F &f) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
        !p) {
        cudaGetLastError();
        return false;
    }
    f = reinterpret_cast<F>(p);
    return true;
}

const Drv &drv() {
    static Drv d = [] {
        Drv x;
        x.ok = entry("cuDeviceGet", x.DeviceGet) && entry("cuDeviceGetAttribute", x.DeviceGetAttribute) &&
               entry("cuMulticastGetGranularity", x.MulticastGetGranularity) &&
               entry("cuMulticastCreate", x.MulticastCreate) && entry("cuMulticastAddDevice", x.MulticastAddDevice) &&
               entry("cuMulticastBindMem", x.MulticastBindMem) && entry("cuMulticastUnbind", x.MulticastUnbind) &&
               entry("cuMemExportToShareableHandle", x.MemExportToShareableHandle) &&
               entry("cuMemImportFromShareableHandle", x.MemImportFromShareableHandle) &&
               entry("cuMemCreate", x.MemCreate) && entry("cuMemRelease", x.MemRelease) &&
               entry("cuMemGetAllocationGranularity", x.MemGetAllocationGranularity) &&
               entry("cuMemAddressReserve", x.MemAddressReserve) && entry("cuMemAddressFree", x.MemAddressFree) &&
               entry("cuMemMap", x.MemMap) && entry("cuMemUnmap", x.MemUnmap) &&
               entry("cuMemSetAccess", x.MemSetAccess);
        return x;
    }();
    return d;
}

// abstract-namespace socket address "\0databin-nvls-<key>-<rank>"
socklen_t sock_addr(sockaddr_un *a, unsigned long long key, int rank) {
    memset(a, 0, sizeof *a);
    a->sun_family = AF_UNIX;
    const int n = snprintf(a->sun_path + 1, sizeof a->sun_path - 1, "databin-nvls-%016llx-%d", key, rank);
    return (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + n);
}

bool send_fd(int sock, unsigned long long key, int to, int fd) {
    sockaddr_un a;
    const socklen_t al = sock_addr(&a, key, to);
    char byte = 'f';
    iovec io{&byte, 1};
    char ctl[CMSG_SPACE(sizeof(int))];
    memset(ctl, 0, sizeof ctl);
    msghdr m{};
    m.msg_name = &a;
    m.msg_namelen = al;
    m.msg_iov = &io;
    m.msg_iovlen = 1;
    m.msg_control = ctl;
    m.msg_controllen = sizeof ctl;
    cmsghdr *c = CMSG_FIRSTHDR(&m);
    c->cmsg_level = SOL_SOCKET;
    c->cmsg_type = SCM_RIGHTS;
    c->cmsg_len = CMSG_LEN(sizeof(int));
    memcpy(CMSG_DATA(c), &fd, sizeof(int));
    return sendmsg(sock, &m, 0) == 1;
}

int recv_fd(int sock, int timeout_ms) {
    pollfd p{sock, POLLIN, 0};
    if (poll(&p, 1, timeout_ms) != 1) return -1;
    char byte;
    iovec io{&byte, 1};
    char ctl[CMSG_SPACE(sizeof(int))];
    msghdr m{};
    m.msg_iov = &io;
    m.msg_iovlen = 1;
    m.msg_control = ctl;
    m.msg_controllen = sizeof ctl;
    if (recvmsg(sock, &m, 0) != 1) return -1;
    cmsghdr *c = CMSG_FIRSTHDR(&m);
    if (!c || c->cmsg_type != SCM_RIGHTS) return -1;
    int fd;
    memcpy(&fd, CMSG_DATA(c), sizeof(int));
    return fd;
}

// all-reduce MIN of one int over the communicator (the setup's barrier + vote)
int vote(ncclComm_t comm, cudaStream_t s, int mine, int *dbuf) {
    int v = mine;
    if (cudaMemcpyAsync(dbuf, &v, sizeof v, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        ncclAllReduce(dbuf, dbuf, 1, ncclInt32, ncclMin, comm, s) != ncclSuccess ||
        cudaMemcpyAsync(&v, dbuf, sizeof v, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return v;
}

bool dbg() {
    static const bool d = getenv("DATABIN_NVLS_DEBUG") != nullptr;
    return d;
}
#define NV_STEP(cond, what)                                                                    \
    do {                                                                                       \
        if (ok && !(cond)) {                                                                   \
            ok = 0;                                                                            \
            if (dbg()) fprintf(stderr, "[databin nvls] rank %d: %s failed\n", rank, what);      \
        }                                                                                      \
    } while (0)

}  // namespace

bool nvls_available(int device) {
    const Drv &d = drv();
    if (!d.ok) return false;
    CUdevice dev;
    int v = 0;
    if (d.DeviceGet(&dev, device) != CUDA_SUCCESS) return false;
    if (d.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) != CUDA_SUCCESS) return false;
    return v != 0;
}

void nvls_free(NvlsRegion &r) {
    const Drv &d = drv();
    if (!d.ok) return;
    if (r.mc) d.MemUnmap((CUdeviceptr)r.mc, r.size), d.MemAddressFree((CUdeviceptr)r.mc, r.size);
    if (r.uc) d.MemUnmap((CUdeviceptr)r.uc, r.size), d.MemAddressFree((CUdeviceptr)r.uc, r.size);
    if (r.bound) {
        CUdevice dev;
        if (d.DeviceGet(&dev, r.device) == CUDA_SUCCESS) d.MulticastUnbind((CUmemGenericAllocationHandle)r.mch, dev, 0, r.size);
    }
    if (r.mem) d.MemRelease((CUmemGenericAllocationHandle)r.mem);
    if (r.mch) d.MemRelease((CUmemGenericAllocationHandle)r.mch);
    r = NvlsRegion{};
}

// Collective over `comm`: every rank gets `bytes` (rounded up) of multicast-
// bound memory on `device`, or every rank gets false.
bool nvls_setup(size_t bytes, int rank, int nranks, int device, ncclComm_t comm, cudaStream_t s,
                const void *nccl_id128, NvlsRegion *out) {
    *out = NvlsRegion{};
    const Drv &d = drv();
    int *dbuf = nullptr;
    if (cudaMalloc(&dbuf, sizeof(int)) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    NvlsRegion r;
    r.device = device;
    CUdevice dev = 0;
    int ok = 1;
    NV_STEP(d.ok, "driver entry points");
    NV_STEP(nvls_available(device), "multicast support");
    NV_STEP(d.DeviceGet(&dev, device) == CUDA_SUCCESS, "cuDeviceGet");
    // sizes (the same on every rank: the larger of both granularities)
    CUmulticastObjectProp mp{};
    mp.numDevices = (unsigned)nranks;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t g1 = 0, g2 = 0;
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = device;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = bytes;
    NV_STEP(d.MulticastGetGranularity(&g1, &mp, CU_MULTICAST_GRANULARITY_MINIMUM) == CUDA_SUCCESS, "granularity");
    NV_STEP(d.MemGetAllocationGranularity(&g2, &ap, CU_MEM_ALLOC_GRANULARITY_MINIMUM) == CUDA_SUCCESS, "alloc granularity");
    const size_t gran = g1 > g2 ? g1 : g2;
    r.size = gran ? (bytes + gran - 1) / gran * gran : 0;
    mp.size = r.size;
    // every rank binds its receiving socket before rank 0 sends
    unsigned long long key = 1469598103934665603ull;  // FNV-1a of the NCCL unique id
    for (int i = 0; i < 128; ++i) key = (key ^ ((const unsigned char *)nccl_id128)[i]) * 1099511628211ull;
    int sock = socket(AF_UNIX, SOCK_DGRAM, 0);
    if (sock >= 0) {
        sockaddr_un a;
        const socklen_t al = sock_addr(&a, key, rank);
        NV_STEP(bind(sock, (sockaddr *)&a, al) == 0, "socket bind");
    } else {
        NV_STEP(false, "socket");
    }
    ok = vote(comm, s, ok, dbuf);
    // rank 0 creates the multicast object and hands its fd to every rank
    int fd = -1;
    if (ok && rank == 0) {
        CUmemGenericAllocationHandle h;
        NV_STEP(d.MulticastCreate(&h, &mp) == CUDA_SUCCESS, "cuMulticastCreate");
        if (ok) r.mch = (unsigned long long)h;
        NV_STEP(d.MemExportToShareableHandle(&fd, h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) == CUDA_SUCCESS,
                "export fd");
        for (int p = 1; p < nranks; ++p) NV_STEP(send_fd(sock, key, p, fd), "send fd");
    }
    ok = vote(comm, s, ok, dbuf);
    if (ok && rank != 0) {
        fd = recv_fd(sock, 10000);
        NV_STEP(fd >= 0, "receive fd");
        CUmemGenericAllocationHandle h;
        NV_STEP(d.MemImportFromShareableHandle(&h, (void *)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR) ==
                    CUDA_SUCCESS,
                "import fd");
        if (ok) r.mch = (unsigned long long)h;
    }
    if (fd >= 0) close(fd);
    if (sock >= 0) close(sock);
    NV_STEP(d.MulticastAddDevice((CUmemGenericAllocationHandle)r.mch, dev) == CUDA_SUCCESS, "cuMulticastAddDevice");
    ok = vote(comm, s, ok, dbuf);  // every device added before any memory is bound
    CUmemGenericAllocationHandle m = 0;
    NV_STEP(d.MemCreate(&m, r.size, &ap, 0) == CUDA_SUCCESS, "cuMemCreate");
    if (ok) r.mem = (unsigned long long)m;
    {
        const CUresult br = ok ? d.MulticastBindMem((CUmemGenericAllocationHandle)r.mch, 0, (CUmemGenericAllocationHandle)r.mem,
                                                    0, r.size, 0)
                               : CUDA_SUCCESS;
        if (ok && dbg())
            fprintf(stderr, "[databin nvls] rank %d: cuMulticastBindMem -> CUresult %d (size %zu, gran %zu/%zu)\n", rank,
                    (int)br, r.size, g1, g2);
        NV_STEP(br == CUDA_SUCCESS, "cuMulticastBindMem");
    }
    r.bound = ok;
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CUdeviceptr va = 0;
    NV_STEP(d.MemAddressReserve(&va, r.size, gran, 0, 0) == CUDA_SUCCESS, "reserve uc");
    if (ok) r.uc = (void *)va;
    NV_STEP(d.MemMap(va, r.size, 0, (CUmemGenericAllocationHandle)r.mem, 0) == CUDA_SUCCESS, "map uc");
    NV_STEP(d.MemSetAccess(va, r.size, &acc, 1) == CUDA_SUCCESS, "access uc");
    va = 0;
    NV_STEP(d.MemAddressReserve(&va, r.size, gran, 0, 0) == CUDA_SUCCESS, "reserve mc");
    if (ok) r.mc = (void *)va;
    NV_STEP(d.MemMap(va, r.size, 0, (CUmemGenericAllocationHandle)r.mch, 0) == CUDA_SUCCESS, "map mc");
    NV_STEP(d.MemSetAccess(va, r.size, &acc, 1) == CUDA_SUCCESS, "access mc");
    NV_STEP(cudaMemset(r.uc, 0, r.size) == cudaSuccess, "memset");
    cudaGetLastError();
    ok = vote(comm, s, ok, dbuf);  // all bound and mapped (or all fall back)
    if (dbg()) fprintf(stderr, "[databin nvls] rank %d: region of %zu bytes %s\n", rank, r.size, ok ? "ready" : "not used");
    cudaFree(dbuf);
    if (!ok) {
        nvls_free(r);
        return false;
    }
    *out = r;
    return true;
}

}  // namespace db
