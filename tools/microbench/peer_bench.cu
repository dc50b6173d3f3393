// Peer-memory (NVLink) microbenchmark for the combine design: from GPU 0,
// uniform-random REDG.ADD.64 / REDG.ADD.F64 / REDG.MIN.64 into a 262,144-bin
// array that lives on GPU 1 (peer access enabled) vs on GPU 0; coalesced
// remote loads and stores of 8 MB.  Not product code: a standalone executable.
// One JSON object per line on stdout.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peer_bench peer_bench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

constexpr int ITERS = 32;

template <int OP>
__global__ void k_red(unsigned long long *a, uint32_t nbins, uint32_t seed) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll 4
    for (int i = 0; i < ITERS; ++i) {
        const uint32_t b = hash32(t * ITERS + i + seed) % nbins;
        if (OP == 0) atomicAdd(a + b, 1ull);
        if (OP == 1) atomicAdd((double *)(a + b), 1.0);
        if (OP == 2) atomicMin(a + b, (unsigned long long)(t ^ i));
    }
}

__global__ void k_load(const double2 *src, double2 *dst, size_t n2) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = __ldcg(src + i);
}

int main() {
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (ndev < 2) {
        printf("{\"error\": \"needs 2 GPUs\"}\n");
        return 0;
    }
    const uint32_t nbins = 262144;
    unsigned long long *loc, *rem;
    double2 *bufl, *bufr;
    const size_t bytes = 8u << 20;
    CK(cudaSetDevice(1));
    CK(cudaMalloc(&rem, nbins * 8));
    CK(cudaMalloc(&bufr, bytes));
    CK(cudaMemset(rem, 0, nbins * 8));
    CK(cudaSetDevice(0));
    CK(cudaDeviceEnablePeerAccess(1, 0));
    CK(cudaMalloc(&loc, nbins * 8));
    CK(cudaMalloc(&bufl, bytes));
    CK(cudaMemset(loc, 0, nbins * 8));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int blocks = 148 * 8, threads = 256;
    const double nops = (double)blocks * threads * ITERS;
    const char *names[3] = {"red_add_u64", "red_add_f64", "red_min_u64"};
    for (int where = 0; where < 2; ++where) {
        unsigned long long *a = where ? rem : loc;
        for (int op = 0; op < 3; ++op) {
            float best = 1e30f;
            for (int rep = 0; rep < 5; ++rep) {
                CK(cudaEventRecord(e0));
                if (op == 0) k_red<0><<<blocks, threads>>>(a, nbins, rep);
                if (op == 1) k_red<1><<<blocks, threads>>>(a, nbins, rep);
                if (op == 2) k_red<2><<<blocks, threads>>>(a, nbins, rep);
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                if (ms < best) best = ms;
            }
            printf("{\"op\": \"%s\", \"target\": \"%s\", \"Gops\": %.2f}\n", names[op], where ? "peer" : "local",
                   nops / (best * 1e-3) / 1e9);
        }
    }
    // coalesced remote read (pull) and remote write (push) of 8 MB
    for (int dir = 0; dir < 2; ++dir) {
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            CK(cudaEventRecord(e0));
            if (dir == 0) k_load<<<148 * 4, 256>>>(bufr, bufl, bytes / 16);
            else k_load<<<148 * 4, 256>>>(bufl, bufr, bytes / 16);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (ms < best) best = ms;
        }
        printf("{\"op\": \"%s\", \"bytes\": %zu, \"us\": %.1f, \"GBps\": %.0f}\n", dir ? "peer_store" : "peer_load",
               bytes, best * 1e3, bytes / (best * 1e-3) / 1e9);
    }
    return 0;
}
