// synth.cu -- host (threaded) and device fills for the generator in
// synth.cuh.  Built into synth/libsynth.so.  Input generation only.
#include <cuda_runtime.h>
#include <stdint.h>
#include <thread>
#include <vector>

#include "synth.cuh"

__global__ void syn_fill_kernel(int dist, int central, uint64_t seed, int column, uint64_t start,
                                int64_t n, double *out) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = syn_value(dist, central, seed, column, start + (uint64_t)i);
}

extern "C" {

// Fill out[0..n) with column `column` of rows start..start+n-1 on the host.
int synth_fill_host(int dist, int central, uint64_t seed, int column, uint64_t start, int64_t n,
                    double *out, int nthreads) {
    if (n <= 0) return 0;
    if (nthreads < 1) nthreads = (int)std::thread::hardware_concurrency();
    if (nthreads < 1) nthreads = 1;
    if (n < 65536) nthreads = 1;
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; ++t) {
        int64_t b0 = n * t / nthreads, b1 = n * (t + 1) / nthreads;
        th.emplace_back([=]() {
            for (int64_t i = b0; i < b1; ++i) out[i] = syn_value(dist, central, seed, column, start + (uint64_t)i);
        });
    }
    for (auto &x : th) x.join();
    return 0;
}

// Same on the device, enqueued on `stream`.  Returns a cudaError_t value.
int synth_fill_device(int dist, int central, uint64_t seed, int column, uint64_t start, int64_t n,
                      double *out, void *stream) {
    if (n <= 0) return 0;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t blocks = (n + 255) / 256;
    if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
    syn_fill_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(dist, central, seed, column, start, n, out);
    return (int)cudaGetLastError();
}

}  // extern "C"
