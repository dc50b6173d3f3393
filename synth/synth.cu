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

// A Newton++-shaped O(N) producer for the placement study (BASELINE.json
// configs[4]): one second-order, time-reversible kick-drift-kick leapfrog step
// of every body in the softened field of the massive body at the origin
// (G = 1).  It stands in for the paper's O(N^2) direct-sum solver (out of
// scope); it reads 7 and writes 6 columns per body (104 B), like a solver
// step's streaming cost.  Not part of the binning method.
__global__ void syn_kdk_kernel(double *x, double *y, double *z, double *vx, double *vy, double *vz, int64_t n,
                               int64_t start, double central_mass, double eps2, double dt) {
    const double hdt = 0.5 * dt;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        if (start + i == 0) continue;  // the massive body (global row 0) stays at the origin
        double px = x[i], py = y[i], pz = z[i], ux = vx[i], uy = vy[i], uz = vz[i];
        double r2 = SYN_ADD(SYN_ADD(SYN_ADD(SYN_MUL(px, px), SYN_MUL(py, py)), SYN_MUL(pz, pz)), eps2);
        double inv = SYN_DIV(central_mass, SYN_MUL(r2, SYN_SQRT(r2)));
        ux = SYN_SUB(ux, SYN_MUL(hdt, SYN_MUL(px, inv)));
        uy = SYN_SUB(uy, SYN_MUL(hdt, SYN_MUL(py, inv)));
        uz = SYN_SUB(uz, SYN_MUL(hdt, SYN_MUL(pz, inv)));
        px = SYN_ADD(px, SYN_MUL(dt, ux));
        py = SYN_ADD(py, SYN_MUL(dt, uy));
        pz = SYN_ADD(pz, SYN_MUL(dt, uz));
        r2 = SYN_ADD(SYN_ADD(SYN_ADD(SYN_MUL(px, px), SYN_MUL(py, py)), SYN_MUL(pz, pz)), eps2);
        inv = SYN_DIV(central_mass, SYN_MUL(r2, SYN_SQRT(r2)));
        vx[i] = SYN_SUB(ux, SYN_MUL(hdt, SYN_MUL(px, inv)));
        vy[i] = SYN_SUB(uy, SYN_MUL(hdt, SYN_MUL(py, inv)));
        vz[i] = SYN_SUB(uz, SYN_MUL(hdt, SYN_MUL(pz, inv)));
        x[i] = px;
        y[i] = py;
        z[i] = pz;
    }
}

// Direct-sum gravity (the Newton++ solver class): every body
// feels every other body (softened, G = 1).  One symplectic-Euler step: the
// velocity kick from the O(N^2) force, then the drift (separate kernel, so no
// position is overwritten while another thread still reads it).  Tiles of
// DS_TILE bodies are staged in shared memory; j runs in the same order for
// every i and every launch, so trajectories are reproducible bit for bit.
constexpr int DS_TILE = 256;
__global__ void __launch_bounds__(DS_TILE) syn_direct_kick(const double *x, const double *y, const double *z,
                                                           double *vx, double *vy, double *vz, const double *m,
                                                           int64_t n, double eps2, double dt) {
    __shared__ double sx[DS_TILE], sy[DS_TILE], sz[DS_TILE], sm[DS_TILE];
    const int64_t i = (int64_t)blockIdx.x * DS_TILE + threadIdx.x;
    const double px = i < n ? x[i] : 0.0, py = i < n ? y[i] : 0.0, pz = i < n ? z[i] : 0.0;
    double ax = 0.0, ay = 0.0, az = 0.0;
    for (int64_t j0 = 0; j0 < n; j0 += DS_TILE) {
        const int64_t j = j0 + threadIdx.x;
        __syncthreads();
        sx[threadIdx.x] = j < n ? x[j] : 0.0;
        sy[threadIdx.x] = j < n ? y[j] : 0.0;
        sz[threadIdx.x] = j < n ? z[j] : 0.0;
        sm[threadIdx.x] = j < n ? m[j] : 0.0;
        __syncthreads();
        const int cnt = (int)(n - j0 < DS_TILE ? n - j0 : DS_TILE);
#pragma unroll 8
        for (int k = 0; k < cnt; ++k) {
            const double dx = sx[k] - px, dy = sy[k] - py, dz = sz[k] - pz;
            const double r2 = fma(dx, dx, fma(dy, dy, fma(dz, dz, eps2)));
            const double ri = rsqrt(r2);
            const double f = sm[k] * ri * ri * ri;  // the self term has dx = dy = dz = 0
            ax = fma(f, dx, ax);
            ay = fma(f, dy, ay);
            az = fma(f, dz, az);
        }
    }
    if (i < n) {
        vx[i] += dt * ax;
        vy[i] += dt * ay;
        vz[i] += dt * az;
    }
}
__global__ void syn_drift(double *x, double *y, double *z, const double *vx, const double *vy, const double *vz,
                          int64_t n, double dt) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        x[i] += dt * vx[i];
        y[i] += dt * vy[i];
        z[i] += dt * vz[i];
    }
}

extern "C" {

// One direct-sum step of n bodies (device columns x y z vx vy vz m), on `stream`.
int synth_direct_step(double *x, double *y, double *z, double *vx, double *vy, double *vz, const double *m,
                      int64_t n, double eps2, double dt, void *stream) {
    if (n <= 0) return 0;
    const unsigned blocks = (unsigned)((n + DS_TILE - 1) / DS_TILE);
    syn_direct_kick<<<blocks, DS_TILE, 0, (cudaStream_t)stream>>>(x, y, z, vx, vy, vz, m, n, eps2, dt);
    syn_drift<<<(unsigned)((n + 255) / 256 < 148 * 8 ? (n + 255) / 256 : 148 * 8), 256, 0, (cudaStream_t)stream>>>(
        x, y, z, vx, vy, vz, n, dt);
    return (int)cudaGetLastError();
}

// One KDK step of n bodies (device columns; row 0 is global row `start`), enqueued on `stream`.
int synth_kdk_step(double *x, double *y, double *z, double *vx, double *vy, double *vz, int64_t n, int64_t start,
                   double central_mass, double eps2, double dt, void *stream) {
    if (n <= 0) return 0;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t blocks = (n + 255) / 256;
    if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
    syn_kdk_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(x, y, z, vx, vy, vz, n, start, central_mass, eps2, dt);
    return (int)cudaGetLastError();
}


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
