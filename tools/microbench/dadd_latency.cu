#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, double a, int n, long long *cyc) {
    double s = out[threadIdx.x];
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        s = __dadd_rn(s, a); s = __dadd_rn(s, a); s = __dadd_rn(s, a); s = __dadd_rn(s, a);
        s = __dadd_rn(s, a); s = __dadd_rn(s, a); s = __dadd_rn(s, a); s = __dadd_rn(s, a);
    }
    long long t1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void kf(float *out, float a, int n, long long *cyc) {
    float s = out[threadIdx.x];
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        s = __fadd_rn(s, a); s = __fadd_rn(s, a); s = __fadd_rn(s, a); s = __fadd_rn(s, a);
        s = __fadd_rn(s, a); s = __fadd_rn(s, a); s = __fadd_rn(s, a); s = __fadd_rn(s, a);
    }
    long long t1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    double *o; float *of; long long *c, h;
    cudaMalloc(&o, 1024 * 8); cudaMalloc(&of, 1024 * 4); cudaMalloc(&c, 8);
    cudaMemset(o, 0, 8192); cudaMemset(of, 0, 4096);
    int n = 100000;
    for (int th : {1, 32}) {
        k<<<1, th>>>(o, 1e-3, n, c); cudaDeviceSynchronize();
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("{\"op\": \"DADD dependent chain\", \"threads\": %d, \"cycles_per_op\": %.2f}\n", th, (double)h / (8.0 * n));
        kf<<<1, th>>>(of, 1e-3f, n, c); cudaDeviceSynchronize();
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("{\"op\": \"FADD dependent chain\", \"threads\": %d, \"cycles_per_op\": %.2f}\n", th, (double)h / (8.0 * n));
    }
    return 0;
}
