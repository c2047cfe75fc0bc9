// Latency microbenchmark (one thread, dependent chains): fp64 div / sqrt / rsqrt / fma, a
// dependent global load (L2 hit), and __syncthreads in a 256-thread CTA.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, long long *cyc, const double *buf, int n) {
    double x = out[0], y = 1.0000001;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = y / x;
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) x = sqrt(x + 1.0);
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) x = rsqrt(x + 1.0);
    long long t3 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, y, 1e-9);
    long long t4 = clock64();
    int idx = 0;
    for (int i = 0; i < n; ++i) idx = (int)__ldcg(buf + idx);   // dependent L2 hits
    long long t5 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    long long t6 = clock64();
    if (threadIdx.x == 0) {
        out[1] = x + idx;
        cyc[0] = (t1 - t0) / n; cyc[1] = (t2 - t1) / n; cyc[2] = (t3 - t2) / n;
        cyc[3] = (t4 - t3) / n; cyc[4] = (t5 - t4) / n; cyc[5] = (t6 - t5) / n;
    }
}
int main() {
    double *out, *buf; long long *cyc;
    cudaMalloc(&out, 16); cudaMalloc(&buf, 1 << 20); cudaMallocManaged(&cyc, 64);
    double h[2] = {1.5, 0}; cudaMemcpy(out, h, 16, cudaMemcpyHostToDevice);
    cudaMemset(buf, 0, 1 << 20);
    for (int rep = 0; rep < 2; ++rep) { k<<<1, 256>>>(out, cyc, buf, 1000); cudaDeviceSynchronize(); }
    printf("cycles per op: div %lld sqrt %lld rsqrt %lld fma %lld ldcg_L2 %lld syncthreads256 %lld\n",
           cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cyc[5]);
    return 0;
}
