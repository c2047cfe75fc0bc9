// L2 / HBM read bandwidth on one B200: each CTA streams a slice of a buffer with 16-B loads,
// repeated `reps` times inside the kernel (buffer <= L2: L2-resident after the first pass).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const double2 *__restrict__ p, size_t n, int reps, double *out) {
    double acc = 0;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
            double2 v = __ldcg(p + ((i + r * 4096) % n));
            acc += v.x + v.y;
        }
    if (acc == 12345.678) *out = acc;
}
__global__ void rd_unroll(const double2 *__restrict__ p, size_t n, int reps, double *out) {
    double acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r) {
        size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
        for (; i + 3 * stride < n; i += 4 * stride) {
            double2 v0 = __ldcg(p + i), v1 = __ldcg(p + i + stride), v2 = __ldcg(p + i + 2 * stride), v3 = __ldcg(p + i + 3 * stride);
            acc += v0.x + v1.x + v2.x + v3.x + v0.y + v1.y + v2.y + v3.y;
        }
    }
    if (acc == 12345.678) *out = acc;
}
int main() {
    size_t sizes[] = {4u << 20, 16u << 20, 32u << 20, 64u << 20, 1024u << 20};
    double2 *p; double *o;
    cudaMalloc(&p, 1024u << 20); cudaMalloc(&o, 8); cudaMemset(p, 0, 1024u << 20);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (size_t bytes : sizes) {
        size_t n = bytes / 16;
        int reps = bytes >= (512u << 20) ? 2 : 40;
        for (int g : {148 * 4, 148 * 8, 148 * 16}) {
            rd_unroll<<<g, 256>>>(p, n, 1, o);
            cudaEventRecord(a);
            rd_unroll<<<g, 256>>>(p, n, reps, o);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("bytes %zu MB grid %d: %.1f GB/s\n", bytes >> 20, g, bytes * (double)reps / (ms * 1e-3) / 1e9);
        }
    }
    return 0;
}
