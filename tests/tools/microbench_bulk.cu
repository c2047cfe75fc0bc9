// Throughput of cp.async.bulk global->shared streams (16 KB chunks from an L2-resident buffer)
// per SM, vs ring depth and CTAs per SM; consumers only wait + release (no math).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t *b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mb_expect(uint64_t *b, unsigned n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mb_arrive(uint64_t *b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory"); }
__device__ __forceinline__ void mb_wait(uint64_t *b, unsigned p) { unsigned d = 0; while (!d) asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0, 1, 0, q; }" : "=r"(d) : "r"(sa(b)), "r"(p) : "memory"); }
__device__ __forceinline__ void bulk(void *d, const void *s, unsigned n, uint64_t *b) { asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(d)), "l"(s), "r"(n), "r"(sa(b)) : "memory"); }

template <int NS, int CH, int P>
__global__ void stream(const char *src, size_t bytes, int items, double *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ uint64_t full[NS], empty[NS];
    if (threadIdx.x == 0) { for (int i = 0; i < NS; ++i) { mb_init(&full[i], 1); mb_init(&empty[i], 8); } asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    __syncthreads();
    const size_t nch = bytes / CH;
    double acc = 0;
    if (threadIdx.x >= 256 && threadIdx.x < 256 + P) {
        for (int it = threadIdx.x - 256; it < items; it += P) {
            int s = it % NS;
            mb_wait(&empty[s], ((it / NS) & 1) ^ 1);
            mb_expect(&full[s], CH);
            size_t c = ((size_t)blockIdx.x * 7919 + (size_t)it * 104729) % nch;
            bulk(sm + s * CH, src + c * CH, CH, &full[s]);
        }
    } else if (threadIdx.x < 256) {
        for (int it = 0; it < items; ++it) {
            int s = it % NS;
            mb_wait(&full[s], (it / NS) & 1);
            acc += ((const double *)(sm + s * CH))[threadIdx.x];
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mb_arrive(&empty[s]);
        }
    }
    if (acc == 1234.5) *out = acc;
}
template <int NS, int CH, int P = 1>
void run(const char *p, size_t bytes, double *o, int ctas_per_sm) {
    const int smem = NS * CH;
    cudaFuncSetAttribute(stream<NS, CH, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int grid = 148 * ctas_per_sm, items = 200;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    stream<NS, CH, P><<<grid, 288, smem>>>(p, bytes, items, o);
    cudaEventRecord(a);
    stream<NS, CH, P><<<grid, 288, smem>>>(p, bytes, items, o);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    double tot = (double)grid * items * CH;
    printf("P=%d NS=%d CH=%d ctas/SM=%d: %.0f GB/s (%.1f B/clk/SM @1.9GHz) %s\n", P, NS, CH, ctas_per_sm, tot / (ms * 1e-3) / 1e9,
           tot / (ms * 1e-3) / 148 / 1.9e9, e ? cudaGetErrorString(e) : "");
}
int main() {
    size_t bytes = 16u << 20;
    char *p; double *o;
    cudaMalloc(&p, bytes); cudaMalloc(&o, 8); cudaMemset(p, 0, bytes);
    run<4, 16384>(p, bytes, o, 1);
    run<4, 16384, 2>(p, bytes, o, 1);
    run<4, 16384, 4>(p, bytes, o, 1);
    run<8, 16384, 8>(p, bytes, o, 1);
    run<2, 16384>(p, bytes, o, 4);
    run<2, 16384>(p, bytes, o, 6);
    run<3, 16384>(p, bytes, o, 4);
    run<4, 16384, 4>(p, bytes, o, 2);
    run<6, 16384, 6>(p, bytes, o, 2);
    run<12, 4096, 12>(p, bytes, o, 2);
    run<4, 65536>(p, bytes, o, 1);
    return 0;
}
