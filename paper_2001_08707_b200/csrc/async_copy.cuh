// async_copy.cuh — PTX wrappers for the asynchronous copies of the streaming kernels: mbarrier
// (init / expect_tx / arrive / parity wait), cp.async.bulk global -> shared with mbarrier
// completion, and 256-bit global loads/stores (LDG.256 / STG.256 on sm_100a).
#pragma once
#include "common.cuh"

namespace sk {

static __device__ __forceinline__ uint32_t sa(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
static __device__ __forceinline__ void mb_init(uint64_t *b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(count) : "memory");
}
static __device__ __forceinline__ void mb_expect(uint64_t *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
static __device__ __forceinline__ void mb_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
static __device__ __forceinline__ void mb_wait(uint64_t *b, unsigned parity) {
    unsigned done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(sa(b)), "r"(parity) : "memory");
}
static __device__ __forceinline__ void bulk_load(void *dst, const void *src, unsigned bytes, uint64_t *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa(dst)), "l"(src), "r"(bytes), "r"(sa(b)) : "memory");
}

// 32-byte (two complex128) streaming load / store: one LDG.256 / STG.256 per lane (sm_100a)
static __device__ __forceinline__ void ldg2_cs(const cplx *p, cplx &a, cplx &b) {
    asm volatile("ld.global.cs.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y) : "l"(p));
}
static __device__ __forceinline__ void stg2(cplx *p, cplx a, cplx b) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y) : "memory");
}

}  // namespace sk
