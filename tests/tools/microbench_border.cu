// Memory-pattern prototype of the split-bond update: does an update that walks
// the rows in "B order" — tiles made of 2^PB-state pieces (16·2^PB B contiguous) taken at every
// combination of the HB top spin bits (pieces 2^AHI states apart) — stream r_n, q, r_{n-1}, b
// and write r_{n+1} as fast as the linear update?  Each B-tile is staged in shared memory and
// the off-diagonal bonds among its bits are applied twice (to r_n and to r_{n+1}), as the real
// kernel does.  Prints GB/s of the 80 algorithmic bytes per row.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbb microbench_border.cu && /tmp/mbb
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

typedef double2 cplx;
__device__ __forceinline__ cplx ldcs(const cplx *p) { return __ldcs(p); }

__global__ void lin(const cplx *__restrict__ rc, const cplx *__restrict__ rp, const cplx *__restrict__ q,
                    const cplx *__restrict__ b, cplx *__restrict__ rn, int64_t M, double2 *part) {
    double ax = 0, ay = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
        cplx a = ldcs(rc + i), c = ldcs(rp + i), d = ldcs(q + i), e = ldcs(b + i);
        cplx o = make_double2(0.5 * a.x + 0.25 * d.x - 0.125 * c.x, 0.5 * a.y + 0.25 * d.y - 0.125 * c.y);
        __stcs(rn + i, o);
        ax += o.x * e.x;
        ay += o.y * e.y;
    }
    if (ax == 1234.5) part[0] = make_double2(ax, ay);
}

template <int L, int AHI, int PB, int NT>
__global__ void __launch_bounds__(NT, 1) bord(const cplx *__restrict__ rc, const cplx *__restrict__ rp,
                                              const cplx *__restrict__ q, const cplx *__restrict__ b,
                                              cplx *__restrict__ rn, double2 *part, unsigned long long *work,
                                              int dyn) {
    constexpr int HB = L - AHI, TB = PB + HB, TS = 1 << TB, PER = TS / NT;
    static_assert(PER * NT == TS, "");
    extern __shared__ cplx S[];
    __shared__ int64_t tnext;
    const int64_t ntiles = int64_t(1) << (AHI - PB);
    const int tid = threadIdx.x;
    double wx = 0, wy = 0, ax = 0;
    int64_t t = dyn ? 0 : blockIdx.x;
    if (dyn) {
        if (tid == 0) tnext = (int64_t)atomicAdd(work, 1ull);
        __syncthreads();
        t = tnext;
    }
    while (t < ntiles) {
        cplx v[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int e = tid + k * NT;
            const int64_t s = ((int64_t)(e >> PB) << AHI) | (t << PB) | (e & ((1 << PB) - 1));
            v[k] = ldcs(rc + s);
            S[e] = v[k];
        }
        __syncthreads();
        if (dyn && tid == 0) tnext = (int64_t)atomicAdd(work, 1ull);
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int e = tid + k * NT;
            const int64_t s = ((int64_t)(e >> PB) << AHI) | (t << PB) | (e & ((1 << PB) - 1));
            cplx h = ldcs(q + s);
            const cplx c = ldcs(rp + s), d = ldcs(b + s);
#pragma unroll
            for (int j = 0; j < HB - 1; ++j)
                if (((e >> (PB + j)) ^ (e >> (PB + j + 1))) & 1) {
                    const cplx p = S[e ^ (3 << (PB + j))];
                    h.x += 0.5 * p.x;
                    h.y += 0.5 * p.y;
                }
            if (((e >> (TB - 1)) ^ e) & 1) {
                const cplx p = S[e ^ ((1 << (TB - 1)) | 1)];
                h.x += 0.5 * p.x;
                h.y += 0.5 * p.y;
            }
            const cplx o = make_double2(0.5 * v[k].x + 0.25 * h.x - 0.125 * c.x, 0.5 * v[k].y + 0.25 * h.y - 0.125 * c.y);
            __stcs(rn + s, o);
            ax += o.x * d.x + o.y * d.y;
            v[k] = o;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < PER; ++k) S[tid + k * NT] = v[k];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int e = tid + k * NT;
            cplx h = make_double2(0, 0);
#pragma unroll
            for (int j = 0; j < HB - 1; ++j)
                if (((e >> (PB + j)) ^ (e >> (PB + j + 1))) & 1) {
                    const cplx p = S[e ^ (3 << (PB + j))];
                    h.x += p.x;
                    h.y += p.y;
                }
            if (((e >> (TB - 1)) ^ e) & 1) {
                const cplx p = S[e ^ ((1 << (TB - 1)) | 1)];
                h.x += p.x;
                h.y += p.y;
            }
            wx += v[k].x * h.x - v[k].y * h.y;
            wy += v[k].x * h.y + v[k].y * h.x;
        }
        if (dyn) {
            __syncthreads();
            t = tnext;
        } else {
            __syncthreads();
            t += gridDim.x;
        }
    }
    if (wx + ax == 1234.5) part[0] = make_double2(wx, wy);
}

// Variant: r_n tiles staged with cp.async (16 B per thread-row, no registers held), double
// buffered so tile t+1's r_n is in flight while tile t is computed; r_{n+1} written in place.
__device__ __forceinline__ void cpa16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src) : "memory");
}
template <int L, int AHI, int PB, int NT>
__global__ void __launch_bounds__(NT, 1) bord2(const cplx *__restrict__ rc, const cplx *__restrict__ rp,
                                               const cplx *__restrict__ q, const cplx *__restrict__ b,
                                               cplx *__restrict__ rn, double2 *part, int64_t pad) {
    constexpr int HB = L - AHI, TB = PB + HB, TS = 1 << TB, PER = TS / NT;
    static_assert(PER * NT == TS, "");
    extern __shared__ cplx S2[];   // [2][TS]
    const int64_t ntiles = int64_t(1) << (AHI - PB);
    const int tid = threadIdx.x;
    double wx = 0, wy = 0, ax = 0;
    // high-bit segments of 2^AHI rows stored `pad` rows apart (pad 0: the natural layout)
    const int64_t seg = (int64_t(1) << AHI) + pad;
    auto row = [&](int64_t t, int e) { return (int64_t)(e >> PB) * seg + (t << PB) + (e & ((1 << PB) - 1)); };
    int64_t t = blockIdx.x;
    if (t < ntiles)
        for (int k = 0; k < PER; ++k) cpa16(S2 + tid + k * NT, rc + row(t, tid + k * NT));
    asm volatile("cp.async.commit_group;" ::: "memory");
    for (int it = 0; t < ntiles; ++it, t += gridDim.x) {
        cplx *S = S2 + (it & 1) * TS;
        const int64_t tn = t + gridDim.x;
        if (tn < ntiles)
            for (int k = 0; k < PER; ++k) cpa16(S2 + ((it + 1) & 1) * TS + tid + k * NT, rc + row(tn, tid + k * NT));
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();
        cplx o[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int e = tid + k * NT;
            const int64_t s = row(t, e);
            cplx h = ldcs(q + s);
            const cplx c = ldcs(rp + s), d = ldcs(b + s);
            const cplx v = S[e];
#pragma unroll
            for (int j = 0; j < HB - 1; ++j)
                if (((e >> (PB + j)) ^ (e >> (PB + j + 1))) & 1) {
                    const cplx p = S[e ^ (3 << (PB + j))];
                    h.x += 0.5 * p.x;
                    h.y += 0.5 * p.y;
                }
            if (((e >> (TB - 1)) ^ e) & 1) {
                const cplx p = S[e ^ ((1 << (TB - 1)) | 1)];
                h.x += 0.5 * p.x;
                h.y += 0.5 * p.y;
            }
            o[k] = make_double2(0.5 * v.x + 0.25 * h.x - 0.125 * c.x, 0.5 * v.y + 0.25 * h.y - 0.125 * c.y);
            __stcs(rn + s, o[k]);
            ax += o[k].x * d.x + o[k].y * d.y;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < PER; ++k) S[tid + k * NT] = o[k];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int e = tid + k * NT;
            cplx h = make_double2(0, 0);
#pragma unroll
            for (int j = 0; j < HB - 1; ++j)
                if (((e >> (PB + j)) ^ (e >> (PB + j + 1))) & 1) {
                    const cplx p = S[e ^ (3 << (PB + j))];
                    h.x += p.x;
                    h.y += p.y;
                }
            if (((e >> (TB - 1)) ^ e) & 1) {
                const cplx p = S[e ^ ((1 << (TB - 1)) | 1)];
                h.x += p.x;
                h.y += p.y;
            }
            wx += o[k].x * h.x - o[k].y * h.y;
            wy += o[k].x * h.y + o[k].y * h.x;
        }
        __syncthreads();   // S (this buffer) is refilled two tiles later
    }
    if (wx + ax == 1234.5) part[0] = make_double2(wx, wy);
}

// Pure B-order streaming (no shared memory, no bonds): the DRAM-pattern cost of the piece size.
template <int L, int AHI, int PB>
__global__ void bpure(const cplx *__restrict__ rc, const cplx *__restrict__ rp, const cplx *__restrict__ q,
                      const cplx *__restrict__ b, cplx *__restrict__ rn, int64_t M, double2 *part) {
    constexpr int HB = L - AHI, TB = PB + HB;
    double ax = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
        const int e = (int)(i & ((1 << TB) - 1));
        const int64_t t = i >> TB;
        const int64_t s = ((int64_t)(e >> PB) << AHI) | (t << PB) | (e & ((1 << PB) - 1));
        cplx a = ldcs(rc + s), c = ldcs(rp + s), d = ldcs(q + s), f = ldcs(b + s);
        cplx o = make_double2(0.5 * a.x + 0.25 * d.x - 0.125 * c.x, 0.5 * a.y + 0.25 * d.y - 0.125 * c.y);
        __stcs(rn + s, o);
        ax += o.x * f.x + o.y * f.y;
    }
    if (ax == 1234.5) part[0] = make_double2(ax, ax);
}


// ---- v3 variants (the update_split2 structure): staging by 16-B cp.async per row or by one
// cp.async.bulk per piece (mbarrier), row streams by 128-bit or 256-bit (pair) loads
__device__ __forceinline__ uint32_t sa3(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbi(uint64_t *b) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa3(b)) : "memory"); }
__device__ __forceinline__ void mbx(uint64_t *b, unsigned n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa3(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mbw(uint64_t *b, unsigned ph) { unsigned d = 0; while (!d) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(d) : "r"(sa3(b)), "r"(ph) : "memory"); }
__device__ __forceinline__ void bulk3(void *d, const void *s, unsigned n, uint64_t *b) { asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa3(d)), "l"(s), "r"(n), "r"(sa3(b)) : "memory"); }
__device__ __forceinline__ void ld2(const cplx *p, cplx &a, cplx &b) { asm volatile("ld.global.cs.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y) : "l"(p)); }
__device__ __forceinline__ void st2(cplx *p, cplx a, cplx b) { asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y) : "memory"); }

template <int L, int AHI, int PB, int NT, bool BULK, bool LD256, bool EARLY = false>
__global__ void __launch_bounds__(NT, 1) bord3(const cplx *__restrict__ rc, const cplx *__restrict__ rp,
                                               const cplx *__restrict__ q, const cplx *__restrict__ b,
                                               cplx *__restrict__ rn, double2 *part) {
    constexpr int HB = L - AHI, TB = PB + HB, TS = 1 << TB, NPIECE = 1 << HB;
    constexpr int G = LD256 ? 2 : 1, PER = TS / G / NT;
    extern __shared__ __align__(16) cplx S3[];
    __shared__ uint64_t full[2];
    const int64_t ntiles = int64_t(1) << (AHI - PB);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    auto row = [&](int64_t t, int e) { return ((int64_t)(e >> PB) << AHI) | (t << PB) | (e & ((1 << PB) - 1)); };
    if (tid == 0) { mbi(&full[0]); mbi(&full[1]); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    __syncthreads();
    auto stage = [&](int64_t t, int k) {
        if (BULK) {
            if (warp == 0) {
                if (lane == 0) mbx(&full[k], TS * 16);
                __syncwarp();
                for (int h = lane; h < NPIECE; h += 32) bulk3(S3 + k * TS + (h << PB), rc + (t << PB) + ((int64_t)h << AHI), 16u << PB, &full[k]);
            }
        } else {
            for (int j = 0; j < TS / NT; ++j) cpa16(S3 + k * TS + tid + j * NT, rc + row(t, tid + j * NT));
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
    };
    double wx = 0, ax = 0;
    int64_t t = blockIdx.x;
    if (t < ntiles) stage(t, 0);
    for (int it = 0; t < ntiles; ++it, t += gridDim.x) {
        const int k = it & 1;
        cplx *S = S3 + k * TS;
        if (t + gridDim.x < ntiles) stage(t + gridDim.x, k ^ 1);
        cplx QA[PER][G], C[PER][G], D[PER][G];
        auto loads = [&]() {
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const int64_t s = row(t, (tid + j * NT) * G);
                if (LD256) { ld2(q + s, QA[j][0], QA[j][1]); ld2(rp + s, C[j][0], C[j][1]); ld2(b + s, D[j][0], D[j][1]); }
                else { QA[j][0] = ldcs(q + s); C[j][0] = ldcs(rp + s); D[j][0] = ldcs(b + s); }
            }
        };
        if (EARLY) loads();
        if (BULK) mbw(&full[k], (it >> 1) & 1);
        else {
            if (t + gridDim.x < ntiles) asm volatile("cp.async.wait_group 1;" ::: "memory");
            else asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncthreads();
        }
        if (!EARLY) loads();
        cplx o[PER][G];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int e0 = (tid + j * NT) * G;
            const int64_t s = row(t, e0);
            cplx *qa = QA[j], *c = C[j], *d = D[j];
#pragma unroll
            for (int m = 0; m < G; ++m) {
                const int e = e0 + m;
                cplx h = qa[m];
#pragma unroll
                for (int jj = 0; jj < HB - 1; ++jj)
                    if (((e >> (PB + jj)) ^ (e >> (PB + jj + 1))) & 1) { const cplx p = S[e ^ (3 << (PB + jj))]; h.x += 0.5 * p.x; h.y += 0.5 * p.y; }
                if (((e >> (TB - 1)) ^ e) & 1) { const cplx p = S[e ^ ((1 << (TB - 1)) | 1)]; h.x += 0.5 * p.x; h.y += 0.5 * p.y; }
                const cplx v = S[e];
                o[j][m] = make_double2(0.5 * v.x + 0.25 * h.x - 0.125 * c[m].x, 0.5 * v.y + 0.25 * h.y - 0.125 * c[m].y);
                ax += o[j][m].x * d[m].x + o[j][m].y * d[m].y;
            }
            if (LD256) st2(rn + s, o[j][0], o[j][1]); else __stcs(rn + s, o[j][0]);
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < PER; ++j) for (int m = 0; m < G; ++m) S[(tid + j * NT) * G + m] = o[j][m];
        __syncthreads();
#pragma unroll
        for (int j = 0; j < PER; ++j) for (int m = 0; m < G; ++m) {
            const int e = (tid + j * NT) * G + m;
            cplx h = make_double2(0, 0);
#pragma unroll
            for (int jj = 0; jj < HB - 1; ++jj)
                if (!((e >> (PB + jj)) & 1) && ((e >> (PB + jj + 1)) & 1)) { const cplx p = S[e ^ (3 << (PB + jj))]; h.x += p.x; h.y += p.y; }
            wx += o[j][m].x * h.x - o[j][m].y * h.y;
        }
        __syncthreads();
    }
    if (wx + ax == 1234.5) part[0] = make_double2(wx, ax);
}

static float timeit(void (*f)(void *), void *arg, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f(arg);
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) f(arg);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

struct Bufs {
    cplx *v[5];
    double2 *part;
    unsigned long long *work;
    int64_t M;
    int grid, dyn;
    int64_t pad;
};
static Bufs G;

static void run_lin(void *) { lin<<<148 * 8, 256>>>(G.v[0], G.v[1], G.v[2], G.v[3], G.v[4], G.M, G.part); }
template <int L, int AHI, int PB, int NT>
static void run_b(void *) {
    constexpr int TS = 1 << (PB + L - AHI);
    cudaMemsetAsync(G.work, 0, 8);
    bord<L, AHI, PB, NT><<<G.grid, NT, TS * sizeof(cplx)>>>(G.v[0], G.v[1], G.v[2], G.v[3], G.v[4], G.part, G.work, G.dyn);
}
template <int L, int AHI, int PB, int NT>
static void bench(int ctas) {
    constexpr int TS = 1 << (PB + L - AHI);
    cudaFuncSetAttribute(bord<L, AHI, PB, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, TS * (int)sizeof(cplx));
    for (int dyn = 0; dyn < 2; ++dyn) {
        G.grid = 148 * ctas;
        G.dyn = dyn;
        float ms = timeit(run_b<L, AHI, PB, NT>, nullptr, 3);
        cudaError_t e = cudaGetLastError();
        printf("B-order L=%d AHI=%d PB=%d (piece %4d B, tile %3d KB) NT=%4d ctas/SM=%d %s: %8.3f ms  %7.1f GB/s  %s\n", L, AHI, PB,
               16 << PB, TS * 16 / 1024, NT, ctas, dyn ? "queue " : "static", ms, 80.0 * G.M / (ms * 1e6),
               cudaGetErrorString(e));
    }
}

template <int L, int AHI, int PB, int NT>
static void run_b2(void *) {
    constexpr int TS = 1 << (PB + L - AHI);
    bord2<L, AHI, PB, NT><<<G.grid, NT, 2 * TS * sizeof(cplx)>>>(G.v[0], G.v[1], G.v[2], G.v[3], G.v[4], G.part, G.pad);
}
template <int L, int AHI, int PB, int NT>
static void bench2(int ctas, int64_t pad = 0) {
    G.pad = pad;
    constexpr int TS = 1 << (PB + L - AHI);
    cudaFuncSetAttribute(bord2<L, AHI, PB, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * TS * (int)sizeof(cplx));
    G.grid = 148 * ctas;
    float ms = timeit(run_b2<L, AHI, PB, NT>, nullptr, 3);
    cudaError_t e = cudaGetLastError();
    printf("B-order/cp.async x2 L=%d AHI=%d PB=%d (piece %4d B, tile %3d KB) NT=%4d ctas/SM=%d pad=%7lld rows: %8.3f ms  %7.1f GB/s  %s\n", L, AHI, PB,
           16 << PB, TS * 16 / 1024, NT, ctas, (long long)pad, ms, 80.0 * G.M / (ms * 1e6), cudaGetErrorString(e));
}

template <int L, int AHI, int PB>
static void run_p(void *) { bpure<L, AHI, PB><<<148 * 8, 256>>>(G.v[0], G.v[1], G.v[2], G.v[3], G.v[4], G.M, G.part); }
template <int L, int AHI, int PB>
static void benchp() {
    float ms = timeit(run_p<L, AHI, PB>, nullptr, 3);
    printf("pure B-order L=%d AHI=%d PB=%d (piece %4d B, tile %d states): %8.3f ms  %7.1f GB/s  %s\n", L, AHI, PB, 16 << PB,
           1 << (PB + L - AHI), ms, 80.0 * G.M / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
}

template <bool BULK, bool LD256, int NT, bool EARLY>
static void run_b3(void *) {
    bord3<30, 22, 4, NT, BULK, LD256, EARLY><<<148, NT, 2 * 4096 * 16>>>(G.v[0], G.v[1], G.v[2], G.v[3], G.v[4], G.part);
}
template <bool BULK, bool LD256, int NT, bool EARLY = false>
static void bench3() {
    cudaFuncSetAttribute(bord3<30, 22, 4, NT, BULK, LD256, EARLY>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 4096 * 16);
    float ms = timeit(run_b3<BULK, LD256, NT, EARLY>, nullptr, 3);
    printf("v3 AHI=22 PB=4 NT=%d staging=%s loads=%s early=%d: %8.3f ms  %7.1f GB/s  %s\n", NT, BULK ? "bulk/piece" : "cp.async16",
           LD256 ? "256-bit" : "128-bit", (int)EARLY, ms, 80.0 * G.M / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
}

int main() {
    G.M = int64_t(1) << 30;
    const int64_t alloc = G.M + 512 * ((int64_t(1) << 17) + 4096);   // room for padded layouts
    for (int i = 0; i < 5; ++i) {
        if (cudaMalloc(&G.v[i], alloc * sizeof(cplx)) != cudaSuccess) { printf("alloc failed\n"); return 1; }
        cudaMemset(G.v[i], 0, alloc * sizeof(cplx));
    }
    cudaMalloc(&G.part, 64);
    cudaMalloc(&G.work, 64);
    float ms = timeit(run_lin, nullptr, 3);
    printf("linear update                      : %8.3f ms  %7.1f GB/s\n", ms, 80.0 * G.M / (ms * 1e6));
    for (int rep = 0; rep < 2; ++rep) {
        bench3<false, false, 1024>();
        bench3<false, true, 1024>();
        bench3<false, false, 1024, true>();
        bench3<false, true, 1024, true>();
        bench3<false, true, 512>();
        bench3<false, true, 512, true>();
        bench3<false, false, 512, true>();
    }
    return 0;
}
