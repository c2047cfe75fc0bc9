// kernels.cu — the sm_100a kernels of one shifted COCG / BiCG iteration.
//
//   a1+a2  heisenberg_kernel / csr_kernel : q = H r_n (BiCG: also qt = H r~_n), fused partial
//          w = <r~|r, q> per CTA (unconjugated for COCG, App. A; conjugated for BiCG,
//          P:L1014)
//   a3-a9  scalar_kernel (1 CTA)           : deterministic reduction of the partials, seed
//          recurrences, per-shift pi/alpha/beta, projected
//          u/y update (corrected index R1), residuals, retirement,
//          seed switching
//   a5+a7  update_kernel                    : r_{n+1} = (1+c-alpha z_s) r_n + alpha q - c r_{n-1}
//          (EQ-CG-RN-3REC P:L269; shadow P:L1029) fused with the dots of the next iteration
//          (rho, ||r||^2, a_l^dag r) and, in full mode, the all-shift update
//          p^k = r_n/pi^k + beta^k p^k, x^k += alpha^k p^k for every active shift.
//
// All reductions are two-stage and deterministic: each CTA reduces its grid-stride rows in a
// fixed order, the scalar kernel sums the CTA partials in CTA order.
#include <type_traits>

#include "kernels.cuh"

namespace sk {

enum { ST_ITERATING = 0, ST_CONVERGED = 1, ST_MAXITER = 2, ST_BREAKDOWN = 3 };

// select one of three by-value pointers without dynamic indexing (keeps them in registers)
template <typename T>
__device__ __forceinline__ T pick3(T const (&a)[3], int64_t i) {
    const int k = (int)(i % 3);
    return k == 0 ? a[0] : (k == 1 ? a[1] : a[2]);
}

int heisenberg_blocks(int L, int64_t M) {
    if (L > kTileBitsPublic && L <= 34) {
        const int64_t ntiles = M >> kTileBitsPublic;
        return (int)(ntiles < (int64_t)kMaxBlocks ? ntiles : (int64_t)kMaxBlocks);
    }
    return stream_blocks(M);
}

int stream_blocks(int64_t M) {
    int64_t b = (M + kThreads - 1) / kThreads;
    if (b > kMaxBlocks) b = kMaxBlocks;
    if (b < 1) b = 1;
    return (int)b;
}

// ============================================================================ Heisenberg H.v
// H = J sum_{i<L} S_i.S_{i+1}, periodic.  x = s XOR rot(s) has bit i set iff sites i,
// i+1 are anti-aligned; diagonal = J/4 (L - 2 popc(x)); each anti-aligned bond flips both spins
// with amplitude J/2.  Bond loop is uniform across the warp so every gather r[s ^ m_i] of a
// warp reads one contiguous 512-byte block (coalesced).
template <int NRHS>
__global__ void __launch_bounds__(kThreads) heisenberg_kernel(SpmvArgs a, int L, double J) {
    int buf = 0;
    if (a.st) {
        if (a.st->status != ST_ITERATING) return;
        buf = (int)(a.st->n_started % 3);
    }
    const cplx *__restrict__ r = pick3(a.r, buf);
    const cplx *__restrict__ t = pick3(a.t, buf);
    const double qJ = 0.25 * J, hJ = 0.5 * J;
    const int64_t M = a.M;
    cplx w = mk(0.0, 0.0);
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < M;
         s += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t us = (uint64_t)s;
        const uint64_t rot = (us >> 1) | ((us & 1ull) << (L - 1));
        const uint64_t x = us ^ rot;
        const double d = qJ * (double)(L - 2 * __popcll(x));
        const cplx rs = r[s];
        cplx q = mk(d * rs.x, d * rs.y);
        cplx ts, qt;
        if (NRHS == 2) {
            ts = t[s];
            qt = mk(d * ts.x, d * ts.y);
        }
        for (int i = 0; i < L; ++i) {
            if ((x >> i) & 1ull) {
                const int j = (i + 1 == L) ? 0 : i + 1;
                const uint64_t s2 = us ^ ((1ull << i) | (1ull << j));
                const cplx v = r[s2];
                q.x = fma(hJ, v.x, q.x);
                q.y = fma(hJ, v.y, q.y);
                if (NRHS == 2) {
                    const cplx vt = t[s2];
                    qt.x = fma(hJ, vt.x, qt.x);
                    qt.y = fma(hJ, vt.y, qt.y);
                }
            }
        }
        a.q[s] = q;
        if (NRHS == 2) {
            a.qt[s] = qt;
            w = cfma_conj(ts, q, w);
        } else {
            w = cfma(rs, q, w);
        }
    }
    if (a.part_w) {
        __shared__ cplx scratch[kThreads / 32];
        cplx v[1] = {w};
        block_sum<1>(v, scratch);
        if (threadIdx.x == 0) a.part_w[blockIdx.x] = v[0];
    }
}

// Shared-memory tiled variant: a CTA stages a tile of 2^T consecutive states of r in shared
// memory (one coalesced pass), applies the T-1 bonds inside the tile from shared memory, and
// gathers only the L-T+1 bonds that leave the tile (bond (T-1,T), the tile-level bonds, and the
// periodic bond (L-1,0)) from global memory — each a contiguous, coalesced 512-byte warp read
// issued predicated and fully unrolled so that they are all in flight together.
constexpr int kTileBits = kTileBitsPublic;

template <int L, int T, int NRHS>
__global__ void __launch_bounds__(kThreads, NRHS == 1 ? 4 : 2)
heisenberg_tiled_kernel(SpmvArgs a, double J) {
    // Bond-major within a tile of 2^T states.  Each thread owns PER = 2^T/256 states
    // (ls = tid + 256 k) and keeps their q in registers.
    //   round 1: own tile (-> shared memory + diagonal), bond (T-1,T) and the periodic bond
    //            (L-1,0) — 3*PER independent loads in flight per thread;
    //   rounds 2..: the ACTIVE tile-level bonds i >= T (a bond flips two tile-index bits, so the
    //            whole tile takes part or none: the active set is uniform per CTA), three partner
    //            tiles per round, each a coalesced stream;
    //   then the T-1 bonds inside the tile from shared memory.
    extern __shared__ cplx tile[];   // [NRHS][2^T]
    using U = typename std::conditional<(L <= 31), uint32_t, uint64_t>::type;
    int buf = 0;
    if (a.st) {
        if (a.st->status != ST_ITERATING) return;
        buf = (int)(a.st->n_started % 3);
    }
    constexpr int TS = 1 << T;
    constexpr int PER = TS / kThreads;
    constexpr int NB = 3;   // tile-level bonds per round
    static_assert(PER * kThreads == TS, "tile must be a multiple of the CTA size");
    const cplx *__restrict__ r = pick3(a.r, buf);
    const cplx *__restrict__ t = pick3(a.t, buf);
    const double qJ = 0.25 * J, hJ = 0.5 * J;
    const int64_t ntiles = a.M >> T;
    const int tid = threadIdx.x;
    cplx w = mk(0.0, 0.0);
    for (int64_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
        const U base = (U)(ti << T);
        __syncthreads();   // previous tile's shared-memory reads are done
        cplx q[PER], qt[NRHS == 2 ? PER : 1];
        // ---- round 1 ---------------------------------------------------------------------
        {
            cplx v0[PER], v1[PER], v2[PER], t0[NRHS == 2 ? PER : 1], t1[NRHS == 2 ? PER : 1],
                t2[NRHS == 2 ? PER : 1];
            const U tb = (base >> T) & (U)1, hb = (base >> (L - 1)) & (U)1;
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int ls = tid + k * kThreads;
                const U s = base + (U)ls;
                v0[k] = r[s];
                if (NRHS == 2) t0[k] = t[s];
                const bool on1 = ((U)((ls >> (T - 1)) & 1) ^ tb) != 0;    // bond (T-1, T)
                const U s1 = s ^ ((U)3 << (T - 1));
                v1[k] = on1 ? r[s1] : mk(0.0, 0.0);
                if (NRHS == 2) t1[k] = on1 ? t[s1] : mk(0.0, 0.0);
                const bool on2 = ((U)(ls & 1) ^ hb) != 0;                 // bond (L-1, 0)
                const U s2 = s ^ (((U)1 << (L - 1)) | (U)1);
                v2[k] = on2 ? r[s2] : mk(0.0, 0.0);
                if (NRHS == 2) t2[k] = on2 ? t[s2] : mk(0.0, 0.0);
            }
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int ls = tid + k * kThreads;
                const U s = base + (U)ls;
                const U x = s ^ ((s >> 1) | ((s & (U)1) << (L - 1)));
                const int na = (L <= 31) ? __popc((unsigned)x) : __popcll((unsigned long long)x);
                const double d = qJ * (double)(L - 2 * na);
                tile[ls] = v0[k];
                q[k].x = fma(hJ, v1[k].x + v2[k].x, d * v0[k].x);
                q[k].y = fma(hJ, v1[k].y + v2[k].y, d * v0[k].y);
                if (NRHS == 2) {
                    tile[TS + ls] = t0[k];
                    qt[k].x = fma(hJ, t1[k].x + t2[k].x, d * t0[k].x);
                    qt[k].y = fma(hJ, t1[k].y + t2[k].y, d * t0[k].y);
                }
            }
        }
        // ---- rounds 2..: active tile-level bonds (uniform per CTA) ----------------------------
        if (L - 1 > T) {
            const U tbits = base >> T;   // bit (i - T) of tbits = site i, for i >= T
            U act = (tbits ^ (tbits >> 1)) & ((((U)1) << (L - 1 - T)) - (U)1);   // bonds T..L-2
            while (act) {
                int bi[NB];
#pragma unroll
                for (int m = 0; m < NB; ++m) {
                    bi[m] = -1;
                    if (act) {
                        const int pos = (L <= 31) ? __ffs((int)act) - 1 : __ffsll((long long)act) - 1;
                        bi[m] = pos + T;
                        act &= act - (U)1;
                    }
                }
                cplx v[NB][PER], vt[NB][NRHS == 2 ? PER : 1];
#pragma unroll
                for (int m = 0; m < NB; ++m) {
                    const U pb = base ^ ((U)3 << (bi[m] < 0 ? 0 : bi[m]));
#pragma unroll
                    for (int k = 0; k < PER; ++k) {
                        v[m][k] = bi[m] >= 0 ? r[pb + (U)(tid + k * kThreads)] : mk(0.0, 0.0);
                        if (NRHS == 2) vt[m][k] = bi[m] >= 0 ? t[pb + (U)(tid + k * kThreads)] : mk(0.0, 0.0);
                    }
                }
#pragma unroll
                for (int m = 0; m < NB; ++m)
#pragma unroll
                    for (int k = 0; k < PER; ++k) {
                        q[k].x = fma(hJ, v[m][k].x, q[k].x);
                        q[k].y = fma(hJ, v[m][k].y, q[k].y);
                        if (NRHS == 2) { qt[k].x = fma(hJ, vt[m][k].x, qt[k].x); qt[k].y = fma(hJ, vt[m][k].y, qt[k].y); }
                    }
            }
        }
        __syncthreads();   // tile staged
        // ---- bonds inside the tile (i = 0 .. T-2) from shared memory -------------------------
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int ls = tid + k * kThreads;
            const U s = base + (U)ls;
            const U x = s ^ (s >> 1);   // bit i (< T-1): sites i, i+1 anti-aligned
#pragma unroll
            for (int i = 0; i < T - 1; ++i) {
                if ((x >> i) & (U)1) {
                    const cplx v = tile[ls ^ (3 << i)];
                    q[k].x = fma(hJ, v.x, q[k].x);
                    q[k].y = fma(hJ, v.y, q[k].y);
                    if (NRHS == 2) {
                        const cplx vt = tile[TS + (ls ^ (3 << i))];
                        qt[k].x = fma(hJ, vt.x, qt[k].x);
                        qt[k].y = fma(hJ, vt.y, qt[k].y);
                    }
                }
            }
            a.q[s] = q[k];
            if (NRHS == 2) {
                a.qt[s] = qt[k];
                w = cfma_conj(tile[TS + ls], q[k], w);
            } else {
                w = cfma(tile[ls], q[k], w);
            }
        }
    }
    if (a.part_w) {
        __shared__ cplx scratch[kThreads / 32];
        cplx v[1] = {w};
        block_sum<1>(v, scratch);
        if (threadIdx.x == 0) a.part_w[blockIdx.x] = v[0];
    }
}

// ============================================================================ CSR SpMV
// LPR lanes per row (LPR | 32), lanes stride over the row's entries, shuffle-reduce in the
// group.  Column ids are int32, row pointers int64, values fp64 or complex128.
template <int LPR, bool CV, int NRHS>
__global__ void __launch_bounds__(kThreads)
csr_kernel(SpmvArgs a, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
           const void *__restrict__ valv) {
    int buf = 0;
    if (a.st) {
        if (a.st->status != ST_ITERATING) return;
        buf = (int)(a.st->n_started % 3);
    }
    const cplx *__restrict__ r = pick3(a.r, buf);
    const cplx *__restrict__ t = pick3(a.t, buf);
    const int lane = threadIdx.x & (LPR - 1);
    const unsigned gmask = (LPR == 32) ? 0xffffffffu
                                       : (((1u << LPR) - 1u) << ((threadIdx.x & 31) & ~(LPR - 1)));
    const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / LPR;
    cplx w = mk(0.0, 0.0);
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPR; i < a.M; i += ngroups) {
        const int64_t e0 = rp[i], e1 = rp[i + 1];
        cplx acc = mk(0.0, 0.0), acct = mk(0.0, 0.0);
        for (int64_t e = e0 + lane; e < e1; e += LPR) {
            const int c = col[e];
            const cplx rv = r[c];
            if (CV) {
                const cplx v = ((const cplx *)valv)[e];
                acc = cfma(v, rv, acc);
                if (NRHS == 2) acct = cfma(v, t[c], acct);
            } else {
                const double v = ((const double *)valv)[e];
                acc.x = fma(v, rv.x, acc.x);
                acc.y = fma(v, rv.y, acc.y);
                if (NRHS == 2) {
                    const cplx tv = t[c];
                    acct.x = fma(v, tv.x, acct.x);
                    acct.y = fma(v, tv.y, acct.y);
                }
            }
        }
#pragma unroll
        for (int o = LPR / 2; o > 0; o >>= 1) {
            acc.x += __shfl_xor_sync(gmask, acc.x, o);
            acc.y += __shfl_xor_sync(gmask, acc.y, o);
            if (NRHS == 2) {
                acct.x += __shfl_xor_sync(gmask, acct.x, o);
                acct.y += __shfl_xor_sync(gmask, acct.y, o);
            }
        }
        if (lane == 0) {
            a.q[i] = acc;
            if (NRHS == 2) {
                a.qt[i] = acct;
                w = cfma_conj(t[i], acc, w);
            } else {
                w = cfma(r[i], acc, w);
            }
        }
    }
    if (a.part_w) {
        __shared__ cplx scratch[kThreads / 32];
        cplx v[1] = {w};
        block_sum<1>(v, scratch);
        if (threadIdx.x == 0) a.part_w[blockIdx.x] = v[0];
    }
}

template <int L>
static cudaError_t launch_tiled(const SpmvArgs &a, double J, int nblk, cudaStream_t s) {
    constexpr int T = kTileBits;
    const int grid = nblk;   // == heisenberg_blocks(L, M): one partial per CTA
    const size_t shm = sizeof(cplx) << T;
    if (a.bicg) {
        static bool cfg = false;
        if (!cfg) {
            cudaFuncSetAttribute(heisenberg_tiled_kernel<L, T, 2>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * shm));
            cfg = true;
        }
        heisenberg_tiled_kernel<L, T, 2><<<grid, kThreads, 2 * shm, s>>>(a, J);
    } else {
        heisenberg_tiled_kernel<L, T, 1><<<grid, kThreads, shm, s>>>(a, J);
    }
    return cudaGetLastError();
}

cudaError_t launch_heisenberg(const SpmvArgs &a, int L, double J, int nblk, cudaStream_t s) {
    switch (L) {
#define SK_TILED_CASE(LL) case LL: return launch_tiled<LL>(a, J, nblk, s);
        SK_TILED_CASE(11) SK_TILED_CASE(12) SK_TILED_CASE(13) SK_TILED_CASE(14) SK_TILED_CASE(15) SK_TILED_CASE(16)
        SK_TILED_CASE(17) SK_TILED_CASE(18) SK_TILED_CASE(19) SK_TILED_CASE(20) SK_TILED_CASE(21)
        SK_TILED_CASE(22) SK_TILED_CASE(23) SK_TILED_CASE(24) SK_TILED_CASE(25) SK_TILED_CASE(26)
        SK_TILED_CASE(27) SK_TILED_CASE(28) SK_TILED_CASE(29) SK_TILED_CASE(30) SK_TILED_CASE(31)
        SK_TILED_CASE(32) SK_TILED_CASE(33) SK_TILED_CASE(34)
#undef SK_TILED_CASE
        default: break;
    }
    if (a.bicg)
        heisenberg_kernel<2><<<nblk, kThreads, 0, s>>>(a, L, J);
    else
        heisenberg_kernel<1><<<nblk, kThreads, 0, s>>>(a, L, J);
    return cudaGetLastError();
}

template <int LPR>
static void csr_dispatch(const SpmvArgs &a, const int64_t *rp, const int32_t *col, const void *val,
                         bool cv, int nblk, cudaStream_t s) {
    if (cv) {
        if (a.bicg) csr_kernel<LPR, true, 2><<<nblk, kThreads, 0, s>>>(a, rp, col, val);
        else csr_kernel<LPR, true, 1><<<nblk, kThreads, 0, s>>>(a, rp, col, val);
    } else {
        if (a.bicg) csr_kernel<LPR, false, 2><<<nblk, kThreads, 0, s>>>(a, rp, col, val);
        else csr_kernel<LPR, false, 1><<<nblk, kThreads, 0, s>>>(a, rp, col, val);
    }
}

cudaError_t launch_csr(const SpmvArgs &a, const int64_t *rp, const int32_t *col, const void *val,
                       bool cv, double avg_nnz, int nblk, cudaStream_t s) {
    if (avg_nnz <= 3.0) csr_dispatch<2>(a, rp, col, val, cv, nblk, s);
    else if (avg_nnz <= 6.0) csr_dispatch<4>(a, rp, col, val, cv, nblk, s);
    else if (avg_nnz <= 24.0) csr_dispatch<8>(a, rp, col, val, cv, nblk, s);
    else csr_dispatch<32>(a, rp, col, val, cv, nblk, s);
    return cudaGetLastError();
}

// ============================================================================ RC dot / init
__global__ void __launch_bounds__(kThreads) rc_dot_kernel(KParams kp, const cplx *__restrict__ q) {
    if (kp.st->status != ST_ITERATING) return;
    const int buf = (int)(kp.st->n_started % 3);
    const cplx *__restrict__ tv = kp.bicg ? pick3(kp.t, buf) : pick3(kp.r, buf);
    cplx w = mk(0.0, 0.0);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < kp.M;
         i += (int64_t)gridDim.x * blockDim.x)
        w = kp.bicg ? cfma_conj(tv[i], q[i], w) : cfma(tv[i], q[i], w);
    __shared__ cplx scratch[kThreads / 32];
    cplx v[1] = {w};
    block_sum<1>(v, scratch);
    if (threadIdx.x == 0) kp.part_w[blockIdx.x] = v[0];
}

cudaError_t launch_rc_dot(const KParams &kp, const cplx *q, cudaStream_t s) {
    rc_dot_kernel<<<kp.nblk_spmv, kThreads, 0, s>>>(kp, q);
    return cudaGetLastError();
}

template <int NLMAX>
__global__ void __launch_bounds__(kThreads) init_kernel(KParams kp, const cplx *__restrict__ b) {
    cplx acc[2 + NLMAX];
#pragma unroll
    for (int j = 0; j < 2 + NLMAX; ++j) acc[j] = mk(0.0, 0.0);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < kp.M;
         i += (int64_t)gridDim.x * blockDim.x) {
        const cplx bi = b[i];
        kp.r[0][i] = bi;
        if (kp.bicg) kp.t[0][i] = cconj(bi);   // r~_0 = conj(b)  (R3)
        acc[0] = cfma(bi, bi, acc[0]);          // rho_0 = <r~_0, r_0> = sum b_i^2 for both methods
        acc[1].x = fma(bi.x, bi.x, fma(bi.y, bi.y, acc[1].x));
#pragma unroll
        for (int l = 0; l < NLMAX; ++l)
            if (l < kp.nl) acc[2 + l] = cfma_conj(kp.left[(int64_t)l * kp.M + i], bi, acc[2 + l]);
    }
    __shared__ cplx scratch[(2 + NLMAX) * (kThreads / 32)];
    block_sum<2 + NLMAX>(acc, scratch);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int j = 0; j < 2 + NLMAX; ++j)
            if (j < 2 + kp.nl) kp.part_u[(int64_t)blockIdx.x * (2 + kp.nl) + j] = acc[j];
    }
}

// ============================================================================ fused update
// Each thread owns R rows per sweep (rows tid, tid+256, ... of a 256*R chunk) and issues all of
// their loads before any arithmetic, so 4R+ independent 16-byte loads are in flight per thread.
template <int NLMAX, bool BICG, bool FULL, int R>
__global__ void __launch_bounds__(kThreads)
update_kernel(KParams kp, const cplx *__restrict__ q, const cplx *__restrict__ qt) {
    extern __shared__ cplx dyn[];  // FULL: coef[3 * nz], then act list (int32)
    DevState *st = kp.st;
    if (st->status != ST_ITERATING) return;
    const int64_t ns = st->n_started;            // start(n) ran: ns = n + 1
    const cplx *__restrict__ rc_ = pick3(kp.r, ns + 2);
    const cplx *__restrict__ rp_ = pick3(kp.r, ns + 1);
    cplx *__restrict__ rn_ = pick3(kp.r, ns);
    const cplx *__restrict__ tc_ = pick3(kp.t, ns + 2);
    const cplx *__restrict__ tp_ = pick3(kp.t, ns + 1);
    cplx *__restrict__ tn_ = pick3(kp.t, ns);
    const cplx a_cur = st->a_cur, a_q = st->a_q, a_prev = st->a_prev;
    const cplx ac_cur = cconj(a_cur), ac_q = cconj(a_q), ac_prev = cconj(a_prev);
    int nact = 0;
    cplx *coef = dyn;
    int *act = nullptr;
    if (FULL) {
        nact = *kp.n_act_list;
        act = (int *)(dyn + 3 * kp.nz);
        for (int j = threadIdx.x; j < 3 * nact; j += blockDim.x) coef[j] = kp.coef[j];
        for (int j = threadIdx.x; j < nact; j += blockDim.x) act[j] = kp.act_list[j];
        __syncthreads();
    }
    cplx acc[2 + NLMAX];
#pragma unroll
    for (int j = 0; j < 2 + NLMAX; ++j) acc[j] = mk(0.0, 0.0);
    const int64_t M = kp.M;
    const int nl = kp.nl;
    const int64_t chunk = (int64_t)kThreads * R;
    for (int64_t base = (int64_t)blockIdx.x * chunk; base < M; base += (int64_t)gridDim.x * chunk) {
        cplx rc[R], rp[R], qi[R], tc[R], tp[R], qti[R], lv[R][NLMAX];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int64_t i = base + threadIdx.x + (int64_t)k * kThreads;
            if (i < M) {
                rc[k] = ldg_cs(rc_ + i);
                rp[k] = ldg_cs(rp_ + i);
                qi[k] = ldg_cs(q + i);
                if (BICG) { tc[k] = ldg_cs(tc_ + i); tp[k] = ldg_cs(tp_ + i); qti[k] = ldg_cs(qt + i); }
#pragma unroll
                for (int l = 0; l < NLMAX; ++l)
                    if (l < nl) lv[k][l] = ldg_cs(kp.left + (int64_t)l * M + i);
            }
        }
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int64_t i = base + threadIdx.x + (int64_t)k * kThreads;
            if (i >= M) continue;
            cplx rn = cmul(a_cur, rc[k]);
            rn = cfma(a_q, qi[k], rn);
            rn = cfma(a_prev, rp[k], rn);
            rn_[i] = rn;
            if (BICG) {
                cplx tn = cmul(ac_cur, tc[k]);
                tn = cfma(ac_q, qti[k], tn);
                tn = cfma(ac_prev, tp[k], tn);
                tn_[i] = tn;
                acc[0] = cfma_conj(tn, rn, acc[0]);
            } else {
                acc[0] = cfma(rn, rn, acc[0]);
            }
            acc[1].x = fma(rn.x, rn.x, fma(rn.y, rn.y, acc[1].x));
#pragma unroll
            for (int l = 0; l < NLMAX; ++l)
                if (l < nl) acc[2 + l] = cfma_conj(lv[k][l], rn, acc[2 + l]);
            if (FULL) {
                const cplx r0 = rc[k];
                int j = 0;
                for (; j + 4 <= nact; j += 4) {
                    cplx pk[4], xk[4];
#pragma unroll
                    for (int uu = 0; uu < 4; ++uu) {
                        const int64_t off = (int64_t)act[j + uu] * M + i;
                        pk[uu] = ldg_cs(kp.p + off);
                        xk[uu] = ldg_cs(kp.x + off);
                    }
#pragma unroll
                    for (int uu = 0; uu < 4; ++uu) {
                        const int64_t off = (int64_t)act[j + uu] * M + i;
                        cplx pn = cmul(coef[3 * (j + uu)], r0);
                        pn = cfma(coef[3 * (j + uu) + 1], pk[uu], pn);
                        stg_cs(kp.p + off, pn);
                        stg_cs(kp.x + off, cfma(coef[3 * (j + uu) + 2], pn, xk[uu]));
                    }
                }
                for (; j < nact; ++j) {
                    const int64_t off = (int64_t)act[j] * M + i;
                    const cplx pk = ldg_cs(kp.p + off), xk = ldg_cs(kp.x + off);
                    cplx pn = cmul(coef[3 * j], r0);
                    pn = cfma(coef[3 * j + 1], pk, pn);
                    stg_cs(kp.p + off, pn);
                    stg_cs(kp.x + off, cfma(coef[3 * j + 2], pn, xk));
                }
            }
        }
    }
    __shared__ cplx scratch[(2 + NLMAX) * (kThreads / 32)];
    block_sum<2 + NLMAX>(acc, scratch);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int j = 0; j < 2 + NLMAX; ++j)
            if (j < 2 + kp.nl) kp.part_u[(int64_t)blockIdx.x * (2 + kp.nl) + j] = acc[j];
    }
}

template <int NLMAX, bool BICG, bool FULL>
static cudaError_t launch_update_t(const KParams &kp, const cplx *q, const cplx *qt, cudaStream_t s) {
    constexpr int R = FULL ? 1 : (NLMAX <= 4 ? 4 : (NLMAX <= 8 ? 2 : 1));
    const size_t shm = FULL ? (size_t)kp.nz * (3 * sizeof(cplx) + sizeof(int)) : 0;
    if (FULL && shm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(update_kernel<NLMAX, BICG, FULL, R>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
        if (e != cudaSuccess) return e;
    }
    update_kernel<NLMAX, BICG, FULL, R><<<kp.nblk_upd, kThreads, shm, s>>>(kp, q, qt);
    return cudaGetLastError();
}

template <int NLMAX>
static cudaError_t launch_update_nl(const KParams &kp, const cplx *q, const cplx *qt, cudaStream_t s) {
    if (kp.full)
        return kp.bicg ? launch_update_t<NLMAX, true, true>(kp, q, qt, s)
                       : launch_update_t<NLMAX, false, true>(kp, q, qt, s);
    return kp.bicg ? launch_update_t<NLMAX, true, false>(kp, q, qt, s)
                   : launch_update_t<NLMAX, false, false>(kp, q, qt, s);
}

cudaError_t launch_update(const KParams &kp, const cplx *q, const cplx *qt, cudaStream_t s) {
    if (kp.nl <= 1) return launch_update_nl<1>(kp, q, qt, s);
    if (kp.nl <= 4) return launch_update_nl<4>(kp, q, qt, s);
    if (kp.nl <= 8) return launch_update_nl<8>(kp, q, qt, s);
    if (kp.nl <= 16) return launch_update_nl<16>(kp, q, qt, s);
    return launch_update_nl<32>(kp, q, qt, s);
}

cudaError_t launch_init(const KParams &kp, const cplx *b, cudaStream_t s) {
    if (kp.nl <= 1) init_kernel<1><<<kp.nblk_upd, kThreads, 0, s>>>(kp, b);
    else if (kp.nl <= 4) init_kernel<4><<<kp.nblk_upd, kThreads, 0, s>>>(kp, b);
    else if (kp.nl <= 8) init_kernel<8><<<kp.nblk_upd, kThreads, 0, s>>>(kp, b);
    else if (kp.nl <= 16) init_kernel<16><<<kp.nblk_upd, kThreads, 0, s>>>(kp, b);
    else init_kernel<32><<<kp.nblk_upd, kThreads, 0, s>>>(kp, b);
    return cudaGetLastError();
}

}  // namespace sk
