// spmv_tiled.cuh — the tiled Heisenberg SpMV kernel (one instantiation per chain length L;
// the instantiations are spread over spmv_tiled_*.cu so they compile in parallel).
#pragma once
#include "spmv_common.cuh"
#include "spmv_stream.cuh"

namespace sk {

// Tiled kernel (bond-major within a tile of 2^T states).  Each thread owns PER = 2^T/256
// states (ls = tid + 256 k) with q in registers.
//   round 1: own tile (-> shared memory + diagonal), bond (T-1,T) and the periodic bond (L-1,0),
//            3*PER independent loads in flight per thread;
//   rounds 2..: the ACTIVE tile-level bonds i >= T (a bond flips two tile-index bits, so the
//            whole tile takes part or none: the active set is uniform per CTA), three partner
//            tiles per round, each a coalesced stream;
//   then the T-1 bonds inside the tile from shared memory.
// SPLIT (one GPU, COCG, N_left = 1): only H_A — the diagonal and the bonds
// (i, i+1), i < kp.split_ahi; the periodic bond and the bonds i >= split_ahi are applied by the
// update kernel (update_split.cu).
// TILED_SPLIT_QCS = 1: the SPLIT kernel's output is stored evict-first (st.global.cs): at the
// chain lengths of the split the update reads it from DRAM anyway, and L2 keeps more of r.
#ifndef TILED_SPLIT_QCS
#define TILED_SPLIT_QCS 1
#endif

// Worker CTAs of the fused SPLIT kernel, once per launch (CTA-uniform; ends with a barrier): wait
// until CTA 0 has published the final state (kp.kflag), then -kappa = -gamma sr_prev / sr_cur
// (steps.cuh seed_compute: a_prev / a_q) into *out.  Returns 1 when kappa == 0 (first iteration:
// r_{n-1} does not exist yet), else 2.
static __device__ __noinline__ int wait_kappa(const uint32_t *kflag, const DevState *st, cplx *out) {
    if (threadIdx.x == 0) {
        unsigned f;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(kflag) : "memory");
            if (!f) __nanosleep(100);
        } while (!f);
        const cplx g = __ldcg(&st->gamma_nx), sp = __ldcg(&st->sr_prev), sc_ = __ldcg(&st->sr_cur);
        cplx kap = mk(0.0, 0.0);
        if (g.x != 0.0 || g.y != 0.0) kap = xdiv(cmul(g, sp), sc_);
        *out = mk(-kap.x, -kap.y);
    }
    __syncthreads();
    return (out->x == 0.0 && out->y == 0.0) ? 1 : 2;
}

template <int L, int T, int NRHS, bool MULTI, bool SPLIT = false>
__global__ void __launch_bounds__(kThreads, NRHS == 1 ? (SPLIT ? TILED_SPLIT_MINB : 4) : 2)
heisenberg_tiled_kernel(SpmvArgs a, KParams kp, double J) {
    extern __shared__ cplx tile[];   // [NRHS][2^T]
    __shared__ StepScratch sc;
    using U = typename std::conditional<(L <= 31), uint32_t, uint64_t>::type;
    bool agent;
    int buf;
    if (!spmv_enter(a, agent, buf, sc, kp)) return;
    constexpr int TS = 1 << T;
    constexpr int PER = TS / kThreads;
#ifndef TILED_SPLIT_NB
#define TILED_SPLIT_NB 3
#endif
    constexpr int NB = SPLIT ? TILED_SPLIT_NB : 3;   // partner tiles per round
    static_assert(PER * kThreads == TS, "tile must be a multiple of the CTA size");
    const cplx *__restrict__ r = pick3(a.r, buf);
    const cplx *__restrict__ t = pick3(a.t, buf);
    // global view of r (and r~): with world > 1 partner tiles on other ranks are read in place
    // through peer memory; every partner tile below is resolved once per tile (its shard is
    // uniform over the tile).
    const RViewT<MULTI> rv = rview<MULTI>(r, kp.shard_r, buf, kp), tv = rview<MULTI>(t, kp.shard_t, buf, kp);
    // SPLIT with the fused r_{n-1} term (kp.split_fuse, §5.9): q <- H_A r_n - kappa r_{n-1}.  CTA 0
    // publishes that the state is final (its finish fixed gamma and the lazy scales); a worker
    // needs kappa only at the end of its first tile.
    const bool fuse = SPLIT && kp.split_fuse != 0;
    __shared__ cplx s_nkap;   // -kappa
    int kstate = 0;           // 0: not read yet, 1: kappa == 0 (first iteration), 2: kappa != 0
    if (SPLIT && fuse && agent) {
        __threadfence();
        __syncthreads();   // the finish's state_store is complete
        if (threadIdx.x == 0) {
            __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(kp.kflag), "r"(1u) : "memory");
        }
    }
    const double qJ = 0.25 * J, hJ = 0.5 * J;
    const int64_t ntiles = a.M >> T;
    const int tid = threadIdx.x;
    const int off = a.st ? 1 : 0;
    cplx w = mk(0.0, 0.0);
    for (int64_t ti = (int64_t)blockIdx.x - off; !agent && ti < ntiles; ti += gridDim.x - off) {
        const int64_t lbase = ti << T;                  // local row of the tile
        const U base = (U)((MULTI ? rv.row0 : 0) + lbase);   // global basis state of the tile
        __syncthreads();   // previous tile's shared-memory reads are done
        // r_{n-1} of the tile's rows is needed last: one bulk L2 prefetch now (no register or L1
        // cost; a normal-priority fill — evict-first loads that MISS L2 wrecked the partner tiles'
        // hit rate, 52% -> 22%), the loads themselves after the in-tile bonds
        if (SPLIT && fuse && kstate != 1 && tid == 0)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pick3(a.r, buf + 2) + lbase), "r"((unsigned)(sizeof(cplx) << T)) : "memory");
        cplx q[PER], qt[NRHS == 2 ? PER : 1];
        {
            cplx v0[PER], v1[PER], v2[PER], t0[NRHS == 2 ? PER : 1], t1[NRHS == 2 ? PER : 1],
                t2[NRHS == 2 ? PER : 1];
            const U tb = (base >> T) & (U)1, hb = (base >> (L - 1)) & (U)1;
            // partner tiles: bond (T-1, T) flips bit T (and bit T-1 inside the tile); the
            // periodic bond (L-1, 0) flips bit L-1 (and bit 0 inside the tile)
            const cplx *p1 = rv.at(base ^ ((U)1 << T)), *p2 = rv.at(base ^ ((U)1 << (L - 1)));
            const cplx *p1t = nullptr, *p2t = nullptr;
            if (NRHS == 2) { p1t = tv.at(base ^ ((U)1 << T)); p2t = tv.at(base ^ ((U)1 << (L - 1))); }
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int ls = tid + k * kThreads;
                v0[k] = r[lbase + ls];
                if (NRHS == 2) t0[k] = t[lbase + ls];
                const bool on1 = ((U)((ls >> (T - 1)) & 1) ^ tb) != 0;    // bond (T-1, T)
                const int l1 = ls ^ (1 << (T - 1));
                v1[k] = on1 ? p1[l1] : mk(0.0, 0.0);
                if (NRHS == 2) t1[k] = on1 ? p1t[l1] : mk(0.0, 0.0);
                const bool on2 = !SPLIT && ((U)(ls & 1) ^ hb) != 0;      // bond (L-1, 0)
                v2[k] = on2 ? p2[ls ^ 1] : mk(0.0, 0.0);
                if (NRHS == 2) t2[k] = on2 ? p2t[ls ^ 1] : mk(0.0, 0.0);
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
            // bond (T-2, T-1) = local bits (8, 9) = the thread's own k: states k = 1, 2 are each
            // other's partner, still in registers here
            if (PER == 4) {
                q[1].x = fma(hJ, v0[2].x, q[1].x); q[1].y = fma(hJ, v0[2].y, q[1].y);
                q[2].x = fma(hJ, v0[1].x, q[2].x); q[2].y = fma(hJ, v0[1].y, q[2].y);
                if (NRHS == 2) {
                    qt[1].x = fma(hJ, t0[2].x, qt[1].x); qt[1].y = fma(hJ, t0[2].y, qt[1].y);
                    qt[2].x = fma(hJ, t0[1].x, qt[2].x); qt[2].y = fma(hJ, t0[1].y, qt[2].y);
                }
            }
        }
        if (L - 1 > T) {
            const U tbits = base >> T;   // bit (i - T) of tbits = site i, for i >= T
            U act = (tbits ^ (tbits >> 1)) & ((((U)1) << (L - 1 - T)) - (U)1);   // bonds T..L-2
            if (SPLIT) act &= (((U)1) << (kp.split_ahi - T)) - (U)1;             // ... below split_ahi
            // full rounds of NB partner tiles without predication (the active set is uniform per
            // tile), then at most one predicated round for the remainder
            while (((L <= 31) ? __popc((unsigned)act) : __popcll((unsigned long long)act)) >= NB) {
                const cplx *pt[NB], *ptt[NB];
#pragma unroll
                for (int m = 0; m < NB; ++m) {
                    const int pos = (L <= 31) ? __ffs((int)act) - 1 : __ffsll((long long)act) - 1;
                    act &= act - (U)1;
                    const U pb = base ^ ((U)3 << (pos + T));
                    pt[m] = rv.at(pb) + tid;
                    ptt[m] = NRHS == 2 ? tv.at(pb) + tid : nullptr;
                }
                cplx v[NB][PER], vt[NB][NRHS == 2 ? PER : 1];
#pragma unroll
                for (int m = 0; m < NB; ++m)
#pragma unroll
                    for (int k = 0; k < PER; ++k) {
                        v[m][k] = pt[m][k * kThreads];
                        if (NRHS == 2) vt[m][k] = ptt[m][k * kThreads];
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
            if (act) {
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
                    const U pb = base ^ ((U)3 << (bi[m] < 0 ? T : bi[m]));
                    const cplx *pt = rv.at(pb);
                    const cplx *ptt = NRHS == 2 ? tv.at(pb) : nullptr;
#pragma unroll
                    for (int k = 0; k < PER; ++k) {
                        v[m][k] = bi[m] >= 0 ? pt[tid + k * kThreads] : mk(0.0, 0.0);
                        if (NRHS == 2) vt[m][k] = bi[m] >= 0 ? ptt[tid + k * kThreads] : mk(0.0, 0.0);
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
        // Bonds (i, i+1), i < T-1, inside the tile.  The tile's low bits of state ls = tid + 256 k
        // are tid (bits 0..7) and k (bits 8, 9), so: bonds i <= 6 are decided by tid alone (one
        // test per thread, the four states' partners at tid ^ (3 << i) + 256 k: constant
        // offsets); bond 7 by tid bit 7 and k bit 0 (partner k ^ 1); bond 8 by k alone — between
        // the thread's own states, applied in round 1 while they were in registers.
        static_assert(T == 10 && kThreads == 256 && PER == 4, "bit split assumes 1024-state tiles");
        {
            const unsigned xt = (unsigned)(tid ^ (tid >> 1));
#pragma unroll
            for (int i = 0; i < 7; ++i) {
                if (SPLIT && i < kp.split_lo) continue;   // in H_B (the update's B-tiles, §5.9)
                if ((xt >> i) & 1u) {
                    const int lp = tid ^ (3 << i);
#pragma unroll
                    for (int k = 0; k < PER; ++k) {
                        const cplx v = tile[lp + k * kThreads];
                        q[k].x = fma(hJ, v.x, q[k].x);
                        q[k].y = fma(hJ, v.y, q[k].y);
                        if (NRHS == 2) {
                            const cplx vt = tile[TS + lp + k * kThreads];
                            qt[k].x = fma(hJ, vt.x, qt[k].x);
                            qt[k].y = fma(hJ, vt.y, qt[k].y);
                        }
                    }
                }
            }
            const int b7 = (tid >> 7) & 1, lp7 = tid ^ 128;
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                if (b7 ^ (k & 1)) {   // bond (7, 8)
                    const cplx v = tile[lp7 + (k ^ 1) * kThreads];
                    q[k].x = fma(hJ, v.x, q[k].x);
                    q[k].y = fma(hJ, v.y, q[k].y);
                    if (NRHS == 2) {
                        const cplx vt = tile[TS + lp7 + (k ^ 1) * kThreads];
                        qt[k].x = fma(hJ, vt.x, qt[k].x);
                        qt[k].y = fma(hJ, vt.y, qt[k].y);
                    }
                }
                // (bond (8, 9) was applied from registers in round 1)
            }
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {   // w = <r~|r, H r> of the tile (before the fused term)
            const int ls = tid + k * kThreads;
            if (NRHS == 2) w = cfma_conj(tile[TS + ls], q[k], w);
            else w = cfma(tile[ls], q[k], w);
        }
        if (SPLIT && fuse) {
            if (kstate == 0) kstate = wait_kappa(kp.kflag, a.st, &s_nkap);   // once per CTA (uniform)
            if (kstate == 2) {
                const cplx *__restrict__ rpv = pick3(a.r, buf + 2) + lbase + tid;   // r_{n-1} (stored form)
                cplx rp[PER];
#pragma unroll
                for (int k = 0; k < PER; ++k) rp[k] = ldg_cs(rpv + k * kThreads);
                const cplx nkap = s_nkap;
#pragma unroll
                for (int k = 0; k < PER; ++k) q[k] = cfma(nkap, rp[k], q[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int ls = tid + k * kThreads;
            if (SPLIT && TILED_SPLIT_QCS) stg_cs(a.q + lbase + ls, q[k]);
            else a.q[lbase + ls] = q[k];
            if (NRHS == 2) a.qt[lbase + ls] = qt[k];
        }
    }
    spmv_exit(a, kp, agent, w, sc);
}

template <int L>
static cudaError_t launch_tiled(const SpmvArgs &a, const KParams &kp, double J, int grid, cudaStream_t s) {
    constexpr int T = kTileBits;
    if (a.work && heis_stream(L, a.M, a.bicg, kp.split_ahi > 0 && a.st)) return launch_stream<L>(a, kp, J, grid, s);
    const size_t shm = sizeof(cplx) << T;
    const bool p = a.st != nullptr;
    if (a.bicg) {
        static PerDevice cfg;
        const cudaError_t e = once_per_device(cfg, [&] {
            cudaError_t r = cudaFuncSetAttribute(heisenberg_tiled_kernel<L, T, 2, false>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * shm));
            if (r == cudaSuccess)
                r = cudaFuncSetAttribute(heisenberg_tiled_kernel<L, T, 2, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * shm));
            return r;
        });
        if (e != cudaSuccess) return e;
        if (kp.world > 1)
            return launch_k(heisenberg_tiled_kernel<L, T, 2, true>, grid, kThreads, 2 * shm, s, p, a, kp, J);
        return launch_k(heisenberg_tiled_kernel<L, T, 2, false>, grid, kThreads, 2 * shm, s, p, a, kp, J);
    }
    if (kp.world > 1)
        return launch_k(heisenberg_tiled_kernel<L, T, 1, true>, grid, kThreads, shm, s, p, a, kp, J);
    if (kp.split_ahi > 0 && a.st)   // solver mode with the bond split: H_A only
        return launch_k(heisenberg_tiled_kernel<L, T, 1, false, true>, grid, kThreads, shm, s, p, a, kp, J);
    return launch_k(heisenberg_tiled_kernel<L, T, 1, false>, grid, kThreads, shm, s, p, a, kp, J);
}

}  // namespace sk

#define SK_TILED_CASE(LL) case LL: return launch_tiled<LL>(a, kp, J, grid, s);
#define SK_TILED_RANGE(NAME, CASES)                                                          \
    namespace sk {                                                                           \
    cudaError_t NAME(int L, const SpmvArgs &a, const KParams &kp, double J, int grid,        \
                     cudaStream_t s) {                                                       \
        switch (L) { CASES default: return cudaErrorInvalidValue; }                          \
    }                                                                                        \
    }
