// spmv.cu — a1 + a2 of one iteration: q = H r_n (BiCG: also qt = H r~_n) with the fused
// partial dot w = <r~|r, q> (unconjugated for COCG, App. A; conjugated for BiCG,
// P:L1014), plus the scalar work that rides along the SpMV launch:
//   * CTA 0 is the finish agent: residuals, retirement and seed switch of the previous
//     iteration (steps.cuh finish_step) — concurrent with the SpMV of the other CTAs;
//   * the last CTA to finish (ticket) reduces the w partials in CTA order and computes the seed
//     scalars of this iteration (steps.cuh seed_step).
// Operators: on-the-fly S=1/2 Heisenberg chain (generated as in P:L508) and CSR.
#include <cstdlib>
#include <type_traits>

#include "kernels.cuh"
#include "steps.cuh"

namespace sk {

int stream_blocks(int64_t M) {
    int64_t b = (M + kThreads - 1) / kThreads;
    if (b > kMaxBlocks) b = kMaxBlocks;
    if (b < 1) b = 1;
    return (int)b;
}

int heisenberg_blocks(int L, int64_t M) {
    if (L > kTileBits && L <= 34 && M >= (int64_t(1) << kTileBits)) {
        const int64_t ntiles = M >> kTileBits;
        return (int)(ntiles < (int64_t)kMaxBlocks ? ntiles : (int64_t)kMaxBlocks);
    }
    return stream_blocks(M);
}

// View of one rotating r buffer as the GLOBAL vector: this rank's rows are local; with
// world > 1 every other rank's rows are reached through the shard table (peer memory over
// NVLink, or the other contexts of a loopback group) — the exchange of the operator is fused
// into the SpMV's own loads.
struct RView {
    const cplx *loc;
    const cplx *const *tab;   // [world] for this buffer index, or null (world <= 1)
    int64_t row0;
    int lloc, world;
    __device__ __forceinline__ const cplx *at(uint64_t g) const {
        if (world <= 1) return loc + (int64_t)(g - (uint64_t)row0);
        return tab[g >> lloc] + (g & ((1ull << lloc) - 1ull));
    }
};
__device__ __forceinline__ RView rview(const cplx *loc, const cplx *const *shard, int buf, const KParams &kp) {
    RView v;
    v.loc = loc;
    v.world = kp.world;
    v.tab = (kp.world > 1 && shard) ? shard + (size_t)buf * kp.world : nullptr;
    v.row0 = kp.world > 1 ? kp.row0 : 0;
    v.lloc = kp.lloc_bits;
    return v;
}

// Common prologue/epilogue of the solver-mode SpMV kernels.  Returns false when the kernel
// should do nothing (terminal state).  `agent` is true for CTA 0 in solver mode.
__device__ __forceinline__ bool spmv_enter(const SpmvArgs &a, bool &agent, int &buf, StepScratch &sc,
                                          const KParams &kp) {
    agent = false;
    buf = 0;
    if (!a.st) return true;
    if (a.st->status != ST_ITERATING) return false;
    buf = (int)(a.st->n_started % 3);
    if (blockIdx.x == 1) dbg_stamp(kp.dbg_ts, 0);                 // first worker CTA starts
    if (blockIdx.x == 0) {
        agent = true;
        dbg_stamp(kp.dbg_ts, 1);
        if (a.st->pending) finish_step(kp, sc, /*eager=*/false);
        dbg_stamp(kp.dbg_ts, 2);                                   // finish agent done
    }
    return true;
}

__device__ __forceinline__ void spmv_exit(const SpmvArgs &a, const KParams &kp, bool agent, cplx w,
                                          StepScratch &sc) {
    __shared__ cplx scratch[kThreads / 32];
    __shared__ int last;
    if (!agent && a.part_w) {
        cplx v[1] = {w};
        block_sum<1>(v, scratch);
        if (threadIdx.x == 0) a.part_w[blockIdx.x - (a.st ? 1 : 0)] = v[0];
    }
    if (!a.st) return;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(kp.ticket, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!last) return;
    dbg_stamp(kp.dbg_ts, 3);                                       // last CTA arrives
    __threadfence();
    if (kp.world > 1) {   // this rank's w only: the all-reduce and the seed step follow
        reduce_columns(a.part_w, gridDim.x - 1, 1, 1, sc);
        if (threadIdx.x == 0) {
            kp.wloc[0] = sc.col[0];
            *kp.ticket = 0u;
        }
        return;
    }
    state_load_nosync(sc.S, kp.st);
    reduce_columns(a.part_w, gridDim.x - 1, 1, 1, sc);   // (its barriers publish sc.S)
    if (threadIdx.x == 0) {
        if (sc.S.status == ST_ITERATING) seed_step(&sc.S, sc.col[0], a.bicg, kp);
        *kp.ticket = 0u;
    }
    __syncthreads();
    // breakdown ends the run here: apply the pending retirement test so results are final
    if (sc.S.status == ST_BREAKDOWN && sc.S.lz_pending) retire_pass(kp, sc);
    state_store(kp.st, sc.S);
    dbg_stamp(kp.dbg_ts, 4);                                       // seed step done
}

// ============================================================================ Heisenberg H.v
// Simple kernel (L <= kTileBits, and standalone use): one thread per state.  x = s XOR rot(s)
// has bit i set iff sites i, i+1 are anti-aligned; diagonal J/4 (L - 2 popc x); each
// anti-aligned bond flips both spins with amplitude J/2.
template <int NRHS>
__global__ void __launch_bounds__(kThreads) heisenberg_kernel(SpmvArgs a, KParams kp, int L, double J) {
    __shared__ StepScratch sc;
    bool agent;
    int buf;
    if (!spmv_enter(a, agent, buf, sc, kp)) return;
    const cplx *__restrict__ r = pick3(a.r, buf);
    const cplx *__restrict__ t = pick3(a.t, buf);
    const RView rv = rview(r, kp.shard_r, buf, kp), tv = rview(t, kp.shard_t, buf, kp);
    const double qJ = 0.25 * J, hJ = 0.5 * J;
    const int64_t M = a.M;
    const uint64_t row0 = (uint64_t)rv.row0;
    const int off = a.st ? 1 : 0;
    cplx w = mk(0.0, 0.0);
    if (!agent) {
        for (int64_t s = (int64_t)(blockIdx.x - off) * blockDim.x + threadIdx.x; s < M;
             s += (int64_t)(gridDim.x - off) * blockDim.x) {
            const uint64_t us = row0 + (uint64_t)s;   // global basis state
            const uint64_t x = us ^ ((us >> 1) | ((us & 1ull) << (L - 1)));
            const double d = qJ * (double)(L - 2 * __popcll(x));
            const cplx rs = r[s];
            cplx q = mk(d * rs.x, d * rs.y);
            cplx ts = mk(0, 0), qt = mk(0, 0);
            if (NRHS == 2) { ts = t[s]; qt = mk(d * ts.x, d * ts.y); }
            for (int i = 0; i < L; ++i) {
                if ((x >> i) & 1ull) {
                    const int j = (i + 1 == L) ? 0 : i + 1;
                    const uint64_t s2 = us ^ ((1ull << i) | (1ull << j));
                    const cplx v = *rv.at(s2);
                    q.x = fma(hJ, v.x, q.x);
                    q.y = fma(hJ, v.y, q.y);
                    if (NRHS == 2) {
                        const cplx vt = *tv.at(s2);
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
    }
    spmv_exit(a, kp, agent, w, sc);
}

// Tiled kernel (bond-major within a tile of 2^T states).  Each thread owns PER = 2^T/256
// states (ls = tid + 256 k) with q in registers.
//   round 1: own tile (-> shared memory + diagonal), bond (T-1,T) and the periodic bond (L-1,0),
//            3*PER independent loads in flight per thread;
//   rounds 2..: the ACTIVE tile-level bonds i >= T (a bond flips two tile-index bits, so the
//            whole tile takes part or none: the active set is uniform per CTA), three partner
//            tiles per round, each a coalesced stream;
//   then the T-1 bonds inside the tile from shared memory.
template <int L, int T, int NRHS>
__global__ void __launch_bounds__(kThreads, NRHS == 1 ? 4 : 2)
heisenberg_tiled_kernel(SpmvArgs a, KParams kp, double J) {
    extern __shared__ cplx tile[];   // [NRHS][2^T]
    __shared__ StepScratch sc;
    using U = typename std::conditional<(L <= 31), uint32_t, uint64_t>::type;
    bool agent;
    int buf;
    if (!spmv_enter(a, agent, buf, sc, kp)) return;
    constexpr int TS = 1 << T;
    constexpr int PER = TS / kThreads;
    constexpr int NB = 3;
    static_assert(PER * kThreads == TS, "tile must be a multiple of the CTA size");
    const cplx *__restrict__ r = pick3(a.r, buf);
    const cplx *__restrict__ t = pick3(a.t, buf);
    // global view of r (and r~): with world > 1 partner tiles on other ranks are read in place
    // through peer memory; every partner tile below is resolved once per tile (its shard is
    // uniform over the tile).
    const RView rv = rview(r, kp.shard_r, buf, kp), tv = rview(t, kp.shard_t, buf, kp);
    const double qJ = 0.25 * J, hJ = 0.5 * J;
    const int64_t ntiles = a.M >> T;
    const int tid = threadIdx.x;
    const int off = a.st ? 1 : 0;
    cplx w = mk(0.0, 0.0);
    for (int64_t ti = (int64_t)blockIdx.x - off; !agent && ti < ntiles; ti += gridDim.x - off) {
        const int64_t lbase = ti << T;                  // local row of the tile
        const U base = (U)(rv.row0 + lbase);            // global basis state of the tile
        __syncthreads();   // previous tile's shared-memory reads are done
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
                const bool on2 = ((U)(ls & 1) ^ hb) != 0;                 // bond (L-1, 0)
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
        }
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
            a.q[lbase + ls] = q[k];
            if (NRHS == 2) {
                a.qt[lbase + ls] = qt[k];
                w = cfma_conj(tile[TS + ls], q[k], w);
            } else {
                w = cfma(tile[ls], q[k], w);
            }
        }
    }
    spmv_exit(a, kp, agent, w, sc);
}

template <int L>
static cudaError_t launch_tiled(const SpmvArgs &a, const KParams &kp, double J, int grid, cudaStream_t s) {
    constexpr int T = kTileBits;
    const size_t shm = sizeof(cplx) << T;
    if (a.bicg) {
        static bool cfg = false;
        if (!cfg) {
            cudaFuncSetAttribute(heisenberg_tiled_kernel<L, T, 2>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * shm));
            cfg = true;
        }
        heisenberg_tiled_kernel<L, T, 2><<<grid, kThreads, 2 * shm, s>>>(a, kp, J);
    } else {
        heisenberg_tiled_kernel<L, T, 1><<<grid, kThreads, shm, s>>>(a, kp, J);
    }
    return cudaGetLastError();
}

cudaError_t launch_heisenberg(const SpmvArgs &a, const KParams &kp, int L, double J, cudaStream_t s) {
    const int workers = heisenberg_blocks(L, a.M);
    const int grid = workers + (a.st ? 1 : 0);
    if (a.M >= (int64_t(1) << kTileBits)) switch (L) {
#define SK_TILED_CASE(LL) case LL: return launch_tiled<LL>(a, kp, J, grid, s);
        SK_TILED_CASE(11) SK_TILED_CASE(12) SK_TILED_CASE(13) SK_TILED_CASE(14) SK_TILED_CASE(15)
        SK_TILED_CASE(16) SK_TILED_CASE(17) SK_TILED_CASE(18) SK_TILED_CASE(19) SK_TILED_CASE(20)
        SK_TILED_CASE(21) SK_TILED_CASE(22) SK_TILED_CASE(23) SK_TILED_CASE(24) SK_TILED_CASE(25)
        SK_TILED_CASE(26) SK_TILED_CASE(27) SK_TILED_CASE(28) SK_TILED_CASE(29) SK_TILED_CASE(30)
        SK_TILED_CASE(31) SK_TILED_CASE(32) SK_TILED_CASE(33) SK_TILED_CASE(34)
#undef SK_TILED_CASE
        default: break;
    }
    if (a.bicg) heisenberg_kernel<2><<<grid, kThreads, 0, s>>>(a, kp, L, J);
    else heisenberg_kernel<1><<<grid, kThreads, 0, s>>>(a, kp, L, J);
    return cudaGetLastError();
}

// ============================================================================ CSR SpMV
// LPR lanes per row (LPR | 32), lanes stride over the row's entries, shuffle-reduce in the
// group.  Column ids are int32, row pointers int64, values fp64 or complex128.
template <int LPR, bool CV, int NRHS>
__global__ void __launch_bounds__(kThreads)
csr_kernel(SpmvArgs a, KParams kp, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
           const void *__restrict__ valv) {
    __shared__ StepScratch sc;
    bool agent;
    int buf;
    if (!spmv_enter(a, agent, buf, sc, kp)) return;
    const cplx *__restrict__ r = pick3(a.r, buf);
    const cplx *__restrict__ t = pick3(a.t, buf);
    const RView rv = rview(r, kp.shard_r, buf, kp), tv = rview(t, kp.shard_t, buf, kp);
    const int off = a.st ? 1 : 0;
    const int lane = threadIdx.x & (LPR - 1);
    const unsigned gmask = (LPR == 32) ? 0xffffffffu
                                       : (((1u << LPR) - 1u) << ((threadIdx.x & 31) & ~(LPR - 1)));
    const int64_t ngroups = (int64_t)(gridDim.x - off) * blockDim.x / LPR;
    cplx w = mk(0.0, 0.0);
    if (!agent) {
        for (int64_t i = ((int64_t)(blockIdx.x - off) * blockDim.x + threadIdx.x) / LPR; i < a.M; i += ngroups) {
            const int64_t e0 = rp[i], e1 = rp[i + 1];
            cplx acc = mk(0.0, 0.0), acct = mk(0.0, 0.0);
            for (int64_t e = e0 + lane; e < e1; e += LPR) {
                const int c = col[e];                      // global column id
                const cplx x = *rv.at((uint64_t)c);
                if (CV) {
                    const cplx v = ((const cplx *)valv)[e];
                    acc = cfma(v, x, acc);
                    if (NRHS == 2) acct = cfma(v, *tv.at((uint64_t)c), acct);
                } else {
                    const double v = ((const double *)valv)[e];
                    acc.x = fma(v, x.x, acc.x);
                    acc.y = fma(v, x.y, acc.y);
                    if (NRHS == 2) {
                        const cplx xt = *tv.at((uint64_t)c);
                        acct.x = fma(v, xt.x, acct.x);
                        acct.y = fma(v, xt.y, acct.y);
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
    }
    spmv_exit(a, kp, agent, w, sc);
}

// Row-per-thread CSR variant: each thread owns whole rows and issues the loads of four entries
// (column ids, values, then the four gathers) before their FMAs, so a warp keeps 32 rows'
// dependent chains (row_ptr -> col -> r[col]) in flight instead of 32/LPR.
template <bool CV, int NRHS>
__global__ void __launch_bounds__(kThreads)
csr_row_kernel(SpmvArgs a, KParams kp, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
               const void *__restrict__ valv) {
    __shared__ StepScratch sc;
    bool agent;
    int buf;
    if (!spmv_enter(a, agent, buf, sc, kp)) return;
    const cplx *__restrict__ r = pick3(a.r, buf);
    const cplx *__restrict__ t = pick3(a.t, buf);
    const RView rv = rview(r, kp.shard_r, buf, kp), tv = rview(t, kp.shard_t, buf, kp);
    const int off = a.st ? 1 : 0;
    cplx w = mk(0.0, 0.0);
    if (!agent) {
        for (int64_t i = (int64_t)(blockIdx.x - off) * blockDim.x + threadIdx.x; i < a.M;
             i += (int64_t)(gridDim.x - off) * blockDim.x) {
            const int64_t e0 = rp[i], e1 = rp[i + 1];
            cplx acc = mk(0.0, 0.0), acct = mk(0.0, 0.0);
            for (int64_t e = e0; e < e1; e += 4) {
                int c[4];
                cplx v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const bool in = e + u < e1;
                    c[u] = in ? col[e + u] : -1;
                    if (CV) v[u] = in ? ((const cplx *)valv)[e + u] : mk(0, 0);
                    else v[u] = mk(in ? ((const double *)valv)[e + u] : 0.0, 0.0);
                }
                cplx x[4], xt[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    x[u] = c[u] >= 0 ? *rv.at((uint64_t)c[u]) : mk(0, 0);
                    if (NRHS == 2) xt[u] = c[u] >= 0 ? *tv.at((uint64_t)c[u]) : mk(0, 0);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (CV) {
                        acc = cfma(v[u], x[u], acc);
                        if (NRHS == 2) acct = cfma(v[u], xt[u], acct);
                    } else {
                        acc.x = fma(v[u].x, x[u].x, acc.x);
                        acc.y = fma(v[u].x, x[u].y, acc.y);
                        if (NRHS == 2) { acct.x = fma(v[u].x, xt[u].x, acct.x); acct.y = fma(v[u].x, xt[u].y, acct.y); }
                    }
                }
            }
            a.q[i] = acc;
            if (NRHS == 2) {
                a.qt[i] = acct;
                w = cfma_conj(t[i], acc, w);
            } else {
                w = cfma(r[i], acc, w);
            }
        }
    }
    spmv_exit(a, kp, agent, w, sc);
}

template <int LPR>
static void csr_dispatch(const SpmvArgs &a, const KParams &kp, const int64_t *rp, const int32_t *col,
                         const void *val, bool cv, int grid, cudaStream_t s) {
    if (cv) {
        if (a.bicg) csr_kernel<LPR, true, 2><<<grid, kThreads, 0, s>>>(a, kp, rp, col, val);
        else csr_kernel<LPR, true, 1><<<grid, kThreads, 0, s>>>(a, kp, rp, col, val);
    } else {
        if (a.bicg) csr_kernel<LPR, false, 2><<<grid, kThreads, 0, s>>>(a, kp, rp, col, val);
        else csr_kernel<LPR, false, 1><<<grid, kThreads, 0, s>>>(a, kp, rp, col, val);
    }
}

int csr_mode() {   // 0: lanes-per-row kernel, 1: row-per-thread kernel (default)
    static int m = -1;
    if (m < 0) {
        const char *e = getenv("SHIFTK_CSR_ROW");
        m = e ? atoi(e) : 1;
    }
    return m;
}

int csr_blocks(int64_t M) {
    if (csr_mode() == 0) return stream_blocks(M);
    int64_t b = (M + kThreads - 1) / kThreads;
    return (int)(b > kMaxSpmvBlocks ? kMaxSpmvBlocks : (b < 1 ? 1 : b));
}

cudaError_t launch_csr(const SpmvArgs &a, const KParams &kp, const int64_t *rp, const int32_t *col,
                       const void *val, bool cv, double avg_nnz, cudaStream_t s) {
    const int grid = csr_blocks(a.M) + (a.st ? 1 : 0);
    if (csr_mode() == 1) {
        if (cv) {
            if (a.bicg) csr_row_kernel<true, 2><<<grid, kThreads, 0, s>>>(a, kp, rp, col, val);
            else csr_row_kernel<true, 1><<<grid, kThreads, 0, s>>>(a, kp, rp, col, val);
        } else {
            if (a.bicg) csr_row_kernel<false, 2><<<grid, kThreads, 0, s>>>(a, kp, rp, col, val);
            else csr_row_kernel<false, 1><<<grid, kThreads, 0, s>>>(a, kp, rp, col, val);
        }
        return cudaGetLastError();
    }
    if (avg_nnz <= 3.0) csr_dispatch<2>(a, kp, rp, col, val, cv, grid, s);
    else if (avg_nnz <= 6.0) csr_dispatch<4>(a, kp, rp, col, val, cv, grid, s);
    else if (avg_nnz <= 24.0) csr_dispatch<8>(a, kp, rp, col, val, cv, grid, s);
    else csr_dispatch<32>(a, kp, rp, col, val, cv, grid, s);
    return cudaGetLastError();
}

// ============================================================================ RC dot
// Reverse communication: the caller supplied q = H r; only the w partial (and the
// agent / seed-scalar tail) run here.
__global__ void __launch_bounds__(kThreads) rc_dot_kernel(SpmvArgs a, KParams kp) {
    __shared__ StepScratch sc;
    bool agent;
    int buf;
    if (!spmv_enter(a, agent, buf, sc, kp)) return;
    const cplx *__restrict__ tv = a.bicg ? pick3(a.t, buf) : pick3(a.r, buf);
    cplx w = mk(0.0, 0.0);
    if (!agent) {
        for (int64_t i = (int64_t)(blockIdx.x - 1) * blockDim.x + threadIdx.x; i < a.M;
             i += (int64_t)(gridDim.x - 1) * blockDim.x)
            w = a.bicg ? cfma_conj(tv[i], a.q[i], w) : cfma(tv[i], a.q[i], w);
    }
    spmv_exit(a, kp, agent, w, sc);
}

cudaError_t launch_rc_dot(const SpmvArgs &a, const KParams &kp, cudaStream_t s) {
    rc_dot_kernel<<<stream_blocks(a.M) + 1, kThreads, 0, s>>>(a, kp);
    return cudaGetLastError();
}

}  // namespace sk
