// update.cu — a5 + a7 of one iteration: the fused three-term seed update
//   r_{n+1} = (1 + c - alpha z_s) r_n + alpha q - c r_{n-1}      (EQ-CG-RN-3REC P:L269, A r = z_s r - q)
//   (BiCG shadow with conjugated coefficients)
// with the reductions of the next iteration (rho_{n+1}, ||r_{n+1}||^2, a_l^dagger r_{n+1}) and,
// in full mode, the all-shift update p^k = r_n/pi^k + beta^k p^k, x^k += alpha^k p^k
// (EQ-SHIFTEDCG-x/p P:L327-328) for every active shift in the same pass over r_n.
// CTA 0 is the shift agent: the projected per-shift recurrences (steps.cuh shift_step) run
// beside the streaming CTAs.
#include "kernels.cuh"
#include "steps.cuh"

namespace sk {

int shift_agents(int nz) {
    int a = (nz + kThreads - 1) / kThreads;   // ~one shift per agent thread
    return a < 1 ? 1 : (a > 8 ? 8 : a);
}

#ifndef UPD_MINB
#define UPD_MINB 4
#endif
int update_blocks(int64_t M, int nl, int full, int nz) {
    const int R = 1;   // rows per thread per chunk (the non-full kernel pipelines two chunks)
    int64_t b = (M + (int64_t)kThreads * R - 1) / ((int64_t)kThreads * R);
    const int64_t cap = (int64_t)sm_count() * UPD_MINB - shift_agents(nz);   // + the agents = one full wave at 4 CTAs/SM
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
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


// Seed scalars of the iteration this update kernel advances.  Deferred mode (world == 1): every
// CTA reduces the SpMV's w partials in the fixed order of reduce_w_fixed and evaluates
// seed_compute itself (thread 0, broadcast through shared memory) — the same bits the next
// finish will commit; no last-CTA hand-off, no serial tail on the critical path.  Otherwise the
// seed step already ran (SpMV's last CTA, or seed_kernel after the all-reduce) and the scalars
// are read from the state.  Returns false on a breakdown (deferred mode; the commit reports it).
// CTA 0 publishes seq (the SpMV's buffer / partial-half counter) and, deferred, pending.
struct UpdSeed {
    DevState S;
    SeedOut o;
    int64_t nsx;   // n_started after the seed step of this iteration
    cplx red8[8];
};
static __device__ __forceinline__ bool update_seed(const KParams &kp, UpdSeed &us) {
    DevState *st = kp.st;
    if (kp.defer) {
        const int64_t m = st->n_started;
        state_load_nosync(us.S, st);   // (published by the barriers of the reduction)
        const cplx w = reduce_w_fixed(kp.part_w + (m & 1) * kp.wred_stride + kp.wred_off, kp.wred_n, us.red8);
        if (threadIdx.x == 0) {
            us.o = seed_compute(us.S, w);
            us.nsx = m + 1;
            if (blockIdx.x == 0) {   // (nothing in this kernel reads rec, pending or seq)
                st->rec = us.o;
                st->pending = 1;     // the next finish commits rec (or reports the breakdown)
                if (us.o.ok) st->seq = m + 1;
            }
        }
        __syncthreads();
        return us.o.ok != 0;
    }
    if (threadIdx.x == 0) {
        us.o.alpha = st->alpha;
        us.o.beta = st->beta;
        us.o.c = st->c;
        us.o.a_cur = st->a_cur;
        us.o.a_q = st->a_q;
        us.o.a_prev = st->a_prev;
        us.o.sr = st->sr_it;
        us.o.ok = 1;
        us.nsx = st->n_started;
        if (blockIdx.x == 0) st->seq = us.nsx;
    }
    __syncthreads();
    return true;
}

// ============================================================================ fused update
// Each thread owns R rows per sweep (rows tid, tid+256, ... of a 256*R chunk) and issues all of
// their loads before any arithmetic, so 4R+ independent 16-byte loads are in flight per thread.
template <int NLMAX, bool BICG, bool FULL, int R>
__global__ void __launch_bounds__(kThreads, FULL ? 2 : UPD_MINB)
update_kernel(KParams kp, const cplx *__restrict__ q, const cplx *__restrict__ qt) {
    extern __shared__ cplx dyn[];  // FULL: coef[3 nz], flags[nz], list[nz]
    __shared__ ShiftScratch ss;
    __shared__ UpdSeed us;
    pdl_wait();
    DevState *st = kp.st;
    if (st->status != ST_ITERATING) return;
    const int wb = blockIdx.x - kp.n_agents, nwb = gridDim.x - kp.n_agents;
    const int64_t ns = st->n_started + (kp.defer ? 1 : 0);   // after the seed step of iteration n
    const cplx *__restrict__ rc_ = pick3(kp.r, ns + 2);
    const cplx *__restrict__ rp_ = pick3(kp.r, ns + 1);
    cplx *__restrict__ rn_ = pick3(kp.r, ns);
    const cplx *__restrict__ tc_ = pick3(kp.t, ns + 2);
    const cplx *__restrict__ tp_ = pick3(kp.t, ns + 1);
    cplx *__restrict__ tn_ = pick3(kp.t, ns);
    const int64_t M = kp.M;
    const int nl = kp.nl;
    const int64_t chunk = (int64_t)kThreads * R;
    const int64_t base0 = (int64_t)wb * chunk;
    // streamed rows of a chunk; the first chunk's loads do not depend on the seed scalars and
    // are issued before them (their latency overlaps the w reduction and the seed step)
    struct Chunk {
        cplx rc[R], rp[R], qi[R], tc[R], tp[R], qti[R], lv[R][NLMAX];
    };
    Chunk A;
    auto load_chunk = [&](Chunk &C, int64_t base) {
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int64_t i = base + threadIdx.x + (int64_t)k * kThreads;
            if (i < M) {
                C.rc[k] = ldg_cs(rc_ + i);
                C.rp[k] = ldg_cs(rp_ + i);
                C.qi[k] = ldg_cs(q + i);
                if (BICG) { C.tc[k] = ldg_cs(tc_ + i); C.tp[k] = ldg_cs(tp_ + i); C.qti[k] = ldg_cs(qt + i); }
#pragma unroll
                for (int l = 0; l < NLMAX; ++l)
                    if (l < nl) C.lv[k][l] = ldg_cs(kp.left + (int64_t)l * M + i);
            }
        }
    };
    Chunk B;   // (non-full: the second chunk is also loaded before the seed scalars)
    const int64_t step = (int64_t)nwb * chunk;
    if (wb >= 0 && base0 < M) load_chunk(A, base0);
    if (!FULL && wb >= 0 && base0 + step < M) load_chunk(B, base0 + step);
    if (blockIdx.x == kp.n_agents) dbg_stamp(kp.dbg_ts, 13);
    if (!update_seed(kp, us)) return;
    if (blockIdx.x == kp.n_agents) dbg_stamp(kp.dbg_ts, 14);
    if (blockIdx.x < kp.n_agents) {   // shift agents (a4 + a6 + pending a8), beside the streaming CTAs
        if (blockIdx.x == 0) dbg_stamp(kp.dbg_ts, 5);
        shift_step(kp, ss, blockIdx.x, us.o.alpha, us.o.beta, us.o.c);
        __syncthreads();
        if (blockIdx.x == 0) dbg_stamp(kp.dbg_ts, 6);
        return;
    }
    if (blockIdx.x == kp.n_agents) dbg_stamp(kp.dbg_ts, 7);
    const cplx a_cur = us.o.a_cur, a_q = us.o.a_q, a_prev = us.o.a_prev;
    const cplx ac_cur = cconj(a_cur), ac_q = cconj(a_q), ac_prev = cconj(a_prev);
    int nact = 0;
    cplx *coef = dyn;      // FULL: [3 nz] coefficients, dense by shift index
    int *act = nullptr;    // FULL: compacted list of the shifts streamed this iteration
    if (FULL) {
        // Every streaming CTA evaluates the pending retirement test and the coefficients of
        // the active shifts itself — the same arithmetic as the shift agent, so identical
        // decisions and bit-identical values: p^k = sr_n r_stored / pi_n^k + beta^k p^k.
        const int nz = kp.nz;
        int *flag = (int *)(dyn + 3 * nz);
        act = flag + nz;
        const int64_t n = st->n;
        const cplx *cur = kp.pibuf + (size_t)(n % 3) * nz;
        const cplx *prv = kp.pibuf + (size_t)((n + 2) % 3) * nz;
        const cplx bc = st->bscale[n % 3], bp = st->bscale[(n + 2) % 3];
        const bool lz = st->lz_pending != 0 && st->lz_iter == n;
        const double lz_nu = st->lz_nu, tol = st->tol;
        const cplx alpha = us.o.alpha, beta = us.o.beta, c = us.o.c, zs = st->zs, sr = us.o.sr;
        for (int k = threadIdx.x; k < nz; k += blockDim.x) {
            bool on = kp.active[k] != 0;
            const cplx pik = cmul(cur[k], bc), piok = cmul(prv[k], bp);
            if (on && lz) {
                double rk;
                if (retire_test(lz_nu, pik, tol, rk)) on = false;
            }
            flag[k] = on;
            if (on) {
                const ShiftCoef sc = shift_coef(pik, piok, kp.z[k], zs, alpha, beta, c, n);
                coef[3 * k] = cmul(sr, sc.ipik);
                coef[3 * k + 1] = sc.bk;
                coef[3 * k + 2] = sc.ak;
            }
        }
        __syncthreads();
        // ascending compaction of the flags (warp ballots + a warp scan of the warp counts)
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        for (int base = 0; base < nz; base += blockDim.x) {
            const int k = base + threadIdx.x;
            const int f = k < nz ? flag[k] : 0;
            const unsigned bal = __ballot_sync(0xffffffffu, f);
            if (lane == 0) ss.ri[warp] = __popc(bal);
            __syncthreads();
            if (warp == 0) {
                const int v = lane < nw ? ss.ri[lane] : 0;
                int incl = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += t;
                }
                if (lane < nw) ss.rc[lane] = incl - v;
                if (lane == 31) ss.ri[31] = incl;   // (nw <= 8: slot 31 is free)
            }
            __syncthreads();
            if (f) act[nact + ss.rc[warp] + __popc(bal & ((1u << lane) - 1u))] = k;
            nact += ss.ri[31];
            __syncthreads();
        }
    }
    cplx acc[2 + NLMAX];
#pragma unroll
    for (int j = 0; j < 2 + NLMAX; ++j) acc[j] = mk(0.0, 0.0);
    auto compute = [&](Chunk &C, int64_t base) {
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int64_t i = base + threadIdx.x + (int64_t)k * kThreads;
            if (i >= M) continue;
            cplx rn = cmul(a_cur, C.rc[k]);
            rn = cfma(a_q, C.qi[k], rn);
            rn = cfma(a_prev, C.rp[k], rn);
            rn_[i] = rn;
            if (BICG) {
                cplx tn = cmul(ac_cur, C.tc[k]);
                tn = cfma(ac_q, C.qti[k], tn);
                tn = cfma(ac_prev, C.tp[k], tn);
                tn_[i] = tn;
                acc[0] = cfma_conj(tn, rn, acc[0]);
            } else {
                acc[0] = cfma(rn, rn, acc[0]);
            }
            acc[1].x = fma(rn.x, rn.x, fma(rn.y, rn.y, acc[1].x));
#pragma unroll
            for (int l = 0; l < NLMAX; ++l)
                if (l < nl) acc[2 + l] = cfma_conj(C.lv[k][l], rn, acc[2 + l]);
            if (FULL) {
                const cplx r0 = C.rc[k];
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
                        const int kk = act[j + uu];
                        cplx pn = cmul(coef[3 * kk], r0);
                        pn = cfma(coef[3 * kk + 1], pk[uu], pn);
                        stg_cs(kp.p + off, pn);
                        stg_cs(kp.x + off, cfma(coef[3 * kk + 2], pn, xk[uu]));
                    }
                }
                for (; j < nact; ++j) {
                    const int64_t off = (int64_t)act[j] * M + i;
                    const cplx pk = ldg_cs(kp.p + off), xk = ldg_cs(kp.x + off);
                    const int kk = act[j];
                    cplx pn = cmul(coef[3 * kk], r0);
                    pn = cfma(coef[3 * kk + 1], pk, pn);
                    stg_cs(kp.p + off, pn);
                    stg_cs(kp.x + off, cfma(coef[3 * kk + 2], pn, xk));
                }
            }
        }
    };
    if (!FULL) {
        // software pipeline (two register sets, loop unrolled by two): A holds the chunk at
        // `base`, B the next one; a set is refilled with the chunk after next once computed
        int64_t base = base0;
        while (base < M) {
            compute(A, base);
            if (base + 2 * step < M) load_chunk(A, base + 2 * step);
            base += step;
            if (base >= M) break;
            compute(B, base);
            if (base + 2 * step < M) load_chunk(B, base + 2 * step);
            base += step;
        }
    } else {
        for (int64_t base = base0; base < M; base += step) {
            if (base != base0) load_chunk(A, base);
            compute(A, base);
        }
    }
    __shared__ cplx scratch[(2 + NLMAX) * (kThreads / 32)];
    block_sum<2 + NLMAX>(acc, scratch);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int j = 0; j < 2 + NLMAX; ++j)
            if (j < 2 + kp.nl) kp.part_u[(int64_t)wb * (2 + kp.nl) + j] = acc[j];
    }
    if (blockIdx.x == gridDim.x - 1) dbg_stamp(kp.dbg_ts, 8);
    if (kp.world > 1) {   // this rank's dots for the all-reduce: the last worker CTA sums them
        __shared__ RedScratch rs;
        __shared__ int last;
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) last = (atomicAdd(kp.ticket_u, 1u) == (unsigned)nwb - 1u);
        __syncthreads();
        if (!last) return;
        __threadfence();
        reduce_columns(kp.part_u, nwb, 2 + kp.nl, 2 + kp.nl, rs);
        if (threadIdx.x < 2 + kp.nl) kp.uloc[threadIdx.x] = rs.col[threadIdx.x];
        if (threadIdx.x == 0) *kp.ticket_u = 0u;
    }
}

// Projection-heavy variant (N_left > 4, projections only; C4 has 32 left vectors = 512 B/row,
// 63% of its bytes).  Holding N_left accumulators per thread would spill, so a CTA works on
// 256-row chunks: every thread forms r_{n+1} (+ shadow) for one row and parks it in shared
// memory; then warp w owns left vectors l = w, w+8, w+16, w+24 and streams a_l over the chunk
// (8 rows per lane, eight coalesced 16-byte loads in flight) into 4 per-lane accumulators.
template <bool BICG>
__global__ void __launch_bounds__(kThreads, 4)
update_proj_kernel(KParams kp, const cplx *__restrict__ q, const cplx *__restrict__ qt) {
    __shared__ ShiftScratch ss;
    __shared__ cplx rtile[kThreads];
    __shared__ cplx scratch[4 * (kThreads / 32)];
    __shared__ cplx lsum[32][1];
    __shared__ UpdSeed us;
    pdl_wait();
    DevState *st = kp.st;
    if (st->status != ST_ITERATING) return;
    if (!update_seed(kp, us)) return;
    if (blockIdx.x < kp.n_agents) {   // shift agents, beside the streaming CTAs
        shift_step(kp, ss, blockIdx.x, us.o.alpha, us.o.beta, us.o.c);
        return;
    }
    const int wb = blockIdx.x - kp.n_agents, nwb = gridDim.x - kp.n_agents;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ns = us.nsx;
    const cplx *__restrict__ rc_ = pick3(kp.r, ns + 2);
    const cplx *__restrict__ rp_ = pick3(kp.r, ns + 1);
    cplx *__restrict__ rn_ = pick3(kp.r, ns);
    const cplx *__restrict__ tc_ = pick3(kp.t, ns + 2);
    const cplx *__restrict__ tp_ = pick3(kp.t, ns + 1);
    cplx *__restrict__ tn_ = pick3(kp.t, ns);
    const cplx a_cur = us.o.a_cur, a_q = us.o.a_q, a_prev = us.o.a_prev;
    const cplx ac_cur = cconj(a_cur), ac_q = cconj(a_q), ac_prev = cconj(a_prev);
    const int64_t M = kp.M;
    const int nl = kp.nl;
    cplx rho = mk(0, 0), nu = mk(0, 0);
    cplx pa[4] = {mk(0, 0), mk(0, 0), mk(0, 0), mk(0, 0)};   // l = warp + 8 j
    for (int64_t base = (int64_t)wb * kThreads; base < M; base += (int64_t)nwb * kThreads) {
        const int64_t i = base + tid;
        cplx rn = mk(0, 0);
        if (i < M) {
            const cplx rc = ldg_cs(rc_ + i), rp = ldg_cs(rp_ + i), qi = ldg_cs(q + i);
            rn = cmul(a_cur, rc);
            rn = cfma(a_q, qi, rn);
            rn = cfma(a_prev, rp, rn);
            rn_[i] = rn;
            if (BICG) {
                const cplx tc = ldg_cs(tc_ + i), tp = ldg_cs(tp_ + i), qti = ldg_cs(qt + i);
                cplx tn = cmul(ac_cur, tc);
                tn = cfma(ac_q, qti, tn);
                tn = cfma(ac_prev, tp, tn);
                tn_[i] = tn;
                rho = cfma_conj(tn, rn, rho);
            } else {
                rho = cfma(rn, rn, rho);
            }
            nu.x = fma(rn.x, rn.x, fma(rn.y, rn.y, nu.x));
        }
        __syncthreads();   // previous chunk's tile reads done
        rtile[tid] = rn;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int l = warp + 8 * j;
            if (l >= nl) break;
            const cplx *al = kp.left + (int64_t)l * M + base;
            cplx av[8];
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int row = lane + 32 * m;
                av[m] = (base + row < M) ? ldg_cs(al + row) : mk(0, 0);
            }
#pragma unroll
            for (int m = 0; m < 8; ++m) pa[j] = cfma_conj(av[m], rtile[lane + 32 * m], pa[j]);
        }
    }
    // CTA partials: rho, ||r||^2 (block sum) and a_l^dagger r (per-warp sums)
    cplx v2[2] = {rho, nu};
    block_sum<2>(v2, scratch);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const cplx s = warp_sum(pa[j]);
        const int l = warp + 8 * j;
        if (lane == 0 && l < nl) lsum[l][0] = s;   // (one warp owns each l)
    }
    __syncthreads();
    cplx *dst = kp.part_u + (int64_t)wb * (2 + nl);
    if (tid == 0) { dst[0] = v2[0]; dst[1] = v2[1]; }
    if (tid < nl) dst[2 + tid] = lsum[tid][0];
    if (kp.world > 1) {   // this rank's dots for the all-reduce: the last worker CTA sums them
        __shared__ RedScratch rs;
        __shared__ int last;
        __threadfence();
        __syncthreads();
        if (tid == 0) last = (atomicAdd(kp.ticket_u, 1u) == (unsigned)nwb - 1u);
        __syncthreads();
        if (!last) return;
        __threadfence();
        reduce_columns(kp.part_u, nwb, 2 + nl, 2 + nl, rs);
        if (tid < 2 + nl) kp.uloc[tid] = rs.col[tid];
        if (tid == 0) *kp.ticket_u = 0u;
    }
}

template <int NLMAX, bool BICG, bool FULL>
static cudaError_t launch_update_t(const KParams &kp, const cplx *q, const cplx *qt, cudaStream_t s) {
    constexpr int R = 1;   // must match update_blocks()
    const size_t shm = FULL ? (size_t)kp.nz * (3 * sizeof(cplx) + 2 * sizeof(int)) : 0;
    if (FULL && shm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(update_kernel<NLMAX, BICG, FULL, R>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
        if (e != cudaSuccess) return e;
    }
    return launch_k(update_kernel<NLMAX, BICG, FULL, R>, kp.nblk_upd + kp.n_agents, kThreads, shm, s, true,
                    kp, q, qt);
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
    if (kp.split_ahi > 0) return launch_update_split(kp, q, s);
    if (kp.nl > 4 && !kp.full) {
        if (kp.bicg)
            return launch_k(update_proj_kernel<true>, kp.nblk_upd + kp.n_agents, kThreads, 0, s, true, kp, q, qt);
        return launch_k(update_proj_kernel<false>, kp.nblk_upd + kp.n_agents, kThreads, 0, s, true, kp, q, qt);
    }
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
