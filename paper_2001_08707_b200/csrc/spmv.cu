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
#include "spmv_common.cuh"

namespace sk {

bool pdl_enabled() {
    static int m = -1;
    if (m < 0) {
        const char *e = getenv("SHIFTK_PDL");
        m = e ? atoi(e) : 1;
    }
    return m != 0;
}

int stream_blocks(int64_t M) {
    int64_t b = (M + kThreads - 1) / kThreads;
    if (b > 8 * (int64_t)sm_count()) b = 8 * (int64_t)sm_count();
    if (b < 1) b = 1;
    return (int)b;
}

int sm_count() {   // per device (cached): grids are sized for the device the launch goes to
    static int n[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (!n[dev]) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        n[dev] = v > kMaxSms ? kMaxSms : v;
    }
    return n[dev];
}

// The streaming (TMA-fed) kernel wins once the vector outgrows L2 (measured: L=24 215 vs 233 us,
// L=26 0.98 vs 1.25 ms, L=28 4.8 vs 6.8 ms); below that the tiled kernel's shorter per-tile
// latency chain wins (L=20 13.4 vs 14.6 us).  SHIFTK_HEIS_STREAM=0/1 forces either.
static int stream_env() {
    static int en = -2;
    if (en == -2) {
        const char *e = getenv("SHIFTK_HEIS_STREAM");
        en = !e ? -1 : (e[0] == '0' ? 0 : 1);
    }
    return en;
}
bool heis_stream(int L, int64_t M, int bicg, bool split) {
    const int en = stream_env();
    if (en == 0 || bicg || L <= kTileBits || L > 34 || M < (int64_t(1) << kTileBits)) return false;
    // H_A of the bond split reaches only L2-resident partner tiles: there the
    // tiled kernel's direct loads win (L=30: 11.7 vs 16.3 ms); SHIFTK_HEIS_STREAM=1 forces it
    if (split) return en == 1;
    return en == 1 || (M >> kTileBits) >= 8192;
}

// Tile pairs across the top spin bit (spmv_stream.cuh heisenberg_pair_kernel) on one GPU from
// L = 24, where the periodic partner would otherwise come from DRAM; SHIFTK_HEIS_PAIRS=0/1.
bool heis_pairs(int L, int64_t M) {
    static int en = -1;
    if (en < 0) {
        const char *e = getenv("SHIFTK_HEIS_PAIRS");
        en = (e && e[0] == '0') ? 0 : 1;
    }
    return en && L >= 24 && M == (int64_t(1) << L);
}

int heisenberg_blocks(int L, int64_t M, int bicg, bool split) {
    if (heis_stream(L, M, bicg, split)) {   // two CTAs per SM, one slot left for the finish agent
        const int64_t ntiles = M >> kTileBits, slots = 2 * (int64_t)sm_count() - 1;
        return (int)(ntiles < slots ? ntiles : slots);
    }
    if (L > kTileBits && L <= 34 && M >= (int64_t(1) << kTileBits)) {
        const int64_t ntiles = M >> kTileBits;
        // one resident wave (4 CTAs per SM, one slot for the finish agent), tiles grid-strided:
        // no second-wave launches and prologues (measured at C2: 41.1 -> 41.0 us flushed step,
        // 30.7 -> 29.3 us per graph iteration)
        const int64_t cap = (split ? TILED_SPLIT_MINB : 4) * (int64_t)sm_count() - 1;
        return (int)(ntiles < cap ? ntiles : cap);
    }
    return stream_blocks(M);
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

cudaError_t launch_heisenberg(const SpmvArgs &a, const KParams &kp, int L, double J, cudaStream_t s) {
    const int workers = heisenberg_blocks(L, a.M, a.bicg, kp.split_ahi > 0 && a.st);
    const int grid = workers + (a.st ? 1 : 0);
    if (a.M >= (int64_t(1) << kTileBits) && L > kTileBits && L <= 34) {
        if (L <= 16) return launch_tiled_a(L, a, kp, J, grid, s);
        if (L <= 22) return launch_tiled_b(L, a, kp, J, grid, s);
        if (L <= 28) return launch_tiled_c(L, a, kp, J, grid, s);
        return launch_tiled_d(L, a, kp, J, grid, s);
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
template <bool CV, int NRHS, bool MULTI>
__global__ void __launch_bounds__(kThreads)
csr_row_kernel(SpmvArgs a, KParams kp, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
               const void *__restrict__ valv) {
    __shared__ StepScratch sc;
    bool agent;
    int buf;
    if (!spmv_enter(a, agent, buf, sc, kp)) return;
    const cplx *__restrict__ r = pick3(a.r, buf);
    const cplx *__restrict__ t = pick3(a.t, buf);
    const RViewT<MULTI> rv = rview<MULTI>(r, kp.shard_r, buf, kp), tv = rview<MULTI>(t, kp.shard_t, buf, kp);
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

// Column-blocked variant of csr_row_kernel (kp.csr_nblk passes, one launch each):
// pass b applies the entries whose column lies in block b = [b << bshift, (b + 1) << bshift), so
// the gathers of one pass fall into a slice of r that stays in L2 (a random 16-B gather from a
// vector larger than L2 costs ~100-128 B of DRAM traffic each).  MODE 0: first pass (q written),
// 1: middle (q accumulated), 2: last (q accumulated, w partials, CTA 0 = finish agent).
template <bool CV, int NRHS, int MODE>
__global__ void __launch_bounds__(kThreads)
csr_block_kernel(SpmvArgs a, KParams kp, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                 const void *__restrict__ valv, int b) {
    __shared__ StepScratch sc;
    bool agent = false;
    int buf = 0;
    if (MODE == 2) {
        if (!spmv_enter(a, agent, buf, sc, kp)) return;
    } else {
        pdl_wait();
        if (a.st) {   // (the finish of the previous iteration runs in the last pass: a terminal
                      // state decided there leaves the earlier passes' work unused)
            if (a.st->status != ST_ITERATING) return;
            buf = (int)(a.st->seq % 3);
        }
    }
    const cplx *__restrict__ r = pick3(a.r, buf);
    const cplx *__restrict__ t = pick3(a.t, buf);
    const uint8_t *__restrict__ s0p = kp.csr_split + (int64_t)b * a.M, *__restrict__ s1p = s0p + a.M;
    const int off = (MODE == 2 && a.st) ? 1 : 0;
    cplx w = mk(0.0, 0.0);
    if (!agent) {
        for (int64_t i = (int64_t)(blockIdx.x - off) * blockDim.x + threadIdx.x; i < a.M;
             i += (int64_t)(gridDim.x - off) * blockDim.x) {
            const int64_t e00 = rp[i];
            const int64_t e0 = e00 + s0p[i], e1 = e00 + s1p[i];
            cplx acc = mk(0.0, 0.0), acct = mk(0.0, 0.0);
            if (MODE != 0) {
                acc = a.q[i];
                if (NRHS == 2) acct = a.qt[i];
            }
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
                    x[u] = c[u] >= 0 ? r[c[u]] : mk(0, 0);
                    if (NRHS == 2) xt[u] = c[u] >= 0 ? t[c[u]] : mk(0, 0);
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
            if (NRHS == 2) a.qt[i] = acct;
            if (MODE == 2) w = NRHS == 2 ? cfma_conj(t[i], acc, w) : cfma(r[i], acc, w);
        }
    }
    if (MODE == 2) spmv_exit(a, kp, agent, w, sc);
}

// Per-row split points of the column blocks (see KParams::csr_split) and what decides whether
// blocking applies: stats[0] |= 1 when a row is longer than 255 entries or not sorted by column;
// stats[1] += entries whose column is at least half a block away from the row (the far gathers).
__global__ void csr_split_kernel(int64_t M, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                                 int nblk, int bshift, uint8_t *split, unsigned long long *stats) {
    unsigned long long far = 0;
    bool bad = false;
    const int64_t half = (int64_t(1) << bshift) >> 1;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e0 = rp[i], e1 = rp[i + 1];
        if (e1 - e0 > 255) { bad = true; continue; }
        int bnext = 0, prev = -1;   // split[b][i] for b < bnext is written
        for (int64_t e = e0; e < e1; ++e) {
            const int c = col[e];
            bad |= c < prev;
            prev = c;
            const int cb = c >> bshift;
            for (; bnext <= cb && bnext <= nblk; ++bnext) split[(int64_t)bnext * M + i] = (uint8_t)(e - e0);
            const int64_t d = c > i ? c - i : i - c;
            far += d >= half;
        }
        for (; bnext <= nblk; ++bnext) split[(int64_t)bnext * M + i] = (uint8_t)(e1 - e0);
    }
    if (bad) atomicOr(stats, 1ull);
    if (far) atomicAdd(stats + 1, far);
}

cudaError_t launch_csr_split(int64_t M, const int64_t *rp, const int32_t *col, int nblk, int bshift,
                             uint8_t *split, unsigned long long *stats, cudaStream_t s) {
    csr_split_kernel<<<8 * sm_count(), kThreads, 0, s>>>(M, rp, col, nblk, bshift, split, stats);
    return cudaGetLastError();
}

// Column blocks of 2^bshift rows (SHIFTK_CSR_BSHIFT; default 22 = 64 MiB of r per block, half of
// L2).  SHIFTK_CSR_BLOCKED=1 enables blocking wherever the rows qualify (default: one pass).
int csr_block_shift() {
    static int b = -1;
    if (b < 0) {
        const char *e = getenv("SHIFTK_CSR_BSHIFT");
        b = e ? atoi(e) : 22;
        if (b < 4) b = 4;
        if (b > 30) b = 30;
    }
    return b;
}
int csr_blocked_env() {
    static int m = -2;
    if (m == -2) {
        const char *e = getenv("SHIFTK_CSR_BLOCKED");
        m = !e ? -1 : (e[0] == '0' ? 0 : 1);
    }
    return m;
}

template <bool CV, int NRHS>
static cudaError_t launch_csr_blocked_t(const SpmvArgs &a, const KParams &kp, const int64_t *rp, const int32_t *col,
                                        const void *val, cudaStream_t s) {
    const int g = csr_blocks(a.M);
    cudaError_t e = launch_k(csr_block_kernel<CV, NRHS, 0>, g, kThreads, 0, s, true, a, kp, rp, col, val, 0);
    for (int b = 1; e == cudaSuccess && b + 1 < kp.csr_nblk; ++b)
        e = launch_k(csr_block_kernel<CV, NRHS, 1>, g, kThreads, 0, s, true, a, kp, rp, col, val, b);
    if (e == cudaSuccess)
        e = launch_k(csr_block_kernel<CV, NRHS, 2>, g + 1, kThreads, 0, s, true, a, kp, rp, col, val, kp.csr_nblk - 1);
    return e;
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
    if (kp.csr_nblk >= 2 && a.st && kp.world <= 1) {   // solver mode, column-blocked passes
        if (cv) return a.bicg ? launch_csr_blocked_t<true, 2>(a, kp, rp, col, val, s)
                              : launch_csr_blocked_t<true, 1>(a, kp, rp, col, val, s);
        return a.bicg ? launch_csr_blocked_t<false, 2>(a, kp, rp, col, val, s)
                      : launch_csr_blocked_t<false, 1>(a, kp, rp, col, val, s);
    }
    if (csr_mode() == 1) {
        if (cv) {
            const bool p = a.st != nullptr;
            if (kp.world > 1) {
                if (a.bicg) return launch_k(csr_row_kernel<true, 2, true>, grid, kThreads, 0, s, p, a, kp, rp, col, val);
                return launch_k(csr_row_kernel<true, 1, true>, grid, kThreads, 0, s, p, a, kp, rp, col, val);
            }
            if (a.bicg) return launch_k(csr_row_kernel<true, 2, false>, grid, kThreads, 0, s, p, a, kp, rp, col, val);
            return launch_k(csr_row_kernel<true, 1, false>, grid, kThreads, 0, s, p, a, kp, rp, col, val);
        } else {
            const bool p = a.st != nullptr;
            if (kp.world > 1) {
                if (a.bicg) return launch_k(csr_row_kernel<false, 2, true>, grid, kThreads, 0, s, p, a, kp, rp, col, val);
                return launch_k(csr_row_kernel<false, 1, true>, grid, kThreads, 0, s, p, a, kp, rp, col, val);
            }
            if (a.bicg) return launch_k(csr_row_kernel<false, 2, false>, grid, kThreads, 0, s, p, a, kp, rp, col, val);
            return launch_k(csr_row_kernel<false, 1, false>, grid, kThreads, 0, s, p, a, kp, rp, col, val);
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
