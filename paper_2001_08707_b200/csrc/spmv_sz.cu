// spmv_sz.cu — the Heisenberg chain restricted to a sector of fixed S^z.
// H conserves the number n of up spins, so it is block diagonal over sectors; HPhi runs the
// 2Sz = 0 sector (dimension C(L, L/2): 924 at L=12).  Sector basis
// (R28): the L-bit states with popcount n in ascending integer order, row i = the
// i-th one.  rank(s) = sum over the set bits of s, taken in ascending position p_1 < p_2 < ...,
// of C(p_m, m) (the states below s, counted by their highest differing bit).
//
// Two kernels: the block-structured heisenberg_szb_kernel (default, described above it) and the
// earlier rank-stepping heisenberg_sz_kernel (SHIFTK_SZ_RANK=1, kept for comparison), which runs
// one thread per sector row, consecutive rows on consecutive lanes:
//  * unranking — lane 0 of a warp unranks the warp's first row bit by bit from the top; the
//    other lanes step from it inside the block of states that share the bits >= 12: there the
//    12 low bits run through the 12-bit patterns with a fixed popcount in ascending order, a
//    shared-memory table (lo_list; lo_idx gives a pattern's position).  Only lanes whose row
//    leaves that block (a few per cent) unrank themselves.
//  * bonds — the diagonal is J/4 (L - 2 popc(s XOR rot s)); for every anti-aligned open bond
//    (j, j+1) the partner's row follows from the row's own rank: moving the m-th set bit between
//    j and j+1 changes one term, C(j, m) <-> C(j+1, m), i.e. the rank by +-C(j, m-1).  Only the
//    periodic bond (L-1, 0) renumbers the set bits: its partner is ranked from the low-bit table
//    plus the high set bits.
//  * 32-bit state arithmetic for L <= 31 (popc/ffs/shifts are single instructions).
// The gathers r[partner] are the remaining cost: a low bond's partner is a neighbouring row
// (coalesced over the warp), a high bond's C(j, m-1) rows away (still consecutive across the
// warp, since the warp's states share their high bits).
#include <cstdlib>
#include <mutex>

#include "kernels.cuh"
#include "spmv_common.cuh"

namespace sk {

constexpr int kSzMaxL = 34;
constexpr int kSzLoBits = 12;
constexpr int kSzLo = 1 << kSzLoBits;
#ifndef SZB_MINB
#define SZB_MINB 4
#endif
#ifndef SZB_HB
#define SZB_HB 4
#endif
#ifndef SZB_BATCH
#define SZB_BATCH 7
#endif
constexpr int kSzBatch = 8;   // partner gathers in flight per thread

// host-built tables, copied into every CTA's shared memory
struct __align__(16) SzTables {
    unsigned long long C[kSzMaxL + 1][kSzMaxL + 1];   // binomials, zero for k > n
    uint16_t lo_list[kSzLo];   // 12-bit patterns sorted by (popcount, value)
    uint16_t lo_idx[kSzLo];    // position of a pattern within its popcount class
    int32_t lo_off[kSzLoBits + 2];   // start of each popcount class in lo_list
};
__device__ SzTables g_sz_tab;

template <typename U>
static __device__ __forceinline__ int popcU(U v) {
    return sizeof(U) == 4 ? __popc((unsigned)v) : __popcll((unsigned long long)v);
}
template <typename U>
static __device__ __forceinline__ int ffsU(U v) {
    return sizeof(U) == 4 ? __ffs((int)v) - 1 : __ffsll((long long)v) - 1;
}

template <int NRHS, typename U>
__global__ void __launch_bounds__(kThreads) heisenberg_sz_kernel(SpmvArgs a, KParams kp, int L, int nup, double J) {
    __shared__ StepScratch sc;
    __shared__ SzTables tab;
    bool agent;
    int buf;
    if (!spmv_enter(a, agent, buf, sc, kp)) return;
    const cplx *__restrict__ r = pick3(a.r, buf);
    const cplx *__restrict__ t = pick3(a.t, buf);
    const double qJ = 0.25 * J, hJ = 0.5 * J;
    const int64_t M = a.M;
    const int off = a.st ? 1 : 0;
    const int lane = threadIdx.x & 31;
    cplx w = mk(0.0, 0.0);
    if (!agent) {
        {   // tables -> shared memory
            const uint4 *src = (const uint4 *)&g_sz_tab;
            uint4 *dst = (uint4 *)&tab;
            for (int e = threadIdx.x; e < (int)(sizeof(SzTables) / 16); e += blockDim.x) dst[e] = src[e];
        }
        __syncthreads();
        auto unrank = [&](uint64_t rank) -> U {
            U s = 0;
            int m = nup;
            for (int p = L - 1; p >= 0 && m > 0; --p) {
                const uint64_t below = tab.C[p][m];
                if (rank >= below) {
                    s |= (U)1 << p;
                    rank -= below;
                    --m;
                }
            }
            return s;
        };
        const int64_t stride = (int64_t)(gridDim.x - off) * blockDim.x;
        for (int64_t i0 = (int64_t)(blockIdx.x - off) * blockDim.x + (threadIdx.x & ~31); i0 < M; i0 += stride) {
            const int64_t i = i0 + lane;   // this lane's row (the warp's rows are i0 .. i0 + 31)
            // warp-cooperative unranking
            U s0 = 0;
            if (lane == 0) s0 = unrank((uint64_t)i0);
            s0 = (U)__shfl_sync(0xffffffffu, (unsigned long long)s0, 0);
            const U hi0 = s0 >> kSzLoBits;
            const int c = nup - popcU<U>(hi0);
            const int idx = (int)tab.lo_idx[s0 & (kSzLo - 1)] + lane;
            if (i >= M) continue;
            U s;
            if (c >= 0 && c <= kSzLoBits && idx < (int)tab.C[kSzLoBits][c])
                s = (hi0 << kSzLoBits) | (U)tab.lo_list[tab.lo_off[c] + idx];
            else
                s = unrank((uint64_t)i);
            const U x = s ^ ((s >> 1) | ((s & (U)1) << (L - 1)));
            const double d = qJ * (double)(L - 2 * popcU<U>(x));
            const cplx rs = r[i];
            cplx q = mk(d * rs.x, d * rs.y);
            cplx ts = mk(0, 0), qt = mk(0, 0);
            if (NRHS == 2) { ts = t[i]; qt = mk(d * ts.x, d * ts.y); }
            // open bonds (j, j+1), j < L-1: this lane's active ones in batches of kSzBatch, all
            // of a batch's gathers in flight at once (a data-dependent loop over single bonds
            // would leave one gather in flight per thread)
            U xb = x & (((U)1 << (L - 1)) - (U)1);
            while (xb) {
                int64_t pr[kSzBatch];
                bool on[kSzBatch];
#pragma unroll
                for (int u = 0; u < kSzBatch; ++u) {
                    on[u] = xb != 0;
                    pr[u] = i;
                    if (on[u]) {
                        const int j = ffsU<U>(xb);
                        xb &= xb - (U)1;
                        const int m = popcU<U>(s & (((U)2 << (j + 1)) - (U)1));   // index of the moving bit
                        const int64_t delta = (int64_t)tab.C[j][m - 1];
                        pr[u] = ((s >> j) & (U)1) ? i + delta : i - delta;
                    }
                }
                cplx v[kSzBatch], vt[kSzBatch];
#pragma unroll
                for (int u = 0; u < kSzBatch; ++u) {
                    v[u] = on[u] ? r[pr[u]] : mk(0.0, 0.0);
                    if (NRHS == 2) vt[u] = on[u] ? t[pr[u]] : mk(0.0, 0.0);
                }
#pragma unroll
                for (int u = 0; u < kSzBatch; ++u) {
                    if (!on[u]) continue;
                    q.x = fma(hJ, v[u].x, q.x);
                    q.y = fma(hJ, v[u].y, q.y);
                    if (NRHS == 2) {
                        qt.x = fma(hJ, vt[u].x, qt.x);
                        qt.y = fma(hJ, vt[u].y, qt.y);
                    }
                }
            }
            if ((x >> (L - 1)) & (U)1) {   // periodic bond (L-1, 0): rank the partner afresh
                const U s2 = s ^ ((U)1 | ((U)1 << (L - 1)));
                const U lo = s2 & (U)(kSzLo - 1);
                int64_t pr = (int64_t)tab.lo_idx[lo];   // sum over the low set bits
                U h = s2 >> kSzLoBits;
                for (int m = popcU<U>(lo) + 1; h; ++m) {
                    const int p = ffsU<U>(h);
                    h &= h - (U)1;
                    pr += (int64_t)tab.C[p + kSzLoBits][m];
                }
                const cplx v = r[pr];
                q.x = fma(hJ, v.x, q.x);
                q.y = fma(hJ, v.y, q.y);
                if (NRHS == 2) {
                    const cplx vt = t[pr];
                    qt.x = fma(hJ, vt.x, qt.x);
                    qt.y = fma(hJ, vt.y, qt.y);
                }
            }
            a.q[i] = q;
            if (NRHS == 2) {
                a.qt[i] = qt;
                w = cfma_conj(ts, q, w);
            } else {
                w = cfma(rs, q, w);
            }
        }
    }
    spmv_exit(a, kp, agent, w, sc);
}

// Block-structured variant (the default from L = 2).  Split a state s into its high part H
// (bits kb .. L-1, kb = min(12, L-1)) and its low pattern lo (bits 0 .. kb-1, popcount
// c = n - popc(H)).  In the ascending sector order the states sharing H are consecutive rows,
// the block off(H) .. off(H) + C(kb, c) - 1, and row(H, lo) = off(H) + lo_idx[lo] with
// off(H) = sum over H's set bits p (the (c+1)-th, (c+2)-th ... set bit of s) of C(p, m) — the low
// terms of the rank are exactly lo_idx[lo] (the combinatorial number system, R28).  One warp per
// block, everything that depends on H is warp-uniform and computed once per block:
//  * high bonds (j, j+1), kb <= j <= L-2: the partner has the same lo, its block is a fixed
//    +-C(j, m-1) rows away — a coalesced read at a per-block offset (no per-row index work);
//  * the boundary bond (kb-1, kb) and the periodic bond (L-1, 0) move one bit between the parts:
//    the partner's block H' is uniform, its index lo_idx[lo'] per lane;
//  * low bonds (j, j+1), j <= kb-2: the partner is in the same block (<= 924 rows, L1-resident).
// Blocks are dealt to warps in ascending order over one resident wave (sz_blocks), so at any
// time the warps sweep a window of ~4700 consecutive blocks and a partner block within a few
// thousand blocks is read from L2 (measured at L = 30: one CTA per block, or a second wave,
// read more from DRAM and ran 1.4-1.9x slower).
// No per-row unranking; ~4x fewer instructions per row than the rank-stepping kernel above.
// Measured (sk_apply_operator, n = L/2): L = 26 583 -> 358 us, L = 30 9.84 -> 5.76 ms.
template <int NRHS>
__global__ void __launch_bounds__(kThreads, NRHS == 2 ? SZB_MINB - 1 : SZB_MINB) heisenberg_szb_kernel(SpmvArgs a, KParams kp, int L, int nup, double J, int fl) {
    __shared__ StepScratch sc;
    __shared__ SzTables tab;
    __shared__ long long dl[kThreads / 32][kSzMaxL];   // per-warp high-bond row offsets
    __shared__ long long bo[kThreads / 32][3];          // per-warp block bases o, oB, oP
    bool agent;
    int buf;
    if (!spmv_enter(a, agent, buf, sc, kp)) return;
    const cplx *__restrict__ r = pick3(a.r, buf);
    const cplx *__restrict__ t = pick3(a.t, buf);
    const double qJ = 0.25 * J, hJ = 0.5 * J;
    const int off = a.st ? 1 : 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (!agent) {
        {   // tables -> shared memory
            const uint4 *src = (const uint4 *)&g_sz_tab;
            uint4 *dst = (uint4 *)&tab;
            for (int e = threadIdx.x; e < (int)(sizeof(SzTables) / 16); e += blockDim.x) dst[e] = src[e];
        }
        __syncthreads();
        const int kb = L - 1 < kSzLoBits ? L - 1 : kSzLoBits;
        const int nh = L - kb;
        long long *dw = dl[warp];
        // off(H) for the block of H with low class c
        auto off_hi = [&](uint32_t H, int c) -> int64_t {
            int64_t o = 0;
            for (int m = c + 1; H; ++m) {
                const int p = __ffs((int)H) - 1;
                H &= H - 1u;
                o += (int64_t)tab.C[p + kb][m];
            }
            return o;
        };
        const int64_t nH = int64_t(1) << nh;
        // hint (vectors beyond L2): q is written streaming (evict-first); evict-first loads of
        // the far partners were measured to make no difference (5.93 vs 5.95 ms at L = 30)
        const bool hint = fl & 2;
        // blocks are dealt in ascending order from a queue (a.work[0]), so all warps stay within
        // a narrow window of the sweep; a static deal lets warps drift apart by several thousand
        // blocks (random block sizes), and partners then miss L2 (measured at L = 30: 24.7 ->
        // 14.6 GB of DRAM reads, 5.8 -> 4.4 ms).  w is summed per block (fixed order, whichever
        // warp runs it) and per group of kStreamGroup blocks, as in the streaming Heisenberg SpMV.
        cplx *const pw = (a.part_w && a.st && kp.defer) ? a.part_w + (a.st->seq & 1) * kp.wred_stride : a.part_w;
        auto grab = [&]() -> int64_t {
            unsigned long long v = 0;
            if (lane == 0) v = atomicAdd(a.work, 1ull);
            return (int64_t)__shfl_sync(0xffffffffu, v, 0);
        };
        for (int64_t hw = grab(); hw < nH; hw = grab()) {
            const uint32_t H = (uint32_t)hw;
            const int c = nup - __popc(H);
            cplx wb = mk(0.0, 0.0);
            if (c >= 0 && c <= kb) {
            const int cnt = (int)tab.C[kb][c];
            const int64_t o = off_hi(H, c);
            // high bonds: bit b of xh <-> bond (kb + b, kb + b + 1)
            const uint32_t xh = (H ^ (H >> 1)) & ((1u << (nh - 1)) - 1u);
            int nb = 0;
            __syncwarp();   // the previous block's reads of dw are done
            for (uint32_t xx = xh; xx; xx &= xx - 1u, ++nb) {
                const int b = __ffs((int)xx) - 1;
                const int m = c + __popc(H & ((2u << (b + 1)) - 1u));   // index of the moving bit
                const long long d = (long long)tab.C[kb + b][m - 1];
                if (lane == 0) dw[nb] = ((H >> b) & 1u) ? d : -d;
            }
            __syncwarp();
            // boundary bond (kb-1, kb) and periodic bond (L-1, 0): uniform partner blocks
            const uint32_t hb = H & 1u, ht = (H >> (nh - 1)) & 1u;
            const int cB = hb ? c + 1 : c - 1, cP = ht ? c + 1 : c - 1;
            const int64_t oB = (cB >= 0 && cB <= kb) ? off_hi(H ^ 1u, cB) : 0;
            const int64_t oP = (cP >= 0 && cP <= kb) ? off_hi(H ^ (1u << (nh - 1)), cP) : 0;
            const int nhb = __popc(xh);
            // the block bases are re-read from shared memory per row (volatile): keeping them
            // in registers across the row loop costs more than the loads (3.91 -> 3.77 ms, L=30)
            if (lane == 0) { bo[warp][0] = o; bo[warp][1] = oB; bo[warp][2] = oP; }
            __syncwarp();
            volatile long long *vb = bo[warp];
            for (int i0 = 0; i0 < cnt; i0 += 32) {
                const int idx = i0 + lane;
                if (idx >= cnt) break;
                const uint32_t lo = tab.lo_list[tab.lo_off[c] + idx];
                const int64_t i = vb[0] + idx;
                const uint32_t xl = (lo ^ (lo >> 1)) & ((1u << (kb - 1)) - 1u);
                const bool onB = ((lo >> (kb - 1)) & 1u) != hb, onP = (lo & 1u) != ht;
                const double d = qJ * (double)(L - 2 * (__popc(xl) + nhb + (int)onB + (int)onP));
                const cplx rs = r[i];
                cplx q = mk(d * rs.x, d * rs.y);
                cplx ts = mk(0, 0), qt = mk(0, 0);
                if (NRHS == 2) { ts = t[i]; qt = mk(d * ts.x, d * ts.y); }
                // high bonds, SZB_HB coalesced reads in flight
                const cplx *ri = r + i, *ti = t + i;
                for (int u0 = 0; u0 < nb; u0 += SZB_HB) {
                    cplx v[SZB_HB], vt[SZB_HB];
#pragma unroll
                    for (int u = 0; u < SZB_HB; ++u) {
                        const bool on = u0 + u < nb;
                        const long long dd = on ? dw[u0 + u] : 0;
                        v[u] = on ? ri[dd] : mk(0.0, 0.0);
                        if (NRHS == 2) vt[u] = on ? ti[dd] : mk(0.0, 0.0);
                    }
#pragma unroll
                    for (int u = 0; u < SZB_HB; ++u) {
                        q.x = fma(hJ, v[u].x, q.x);
                        q.y = fma(hJ, v[u].y, q.y);
                        if (NRHS == 2) {
                            qt.x = fma(hJ, vt[u].x, qt.x);
                            qt.y = fma(hJ, vt[u].y, qt.y);
                        }
                    }
                }
                // low bonds, boundary and periodic bond: the partner is the lo_idx-th row of a
                // block with a uniform base (own block, H ^ 1, H ^ top bit), two batches in flight
                const cplx *rb[3] = {r + vb[0], r + vb[1], r + vb[2]}, *tb[3] = {t + vb[0], t + vb[1], t + vb[2]};
                const uint32_t onm = xl | ((uint32_t)onB << (kSzLoBits - 1)) | ((uint32_t)onP << kSzLoBits);
                constexpr int kHalf = SZB_BATCH;
#pragma unroll
                for (int j0 = 0; j0 <= kSzLoBits; j0 += kHalf) {
                    cplx v[kHalf], vt[kHalf];
#pragma unroll
                    for (int u = 0; u < kHalf; ++u) {
                        const int j = j0 + u;
                        if (j > kSzLoBits) break;
                        const int sel = j < kSzLoBits - 1 ? 0 : j - (kSzLoBits - 2);
                        const bool on = (onm >> j) & 1u;
                        const uint32_t flip = j < kSzLoBits - 1 ? 3u << j : (j == kSzLoBits - 1 ? 1u << (kb - 1) : 1u);
                        const uint32_t pj = tab.lo_idx[(lo ^ flip) & (kSzLo - 1)];
                        v[u] = on ? rb[sel][pj] : mk(0.0, 0.0);
                        if (NRHS == 2) vt[u] = on ? tb[sel][pj] : mk(0.0, 0.0);
                    }
#pragma unroll
                    for (int u = 0; u < kHalf; ++u) {
                        if (j0 + u > kSzLoBits) break;
                        q.x = fma(hJ, v[u].x, q.x);
                        q.y = fma(hJ, v[u].y, q.y);
                        if (NRHS == 2) {
                            qt.x = fma(hJ, vt[u].x, qt.x);
                            qt.y = fma(hJ, vt[u].y, qt.y);
                        }
                    }
                }
                if (hint) __stcs(a.q + i, q); else a.q[i] = q;
                if (NRHS == 2) {
                    a.qt[i] = qt;
                    wb = cfma_conj(ts, q, wb);
                } else {
                    wb = cfma(rs, q, wb);
                }
            }
            }
            if (pw) {   // this block's partial of w; the last block of a group sums the group
                wb = warp_sum(wb);
                bool reduce_group = false;
                if (lane == 0) {
                    pw[hw] = wb;
                    if (nH > kStreamDirect) {
                        const int64_t g = hw / kStreamGroup, g0 = g * kStreamGroup;
                        const uint32_t gn = (uint32_t)((nH - g0) < kStreamGroup ? (nH - g0) : kStreamGroup);
                        __threadfence();
                        reduce_group = atomicAdd(a.grp + g, 1u) == gn - 1u;
                    }
                }
                reduce_group = __shfl_sync(0xffffffffu, reduce_group, 0);
                if (reduce_group) {
                    __threadfence();
                    const int64_t g = hw / kStreamGroup, g0 = g * kStreamGroup;
                    const int64_t g1 = (g0 + kStreamGroup) < nH ? g0 + kStreamGroup : nH;
                    cplx v = mk(0.0, 0.0);
                    for (int64_t j = g0 + lane; j < g1; j += 32) v = cadd(v, ldcg(pw + j));
                    v = warp_sum(v);
                    if (lane == 0) {
                        pw[nH + g] = v;
                        a.grp[g] = 0u;
                    }
                }
            }
        }
        // queue bookkeeping: the last worker CTA rewinds the queue for the next launch
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(a.work + 1, 1ull) == (unsigned long long)(gridDim.x - off) - 1ull) {
                a.work[0] = 0ull;
                a.work[1] = 0ull;
            }
        }
    }
    const int64_t nH = int64_t(1) << (L - (L - 1 < kSzLoBits ? L - 1 : kSzLoBits));
    cplx *const pw = (a.part_w && a.st && kp.defer) ? a.part_w + (a.st->seq & 1) * kp.wred_stride : a.part_w;
    spmv_exit(a, kp, agent, mk(0.0, 0.0), sc, nH <= kStreamDirect ? pw : pw + nH,
              (int)(nH <= kStreamDirect ? nH : stream_partials(nH) - nH));
}


// g_sz_tab is a __device__ symbol: one copy per device, so it is written on every device a
// sector operator runs on (once each).
static cudaError_t sz_tables_init() {
    static PerDevice once;
    return once_per_device(once, [] {
        static SzTables h;
        for (int n = 0; n <= kSzMaxL; ++n)
            for (int k = 0; k <= kSzMaxL; ++k)
                h.C[n][k] = k > n ? 0ull : (k == 0 || k == n ? 1ull : h.C[n - 1][k - 1] + h.C[n - 1][k]);
        int pos = 0;
        for (int c = 0; c <= kSzLoBits; ++c) {
            h.lo_off[c] = pos;
            int within = 0;
            for (int v = 0; v < kSzLo; ++v)
                if (__builtin_popcount((unsigned)v) == c) {
                    h.lo_list[pos++] = (uint16_t)v;
                    h.lo_idx[v] = (uint16_t)within++;
                }
        }
        h.lo_off[kSzLoBits + 1] = pos;
        return cudaMemcpyToSymbol(g_sz_tab, &h, sizeof(h));
    });
}

// SHIFTK_SZ_RANK=1 selects the rank-stepping kernel (kept for comparison)
static bool sz_rank_kernel() {
    static int en = -1;
    if (en < 0) {
        const char *e = getenv("SHIFTK_SZ_RANK");
        en = (e && e[0] == '1') ? 1 : 0;
    }
    return en == 1;
}

int64_t sz_partials(int L) {   // w partials of the block kernel (0: per-CTA partials)
    if (L < 2 || sz_rank_kernel()) return 0;
    return stream_partials(int64_t(1) << (L - (L - 1 < kSzLoBits ? L - 1 : kSzLoBits)));
}

// One resident wave (SZB_MINB CTAs per SM, one slot for the finish agent): the warps sweep the
// blocks H once in ascending order; a second wave would start a second sweep over the partners.
int sz_blocks(int L, int64_t M, int bicg) {
    const int b = stream_blocks(M);
    if (L < 2 || sz_rank_kernel()) return b;
    const int cap = (bicg ? SZB_MINB - 1 : SZB_MINB) * sm_count() - 1;
    return b < cap ? b : cap;
}

cudaError_t launch_heisenberg_sz(const SpmvArgs &a, const KParams &kp, int L, int nup, double J, cudaStream_t s) {
    const cudaError_t e = sz_tables_init();
    if (e != cudaSuccess) return e;
    const int grid = sz_blocks(L, a.M, a.bicg) + (a.st ? 1 : 0);
    const bool p = a.st != nullptr;
    if (L >= 2 && !sz_rank_kernel()) {
        const int fl = a.M * (int64_t)sizeof(cplx) >= (int64_t(64) << 20) ? 2 : 0;
        if (a.bicg) return launch_k(heisenberg_szb_kernel<2>, grid, kThreads, 0, s, p, a, kp, L, nup, J, fl);
        return launch_k(heisenberg_szb_kernel<1>, grid, kThreads, 0, s, p, a, kp, L, nup, J, fl);
    }
    if (L <= 31) {
        if (a.bicg) return launch_k(heisenberg_sz_kernel<2, uint32_t>, grid, kThreads, 0, s, p, a, kp, L, nup, J);
        return launch_k(heisenberg_sz_kernel<1, uint32_t>, grid, kThreads, 0, s, p, a, kp, L, nup, J);
    }
    if (a.bicg) return launch_k(heisenberg_sz_kernel<2, uint64_t>, grid, kThreads, 0, s, p, a, kp, L, nup, J);
    return launch_k(heisenberg_sz_kernel<1, uint64_t>, grid, kThreads, 0, s, p, a, kp, L, nup, J);
}

}  // namespace sk
