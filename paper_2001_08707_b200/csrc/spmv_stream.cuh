// spmv_stream.cuh — the Heisenberg SpMV q = H r (COCG, one right-hand side) as a TMA-fed
// streaming kernel.  Same decomposition as the tiled kernel (spmv_tiled.cuh): a tile is 2^T
// consecutive basis states; the T-1 bonds inside a tile read the tile itself, the bond (T-1, T)
// reads half of the tile that differs in bit T, the periodic bond (L-1, 0) the tile that differs
// in bit L-1, and each ACTIVE tile-level bond i >= T (sites i, i+1 anti-aligned in the tile
// index — uniform over the tile) the tile that differs in bits i and i+1 (P:L831 H, P:L508 bit
// flips).  What changes is how the data moves:
//   * one producer thread per CTA streams the tile and its partner tiles into shared memory
//     with cp.async.bulk (global -> shared, mbarrier completion): a double-buffered own-tile
//     slot and a ring of NS partner slots, so ~100 KB per CTA is in flight and the consumer
//     warps never wait on an L2 round trip per element;
//   * the tiles come from a dynamic queue (one 64-bit atomic per tile), so the CTAs, two per
//     SM, stay busy until the last tile and concurrently processed tiles are adjacent in index
//     (their partners across low tile bits are L2 hits);
//   * 8 consumer warps accumulate q in registers (4 states per thread), then the internal bonds
//     from the staged own tile, store q and the partial w = <r, q> (unconjugated, App. A).
// Multi-rank (MULTI): the partner tile's address comes from the shard table — a bulk copy
// straight from the owning rank's buffer (peer memory), fused into the same pipeline.
#pragma once
#include "async_copy.cuh"
#include "spmv_common.cuh"

namespace sk {

constexpr int kStreamConsumers = 256;            // 8 consumer warps
constexpr int kStreamThreads = kStreamConsumers + 32;   // + 1 producer warp
constexpr int kStreamSlots = 4;                  // partner ring depth (tiles)

// active tile-level bonds T..L-2 of the tile with global first state `base` (bit j = bond j+T)
template <int L, int T, typename U>
static __device__ __forceinline__ U tile_bonds(U base) {
    if (L - 1 <= T) return (U)0;
    const U tbits = base >> T;
    return (tbits ^ (tbits >> 1)) & ((((U)1) << (L - 1 - T)) - (U)1);
}

// SPLIT (one GPU, COCG, projection mode): this kernel applies only H_A — the
// diagonal and the bonds (i, i+1) with i < kp.split_ahi (the arc kept local by the tile + the L2
// window) — and leaves H_B (bonds i >= split_ahi and the periodic bond) to the update kernel,
// which applies it from shared memory in its own row order (update_split.cu).
template <int L, int T, bool MULTI, bool SPLIT = false>
__global__ void __launch_bounds__(kStreamThreads, 2)
heisenberg_stream_kernel(SpmvArgs a, KParams kp, double J) {
    constexpr int TS = 1 << T;
    constexpr int NS = kStreamSlots;
    constexpr int PER = TS / kStreamConsumers;
    static_assert(PER * kStreamConsumers == TS, "tile must be a multiple of the consumer count");
    using U = typename std::conditional<(L <= 31), uint32_t, uint64_t>::type;
    extern __shared__ __align__(128) unsigned char dsm[];
    cplx *own = (cplx *)dsm;                       // [2][TS]
    cplx *ring = own + 2 * TS;                     // [NS][TS]
    __shared__ StepScratch sc;
    __shared__ uint64_t own_full[2], own_empty[2], ring_full[NS], ring_empty[NS];
    __shared__ int64_t tile_of[2];
    __shared__ cplx wsm[2][kStreamConsumers / 32];
    bool agent;
    int buf;
    if (!spmv_enter(a, agent, buf, sc, kp)) return;
    const cplx *__restrict__ r = pick3(a.r, buf);
    const RViewT<MULTI> rv = rview<MULTI>(r, kp.shard_r, buf, kp);
    const int tid = threadIdx.x;
    const int64_t ntiles = a.M >> T;
    const U row0 = (U)(MULTI ? rv.row0 : 0);
    cplx *const pw = (a.part_w && a.st && kp.defer) ? a.part_w + (a.st->seq & 1) * kp.wred_stride : a.part_w;
    // tile-level bonds applied here: all, or (SPLIT) those with i < split_ahi (bit j = bond j + T)
    const U amask = SPLIT ? (U)((((U)1) << (kp.split_ahi - T)) - (U)1) : ~(U)0;
    cplx w = mk(0.0, 0.0);
    if (!agent) {
        if (tid == 0) {
            for (int i = 0; i < 2; ++i) { mb_init(&own_full[i], 1); mb_init(&own_empty[i], kStreamConsumers / 32); }
            for (int i = 0; i < NS; ++i) { mb_init(&ring_full[i], 1); mb_init(&ring_empty[i], kStreamConsumers / 32); }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();   // barriers initialised before anyone waits on them
        if (tid >= kStreamConsumers) {
            // ------------------------------------------------------------ producer lanes
            // lane 0 takes tiles from the queue and loads the own tile; ring item `it` is issued
            // by lane it % NS (several issuing lanes keep more bulk copies in flight per CTA)
            const int pl = tid - kStreamConsumers;
            if (pl < NS) {
                constexpr unsigned pmask = (1u << NS) - 1u;
                uint32_t it = 0;
                int64_t ti_next = 0;
                if (pl == 0) ti_next = (int64_t)atomicAdd(a.work, 1ull);
                for (uint32_t j = 0;; ++j) {
                    const int k = j & 1;
                    const int64_t ti = __shfl_sync(pmask, ti_next, 0);
                    if (pl == 0) mb_wait(&own_empty[k], ((j >> 1) & 1) ^ 1);
                    if (ti >= ntiles) {
                        if (pl == 0) {
                            tile_of[k] = -1;
                            mb_arrive(&own_full[k]);
                        }
                        break;
                    }
                    const U base = row0 + (U)(ti << T);
                    if (pl == 0) {
                        tile_of[k] = ti;
                        mb_expect(&own_full[k], TS * sizeof(cplx));
                        bulk_load(own + k * TS, rv.at(base), TS * sizeof(cplx), &own_full[k]);
                    }
                    // partner items, in the consumers' order
                    const U tb = (base >> T) & (U)1;
                    U act = tile_bonds<L, T, U>(base) & amask;
                    for (int m = -2;; ++m) {
                        if (SPLIT && m == -1) continue;   // the periodic bond is in H_B
                        const cplx *src;
                        unsigned bytes = TS * sizeof(cplx);
                        if (m == -2) {          // bond (T-1, T): the half with bit T-1 = tb
                            src = rv.at(base ^ ((U)1 << T)) + ((int64_t)tb << (T - 1));
                            bytes = (TS / 2) * sizeof(cplx);
                        } else if (m == -1) {   // periodic bond (L-1, 0)
                            src = rv.at(base ^ ((U)1 << (L - 1)));
                        } else {
                            if (!act) break;
                            const int pos = (L <= 31) ? __ffs((int)act) - 1 : __ffsll((long long)act) - 1;
                            act &= act - (U)1;
                            src = rv.at(base ^ ((U)3 << (pos + T)));
                        }
                        const int s = it % NS;
                        if (s == pl) {
                            mb_wait(&ring_empty[s], ((it / NS) & 1) ^ 1);
                            mb_expect(&ring_full[s], bytes);
                            bulk_load(ring + s * TS, src, bytes, &ring_full[s]);
                        }
                        ++it;
                    }
                    // next tile: claimed once this tile's loads are all issued (the consumers
                    // still have the last NS items to process)
                    if (pl == 0) ti_next = (int64_t)atomicAdd(a.work, 1ull);
                }
            }
        } else {
            // ------------------------------------------------------------ consumers
            const double qJ = 0.25 * J, hJ = 0.5 * J;
            const int lane = tid & 31;
            uint32_t it = 0;
            for (uint32_t j = 0;; ++j) {
                const int k = j & 1;
                mb_wait(&own_full[k], (j >> 1) & 1);
                const int64_t ti = tile_of[k];
                if (ti < 0) break;
                const cplx *ot = own + k * TS;
                const U base = row0 + (U)(ti << T);
                const U tb = (base >> T) & (U)1, hb = (base >> (L - 1)) & (U)1;
                cplx v0[PER], q[PER];
#pragma unroll
                for (int e = 0; e < PER; ++e) {
                    const int ls = tid + e * kStreamConsumers;
                    const U s = base + (U)ls;
                    const U x = s ^ ((s >> 1) | ((s & (U)1) << (L - 1)));
                    const int na = (L <= 31) ? __popc((unsigned)x) : __popcll((unsigned long long)x);
                    const double d = qJ * (double)(L - 2 * na);
                    v0[e] = ot[ls];
                    q[e] = mk(d * v0[e].x, d * v0[e].y);
                }
                U act = tile_bonds<L, T, U>(base) & amask;
                for (int m = -2;; ++m) {
                    if (SPLIT && m == -1) continue;
                    if (m >= 0) {
                        if (!act) break;
                        act &= act - (U)1;
                    }
                    const int s = it % NS;
                    mb_wait(&ring_full[s], (it / NS) & 1);
                    const cplx *pt = ring + s * TS;
#pragma unroll
                    for (int e = 0; e < PER; ++e) {
                        const int ls = tid + e * kStreamConsumers;
                        bool on = true;
                        cplx v;
                        if (m == -2) {
                            on = (((U)((ls >> (T - 1)) & 1)) ^ tb) != 0;
                            v = pt[ls & (TS / 2 - 1)];
                        } else if (m == -1) {
                            on = (((U)(ls & 1)) ^ hb) != 0;
                            v = pt[ls ^ 1];
                        } else {
                            v = pt[ls];
                        }
                        if (on) {
                            q[e].x = fma(hJ, v.x, q[e].x);
                            q[e].y = fma(hJ, v.y, q[e].y);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mb_arrive(&ring_empty[s]);
                    ++it;
                }
                // bonds (i, i+1), i < T-1, inside the tile, split by bit position as in the
                // tiled kernel: bonds 0..6 by the consumer index alone (constant-offset
                // partners), bond 7 by its bit 7 and e bit 0, bond 8 by e alone
                static_assert(T == 10 && kStreamConsumers == 256 && PER == 4, "bit split assumes 1024-state tiles");
                {
                    const unsigned xt = (unsigned)(tid ^ (tid >> 1));
#pragma unroll
                    for (int i = 0; i < 7; ++i) {
                        if ((xt >> i) & 1u) {
                            const int lp = tid ^ (3 << i);
#pragma unroll
                            for (int e = 0; e < PER; ++e) {
                                const cplx v = ot[lp + e * kStreamConsumers];
                                q[e].x = fma(hJ, v.x, q[e].x);
                                q[e].y = fma(hJ, v.y, q[e].y);
                            }
                        }
                    }
                    const int b7 = (tid >> 7) & 1, lp7 = tid ^ 128;
#pragma unroll
                    for (int e = 0; e < PER; ++e) {
                        if (b7 ^ (e & 1)) {   // bond (7, 8)
                            const cplx v = ot[lp7 + (e ^ 1) * kStreamConsumers];
                            q[e].x = fma(hJ, v.x, q[e].x);
                            q[e].y = fma(hJ, v.y, q[e].y);
                        }
                        if ((e ^ (e >> 1)) & 1) {   // bond (8, 9): partner e ^ 3 (own registers)
                            const cplx v = v0[e ^ 3];
                            q[e].x = fma(hJ, v.x, q[e].x);
                            q[e].y = fma(hJ, v.y, q[e].y);
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mb_arrive(&own_empty[k]);
                cplx *qo = a.q + (ti << T);
                cplx wt = mk(0.0, 0.0);
#pragma unroll
                for (int e = 0; e < PER; ++e) {
                    qo[tid + e * kStreamConsumers] = q[e];
                    wt = cfma(v0[e], q[e], wt);
                }
                if (pw) {   // this tile's partial of w, fixed order
                    wt = warp_sum(wt);
                    if (lane == 0) wsm[k][tid >> 5] = wt;
                    asm volatile("bar.sync 1, %0;" ::"n"(kStreamConsumers) : "memory");
                    if (tid < 32) {
                        bool reduce_group = false;
                        if (tid == 0) {
                            cplx v = wsm[k][0];
#pragma unroll
                            for (int m = 1; m < kStreamConsumers / 32; ++m) v = cadd(v, wsm[k][m]);
                            pw[ti] = v;
                            if (ntiles > kStreamDirect) {
                                const int64_t g = ti / kStreamGroup;
                                const int64_t g0 = g * kStreamGroup;
                                const uint32_t gn = (uint32_t)((ntiles - g0) < kStreamGroup ? (ntiles - g0) : kStreamGroup);
                                __threadfence();
                                reduce_group = atomicAdd(a.grp + g, 1u) == gn - 1u;
                            }
                        }
                        reduce_group = __shfl_sync(0xffffffffu, reduce_group, 0);
                        if (reduce_group) {   // sum the group's tile partials (lane-strided, tree)
                            __threadfence();
                            const int64_t g = ti / kStreamGroup, g0 = g * kStreamGroup;
                            const int64_t g1 = (g0 + kStreamGroup) < ntiles ? g0 + kStreamGroup : ntiles;
                            cplx v = mk(0.0, 0.0);
                            for (int64_t i = g0 + lane; i < g1; i += 32) v = cadd(v, ldcg(pw + i));
                            v = warp_sum(v);
                            if (lane == 0) {
                                pw[ntiles + g] = v;
                                a.grp[g] = 0u;
                            }
                        }
                    }
                }
            }
        }
        // queue bookkeeping: the last worker CTA rewinds the tile queue for the next launch
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            if (atomicAdd(a.work + 1, 1ull) == (unsigned long long)(gridDim.x - (a.st ? 1 : 0)) - 1ull) {
                a.work[0] = 0ull;
                a.work[1] = 0ull;
            }
        }
    }
    // the seed CTA reduces the per-tile (or per-group) partials in index order
    const int64_t np = stream_partials(ntiles);
    spmv_exit(a, kp, agent, w, sc, ntiles <= kStreamDirect ? pw : pw + ntiles,
              (int)(ntiles <= kStreamDirect ? ntiles : np - ntiles));
}

// ---------------------------------------------------------------------------- tile pairs
// One GPU, L >= 24: the work unit is the pair of tiles t, t + ntiles/2 that differ in the top
// spin bit — each the other's partner across the periodic bond (L-1, 0), otherwise a tile
// 2^(L-1) states away read from DRAM by every tile (16 B/row).  One own-tile slot holds the pair
// (32 KB) and the ring the partner tiles; the consumers take a tile's ring items BEFORE its own
// tile (the partner sums need nothing of it), so the pair's own tiles are issued when the previous
// pair releases the slot and arrive while the first tile's items are processed.  Producer order
// per unit: unit id -> items of t0 -> (slot free) own tiles -> items of t1; consumer order:
// items of t0 -> own part of t0 (diagonal, periodic from t1, in-tile bonds) -> items of t1 ->
// own part of t1 -> release.  (No deadlock: the own tiles are issued before any t1 item.)
template <int L, int T>
__global__ void __launch_bounds__(kStreamThreads, 2)
heisenberg_pair_kernel(SpmvArgs a, KParams kp, double J) {
    constexpr int TS = 1 << T;
    constexpr int NS = kStreamSlots;
    constexpr int PER = TS / kStreamConsumers;
    static_assert(PER * kStreamConsumers == TS && T == 10, "bit split assumes 1024-state tiles");
    using U = typename std::conditional<(L <= 31), uint32_t, uint64_t>::type;
    extern __shared__ __align__(128) unsigned char dsm[];
    cplx *own = (cplx *)dsm;                       // [2][TS]: the pair
    cplx *ring = own + 2 * TS;                     // [NS][TS]
    __shared__ StepScratch sc;
    __shared__ uint64_t own_full, own_empty, unit_full[2], unit_empty[2], ring_full[NS], ring_empty[NS];
    __shared__ int64_t unit_of[2];
    __shared__ cplx wsm[2][kStreamConsumers / 32];
    bool agent;
    int buf;
    if (!spmv_enter(a, agent, buf, sc, kp)) return;
    const cplx *__restrict__ r = pick3(a.r, buf);
    const int tid = threadIdx.x;
    const int64_t ntiles = a.M >> T, half = ntiles / 2;
    cplx *const pw = (a.part_w && a.st && kp.defer) ? a.part_w + (a.st->seq & 1) * kp.wred_stride : a.part_w;
    cplx w = mk(0.0, 0.0);
    if (!agent) {
        if (tid == 0) {
            mb_init(&own_full, 1);
            mb_init(&own_empty, kStreamConsumers / 32);
            for (int i = 0; i < 2; ++i) { mb_init(&unit_full[i], 1); mb_init(&unit_empty[i], kStreamConsumers / 32); }
            for (int i = 0; i < NS; ++i) { mb_init(&ring_full[i], 1); mb_init(&ring_empty[i], kStreamConsumers / 32); }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (tid >= kStreamConsumers) {
            // ------------------------------------------------------------ producer lanes
            const int pl = tid - kStreamConsumers;
            if (pl < NS) {
                constexpr unsigned pmask = (1u << NS) - 1u;
                uint32_t it = 0;
                int64_t u_next = 0;
                if (pl == 0) u_next = (int64_t)atomicAdd(a.work, 1ull);
                auto issue_items = [&](U base) {   // bond (T-1, T) half, then the active tile bonds
                    const U tb = (base >> T) & (U)1;
                    U act = tile_bonds<L, T, U>(base);
                    for (int m = -1;; ++m) {
                        const cplx *src;
                        unsigned bytes = TS * sizeof(cplx);
                        if (m < 0) {
                            src = r + (int64_t)(base ^ ((U)1 << T)) + ((int64_t)tb << (T - 1));
                            bytes = (TS / 2) * sizeof(cplx);
                        } else {
                            if (!act) break;
                            const int pos = (L <= 31) ? __ffs((int)act) - 1 : __ffsll((long long)act) - 1;
                            act &= act - (U)1;
                            src = r + (int64_t)(base ^ ((U)3 << (pos + T)));
                        }
                        const int s = it % NS;
                        if (s == pl) {
                            mb_wait(&ring_empty[s], ((it / NS) & 1) ^ 1);
                            mb_expect(&ring_full[s], bytes);
                            bulk_load(ring + s * TS, src, bytes, &ring_full[s]);
                        }
                        ++it;
                    }
                };
                for (uint32_t j = 0;; ++j) {
                    const int g = j & 1;
                    const int64_t uid = __shfl_sync(pmask, u_next, 0);
                    if (pl == 0) {
                        mb_wait(&unit_empty[g], ((j >> 1) & 1) ^ 1);
                        unit_of[g] = uid < half ? uid : -1;
                        mb_arrive(&unit_full[g]);
                    }
                    if (uid >= half) break;
                    const U b0 = (U)(uid << T), b1 = (U)((uid + half) << T);
                    issue_items(b0);
                    if (pl == 0) {
                        mb_wait(&own_empty, (j & 1) ^ 1);
                        mb_expect(&own_full, 2 * TS * sizeof(cplx));
                        bulk_load(own, r + (int64_t)b0, TS * sizeof(cplx), &own_full);
                        bulk_load(own + TS, r + (int64_t)b1, TS * sizeof(cplx), &own_full);
                    }
                    issue_items(b1);
                    if (pl == 0) u_next = (int64_t)atomicAdd(a.work, 1ull);
                }
            }
        } else {
            // ------------------------------------------------------------ consumers
            const double qJ = 0.25 * J, hJ = 0.5 * J;
            const int lane = tid & 31;
            uint32_t it = 0, tcount = 0;
            for (uint32_t j = 0;; ++j) {
                const int g = j & 1;
                mb_wait(&unit_full[g], (j >> 1) & 1);
                const int64_t uid = unit_of[g];
                if (uid < 0) break;
                for (int h = 0; h < 2; ++h, ++tcount) {
                    const int64_t ti = uid + h * half;
                    const U base = (U)(ti << T);
                    const U tb = (base >> T) & (U)1, hb = (base >> (L - 1)) & (U)1;
                    cplx q[PER];
#pragma unroll
                    for (int e = 0; e < PER; ++e) q[e] = mk(0.0, 0.0);
                    // partner tiles from the ring (nothing of the own tile needed)
                    U act = tile_bonds<L, T, U>(base);
                    for (int m = -1;; ++m) {
                        if (m >= 0) {
                            if (!act) break;
                            act &= act - (U)1;
                        }
                        const int s = it % NS;
                        mb_wait(&ring_full[s], (it / NS) & 1);
                        const cplx *pt = ring + s * TS;
#pragma unroll
                        for (int e = 0; e < PER; ++e) {
                            const int ls = tid + e * kStreamConsumers;
                            if (m < 0) {
                                if ((((U)((ls >> (T - 1)) & 1)) ^ tb) != 0) {
                                    const cplx v = pt[ls & (TS / 2 - 1)];
                                    q[e].x = fma(hJ, v.x, q[e].x);
                                    q[e].y = fma(hJ, v.y, q[e].y);
                                }
                            } else {
                                const cplx v = pt[ls];
                                q[e].x = fma(hJ, v.x, q[e].x);
                                q[e].y = fma(hJ, v.y, q[e].y);
                            }
                        }
                        __syncwarp();
                        if (lane == 0) mb_arrive(&ring_empty[s]);
                        ++it;
                    }
                    // own part: diagonal, periodic bond from the pair's other tile, in-tile bonds
                    if (h == 0) mb_wait(&own_full, j & 1);
                    const cplx *ot = own + h * TS, *op = own + (1 - h) * TS;
                    cplx v0[PER];
#pragma unroll
                    for (int e = 0; e < PER; ++e) {
                        const int ls = tid + e * kStreamConsumers;
                        const U s = base + (U)ls;
                        const U x = s ^ ((s >> 1) | ((s & (U)1) << (L - 1)));
                        const int na = (L <= 31) ? __popc((unsigned)x) : __popcll((unsigned long long)x);
                        const double d = qJ * (double)(L - 2 * na);
                        v0[e] = ot[ls];
                        q[e].x = fma(d, v0[e].x, q[e].x);
                        q[e].y = fma(d, v0[e].y, q[e].y);
                        if ((((U)(ls & 1)) ^ hb) != 0) {
                            const cplx v = op[ls ^ 1];
                            q[e].x = fma(hJ, v.x, q[e].x);
                            q[e].y = fma(hJ, v.y, q[e].y);
                        }
                    }
                    {
                        const unsigned xt = (unsigned)(tid ^ (tid >> 1));
#pragma unroll
                        for (int i = 0; i < 7; ++i) {
                            if ((xt >> i) & 1u) {
                                const int lp = tid ^ (3 << i);
#pragma unroll
                                for (int e = 0; e < PER; ++e) {
                                    const cplx v = ot[lp + e * kStreamConsumers];
                                    q[e].x = fma(hJ, v.x, q[e].x);
                                    q[e].y = fma(hJ, v.y, q[e].y);
                                }
                            }
                        }
                        const int b7 = (tid >> 7) & 1, lp7 = tid ^ 128;
#pragma unroll
                        for (int e = 0; e < PER; ++e) {
                            if (b7 ^ (e & 1)) {
                                const cplx v = ot[lp7 + (e ^ 1) * kStreamConsumers];
                                q[e].x = fma(hJ, v.x, q[e].x);
                                q[e].y = fma(hJ, v.y, q[e].y);
                            }
                            if ((e ^ (e >> 1)) & 1) {
                                const cplx v = v0[e ^ 3];
                                q[e].x = fma(hJ, v.x, q[e].x);
                                q[e].y = fma(hJ, v.y, q[e].y);
                            }
                        }
                    }
                    if (h == 1) {   // the pair's own tiles and unit id are no longer read
                        __syncwarp();
                        if (lane == 0) {
                            mb_arrive(&own_empty);
                            mb_arrive(&unit_empty[g]);
                        }
                    }
                    cplx *qo = a.q + (ti << T);
                    cplx wt = mk(0.0, 0.0);
#pragma unroll
                    for (int e = 0; e < PER; ++e) {
                        stg_cs(qo + tid + e * kStreamConsumers, q[e]);
                        wt = cfma(v0[e], q[e], wt);
                    }
                    if (pw) {   // this tile's partial of w, fixed order
                        const int wk = tcount & 1;
                        wt = warp_sum(wt);
                        if (lane == 0) wsm[wk][tid >> 5] = wt;
                        asm volatile("bar.sync 1, %0;" ::"n"(kStreamConsumers) : "memory");
                        if (tid < 32) {
                            bool reduce_group = false;
                            if (tid == 0) {
                                cplx v = wsm[wk][0];
#pragma unroll
                                for (int mm = 1; mm < kStreamConsumers / 32; ++mm) v = cadd(v, wsm[wk][mm]);
                                pw[ti] = v;
                                if (ntiles > kStreamDirect) {
                                    const int64_t gg = ti / kStreamGroup, g0 = gg * kStreamGroup;
                                    const uint32_t gn = (uint32_t)((ntiles - g0) < kStreamGroup ? (ntiles - g0) : kStreamGroup);
                                    __threadfence();
                                    reduce_group = atomicAdd(a.grp + gg, 1u) == gn - 1u;
                                }
                            }
                            reduce_group = __shfl_sync(0xffffffffu, reduce_group, 0);
                            if (reduce_group) {
                                __threadfence();
                                const int64_t gg = ti / kStreamGroup, g0 = gg * kStreamGroup;
                                const int64_t g1 = (g0 + kStreamGroup) < ntiles ? g0 + kStreamGroup : ntiles;
                                cplx v = mk(0.0, 0.0);
                                for (int64_t i = g0 + lane; i < g1; i += 32) v = cadd(v, ldcg(pw + i));
                                v = warp_sum(v);
                                if (lane == 0) {
                                    pw[ntiles + gg] = v;
                                    a.grp[gg] = 0u;
                                }
                            }
                        }
                    }
                }
            }
        }
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            if (atomicAdd(a.work + 1, 1ull) == (unsigned long long)(gridDim.x - (a.st ? 1 : 0)) - 1ull) {
                a.work[0] = 0ull;
                a.work[1] = 0ull;
            }
        }
    }
    const int64_t np = stream_partials(ntiles);
    spmv_exit(a, kp, agent, w, sc, ntiles <= kStreamDirect ? pw : pw + ntiles,
              (int)(ntiles <= kStreamDirect ? ntiles : np - ntiles));
}

template <int L>
static cudaError_t launch_stream(const SpmvArgs &a, const KParams &kp, double J, int grid, cudaStream_t s) {
    constexpr int T = kTileBits;
    const size_t shm = (size_t)(2 + kStreamSlots) * sizeof(cplx) << T;
    static PerDevice cfg;
    cudaError_t e = once_per_device(cfg, [&] {
        cudaError_t r = cudaFuncSetAttribute(heisenberg_stream_kernel<L, T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
        if (r == cudaSuccess) r = cudaFuncSetAttribute(heisenberg_stream_kernel<L, T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
        if (r == cudaSuccess) r = cudaFuncSetAttribute(heisenberg_pair_kernel<L, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
        if (r == cudaSuccess) r = cudaFuncSetAttribute(heisenberg_stream_kernel<L, T, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
        return r;
    });
    if (e != cudaSuccess) return e;
    const bool p = a.st != nullptr;
    if (kp.split_ahi > 0 && a.st)   // solver mode with the bond split: H_A only
        return launch_k(heisenberg_stream_kernel<L, T, false, true>, grid, kStreamThreads, shm, s, p, a, kp, J);
    if (kp.world > 1)
        return launch_k(heisenberg_stream_kernel<L, T, true>, grid, kStreamThreads, shm, s, p, a, kp, J);
    if (heis_pairs(L, a.M))
        return launch_k(heisenberg_pair_kernel<L, T>, grid, kStreamThreads, shm, s, p, a, kp, J);
    return launch_k(heisenberg_stream_kernel<L, T, false>, grid, kStreamThreads, shm, s, p, a, kp, J);
}

}  // namespace sk
