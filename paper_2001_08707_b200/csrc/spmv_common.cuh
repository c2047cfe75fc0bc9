// spmv_common.cuh — the view of the rotating r buffers as the global vector (shard tables)
// and the common prologue/epilogue of the solver-mode SpMV kernels (finish agent, seed tail).
#pragma once
#include "kernels.cuh"
#include "steps.cuh"

namespace sk {

// View of one rotating r buffer as the GLOBAL vector: this rank's rows are local; with
// world > 1 every other rank's rows are reached through the shard table (peer memory over
// NVLink, or the other contexts of a loopback group) — the exchange of the operator is fused
// into the SpMV's own loads.
// MULTI = false compiles the single-GPU case down to a plain pointer offset.
template <bool MULTI>
struct RViewT {
    const cplx *loc;
    const cplx *const *tab;   // [world] for this buffer index, or null (world <= 1)
    int64_t row0;
    int lloc, world;
    __device__ __forceinline__ const cplx *at(uint64_t g) const {
        if (!MULTI) return loc + (int64_t)g;
        if (world <= 1) return loc + (int64_t)(g - (uint64_t)row0);
        return tab[g >> lloc] + (g & ((1ull << lloc) - 1ull));
    }
};
using RView = RViewT<true>;
template <bool MULTI = true>
static __device__ __forceinline__ RViewT<MULTI> rview(const cplx *loc, const cplx *const *shard, int buf, const KParams &kp) {
    RViewT<MULTI> v;
    v.loc = loc;
    v.world = kp.world;
    v.tab = (kp.world > 1 && shard) ? shard + (size_t)buf * kp.world : nullptr;
    v.row0 = kp.world > 1 ? kp.row0 : 0;
    v.lloc = kp.lloc_bits;
    return v;
}

// Common prologue/epilogue of the solver-mode SpMV kernels.  Returns false when the kernel
// should do nothing (terminal state).  `agent` is true for CTA 0 in solver mode.
static __device__ __forceinline__ bool spmv_enter(const SpmvArgs &a, bool &agent, int &buf, StepScratch &sc,
                                          const KParams &kp) {
    agent = false;
    buf = 0;
    pdl_wait();
    if (!a.st) return true;
    // the three words read together (one round trip; seq is written only by the update kernel)
    const int32_t status = a.st->status;
    const int64_t seq = a.st->seq;
    const int32_t pending = a.st->pending;
    if (status != ST_ITERATING) return false;
    buf = (int)(seq % 3);
    if (blockIdx.x == 1) dbg_stamp(kp.dbg_ts, 0);                 // first worker CTA starts
    if (blockIdx.x == 0) {
        agent = true;
        dbg_stamp(kp.dbg_ts, 1);
        if (pending) agent_finish(kp, sc, /*eager=*/false);
        dbg_stamp(kp.dbg_ts, 2);                                   // finish agent done
    }
    return true;
}

// `red`/`red_n`: the partials the last CTA reduces when the kernel wrote its own (fixed-order
// per-tile / per-group partials of the streaming kernel); default: one partial per worker CTA.
static __device__ __forceinline__ void spmv_exit(const SpmvArgs &a, const KParams &kp, bool agent, cplx w,
                                          StepScratch &sc, const cplx *red = nullptr, int red_n = 0) {
    __shared__ cplx scratch[32];
    __shared__ int last;
    const bool per_cta = red == nullptr;
    // deferred seed step: this iteration's half of part_w; the update CTAs reduce it
    cplx *pw = a.part_w;
    if (a.st && kp.defer && pw) pw += (a.st->seq & 1) * kp.wred_stride;
    if (per_cta) { red = pw; red_n = gridDim.x - 1; }
    if (per_cta && !agent && pw) {
        cplx v[1] = {w};
        block_sum<1>(v, scratch);
        if (threadIdx.x == 0) pw[blockIdx.x - (a.st ? 1 : 0)] = v[0];
    }
    if (!a.st || kp.defer) return;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(kp.ticket, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!last) return;
    dbg_stamp(kp.dbg_ts, 3);                                       // last CTA arrives
    __threadfence();
    if (kp.world > 1) {   // this rank's w only: the all-reduce and the seed step follow
        reduce_columns(red, red_n, 1, 1, sc);
        if (threadIdx.x == 0) {
            kp.wloc[0] = sc.col[0];
            *kp.ticket = 0u;
        }
        return;
    }
    state_load_nosync(sc.S, kp.st);
    reduce_columns(red, red_n, 1, 1, sc);   // (its barriers publish sc.S)
    dbg_stamp(kp.dbg_ts, 9);                                       // partials reduced
    if (threadIdx.x == 0) {
        if (sc.S.status == ST_ITERATING) seed_step(&sc.S, sc.col[0], a.bicg, kp);
        *kp.ticket = 0u;
    }
    // (a breakdown here leaves the pending retirement test to the stand-alone finish)
    state_store(kp.st, sc.S);
    dbg_stamp(kp.dbg_ts, 4);                                       // seed step done
}

}  // namespace sk
