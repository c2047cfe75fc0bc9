// update_split.cu — the bond-split iteration of the Heisenberg chain at large L (one GPU, COCG,
// N_left = 1).
//
// H = H_A + H_B (EQ heisenberg P:L831: H = J sum_i S_i.S_{i+1}; every bond's off-diagonal part
// flips the two spins, amplitude J/2).  H_A holds the diagonal and the bonds (i, i+1) with
// i < AHI = L - HB; H_B the bonds i = AHI..L-2 and the periodic bond (L-1, 0).  The SpMV applies
// H_A in natural order (spmv_stream.cuh, SPLIT): its bonds stay inside a 2^10-state tile or
// reach a partner tile that is still in L2.  H_B would need partners 2^AHI states away — from
// DRAM on every use — so this kernel applies it instead, in its own row order: a B-tile is the
// 2^TB states {2^PB-state contiguous piece} x {all 2^HB combinations of spins AHI..L-1}, staged
// in shared memory, so every H_B partner of a B-tile row is in the same B-tile.
//
// Per B-tile (one CTA, double-buffered cp.async staging of r_n):
//   q_n     = q_A + H_B r_n                                   (q_A: the SpMV's output)
//   r_{n+1} = (1 + c - alpha z_s) r_n + alpha q_n - c r_{n-1}  (EQ-CG-RN-3REC P:L269, stored form)
//   dots of the next iteration: rho_{n+1} = <r_{n+1}, r_{n+1}>, ||r_{n+1}||^2, a^dag r_{n+1}
//   w_B     = <r_{n+1}, H_B r_{n+1}>  (r_{n+1} parked in shared memory; each anti-aligned pair
//            counted once, doubled)
// so the next iteration's w_{n+1} = <r_{n+1}, H r_{n+1}> (EQ-REC-ALPHA-N2 P:L276) is w_A (SpMV
// partials) + w_B (these partials): both sit in the half of part_w the next update's seed step
// reduces, in fixed order.  Bytes per row: SpMV 32 (r, q_A) + update 80 (r_n, q_A, r_{n-1}, b
// read; r_{n+1} written) = the algorithmic 112 of SURVEY §8(d.3): the far bonds' partner reads
// (the pair kernel's 3.5x DRAM excess at L = 30) are gone.
#include "kernels.cuh"
#include "steps.cuh"

namespace sk {

constexpr int kSplitHB = 8;      // spins AHI..L-1 in a B-tile
constexpr int kSplitTB = 12;     // 2^12 states per B-tile (64 KB per buffer, two buffers)
constexpr int kSplitNT = 512;    // threads per CTA (one CTA per SM)
// SPLIT_UPD_RK = 1: the w_B pass takes the thread's own r_{n+1} rows from registers instead of
// re-reading them from shared memory (one LDS.128 per row less).
#ifndef SPLIT_UPD_RK
#define SPLIT_UPD_RK 1
#endif

static __device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src) : "memory");
}
static __device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
static __device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Global row of B-tile t, local index e: piece bits e[0, PB) -> spins 0..PB-1, high bits
// e[PB, TB) -> spins AHI..L-1, tile index t -> spins PB..AHI-1.
template <int HB, int TB>
static __device__ __forceinline__ int64_t split_row(int64_t t, int e, int ahi) {
    constexpr int PB = TB - HB;
    return ((int64_t)(e >> PB) << ahi) | (t << PB) | (int64_t)(e & ((1 << PB) - 1));
}

template <int HB, int TB, int NT>
static __device__ __forceinline__ void stage_tile(cplx *S, const cplx *__restrict__ r, int64_t t, int ahi) {
    constexpr int TS = 1 << TB;
#pragma unroll
    for (int k = 0; k < TS / NT; ++k) {
        const int e = threadIdx.x + k * NT;
        cp_async16(S + e, r + split_row<HB, TB>(t, e, ahi));
    }
}

// Seed scalars, as in update.cu (deferred mode: every CTA reduces the w partials — here w_A
// groups + w_B partials — in fixed order and evaluates the seed step itself).
struct SplitSeed {
    DevState S;
    SeedOut o;
    int64_t nsx;
    cplx red8[8];
};

// Per-thread view of the H_B bonds of the rows e = tid | (k << NB) (k < PER, NT = 2^NB threads):
// a bond between two local bits is decided by tid alone (both bits < NB: a per-thread constant),
// by tid and k (one bit each), or by k alone (a compile-time constant once k is unrolled); its
// partner index is e ^ (bit mask) = (tid ^ low mask) | ((k ^ high mask) << NB).  Precomputing the
// per-thread parts turns every partner read into one LDS at a per-thread base + an immediate
// (ncu: the generic bit tests and index arithmetic were ~75 of 184 instructions per row).
template <int HB, int TB, int NB>
struct BondView {
    // bonds of H_B in local bits: j < NPIECE: (j, j+1) inside the piece (moved from H_A when
    // kp.split_lo = NPIECE, §5.9); then the chain (PB+i, PB+i+1), i < HB-1; last the periodic
    // (TB-1, 0).  For the pair count of w_B, `lower` is the bond's lower spin site.
    static constexpr int PB = TB - HB, NPIECE = PB - 1, NBOND = NPIECE + HB;
    __device__ __forceinline__ static constexpr int b1(int j) {
        return j < NPIECE ? j : (j < NBOND - 1 ? PB + (j - NPIECE) : TB - 1);
    }
    __device__ __forceinline__ static constexpr int b2(int j) {
        return j < NPIECE ? j + 1 : (j < NBOND - 1 ? PB + (j - NPIECE) + 1 : 0);
    }
    __device__ __forceinline__ static constexpr int lower(int j) { return j < NBOND - 1 ? b1(j) : b2(j); }
    __device__ __forceinline__ static constexpr int upper(int j) { return j < NBOND - 1 ? b2(j) : b1(j); }
    __device__ __forceinline__ static constexpr int mask(int j) { return (1 << b1(j)) | (1 << b2(j)); }
    __device__ __forceinline__ static constexpr bool piece(int j) { return j < NPIECE; }
    // bit `b` of e = tid | (k << NB)
    __device__ __forceinline__ static int bit(int tid, int k, int b) {
        return b < NB ? (tid >> b) & 1 : (k >> (b - NB)) & 1;
    }
};

// FUSE: q holds u = H_A r_n - kappa r_{n-1} (the SpMV's fused r_{n-1} term, kp.split_fuse), so
// r_{n+1} = a_cur r_n + a_q (u + H_B r_n) and r_{n-1} is not read.  LRE: the left vector is real
// (Im a = 0 at initialisation) and kp.left_re holds it in B-tile order (8 B/row, linear).
template <int HB, int TB, int NT, bool FUSE, bool LRE>
__global__ void __launch_bounds__(NT, 1) update_split_kernel(KParams kp, const cplx *__restrict__ q) {
    constexpr int TS = 1 << TB, PER = TS / NT, PB = TB - HB;
    constexpr int NB = NT == 256 ? 8 : NT == 512 ? 9 : 10;
    static_assert((1 << NB) == NT && PER * NT == TS && NT % (1 << PB) == 0, "CTA / B-tile / piece shape");
    using BV = BondView<HB, TB, NB>;
    // [2][TS]: r_n of the tile (cp.async staging) and r_{n+1} of the tile.  Shared memory is kept
    // to 128 KB + a few KB so ~95 KB of L1 remain for the row-stream loads in flight (with a
    // third 64-KB buffer the update ran 16 -> 22 ms: the loads had no L1 to land in).  The shift
    // agents' scratch lives in the same dynamic region (agents do not stream).
    extern __shared__ __align__(16) cplx S3[];
    __shared__ SplitSeed us;
    __shared__ cplx scratch[4 * (NT / 32)];
    pdl_wait();
    DevState *st = kp.st;
    if (FUSE && blockIdx.x == 0 && threadIdx.x == 0) *kp.kflag = 0u;   // the SpMV grid is complete
    if (st->status != ST_ITERATING) return;
    const int wb = blockIdx.x - kp.n_agents, nwb = gridDim.x - kp.n_agents;
    const int ahi = kp.split_ahi;
    const int64_t ntiles = kp.M >> TB;
    const int64_t ns = st->n_started + 1;   // after the seed step of iteration n (deferred mode)
    const cplx *__restrict__ rc_ = pick3(kp.r, ns + 2);   // r_n
    const cplx *__restrict__ rp_ = pick3(kp.r, ns + 1);   // r_{n-1}
    cplx *__restrict__ rn_ = pick3(kp.r, ns);             // r_{n+1}
    // tid < NT explicit (e = tid | (k << NB)); row of e in B-tile t: row0 + k kstep + (t << PB)
    const int tid = threadIdx.x & (NT - 1);
    const int64_t row0 = split_row<HB, TB>(0, tid, ahi);
    const int64_t kstep = (int64_t)(NT >> PB) << ahi;
    cplx *const S = S3, *const W = S3 + TS;   // r_n, r_{n+1} of the current tile
    auto stage = [&](int64_t t) {
        const cplx *src = rc_ + row0 + (t << PB);
#pragma unroll
        for (int k = 0; k < PER; ++k) cp_async16(S + (tid | (k << NB)), src + k * kstep);
        cp_async_commit();
    };
    // the first tile's r_n does not depend on the seed scalars: in flight during the w reduction
    if (wb >= 0 && wb < ntiles) stage(wb);
    // ---- seed step (a3): w = w_A + w_B partials of this iteration's half, fixed order
    {
        const int64_t m = st->n_started;
        state_load_nosync(us.S, st);
        const cplx w = reduce_w_fixed(kp.part_w + (m & 1) * kp.wred_stride + kp.wred_off, kp.wred_n, us.red8);
        if (threadIdx.x == 0) {
            us.o = seed_compute(us.S, w);
            us.nsx = m + 1;
            if (blockIdx.x == 0) {
                st->rec = us.o;
                st->pending = 1;
                if (us.o.ok) st->seq = m + 1;
            }
        }
        __syncthreads();
        if (!us.o.ok) {
            cp_async_wait<0>();
            return;
        }
    }
    if (blockIdx.x < kp.n_agents) {   // shift agents (a4 + a6 + pending a8)
        static_assert(sizeof(ShiftScratch) <= 2 * TS * sizeof(cplx), "agent scratch fits the tile buffers");
        shift_step(kp, *reinterpret_cast<ShiftScratch *>(S3), blockIdx.x, us.o.alpha, us.o.beta, us.o.c);
        return;
    }
    const cplx a_cur = us.o.a_cur, a_q = us.o.a_q, a_prev = us.o.a_prev;
    const double hJ = 0.5 * kp.J;
    const cplx *__restrict__ left = kp.left;
    const double *__restrict__ left_re = kp.left_re;
    const bool lo = kp.split_lo != 0;   // the piece bonds (0,1)..(PB-2,PB-1) are in H_B
    cplx rho = mk(0.0, 0.0), nu = mk(0.0, 0.0), g = mk(0.0, 0.0), wbp = mk(0.0, 0.0);
    for (int64_t t = wb; t < ntiles; t += nwb) {
        // every row-stream load of the tile is issued before waiting for its staged r_n (they do
        // not depend on it): 3 PER loads in flight per thread across the wait and the barrier
        const int64_t rt = row0 + (t << PB);
        cplx qa[PER], rp[FUSE ? 1 : PER], lv[LRE ? 1 : PER];
        double lr[LRE ? PER : 1];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int64_t s = rt + k * kstep;
            qa[k] = ldg_cs(q + s);
            if (!FUSE) rp[FUSE ? 0 : k] = ldg_cs(rp_ + s);
            if (LRE) lr[LRE ? k : 0] = __ldcs(left_re + (t << TB) + (tid | (k << NB)));
            else lv[LRE ? 0 : k] = ldg_cs(left + s);
        }
        cp_async_wait<0>();   // this tile's r_n has landed (staged during the previous w_B pass)
        __syncthreads();      // ... for every thread; and W of the previous tile is consumed
        cplx rk[SPLIT_UPD_RK ? PER : 1];   // the thread's own r_{n+1} rows, kept for the w_B pass
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int e = tid | (k << NB);
            cplx h = mk(0.0, 0.0);   // (H_B r_n)_e / (J/2): anti-aligned bonds' partners
#pragma unroll
            for (int j = 0; j < BV::NBOND; ++j) {
                if ((!BV::piece(j) || lo) && BV::bit(tid, k, BV::b1(j)) != BV::bit(tid, k, BV::b2(j))) {
                    const cplx p = S[e ^ BV::mask(j)];
                    h.x += p.x;
                    h.y += p.y;
                }
            }
            const cplx qf = mk(fma(hJ, h.x, qa[k].x), fma(hJ, h.y, qa[k].y));   // (H r_n)_s
            cplx rn = cmul(a_cur, S[e]);
            rn = cfma(a_q, qf, rn);
            if (!FUSE) rn = cfma(a_prev, rp[FUSE ? 0 : k], rn);
            rn_[rt + k * kstep] = rn;
            W[e] = rn;
            if (SPLIT_UPD_RK) rk[SPLIT_UPD_RK ? k : 0] = rn;
            rho = cfma(rn, rn, rho);
            nu.x = fma(rn.x, rn.x, fma(rn.y, rn.y, nu.x));
            if (LRE) g = mk(fma(lr[LRE ? k : 0], rn.x, g.x), fma(lr[LRE ? k : 0], rn.y, g.y));
            else g = cfma_conj(lv[LRE ? 0 : k], rn, g);
        }
        __syncthreads();   // r_{n+1} of the tile complete in W; r_n no longer read
        if (t + nwb < ntiles) stage(t + nwb);   // in flight during the w_B pass
#pragma unroll
        for (int k = 0; k < PER; ++k) {   // w_B: each anti-aligned pair once (lower bit 0, upper 1)
            const int e = tid | (k << NB);
            cplx h = mk(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < BV::NBOND; ++j) {
                if ((!BV::piece(j) || lo) && !BV::bit(tid, k, BV::lower(j)) && BV::bit(tid, k, BV::upper(j))) {
                    const cplx p = W[e ^ BV::mask(j)];
                    h.x += p.x;
                    h.y += p.y;
                }
            }
            wbp = cfma(SPLIT_UPD_RK ? rk[SPLIT_UPD_RK ? k : 0] : W[e], h, wbp);
        }
    }
    // CTA partials: rho, ||r||^2, a^dag r (part_u) and w_B (the next half of part_w)
    wbp = mk(2.0 * hJ * wbp.x, 2.0 * hJ * wbp.y);
    cplx v[4] = {rho, nu, g, wbp};
    block_sum<4>(v, scratch);
    if (threadIdx.x == 0) {
        cplx *pu = kp.part_u + (int64_t)wb * 3;
        pu[0] = v[0];
        pu[1] = v[1];
        pu[2] = v[2];
        kp.part_w[(us.nsx & 1) * kp.wred_stride + kp.wsplit_off + wb] = v[3];
    }
}

// w_B partials of r_0 = b (initialisation; half 0 of part_w, which the first update reduces):
// the same B-tiles and per-CTA tile order as the update kernel.
template <int HB, int TB, int NT>
__global__ void __launch_bounds__(NT, 1) split_wb_kernel(KParams kp, const cplx *__restrict__ r, cplx *out) {
    constexpr int TS = 1 << TB, PER = TS / NT;
    extern __shared__ __align__(16) cplx S2[];
    __shared__ cplx scratch[NT / 32];
    const int ahi = kp.split_ahi;
    const int64_t ntiles = kp.M >> TB;
    cplx wbp = mk(0.0, 0.0);
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        stage_tile<HB, TB, NT>(S2, r, t, ahi);
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        constexpr int NB = NT == 256 ? 8 : NT == 512 ? 9 : 10;
        using BV = BondView<HB, TB, NB>;
        const int tid = threadIdx.x & (NT - 1);
        const bool lo = kp.split_lo != 0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {   // as the update's w_B pass
            const int e = tid | (k << NB);
            cplx h = mk(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < BV::NBOND; ++j)
                if ((!BV::piece(j) || lo) && !BV::bit(tid, k, BV::lower(j)) && BV::bit(tid, k, BV::upper(j))) {
                    const cplx p = S2[e ^ BV::mask(j)];
                    h.x += p.x;
                    h.y += p.y;
                }
            wbp = cfma(S2[e], h, wbp);
        }
        __syncthreads();
    }
    const double hJ = 0.5 * kp.J;
    cplx v[1] = {mk(2.0 * hJ * wbp.x, 2.0 * hJ * wbp.y)};
    block_sum<1>(v, scratch);
    if (threadIdx.x == 0) out[blockIdx.x] = v[0];
}

// Re a in B-tile order (left_re[(t << TB) | e] = Re a[split_row(t, e)]) and a flag word that is
// nonzero when some Im a != 0 (then the complex left vector is read as before).
template <int HB, int TB>
__global__ void split_left_kernel(KParams kp, double *out, uint32_t *any_imag) {
    const int ahi = kp.split_ahi;
    bool im = false;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < kp.M; j += (int64_t)gridDim.x * blockDim.x) {
        const cplx v = kp.left[split_row<HB, TB>(j >> TB, (int)(j & ((1 << TB) - 1)), ahi)];
        out[j] = v.x;
        im |= v.y != 0.0;
    }
    if (__syncthreads_or(im) && threadIdx.x == 0) atomicOr(any_imag, 1u);
}

// ---- host side --------------------------------------------------------------------------------
int split_ahi_for(int L, int64_t M, int world, int bicg, int full, int nl, int kind_heisenberg) {
    static int en = -2;
    if (en == -2) {
        const char *e = getenv("SHIFTK_HEIS_SPLIT");
        en = !e ? -1 : (e[0] == '0' ? 0 : 1);
    }
    if (en == 0 || !kind_heisenberg || world != 1 || bicg || full || nl != 1) return 0;
    const int ahi = L - kSplitHB;
    if (ahi < kTileBits || ahi < kSplitTB - kSplitHB || M != (int64_t(1) << L) || L > 31) return 0;
    return (en == 1 || L >= 24) ? ahi : 0;
}

// SHIFTK_SPLIT_LO=1 moves the piece bonds (0,1)..(PB-2,PB-1) from H_A (the SpMV) to H_B (the
// update).  Measured at C5: SpMV 10.5 -> 9.8 ms, update 15.3 -> 17.2 ms (the update's predicated
// bond loads: 4.4e9 -> 5.9e9 instructions) — so off by default.
int split_lo_bonds() {
    static int lo = -1;
    if (lo < 0) {
        const char *e = getenv("SHIFTK_SPLIT_LO");
        lo = (e && e[0] == '1') ? kSplitTB - kSplitHB - 1 : 0;
    }
    return lo;
}

int split_blocks() { return sm_count(); }   // one CTA per SM (128 KB of shared memory each)

// dynamic shared memory: the update stages r_n in one buffer and parks r_{n+1} in a second; the
// init kernel uses one
static size_t split_smem_update() { return 2 * (sizeof(cplx) << kSplitTB); }
static size_t split_smem_init() { return sizeof(cplx) << kSplitTB; }

template <bool FUSE, bool LRE>
static cudaError_t split_attr() {
    return cudaFuncSetAttribute(update_split_kernel<kSplitHB, kSplitTB, kSplitNT, FUSE, LRE>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)split_smem_update());
}

static cudaError_t split_setup() {
    static PerDevice once;
    return once_per_device(once, [] {
        cudaError_t e = split_attr<false, false>();
        if (e == cudaSuccess) e = split_attr<false, true>();
        if (e == cudaSuccess) e = split_attr<true, false>();
        if (e == cudaSuccess) e = split_attr<true, true>();
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(split_wb_kernel<kSplitHB, kSplitTB, kSplitNT>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)split_smem_init());
        return e;
    });
}

template <bool FUSE, bool LRE>
static cudaError_t launch_update_split_t(const KParams &kp, const cplx *q, cudaStream_t s) {
    return launch_k(update_split_kernel<kSplitHB, kSplitTB, kSplitNT, FUSE, LRE>, kp.nblk_upd + kp.n_agents,
                    kSplitNT, split_smem_update(), s, true, kp, q);
}

cudaError_t launch_update_split(const KParams &kp, const cplx *q, cudaStream_t s) {
    const cudaError_t e = split_setup();
    if (e != cudaSuccess) return e;
    if (kp.split_fuse)
        return kp.left_real ? launch_update_split_t<true, true>(kp, q, s) : launch_update_split_t<true, false>(kp, q, s);
    return kp.left_real ? launch_update_split_t<false, true>(kp, q, s) : launch_update_split_t<false, false>(kp, q, s);
}

// SHIFTK_SPLIT_FUSE=0: the SpMV writes plain q = H_A r and the update reads r_{n-1} itself.
// (The streaming H_A kernel never fuses.)
int split_fuse_enabled() {
    static int en = -1;
    if (en < 0) {
        const char *e = getenv("SHIFTK_SPLIT_FUSE");
        en = (e && e[0] == '0') ? 0 : 1;
    }
    return en;
}

// SHIFTK_LEFT_REAL=0: never use the compressed real left vector.
int split_left_real_enabled() {
    static int en = -1;
    if (en < 0) {
        const char *e = getenv("SHIFTK_LEFT_REAL");
        en = (e && e[0] == '0') ? 0 : 1;
    }
    return en;
}

// out = Re(kp.left) in B-tile order; *any_imag |= 1 when some Im != 0 (zeroed by the caller)
cudaError_t launch_split_left(const KParams &kp, double *out, uint32_t *any_imag, cudaStream_t s) {
    split_left_kernel<kSplitHB, kSplitTB><<<8 * sm_count(), 256, 0, s>>>(kp, out, any_imag);
    return cudaGetLastError();
}

cudaError_t launch_split_init(const KParams &kp, cudaStream_t s) {
    const cudaError_t e = split_setup();
    if (e != cudaSuccess) return e;
    split_wb_kernel<kSplitHB, kSplitTB, kSplitNT><<<kp.nblk_upd, kSplitNT, split_smem_init(), s>>>(
        kp, kp.r[0], kp.part_w + kp.wsplit_off);
    return cudaGetLastError();
}

}  // namespace sk
