// common.cuh — device-side types and complex fp64 helpers shared by the CUDA kernels of
// libshiftk.so.  (The CPU oracle in oracle/ shares nothing with this file.)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

typedef double2 cplx;  // (x = re, y = im), 16-byte aligned -> LDG.128 / STG.128

__host__ __device__ __forceinline__ cplx mk(double re, double im) { return make_double2(re, im); }
__host__ __device__ __forceinline__ cplx cadd(cplx a, cplx b) { return mk(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ cplx csub(cplx a, cplx b) { return mk(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ cplx cmul(cplx a, cplx b) {
    return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ cplx cconj(cplx a) { return mk(a.x, -a.y); }
__host__ __device__ __forceinline__ double cabs2(cplx a) { return a.x * a.x + a.y * a.y; }
// acc + a * b
__host__ __device__ __forceinline__ cplx cfma(cplx a, cplx b, cplx acc) {
    return mk(fma(a.x, b.x, fma(-a.y, b.y, acc.x)), fma(a.x, b.y, fma(a.y, b.x, acc.y)));
}
// acc + conj(a) * b
__host__ __device__ __forceinline__ cplx cfma_conj(cplx a, cplx b, cplx acc) {
    return mk(fma(a.x, b.x, fma(a.y, b.y, acc.x)), fma(a.x, b.y, fma(-a.y, b.x, acc.y)));
}

__device__ __forceinline__ cplx ldg_cs(const cplx *p) { return __ldcs(p); }   // read once
__device__ __forceinline__ void stg_cs(cplx *p, cplx v) { __stcs(p, v); }
__device__ __forceinline__ cplx ldcg(const cplx *p) { return __ldcg(p); }     // L2 (coherent)

__device__ __forceinline__ void dbg_stamp(int64_t *ts, int i) {
    if (ts && threadIdx.x == 0) {
        int64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        ts[i] = t;
    }
}

// griddepcontrol.wait: returns when the programmatic predecessor grid has completed (a no-op for
// kernels launched without the PDL attribute).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ cplx warp_sum(cplx v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    }
    return v;
}

// Deterministic block sum of NV complex values per thread; result valid in thread 0.
// scratch: >= NV * (blockDim.x/32) cplx in shared memory.
template <int NV>
__device__ __forceinline__ void block_sum(cplx (&v)[NV], cplx *scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = warp_sum(v[j]);
    if (lane == 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j) scratch[j * nw + warp] = v[j];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            cplx s = scratch[j * nw];
            for (int w = 1; w < nw; ++w) s = cadd(s, scratch[j * nw + w]);
            v[j] = s;
        }
    }
    __syncthreads();
}

// select one of three by-value pointers without dynamic indexing (keeps them in registers)
template <typename T>
__host__ __device__ __forceinline__ T pick3(T const (&a)[3], int64_t i) {
    const int k = (int)(i % 3);
    return k == 0 ? a[0] : (k == 1 ? a[1] : a[2]);
}

// ---------------------------------------------------------------------------------------------
// Device-resident solver state (one per context).  Everything a kernel needs per iteration is
// read from here, so a captured CUDA graph can replay iterations without host involvement.
//
// Iteration bookkeeping: `n` completed iterations.  r_n lives in r[n % 3] (stored form,
// r_true = sr_cur * r_stored).  pi_n^k = pibuf[n % 3][k] * bscale[n % 3] and
// pi_{n-1}^k = pibuf[(n + 2) % 3][k] * bscale[(n + 2) % 3]: a seed switch rescales the two
// buffers' scale factors, never their elements (O(1) instead of O(N_z)).
// Retirement after a finish is applied lazily by the next per-shift pass (lz_pending).
// ---------------------------------------------------------------------------------------------
// Seed scalars of one iteration (steps.cuh seed_compute).
struct SeedOut {
    cplx w, alpha, beta, c, a_cur, a_q, a_prev, sr;
    int32_t ok, pad_;
};

struct DevState {
    int64_t n;           // completed iterations
    int64_t n_started;   // iterations whose seed scalars were computed
    int64_t nswitch;
    int64_t nspmv;
    int32_t status;      // sk_status
    int32_t pending;     // 1: iteration n was updated, its finish (residuals/switch) not yet run
    int32_t seed;        // current seed index s
    int32_t n_active;
    cplx zs;             // seed shift z_s
    cplx alpha_prev;     // alpha_{n-1} (current-seed normalisation)
    cplx rho_cur;        // rho_n of the current r_n (current-seed normalisation)
    cplx rho_prev;       // rho_{n-1}
    cplx sr_cur, sr_prev;   // lazy scale: r_true = sr * r_stored (shadow: conj(sr))
    cplx a_cur, a_q, a_prev; // r_{n+1} = a_cur r_cur_st + a_q q_raw + a_prev r_prev_st
    cplx alpha, beta, c; // seed scalars of the current iteration (read by the shift step)
    cplx sr_it;          // sr_cur used by the current iteration (full-mode coefficient)
    cplx w;              // diagnostics
    cplx bscale[3];      // lazy scale factors of the three pi buffers
    int32_t lz_pending;  // a retirement test of iteration lz_iter is due
    int32_t pad_;
    double lz_nu;        // ||r|| (current normalisation) for the pending retirement test
    int64_t lz_iter;
    double nu;           // ||r_n||_2 (true scale)
    double tol;
    int64_t itermax;
    int64_t seq;         // iterations whose update ran: the SpMV reads r[seq % 3] and writes its w
                         // partials to half (seq & 1) of part_w (written only by the update kernel)
    // the parts of the next seed step that do not depend on w, evaluated by the finish that
    // fixed rho_n (so the seed step on the critical path is one complex division):
    cplx beta_nx;        // beta_{n-1} = rho_n / rho_{n-1}   (0 at n = 0)
    cplx gamma_nx;       // beta_{n-1} / alpha_{n-1}          (0 at n = 0)
    int32_t rho_small;   // |rho_n| < 1e-300 (R12)
    int32_t pad2_;
    SeedOut rec;         // deferred mode: the seed scalars the update kernel used (committed by
                         // the next finish; written only by the update kernel's CTA 0)
};

// Pointers/sizes passed by value to every kernel.
struct KParams {
    DevState *st;
    int64_t M;           // local rows
    int32_t nz, nl;      // shifts, projections
    int32_t bicg, full;
    int32_t a_is_b;
    int32_t flags;
    cplx *r[3];          // rotating seed residual buffers
    cplx *t[3];          // shadow (BiCG)
    cplx *q, *qt;        // H r, H t (raw, i.e. applied to stored vectors)
    const cplx *left;    // [nl][M] (== b when a = b)
    cplx *part_w;        // [2][wred_stride]: SpMV w partials, half (seq & 1) per iteration
    cplx *part_u;        // [nblk_upd][2 + nl]
    int32_t nblk_spmv, nblk_upd;   // worker CTAs (= partial count) of the SpMV / update kernels
    // deferred seed step (world == 1, built-in operator): the update CTAs evaluate the seed
    // scalars themselves from the w partials [wred_off, wred_off + wred_n) of the current half;
    // the next finish commits them to the state (steps.cuh agent_finish)
    int32_t defer;
    int32_t wred_n;
    int64_t wred_off, wred_stride;
    // bond split (one GPU, Heisenberg chain, COCG, N_left = 1): the SpMV applies
    // H_A (diagonal + bonds i < split_ahi), the update H_B (the other bonds) in its own row order
    // and the partials of w_B = <r, H_B r> of the r it writes, at [wsplit_off, + nblk_upd) of
    // the next half of part_w (inside the range the seed step reduces).  split_ahi = 0: off.
    int32_t split_ahi;
    int32_t split_lo;            // bonds (i, i+1), i < split_lo, are in H_B too (B-tile piece bits)
    int64_t wsplit_off;
    double J;                    // exchange coupling of the Heisenberg operator (H_B amplitudes)
    // fused r_{n-1} term (§5.9): the H_A SpMV writes u = H_A r_n - kappa r_{n-1} with
    // kappa = gamma sr_prev / sr_cur (= -a_prev / a_q: known once the finish has fixed rho_n,
    // before w_n), so the update reads u instead of q and r_{n-1} (80 -> 64 B/row there, 32 -> 48
    // in the SpMV, which has DRAM headroom).  kflag: set by the SpMV's CTA 0 once the state is
    // final (after its finish), awaited by the worker CTAs, cleared by the update kernel.
    int32_t split_fuse;
    int32_t left_real;           // kp.left_re holds Re a (Im a = 0) in B-tile order, 8 B/row
    uint32_t *kflag;
    const double *left_re;
    // column-blocked CSR SpMV (spmv.cu): csr_nblk >= 2 passes over column blocks
    // of 2^csr_bshift rows, so the gathered slice of r stays in L2; csr_split[b * M + i] = entries
    // of row i with column < (b << csr_bshift) (rows sorted by column, <= 255 entries).  0: off.
    int32_t csr_nblk, csr_bshift;
    const uint8_t *csr_split;
    // per-shift arrays [nz]
    const cplx *z;
    cplx *pibuf;         // [3][nz] rotating pi_n^k
    cplx *pi_frozen;     // [nz] value at retirement
    uint8_t *active;
    double *res;
    int64_t *retired_at;
    cplx *u, *y;         // [nz][nl]
    cplx *g;             // [nl] projection of current r (true scale)
    // full mode
    cplx *p, *x;         // [nz][M]
    int64_t *dbg_ts;     // optional [16] %globaltimer stamps
    uint32_t *ticket;    // [1] last-CTA detection in the SpMV kernel (reset by the last CTA)
    unsigned long long *work;   // [2] tile queue of the streaming Heisenberg SpMV (reset by its last CTA)
    uint32_t *grp;              // [ngroups] tile-group counters of the streaming SpMV (reset by their reducers)
    int32_t n_agents;    // shift-agent CTAs of the update kernel (each a slice of the shifts)
    struct AminPart *amin_part;   // [n_agents] per-agent argmin |pi_{n+1}| and survivor count
    // ---- multi-rank (world > 1): this rank owns global rows [row0, row0 + M); every rank's r
    // (and r~) buffers are reachable through shard tables (NVLink peer mappings of the other
    // ranks' arenas, or the other contexts of a single-GPU loopback group).
    int32_t world, rank;
    int32_t lloc_bits;           // log2(M): M (rows per rank) is a power of two when world > 1
    int32_t pad_;
    int64_t row0;
    const cplx *const *shard_r;  // device [3 * world]: shard_r[b * world + g] = rank g's r[b]
    const cplx *const *shard_t;  // device [3 * world] (BiCG shadow)
    cplx *wloc, *wsum;           // [1] this rank's / all-reduced SpMV dot  (world > 1)
    cplx *uloc, *usum;           // [2 + nl] this rank's / all-reduced update dots (world > 1)
    uint32_t *ticket_u;          // [1] last-CTA detection in the update kernel (world > 1)
    // ---- coefficient log for recalculation (SK_FLAG_LOG) ----
    cplx *lg;                    // [lg_cap][6]: alpha_n, beta_{n-1}, c_n, z_s(n), 1/f, 1/f'
    double *lg_nu;               // [lg_cap]: ||r_{n+1}|| (before the switch of iteration n)
    cplx *lg_g;                  // [lg_cap][nl]: P r_n
    int64_t lg_cap;
};

// Per shift-agent result: argmin over its slice of |pi_{n+1}|^2 (lowest index on ties).
struct AminPart {
    double a2;
    int32_t idx, cnt;
    cplx f, fp;          // pi_{n+1}, pi_n of that shift
};

enum { ST_ITERATING = 0, ST_CONVERGED = 1, ST_MAXITER = 2, ST_BREAKDOWN = 3 };
