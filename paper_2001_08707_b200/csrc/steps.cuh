// steps.cuh — the scalar parts of one iteration as
// CTA-level device functions.  They run inside the streaming kernels, off the critical path:
//
//   finish_step  (an extra CTA of the SpMV kernel of iteration n+1, concurrent with the SpMV):
//       rho_{n+1}, nu = ||r_{n+1}||, g = P r_{n+1} from the update partials; residuals
//       res_k = nu/|pi_{n+1}^k| (EQ-COLLINEAR P:L300); retirement res_k < tol (R8);
//       seed switch to argmin_active |pi| (R9-R11); compacted active list.
//   seed_step    (the last CTA of the SpMV kernel, after every partial is written):
//       beta_{n-1} = rho_n/rho_{n-1}, gamma = beta/alpha_{n-1}, alpha_n =
//       rho_n/(z_s rho_n - w_n - gamma rho_n) (EQ-REC-ALPHA-N2 P:L276), c = alpha gamma.
//   shift_step   (an extra CTA of the update kernel, concurrent with the streaming update):
//       pi_{n+1} = (1 + c + alpha sigma) pi_n - c pi_{n-1} (EQ-SHIFTEDCG-PI P:L317),
//       alpha^k = (pi_n/pi_{n+1}) alpha, beta^k = (pi_{n-1}/pi_n)^2 beta,
//       u^k = g/pi_n^k + beta^k u^k, y^k += alpha^k u^k (EQ-SHIFTEDCG-y/u P:L372-376, R1).
//
// Because seed switching is applied lazily (scale factors, no vector pass), the SpMV of
// iteration n+1 does not depend on the finish of iteration n, which is what lets the finish
// run beside it.
//
// Latency rule used throughout (measured: one dependent L2/DRAM round trip costs ~0.5-1 us):
// every loop issues all of its loads for a block of shifts before any dependent arithmetic or
// branch, so a step over N_z shifts costs ~N_z/(4*256) round trips, not N_z/256 * (chain).
#pragma once
#include "common.cuh"

namespace sk {

// ---- complex helpers kept out of line (one copy of the division code) ---------------------
// 1/b with a scaling by max(|re|,|im|) so |b|^2 neither overflows nor underflows.
static __device__ __noinline__ cplx xrecip(cplx b) {
    const double s = fmax(fabs(b.x), fabs(b.y));
    const double is = 1.0 / s;
    const double xr = b.x * is, xi = b.y * is;
    const double d = is / (xr * xr + xi * xi);
    return mk(xr * d, -xi * d);
}
static __device__ __forceinline__ cplx xdiv(cplx a, cplx b) { return cmul(a, xrecip(b)); }
static __device__ __noinline__ double xabs(cplx b) {
    const double s = fmax(fabs(b.x), fabs(b.y));
    if (s == 0.0) return 0.0;
    const double is = 1.0 / s;
    const double xr = b.x * is, xi = b.y * is;
    return s * sqrt(xr * xr + xi * xi);
}

// The device state is read through L2 (ld.cg) into a shared-memory copy and written back
// word by word: the agent CTA and the last CTA of a kernel exchange it within one launch.
constexpr int kStateWords = sizeof(DevState) / 8;
static_assert(sizeof(DevState) % 8 == 0, "DevState is copied as 8-byte words");
static_assert(kStateWords <= 256, "DevState copy uses one word per thread");
static __device__ __forceinline__ void state_load_nosync(DevState &dst, const DevState *src) {
    if (threadIdx.x < kStateWords)
        ((long long *)&dst)[threadIdx.x] = __ldcg((const long long *)src + threadIdx.x);
}
static __device__ __forceinline__ void state_store(DevState *dst, const DevState &src) {
    __syncthreads();
    if (threadIdx.x < kStateWords) ((long long *)dst)[threadIdx.x] = ((const long long *)&src)[threadIdx.x];
}

constexpr int kSpt = 4;             // shifts per thread per block of a step loop
constexpr int kSmemShifts = 4096;   // shifts whose active flags fit in the scratch copy

// Scratch of a column reduction.
struct RedScratch {
    cplx col[40];                // reduced partial columns
    cplx red[4][32];             // per-warp partial sums (4 columns at a time)
};

// Shared scratch of the step functions (one instance per CTA that runs them).
struct StepScratch {
    DevState S;                  // shared copy of the device state
    cplx col[40];                // reduced partial columns
    cplx red[4][32];             // per-warp partial sums (4 columns at a time)
    double rd[32];
    int ri[32], rc[32];
    cplx bc[4];
    int bi[4];
    uint8_t act[kSmemShifts];    // active flags after retirement (compaction source)
};

// Sum columns [0, ncol) of part[nblk][stride] into sc.col — fixed order (per-thread strided
// sum over b = tid + 4k*NT.., then warps in index order): deterministic.  Loads of 4 blocks x
// up to 4 columns are issued before they are summed.  All threads call it; ends with a barrier.
template <typename Scratch>
static __device__ __forceinline__ void reduce_columns(const cplx *part, int nblk, int stride, int ncol,
                                                      Scratch &sc) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int NT = blockDim.x;
    for (int cb = 0; cb < ncol; cb += 4) {
        const int nc = ncol - cb < 4 ? ncol - cb : 4;
        cplx v[4] = {mk(0, 0), mk(0, 0), mk(0, 0), mk(0, 0)};
        for (int b0 = tid; b0 < nblk; b0 += 4 * NT) {
            cplx x[4][4];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int b = b0 + m * NT;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    x[m][j] = (b < nblk && j < nc) ? ldcg(part + (int64_t)b * stride + cb + j) : mk(0, 0);
            }
#pragma unroll
            for (int m = 0; m < 4; ++m)
#pragma unroll
                for (int j = 0; j < 4; ++j) v[j] = cadd(v[j], x[m][j]);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const cplx s = warp_sum(v[j]);
            if (lane == 0) sc.red[j][warp] = s;
        }
        __syncthreads();
        if (tid < nc) {
            cplx s = sc.red[tid][0];
            for (int w = 1; w < nw; ++w) s = cadd(s, sc.red[tid][w]);
            sc.col[cb + tid] = s;
        }
        __syncthreads();
    }
}

// Block exclusive scan of 0/1 flags over [0, n) in chunks of blockDim: writes the compacted
// ascending index list, returns the count (all threads).  Flags come from shared memory when
// n <= kSmemShifts (the caller filled sc.act), else from `act_g`.
static __device__ int compact_active(const uint8_t *act_g, int n, int32_t *list, StepScratch &sc) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const bool sm = n <= kSmemShifts;
    int total = 0;
    for (int base = 0; base < n; base += blockDim.x) {
        const int k = base + tid;
        const int a = (k < n) ? (int)(sm ? sc.act[k] : act_g[k]) : 0;
        const unsigned bal = __ballot_sync(0xffffffffu, a);
        if (lane == 0) sc.ri[warp] = __popc(bal);
        __syncthreads();
        if (warp == 0) {   // warp-level exclusive scan of the per-warp counts
            const int v = lane < nw ? sc.ri[lane] : 0;
            int incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += u;
            }
            if (lane < nw) sc.rc[lane] = incl - v;
            if (lane == 31) sc.bi[3] = incl;
        }
        __syncthreads();
        if (a) list[total + sc.rc[warp] + __popc(bal & ((1u << lane) - 1u))] = k;
        total += sc.bi[3];
        __syncthreads();
    }
    return total;
}

// ------------------------------------------------------------------------------- retirement
// The retirement test of iteration it = S->lz_iter: res_k = ||r_it|| / |pi_it^k|
// (EQ-COLLINEAR P:L300), retire when res_k < tol (R8).  Evaluated with the pi buffer
// of iteration it and its lazy scale, so every evaluator (shift agent, full-mode streaming
// CTAs, eager pass) takes the identical decision.
static __device__ __forceinline__ bool retire_test(double lz_nu, cplx pik, double tol, double &res) {
    res = lz_nu / sqrt(cabs2(pik));
    return res < tol;
}

// Eager application of a pending retirement test to every active shift (CTA-wide; operates on
// the shared state copy sc.S; the caller stores it).  Used when no further per-shift pass will
// run: the stand-alone finish, terminal states, breakdown.
static __device__ void retire_pass(const KParams &kp, StepScratch &sc) {
    DevState *S = &sc.S;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int NT = blockDim.x, nz = kp.nz;
    int cnt = 0;
    if (S->lz_pending && S->lz_iter == S->n) {
        const int64_t it = S->lz_iter;
        const cplx *buf = kp.pibuf + (size_t)(it % 3) * nz;
        const cplx bs = S->bscale[it % 3];
        const double lz_nu = S->lz_nu, tol = S->tol;
        for (int k0 = tid; k0 < nz; k0 += kSpt * NT) {
            uint8_t a[kSpt];
            cplx pk[kSpt];
#pragma unroll
            for (int s = 0; s < kSpt; ++s) {          // all loads of the block first
                const int k = k0 + s * NT;
                a[s] = k < nz ? kp.active[k] : (uint8_t)0;
                pk[s] = k < nz ? buf[k] : mk(1, 0);
            }
#pragma unroll
            for (int s = 0; s < kSpt; ++s) {
                const int k = k0 + s * NT;
                if (k >= nz || !a[s]) continue;
                const cplx p = cmul(pk[s], bs);
                double rk;
                if (retire_test(lz_nu, p, tol, rk)) {
                    kp.active[k] = 0;
                    kp.retired_at[k] = it;
                    kp.pi_frozen[k] = p;
                } else {
                    ++cnt;
                }
                kp.res[k] = rk;
            }
        }
    } else {
        for (int k = tid; k < nz; k += NT) cnt += kp.active[k] ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) sc.rc[warp] = cnt;
    __syncthreads();
    if (tid == 0) {
        int c = 0;
        for (int w = 0; w < nw; ++w) c += sc.rc[w];
        S->n_active = c;
        S->lz_pending = 0;
        if (c == 0) S->status = ST_CONVERGED;
    }
    __syncthreads();
}

// ------------------------------------------------------------------------------- finish_step
static __device__ __forceinline__ void seed_prepare(DevState *S);

// Finishes iteration m = S->n (pending): consumes the update partials of r_{m+1} and the
// argmin of |pi_{m+1}| found by the shift step of iteration m.  O(1) work besides the partial
// reduction: the switch rescales buffer scale factors, and the retirement test is left pending
// for the next per-shift pass (eager = true applies it here).  Retirement removes the shifts
// with the LARGEST |pi| (res = nu/|pi| < tol), so the argmin over the survivors is the argmin
// over the shifts active before the test unless every shift retires — which is exactly the
// test nu/|pi_{s*}| < tol on that argmin (R10, R11).
static __device__ void finish_step(const KParams &kp, StepScratch &sc, bool eager, bool loaded = false) {
    if (!loaded) state_load_nosync(sc.S, kp.st);
    DevState *S = &sc.S;
    const int nl = kp.nl, nred = 2 + nl;
    if (kp.usum) reduce_columns(kp.usum, 1, nred, nred, sc);         // all-reduced (world > 1)
    else reduce_columns(kp.part_u, kp.nblk_upd, nred, nred, sc);   // (barriers publish sc.S)
    const int64_t m = S->n;
    const double nu = sqrt(sc.col[1].x);
    if (blockIdx.x == 0) dbg_stamp(kp.dbg_ts, 12);
    if (threadIdx.x == 0) {
        // argmin over the shift agents' slices (ascending: ties keep the lowest index)
        AminPart best = kp.amin_part[0];
        int survivors = best.cnt;
        for (int a = 1; a < kp.n_agents; ++a) {
            const AminPart p = kp.amin_part[a];
            survivors += p.cnt;
            if (p.idx >= 0 && (best.idx < 0 || p.a2 < best.a2)) best = p;
        }
        S->n_active = survivors;
        const cplx f = best.f, fp = best.fp;
        const int bst = best.idx;
        double rmin;
        // (bst < 0: no agent kept a survivor — possible only when the lazy test of the agents and
        // this one differ by an ulp at res == tol; nothing is left to switch to, so it is the
        // all-retire case: retire_pass below makes it CONVERGED)
        const bool all_retire = bst < 0 || retire_test(nu, f, S->tol, rmin);
        const bool sw = !all_retire && !(kp.flags & 1) && bst != S->seed;
        cplx rf = mk(1, 0);
        if (sw) {   // a9 / R9: the new seed's r, r_prev, pi, alpha, rho in its own normalisation
            rf = xrecip(f);
            const cplx rfp = xrecip(fp);
            S->bscale[(m + 1) % 3] = cmul(S->bscale[(m + 1) % 3], rf);   // pi_{m+1} /= f
            S->bscale[m % 3] = cmul(S->bscale[m % 3], rfp);               // pi_m /= f'
            S->sr_cur = cmul(S->sr_cur, rf);                               // r_{m+1} /= f
            S->sr_prev = cmul(S->sr_prev, rfp);                            // r_m /= f'
            S->alpha_prev = cmul(S->alpha_prev, cmul(fp, rf));             // alpha_m^{s*}
            S->rho_prev = cmul(S->rho_prev, cmul(rfp, rfp));               // rho_m / f'^2
            S->zs = kp.z[bst];
            S->seed = bst;
            S->nswitch += 1;
        }
        if (m < kp.lg_cap) {   // coefficient log (recalc): nu before the switch, switch factors
            kp.lg_nu[m] = nu;
            kp.lg[6 * m + 4] = rf;
            kp.lg[6 * m + 5] = sw ? xrecip(fp) : mk(1, 0);
        }
        S->rho_cur = cmul(sc.col[0], cmul(rf, rf));                       // rho_{m+1} / f^2
        S->n = m + 1;
        seed_prepare(S);
        S->nu = nu * sqrt(cabs2(rf));
        S->lz_pending = 1;
        S->lz_nu = S->nu;   // current normalisation (matches the rescaled pi buffers)
        S->lz_iter = m + 1;
        S->pending = 0;
        if (!all_retire && m + 1 >= S->itermax) S->status = ST_MAXITER;
        sc.bc[0] = rf;
        sc.bi[0] = all_retire || S->status != ST_ITERATING;
    }
    __syncthreads();
    if (threadIdx.x < nl) {
        const cplx gl = cmul(sc.col[2 + threadIdx.x], sc.bc[0]);
        kp.g[threadIdx.x] = gl;
        if (m + 1 < kp.lg_cap) kp.lg_g[(m + 1) * nl + threadIdx.x] = gl;   // P r_{m+1}
    }
    if (eager || sc.bi[0]) retire_pass(kp, sc);
    state_store(kp.st, sc.S);
}

// ------------------------------------------------------------------------------- seed_step
// Seed scalars of iteration n from the state before the seed step and w_raw = <r~|r, q> of the
// stored vectors.  Pure: evaluated identically by the update CTAs (deferred mode) and by the
// commit (seed_step), so both hold bit-identical values.
static __device__ __forceinline__ bool tiny_abs(cplx v) {   // xabs(v) < 1e-300, cheap path first
    const double s = fmax(fabs(v.x), fabs(v.y));
    if (s >= 1e-300) return false;
    return xabs(v) < 1e-300;
}
static __device__ __forceinline__ SeedOut seed_compute(const DevState &S, cplx wraw) {
    SeedOut o;
    const cplx sr = S.sr_cur;
    o.sr = sr;
    o.w = cmul(cmul(sr, sr), wraw);   // true-scale w_n (shadow scale = conj(sr))
    const cplx rho = S.rho_cur;
    const cplx beta = S.beta_nx, gamma = S.gamma_nx;   // EQ-REC-BETA P:L262 (by the finish)
    // EQ-REC-ALPHA-N2: alpha = rho / (<r, A r> - gamma rho), <r, A r> = z_s rho - w
    const cplx den = csub(csub(cmul(S.zs, rho), o.w), cmul(gamma, rho));
    o.ok = !(S.rho_small || tiny_abs(den));   // R12
    o.pad_ = 0;
    const cplx alpha = o.ok ? xdiv(rho, den) : mk(0, 0);
    const cplx c = cmul(alpha, gamma);
    o.alpha = alpha;
    o.beta = beta;
    o.c = c;
    const cplx c1 = cadd(mk(1.0, 0.0), c);
    o.a_cur = cmul(csub(c1, cmul(alpha, S.zs)), sr);   // EQ-CG-RN-3REC with A r = z_s r - q
    o.a_q = cmul(alpha, sr);
    o.a_prev = cmul(mk(-c.x, -c.y), S.sr_prev);
    return o;
}

// Next seed step's w-independent parts (beta_{n-1}, gamma, |rho_n| test), from the state after a
// finish (or the initialisation) — the same operations the seed step itself would do.
static __device__ __forceinline__ void seed_prepare(DevState *S) {
    if (S->n > 0) {
        S->beta_nx = xdiv(S->rho_cur, S->rho_prev);
        S->gamma_nx = xdiv(S->beta_nx, S->alpha_prev);
    } else {
        S->beta_nx = mk(0, 0);
        S->gamma_nx = mk(0, 0);
    }
    S->rho_small = tiny_abs(S->rho_cur);
}

// Commit evaluated seed scalars to a shared copy of the state (one thread).
static __device__ void seed_apply(DevState *S, const SeedOut &o, int bicg, const KParams &kp) {
    const int64_t n = S->n;
    S->w = o.w;
    if (!o.ok) {
        S->status = ST_BREAKDOWN;
        return;
    }
    S->alpha = o.alpha;
    S->beta = o.beta;
    S->c = o.c;
    S->sr_it = o.sr;
    if (n < kp.lg_cap) {   // coefficient log (recalc)
        kp.lg[6 * n] = o.alpha;
        kp.lg[6 * n + 1] = o.beta;
        kp.lg[6 * n + 2] = o.c;
        kp.lg[6 * n + 3] = S->zs;
        kp.lg[6 * n + 4] = mk(1, 0);
        kp.lg[6 * n + 5] = mk(1, 0);
    }
    S->a_cur = o.a_cur;
    S->a_q = o.a_q;
    S->a_prev = o.a_prev;
    S->sr_prev = o.sr;
    S->sr_cur = mk(1.0, 0.0);
    S->alpha_prev = o.alpha;
    S->rho_prev = S->rho_cur;
    S->n_started = n + 1;
    S->pending = 1;
    S->bscale[(n + 1) % 3] = mk(1.0, 0.0);   // the shift step writes pi_{n+1} unscaled
    S->nspmv += bicg ? 2 : 1;
}

// One thread, on a shared copy of the state: evaluate and commit the seed step.
static __device__ void seed_step(DevState *S, cplx wraw, int bicg, const KParams &kp) {
    seed_apply(S, seed_compute(*S, wraw), bicg, kp);
}

// w_raw of the deferred seed step: the partials of the current half reduced in a fixed order
// that does not depend on the CTA size (threads 0..255 take strided subsequences, then a fixed
// warp tree, then warps 0..7 in order), so every CTA that evaluates it gets the same bits.  All
// threads call it (blockDim >= 256); ends with a barrier.
static __device__ __noinline__ cplx reduce_w_fixed(const cplx *part, int n, cplx *red8) {
    const int tid = threadIdx.x;
    cplx v = mk(0.0, 0.0);
    if (tid < 256) {
        for (int i = tid; i < n; i += 4 * 256) {   // four loads in flight, predicated at the end
            const cplx z = mk(0.0, 0.0);
            const cplx a = ldcg(part + i);
            const cplx b = i + 256 < n ? ldcg(part + i + 256) : z;
            const cplx c = i + 512 < n ? ldcg(part + i + 512) : z;
            const cplx d = i + 768 < n ? ldcg(part + i + 768) : z;
            v = cadd(cadd(cadd(cadd(v, a), b), c), d);
        }
        v = warp_sum(v);
        if ((tid & 31) == 0) red8[tid >> 5] = v;
    }
    __syncthreads();
    cplx s = red8[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) s = cadd(s, red8[w]);
    __syncthreads();
    return s;
}

// The finish of a pending iteration as the agents run it.  Deferred mode: first commit the seed
// step of that iteration (the scalars the update CTAs evaluated, recorded in S.rec by CTA 0);
// a breakdown there ends the run (with the retirement test left pending by the previous finish
// applied eagerly).  Then finish_step.
static __device__ void agent_finish(const KParams &kp, StepScratch &sc, bool eager) {
    if (!kp.defer) {
        finish_step(kp, sc, eager);
        return;
    }
    state_load_nosync(sc.S, kp.st);
    __syncthreads();
    if (threadIdx.x == 0 && sc.S.status == ST_ITERATING) seed_apply(&sc.S, sc.S.rec, kp.bicg, kp);
    __syncthreads();
    if (blockIdx.x == 0) dbg_stamp(kp.dbg_ts, 11);
    if (sc.S.status == ST_BREAKDOWN) {
        if (sc.S.lz_pending) retire_pass(kp, sc);
        if (threadIdx.x == 0) sc.S.pending = 0;
        state_store(kp.st, sc.S);
        return;
    }
    finish_step(kp, sc, eager, /*loaded=*/true);
}

// ------------------------------------------------------------------------------- shift recurrences
// Per-shift coefficients of iteration n (identical arithmetic wherever it is evaluated).
struct ShiftCoef {
    cplx pin, ak, bk, ipik;
};
static __device__ __forceinline__ ShiftCoef shift_coef(cplx pik, cplx piok, cplx zk, cplx zs, cplx alpha,
                                                       cplx beta, cplx c, int64_t n) {
    ShiftCoef o;
    const cplx sigma = csub(zk, zs);
    // EQ-SHIFTEDCG-PI: pi_{n+1} = (1 + c + alpha sigma) pi_n - c pi_{n-1}
    o.pin = csub(cmul(cadd(cadd(mk(1.0, 0.0), c), cmul(alpha, sigma)), pik), cmul(c, piok));
    o.ipik = xrecip(pik);
    o.ak = cmul(cmul(pik, xrecip(o.pin)), alpha);
    o.bk = mk(0, 0);
    if (n > 0) {
        const cplx rat = cmul(piok, o.ipik);
        o.bk = cmul(cmul(rat, rat), beta);
    }
    return o;
}

// Per-shift pass of iteration n (a4 + a6, and the pending retirement test of a8): for every
// shift active at the previous finish, apply the retirement test; for the survivors compute
// pi_{n+1}, u, y; find argmin |pi_{n+1}| (lowest index on ties) for the next finish.  Shifts
// are visited directly in blocks of 2 per thread with all loads issued first.  For
// N_left > 1 the (shift, l) pairs of a block are spread over the threads.  All threads call
// it.  Writes only per-shift arrays and the amin / n_active / lz_pending words of the state.
struct ShiftScratch {
    cplx g[32];
    cplx ak[512], bk[512], ip[512];   // per-shift coefficients of a block (2 per thread, <= 256 threads)
    uint8_t act[512];
    double rd[32];
    int ri[32], rc[32];
    cplx f, fp;
};
static __device__ void shift_step(const KParams &kp, ShiftScratch &ss, int agent, cplx alpha, cplx beta, cplx c) {
    DevState *S = kp.st;
    const int64_t n = S->n;
    const int nzt = kp.nz, nl = kp.nl, NT = blockDim.x, tid = threadIdx.x;
    const int per = (nzt + kp.n_agents - 1) / kp.n_agents;   // this agent's slice [k_lo, k_lo+nz)
    const int k_lo = agent * per;
    const int nz = nzt - k_lo < per ? (nzt - k_lo > 0 ? nzt - k_lo : 0) : per;
    const int lane = tid & 31, warp = tid >> 5, nw = NT >> 5;
    const cplx *cur = kp.pibuf + (size_t)(n % 3) * nzt + k_lo;
    const cplx *prv = kp.pibuf + (size_t)((n + 2) % 3) * nzt + k_lo;
    cplx *nxt = kp.pibuf + (size_t)((n + 1) % 3) * nzt + k_lo;
    const cplx *zz = kp.z + k_lo;
    uint8_t *actv = kp.active + k_lo;
    const cplx bc = S->bscale[n % 3], bp = S->bscale[(n + 2) % 3];
    const cplx zs = S->zs;
    const bool lz = S->lz_pending != 0 && S->lz_iter == n;
    const double lz_nu = S->lz_nu, tol = S->tol;
    int cnt = 0, bi = -1;
    double best = 0.0;
    if (tid < nl) ss.g[tid] = kp.g[tid];
    __syncthreads();
    for (int k0 = 0; k0 < nz; k0 += 2 * NT) {
        uint8_t a[2];
        cplx pc[2], pp[2], zk[2], uk[2], yk[2];
#pragma unroll
        for (int s = 0; s < 2; ++s) {            // all loads of the block first
            const int k = k0 + tid + s * NT;
            const bool in = k < nz;
            a[s] = in ? actv[k] : (uint8_t)0;
            pc[s] = in ? cur[k] : mk(1, 0);
            pp[s] = in ? prv[k] : mk(1, 0);
            zk[s] = in ? zz[k] : mk(0, 0);
            uk[s] = (in && nl == 1) ? kp.u[k_lo + k] : mk(0, 0);
            yk[s] = (in && nl == 1) ? kp.y[k_lo + k] : mk(0, 0);
        }
        if (nl > 1) __syncthreads();   // previous block's coefficients are consumed
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int k = k0 + tid + s * NT;
            bool on = k < nz && a[s];
            const cplx pik = cmul(pc[s], bc), piok = cmul(pp[s], bp);
            if (on && lz) {
                double rk;
                if (retire_test(lz_nu, pik, tol, rk)) {
                    on = false;
                    actv[k] = 0;
                    kp.retired_at[k_lo + k] = n;
                    kp.pi_frozen[k_lo + k] = pik;
                }
                kp.res[k_lo + k] = rk;
            }
            if (nl > 1) ss.act[tid + s * NT] = on;
            if (!on) continue;
            const ShiftCoef sc = shift_coef(pik, piok, zk[s], zs, alpha, beta, c, n);
            nxt[k] = sc.pin;
            ++cnt;
            const double a2 = cabs2(sc.pin);
            if (bi < 0 || a2 < best) { best = a2; bi = k; }   // ascending k: ties keep the lowest
            if (nl == 1) {
                const cplx uu = cadd(cmul(ss.g[0], sc.ipik), cmul(sc.bk, uk[s]));   // P:L372-376 (R1)
                kp.u[k_lo + k] = uu;
                kp.y[k_lo + k] = cfma(sc.ak, uu, yk[s]);
            } else {
                ss.ak[tid + s * NT] = sc.ak;
                ss.bk[tid + s * NT] = sc.bk;
                ss.ip[tid + s * NT] = sc.ipik;
            }
        }
        if (nl > 1) {
            __syncthreads();
            const int nk = nz - k0 < 2 * NT ? nz - k0 : 2 * NT;
            for (int e0 = tid; e0 < nk * nl; e0 += 2 * NT) {   // (shift, l) pairs
                cplx uv[2], yv[2];
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const int e = e0 + s * NT;
                    const int64_t o = (int64_t)(k_lo + k0) * nl + e;
                    uv[s] = e < nk * nl ? kp.u[o] : mk(0, 0);
                    yv[s] = e < nk * nl ? kp.y[o] : mk(0, 0);
                }
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const int e = e0 + s * NT;
                    if (e >= nk * nl) continue;
                    const int kk = e / nl, l = e - kk * nl;
                    if (!ss.act[kk]) continue;
                    const int64_t o = (int64_t)(k_lo + k0) * nl + e;
                    const cplx uu = cadd(cmul(ss.g[l], ss.ip[kk]), cmul(ss.bk[kk], uv[s]));
                    kp.u[o] = uu;
                    kp.y[o] = cfma(ss.ak[kk], uu, yv[s]);
                }
            }
        }
    }
    // block reduction: survivor count + argmin |pi_{n+1}|
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (oi >= 0 && (bi < 0 || ov < best || (ov == best && oi < bi))) { best = ov; bi = oi; }
    }
    if (lane == 0) { ss.rc[warp] = cnt; ss.rd[warp] = best; ss.ri[warp] = bi; }
    __syncthreads();
    if (tid == 0) {
        int cc = 0, i = -1;
        double b = 0.0;
        for (int w = 0; w < nw; ++w) {
            cc += ss.rc[w];
            const int oi = ss.ri[w];
            const double ov = ss.rd[w];
            if (oi >= 0 && (i < 0 || ov < b || (ov == b && oi < i))) { b = ov; i = oi; }
        }
        AminPart p;
        p.a2 = b;
        p.idx = i < 0 ? -1 : k_lo + i;
        p.cnt = cc;
        p.f = i < 0 ? mk(1, 0) : nxt[i];          // written by this CTA above
        p.fp = i < 0 ? mk(1, 0) : cmul(cur[i], bc);
        kp.amin_part[agent] = p;
    }
}

}  // namespace sk
