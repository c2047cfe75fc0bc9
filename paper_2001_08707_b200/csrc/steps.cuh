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
static __device__ __forceinline__ void state_load(DevState &dst, const DevState *src) {
    if (threadIdx.x < kStateWords)
        ((long long *)&dst)[threadIdx.x] = __ldcg((const long long *)src + threadIdx.x);
    __syncthreads();
}
static __device__ __forceinline__ void state_store(DevState *dst, const DevState &src) {
    __syncthreads();
    if (threadIdx.x < kStateWords) ((long long *)dst)[threadIdx.x] = ((const long long *)&src)[threadIdx.x];
}

// Shared scratch of the step functions (one instance per CTA that runs them).
struct StepScratch {
    DevState S;        // shared copy of the device state
    cplx col[40];      // reduced partial columns
    cplx red[4][32];   // per-warp partial sums (4 columns at a time)
    double rd[32];
    int ri[32], rc[32];
    cplx bc[4];
    int bi[4];
};

// Sum columns [c0, c0 + ncol) of part[nblk][stride] into sc.col[c0 ..] — fixed order
// (per-thread strided sum, then warps in index order): deterministic.  Up to four columns per
// sweep so that their loads are in flight together.  All threads of the CTA must call it.
static __device__ __forceinline__ void reduce_columns(const cplx *part, int nblk, int stride, int c0,
                                               int ncol, StepScratch &sc) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    for (int cb = 0; cb < ncol; cb += 4) {
        const int nc = ncol - cb < 4 ? ncol - cb : 4;
        cplx v[4] = {mk(0, 0), mk(0, 0), mk(0, 0), mk(0, 0)};
        for (int b = tid; b < nblk; b += blockDim.x) {
            const cplx *row = part + (int64_t)b * stride + c0 + cb;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (j < nc) v[j] = cadd(v[j], ldcg(row + j));
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
            sc.col[c0 + cb + tid] = s;
        }
        __syncthreads();
    }
}

// Block exclusive scan of 0/1 flags over [0, n) in chunks of blockDim: writes the compacted
// ascending index list, returns the count (all threads).
static __device__ __forceinline__ int compact_active(const uint8_t *act, int n, int32_t *list, StepScratch &sc) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    int total = 0;
    for (int base = 0; base < n; base += blockDim.x) {
        const int k = base + tid;
        const int a = (k < n) ? (int)act[k] : 0;
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

// ------------------------------------------------------------------------------- finish_step
// Finishes iteration m = S->n (pending): consumes the update partials of r_{m+1}.  All threads
// of the CTA call it; reads and writes the device state in global memory.
static __device__ void finish_step(const KParams &kp, StepScratch &sc) {
    state_load(sc.S, kp.st);
    DevState *S = &sc.S;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int nz = kp.nz, nl = kp.nl, nred = 2 + nl;
    reduce_columns(kp.part_u, kp.nblk_upd, nred, 0, nred, sc);
    const int64_t m = S->n;
    cplx *cur = kp.pibuf + (size_t)((m + 1) % 3) * nz;   // pi_{m+1}
    cplx *prv = kp.pibuf + (size_t)(m % 3) * nz;         // pi_m
    const double nu2 = sc.col[1].x;
    const double nu = sqrt(nu2);
    const double tol = S->tol;
    // a8: residuals and retirement; local count + argmin of |pi|^2 over survivors
    int cnt = 0, bi = -1;
    double best = 0.0;
    for (int k = tid; k < nz; k += blockDim.x) {
        if (!kp.active[k]) continue;
        const cplx pk = cur[k];
        const double a2 = cabs2(pk);
        const double rk = nu * rsqrt(a2);      // ||r_{m+1}|| / |pi_{m+1}^k|
        kp.res[k] = rk;
        if (rk < tol) {
            kp.active[k] = 0;
            kp.retired_at[k] = m + 1;
            kp.pi_frozen[k] = pk;
            continue;
        }
        ++cnt;
        if (bi < 0 || a2 < best) { best = a2; bi = k; }   // ascending k: ties keep the lowest
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (oi >= 0 && (bi < 0 || ov < best || (ov == best && oi < bi))) { best = ov; bi = oi; }
    }
    if (lane == 0) { sc.rc[warp] = cnt; sc.rd[warp] = best; sc.ri[warp] = bi; }
    __syncthreads();
    if (warp == 0) {
        int c = lane < nw ? sc.rc[lane] : 0;
        double b = lane < nw ? sc.rd[lane] : 0.0;
        int i = lane < nw ? sc.ri[lane] : -1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            c += __shfl_xor_sync(0xffffffffu, c, o);
            const double ov = __shfl_xor_sync(0xffffffffu, b, o);
            const int oi = __shfl_xor_sync(0xffffffffu, i, o);
            if (oi >= 0 && (i < 0 || ov < b || (ov == b && oi < i))) { b = ov; i = oi; }
        }
        if (lane == 0) { sc.bi[0] = c; sc.bi[1] = i; }
    }
    __syncthreads();
    cnt = sc.bi[0];
    const int bst = sc.bi[1];
    const bool sw = cnt > 0 && !(kp.flags & 1) && bst != S->seed;
    cplx rf = mk(1, 0), rfp = mk(1, 0);
    if (sw) {   // a9 / R9: the new seed's r, r_prev, pi, alpha, rho in its own normalisation
        const cplx f = cur[bst], fp = prv[bst];
        rf = xrecip(f);
        rfp = xrecip(fp);
        __syncthreads();   // everyone has read pi[best] before it is rescaled
        for (int k = tid; k < nz; k += blockDim.x) {
            if (!kp.active[k]) continue;   // retired shifts are not rescaled (R13)
            cur[k] = cmul(cur[k], rf);
            prv[k] = cmul(prv[k], rfp);
        }
        if (tid == 0) {
            S->sr_cur = cmul(S->sr_cur, rf);                        // r_{m+1} /= f
            S->sr_prev = cmul(S->sr_prev, rfp);                     // r_m /= f'
            S->alpha_prev = cmul(S->alpha_prev, cmul(fp, rf));      // alpha_m^{s*}
            S->rho_prev = cmul(S->rho_prev, cmul(rfp, rfp));        // rho_m / f'^2
            S->zs = kp.z[bst];
            S->seed = bst;
            S->nswitch += 1;
        }
    }
    if (tid < nl) kp.g[tid] = sw ? cmul(sc.col[2 + tid], rf) : sc.col[2 + tid];
    const int nact = compact_active(kp.active, nz, kp.act_list, sc);
    if (tid == 0) {
        *kp.n_act = nact;
        S->rho_cur = sw ? cmul(sc.col[0], cmul(rf, rf)) : sc.col[0];   // rho_{m+1} / f^2
        S->nu = sw ? nu * sqrt(cabs2(rf)) : nu;
        S->n = m + 1;
        S->pending = 0;
        S->n_active = cnt;
        if (cnt == 0) S->status = ST_CONVERGED;
        else if (m + 1 >= S->itermax) S->status = ST_MAXITER;
    }
    state_store(kp.st, sc.S);
}

// ------------------------------------------------------------------------------- seed_step
// One thread, on a shared copy of the state.  w_raw = <r~|r, q> of the stored vectors.  Writes the update coefficients.
static __device__ void seed_step(DevState *S, cplx wraw, int bicg) {
    const cplx sr = S->sr_cur;
    const cplx w = cmul(cmul(sr, sr), wraw);   // true-scale w_n (shadow scale = conj(sr))
    const cplx rho = S->rho_cur;
    const int64_t n = S->n;
    cplx beta = mk(0, 0), gamma = mk(0, 0);
    if (n > 0) {
        beta = xdiv(rho, S->rho_prev);             // EQ-REC-BETA P:L262
        gamma = xdiv(beta, S->alpha_prev);
    }
    // EQ-REC-ALPHA-N2: alpha = rho / (<r, A r> - gamma rho), <r, A r> = z_s rho - w
    const cplx den = csub(csub(cmul(S->zs, rho), w), cmul(gamma, rho));
    S->w = w;
    if (xabs(rho) < 1e-300 || xabs(den) < 1e-300) {   // R12
        S->status = ST_BREAKDOWN;
        return;
    }
    const cplx alpha = xdiv(rho, den);
    const cplx c = cmul(alpha, gamma);
    S->alpha = alpha;
    S->beta = beta;
    S->c = c;
    S->sr_it = sr;
    const cplx c1 = cadd(mk(1.0, 0.0), c);
    S->a_cur = cmul(csub(c1, cmul(alpha, S->zs)), sr);   // EQ-CG-RN-3REC with A r = z_s r - q
    S->a_q = cmul(alpha, sr);
    S->a_prev = cmul(mk(-c.x, -c.y), S->sr_prev);
    S->sr_prev = sr;
    S->sr_cur = mk(1.0, 0.0);
    S->alpha_prev = alpha;
    S->rho_prev = rho;
    S->n_started = n + 1;
    S->pending = 1;
    S->nspmv += bicg ? 2 : 1;
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

// Projected update of every active shift (a4 + a6); writes pi_{n+1}.  All threads call it.
static __device__ void shift_step(const KParams &kp) {
    const DevState *S = kp.st;
    const int64_t n = S->n;
    const int nz = kp.nz, nl = kp.nl;
    const cplx *cur = kp.pibuf + (size_t)(n % 3) * nz;
    const cplx *prv = kp.pibuf + (size_t)((n + 2) % 3) * nz;
    cplx *nxt = kp.pibuf + (size_t)((n + 1) % 3) * nz;
    const cplx alpha = S->alpha, beta = S->beta, c = S->c, zs = S->zs;
    const int nact = *kp.n_act;
    for (int j = threadIdx.x; j < nact; j += blockDim.x) {
        const int k = kp.act_list[j];
        const ShiftCoef sc = shift_coef(cur[k], prv[k], kp.z[k], zs, alpha, beta, c, n);
        for (int l = 0; l < nl; ++l) {                                // P:L372-376 (R1)
            const int64_t o = (int64_t)k * nl + l;
            const cplx uu = cadd(cmul(kp.g[l], sc.ipik), cmul(sc.bk, kp.u[o]));
            kp.u[o] = uu;
            kp.y[o] = cfma(sc.ak, uu, kp.y[o]);
        }
        nxt[k] = sc.pin;
    }
}

}  // namespace sk
