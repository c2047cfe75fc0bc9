// scalar.cu — the per-iteration scalar step as ONE CTA.
//
// Latency design (the step is a few microseconds of dependent work on one SM):
//   * the per-shift arrays (pi, pi_old, z, u, y, res, active, retired_at) are staged into shared
//     memory with TMA bulk copies (cp.async.bulk, one elected thread, mbarrier completion) and
//     written back with bulk stores — a single DRAM round trip in each direction;
//   * the CTA partials of the SpMV / update kernels are reduced while the bulk copies fly;
//   * the code is kept compact (complex division / modulus are out-of-line helpers) because a
//     kernel executed by a single CTA pays an instruction-cache miss for every 128 bytes of
//     straight-line code (profiled: 26% `no_instructions` stalls with inlined arithmetic).
//
//   FINISH (of iteration n, after its update kernel):  rho_{n+1}, nu = ||r_{n+1}||, g = P r_{n+1}
//     from the update partials; res_k = nu/|pi_{n+1}^k| (EQ-COLLINEAR P:L300); retire
//     res_k < tol (R8); seed switch to argmin_active |pi| (R9-R11).
//   START (of iteration n+1, after its SpMV):  w from the SpMV partials; beta, gamma, alpha, c
//     (P:L262); per active shift pi_{n+1}, alpha^k, beta^k and the
//     projected u, y update (R1); full-mode coefficients for the update kernel.
#include "kernels.cuh"

namespace sk {

namespace {
enum { ST_ITERATING = 0, ST_CONVERGED = 1, ST_MAXITER = 2, ST_BREAKDOWN = 3 };
constexpr int NT = kScalarThreads;
constexpr int NW = NT / 32;
constexpr int kMaxCols = 40;   // 2 + nl (<= 34) update columns + 1 SpMV column

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

struct Layout {
    size_t pi, pio, z, u, y, res, ret, act, alist, total;
};

__host__ __device__ inline Layout layout(int nz, int nl) {
    Layout L{};
    size_t o = 0;
    L.pi = o;    o += al16(sizeof(cplx) * nz);
    L.pio = o;   o += al16(sizeof(cplx) * nz);
    L.z = o;     o += al16(sizeof(cplx) * nz);
    L.u = o;     o += al16(sizeof(cplx) * (size_t)nz * nl);
    L.y = o;     o += al16(sizeof(cplx) * (size_t)nz * nl);
    L.res = o;   o += al16(sizeof(double) * nz);
    L.ret = o;   o += al16(sizeof(int64_t) * nz);
    L.act = o;   o += al16(nz);
    L.alist = o; o += al16(sizeof(int32_t) * nz);
    L.total = o;
    return L;
}

struct Shared {
    DevState S;
    unsigned long long mbar;
    cplx wsum[NW];
    cplx col[kMaxCols];     // reduced partial columns
    cplx g[64];             // projections of the current r
    cplx bc[4];
    double redd[NW];
    int redi[NW], redc[NW];
    int bci[4];
};

// ---- out-of-line complex helpers (code size matters more than call overhead here) --------
// 1/b with a scaling by max(|re|,|im|) so that |b|^2 neither overflows nor underflows.
__device__ __noinline__ cplx xrecip(cplx b) {
    const double s = fmax(fabs(b.x), fabs(b.y));
    const double is = 1.0 / s;
    const double xr = b.x * is, xi = b.y * is;
    const double d = is / (xr * xr + xi * xi);
    return mk(xr * d, -xi * d);
}
__device__ __noinline__ cplx xdiv(cplx a, cplx b) { return cmul(a, xrecip(b)); }
__device__ __noinline__ double xabs(cplx b) {
    const double s = fmax(fabs(b.x), fabs(b.y));
    if (s == 0.0) return 0.0;
    const double xr = b.x / s, xi = b.y / s;
    return s * sqrt(xr * xr + xi * xi);
}

// ---- TMA bulk copies (1-D, no tensor map): global <-> shared ---------------------------------
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(mbar)) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(dst), "r"(smem_u32(src)), "r"(bytes) : "memory");
}
}  // namespace

__global__ void __launch_bounds__(NT) scalar_kernel(KParams kp, int phases, int use_smem) {
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ Shared sh;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nz = kp.nz, nl = kp.nl, nred = 2 + nl;
    const Layout LY = layout(nz, nl);
    dbg_stamp(kp.dbg_ts, 0);

    // ---------------------------------------------------------------- prologue: one load wave
    cplx *pi = kp.pi, *pio = kp.pi_old, *u = kp.u, *y = kp.y;
    const cplx *z = kp.z;
    double *res = kp.res;
    int64_t *ret = kp.retired_at;
    uint8_t *act = kp.active;
    int32_t *alist = kp.act_list;
    if (use_smem) {
        pi = (cplx *)(dsm + LY.pi);
        pio = (cplx *)(dsm + LY.pio);
        z = (const cplx *)(dsm + LY.z);
        u = (cplx *)(dsm + LY.u);
        y = (cplx *)(dsm + LY.y);
        res = (double *)(dsm + LY.res);
        ret = (int64_t *)(dsm + LY.ret);
        act = (uint8_t *)(dsm + LY.act);
        alist = (int32_t *)(dsm + LY.alist);
        if (tid == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&sh.mbar)));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();   // the barrier is initialised before anyone waits on it
        if (tid == 0) {
            const unsigned mb = smem_u32(&sh.mbar);
            const unsigned bytes = (unsigned)(LY.alist);   // everything before alist
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(mb), "r"(bytes) : "memory");
            bulk_g2s(pi, kp.pi, (unsigned)(LY.pio - LY.pi), &sh.mbar);
            bulk_g2s(pio, kp.pi_old, (unsigned)(LY.z - LY.pio), &sh.mbar);
            bulk_g2s((void *)z, kp.z, (unsigned)(LY.u - LY.z), &sh.mbar);
            bulk_g2s(u, kp.u, (unsigned)(LY.y - LY.u), &sh.mbar);
            bulk_g2s(y, kp.y, (unsigned)(LY.res - LY.y), &sh.mbar);
            bulk_g2s(res, kp.res, (unsigned)(LY.ret - LY.res), &sh.mbar);
            bulk_g2s(ret, kp.retired_at, (unsigned)(LY.act - LY.ret), &sh.mbar);
            bulk_g2s(act, kp.active, (unsigned)(LY.alist - LY.act), &sh.mbar);
        }
    }
    if (tid < (int)(sizeof(DevState) / 8)) ((int64_t *)&sh.S)[tid] = ((const int64_t *)kp.st)[tid];
    if (tid < nl) sh.g[tid] = kp.g[tid];
    // partial columns (update: INIT/FINISH; SpMV: START), one warp per column, fixed order
    const bool want_u = (phases & (PH_INIT | PH_FINISH)) != 0;
    const bool want_w = (phases & PH_START) != 0;
    const int ncol = (want_u ? nred : 0) + (want_w ? 1 : 0);
    for (int c = warp; c < ncol; c += NW) {
        const bool isu = want_u && c < nred;
        const cplx *part = isu ? kp.part_u : kp.part_w;
        const int nb = isu ? kp.nblk_upd : kp.nblk_spmv, stride = isu ? nred : 1, j = isu ? c : 0;
        cplx s0 = mk(0, 0), s1 = mk(0, 0), s2 = mk(0, 0), s3 = mk(0, 0);
        int b = lane;
        for (; b + 96 < nb; b += 128) {   // four independent loads in flight per lane
            const cplx v0 = part[(int64_t)b * stride + j], v1 = part[(int64_t)(b + 32) * stride + j];
            const cplx v2 = part[(int64_t)(b + 64) * stride + j], v3 = part[(int64_t)(b + 96) * stride + j];
            s0 = cadd(s0, v0); s1 = cadd(s1, v1); s2 = cadd(s2, v2); s3 = cadd(s3, v3);
        }
        for (; b < nb; b += 32) s0 = cadd(s0, part[(int64_t)b * stride + j]);
        const cplx v = warp_sum(cadd(cadd(s0, s1), cadd(s2, s3)));
        if (lane == 0) sh.col[c] = v;
    }
    if (use_smem) {   // wait for the bulk copies (phase 0 of the mbarrier)
        const unsigned mb = smem_u32(&sh.mbar);
        unsigned done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(mb) : "memory");
    }
    __syncthreads();
    DevState &S = sh.S;

    if (phases & PH_INIT) {
        const double nu = sqrt(sh.col[1].x);
        for (int k = tid; k < nz; k += NT) res[k] = nu;
        if (tid < nl) sh.g[tid] = sh.col[2 + tid];
        if (tid == 0) { S.rho_cur = sh.col[0]; S.nu = nu; }
        __syncthreads();
    }

    dbg_stamp(kp.dbg_ts, 1);
    // ---------------------------------------------------------------- FINISH(n)
    if ((phases & PH_FINISH) && S.pending) {
        cplx rho = sh.col[0];
        double nu = sqrt(sh.col[1].x);
        const int64_t n = S.n + 1;
        const double tol = S.tol;
        int cnt = 0, bi = -1;
        double best = 0.0;
        for (int k = tid; k < nz; k += NT) {
            if (!act[k]) continue;
            const double a = xabs(pi[k]);
            const double rk = nu / a;
            res[k] = rk;
            if (rk < tol) { act[k] = 0; ret[k] = n; continue; }
            ++cnt;
            if (bi < 0 || a < best) { best = a; bi = k; }   // ascending k: ties keep lowest
        }
        // combined block reduction: active count + argmin (lowest index on ties)
        for (int o = 16; o > 0; o >>= 1) {
            cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
            const double ov = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (oi >= 0 && (bi < 0 || ov < best || (ov == best && oi < bi))) { best = ov; bi = oi; }
        }
        if (lane == 0) { sh.redc[warp] = cnt; sh.redd[warp] = best; sh.redi[warp] = bi; }
        __syncthreads();
        if (tid == 0) {
            int c = 0, i = -1;
            double bb = 0.0;
            for (int w = 0; w < NW; ++w) {
                c += sh.redc[w];
                const int oi = sh.redi[w];
                const double ov = sh.redd[w];
                if (oi >= 0 && (i < 0 || ov < bb || (ov == bb && oi < i))) { bb = ov; i = oi; }
            }
            sh.bci[0] = c;
            sh.bci[1] = i;
            const bool sw = c > 0 && !(kp.flags & 1) && i != S.seed;
            sh.bci[2] = sw;
            if (sw) {   // R9: the new seed's r, r_prev, alpha, rho in its own normalisation
                const cplx f = pi[i], fp = pio[i];
                const cplx rf = xrecip(f), rfp = xrecip(fp);
                sh.bc[0] = rf;
                sh.bc[1] = rfp;
                S.sr_cur = cmul(S.sr_cur, rf);                        // r_{n+1} /= f
                S.sr_prev = cmul(S.sr_prev, rfp);                     // r_n /= f'
                S.alpha_prev = cmul(S.alpha_prev, cmul(fp, rf));      // alpha_n^{s*}
                S.rho_prev = cmul(S.rho_prev, cmul(rfp, rfp));        // rho_n / f'^2
                rho = cmul(rho, cmul(rf, rf));                        // rho_{n+1} / f^2
                nu = nu / xabs(f);
                S.zs = z[i];
                S.seed = i;
                S.nswitch += 1;
            }
            S.rho_cur = rho;
            S.nu = nu;
            S.n = n;
            S.pending = 0;
            S.n_active = c;
            if (c == 0) S.status = ST_CONVERGED;
            else if (n >= S.itermax) S.status = ST_MAXITER;
        }
        __syncthreads();
        const bool sw = sh.bci[2];
        if (sw) {
            const cplx rf = sh.bc[0], rfp = sh.bc[1];
            for (int k = tid; k < nz; k += NT) {
                if (!act[k]) continue;   // retired shifts are not rescaled (R13)
                pi[k] = cmul(pi[k], rf);
                pio[k] = cmul(pio[k], rfp);
            }
        }
        if (tid < nl) sh.g[tid] = sw ? cmul(sh.col[2 + tid], sh.bc[0]) : sh.col[2 + tid];
        __syncthreads();
    }

    dbg_stamp(kp.dbg_ts, 2);
    // ---------------------------------------------------------------- START(n)
    if ((phases & PH_START) && S.status == ST_ITERATING) {
        if (tid == 0) {
            const cplx sr = S.sr_cur;
            const cplx w = cmul(cmul(sr, sr), sh.col[ncol - 1]);   // true-scale w_n
            const cplx rho = S.rho_cur;
            cplx beta = mk(0, 0), gamma = mk(0, 0);
            if (S.n > 0) {
                beta = xdiv(rho, S.rho_prev);          // EQ-REC-BETA P:L262
                gamma = xdiv(beta, S.alpha_prev);
            }
            // EQ-REC-ALPHA-N2: alpha = rho / (<r, A r> - gamma rho), <r, A r> = z_s rho - w
            const cplx den = csub(csub(cmul(S.zs, rho), w), cmul(gamma, rho));
            const int brk = (xabs(rho) < 1e-300) || (xabs(den) < 1e-300);
            cplx alpha = mk(0, 0), c = mk(0, 0);
            if (!brk) {
                alpha = xdiv(rho, den);
                c = cmul(alpha, gamma);
            }
            sh.bc[0] = alpha; sh.bc[1] = beta; sh.bc[2] = c;
            sh.bci[2] = brk;
            S.alpha = alpha; S.beta = beta; S.w = w;
            if (brk) S.status = ST_BREAKDOWN;
        }
        __syncthreads();
        dbg_stamp(kp.dbg_ts, 5);
        if (!sh.bci[2]) {
            const cplx alpha = sh.bc[0], beta = sh.bc[1], c = sh.bc[2];
            const cplx zs = S.zs, sr = S.sr_cur;
            const int64_t n = S.n;
            // compacted active list, ascending k (the full-mode update streams only these)
            int nact = 0;
            for (int base = 0; base < nz; base += NT) {
                const int k = base + tid;
                const int a = (k < nz) ? (int)act[k] : 0;
                const unsigned bal = __ballot_sync(0xffffffffu, a);
                if (lane == 0) sh.redi[warp] = __popc(bal);
                __syncthreads();
                if (tid == 0) {
                    int acc = 0;
                    for (int w = 0; w < NW; ++w) { const int v = sh.redi[w]; sh.redi[w] = acc; acc += v; }
                    sh.bci[3] = acc;
                }
                __syncthreads();
                if (a) alist[nact + sh.redi[warp] + __popc(bal & ((1u << lane) - 1u))] = k;
                nact += sh.bci[3];
                __syncthreads();
            }
            dbg_stamp(kp.dbg_ts, 6);
            const cplx c1 = cadd(mk(1.0, 0.0), c);
            for (int j = tid; j < nact; j += NT) {
                const int k = alist[j];
                const cplx pik = pi[k], piok = pio[k];
                // EQ-SHIFTEDCG-PI: pi_{n+1} = (1 + c + alpha sigma) pi_n - c pi_{n-1}
                const cplx sigma = csub(z[k], zs);
                const cplx pin = csub(cmul(cadd(c1, cmul(alpha, sigma)), pik), cmul(c, piok));
                const cplx ipik = xrecip(pik);
                const cplx ak = cmul(xdiv(pik, pin), alpha);
                cplx bk = mk(0, 0);
                if (n > 0) { const cplx rat = cmul(piok, ipik); bk = cmul(cmul(rat, rat), beta); }
                for (int l = 0; l < nl; ++l) {                                // P:L372-376 (R1)
                    const int64_t o = (int64_t)k * nl + l;
                    const cplx uu = cadd(cmul(sh.g[l], ipik), cmul(bk, u[o]));
                    u[o] = uu;
                    y[o] = cfma(ak, uu, y[o]);
                }
                pio[k] = pik;
                pi[k] = pin;
                if (kp.full) {
                    kp.coef[3 * j] = cmul(sr, ipik);   // p^k = r_n/pi_n^k + ...  (r_n = sr r_stored)
                    kp.coef[3 * j + 1] = bk;
                    kp.coef[3 * j + 2] = ak;
                }
            }
            if (tid == 0) {
                *kp.n_act_list = nact;
                S.a_cur = cmul(csub(c1, cmul(alpha, zs)), sr);
                S.a_q = cmul(alpha, sr);
                S.a_prev = cmul(mk(-c.x, -c.y), S.sr_prev);
                S.sr_prev = sr;
                S.sr_cur = mk(1.0, 0.0);
                S.alpha_prev = alpha;
                S.rho_prev = S.rho_cur;
                S.n_started = n + 1;
                S.pending = 1;
                S.nspmv += kp.bicg ? 2 : 1;
            }
        }
    }

    dbg_stamp(kp.dbg_ts, 3);
    // ---------------------------------------------------------------- epilogue: write back
    if (use_smem) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid < (int)(sizeof(DevState) / 8)) ((int64_t *)kp.st)[tid] = ((const int64_t *)&sh.S)[tid];
    if (tid < nl) kp.g[tid] = sh.g[tid];
    if (use_smem && tid == 0) {
        bulk_s2g(kp.pi, pi, (unsigned)(LY.pio - LY.pi));
        bulk_s2g(kp.pi_old, pio, (unsigned)(LY.z - LY.pio));
        bulk_s2g(kp.u, u, (unsigned)(LY.y - LY.u));
        bulk_s2g(kp.y, y, (unsigned)(LY.res - LY.y));
        bulk_s2g(kp.res, res, (unsigned)(LY.ret - LY.res));
        bulk_s2g(kp.retired_at, ret, (unsigned)(LY.act - LY.ret));
        bulk_s2g(kp.active, act, (unsigned)(LY.alist - LY.act));
        bulk_s2g(kp.act_list, alist, (unsigned)(LY.total - LY.alist));
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    dbg_stamp(kp.dbg_ts, 4);
}

static_assert(sizeof(DevState) % 8 == 0, "DevState is copied as int64 words");
static_assert(sizeof(DevState) / 8 <= NT, "DevState copy uses one word per thread");

size_t scalar_smem_bytes(int nz, int nl) { return layout(nz, nl).total; }

cudaError_t launch_scalar(const KParams &kp, int phases, cudaStream_t s) {
    const size_t need = scalar_smem_bytes(kp.nz, kp.nl);
    const int use_smem = need <= 200 * 1024;
    const size_t shm = use_smem ? need : 0;
    static size_t configured = 0;   // max dynamic smem requested so far
    if (shm > configured) {
        cudaError_t e = cudaFuncSetAttribute(scalar_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
        if (e != cudaSuccess) return e;
        configured = shm;
    }
    scalar_kernel<<<1, NT, shm, s>>>(kp, phases, use_smem);
    return cudaGetLastError();
}

}  // namespace sk
