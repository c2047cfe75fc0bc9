// scalar.cu — single-CTA steps outside the per-iteration kernels:
//   INIT   : rho_0, ||b||, g_0 = P b from the init partials; res_k = ||b|| (pi_0 = 1, SPEC
//            S:L181); the compacted active list (all shifts).
//   FINISH : residuals / retirement / seed switch of a pending iteration (steps.cuh
//            finish_step) when no further SpMV launch will carry it (sk_update, end of sk_run,
//            getters).
#include "kernels.cuh"
#include "steps.cuh"

namespace sk {

__global__ void __launch_bounds__(kThreads) scalar_kernel(KParams kp, int phase) {
    __shared__ StepScratch sc;
    if (phase == PH_INIT) {
        state_load_nosync(sc.S, kp.st);
        if (kp.usum) reduce_columns(kp.usum, 1, 2 + kp.nl, 2 + kp.nl, sc);   // all-reduced
        else reduce_columns(kp.part_u, kp.nblk_upd, 2 + kp.nl, 2 + kp.nl, sc);   // (barriers publish)
        const double nu = sqrt(sc.col[1].x);
        for (int k = threadIdx.x; k < kp.nz; k += blockDim.x) kp.res[k] = nu;
        if (threadIdx.x < kp.nl) {
            kp.g[threadIdx.x] = sc.col[2 + threadIdx.x];
            if (kp.lg_cap > 0) kp.lg_g[threadIdx.x] = sc.col[2 + threadIdx.x];   // P r_0
        }
        if (threadIdx.x == 0) {
            sc.S.rho_cur = sc.col[0];
            seed_prepare(&sc.S);
            sc.S.nu = nu;
            sc.S.n_active = kp.nz;
            sc.S.lz_pending = 0;
            sc.S.lz_iter = -1;
            sc.S.bscale[0] = sc.S.bscale[1] = sc.S.bscale[2] = mk(1.0, 0.0);
        }
        state_store(kp.st, sc.S);
        return;
    }
    // FINISH: of a pending iteration; or, after a breakdown in the seed step, the retirement
    // test that the finish of the previous iteration left pending (the state is read via L2)
    const int pending = __ldcg(&kp.st->pending);
    if (pending) {
        agent_finish(kp, sc, /*eager=*/true);
    } else if (__ldcg(&kp.st->status) == ST_BREAKDOWN && __ldcg(&kp.st->lz_pending)) {
        state_load_nosync(sc.S, kp.st);
        __syncthreads();
        retire_pass(kp, sc);
        state_store(kp.st, sc.S);
    }
}

cudaError_t launch_scalar(const KParams &kp, int phase, cudaStream_t s) {
    scalar_kernel<<<1, kThreads, 0, s>>>(kp, phase);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- recalculation
// Projections at new shifts from the coefficient log: the per-shift recurrences
// (a4, a6) and the residual test (a8) replayed with the logged seed scalars, seed shifts,
// P r_n and switch factors — one thread per new shift, no operator application.
__global__ void recalc_kernel(KParams kp, int64_t nlog, const cplx *__restrict__ znew, int nnew,
                              double tol, double nu0, cplx *__restrict__ y, cplx *__restrict__ u,
                              double *__restrict__ res) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nnew) return;
    const int nl = kp.nl;
    const cplx z = znew[j];
    cplx pi = mk(1, 0), pio = mk(1, 0);
    double rj = nu0;
    for (int l = 0; l < nl; ++l) { u[(int64_t)j * nl + l] = mk(0, 0); y[(int64_t)j * nl + l] = mk(0, 0); }
    for (int64_t n = 0; n < nlog; ++n) {
        const cplx *e = kp.lg + 6 * n;
        const ShiftCoef sc = shift_coef(pi, pio, z, e[3], e[0], e[1], e[2], n);
        for (int l = 0; l < nl; ++l) {
            const int64_t o = (int64_t)j * nl + l;
            const cplx uu = cadd(cmul(kp.lg_g[n * nl + l], sc.ipik), cmul(sc.bk, u[o]));
            u[o] = uu;
            y[o] = cfma(sc.ak, uu, y[o]);
        }
        pio = pi;
        pi = sc.pin;
        double r2;
        if (retire_test(kp.lg_nu[n], pi, tol, r2)) { rj = r2; break; }
        rj = r2;
        pi = cmul(pi, e[4]);
        pio = cmul(pio, e[5]);
    }
    res[j] = rj;
}

cudaError_t launch_recalc(const KParams &kp, int64_t nlog, const cplx *znew, int nnew, double tol,
                          double nu0, cplx *y, cplx *u, double *res, cudaStream_t s) {
    recalc_kernel<<<(nnew + 127) / 128, 128, 0, s>>>(kp, nlog, znew, nnew, tol, nu0, y, u, res);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- multi-rank (world > 1)
// Seed step on the all-reduced w (the single-GPU path runs it in the SpMV's last CTA).
__global__ void __launch_bounds__(kThreads) seed_kernel(KParams kp) {
    __shared__ StepScratch sc;
    state_load_nosync(sc.S, kp.st);
    __syncthreads();
    if (threadIdx.x == 0 && sc.S.status == ST_ITERATING) seed_step(&sc.S, __ldcg(kp.wsum), kp.bicg, kp);
    state_store(kp.st, sc.S);
}

cudaError_t launch_seed(const KParams &kp, cudaStream_t s) {
    seed_kernel<<<1, kThreads, 0, s>>>(kp);
    return cudaGetLastError();
}

// This rank's init partials -> uloc (before the all-reduce of sk_connect).
__global__ void __launch_bounds__(kThreads) reduce_local_kernel(KParams kp) {
    __shared__ RedScratch rs;
    reduce_columns(kp.part_u, kp.nblk_upd, 2 + kp.nl, 2 + kp.nl, rs);
    if (threadIdx.x < 2 + kp.nl) kp.uloc[threadIdx.x] = rs.col[threadIdx.x];
}

cudaError_t launch_reduce_local(const KParams &kp, cudaStream_t s) {
    reduce_local_kernel<<<1, kThreads, 0, s>>>(kp);
    return cudaGetLastError();
}

// Loopback all-reduce of a group living on one GPU: dst_g[j] = sum_{g' in rank order} src_g'[j]
// for every member g (identical on all members, deterministic).
__global__ void loopback_allreduce_kernel(LoopbackPtrs p, int world, int n) {
    const int j = threadIdx.x;
    if (j >= n) return;
    cplx s = p.src[0][j];
    for (int g = 1; g < world; ++g) s = cadd(s, p.src[g][j]);
    for (int g = 0; g < world; ++g) p.dst[g][j] = s;
}

cudaError_t launch_loopback_allreduce(const LoopbackPtrs &p, int world, int n, cudaStream_t s) {
    loopback_allreduce_kernel<<<1, 64, 0, s>>>(p, world, n);
    return cudaGetLastError();
}

}  // namespace sk
