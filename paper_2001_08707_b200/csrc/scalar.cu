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
        reduce_columns(kp.part_u, kp.nblk_upd, 2 + kp.nl, 2 + kp.nl, sc);   // (barriers publish)
        const double nu = sqrt(sc.col[1].x);
        for (int k = threadIdx.x; k < kp.nz; k += blockDim.x) kp.res[k] = nu;
        if (threadIdx.x < kp.nl) kp.g[threadIdx.x] = sc.col[2 + threadIdx.x];
        if (threadIdx.x == 0) {
            sc.S.rho_cur = sc.col[0];
            sc.S.nu = nu;
            sc.S.n_active = kp.nz;
            sc.S.lz_pending = 0;
            sc.S.lz_iter = -1;
            sc.S.bscale[0] = sc.S.bscale[1] = sc.S.bscale[2] = mk(1.0, 0.0);
        }
        state_store(kp.st, sc.S);
        return;
    }
    // FINISH: only when an iteration is pending (the state is read through L2)
    const int pending = __ldcg(&kp.st->pending);
    if (pending) finish_step(kp, sc, /*eager=*/true);
}

cudaError_t launch_scalar(const KParams &kp, int phase, cudaStream_t s) {
    scalar_kernel<<<1, kThreads, 0, s>>>(kp, phase);
    return cudaGetLastError();
}

}  // namespace sk
