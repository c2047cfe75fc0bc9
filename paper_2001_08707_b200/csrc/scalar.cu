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

// ---------------------------------------------------------------- multi-rank (world > 1)
// Seed step on the all-reduced w (the single-GPU path runs it in the SpMV's last CTA).
__global__ void __launch_bounds__(kThreads) seed_kernel(KParams kp) {
    __shared__ StepScratch sc;
    state_load_nosync(sc.S, kp.st);
    __syncthreads();
    if (threadIdx.x == 0 && sc.S.status == ST_ITERATING) seed_step(&sc.S, __ldcg(kp.wsum), kp.bicg);
    __syncthreads();
    if (sc.S.status == ST_BREAKDOWN && sc.S.lz_pending) retire_pass(kp, sc);
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
