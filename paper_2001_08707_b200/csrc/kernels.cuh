// kernels.cuh — launch wrappers of the hot-path kernels (spmv.cu, update.cu, scalar.cu).
#pragma once
#include <mutex>
#include <utility>

#include "common.cuh"

namespace sk {

// Programmatic dependent launch (PDL): the SpMV and update kernels of the iteration loop are
// launched with programmatic stream serialization, so a kernel's CTAs are dispatched while its
// predecessor drains; each such kernel's first instruction is griddepcontrol.wait, which
// returns once the predecessor has completed and its writes are visible — the data order is
// unchanged, only the launch latency is hidden.  SHIFTK_PDL=0 disables it.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kernel)(KArgs...), int grid, int block, size_t smem, cudaStream_t s,
                     bool pdl, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (pdl && pdl_enabled()) ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Per-device one-time setup (cudaFuncSetAttribute, __device__ tables): both are per device, so a
// process that drives several GPUs must run it on each — keyed by the current device.
struct PerDevice {
    std::mutex mu;
    uint64_t done = 0;   // bit d: done on device d (d < 64)
};
template <typename F>
cudaError_t once_per_device(PerDevice &pd, F &&f) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> g(pd.mu);
    if ((pd.done >> dev) & 1ull) return cudaSuccess;
    e = f();
    if (e == cudaSuccess) pd.done |= 1ull << dev;
    return e;
}

constexpr int kThreads = 256;          // streaming kernels
constexpr int kScalarThreads = 1024;   // the single-CTA init / finish kernel
// partial-slot capacities (arena sizes); grids are sized from sm_count() and capped by these
constexpr int kMaxSms = 192;
constexpr int kMaxBlocks = kMaxSms * 8;      // grid cap for grid-stride streaming kernels
constexpr int kMaxSpmvBlocks = kMaxSms * 32; // grid cap (= partial slots) of the SpMV kernels
// w = <r, q> is reduced in a fixed order whatever CTA takes a tile: one partial per tile; up to
// kStreamDirect tiles the seed CTA sums them all, beyond that the CTA completing a group of
// kStreamGroup tiles sums the group (partials [ntiles, ntiles + ngroups) of part_w).
constexpr int kStreamDirect = 4096;
constexpr int kStreamGroup = 1024;
inline __host__ __device__ int64_t stream_partials(int64_t ntiles) {
    return ntiles <= kStreamDirect ? ntiles : ntiles + (ntiles + kStreamGroup - 1) / kStreamGroup;
}
constexpr int kTileBits = 10;          // Heisenberg tile: 2^10 states per CTA
#ifndef TILED_SPLIT_MINB
#define TILED_SPLIT_MINB 4   // resident CTAs per SM of the bond-split tiled kernel (register cap and grid)
#endif

int stream_blocks(int64_t M);
// worker CTAs (= partials) of the Heisenberg SpMV; split: the SpMV of a bond-split solver (H_A)
int heisenberg_blocks(int L, int64_t M, int bicg, bool split = false);
int sz_blocks(int L, int64_t M, int bicg);
int64_t sz_partials(int L);                          // w partials of the sector SpMV (0: per CTA)                     // worker CTAs of the sector SpMV
bool heis_stream(int L, int64_t M, int bicg, bool split = false);   // the TMA-fed streaming kernel is used
bool heis_pairs(int L, int64_t M);                 // ... as tile pairs across the top spin bit (one GPU)
int sm_count();                                  // SMs of the current device
int csr_blocks(int64_t M);                      // worker CTAs (= partials) of the CSR SpMV
int update_blocks(int64_t M, int nl, int full, int nz); // worker CTAs (= partials) of the update
int shift_agents(int nz);                        // shift-agent CTAs of the update

// SpMV q = H r (and qt = H t for BiCG) with the fused partial dot w = <tv, q>.
// Solver mode (st != null): CTA 0 runs the finish step, the last CTA the seed step.
// Standalone mode (st == null, sk_apply_operator): r[0] -> q, no partials.
struct SpmvArgs {
    const DevState *st;
    const cplx *r[3];
    const cplx *t[3];
    cplx *q, *qt;
    cplx *part_w;
    unsigned long long *work;   // [2] tile queue of the streaming Heisenberg SpMV (zero between launches)
    uint32_t *grp;              // [ngroups] tile-group completion counters of the streaming SpMV
    int64_t M;
    int bicg;
};
cudaError_t launch_heisenberg(const SpmvArgs &a, const KParams &kp, int L, double J, cudaStream_t s);
cudaError_t launch_heisenberg_sz(const SpmvArgs &a, const KParams &kp, int L, int nup, double J, cudaStream_t s);
// tiled Heisenberg SpMV by chain length: a 11..16, b 17..22, c 23..28, d 29..34 (spmv_tiled_*.cu)
cudaError_t launch_tiled_a(int L, const SpmvArgs &a, const KParams &kp, double J, int grid, cudaStream_t s);
cudaError_t launch_tiled_b(int L, const SpmvArgs &a, const KParams &kp, double J, int grid, cudaStream_t s);
cudaError_t launch_tiled_c(int L, const SpmvArgs &a, const KParams &kp, double J, int grid, cudaStream_t s);
cudaError_t launch_tiled_d(int L, const SpmvArgs &a, const KParams &kp, double J, int grid, cudaStream_t s);
cudaError_t launch_csr(const SpmvArgs &a, const KParams &kp, const int64_t *row_ptr, const int32_t *col,
                       const void *val, bool cplx_val, double avg_nnz, cudaStream_t s);
// Column-blocked CSR passes (spmv.cu): split points + qualification statistics, block size, switch.
cudaError_t launch_csr_split(int64_t M, const int64_t *rp, const int32_t *col, int nblk, int bshift,
                             uint8_t *split, unsigned long long *stats, cudaStream_t s);
int csr_block_shift();
int csr_blocked_env();   // -1: automatic, 0: off, 1: forced where the rows qualify
// Reverse communication: a.q holds the caller's q = H r.
cudaError_t launch_rc_dot(const SpmvArgs &a, const KParams &kp, cudaStream_t s);

// r_0 = b, t_0 = conj(b); partials of rho_0, nu_0, g_0 into part_u.
cudaError_t launch_init(const KParams &kp, const cplx *b, cudaStream_t s);

// Fused three-term update (+ shadow) + next-iteration dots + (full mode) all-shift x/p update;
// CTA 0 runs the per-shift recurrences.
cudaError_t launch_update(const KParams &kp, const cplx *q, const cplx *qt, cudaStream_t s);

// Bond split (update_split.cu): AHI = L - 8 when the split applies to this
// context (one GPU, Heisenberg chain, COCG, N_left = 1, streaming SpMV), else 0; the update then
// applies H_B and writes the w_B partials; launch_split_init writes those of r_0.
int split_ahi_for(int L, int64_t M, int world, int bicg, int full, int nl, int kind_heisenberg);
int split_blocks();
int split_lo_bonds();   // in-piece bonds (0,1).. moved from H_A to H_B (0: none)
cudaError_t launch_update_split(const KParams &kp, const cplx *q, cudaStream_t s);
cudaError_t launch_split_init(const KParams &kp, cudaStream_t s);
int split_fuse_enabled();        // SHIFTK_SPLIT_FUSE (default 1): the H_A SpMV folds -kappa r_{n-1} into q
int split_left_real_enabled();   // SHIFTK_LEFT_REAL (default 1): a real left vector is kept as Re a in B-tile order
cudaError_t launch_split_left(const KParams &kp, double *out, uint32_t *any_imag, cudaStream_t s);

// Single-CTA steps outside the iteration: INIT (after launch_init) and FINISH (residuals,
// retirement, switch of a pending iteration).
enum : int { PH_INIT = 1, PH_FINISH = 2 };
cudaError_t launch_scalar(const KParams &kp, int phase, cudaStream_t s);

// Recalculation at new shifts from the coefficient log (y, u: device [nnew][nl], res [nnew]).
cudaError_t launch_recalc(const KParams &kp, int64_t nlog, const cplx *znew, int nnew, double tol,
                          double nu0, cplx *y, cplx *u, double *res, cudaStream_t s);

// ---- multi-rank (world > 1) -----------------------------------------------------------------
constexpr int kMaxWorld = 64;
struct LoopbackPtrs {
    const cplx *src[kMaxWorld];
    cplx *dst[kMaxWorld];
};
cudaError_t launch_seed(const KParams &kp, cudaStream_t s);            // seed step on wsum
cudaError_t launch_reduce_local(const KParams &kp, cudaStream_t s);    // init partials -> uloc
cudaError_t launch_loopback_allreduce(const LoopbackPtrs &p, int world, int n, cudaStream_t s);

}  // namespace sk
