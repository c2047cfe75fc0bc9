// kernels.cuh — launch wrappers of the hot-path kernels (implemented in kernels.cu).
#pragma once
#include "common.cuh"

namespace sk {

constexpr int kThreads = 256;          // streaming kernels
constexpr int kScalarThreads = 1024;   // the single-CTA scalar kernel
constexpr int kMaxBlocks = 148 * 8;    // grid cap for grid-stride streaming kernels

// Scalar-kernel phases.
enum : int { PH_INIT = 1, PH_FINISH = 2, PH_START = 4 };

constexpr int kTileBitsPublic = 10;  // Heisenberg tile: 2^10 states per CTA
int stream_blocks(int64_t M);
int heisenberg_blocks(int L, int64_t M);   // grid (and partial count) of the Heisenberg SpMV

// SpMV q = H r (and qt = H t for BiCG) with the fused partial dot w = <tv, q>.
// When `st` is null the kernel runs standalone on r0/t0 (sk_apply_operator) without partials.
struct SpmvArgs {
    const DevState *st;
    const cplx *r[3];
    const cplx *t[3];
    cplx *q, *qt;
    cplx *part_w;
    int64_t M;
    int bicg;
};
cudaError_t launch_heisenberg(const SpmvArgs &a, int L, double J, int nblk, cudaStream_t s);
cudaError_t launch_csr(const SpmvArgs &a, const int64_t *row_ptr, const int32_t *col,
                       const void *val, bool cplx_val, double avg_nnz, int nblk, cudaStream_t s);

// Reverse-communication dot: part_w = <tv, q> on caller-supplied q (and qt ignored).
cudaError_t launch_rc_dot(const KParams &kp, const cplx *q, cudaStream_t s);

// r_0 = b, t_0 = conj(b); partials of rho_0, nu_0, g_0 into part_u.
cudaError_t launch_init(const KParams &kp, const cplx *b, cudaStream_t s);

// Fused three-term update (+ shadow) + next-iteration dots + (full mode) all-shift x/p update.
cudaError_t launch_update(const KParams &kp, const cplx *q, const cplx *qt, cudaStream_t s);

// Single-CTA scalar step (reductions of partials, recurrences, retirement, seed switch).
cudaError_t launch_scalar(const KParams &kp, int phases, cudaStream_t s);

}  // namespace sk
