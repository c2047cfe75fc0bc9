/*
 * shiftk.h — C-ABI of the B200 shifted-Krylov library (libshiftk.so).
 *
 * Solves the shifted linear equations  (z_k I - H) x^(k) = b,  k = 0..N_z-1   (EQ-SHIFT-EQ,
 * PAPER.md P:L136-138) for all shifts at once with the shifted COCG (App. A) or
 * shifted BiCG (App. B) method, and reports the projections
 * y[k][l] = a_l^dagger x^(k)  (EQ-GREEN-ELEM P:L101, EQ-SHIFTEDCG-y P:L372) and, in
 * full mode (P = I), the solution vectors x^(k) themselves.
 *
 * The call sequence follows the paper's library flow (Alg. 1):
 *     sk_init  ->  { sk_update | sk_update_rc | sk_run }*  ->  sk_get_*  ->  sk_finalize
 * with one difference: the library owns the operator H (Heisenberg bit-flip chain or CSR), so
 * sk_update performs the seed SpMV itself.  sk_update_rc keeps the paper's reverse-communication
 * form (caller supplies q = H r).
 *
 * Conventions (all entry points):
 *   - Return value: SK_OK (0) on success, a negative sk_error otherwise.  No exception or
 *     abort crosses the ABI.  Solver outcomes (converged / budget exhausted / breakdown) are NOT
 *     errors: they come back through the `status` out-parameter.
 *   - Complex numbers are sk_cplx {re, im} (binary-compatible with cuDoubleComplex / double2 /
 *     std::complex<double> / numpy complex128).  All arithmetic is IEEE fp64.
 *   - Vectors are dense, contiguous, element i = basis state / row i.  Multi-vector arrays are
 *     row-major [count][M] (each vector contiguous).
 *   - "device" pointers are CUDA device pointers on the context's device; "host" pointers are
 *     ordinary (pageable or pinned) host memory.  sk_mem tells which, where both are accepted.
 *   - Ownership: the library COPIES z, b and host-side left vectors at sk_init; it BORROWS
 *     device-side left vectors and CSR arrays, which must stay valid and unmodified until
 *     sk_finalize; it owns every internal buffer and never frees caller memory.
 *   - Streams: all device work is enqueued on the context's stream (sk_dist.stream, or one the
 *     library creates).  Functions returning host data synchronise that stream.
 *   - A context is used by one host thread at a time.
 */
#ifndef SHIFTK_H
#define SHIFTK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { double re, im; } sk_cplx;
typedef struct sk_ctx sk_ctx;

/* Table 1: COCG for complex-symmetric z I - H (real-symmetric H, complex z);
   BiCG otherwise (here: complex Hermitian H).  Readings: DESIGN.md R2. */
enum sk_method { SK_COCG = 0, SK_BICG = 1 };

enum sk_opkind {
    SK_OP_HEISENBERG = 0, /* S=1/2 chain H = J sum_i S_i.S_{i+1}, periodic, generated on
                             the fly ("matrix elements are internally generated") */
    SK_OP_CSR_REAL = 1,   /* real-symmetric CSR, fp64 values                                   */
    SK_OP_CSR_CPLX = 2,   /* complex Hermitian CSR, complex128 values                          */
    SK_OP_RC = 3,         /* no operator: reverse communication only (sk_update_rc)            */
    SK_OP_HEISENBERG_SZ = 4 /* the chain of SK_OP_HEISENBERG restricted to the sector of n_up up
                               spins (S^z conservation; HPhi's 2Sz sectors, dim 924
                               at L=12, n_up=6).  Rows: the L-bit states with popcount
                               n_up in ascending order (R28); M = C(L, n_up).  One GPU. */
};

/* Outcome of an iteration (returned through `status`, never as an error). */
enum sk_status {
    SK_ITERATING = 0,  /* call again                                                         */
    SK_CONVERGED = 1,  /* every shift has ||r^(k)||_2 < tol                         */
    SK_MAXITER = 2,    /* itermax iterations done                                             */
    SK_BREAKDOWN = 3   /* |rho_n| or |alpha denominator| < 1e-300 (R12)             */
};

enum sk_error {
    SK_OK = 0,
    SK_EINVAL = -1,        /* bad argument (null pointer, size, tol <= 0, ||b|| = 0, ...)    */
    SK_ENOMEM = -2,        /* device allocation failed                                        */
    SK_ECUDA = -3,         /* a CUDA call failed (message: sk_last_error())                   */
    SK_ENCCL = -4,         /* an NCCL call failed                                             */
    SK_ESTATE = -5,        /* wrong call order, or use after sk_finalize                      */
    SK_EUNSUPPORTED = -6   /* valid request this build does not support (e.g. COCG on a
                              complex Hermitian operator, which Table 1 rules out)           */
};

enum sk_mem { SK_MEM_HOST = 0, SK_MEM_DEVICE = 1 };

enum sk_flags {
    SK_FLAG_NO_SWITCH = 1,  /* disable seed switching; diagnostics only           */
    SK_FLAG_LOG = 2         /* keep the coefficient log {alpha_n, beta_n, z_s, P r_n, switch
                               factors, ||r_n||} for sk_recalc; itermax entries,
                               itermax <= 2^24                                                 */
};

/* The operator H.  For SK_OP_HEISENBERG only L and J are read (M = 2^L, basis state s = L-bit
   integer, bit i = site i, 1 = up; R16).  For CSR: this rank's rows
   [row_begin, row_begin + M_local) of the global M x M matrix, row_ptr[M_local + 1] (int64,
   row_ptr[0] = 0), col[nnz] (int32 GLOBAL column ids, ascending within a row),
   val[nnz] (double for SK_OP_CSR_REAL, sk_cplx for SK_OP_CSR_CPLX).  CSR arrays are DEVICE
   pointers, borrowed until sk_finalize. */
typedef struct {
    int32_t kind;        /* sk_opkind */
    int32_t L;           /* Heisenberg: number of sites, 1 <= L <= 34                           */
    double J;            /* Heisenberg: exchange coupling                                        */
    int64_t M;           /* global dimension (Heisenberg: must equal 2^L)                        */
    int64_t M_local;     /* rows held by this rank (== M when world == 1)                        */
    int64_t row_begin;   /* first global row of this rank                                        */
    int64_t nnz;         /* CSR: number of stored entries of this rank                          */
    const int64_t *row_ptr;
    const int32_t *col;
    const void *val;
    int32_t n_up;        /* SK_OP_HEISENBERG_SZ: number of up spins, 0 <= n_up <= L              */
    int32_t reserved;    /* zero                                                                 */
} sk_operator;

/* Solver parameters (the paper's *_init arguments, Alg. 1 P:L541 "init(ndim, nz, ndim,
   x, z)", made explicit: DESIGN.md R26). */
typedef struct {
    int32_t method;          /* sk_method                                                      */
    int32_t flags;           /* sk_flags                                                       */
    int64_t n_shift;         /* N_z >= 1                                                       */
    const sk_cplx *z;        /* [n_shift] HOST, copied.  z[0] is the first seed (R5)  */
    const sk_cplx *b;        /* [M_local] right-hand side rows of this rank, copied; != 0       */
    int32_t b_mem;           /* sk_mem of b                                                     */
    int32_t left_mem;        /* sk_mem of left                                                  */
    int64_t n_left;          /* number of left vectors a_l (0 with left == NULL means a = b)   */
    const sk_cplx *left;     /* [n_left][M_local] or NULL (a = b, one projection y_k = b^dag x) */
    int32_t full_x;          /* 1: store x^(k), p^(k) on device (P = I; memory O(M N_z),
                                P:L434-438); 0: projections only (the paper's default) */
    double tol;              /* retire shift k when ||r^(k)||_2 < tol (absolute)        */
    int64_t itermax;         /* iteration budget >= 1 (maxloops)                    */
} sk_params;

typedef struct sk_group sk_group;

/* Multi-GPU placement (the paper's optional MPI).  world == 1: one GPU.
   world > 1: the vector rows are sharded — rank g owns global rows [g M_local, (g+1) M_local),
   M_local = M / world a power of two (for the Heisenberg chain: the top log2(world) spin bits
   select the rank), and passes its own rows of b, of the left vectors and of the CSR (global
   column ids).  Dot products are all-reduced (NCCL, or a loopback group); the SpMV reads the
   rows it needs from the other ranks IN PLACE through peer memory (CUDA IPC mappings over
   NVLink) — the operator exchange is fused into the SpMV's loads.
   Two ways to run world > 1:
     * one process per GPU (NCCL): group == NULL.  sk_init, then exchange sk_ipc_handle()
       (64 B per rank, all-gathered by the caller) and one sk_nccl_unique_id() (128 B, from
       rank 0), then sk_connect().  All calls are collective in iteration order.
     * loopback group (tests on one GPU): group from sk_group_create(world); sk_init every rank
       with that group, sk_group_connect(), then sk_group_update / sk_group_run drive all ranks.
   Contexts of world > 1 refuse sk_update / sk_run until connected. */
typedef struct {
    int32_t rank;
    int32_t world;
    int32_t device;          /* CUDA device ordinal (ignored for a loopback group)             */
    int32_t reserved;
    const void *nccl_id;     /* unused (see sk_connect); kept for layout stability              */
    void *stream;            /* cudaStream_t to use, or NULL (library creates one)             */
    sk_group *group;         /* loopback group, or NULL                                         */
} sk_dist;

/* Current seed/shift coefficients (the quantities the paper logs in TriDiagComp.dat). */
typedef struct {
    int64_t iterations;      /* completed iterations n                                          */
    int64_t seed_index;      /* current seed shift s                                            */
    int64_t switches;        /* seed switches so far                                            */
    int64_t spmv_count;      /* operator applications so far (1 or 2 per iteration, Table 2)   */
    int64_t n_active;        /* shifts not yet retired                                          */
    int32_t status;          /* sk_status                                                       */
    int32_t reserved;
    sk_cplx z_seed;          /* z_s                                                             */
    sk_cplx alpha;           /* alpha_{n-1} of the current seed (after switch rescaling)        */
    sk_cplx rho;             /* rho_{n-1} of the current seed (after switch rescaling)          */
    sk_cplx beta;            /* beta_{n-2} used in the last iteration                          */
    double seed_residual;    /* ||r_n||_2 of the current seed                                   */
} sk_coeffs;

/* Create a context: allocate device state, copy z and b, set r_0 = b, r_-1 = 0,
   (BiCG) shadow r~_0 = conj(b) (R3), pi_0 = pi_-1 = 1, x_0 = 0, y_0 = 0, p_0/u_0 via
   the first update (R5).  After sk_init every residual equals ||b||_2. */
int sk_init(sk_ctx **out, const sk_operator *H, const sk_params *p, const sk_dist *d);

/* Exactly one iteration: q = H r_n (and q~ = H r~_n for BiCG), the seed and per-shift
   recurrences, the all-shift update, retirement and seed switching ("update and seed
   switching").  Synchronises the stream to return `status`.  Calling after a terminal status
   is a no-op returning that status. */
int sk_update(sk_ctx *ctx, int32_t *status);

/* Reverse-communication iteration: the caller computed q = H r and (BiCG)
   qt = H r~ on the vectors returned by sk_get_seed_vectors (device pointers, [M_local]).
   The operator kind may be SK_OP_RC. */
int sk_update_rc(sk_ctx *ctx, const sk_cplx *q_dev, const sk_cplx *qt_dev, int32_t *status);

/* Device pointers of the current seed residual r_n and shadow r~_n (NULL for COCG).  The
   vectors equal the paper's r_n, r~_n up to one internal scalar factor (seed-switch rescaling
   is applied lazily), which the library accounts for; valid until the next update. */
int sk_get_seed_vectors(sk_ctx *ctx, const sk_cplx **r_dev, const sk_cplx **rt_dev);

/* Up to max_iters iterations without host round trips (CUDA-graph captured); the status word is
   polled every poll_every iterations (<= 0: default 64).  Iterations after the terminal one are
   device-side no-ops, so results equal those of repeated sk_update. */
int sk_run(sk_ctx *ctx, int64_t max_iters, int32_t poll_every, int32_t *status);

/* Enqueue exactly `iters` iterations on the stream and return immediately (no host sync);
   for timing.  Terminal states make the remaining iterations device-side no-ops. */
int sk_enqueue(sk_ctx *ctx, int64_t iters);

/* ||r_n^(k)||_2 = ||r_n||_2 / |pi_n^(k)| per shift (EQ-COLLINEAR P:L300; "2-norm of the
   residual vector"); a retired shift reports its value at retirement.  res: HOST
   [n_shift]. */
int sk_get_residual(sk_ctx *ctx, double *res);

/* y[k][l] = a_l^dagger x_n^(k)  (HOST [n_shift][n_left], n_left = 1 when a = b). */
int sk_get_projection(sk_ctx *ctx, sk_cplx *y);

/* Full mode only: device pointer to x_n^(k) ([M_local]), valid until sk_finalize. */
int sk_get_solution(sk_ctx *ctx, int64_t k, const sk_cplx **x_dev);

/* Full mode only: copy x_n^(k) ([M_local]) into dst (host or device, per dst_mem). */
int sk_copy_solution(sk_ctx *ctx, int64_t k, sk_cplx *dst, int32_t dst_mem);

/* Per-shift state: pi_n^(k) (HOST [n_shift], relative to the current seed; frozen for retired
   shifts), active flags (HOST [n_shift], 1 = active) and retirement iteration (-1 if active).
   Any pointer may be NULL. */
int sk_get_shift_state(sk_ctx *ctx, sk_cplx *pi, uint8_t *active, int64_t *retired_at);

/* The current seed and its scalars (sk_coeffs above; the paper's TriDiagComp.dat quantities,
   P:L638) after finishing any pending iteration.  out: HOST. */
int sk_get_coefficients(sk_ctx *ctx, sk_coeffs *out);

/* Release everything and set *ctx = NULL.  A second call on NULL returns SK_ESTATE. */
int sk_finalize(sk_ctx **ctx);

/* q = H r for the given operator on device vectors (no solver state); for operator parity
   tests.  stream: cudaStream_t or NULL (default stream).  The Heisenberg (streaming) and
   Heisenberg-sector kernels take their work from a per-device queue that each launch rewinds:
   calls for those operators on one device must not run concurrently on different streams. */
int sk_apply_operator(const sk_operator *H, const sk_cplx *r_dev, sk_cplx *q_dev, void *stream);

/* ---- contour-integral eigensolver building blocks ----------
   The moments s_k = (1/2 pi i) oint (z - z0)^k (z - H)^{-1} phi dz are linear
   combinations of the full-mode solutions x^(j) of one solver (sk_get_solution) with the
   trapezoidal weights of the contour points z_j; the Rayleigh-Ritz step
   needs the Gram matrices S^dagger S and U~^dagger H U~.  The small eigenproblems are the
   caller's (host).

   out[c][i] = sum_j W[j * n_out + c] * X[j * ld_x + i] for 0 <= c < n_out, 0 <= i < M.
   X: DEVICE, n_in rows of stride ld_x >= M (e.g. the solutions of one context: ld_x =
   sk_get_solution(k+1) - sk_get_solution(k)); W: HOST [n_in][n_out] (copied); out: DEVICE
   [n_out][M], must not alias X.  Returns after the result is complete (synchronises `stream`).
   SK_EINVAL on null pointers or sizes (n_out <= 4096). */
int sk_combine(const sk_cplx *X, int64_t n_in, int64_t ld_x, int64_t M, const sk_cplx *W, int64_t n_out,
               sk_cplx *out, void *stream);

/* G[a * nb + b] = sum_i conj(A[a * M + i]) * B[b * M + i] (fixed summation order, deterministic).
   A: DEVICE [na][M], B: DEVICE [nb][M], G: HOST [na][nb]; 1 <= na, nb <= 64.  Synchronous on
   `stream`.  SK_EINVAL on null pointers or sizes. */
int sk_gram(const sk_cplx *A, int64_t na, const sk_cplx *B, int64_t nb, int64_t M, sk_cplx *G, void *stream);

/* Human-readable text of the last error on this thread (never NULL). */
const char *sk_last_error(void);

/* Per-kernel device timing (tracing).  While enabled, every iteration is enqueued as individual
   launches bracketed by CUDA events on the context stream (no graph capture), so the summed
   durations of the three kernel classes of one iteration can be read back. */
typedef struct {
    int64_t iterations;      /* iterations timed since the last reset                          */
    int64_t launches;        /* kernels this library launched since sk_init (all modes)        */
    double ms_spmv;          /* summed device time of the SpMV kernels (+ fused w, the finish of
                                the previous iteration and the seed scalars)                    */
    double ms_scalar;        /* summed device time of stand-alone scalar kernels (0 in a loop) */
    double ms_update;        /* summed device time of the fused update kernels (+ per-shift
                                recurrences)                                                    */
} sk_profile;

int sk_profile_enable(sk_ctx *ctx, int32_t on);
/* Synchronises the stream, accumulates the recorded events into *out; reset != 0 clears. */
int sk_get_profile(sk_ctx *ctx, sk_profile *out, int32_t reset);

/* The execution plan sk_init chose for a context (diagnostics; bench.py reports it).
   split_ahi > 0: the Heisenberg bond split — the SpMV applies the diagonal and
   the bonds (i, i+1), i < split_ahi; the update kernel applies the bonds i >= split_ahi and the
   periodic bond in its B-tile row order; 0: one kernel applies the whole operator.
   split_fuse: with the split, the SpMV also folds the r_{n-1} term of EQ-CG-RN-3REC into
   its output, u = H_A r_n - (gamma sr_prev / sr_cur) r_{n-1}, so the update reads u and r_n only.
   left_real: with the split and Im a = 0, the update reads Re a (8 B/row, its own row order).
   csr_col_blocks: opt-in (environment SHIFTK_CSR_BLOCKED=1; measured slower than one pass on the
   C3 workload, so off by default) for a one-GPU CSR operator whose rows are sorted by column and
   at most 255 entries long. */
typedef struct {
    int32_t split_ahi;       /* see above                                                      */
    int32_t spmv_ctas;       /* worker CTAs (= w partials) of the SpMV                         */
    int32_t update_ctas;     /* streaming CTAs of the update kernel                            */
    int32_t shift_agents;    /* shift-agent CTAs of the update kernel                          */
    int64_t arena_bytes;     /* device bytes the context owns                                  */
    int32_t split_fuse;      /* see above                                                      */
    int32_t left_real;       /* see above                                                      */
    int32_t csr_col_blocks;  /* >= 2: the CSR SpMV runs that many passes over column blocks of  */
    int32_t csr_block_shift; /* 2^csr_block_shift rows (the gathered slice of r stays in L2); 0: one pass */
} sk_info;
int sk_get_info(sk_ctx *ctx, sk_info *out);

/* Diagnostics: %globaltimer stamps (ns) written by instrumented kernels (16 slots; see
   csrc/steps.cuh).  Requires the environment variable SHIFTK_DEBUG_TS at sk_init. */
int sk_debug_timestamps(sk_ctx *ctx, int64_t *out16);

/* Recalculation at new shifts (ShiftK "recalc"): the per-shift recurrences
   EQ-SHIFTEDCG-PI/alpha/beta and EQ-SHIFTEDCG-y/u are replayed for z_new from the coefficient
   log recorded so far — no operator application.  Each new shift is frozen when its residual
   ||r_n|| / |pi_n| drops below tol, like the original shifts (R8), so recalc at the original
   shifts reproduces sk_get_projection.  Requires SK_FLAG_LOG.  z_new: HOST [n_new];
   y: HOST [n_new][n_left]; res: HOST [n_new] or NULL (residual at the last replayed step). */
int sk_recalc(sk_ctx *ctx, int64_t n_new, const sk_cplx *z_new, sk_cplx *y, double *res);

/* Checkpoint / restart ("initial values of the coefficients and the vector", P:L575
   calctype = restart; SURVEY f-4).  sk_checkpoint copies the complete solver state (seed
   residuals with their lazy scales, seed and per-shift scalars, projections, full-mode x/p,
   coefficient log) to host memory: call with buf = NULL to get the size in *bytes.
   sk_restore loads it into a context created by sk_init with the SAME operator, parameters and
   placement; the continued run is bit-identical to an uninterrupted one. */
int sk_checkpoint(sk_ctx *ctx, void *buf, size_t *bytes);
int sk_restore(sk_ctx *ctx, const void *buf, size_t bytes);

/* ---- multi-rank setup (see sk_dist) ---- */
/* Host all-reduce supplied by the caller (MPI_Allreduce, a gloo/torch.distributed group, ...):
   sum `n` doubles of `send` over the ranks into `recv` (both HOST memory owned by the library,
   valid for the call only); every rank must receive bit-identical sums.  Returns 0 on success. */
typedef int (*sk_allreduce_fn)(void *user, const double *send, double *recv, int64_t n);

/* CUDA IPC handle (64 bytes) of this context's device arena, for the other ranks. */
int sk_ipc_handle(sk_ctx *ctx, void *out64);
/* A fresh ncclUniqueId (128 bytes); call on one rank and broadcast. */
int sk_nccl_unique_id(void *out128);
/* Self-test of the NCCL plumbing on one device (diagnostics; "MPI optional"):
   a ONE-rank communicator is created on `device` and n doubles (HOST in) are all-reduced with the
   call the iteration uses (ncclDouble, ncclSum, a user stream) — directly into out1 and, replayed
   from a captured CUDA graph, into out2 (both HOST [n]; with one rank each equals in).  Returns
   SK_ENCCL if libnccl cannot be loaded or a NCCL call fails. */
int sk_nccl_selftest(int32_t device, int64_t n, const double *in_host, double *out1_host, double *out2_host);
/* Map every other rank's arena (handles: [world][64] from sk_ipc_handle, in rank order), join
   the NCCL communicator and finish the initialisation (global rho_0, ||b||, P b).  Collective. */
int sk_connect(sk_ctx *ctx, const void *handles, const void *nccl_id);
/* As sk_connect, but the two small all-reduces of every iteration (w; then rho, ||r||^2, P r —
   P:L973's parallel products) go through `fn` on the host instead of NCCL: the
   library copies this rank's partials to host, calls fn, copies the sums back (the stream is
   synchronised around the call, so iterations run without graph capture).  The operator's
   off-rank reads still go through the mapped peer arenas inside the SpMV kernels.  No kernel of
   one rank ever waits on another rank's kernel: ranks meet only inside fn.  For MPI codes (the
   paper's own parallelisation) and for testing the IPC data plane with several processes
   on one GPU.  Collective. */
int sk_connect_host(sk_ctx *ctx, const void *handles, sk_allreduce_fn fn, void *user);
/* Loopback group of `world` virtual ranks on one device (all share one stream). */
int sk_group_create(sk_group **out, int32_t world, int32_t device);
/* After sk_init of every rank with this group: wire the ranks and finish initialisation. */
int sk_group_connect(sk_group *group);
/* One iteration / up to max_iters iterations of every rank (status of the group). */
int sk_group_update(sk_group *group, int32_t *status);
int sk_group_run(sk_group *group, int64_t max_iters, int32_t *status);
/* Release the group (every member context must be finalized first). */
int sk_group_destroy(sk_group **group);

/* Library version / build info string (never NULL). */
const char *sk_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SHIFTK_H */
