/*
 * shiftk_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the shifted COCG / shifted BiCG
 * iteration of the Komega paper (arxiv 2001.08707; PAPER.md = /root/reference/PAPER.md,
 * cited P:Lnnn) and of the two operators on the hot path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or helper with the CUDA path (paper_2001_08707_b200/csrc).
 *
 * Arithmetic: IEEE fp64, C99 `double complex`.  Every reduction has one fixed order: the
 * index range is cut into consecutive chunks of OR_CHUNK elements, each chunk is summed in
 * index order, and the chunk sums are added in index order (SURVEY §8(c.1) "Determinism": "a
 * static chunking, accumulates per chunk in order, and combines the chunks in index order").
 * OR_FLAG_REVERSE runs both levels backwards (used only to measure the self-divergence
 * horizon of SURVEY §8(c.4)).  The same source is built twice: liboracle.so (one thread) and
 * liboracle_omp.so (-fopenmp: the chunks and the element-wise loops are shared out among
 * threads).  The order of every floating-point operation is the same in both, so the two
 * builds give bit-identical results (pinned in tests/test_oracle_pins.py).
 *
 * Memory: b and the left vectors are BORROWED (the caller keeps them alive until or_destroy);
 * with a = b the single left vector is b itself.  r_{n+1} is formed in the buffer of r_{n-1}
 * (each element is read before it is overwritten), so the state holds three M-vectors (r, r_old
 * and, for BiCG, t, t_old) beyond b — the paper's three-vector storage.
 *
 * Algorithm (one call of or_update = one iteration n; step numbers follow SURVEY §8(c.1)):
 *   inner product  <u,v> = sum u_i v_i (COCG, App. A)  |  sum conj(u_i) v_i (BiCG)
 *   A = z_s I - H  (EQ-SHIFT-EQ2), so  A r = z_s r - q  with q = H r supplied by the caller
 *   2  rho_n = <r_n, r_n> | <t_n, r_n>,  w_n = <r_n, q> | <t_n, q>
 *   3  beta_{n-1} = rho_n / rho_{n-1}  (EQ-REC-BETA P:L262), gamma = beta_{n-1}/alpha_{n-1},
 *      gamma = 0 at n = 0 ("start with beta_{-1}/alpha_{-1} = 0")
 *   4  alpha_n = rho_n / (<r, A r> - gamma rho_n),  <r, A r> = z_s rho_n - w_n   (EQ-REC-ALPHA-N2 P:L276)
 *   5  c_n = alpha_n gamma = alpha_n beta_{n-1} / alpha_{n-1}
 *   6  per active shift k, sigma = z_k - z_s:
 *        pi_{n+1} = (1 + c_n + alpha_n sigma) pi_n - c_n pi_{n-1}                  (EQ-SHIFTEDCG-PI P:L317)
 *        alpha_n^k = (pi_n / pi_{n+1}) alpha_n                                       (EQ-SHIFTEDCG-alpha P:L325)
 *        beta_{n-1}^k = (pi_{n-1} / pi_n)^2 beta_{n-1}                              (EQ-SHIFTEDCG-beta P:L326)
 *   7  full:  p_n^k = r_n / pi_n^k + beta_{n-1}^k p_{n-1}^k ; x_{n+1}^k = x_n^k + alpha_n^k p_n^k
 *                                                                                    (EQ-SHIFTEDCG-x/p P:L327-328)
 *      proj:  g_n = P r_n (g_l = a_l^dagger r_n);  u_n^k = g_n / pi_n^k + beta_{n-1}^k u_{n-1}^k ;
 *             y_{n+1}^k = y_n^k + alpha_n^k u_n^k      (EQ-SHIFTEDCG-y/u P:L372-376 with the index
 *             of P:L373 read as pi_{n+1} / r_{n+1} for u_{n+1}, i.e. as EQ-SHIFTEDCG-p; R1)
 *   8  r_{n+1} = (1 + c_n) r_n - alpha_n A r_n - c_n r_{n-1}                       (EQ-CG-RN-3REC P:L269)
 *      BiCG:  t_{n+1} = (1 + c_n^*) t_n - alpha_n^* A^dagger t_n - c_n^* t_{n-1},
 *             A^dagger t = z_s^* t - H t  (H Hermitian)                               (App. B)
 *   9  pi_{n-1} <- pi_n, pi_n <- pi_{n+1}; alpha_prev <- alpha_n; rho_prev <- rho_n
 *  10  nu = ||r_{n+1}||_2 ("2-norm"); res_k = nu / |pi_{n+1}^k| (EQ-COLLINEAR P:L300);
 *      retire k when res_k < tol (frozen thereafter, R8)
 *  11  CONVERGED when no shift is active; MAXITER when n+1 = itermax
 *  log   (recalc) per iteration n: alpha_n, beta_{n-1}, c_n, z_s, g_n = P r_n,
 *        nu = ||r_{n+1}|| and the switch factors 1/f, 1/f' (1 when no switch) — or_recalc replays
 *        steps 6, 7 (projection), 10 for new shifts from this log with no operator application.
 *  12  seed switch ("always ... after an update"): s* = argmin_{k active} |pi_{n+1}^k|,
 *      lowest index on ties; if s* != s:  f = pi_{n+1}^{s*}, f' = pi_n^{s*};
 *      r_{n+1} /= f, r_n /= f' (shadow by conj);  active pi_{n+1} /= f, pi_n /= f';
 *      alpha_prev *= f'/f (EQ-SHIFTEDCG-alpha);  rho_prev /= f'^2;  z_s = z_{s*}   (R9)
 *
 * Breakdown (R12): |rho_n| < 1e-300 or |alpha denominator| < 1e-300 -> OR_BREAKDOWN.
 */
#include <complex.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

#define OR_CHUNK 32768   /* reduction chunk (elements) */

enum { OR_COCG = 0, OR_BICG = 1 };
enum { OR_ITERATING = 0, OR_CONVERGED = 1, OR_MAXITER = 2, OR_BREAKDOWN = 3 };
enum { OR_FLAG_REVERSE = 1, OR_FLAG_NO_SWITCH = 2 };

typedef struct {
    int method, full, flags;
    int64_t M, nz, nleft, itermax;
    double tol;
    const cplx *b, *left;      /* borrowed; left: [nleft][M] (b itself when a = b) */
    cplx *r, *r_old, *t, *t_old;
    cplx *part;                /* chunk sums of one reduction */
    int64_t nchunk;
    cplx *z, zs;
    int64_t s;
    cplx *pi, *pi_old, *pi_new;
    unsigned char *active;
    double *res;
    int64_t *retired_at;
    cplx *g, *u, *y;           /* g: [nleft]; u, y: [nz][nleft] */
    cplx *p, *x;               /* [nz][M] when full (only shifts with keep[k]) */
    unsigned char *keep;       /* full mode: which shifts carry x, p (all by default) */
    cplx alpha_prev, rho_prev;
    cplx alpha, beta, rho, w;  /* last iteration's seed scalars (for inspection) */
    /* coefficient log for recalculation */
    int64_t nlog, caplog;
    cplx *lg_alpha, *lg_beta, *lg_c, *lg_zs, *lg_rf, *lg_rfp, *lg_g;   /* lg_g: [cap][nleft] */
    double *lg_nu;
    int64_t n, nswitch, nspmv;
    int status;
} or_state;

/* ------------------------------------------------------------------ inner products */

/* sum over i of f(u_i, v_i) in the fixed chunked order (see the header); conj_u selects
   conj(u_i) v_i instead of u_i v_i */
static cplx dot_chunked(const or_state *st, const cplx *u, const cplx *v, int conj_u) {
    const int64_t M = st->M, nc = st->nchunk;
    const int rev = (st->flags & OR_FLAG_REVERSE) != 0;
    cplx *part = st->part;
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
    for (int64_t c = 0; c < nc; ++c) {
        const int64_t i0 = c * OR_CHUNK, i1 = (i0 + OR_CHUNK < M) ? i0 + OR_CHUNK : M;
        cplx acc = 0;
        if (rev) {
            for (int64_t i = i1 - 1; i >= i0; --i) acc += (conj_u ? conj(u[i]) : u[i]) * v[i];
        } else {
            for (int64_t i = i0; i < i1; ++i) acc += (conj_u ? conj(u[i]) : u[i]) * v[i];
        }
        part[c] = acc;
    }
    cplx acc = 0;
    if (rev) {
        for (int64_t c = nc - 1; c >= 0; --c) acc += part[c];
    } else {
        for (int64_t c = 0; c < nc; ++c) acc += part[c];
    }
    return acc;
}

static cplx dot_plain(const or_state *st, const cplx *u, const cplx *v) {
    return dot_chunked(st, u, v, 0);
}

static cplx dot_conj(const or_state *st, const cplx *u, const cplx *v) {
    return dot_chunked(st, u, v, 1);
}

/* <u, v> of the method: unconjugated for COCG (App. A), conjugated for BiCG (App. B) */
static cplx dot_method(const or_state *st, const cplx *u, const cplx *v) {
    return st->method == OR_COCG ? dot_plain(st, u, v) : dot_conj(st, u, v);
}

/* g_l = a_l^dagger v  (projection P v) */
static void project(const or_state *st, const cplx *v, cplx *g) {
    for (int64_t l = 0; l < st->nleft; ++l) g[l] = dot_conj(st, st->left + l * st->M, v);
}

/* ------------------------------------------------------------------ lifecycle */

static void *xcalloc(size_t n, size_t sz) { return calloc(n ? n : 1, sz); }

void or_destroy(or_state *st);

/* left == NULL  ->  a = b (one left vector equal to b). */
or_state *or_create_subset(int method, int64_t M, int64_t nz, const cplx *z, const cplx *b,
                           int64_t nleft, const cplx *left, int full, double tol, int64_t itermax,
                           int flags, const unsigned char *keep);

or_state *or_create(int method, int64_t M, int64_t nz, const cplx *z, const cplx *b,
                    int64_t nleft, const cplx *left, int full, double tol, int64_t itermax,
                    int flags) {
    return or_create_subset(method, M, nz, z, b, nleft, left, full, tol, itermax, flags, NULL);
}

/* Full mode with x, p stored only for the shifts with keep[k] != 0 (NULL = all).  The scalar
   recurrences, retirement and seed switching still run over every shift, and they never read
   x or p, so the iterates of the carried shifts are exactly those of a run carrying all. */
or_state *or_create_subset(int method, int64_t M, int64_t nz, const cplx *z, const cplx *b,
                           int64_t nleft, const cplx *left, int full, double tol, int64_t itermax,
                           int flags, const unsigned char *keep) {
    if (M <= 0 || nz <= 0 || (method != OR_COCG && method != OR_BICG) || tol <= 0 || itermax < 1)
        return NULL;
    or_state *st = (or_state *)xcalloc(1, sizeof(or_state));
    st->method = method; st->M = M; st->nz = nz; st->full = full; st->tol = tol;
    st->itermax = itermax; st->flags = flags;
    st->nleft = left ? nleft : 1;
    st->b = b;
    st->left = left ? left : b;
    st->nchunk = (M + OR_CHUNK - 1) / OR_CHUNK;
    st->part = (cplx *)xcalloc(st->nchunk, sizeof(cplx));
    st->r = (cplx *)malloc((size_t)M * sizeof(cplx));
    st->r_old = (cplx *)xcalloc(M, sizeof(cplx));
    if (!st->r || !st->r_old || !st->part) { or_destroy(st); return NULL; }
    if (method == OR_BICG) {
        st->t = (cplx *)xcalloc(M, sizeof(cplx));
        st->t_old = (cplx *)xcalloc(M, sizeof(cplx));
    }
    st->z = (cplx *)xcalloc(nz, sizeof(cplx));
    st->pi = (cplx *)xcalloc(nz, sizeof(cplx));
    st->pi_old = (cplx *)xcalloc(nz, sizeof(cplx));
    st->pi_new = (cplx *)xcalloc(nz, sizeof(cplx));
    st->active = (unsigned char *)xcalloc(nz, 1);
    st->res = (double *)xcalloc(nz, sizeof(double));
    st->retired_at = (int64_t *)xcalloc(nz, sizeof(int64_t));
    st->g = (cplx *)xcalloc(st->nleft, sizeof(cplx));
    st->u = (cplx *)xcalloc(nz * st->nleft, sizeof(cplx));
    st->y = (cplx *)xcalloc(nz * st->nleft, sizeof(cplx));
    st->keep = (unsigned char *)xcalloc(nz, 1);
    int64_t nkeep = 0;
    for (int64_t k = 0; k < nz; ++k) {
        st->keep[k] = keep ? (keep[k] != 0) : 1;
        nkeep += st->keep[k];
    }
    if (full) {
        /* x, p rows of the kept shifts only, addressed through slot[] */
        st->p = (cplx *)xcalloc((size_t)(nkeep * M), sizeof(cplx));
        st->x = (cplx *)xcalloc((size_t)(nkeep * M), sizeof(cplx));
        if (!st->p || !st->x) { or_destroy(st); return NULL; }
    }
    memcpy(st->z, z, nz * sizeof(cplx));

    /* Init: r_0 = b, r_{-1} = 0, t_0 = conj(b) (R3), pi_0 = pi_{-1} = 1,
       x_0 = 0, y_0 = 0, first seed z[0]. */
    memcpy(st->r, b, (size_t)M * sizeof(cplx));
    if (method == OR_BICG)
        for (int64_t i = 0; i < M; ++i) st->t[i] = conj(b[i]);
    double nb = sqrt(creal(dot_conj(st, b, b)));
    for (int64_t k = 0; k < nz; ++k) {
        st->pi[k] = 1; st->pi_old[k] = 1; st->active[k] = 1; st->res[k] = nb;
        st->retired_at[k] = -1;
    }
    st->s = 0; st->zs = z[0];
    st->n = 0; st->status = OR_ITERATING;
    return st;
}

void or_destroy(or_state *st) {
    if (!st) return;
    free(st->part); free(st->r); free(st->r_old);
    free(st->t); free(st->t_old); free(st->z); free(st->pi); free(st->pi_old); free(st->pi_new);
    free(st->active); free(st->res); free(st->retired_at); free(st->g); free(st->u); free(st->y);
    free(st->p); free(st->x); free(st->keep);
    free(st->lg_alpha); free(st->lg_beta); free(st->lg_c); free(st->lg_zs); free(st->lg_rf);
    free(st->lg_rfp); free(st->lg_g); free(st->lg_nu);
    free(st);
}

/* ------------------------------------------------------------------ coefficient log */

static int log_reserve(or_state *st, int64_t n) {
    if (n < st->caplog) return 1;
    int64_t cap = st->caplog ? 2 * st->caplog : 64;
    while (cap <= n) cap *= 2;
#define GROW(f, T, w) do { T *p_ = (T *)realloc(st->f, (size_t)(cap * (w)) * sizeof(T)); \
                           if (!p_) return 0; st->f = p_; } while (0)
    GROW(lg_alpha, cplx, 1); GROW(lg_beta, cplx, 1); GROW(lg_c, cplx, 1); GROW(lg_zs, cplx, 1);
    GROW(lg_rf, cplx, 1); GROW(lg_rfp, cplx, 1); GROW(lg_nu, double, 1);
    GROW(lg_g, cplx, st->nleft);
#undef GROW
    st->caplog = cap;
    return 1;
}

/* ------------------------------------------------------------------ one iteration */

/* q = H r_n (and qt = H t_n for BiCG), computed by the caller (reverse communication,
   P:L503-508; Alg. 1). */
int or_update(or_state *st, const cplx *q, const cplx *qt) {
    if (st->status != OR_ITERATING) return st->status;
    const int64_t M = st->M, nz = st->nz, nl = st->nleft, n = st->n;
    const int bicg = st->method == OR_BICG;
    const cplx *tv = bicg ? st->t : st->r;    /* left operand of the method's inner product */
    st->nspmv += bicg ? 2 : 1;

    /* 2 */
    cplx rho = dot_method(st, tv, st->r);
    cplx w = dot_method(st, tv, q);
    /* 3 */
    cplx beta = 0, gamma = 0;
    if (n > 0) { beta = rho / st->rho_prev; gamma = beta / st->alpha_prev; }
    /* 4 */
    cplx den = st->zs * rho - w - gamma * rho;
    if (cabs(rho) < 1e-300 || cabs(den) < 1e-300) { st->status = OR_BREAKDOWN; return st->status; }
    cplx alpha = rho / den;
    /* 5 */
    cplx c = alpha * gamma;
    st->alpha = alpha; st->beta = beta; st->rho = rho; st->w = w;

    /* 6 + 7 */
    if (nl > 0) project(st, st->r, st->g);
    const int logged = log_reserve(st, n);
    if (logged) {
        st->lg_alpha[n] = alpha; st->lg_beta[n] = beta; st->lg_c[n] = c; st->lg_zs[n] = st->zs;
        for (int64_t l = 0; l < nl; ++l) st->lg_g[n * nl + l] = st->g[l];
        st->lg_rf[n] = 1; st->lg_rfp[n] = 1; st->lg_nu[n] = 0;
        st->nlog = n + 1;
    }
    for (int64_t k = 0; k < nz; ++k) {
        if (!st->active[k]) continue;
        cplx sigma = st->z[k] - st->zs;
        cplx pin = (1.0 + c + alpha * sigma) * st->pi[k] - c * st->pi_old[k];
        cplx ak = (st->pi[k] / pin) * alpha;
        cplx rat = st->pi_old[k] / st->pi[k];
        cplx bk = (n == 0) ? 0 : rat * rat * beta;
        st->pi_new[k] = pin;
        for (int64_t l = 0; l < nl; ++l) {
            cplx *u = st->u + k * nl + l, *y = st->y + k * nl + l;
            *u = st->g[l] / st->pi[k] + bk * (*u);
            *y = *y + ak * (*u);
        }
        if (st->full && st->keep[k]) {
            int64_t slot = 0;
            for (int64_t j = 0; j < k; ++j) slot += st->keep[j];
            cplx *p = st->p + slot * M, *x = st->x + slot * M;
            const cplx *rr = st->r, ipk = st->pi[k];
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
            for (int64_t i = 0; i < M; ++i) {
                p[i] = rr[i] / ipk + bk * p[i];
                x[i] = x[i] + ak * p[i];
            }
        }
    }

    /* 8  (r_{n+1} formed in the buffer of r_{n-1}: element i of r_{n-1} is read before it is
          overwritten, then the buffers rotate) */
    {
        cplx *rn = st->r, *ro = st->r_old;
        const cplx zs = st->zs;
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
        for (int64_t i = 0; i < M; ++i)
            ro[i] = (1.0 + c) * rn[i] - alpha * (zs * rn[i] - q[i]) - c * ro[i];
        st->r = ro; st->r_old = rn;
    }
    if (bicg) {
        cplx cc = conj(c), ac = conj(alpha), zc = conj(st->zs);
        cplx *tn = st->t, *to = st->t_old;
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
        for (int64_t i = 0; i < M; ++i)
            to[i] = (1.0 + cc) * tn[i] - ac * (zc * tn[i] - qt[i]) - cc * to[i];
        st->t = to; st->t_old = tn;
    }

    /* 9 */
    for (int64_t k = 0; k < nz; ++k) {
        if (!st->active[k]) continue;
        st->pi_old[k] = st->pi[k];
        st->pi[k] = st->pi_new[k];
    }
    st->alpha_prev = alpha;
    st->rho_prev = rho;
    st->n = n + 1;

    /* 10 */
    double nu = sqrt(creal(dot_conj(st, st->r, st->r)));
    if (logged) st->lg_nu[n] = nu;
    int64_t nact = 0;
    for (int64_t k = 0; k < nz; ++k) {
        if (!st->active[k]) continue;
        st->res[k] = nu / cabs(st->pi[k]);
        if (st->res[k] < st->tol) { st->active[k] = 0; st->retired_at[k] = n + 1; }
        else ++nact;
    }
    /* 11 */
    if (nact == 0) { st->status = OR_CONVERGED; return st->status; }

    /* 12 */
    if (!(st->flags & OR_FLAG_NO_SWITCH)) {
        int64_t best = -1; double bmin = 0;
        for (int64_t k = 0; k < nz; ++k) {
            if (!st->active[k]) continue;
            double a = cabs(st->pi[k]);
            if (best < 0 || a < bmin) { best = k; bmin = a; }
        }
        if (best != st->s) {
            cplx f = st->pi[best], fp = st->pi_old[best];
            cplx *rr = st->r, *ro = st->r_old;
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
            for (int64_t i = 0; i < M; ++i) { rr[i] /= f; ro[i] /= fp; }
            if (bicg) {
                cplx fc = conj(f), fpc = conj(fp);
                cplx *tt = st->t, *to = st->t_old;
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
                for (int64_t i = 0; i < M; ++i) { tt[i] /= fc; to[i] /= fpc; }
            }
            for (int64_t k = 0; k < nz; ++k) {
                if (!st->active[k]) continue;
                st->pi[k] /= f; st->pi_old[k] /= fp;
            }
            st->alpha_prev *= fp / f;
            st->rho_prev /= fp * fp;
            st->zs = st->z[best];
            st->s = best;
            st->nswitch++;
            if (logged) { st->lg_rf[n] = 1.0 / f; st->lg_rfp[n] = 1.0 / fp; }
        }
    }
    if (st->n >= st->itermax) st->status = OR_MAXITER;
    return st->status;
}

/* ------------------------------------------------------------------ recalculation */

/* Projections y[j][l] = a_l^dagger x^(z_j) for new shifts from the coefficient log (P:L640-651:
   "the recurrence relations for the shifted equation ... can be solved without any expensive
   matrix-vector multiplications"): for each new shift, steps 6, 7 (projection) and 10 of
   or_update replayed with the logged alpha_n, beta_{n-1}, c_n, z_s, g_n, nu and switch
   factors; the shift is frozen (R8) when its residual drops below tol.  res[j]: last residual. */
void or_recalc(const or_state *st, int64_t nnew, const cplx *znew, double tol, cplx *y, double *res) {
    const int64_t nl = st->nleft;
    cplx *u = (cplx *)xcalloc(nl, sizeof(cplx));
    for (int64_t j = 0; j < nnew; ++j) {
        cplx pi = 1, pio = 1;
        double rj = sqrt(creal(dot_conj(st, st->b, st->b)));
        for (int64_t l = 0; l < nl; ++l) { u[l] = 0; y[j * nl + l] = 0; }
        for (int64_t n = 0; n < st->nlog; ++n) {
            const cplx alpha = st->lg_alpha[n], beta = st->lg_beta[n], c = st->lg_c[n];
            const cplx sigma = znew[j] - st->lg_zs[n];
            const cplx pin = (1.0 + c + alpha * sigma) * pi - c * pio;
            const cplx ak = (pi / pin) * alpha;
            const cplx rat = pio / pi;
            const cplx bk = (n == 0) ? 0 : rat * rat * beta;
            for (int64_t l = 0; l < nl; ++l) {
                u[l] = st->lg_g[n * nl + l] / pi + bk * u[l];
                y[j * nl + l] += ak * u[l];
            }
            pio = pi;
            pi = pin;
            rj = st->lg_nu[n] / cabs(pi);
            if (rj < tol) break;
            pi *= st->lg_rf[n];
            pio *= st->lg_rfp[n];
        }
        if (res) res[j] = rj;
    }
    free(u);
}

int64_t or_log_length(const or_state *st) { return st->nlog; }

/* ------------------------------------------------------------------ operators */

/* S=1/2 Heisenberg chain H = J sum_{i=0}^{L-1} S_i . S_{i+1}, periodic.  Basis state s
   is an L-bit integer, bit i = site i, bit value 1 = up (R16).  Per bond (i, i+1):
   S^z S^z gives +J/4 (aligned) or -J/4 (anti-aligned); (S^+S^- + S^-S^+)/2 flips an
   anti-aligned pair with amplitude J/2. */
void or_heisenberg_apply(int L, double J, const cplx *r, cplx *q) {
    const int64_t M = (int64_t)1 << L;
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
    for (int64_t s = 0; s < M; ++s) {
        cplx acc = 0;
        for (int i = 0; i < L; ++i) {
            int j = (i + 1) % L;
            int bi = (int)((s >> i) & 1), bj = (int)((s >> j) & 1);
            if (bi == bj) {
                acc += 0.25 * J * r[s];
            } else {
                acc += -0.25 * J * r[s];
                int64_t s2 = s ^ (((int64_t)1 << i) | ((int64_t)1 << j));
                acc += 0.5 * J * r[s2];
            }
        }
        q[s] = acc;
    }
}

/* q = H r for a CSR matrix with real values (row_ptr int64[M+1], col int32[nnz]). */
void or_csr_real_apply(int64_t M, const int64_t *row_ptr, const int32_t *col, const double *val,
                       const cplx *r, cplx *q) {
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
    for (int64_t i = 0; i < M; ++i) {
        cplx acc = 0;
        for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) acc += val[e] * r[col[e]];
        q[i] = acc;
    }
}

/* q = H r for a CSR matrix with complex values. */
void or_csr_cplx_apply(int64_t M, const int64_t *row_ptr, const int32_t *col, const cplx *val,
                       const cplx *r, cplx *q) {
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
    for (int64_t i = 0; i < M; ++i) {
        cplx acc = 0;
        for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) acc += val[e] * r[col[e]];
        q[i] = acc;
    }
}

/* One output element of the operators (for sampled parity at sizes where a full product is
   too slow): q_s = sum_j H_sj r_j, same arithmetic as the full products above. */
cplx or_heisenberg_row(int L, double J, const cplx *r, int64_t s) {
    cplx acc = 0;
    for (int i = 0; i < L; ++i) {
        const int j = (i + 1) % L;                    /* bond (i, i+1 mod L) */
        const int bi = (int)((s >> i) & 1), bj = (int)((s >> j) & 1);
        if (bi == bj) {
            acc += 0.25 * J * r[s];                   /* parallel spins: +J/4 */
        } else {
            const int64_t flip = ((int64_t)1 << i) | ((int64_t)1 << j);
            acc += -0.25 * J * r[s];                  /* antiparallel: -J/4 */
            acc += 0.5 * J * r[s ^ flip];             /* and J/2 to the flipped pair */
        }
    }
    return acc;
}

cplx or_csr_real_row(const int64_t *row_ptr, const int32_t *col, const double *val, const cplx *r,
                     int64_t i) {
    const int64_t e_begin = row_ptr[i], e_end = row_ptr[i + 1];
    cplx acc = 0;
    for (int64_t e = e_begin; e < e_end; ++e) acc += val[e] * r[col[e]];      /* real row */
    return acc;
}

cplx or_csr_cplx_row(const int64_t *row_ptr, const int32_t *col, const cplx *val, const cplx *r,
                     int64_t i) {
    const int64_t e_begin = row_ptr[i], e_end = row_ptr[i + 1];
    cplx acc = 0;
    for (int64_t e = e_begin; e < e_end; ++e) acc += val[e] * r[col[e]];      /* complex row */
    return acc;
}

/* ------------------------------------------------------------------ accessors */

int or_status(const or_state *st) { return st->status; }
int64_t or_iterations(const or_state *st) { return st->n; }
int64_t or_switches(const or_state *st) { return st->nswitch; }
int64_t or_spmv_count(const or_state *st) { return st->nspmv; }
int64_t or_seed_index(const or_state *st) { return st->s; }
const cplx *or_r(const or_state *st) { return st->r; }
const cplx *or_r_old(const or_state *st) { return st->r_old; }
const cplx *or_t(const or_state *st) { return st->t; }
const cplx *or_pi(const or_state *st) { return st->pi; }
const cplx *or_pi_old(const or_state *st) { return st->pi_old; }
const double *or_res(const or_state *st) { return st->res; }
const unsigned char *or_active(const or_state *st) { return st->active; }
const int64_t *or_retired_at(const or_state *st) { return st->retired_at; }
const cplx *or_y(const or_state *st) { return st->y; }
const cplx *or_x(const or_state *st, int64_t k) {
    if (!st->full || !st->keep[k]) return NULL;
    int64_t slot = 0;
    for (int64_t j = 0; j < k; ++j) slot += st->keep[j];
    return st->x + slot * st->M;
}
void or_scalars(const or_state *st, cplx *out /* [6] */) {
    out[0] = st->alpha; out[1] = st->beta; out[2] = st->rho; out[3] = st->w;
    out[4] = st->zs; out[5] = st->alpha_prev;
}

/* ------------------------------------------------------------------ Sz sector (SURVEY f-3)

   The Heisenberg chain conserves S^z_total, so H is block diagonal over sectors of fixed
   number of up spins n (2 S^z = 2n - L; HPhi's "2Sz=0" sector, of dimension
   C(L, L/2), e.g. 924 at L=12).  Sector basis (R28): the L-bit states with
   popcount n in ASCENDING integer order; row i of the sector operator is the i-th such state.
   The oracle builds that list by brute force and finds ranks by binary search; the rank by
   counting (or_sz_rank) is only used for sampled rows at sizes where the list is too large. */

/* number of states of the sector: C(L, n), by Pascal's rule */
int64_t or_sz_dim(int L, int n) {
    if (n < 0 || n > L) return 0;
    int64_t c[65] = {0};
    c[0] = 1;
    for (int m = 1; m <= L; ++m)
        for (int k = m; k >= 1; --k) c[k] += c[k - 1];
    return c[n];
}

/* the sector states in ascending order (out has or_sz_dim(L, n) entries) */
void or_sz_states(int L, int n, int64_t *out) {
    int64_t i = 0;
    for (int64_t s = 0; s < ((int64_t)1 << L); ++s)
        if (__builtin_popcountll((unsigned long long)s) == n) out[i++] = s;
}

static int64_t sz_find(const int64_t *states, int64_t D, int64_t s) {
    int64_t lo = 0, hi = D - 1;
    while (lo <= hi) {
        int64_t mid = (lo + hi) / 2;
        if (states[mid] == s) return mid;
        if (states[mid] < s) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

/* q = H r restricted to the sector: the same bond sum as or_heisenberg_apply, on the list */
void or_heisenberg_sz_apply(int L, double J, const int64_t *states, int64_t D, const cplx *r, cplx *q) {
    for (int64_t a = 0; a < D; ++a) {
        int64_t s = states[a];
        cplx acc = 0;
        for (int i = 0; i < L; ++i) {
            int j = (i + 1) % L;
            int bi = (int)((s >> i) & 1), bj = (int)((s >> j) & 1);
            if (bi == bj) {
                acc += 0.25 * J * r[a];
            } else {
                acc += -0.25 * J * r[a];
                int64_t s2 = s ^ (((int64_t)1 << i) | ((int64_t)1 << j));
                acc += 0.5 * J * r[sz_find(states, D, s2)];
            }
        }
        q[a] = acc;
    }
}

/* rank of s among the n-bit states by counting the smaller ones: scanning the set bits from the
   top, a set bit at position p with m set bits at positions <= p contributes the C(p, m)
   states that agree above p, have 0 at p and m set bits below p. */
int64_t or_sz_rank(int L, int64_t s) {
    int64_t rank = 0;
    int m = __builtin_popcountll((unsigned long long)s);
    for (int p = L - 1; p >= 0 && m > 0; --p) {
        if ((s >> p) & 1) {
            rank += or_sz_dim(p, m);
            m -= 1;
        }
    }
    return rank;
}

/* the state of rank `rank`: the inverse of the counting above, bit by bit from the top */
int64_t or_sz_unrank(int L, int n, int64_t rank) {
    int64_t s = 0;
    int m = n;
    for (int p = L - 1; p >= 0 && m > 0; --p) {
        int64_t below = or_sz_dim(p, m);   /* states with a 0 here and m set bits below */
        if (rank >= below) {
            s |= (int64_t)1 << p;
            rank -= below;
            m -= 1;
        }
    }
    return s;
}

/* one row of the sector operator (for sampled parity at large L) */
cplx or_heisenberg_sz_row(int L, int n, double J, const cplx *r, int64_t a) {
    int64_t s = or_sz_unrank(L, n, a);
    cplx acc = 0;
    for (int i = 0; i < L; ++i) {
        int j = (i + 1) % L;
        int bi = (int)((s >> i) & 1), bj = (int)((s >> j) & 1);
        if (bi == bj) {
            acc += 0.25 * J * r[a];
        } else {
            acc += -0.25 * J * r[a];
            acc += 0.5 * J * r[or_sz_rank(L, s ^ (((int64_t)1 << i) | ((int64_t)1 << j)))];
        }
    }
    return acc;
}
