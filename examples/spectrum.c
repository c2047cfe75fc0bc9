/* A plain C caller of the boundary (no Python, no torch): the spectral function
   A(w) = -1/pi Im b^dagger (w + i delta - H)^-1 b of an S=1/2 Heisenberg chain on a
   grid of shifts, b a fixed pseudo-random unit vector, through sk_init (host b),
   sk_run, sk_get_projection / sk_get_residual, sk_finalize.

   build: gcc -O2 -I include examples/spectrum.c -L paper_2001_08707_b200 -lshiftk \
              -Wl,-rpath,$PWD/paper_2001_08707_b200 -lm -o spectrum
   run:   ./spectrum L n_shift     (prints "w A(w) residual" lines, then a status line) */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "shiftk.h"

static uint64_t lcg(uint64_t *s) {
    *s = *s * 6364136223846793005ull + 1442695040888963407ull;
    return *s >> 11;
}

int main(int argc, char **argv) {
    const int L = argc > 1 ? atoi(argv[1]) : 12;
    const int64_t nz = argc > 2 ? atoll(argv[2]) : 32;
    const int64_t M = (int64_t)1 << L;
    const double delta = 0.1, wmin = -6.0, wmax = 2.0;
    sk_cplx *b = malloc(sizeof(sk_cplx) * M), *z = malloc(sizeof(sk_cplx) * nz);
    sk_cplx *y = malloc(sizeof(sk_cplx) * nz);
    double *res = malloc(sizeof(double) * nz);
    uint64_t seed = 12345;
    double nrm = 0;
    for (int64_t i = 0; i < M; ++i) {
        b[i].re = (double)lcg(&seed) / 9007199254740992.0 - 0.5;
        b[i].im = 0;
        nrm += b[i].re * b[i].re;
    }
    nrm = sqrt(nrm);
    for (int64_t i = 0; i < M; ++i) b[i].re /= nrm;
    for (int64_t k = 0; k < nz; ++k) {
        z[k].re = wmin + k * (wmax - wmin) / nz;
        z[k].im = delta;
    }
    sk_operator H = {0};
    H.kind = SK_OP_HEISENBERG;
    H.L = L;
    H.J = 1.0;
    H.M = M;
    H.M_local = M;
    sk_params p = {0};
    p.method = SK_COCG;
    p.n_shift = nz;
    p.z = z;
    p.b = b;
    p.b_mem = SK_MEM_HOST;
    p.tol = 1e-10;
    p.itermax = 20000;
    sk_dist d = {0};
    d.world = 1;
    sk_ctx *ctx = NULL;
    if (sk_init(&ctx, &H, &p, &d) != SK_OK) {
        fprintf(stderr, "sk_init: %s\n", sk_last_error());
        return 1;
    }
    int32_t status = 0;
    if (sk_run(ctx, p.itermax, 64, &status) != SK_OK || sk_get_projection(ctx, y) != SK_OK ||
        sk_get_residual(ctx, res) != SK_OK) {
        fprintf(stderr, "shiftk: %s\n", sk_last_error());
        return 1;
    }
    sk_coeffs c;
    sk_get_coefficients(ctx, &c);
    for (int64_t k = 0; k < nz; ++k)
        printf("%.6f %.12e %.3e\n", z[k].re, -y[k].im / M_PI, res[k]);
    printf("status %d iterations %lld switches %lld\n", status, (long long)c.iterations,
           (long long)c.switches);
    sk_finalize(&ctx);
    free(b); free(z); free(y); free(res);
    return status == SK_CONVERGED ? 0 : 2;
}
