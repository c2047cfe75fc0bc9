// spmv_sz.cu — the Heisenberg chain restricted to a sector of fixed S^z.
// H conserves the number n of up spins, so it is block diagonal over sectors; HPhi runs the
// 2Sz = 0 sector (dimension C(L, L/2): 924 at L=12).  Sector basis
// (R28): the L-bit states with popcount n in ascending integer order, row i = the
// i-th one.  rank(s) = sum over the set bits of s, taken in ascending position p_1 < p_2 < ...,
// of C(p_m, m) (the states below s, counted by their highest differing bit).
//
// One thread per row: unrank i bit by bit from the top (C(p, m) from a per-CTA shared-memory
// table), diagonal J/4 (L - 2 popc(s XOR rot s)), and for each anti-aligned bond the partner's
// row from the rank of s itself: moving the m-th set bit between positions j and j+1 changes
// exactly one term, C(j, m) <-> C(j+1, m), i.e. the rank by +-C(j, m-1).  Only the periodic
// bond (L-1, 0) renumbers the set bits; its partner is ranked from scratch.  The gathers are
// the cost: a partner of a low bond lies next to the row (coalesced across the warp), a partner
// of a high bond C(j, m-1) rows away.
#include "kernels.cuh"
#include "spmv_common.cuh"

namespace sk {

constexpr int kSzMaxL = 34;

template <int NRHS>
__global__ void __launch_bounds__(kThreads) heisenberg_sz_kernel(SpmvArgs a, KParams kp, int L, int nup, double J) {
    __shared__ StepScratch sc;
    __shared__ unsigned long long C[kSzMaxL + 1][kSzMaxL + 2];   // C[n][k], zero for k > n
    bool agent;
    int buf;
    if (!spmv_enter(a, agent, buf, sc, kp)) return;
    const cplx *__restrict__ r = pick3(a.r, buf);
    const cplx *__restrict__ t = pick3(a.t, buf);
    const double qJ = 0.25 * J, hJ = 0.5 * J;
    const int64_t M = a.M;
    const int off = a.st ? 1 : 0;
    cplx w = mk(0.0, 0.0);
    if (!agent) {
        for (int e = threadIdx.x; e < (kSzMaxL + 1) * (kSzMaxL + 2); e += blockDim.x) {
            const int n = e / (kSzMaxL + 2), k = e % (kSzMaxL + 2);
            unsigned long long c = 0;
            if (k <= n) {   // exact: C(n, j) * (n - k + j) / j stays below 2^40 for n <= 34
                c = 1;
                for (int j = 1; j <= k; ++j) c = c * (unsigned long long)(n - k + j) / (unsigned long long)j;
            }
            C[n][k] = c;
        }
        __syncthreads();
        for (int64_t i = (int64_t)(blockIdx.x - off) * blockDim.x + threadIdx.x; i < M;
             i += (int64_t)(gridDim.x - off) * blockDim.x) {
            // unrank
            uint64_t s = 0;
            {
                uint64_t rank = (uint64_t)i;
                int m = nup;
                for (int p = L - 1; p >= 0 && m > 0; --p) {
                    const uint64_t below = C[p][m];
                    if (rank >= below) {
                        s |= 1ull << p;
                        rank -= below;
                        --m;
                    }
                }
            }
            const uint64_t x = s ^ ((s >> 1) | ((s & 1ull) << (L - 1)));
            const double d = qJ * (double)(L - 2 * __popcll(x));
            const cplx rs = r[i];
            cplx q = mk(d * rs.x, d * rs.y);
            cplx ts = mk(0, 0), qt = mk(0, 0);
            if (NRHS == 2) { ts = t[i]; qt = mk(d * ts.x, d * ts.y); }
            uint64_t xb = x & ((1ull << (L - 1)) - 1ull);   // open bonds (j, j+1), j < L-1
            while (xb) {
                const int j = __ffsll((long long)xb) - 1;
                xb &= xb - 1ull;
                const int m = __popcll(s & ((2ull << (j + 1)) - 1ull));   // index of the moving bit
                const int64_t delta = (int64_t)C[j][m - 1];
                const int64_t pr = ((s >> j) & 1ull) ? i + delta : i - delta;
                const cplx v = r[pr];
                q.x = fma(hJ, v.x, q.x);
                q.y = fma(hJ, v.y, q.y);
                if (NRHS == 2) {
                    const cplx vt = t[pr];
                    qt.x = fma(hJ, vt.x, qt.x);
                    qt.y = fma(hJ, vt.y, qt.y);
                }
            }
            if ((x >> (L - 1)) & 1ull) {   // periodic bond (L-1, 0): rank the partner afresh
                uint64_t s2 = s ^ (1ull | (1ull << (L - 1)));
                int64_t pr = 0;
                for (int m = 1; s2; ++m) {
                    const int p = __ffsll((long long)s2) - 1;
                    s2 &= s2 - 1ull;
                    pr += (int64_t)C[p][m];
                }
                const cplx v = r[pr];
                q.x = fma(hJ, v.x, q.x);
                q.y = fma(hJ, v.y, q.y);
                if (NRHS == 2) {
                    const cplx vt = t[pr];
                    qt.x = fma(hJ, vt.x, qt.x);
                    qt.y = fma(hJ, vt.y, qt.y);
                }
            }
            a.q[i] = q;
            if (NRHS == 2) {
                a.qt[i] = qt;
                w = cfma_conj(ts, q, w);
            } else {
                w = cfma(rs, q, w);
            }
        }
    }
    spmv_exit(a, kp, agent, w, sc);
}

cudaError_t launch_heisenberg_sz(const SpmvArgs &a, const KParams &kp, int L, int nup, double J, cudaStream_t s) {
    const int grid = stream_blocks(a.M) + (a.st ? 1 : 0);
    const bool p = a.st != nullptr;
    if (a.bicg) return launch_k(heisenberg_sz_kernel<2>, grid, kThreads, 0, s, p, a, kp, L, nup, J);
    return launch_k(heisenberg_sz_kernel<1>, grid, kThreads, 0, s, p, a, kp, L, nup, J);
}

}  // namespace sk
