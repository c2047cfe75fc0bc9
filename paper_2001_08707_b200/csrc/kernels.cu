// kernels.cu — the sm_100a kernels of one shifted COCG / BiCG iteration.
//
//   a1+a2  heisenberg_kernel / csr_kernel : q = H r_n (BiCG: also qt = H r~_n), fused partial
//          w = <r~|r, q> per CTA (unconjugated for COCG, App. A; conjugated for BiCG,
//          P:L1014)
//   a3-a9  scalar_kernel (1 CTA)           : deterministic reduction of the partials, seed
//          recurrences, per-shift pi/alpha/beta, projected
//          u/y update (corrected index R1), residuals, retirement,
//          seed switching
//   a5+a7  update_kernel                    : r_{n+1} = (1+c-alpha z_s) r_n + alpha q - c r_{n-1}
//          (EQ-CG-RN-3REC P:L269; shadow P:L1029) fused with the dots of the next iteration
//          (rho, ||r||^2, a_l^dag r) and, in full mode, the all-shift update
//          p^k = r_n/pi^k + beta^k p^k, x^k += alpha^k p^k for every active shift.
//
// All reductions are two-stage and deterministic: each CTA reduces its grid-stride rows in a
// fixed order, the scalar kernel sums the CTA partials in CTA order.
#include "kernels.cuh"

namespace sk {

enum { ST_ITERATING = 0, ST_CONVERGED = 1, ST_MAXITER = 2, ST_BREAKDOWN = 3 };

// select one of three by-value pointers without dynamic indexing (keeps them in registers)
template <typename T>
__device__ __forceinline__ T pick3(T const (&a)[3], int64_t i) {
    const int k = (int)(i % 3);
    return k == 0 ? a[0] : (k == 1 ? a[1] : a[2]);
}

int stream_blocks(int64_t M) {
    int64_t b = (M + kThreads - 1) / kThreads;
    if (b > kMaxBlocks) b = kMaxBlocks;
    if (b < 1) b = 1;
    return (int)b;
}

// ============================================================================ Heisenberg H.v
// H = J sum_{i<L} S_i.S_{i+1}, periodic.  x = s XOR rot(s) has bit i set iff sites i,
// i+1 are anti-aligned; diagonal = J/4 (L - 2 popc(x)); each anti-aligned bond flips both spins
// with amplitude J/2.  Bond loop is uniform across the warp so every gather r[s ^ m_i] of a
// warp reads one contiguous 512-byte block (coalesced).
template <int NRHS>
__global__ void __launch_bounds__(kThreads) heisenberg_kernel(SpmvArgs a, int L, double J) {
    int buf = 0;
    if (a.st) {
        if (a.st->status != ST_ITERATING) return;
        buf = (int)(a.st->n_started % 3);
    }
    const cplx *__restrict__ r = pick3(a.r, buf);
    const cplx *__restrict__ t = pick3(a.t, buf);
    const double qJ = 0.25 * J, hJ = 0.5 * J;
    const int64_t M = a.M;
    cplx w = mk(0.0, 0.0);
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < M;
         s += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t us = (uint64_t)s;
        const uint64_t rot = (us >> 1) | ((us & 1ull) << (L - 1));
        const uint64_t x = us ^ rot;
        const double d = qJ * (double)(L - 2 * __popcll(x));
        const cplx rs = r[s];
        cplx q = mk(d * rs.x, d * rs.y);
        cplx ts, qt;
        if (NRHS == 2) {
            ts = t[s];
            qt = mk(d * ts.x, d * ts.y);
        }
        for (int i = 0; i < L; ++i) {
            if ((x >> i) & 1ull) {
                const int j = (i + 1 == L) ? 0 : i + 1;
                const uint64_t s2 = us ^ ((1ull << i) | (1ull << j));
                const cplx v = r[s2];
                q.x = fma(hJ, v.x, q.x);
                q.y = fma(hJ, v.y, q.y);
                if (NRHS == 2) {
                    const cplx vt = t[s2];
                    qt.x = fma(hJ, vt.x, qt.x);
                    qt.y = fma(hJ, vt.y, qt.y);
                }
            }
        }
        a.q[s] = q;
        if (NRHS == 2) {
            a.qt[s] = qt;
            w = cfma_conj(ts, q, w);
        } else {
            w = cfma(rs, q, w);
        }
    }
    if (a.part_w) {
        __shared__ cplx scratch[kThreads / 32];
        cplx v[1] = {w};
        block_sum<1>(v, scratch);
        if (threadIdx.x == 0) a.part_w[blockIdx.x] = v[0];
    }
}

// ============================================================================ CSR SpMV
// LPR lanes per row (LPR | 32), lanes stride over the row's entries, shuffle-reduce in the
// group.  Column ids are int32, row pointers int64, values fp64 or complex128.
template <int LPR, bool CV, int NRHS>
__global__ void __launch_bounds__(kThreads)
csr_kernel(SpmvArgs a, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
           const void *__restrict__ valv) {
    int buf = 0;
    if (a.st) {
        if (a.st->status != ST_ITERATING) return;
        buf = (int)(a.st->n_started % 3);
    }
    const cplx *__restrict__ r = pick3(a.r, buf);
    const cplx *__restrict__ t = pick3(a.t, buf);
    const int lane = threadIdx.x & (LPR - 1);
    const unsigned gmask = (LPR == 32) ? 0xffffffffu
                                       : (((1u << LPR) - 1u) << ((threadIdx.x & 31) & ~(LPR - 1)));
    const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / LPR;
    cplx w = mk(0.0, 0.0);
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPR; i < a.M; i += ngroups) {
        const int64_t e0 = rp[i], e1 = rp[i + 1];
        cplx acc = mk(0.0, 0.0), acct = mk(0.0, 0.0);
        for (int64_t e = e0 + lane; e < e1; e += LPR) {
            const int c = col[e];
            const cplx rv = r[c];
            if (CV) {
                const cplx v = ((const cplx *)valv)[e];
                acc = cfma(v, rv, acc);
                if (NRHS == 2) acct = cfma(v, t[c], acct);
            } else {
                const double v = ((const double *)valv)[e];
                acc.x = fma(v, rv.x, acc.x);
                acc.y = fma(v, rv.y, acc.y);
                if (NRHS == 2) {
                    const cplx tv = t[c];
                    acct.x = fma(v, tv.x, acct.x);
                    acct.y = fma(v, tv.y, acct.y);
                }
            }
        }
#pragma unroll
        for (int o = LPR / 2; o > 0; o >>= 1) {
            acc.x += __shfl_xor_sync(gmask, acc.x, o);
            acc.y += __shfl_xor_sync(gmask, acc.y, o);
            if (NRHS == 2) {
                acct.x += __shfl_xor_sync(gmask, acct.x, o);
                acct.y += __shfl_xor_sync(gmask, acct.y, o);
            }
        }
        if (lane == 0) {
            a.q[i] = acc;
            if (NRHS == 2) {
                a.qt[i] = acct;
                w = cfma_conj(t[i], acc, w);
            } else {
                w = cfma(r[i], acc, w);
            }
        }
    }
    if (a.part_w) {
        __shared__ cplx scratch[kThreads / 32];
        cplx v[1] = {w};
        block_sum<1>(v, scratch);
        if (threadIdx.x == 0) a.part_w[blockIdx.x] = v[0];
    }
}

cudaError_t launch_heisenberg(const SpmvArgs &a, int L, double J, int nblk, cudaStream_t s) {
    if (a.bicg)
        heisenberg_kernel<2><<<nblk, kThreads, 0, s>>>(a, L, J);
    else
        heisenberg_kernel<1><<<nblk, kThreads, 0, s>>>(a, L, J);
    return cudaGetLastError();
}

template <int LPR>
static void csr_dispatch(const SpmvArgs &a, const int64_t *rp, const int32_t *col, const void *val,
                         bool cv, int nblk, cudaStream_t s) {
    if (cv) {
        if (a.bicg) csr_kernel<LPR, true, 2><<<nblk, kThreads, 0, s>>>(a, rp, col, val);
        else csr_kernel<LPR, true, 1><<<nblk, kThreads, 0, s>>>(a, rp, col, val);
    } else {
        if (a.bicg) csr_kernel<LPR, false, 2><<<nblk, kThreads, 0, s>>>(a, rp, col, val);
        else csr_kernel<LPR, false, 1><<<nblk, kThreads, 0, s>>>(a, rp, col, val);
    }
}

cudaError_t launch_csr(const SpmvArgs &a, const int64_t *rp, const int32_t *col, const void *val,
                       bool cv, double avg_nnz, int nblk, cudaStream_t s) {
    if (avg_nnz <= 3.0) csr_dispatch<2>(a, rp, col, val, cv, nblk, s);
    else if (avg_nnz <= 6.0) csr_dispatch<4>(a, rp, col, val, cv, nblk, s);
    else if (avg_nnz <= 24.0) csr_dispatch<8>(a, rp, col, val, cv, nblk, s);
    else csr_dispatch<32>(a, rp, col, val, cv, nblk, s);
    return cudaGetLastError();
}

// ============================================================================ RC dot / init
__global__ void __launch_bounds__(kThreads) rc_dot_kernel(KParams kp, const cplx *__restrict__ q) {
    if (kp.st->status != ST_ITERATING) return;
    const int buf = (int)(kp.st->n_started % 3);
    const cplx *__restrict__ tv = kp.bicg ? pick3(kp.t, buf) : pick3(kp.r, buf);
    cplx w = mk(0.0, 0.0);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < kp.M;
         i += (int64_t)gridDim.x * blockDim.x)
        w = kp.bicg ? cfma_conj(tv[i], q[i], w) : cfma(tv[i], q[i], w);
    __shared__ cplx scratch[kThreads / 32];
    cplx v[1] = {w};
    block_sum<1>(v, scratch);
    if (threadIdx.x == 0) kp.part_w[blockIdx.x] = v[0];
}

cudaError_t launch_rc_dot(const KParams &kp, const cplx *q, cudaStream_t s) {
    rc_dot_kernel<<<kp.nblk_spmv, kThreads, 0, s>>>(kp, q);
    return cudaGetLastError();
}

template <int NLMAX>
__global__ void __launch_bounds__(kThreads) init_kernel(KParams kp, const cplx *__restrict__ b) {
    cplx acc[2 + NLMAX];
#pragma unroll
    for (int j = 0; j < 2 + NLMAX; ++j) acc[j] = mk(0.0, 0.0);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < kp.M;
         i += (int64_t)gridDim.x * blockDim.x) {
        const cplx bi = b[i];
        kp.r[0][i] = bi;
        if (kp.bicg) kp.t[0][i] = cconj(bi);   // r~_0 = conj(b)  (R3)
        acc[0] = cfma(bi, bi, acc[0]);          // rho_0 = <r~_0, r_0> = sum b_i^2 for both methods
        acc[1].x = fma(bi.x, bi.x, fma(bi.y, bi.y, acc[1].x));
#pragma unroll
        for (int l = 0; l < NLMAX; ++l)
            if (l < kp.nl) acc[2 + l] = cfma_conj(kp.left[(int64_t)l * kp.M + i], bi, acc[2 + l]);
    }
    __shared__ cplx scratch[(2 + NLMAX) * (kThreads / 32)];
    block_sum<2 + NLMAX>(acc, scratch);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int j = 0; j < 2 + NLMAX; ++j)
            if (j < 2 + kp.nl) kp.part_u[(int64_t)blockIdx.x * (2 + kp.nl) + j] = acc[j];
    }
}

// ============================================================================ fused update
template <int NLMAX, bool BICG, bool FULL>
__global__ void __launch_bounds__(kThreads)
update_kernel(KParams kp, const cplx *__restrict__ q, const cplx *__restrict__ qt) {
    extern __shared__ cplx dyn[];  // FULL: coef[3 * nact], then act list (int32)
    DevState *st = kp.st;
    if (st->status != ST_ITERATING) return;
    const int64_t ns = st->n_started;            // start(n) ran: ns = n + 1
    const cplx *__restrict__ rc_ = pick3(kp.r, ns + 2);
    const cplx *__restrict__ rp_ = pick3(kp.r, ns + 1);
    cplx *__restrict__ rn_ = pick3(kp.r, ns);
    const cplx *__restrict__ tc_ = pick3(kp.t, ns + 2);
    const cplx *__restrict__ tp_ = pick3(kp.t, ns + 1);
    cplx *__restrict__ tn_ = pick3(kp.t, ns);
    const cplx a_cur = st->a_cur, a_q = st->a_q, a_prev = st->a_prev;
    const cplx ac_cur = cconj(a_cur), ac_q = cconj(a_q), ac_prev = cconj(a_prev);
    int nact = 0;
    cplx *coef = dyn;
    int *act = nullptr;
    if (FULL) {
        nact = *kp.n_act_list;
        act = (int *)(dyn + 3 * kp.nz);
        for (int j = threadIdx.x; j < 3 * nact; j += blockDim.x) coef[j] = kp.coef[j];
        for (int j = threadIdx.x; j < nact; j += blockDim.x) act[j] = kp.act_list[j];
        __syncthreads();
    }
    cplx acc[2 + NLMAX];
#pragma unroll
    for (int j = 0; j < 2 + NLMAX; ++j) acc[j] = mk(0.0, 0.0);
    const int64_t M = kp.M;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M;
         i += (int64_t)gridDim.x * blockDim.x) {
        const cplx rc = ldg_cs(rc_ + i);
        const cplx rp = ldg_cs(rp_ + i);
        const cplx qi = ldg_cs(q + i);
        cplx rn = cmul(a_cur, rc);
        rn = cfma(a_q, qi, rn);
        rn = cfma(a_prev, rp, rn);
        rn_[i] = rn;
        if (BICG) {
            const cplx tc = ldg_cs(tc_ + i), tp = ldg_cs(tp_ + i), qti = ldg_cs(qt + i);
            cplx tn = cmul(ac_cur, tc);
            tn = cfma(ac_q, qti, tn);
            tn = cfma(ac_prev, tp, tn);
            tn_[i] = tn;
            acc[0] = cfma_conj(tn, rn, acc[0]);
        } else {
            acc[0] = cfma(rn, rn, acc[0]);
        }
        acc[1].x = fma(rn.x, rn.x, fma(rn.y, rn.y, acc[1].x));
#pragma unroll
        for (int l = 0; l < NLMAX; ++l)
            if (l < kp.nl) acc[2 + l] = cfma_conj(ldg_cs(kp.left + (int64_t)l * M + i), rn, acc[2 + l]);
        if (FULL) {
            int j = 0;
            for (; j + 4 <= nact; j += 4) {
                cplx pk[4], xk[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int64_t off = (int64_t)act[j + u] * M + i;
                    pk[u] = ldg_cs(kp.p + off);
                    xk[u] = ldg_cs(kp.x + off);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int64_t off = (int64_t)act[j + u] * M + i;
                    cplx pn = cmul(coef[3 * (j + u)], rc);
                    pn = cfma(coef[3 * (j + u) + 1], pk[u], pn);
                    const cplx xn = cfma(coef[3 * (j + u) + 2], pn, xk[u]);
                    stg_cs(kp.p + off, pn);
                    stg_cs(kp.x + off, xn);
                }
            }
            for (; j < nact; ++j) {
                const int64_t off = (int64_t)act[j] * M + i;
                const cplx pk = ldg_cs(kp.p + off), xk = ldg_cs(kp.x + off);
                cplx pn = cmul(coef[3 * j], rc);
                pn = cfma(coef[3 * j + 1], pk, pn);
                stg_cs(kp.p + off, pn);
                stg_cs(kp.x + off, cfma(coef[3 * j + 2], pn, xk));
            }
        }
    }
    __shared__ cplx scratch[(2 + NLMAX) * (kThreads / 32)];
    block_sum<2 + NLMAX>(acc, scratch);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int j = 0; j < 2 + NLMAX; ++j)
            if (j < 2 + kp.nl) kp.part_u[(int64_t)blockIdx.x * (2 + kp.nl) + j] = acc[j];
    }
}

template <int NLMAX>
static cudaError_t launch_update_nl(const KParams &kp, const cplx *q, const cplx *qt, cudaStream_t s) {
    const size_t shm = kp.full ? (size_t)kp.nz * (3 * sizeof(cplx) + sizeof(int)) : 0;
    if (kp.full) {
        if (kp.bicg) {
            cudaFuncSetAttribute(update_kernel<NLMAX, true, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
            update_kernel<NLMAX, true, true><<<kp.nblk_upd, kThreads, shm, s>>>(kp, q, qt);
        } else {
            cudaFuncSetAttribute(update_kernel<NLMAX, false, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
            update_kernel<NLMAX, false, true><<<kp.nblk_upd, kThreads, shm, s>>>(kp, q, qt);
        }
    } else {
        if (kp.bicg) update_kernel<NLMAX, true, false><<<kp.nblk_upd, kThreads, 0, s>>>(kp, q, qt);
        else update_kernel<NLMAX, false, false><<<kp.nblk_upd, kThreads, 0, s>>>(kp, q, qt);
    }
    return cudaGetLastError();
}

cudaError_t launch_update(const KParams &kp, const cplx *q, const cplx *qt, cudaStream_t s) {
    if (kp.nl <= 1) return launch_update_nl<1>(kp, q, qt, s);
    if (kp.nl <= 4) return launch_update_nl<4>(kp, q, qt, s);
    if (kp.nl <= 8) return launch_update_nl<8>(kp, q, qt, s);
    if (kp.nl <= 16) return launch_update_nl<16>(kp, q, qt, s);
    return launch_update_nl<32>(kp, q, qt, s);
}

cudaError_t launch_init(const KParams &kp, const cplx *b, cudaStream_t s) {
    if (kp.nl <= 1) init_kernel<1><<<kp.nblk_upd, kThreads, 0, s>>>(kp, b);
    else if (kp.nl <= 4) init_kernel<4><<<kp.nblk_upd, kThreads, 0, s>>>(kp, b);
    else if (kp.nl <= 8) init_kernel<8><<<kp.nblk_upd, kThreads, 0, s>>>(kp, b);
    else if (kp.nl <= 16) init_kernel<16><<<kp.nblk_upd, kThreads, 0, s>>>(kp, b);
    else init_kernel<32><<<kp.nblk_upd, kThreads, 0, s>>>(kp, b);
    return cudaGetLastError();
}

// ============================================================================ scalar kernel
// One CTA of kScalarThreads threads.  Shared broadcast slots + deterministic block reductions.
struct ScalarShared {
    cplx red[kScalarThreads / 32 + 1];
    double redd[kScalarThreads / 32];
    int redi[kScalarThreads / 32];
    cplx g[64];
    cplx bc[8];      // broadcast scalars
    int bci[4];
};

__device__ cplx block_allsum(cplx v, ScalarShared &sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    if (lane == 0) sh.red[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        cplx s = sh.red[0];
        for (int w = 1; w < nw; ++w) s = cadd(s, sh.red[w]);
        sh.red[32] = s;
    }
    __syncthreads();
    const cplx r = sh.red[32];
    __syncthreads();
    return r;
}

__device__ int block_allsum_int(int v, ScalarShared &sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sh.redi[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
        for (int w = 0; w < nw; ++w) s += sh.redi[w];
        sh.bci[3] = s;
    }
    __syncthreads();
    const int r = sh.bci[3];
    __syncthreads();
    return r;
}

// Sum partial column j of part[nblk][stride] in fixed order -> broadcast.
__device__ cplx reduce_partials(const cplx *part, int nblk, int stride, int j, ScalarShared &sh) {
    cplx v = mk(0.0, 0.0);
    for (int b = threadIdx.x; b < nblk; b += blockDim.x) v = cadd(v, part[(int64_t)b * stride + j]);
    return block_allsum(v, sh);
}

// argmin over active shifts of |pi_k|, ties -> lowest k; returns -1 if none active.
__device__ int block_argmin_active(const KParams &kp, ScalarShared &sh) {
    double best = 0.0;
    int bi = -1;
    for (int k = threadIdx.x; k < kp.nz; k += blockDim.x) {
        if (!kp.active[k]) continue;
        const double v = cabsd(kp.pi[k]);
        if (bi < 0 || v < best) { best = v; bi = k; }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (oi >= 0 && (bi < 0 || ov < best || (ov == best && oi < bi))) { best = ov; bi = oi; }
    }
    if (lane == 0) { sh.redd[warp] = best; sh.redi[warp] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = 0.0; int i = -1;
        for (int w = 0; w < nw; ++w) {
            const int oi = sh.redi[w]; const double ov = sh.redd[w];
            if (oi >= 0 && (i < 0 || ov < b || (ov == b && oi < i))) { b = ov; i = oi; }
        }
        sh.bci[2] = i;
    }
    __syncthreads();
    const int r = sh.bci[2];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kScalarThreads) scalar_kernel(KParams kp, int phases) {
    __shared__ ScalarShared sh;
    DevState *st = kp.st;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int nred = 2 + kp.nl;

    if (phases & PH_INIT) {
        const cplx rho = reduce_partials(kp.part_u, kp.nblk_upd, nred, 0, sh);
        const double nu = sqrt(reduce_partials(kp.part_u, kp.nblk_upd, nred, 1, sh).x);
        for (int l = 0; l < kp.nl; ++l) {
            const cplx g = reduce_partials(kp.part_u, kp.nblk_upd, nred, 2 + l, sh);
            if (tid == 0) kp.g[l] = g;
        }
        for (int k = tid; k < kp.nz; k += nt) kp.res[k] = nu;
        if (tid == 0) { st->rho_cur = rho; st->nu = nu; }
        return;
    }

    const int pending = st->pending;
    __syncthreads();
    if ((phases & PH_FINISH) && pending) {
        // --- a8: residuals of r_{n+1} (stored unscaled), retirement ------------------------
        cplx rho = reduce_partials(kp.part_u, kp.nblk_upd, nred, 0, sh);
        double nu = sqrt(reduce_partials(kp.part_u, kp.nblk_upd, nred, 1, sh).x);
        for (int l = 0; l < kp.nl; ++l) {
            const cplx g = reduce_partials(kp.part_u, kp.nblk_upd, nred, 2 + l, sh);
            if (tid == 0) sh.g[l] = g;
        }
        const int64_t n = st->n + 1;
        const double tol = st->tol;
        int cnt = 0;
        for (int k = tid; k < kp.nz; k += nt) {
            if (!kp.active[k]) continue;
            const double res = nu / cabsd(kp.pi[k]);
            kp.res[k] = res;
            if (res < tol) { kp.active[k] = 0; kp.retired_at[k] = n; }
            else ++cnt;
        }
        __syncthreads();
        cnt = block_allsum_int(cnt, sh);
        // --- a9: seed switching --------------------------------------------------------------
        int best = -1;
        if (cnt > 0) best = block_argmin_active(kp, sh);
        const int doswitch = cnt > 0 && !(kp.flags & 1) && best != st->seed;
        cplx f = mk(1.0, 0.0), fp = mk(1.0, 0.0);
        if (doswitch) {
            f = kp.pi[best];
            fp = kp.pi_old[best];
            __syncthreads();   // everyone read pi[best] before it is rescaled
            const cplx rf = crecip(f), rfp = crecip(fp);
            for (int k = tid; k < kp.nz; k += nt) {
                if (!kp.active[k]) continue;
                kp.pi[k] = cmul(kp.pi[k], rf);
                kp.pi_old[k] = cmul(kp.pi_old[k], rfp);
            }
        }
        __syncthreads();
        if (tid == 0) {
            if (doswitch) {   // DESIGN.md R9: the new seed's r, r_prev, pi, alpha, rho
                st->sr_cur = cdiv(st->sr_cur, f);                          // r_{n+1} /= f
                st->sr_prev = cdiv(st->sr_prev, fp);                       // r_n /= f'
                st->alpha_prev = cmul(st->alpha_prev, cdiv(fp, f));        // alpha_n^{s*}
                st->rho_prev = cdiv(st->rho_prev, cmul(fp, fp));           // rho_n / f'^2
                rho = cdiv(rho, cmul(f, f));                               // rho_{n+1} / f^2
                nu = nu / cabsd(f);
                for (int l = 0; l < kp.nl; ++l) sh.g[l] = cdiv(sh.g[l], f);
                st->zs = kp.z[best];
                st->seed = best;
                st->nswitch += 1;
            }
            st->rho_cur = rho;
            st->nu = nu;
            for (int l = 0; l < kp.nl; ++l) kp.g[l] = sh.g[l];
            st->n = n;
            st->pending = 0;
            st->n_active = cnt;
            if (cnt == 0) st->status = ST_CONVERGED;
            else if (n >= st->itermax) st->status = ST_MAXITER;
        }
        __syncthreads();
    }

    if (!(phases & PH_START)) return;
    if (st->status != ST_ITERATING) return;   // uniform: written before the last barrier

    // --- a3: seed scalars ---------------------------------------------------------------------
    const cplx wraw = reduce_partials(kp.part_w, kp.nblk_spmv, 1, 0, sh);
    if (tid == 0) {
        const cplx sr = st->sr_cur;
        const cplx w = cmul(cmul(sr, sr), wraw);   // w_n = <r~_n|r_n, H r_n> (true scale)
        const cplx rho = st->rho_cur;
        const int64_t n = st->n;
        cplx beta = mk(0, 0), gamma = mk(0, 0);
        if (n > 0) {
            beta = cdiv(rho, st->rho_prev);           // EQ-REC-BETA P:L262
            gamma = cdiv(beta, st->alpha_prev);
        }
        // EQ-REC-ALPHA-N2: alpha = rho / (<r, A r> - gamma rho), <r, A r> = z_s rho - w
        const cplx den = csub(csub(cmul(st->zs, rho), w), cmul(gamma, rho));
        int brk = (cabsd(rho) < 1e-300) || (cabsd(den) < 1e-300);
        cplx alpha = mk(0, 0), c = mk(0, 0);
        if (!brk) {
            alpha = cdiv(rho, den);
            c = cmul(alpha, gamma);
        }
        sh.bc[0] = alpha; sh.bc[1] = beta; sh.bc[2] = c;
        sh.bci[0] = brk;
        st->alpha = alpha; st->beta = beta; st->w = w;
        if (brk) st->status = ST_BREAKDOWN;
    }
    __syncthreads();
    if (sh.bci[0]) return;
    const cplx alpha = sh.bc[0], beta = sh.bc[1], c = sh.bc[2];
    const cplx zs = st->zs, sr = st->sr_cur;
    const int64_t n = st->n;
    const int nl = kp.nl;

    // compacted active list (ascending shift order): the full-mode kernel streams only these
    int nact = 0;
    {
        const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
        for (int base = 0; base < kp.nz; base += nt) {
            const int k = base + tid;
            const int a = (k < kp.nz) ? (int)kp.active[k] : 0;
            const unsigned bal = __ballot_sync(0xffffffffu, a);
            const int wpre = __popc(bal & ((1u << lane) - 1u));
            if (lane == 0) sh.redi[warp] = __popc(bal);
            __syncthreads();
            if (tid == 0) {
                int acc = 0;
                for (int w = 0; w < nw; ++w) { const int v = sh.redi[w]; sh.redi[w] = acc; acc += v; }
                sh.bci[1] = acc;
            }
            __syncthreads();
            if (a) kp.act_list[nact + sh.redi[warp] + wpre] = k;
            nact += sh.bci[1];
            __syncthreads();
        }
        if (tid == 0) *kp.n_act_list = nact;
    }
    __syncthreads();

    // --- a4 + a6 + (a7 coefficients): per-shift recurrences -------------------------------------
    const cplx one = mk(1.0, 0.0);
    for (int j = tid; j < nact; j += nt) {
        const int k = kp.act_list[j];
        const cplx pik = kp.pi[k], pio = kp.pi_old[k];
        const cplx sigma = csub(kp.z[k], zs);
        // EQ-SHIFTEDCG-PI: pi_{n+1} = (1 + c + alpha sigma) pi_n - c pi_{n-1}
        const cplx pin = csub(cmul(cadd(cadd(one, c), cmul(alpha, sigma)), pik), cmul(c, pio));
        const cplx ak = cmul(cdiv(pik, pin), alpha);
        cplx bk = mk(0, 0);
        if (n > 0) { const cplx rat = cdiv(pio, pik); bk = cmul(cmul(rat, rat), beta); }
        for (int l = 0; l < nl; ++l) {                                           // P:L372-376 (R1)
            const int64_t o = (int64_t)k * nl + l;
            const cplx u = cadd(cdiv(kp.g[l], pik), cmul(bk, kp.u[o]));
            kp.u[o] = u;
            kp.y[o] = cfma(ak, u, kp.y[o]);
        }
        kp.pi_old[k] = pik;
        kp.pi[k] = pin;
        if (kp.full) {
            kp.coef[3 * j] = cdiv(sr, pik);    // p^k = r_n/pi_n^k + ...   (r_n = sr * r_stored)
            kp.coef[3 * j + 1] = bk;
            kp.coef[3 * j + 2] = ak;
        }
    }
    __syncthreads();
    if (tid == 0) {
        // update coefficients (a5) in stored-vector form, then rotate the lazy scales
        st->a_cur = cmul(csub(cadd(one, c), cmul(alpha, zs)), sr);
        st->a_q = cmul(alpha, sr);
        st->a_prev = cmul(mk(-c.x, -c.y), st->sr_prev);
        st->sr_prev = sr;
        st->sr_cur = one;
        st->alpha_prev = alpha;
        st->rho_prev = st->rho_cur;
        st->n_started = n + 1;
        st->pending = 1;
        st->nspmv += kp.bicg ? 2 : 1;
    }
}

cudaError_t launch_scalar(const KParams &kp, int phases, cudaStream_t s) {
    scalar_kernel<<<1, kScalarThreads, 0, s>>>(kp, phases);
    return cudaGetLastError();
}

}  // namespace sk
