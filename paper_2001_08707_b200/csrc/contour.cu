// contour.cu — the device work of the contour-integral eigensolver
// on top of the shifted solver's full-mode solutions x^(j) = (z_j I - H)^{-1} phi:
//   * sk_combine: out[c] = sum_j W[j][c] X[j] — the moments s_k = sum_j w_j (z_j - z0)^k x^(j)
//     (P:L708-712 by the trapezoidal rule on z_j) and the Rayleigh-Ritz basis
//     U~ = S V Sigma^{-1}; one streaming pass over X per 8 outputs, W broadcast from L1;
//   * sk_gram: G = A^dagger B — S^dagger S (the SVD of the tall S through its Gram matrix) and
//     U~^dagger H U~; per-CTA partials over 32-row chunks staged in shared memory,
//     then a fixed-order sum (deterministic).
// The M_nz x M_nz eigenproblems are solved on the host (a few dozen rows; SURVEY f-2).
#include <cuda_runtime.h>

#include "../../include/shiftk.h"
#include "kernels.cuh"

namespace sk {

constexpr int kCombineOut = 8;     // outputs per pass (accumulators per thread)
constexpr int kGramRows = 32;      // rows per staged chunk
constexpr int kGramMax = 64;       // na, nb limit

__global__ void __launch_bounds__(kThreads) combine_kernel(const cplx *__restrict__ X, int64_t n_in, int64_t ld,
                                                           int64_t M, const cplx *__restrict__ W, int n_out, int c0,
                                                           int nc, cplx *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
        cplx acc[kCombineOut];
#pragma unroll
        for (int c = 0; c < kCombineOut; ++c) acc[c] = mk(0.0, 0.0);
        int64_t j = 0;
        for (; j + 4 <= n_in; j += 4) {
            cplx x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = ldg_cs(X + (j + u) * ld + i);
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int c = 0; c < kCombineOut; ++c)
                    if (c < nc) acc[c] = cfma(__ldg(W + (j + u) * n_out + c0 + c), x[u], acc[c]);
        }
        for (; j < n_in; ++j) {
            const cplx x = ldg_cs(X + j * ld + i);
#pragma unroll
            for (int c = 0; c < kCombineOut; ++c)
                if (c < nc) acc[c] = cfma(__ldg(W + j * n_out + c0 + c), x, acc[c]);
        }
#pragma unroll
        for (int c = 0; c < kCombineOut; ++c)
            if (c < nc) out[(int64_t)(c0 + c) * M + i] = acc[c];
    }
}

__global__ void __launch_bounds__(kThreads) gram_kernel(const cplx *__restrict__ A, int na, const cplx *__restrict__ B,
                                                        int nb, int64_t M, cplx *__restrict__ part) {
    extern __shared__ cplx st[];   // [na][kGramRows] then [nb][kGramRows]
    cplx *As = st, *Bs = st + (size_t)na * kGramRows;
    constexpr int PP = kGramMax * kGramMax / kThreads;   // pairs per thread (max)
    cplx acc[PP];
#pragma unroll
    for (int m = 0; m < PP; ++m) acc[m] = mk(0.0, 0.0);
    const int np = na * nb;
    const int64_t nchunk = (M + kGramRows - 1) / kGramRows;
    for (int64_t ch = blockIdx.x; ch < nchunk; ch += gridDim.x) {
        const int64_t r0 = ch * kGramRows;
        __syncthreads();
        for (int e = threadIdx.x; e < (na + nb) * kGramRows; e += blockDim.x) {
            const int v = e / kGramRows, r = e % kGramRows;
            const int64_t i = r0 + r;
            cplx val = mk(0.0, 0.0);
            if (i < M) val = v < na ? A[(int64_t)v * M + i] : B[(int64_t)(v - na) * M + i];
            st[e] = val;
        }
        __syncthreads();
#pragma unroll
        for (int m = 0; m < PP; ++m) {
            const int p = threadIdx.x + m * kThreads;
            if (p >= np) break;
            const int a = p / nb, b = p % nb;
            cplx s = acc[m];
            for (int r = 0; r < kGramRows; ++r) s = cfma_conj(As[a * kGramRows + r], Bs[b * kGramRows + r], s);
            acc[m] = s;
        }
    }
#pragma unroll
    for (int m = 0; m < PP; ++m) {
        const int p = threadIdx.x + m * kThreads;
        if (p < np) part[(int64_t)blockIdx.x * np + p] = acc[m];
    }
}

__global__ void gram_reduce_kernel(const cplx *__restrict__ part, int nblk, int np, cplx *__restrict__ G) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= np) return;
    cplx s = mk(0.0, 0.0);
    for (int b = 0; b < nblk; ++b) s = cadd(s, part[(int64_t)b * np + p]);
    G[p] = s;
}

}  // namespace sk


int sk_set_error(int code, const char *msg);   // api.cu

extern "C" {

int sk_combine(const sk_cplx *X, int64_t n_in, int64_t ld_x, int64_t M, const sk_cplx *W, int64_t n_out,
               sk_cplx *out, void *stream) {
    if (!X || !W || !out || n_in < 1 || n_out < 1 || M < 1 || ld_x < M || n_out > 4096)
        return sk_set_error(SK_EINVAL, "sk_combine: arguments");
    cudaStream_t s = (cudaStream_t)stream;
    cplx *Wd = nullptr;
    const size_t wb = sizeof(cplx) * (size_t)n_in * (size_t)n_out;
    if (cudaMallocAsync((void **)&Wd, wb, s) != cudaSuccess) return sk_set_error(SK_ECUDA, "sk_combine: W");
    if (cudaMemcpyAsync(Wd, W, wb, cudaMemcpyHostToDevice, s) != cudaSuccess)
        return sk_set_error(SK_ECUDA, "sk_combine: W copy");
    int64_t g = (M + sk::kThreads - 1) / sk::kThreads;
    if (g > 4 * sk::sm_count()) g = 4 * sk::sm_count();
    for (int c0 = 0; c0 < n_out; c0 += sk::kCombineOut) {
        const int nc = (int)(n_out - c0 < sk::kCombineOut ? n_out - c0 : sk::kCombineOut);
        sk::combine_kernel<<<(int)g, sk::kThreads, 0, s>>>((const cplx *)X, n_in, ld_x, M, Wd, (int)n_out, c0, nc,
                                                           (cplx *)out);
    }
    cudaFreeAsync(Wd, s);   // (the copy is stream-ordered before the kernels; W may be reused now)
    if (cudaStreamSynchronize(s) != cudaSuccess || cudaGetLastError() != cudaSuccess)
        return sk_set_error(SK_ECUDA, "sk_combine: kernel");
    return SK_OK;
}

int sk_gram(const sk_cplx *A, int64_t na, const sk_cplx *B, int64_t nb, int64_t M, sk_cplx *G, void *stream) {
    if (!A || !B || !G || na < 1 || nb < 1 || na > sk::kGramMax || nb > sk::kGramMax || M < 1)
        return sk_set_error(SK_EINVAL, "sk_gram: arguments (na, nb <= 64)");
    cudaStream_t s = (cudaStream_t)stream;
    const int np = (int)(na * nb);
    int64_t g = (M + sk::kGramRows - 1) / sk::kGramRows;
    if (g > 2 * sk::sm_count()) g = 2 * sk::sm_count();
    cplx *part = nullptr, *Gd = nullptr;
    if (cudaMallocAsync((void **)&part, sizeof(cplx) * (size_t)g * np, s) != cudaSuccess ||
        cudaMallocAsync((void **)&Gd, sizeof(cplx) * (size_t)np, s) != cudaSuccess)
        return sk_set_error(SK_ECUDA, "sk_gram: scratch");
    const size_t shm = sizeof(cplx) * (size_t)(na + nb) * sk::kGramRows;
    static sk::PerDevice cfg;
    if (sk::once_per_device(cfg, [] {
            return cudaFuncSetAttribute(sk::gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)(sizeof(cplx) * 2 * sk::kGramMax * sk::kGramRows));
        }) != cudaSuccess)
        return sk_set_error(SK_ECUDA, "sk_gram: shared-memory attribute");
    sk::gram_kernel<<<(int)g, sk::kThreads, shm, s>>>((const cplx *)A, (int)na, (const cplx *)B, (int)nb, M, part);
    sk::gram_reduce_kernel<<<(np + 255) / 256, 256, 0, s>>>(part, (int)g, np, Gd);
    const cudaError_t e1 = cudaMemcpyAsync(G, Gd, sizeof(cplx) * (size_t)np, cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(part, s);
    cudaFreeAsync(Gd, s);
    if (e1 != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess || cudaGetLastError() != cudaSuccess)
        return sk_set_error(SK_ECUDA, "sk_gram: kernel");
    return SK_OK;
}

}  // extern "C"
