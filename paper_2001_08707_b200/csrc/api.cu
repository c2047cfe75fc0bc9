// api.cu — the C-ABI of libshiftk.so (include/shiftk.h): context lifecycle, iteration
// enqueueing (single step / CUDA-graph captured loop), getters.  Every step of the method runs in
// the kernels of kernels.cu; this file only allocates, enqueues and copies.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/shiftk.h"
#include "kernels.cuh"

using sk::LoopbackPtrs;


static thread_local std::string g_err = "no error";

static int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

// error reporting for the other translation units (contour.cu)
int sk_set_error(int code, const char *msg) { return fail(code, msg); }

#define CK(call)                                                                                 \
    do {                                                                                         \
        cudaError_t e_ = (call);                                                                 \
        if (e_ != cudaSuccess)                                                                   \
            return fail(SK_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));            \
    } while (0)

// ---- NCCL, loaded on first multi-rank use (the torch-bundled libnccl.so.2; no link-time
// dependency, so single-GPU users never need it) ----------------------------------------------
struct NcclApi {
    bool ok = false;
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char *(*getErrorString)(ncclResult_t) = nullptr;
};
static NcclApi &nccl() {
    static NcclApi api;
    static bool tried = false;
    if (tried) return api;
    tried = true;
    void *h = nullptr;
    if (const char *p = getenv("SHIFTK_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen(SHIFTK_NCCL_DEFAULT, RTLD_NOW | RTLD_GLOBAL);
    if (!h) return api;
    api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
    api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
    api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
    api.getErrorString = (decltype(api.getErrorString))dlsym(h, "ncclGetErrorString");
    api.ok = api.getUniqueId && api.commInitRank && api.allReduce && api.commDestroy && api.getErrorString;
    return api;
}

#define NK(call)                                                                                 \
    do {                                                                                         \
        ncclResult_t e_ = (call);                                                                \
        if (e_ != ncclSuccess)                                                                   \
            return fail(SK_ENCCL, std::string(#call) + ": " + nccl().getErrorString(e_));         \
    } while (0)

struct sk_group {   // single-GPU loopback group: `world` virtual ranks in one process
    int world = 0, device = 0;
    cudaStream_t stream = nullptr;
    std::vector<sk_ctx *> members;
    bool connected = false;
};

struct sk_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    sk_operator op{};
    int method = SK_COCG, full = 0, flags = 0;
    int64_t M = 0;
    int nz = 0, nl = 0;
    bool a_is_b = true;
    double tol = 0, avg_nnz = 0;
    int64_t itermax = 0;
    KParams kp{};
    DevState *st = nullptr;       // device
    DevState *st_host = nullptr;  // pinned mirror
    cplx *b = nullptr;            // device copy of b
    cplx *left_owned = nullptr;
    std::vector<void *> allocs;
    cudaGraphExec_t graph = nullptr;    // `graph_iters` iterations (sk_run chunks)
    int graph_iters = 0;
    cudaGraphExec_t graph1 = nullptr;   // one iteration (the remainders, single sk_enqueue steps)
    int64_t host_started = 0;     // iterations enqueued (host view, for RC pointers)
    bool pending_host = false;    // an update ran whose finish phase is not yet enqueued
    // tracing
    bool capturing = false;
    bool profiling = false;
    int64_t launches = 0;
    std::vector<cudaEvent_t> ev_pool;  // 4 per profiled iteration
    size_t ev_used = 0;
    int64_t prof_iters = 0;
    double prof_ms[3] = {0, 0, 0};
    // multi-rank
    int world = 1, rank = 0;
    sk_group *group = nullptr;      // loopback group (single GPU), or
    ncclComm_t comm = nullptr;      // NCCL communicator (one process per GPU)
    bool connected = true;          // false until sk_connect / sk_group_connect
    void *arena = nullptr;
    size_t arena_bytes = 0;
    double b_norm = 0;              // ||b|| (global), recorded at initialisation
    std::vector<void *> peer_bases; // opened IPC mappings of the other ranks' arenas
    sk_allreduce_fn host_ar = nullptr;   // host all-reduce (sk_connect_host) instead of NCCL
    void *host_ar_user = nullptr;
    double *host_stage = nullptr;        // pinned [2][2 (2 + nl)] doubles: send, recv
};

static cudaError_t prof_mark(sk_ctx *c) {
    if (!c->profiling || c->capturing) return cudaSuccess;
    if (c->ev_used == c->ev_pool.size()) {
        cudaEvent_t e;
        cudaError_t r = cudaEventCreate(&e);
        if (r != cudaSuccess) return r;
        c->ev_pool.push_back(e);
    }
    return cudaEventRecord(c->ev_pool[c->ev_used++], c->stream);
}

static int dalloc(sk_ctx *c, void **p, size_t bytes) {
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(SK_ENOMEM, "cudaMalloc(" + std::to_string(bytes) + " B): " + cudaGetErrorString(e));
    }
    c->allocs.push_back(*p);
    CK(cudaMemsetAsync(*p, 0, bytes, c->stream));
    return SK_OK;
}

static void destroy(sk_ctx *c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->graph) cudaGraphExecDestroy(c->graph);
    if (c->graph1) cudaGraphExecDestroy(c->graph1);
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    for (void *p : c->peer_bases)
        if (p) cudaIpcCloseMemHandle(p);
    if (c->comm && nccl().ok) nccl().commDestroy(c->comm);
    if (c->group && c->rank < (int)c->group->members.size()) c->group->members[c->rank] = nullptr;
    for (void *p : c->allocs) cudaFree(p);
    if (c->st_host) cudaFreeHost(c->st_host);
    if (c->host_stage) cudaFreeHost(c->host_stage);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

// --------------------------------------------------------------------------- enqueue helpers
// One iteration (world == 1) = two launches:
//   SpMV (+ finish of the previous iteration in CTA 0, + seed scalars in the last CTA)
//   update (+ per-shift recurrences in the agent CTAs).
// world > 1: SpMV (peer loads through the shard tables; last CTA -> this rank's w) ->
//   all-reduce(w) -> seed kernel -> update (last CTA -> this rank's dots) -> all-reduce(dots).
static int enqueue_phase_a(sk_ctx *c, const cplx *q_rc, const cplx *qt_rc, sk::SpmvArgs &a) {
    a = sk::SpmvArgs{};
    a.st = c->st;
    for (int i = 0; i < 3; ++i) { a.r[i] = c->kp.r[i]; a.t[i] = c->kp.t[i]; }
    a.q = q_rc ? (cplx *)q_rc : c->kp.q;
    a.qt = q_rc ? (cplx *)qt_rc : c->kp.qt;
    a.part_w = c->kp.part_w;
    a.work = c->kp.work;
    a.grp = c->kp.grp;
    a.M = c->M;
    a.bicg = c->method == SK_BICG;
    CK(prof_mark(c));
    if (q_rc)
        CK(sk::launch_rc_dot(a, c->kp, c->stream));
    else if (c->op.kind == SK_OP_HEISENBERG)
        CK(sk::launch_heisenberg(a, c->kp, c->op.L, c->op.J, c->stream));
    else if (c->op.kind == SK_OP_HEISENBERG_SZ)
        CK(sk::launch_heisenberg_sz(a, c->kp, c->op.L, c->op.n_up, c->op.J, c->stream));
    else
        CK(sk::launch_csr(a, c->kp, c->op.row_ptr, c->op.col, c->op.val, c->op.kind == SK_OP_CSR_CPLX,
                          c->avg_nnz, c->stream));
    CK(prof_mark(c));
    if (!c->capturing) c->launches += (!q_rc && c->kp.csr_nblk >= 2) ? c->kp.csr_nblk : 1;
    return SK_OK;
}

static int enqueue_phase_b(sk_ctx *c, const sk::SpmvArgs &a) {
    CK(sk::launch_update(c->kp, a.q, a.qt, c->stream));
    CK(prof_mark(c));
    if (!c->capturing) c->launches += 1;
    c->host_started += 1;
    c->pending_host = true;
    return SK_OK;
}

static int nccl_allreduce(sk_ctx *c, const cplx *src, cplx *dst, int ncplx) {
    if (c->host_ar) {   // sk_connect_host: through the caller's host collective
        const int64_t n = 2 * (int64_t)ncplx;
        double *snd = c->host_stage, *rcv = c->host_stage + n;
        CK(cudaMemcpyAsync(snd, src, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (c->host_ar(c->host_ar_user, snd, rcv, n) != 0) return fail(SK_ENCCL, "host all-reduce callback failed");
        CK(cudaMemcpyAsync(dst, rcv, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));   // (the staging buffer is reused by the next call)
        return SK_OK;
    }
    NK(nccl().allReduce(src, dst, 2 * (size_t)ncplx, ncclDouble, ncclSum, c->comm, c->stream));
    return SK_OK;
}

static int enqueue_iteration(sk_ctx *c, const cplx *q_rc, const cplx *qt_rc) {
    if (!c->connected) return fail(SK_ESTATE, "multi-rank context not connected (sk_connect)");
    if (c->group) return fail(SK_ESTATE, "loopback group member: use sk_group_update / sk_group_run");
    sk::SpmvArgs a;
    int rc;
    if ((rc = enqueue_phase_a(c, q_rc, qt_rc, a)) != SK_OK) return rc;
    if (c->world > 1) {
        if ((rc = nccl_allreduce(c, c->kp.wloc, c->kp.wsum, 1)) != SK_OK) return rc;
        CK(sk::launch_seed(c->kp, c->stream));
        if (!c->capturing) c->launches += 1;
    }
    if ((rc = enqueue_phase_b(c, a)) != SK_OK) return rc;
    if (c->world > 1 && (rc = nccl_allreduce(c, c->kp.uloc, c->kp.usum, 2 + c->nl)) != SK_OK) return rc;
    return SK_OK;
}

// Loopback all-reduce over the members of a single-GPU group (deterministic, rank order).
static int group_allreduce(sk_group *g, bool dots) {
    LoopbackPtrs p{};
    int n = 0;
    for (int r = 0; r < g->world; ++r) {
        sk_ctx *m = g->members[r];
        p.src[r] = dots ? m->kp.uloc : m->kp.wloc;
        p.dst[r] = dots ? m->kp.usum : m->kp.wsum;
        n = dots ? 2 + m->nl : 1;
    }
    sk_ctx *m0 = g->members[0];
    cudaError_t e = sk::launch_loopback_allreduce(p, g->world, n, g->stream);
    if (e != cudaSuccess) return fail(SK_ECUDA, std::string("loopback all-reduce: ") + cudaGetErrorString(e));
    m0->launches += 1;
    return SK_OK;
}

static int group_iteration(sk_group *g) {
    std::vector<sk::SpmvArgs> a(g->world);
    int rc;
    for (int r = 0; r < g->world; ++r)
        if ((rc = enqueue_phase_a(g->members[r], nullptr, nullptr, a[r])) != SK_OK) return rc;
    if ((rc = group_allreduce(g, false)) != SK_OK) return rc;
    for (int r = 0; r < g->world; ++r) {
        CK(sk::launch_seed(g->members[r]->kp, g->stream));
        g->members[r]->launches += 1;
    }
    for (int r = 0; r < g->world; ++r)
        if ((rc = enqueue_phase_b(g->members[r], a[r])) != SK_OK) return rc;
    return group_allreduce(g, true);
}

// (every context entry point reaches the device through here or read_state: both select the
// context's device first, so a caller whose current device differs is served correctly)
static int enqueue_finish(sk_ctx *c) {
    CK(cudaSetDevice(c->device));
    if (!c->pending_host) return SK_OK;
    CK(sk::launch_scalar(c->kp, sk::PH_FINISH, c->stream));
    c->launches += 1;
    c->pending_host = false;
    return SK_OK;
}

static int read_state(sk_ctx *c) {
    CK(cudaSetDevice(c->device));
    CK(cudaMemcpyAsync(c->st_host, c->st, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return SK_OK;
}

// --------------------------------------------------------------------------- C-ABI
extern "C" {

const char *sk_last_error(void) { return g_err.c_str(); }

const char *sk_version(void) {
    return "shiftk 0.1 (sm_100a; shifted COCG/BiCG, Heisenberg + CSR operators)";
}

int sk_init(sk_ctx **out, const sk_operator *H, const sk_params *p, const sk_dist *d) {
    if (!out || !H || !p) return fail(SK_EINVAL, "null argument");
    *out = nullptr;
    const int world = d ? (d->world < 1 ? 1 : d->world) : 1;
    const int rank = d ? d->rank : 0;
    sk_group *group = d ? (sk_group *)d->group : nullptr;
    if (world > sk::kMaxWorld) return fail(SK_EUNSUPPORTED, "world > 64");
    if (rank < 0 || rank >= world) return fail(SK_EINVAL, "rank out of range");
    if (group && (group->world != world || group->members[rank] != nullptr))
        return fail(SK_EINVAL, "group size mismatch or rank already initialised");
    if (p->method != SK_COCG && p->method != SK_BICG) return fail(SK_EINVAL, "method");
    if (p->n_shift < 1 || !p->z) return fail(SK_EINVAL, "n_shift >= 1 and z required");
    if (!(p->tol > 0)) return fail(SK_EINVAL, "tol must be > 0");
    if (p->itermax < 1) return fail(SK_EINVAL, "itermax must be >= 1");
    if (!p->b) return fail(SK_EINVAL, "b required");
    if (p->n_left < 0 || (p->n_left > 0 && !p->left) || (p->n_left == 0 && p->left))
        return fail(SK_EINVAL, "n_left/left inconsistent");
    if (p->n_left > 32) return fail(SK_EUNSUPPORTED, "n_left > 32");
    if (p->n_shift > (1 << 20)) return fail(SK_EUNSUPPORTED, "n_shift > 2^20");
    if ((p->flags & SK_FLAG_LOG) && p->itermax > (int64_t(1) << 24))
        return fail(SK_EINVAL, "SK_FLAG_LOG needs itermax <= 2^24 (one log entry per iteration)");
    const int64_t M = H->M_local > 0 ? H->M_local : H->M;
    if (world > 1) {   // rows [rank * M_local, (rank + 1) * M_local), M_local a power of two
        if (M * world != H->M || (M & (M - 1)) != 0 || H->row_begin != (int64_t)rank * M)
            return fail(SK_EINVAL, "multi-rank: need M = world * M_local, M_local a power of two, "
                                   "row_begin = rank * M_local");
        if (H->kind == SK_OP_RC) return fail(SK_EUNSUPPORTED, "reverse communication with world > 1");
    }
    switch (H->kind) {
        case SK_OP_HEISENBERG:
            if (H->L < 1 || H->L > 34 || H->M != (int64_t(1) << H->L) || (world == 1 && M != H->M))
                return fail(SK_EINVAL, "Heisenberg: need 1 <= L <= 34, M = 2^L");
            break;
        case SK_OP_CSR_REAL:
        case SK_OP_CSR_CPLX:
            if (!H->row_ptr || !H->col || !H->val || M < 1 || H->nnz < 0)
                return fail(SK_EINVAL, "CSR arrays / sizes");
            if (world == 1 && M != H->M) return fail(SK_EINVAL, "CSR: M_local must equal M when world == 1");
            if (H->kind == SK_OP_CSR_CPLX && p->method == SK_COCG)
                return fail(SK_EUNSUPPORTED,
                            "COCG needs a complex-symmetric z I - H: use BiCG for complex "
                            "Hermitian H (Table 1, P:L211-216)");
            break;
        case SK_OP_RC:
            if (M < 1) return fail(SK_EINVAL, "M");
            break;
        case SK_OP_HEISENBERG_SZ: {
            if (H->L < 1 || H->L > 34 || H->n_up < 0 || H->n_up > H->L)
                return fail(SK_EINVAL, "Heisenberg sector: need 1 <= L <= 34, 0 <= n_up <= L");
            int64_t dim = 1;   // C(L, n_up)
            for (int j = 1; j <= H->n_up; ++j) dim = dim * (H->L - H->n_up + j) / j;
            if (H->M != dim || M != H->M) return fail(SK_EINVAL, "Heisenberg sector: need M = C(L, n_up)");
            if (world > 1) return fail(SK_EUNSUPPORTED, "Heisenberg sector operator with world > 1");
            break;
        }
        default:
            return fail(SK_EINVAL, "operator kind");
    }

    sk_ctx *c = new (std::nothrow) sk_ctx();
    if (!c) return fail(SK_ENOMEM, "host allocation");
    c->device = group ? group->device : (d ? d->device : 0);
    c->world = world;
    c->rank = rank;
    c->group = group;
    c->connected = world == 1;
    c->op = *H;
    c->method = p->method;
    c->full = p->full_x ? 1 : 0;
    c->flags = p->flags;
    c->M = M;
    c->nz = (int)p->n_shift;
    c->a_is_b = p->n_left == 0;
    c->nl = c->a_is_b ? 1 : (int)p->n_left;
    c->tol = p->tol;
    c->itermax = p->itermax;
    c->avg_nnz = (H->kind == SK_OP_CSR_REAL || H->kind == SK_OP_CSR_CPLX) ? double(H->nnz) / double(M) : 0;
    int rc = SK_OK;
    auto bail = [&](int code) { destroy(c); return code; };

    if (cudaSetDevice(c->device) != cudaSuccess) return bail(fail(SK_ECUDA, "cudaSetDevice"));
    if (group) {
        c->stream = group->stream;   // every member of a loopback group shares one stream
    } else if (d && d->stream) {
        c->stream = (cudaStream_t)d->stream;
    } else {
        if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
            return bail(fail(SK_ECUDA, "cudaStreamCreate"));
        c->own_stream = true;
    }
    if (cudaMallocHost((void **)&c->st_host, sizeof(DevState)) != cudaSuccess)
        return bail(fail(SK_ENOMEM, "cudaMallocHost"));

    KParams &kp = c->kp;
    kp.M = M;
    kp.nz = c->nz;
    kp.nl = c->nl;
    kp.bicg = c->method == SK_BICG;
    kp.full = c->full;
    kp.a_is_b = c->a_is_b;
    kp.flags = c->flags;
    kp.J = H->J;
    kp.split_ahi = sk::split_ahi_for(H->L, M, world, kp.bicg, c->full, c->nl, H->kind == SK_OP_HEISENBERG);
    kp.nblk_spmv = H->kind == SK_OP_HEISENBERG ? sk::heisenberg_blocks(H->L, M, kp.bicg, kp.split_ahi > 0)
                   : H->kind == SK_OP_HEISENBERG_SZ ? sk::sz_blocks(H->L, M, kp.bicg)
                   : H->kind == SK_OP_RC ? sk::stream_blocks(M) : sk::csr_blocks(M);
    kp.nblk_upd = sk::update_blocks(M, c->nl, c->full, c->nz);
    if (kp.split_ahi) {
        kp.nblk_upd = sk::split_blocks();
        kp.split_lo = sk::split_lo_bonds();
        // the fused r_{n-1} term lives in the tiled H_A kernel only
        kp.split_fuse = sk::split_fuse_enabled() && !sk::heis_stream(H->L, M, kp.bicg, true);
    }
    // column-blocked CSR passes (spmv.cu): opt-in (SHIFTK_CSR_BLOCKED=1) — measured slower than
    // the one-pass kernel at C3 (4 blocks 4.21 ms, 2 blocks 3.70 ms vs 3.63 ms);
    // the split kernel below still checks that the rows qualify
    int csr_cand_nblk = 0;
    if ((H->kind == SK_OP_CSR_REAL || H->kind == SK_OP_CSR_CPLX) && world == 1 && sk::csr_blocked_env() == 1) {
        const int bs = sk::csr_block_shift();
        const int64_t nb = (M + (int64_t(1) << bs) - 1) >> bs;
        if (nb >= 2 && nb <= 16 && M < (int64_t(1) << 31)) csr_cand_nblk = (int)nb;
    }
    kp.n_agents = sk::shift_agents(c->nz);
    kp.world = world;
    kp.rank = rank;
    kp.row0 = world > 1 ? (int64_t)rank * M : 0;
    kp.lloc_bits = 0;
    while ((int64_t(1) << kp.lloc_bits) < M) ++kp.lloc_bits;
    const size_t vb = (size_t)M * sizeof(cplx);

    // One device arena for everything the context owns (one cudaMalloc / cudaFree); every
    // array is padded to 256 B so bulk (TMA) copies of rounded sizes stay inside it.
    cplx *zdev = nullptr;
    unsigned long long *csr_stats = nullptr;
    {
        struct Item { void **p; size_t bytes; };
        std::vector<Item> items;
        auto add = [&](void *pp, size_t bytes) { items.push_back({(void **)pp, bytes}); };
        add(&c->st, sizeof(DevState));
        for (int i = 0; i < 3; ++i) add(&kp.r[i], vb);
        if (kp.bicg)
            for (int i = 0; i < 3; ++i) add(&kp.t[i], vb);
        if (H->kind != SK_OP_RC) {
            add(&kp.q, vb);
            if (kp.bicg) add(&kp.qt, vb);
        }
        add(&c->b, vb);
        {   // per-CTA partials, or the streaming SpMV's per-tile + per-group partials
            int64_t np = sk::kMaxSpmvBlocks, ng = 1;
            // the w partials the seed step reduces: [wred_off, wred_off + wred_n) of a half
            kp.wred_off = 0;
            kp.wred_n = kp.nblk_spmv;
            if (H->kind == SK_OP_HEISENBERG && sk::heis_stream(H->L, M, kp.bicg, kp.split_ahi > 0)) {
                const int64_t nt = M >> sk::kTileBits;
                np = std::max<int64_t>(np, sk::stream_partials(nt));
                ng = std::max<int64_t>(1, (nt + sk::kStreamGroup - 1) / sk::kStreamGroup);
                kp.wred_off = nt <= sk::kStreamDirect ? 0 : nt;
                kp.wred_n = (int32_t)(nt <= sk::kStreamDirect ? nt : ng);
            }
            if (H->kind == SK_OP_HEISENBERG_SZ && sk::sz_partials(H->L) > 0) {   // per block + per group
                const int64_t nt = int64_t(1) << (H->L - std::min(H->L - 1, 12));
                np = std::max<int64_t>(np, sk::sz_partials(H->L));
                ng = std::max<int64_t>(1, (nt + sk::kStreamGroup - 1) / sk::kStreamGroup);
                kp.wred_off = nt <= sk::kStreamDirect ? 0 : nt;
                kp.wred_n = (int32_t)(nt <= sk::kStreamDirect ? nt : ng);
            }
            // deferred seed step on one GPU with the built-in operator: two halves (iteration
            // parity), because the next SpMV writes its partials while the finish reads these
            kp.defer = (world == 1 && H->kind != SK_OP_RC) ? 1 : 0;
            if (kp.split_ahi) {   // the update's w_B partials follow the SpMV's (same reduced range;
                                  // per-tile/group partials of the streaming kernel, else per CTA)
                kp.wsplit_off = kp.wred_off + kp.wred_n;
                kp.wred_n += kp.nblk_upd;
                np = std::max<int64_t>(np, kp.wsplit_off + kp.nblk_upd);
            }
            kp.wred_stride = np;
            add(&kp.part_w, sizeof(cplx) * np * 2);
            add(&kp.grp, sizeof(uint32_t) * ng);
        }
        add(&kp.part_u, sizeof(cplx) * sk::kMaxBlocks * (2 + c->nl));
        add(&zdev, sizeof(cplx) * c->nz);
        add(&kp.pibuf, sizeof(cplx) * 3 * c->nz);
        add(&kp.pi_frozen, sizeof(cplx) * c->nz);
        add(&kp.ticket, sizeof(uint32_t));
        if (csr_cand_nblk) {
            add(&kp.csr_split, (size_t)(csr_cand_nblk + 1) * (size_t)M);
            add(&csr_stats, 2 * sizeof(unsigned long long));
        }
        if (kp.split_ahi) {
            add(&kp.kflag, 2 * sizeof(uint32_t));   // [0] SpMV kappa flag, [1] "Im a != 0 somewhere"
            if (sk::split_left_real_enabled()) add(&kp.left_re, sizeof(double) * (size_t)M);
        }
        add(&kp.work, 2 * sizeof(unsigned long long));
        add(&kp.amin_part, sizeof(AminPart) * 8);
        add(&kp.active, c->nz);
        add(&kp.res, sizeof(double) * c->nz);
        add(&kp.retired_at, sizeof(int64_t) * c->nz);
        add(&kp.u, sizeof(cplx) * c->nz * c->nl);
        add(&kp.y, sizeof(cplx) * c->nz * c->nl);
        add(&kp.g, sizeof(cplx) * c->nl);
        if (getenv("SHIFTK_DEBUG_TS")) add(&kp.dbg_ts, sizeof(int64_t) * 16);
        if (p->flags & SK_FLAG_LOG) {
            kp.lg_cap = p->itermax;
            add(&kp.lg, sizeof(cplx) * 6 * (size_t)p->itermax);
            add(&kp.lg_nu, sizeof(double) * (size_t)p->itermax);
            add(&kp.lg_g, sizeof(cplx) * (size_t)p->itermax * c->nl);
        }
        if (world > 1) {
            add(&kp.wloc, sizeof(cplx));
            add(&kp.wsum, sizeof(cplx));
            add(&kp.uloc, sizeof(cplx) * (2 + c->nl));
            add(&kp.usum, sizeof(cplx) * (2 + c->nl));
            add(&kp.ticket_u, sizeof(uint32_t));
            add(&kp.shard_r, sizeof(cplx *) * 3 * world);
            add(&kp.shard_t, sizeof(cplx *) * 3 * world);
        }
        if (!c->a_is_b && p->left_mem != SK_MEM_DEVICE) add(&c->left_owned, vb * c->nl);
        if (c->full) {
            add(&kp.p, vb * c->nz);
            add(&kp.x, vb * c->nz);
        }
        size_t total = 0;
        for (auto &it : items) total += (it.bytes + 255) & ~size_t(255);
        void *arena = nullptr;
        if ((rc = dalloc(c, &arena, total)) != SK_OK) return bail(rc);
        c->arena = arena;
        c->arena_bytes = total;
        size_t off = 0;
        for (auto &it : items) {
            *it.p = (char *)arena + off;
            off += (it.bytes + 255) & ~size_t(255);
        }
    }
    kp.st = c->st;
    kp.z = zdev;

    // inputs
    const cudaMemcpyKind kb = p->b_mem == SK_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (cudaMemcpyAsync(c->b, p->b, vb, kb, c->stream) != cudaSuccess) return bail(fail(SK_ECUDA, "copy b"));
    if (cudaMemcpyAsync(zdev, p->z, sizeof(cplx) * c->nz, cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
        return bail(fail(SK_ECUDA, "copy z"));
    if (c->a_is_b) {
        kp.left = c->b;
    } else if (p->left_mem == SK_MEM_DEVICE) {
        kp.left = (const cplx *)p->left;
    } else {
        if (cudaMemcpyAsync(c->left_owned, p->left, vb * c->nl, cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
            return bail(fail(SK_ECUDA, "copy left"));
        kp.left = c->left_owned;
    }
    // per-shift init: pi_0 = pi_{-1} = 1, active, retired_at = -1
    {
        std::vector<cplx> ones(3 * (size_t)c->nz, mk(1.0, 0.0));   // pi_0 = pi_{-1} = 1
        std::vector<uint8_t> act(c->nz, 1);
        std::vector<int64_t> ret(c->nz, -1);
        if (cudaMemcpyAsync(kp.pibuf, ones.data(), sizeof(cplx) * 3 * c->nz, cudaMemcpyHostToDevice, c->stream) ||
            cudaMemcpyAsync(kp.active, act.data(), c->nz, cudaMemcpyHostToDevice, c->stream) ||
            cudaMemcpyAsync(kp.retired_at, ret.data(), sizeof(int64_t) * c->nz, cudaMemcpyHostToDevice, c->stream))
            return bail(fail(SK_ECUDA, "init per-shift arrays"));
        DevState h{};
        h.status = 0;
        h.seed = 0;
        h.n_active = c->nz;
        h.zs = mk(p->z[0].re, p->z[0].im);
        h.sr_cur = mk(1, 0);
        h.sr_prev = mk(1, 0);
        h.tol = c->tol;
        h.itermax = c->itermax;
        *c->st_host = h;
        if (cudaMemcpyAsync(c->st, c->st_host, sizeof(DevState), cudaMemcpyHostToDevice, c->stream))
            return bail(fail(SK_ECUDA, "init state"));
        // the pinned mirror is reused below; make sure the copy has consumed it
        if (cudaStreamSynchronize(c->stream)) return bail(fail(SK_ECUDA, "sync"));
    }
    if (csr_cand_nblk) {   // split points of the column blocks; blocking applies when the rows are
                           // sorted and short
        unsigned long long st2[2] = {1, 0};
        const int bs = sk::csr_block_shift();
        if (sk::launch_csr_split(M, H->row_ptr, H->col, csr_cand_nblk, bs, const_cast<uint8_t *>(kp.csr_split),
                                 csr_stats, c->stream) != cudaSuccess ||
            cudaMemcpyAsync(st2, csr_stats, sizeof(st2), cudaMemcpyDeviceToHost, c->stream) ||
            cudaStreamSynchronize(c->stream))
            return bail(fail(SK_ECUDA, "csr split kernel"));
        if (st2[0] == 0) {
            kp.csr_nblk = csr_cand_nblk;
            kp.csr_bshift = bs;
        }
    }
    if (sk::launch_init(kp, c->b, c->stream) != cudaSuccess) return bail(fail(SK_ECUDA, "init kernel"));
    if (kp.split_ahi && sk::launch_split_init(kp, c->stream) != cudaSuccess)
        return bail(fail(SK_ECUDA, "split init kernel"));
    if (kp.split_ahi && kp.left_re) {   // a real left vector (Im a = 0): 8 B/row in B-tile order
        uint32_t any_imag = 1;
        if (sk::launch_split_left(kp, const_cast<double *>(kp.left_re), kp.kflag + 1, c->stream) != cudaSuccess ||
            cudaMemcpyAsync(&any_imag, kp.kflag + 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream) ||
            cudaStreamSynchronize(c->stream))
            return bail(fail(SK_ECUDA, "split left kernel"));
        kp.left_real = any_imag ? 0 : 1;
    }
    if (world > 1) {   // the global rho_0, ||b||, P b need the other ranks: finished at connect
        if (sk::launch_reduce_local(kp, c->stream) != cudaSuccess) return bail(fail(SK_ECUDA, "init reduce"));
        if (group) group->members[rank] = c;
        *out = c;
        return SK_OK;
    }
    if (sk::launch_scalar(kp, sk::PH_INIT, c->stream) != cudaSuccess) return bail(fail(SK_ECUDA, "init scalar"));
    if ((rc = read_state(c)) != SK_OK) return bail(rc);
    if (!(c->st_host->nu > 0)) return bail(fail(SK_EINVAL, "||b|| must be > 0"));
    c->b_norm = c->st_host->nu;
    *out = c;
    return SK_OK;
}

// Shard tables: entry [b * world + g] = rank g's r[b] (t[b]), given every rank's arena base.
static int write_shard_tables(sk_ctx *c, const std::vector<char *> &bases) {
    std::vector<const cplx *> tr(3 * c->world), tt(3 * c->world);
    char *mine = (char *)c->arena;
    for (int b = 0; b < 3; ++b)
        for (int g = 0; g < c->world; ++g) {
            tr[b * c->world + g] = (const cplx *)(bases[g] + ((char *)c->kp.r[b] - mine));
            tt[b * c->world + g] = c->kp.bicg ? (const cplx *)(bases[g] + ((char *)c->kp.t[b] - mine)) : nullptr;
        }
    CK(cudaMemcpyAsync((void *)c->kp.shard_r, tr.data(), sizeof(cplx *) * tr.size(), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync((void *)c->kp.shard_t, tt.data(), sizeof(cplx *) * tt.size(), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return SK_OK;
}

static int finish_init(sk_ctx *c) {
    CK(sk::launch_scalar(c->kp, sk::PH_INIT, c->stream));
    int rc;
    if ((rc = read_state(c)) != SK_OK) return rc;
    if (!(c->st_host->nu > 0)) return fail(SK_EINVAL, "||b|| must be > 0");
    c->b_norm = c->st_host->nu;
    c->connected = true;
    return SK_OK;
}

int sk_recalc(sk_ctx *c, int64_t n_new, const sk_cplx *z_new, sk_cplx *y, double *res) {
    if (!c || !z_new || !y) return fail(c ? SK_EINVAL : SK_ESTATE, "null argument");
    if (!c->kp.lg) return fail(SK_ESTATE, "context created without SK_FLAG_LOG");
    if (n_new < 1 || n_new > (1 << 24)) return fail(SK_EINVAL, "n_new");
    CK(cudaSetDevice(c->device));
    int rc;
    if ((rc = enqueue_finish(c)) != SK_OK) return rc;
    if ((rc = read_state(c)) != SK_OK) return rc;
    const int64_t nlog = c->st_host->n < c->kp.lg_cap ? c->st_host->n : c->kp.lg_cap;
    // ||b|| = ||r_0||: the residual of a shift before any iteration
    double nu0 = 0;
    {
        const size_t nv = (size_t)n_new * c->nl;
        void *tmp = nullptr;
        const size_t bytes = sizeof(cplx) * (n_new + 2 * nv) + sizeof(double) * n_new;
        CK(cudaMallocAsync(&tmp, bytes, c->stream));
        cplx *zd = (cplx *)tmp, *yd = zd + n_new, *ud = yd + nv;
        double *rd = (double *)(ud + nv);
        CK(cudaMemcpyAsync(zd, z_new, sizeof(cplx) * n_new, cudaMemcpyHostToDevice, c->stream));
        nu0 = c->b_norm;
        CK(sk::launch_recalc(c->kp, nlog, zd, (int)n_new, c->tol, nu0, yd, ud, rd, c->stream));
        CK(cudaMemcpyAsync(y, yd, sizeof(cplx) * nv, cudaMemcpyDeviceToHost, c->stream));
        std::vector<double> rh(n_new);
        CK(cudaMemcpyAsync(rh.data(), rd, sizeof(double) * n_new, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaFreeAsync(tmp, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (res) memcpy(res, rh.data(), sizeof(double) * n_new);
    }
    return SK_OK;
}

// The arena holds every piece of solver state (borrowed inputs — CSR, device left vectors —
// live outside it), so a checkpoint is the arena bytes plus a small header; pointers inside it
// are not stored (buffers are addressed through KParams, rebuilt identically by sk_init).
struct CkptHeader {
    uint64_t magic, arena_bytes;
    int64_t M, nz, nl, world, rank;
    int32_t method, full;
};
static const uint64_t kCkptMagic = 0x324b5054504b4b53ull;   // "SKKPTPK2"

int sk_checkpoint(sk_ctx *c, void *buf, size_t *bytes) {
    if (!c || !bytes) return fail(c ? SK_EINVAL : SK_ESTATE, "null argument");
    const size_t need = sizeof(CkptHeader) + c->arena_bytes;
    if (!buf) { *bytes = need; return SK_OK; }
    if (*bytes < need) return fail(SK_EINVAL, "checkpoint buffer too small");
    CK(cudaSetDevice(c->device));
    int rc;
    if ((rc = enqueue_finish(c)) != SK_OK) return rc;
    CkptHeader h{kCkptMagic, c->arena_bytes, c->M, c->nz, c->nl, c->world, c->rank, c->method, c->full};
    memcpy(buf, &h, sizeof(h));
    CK(cudaMemcpyAsync((char *)buf + sizeof(h), c->arena, c->arena_bytes, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    *bytes = need;
    return SK_OK;
}

int sk_restore(sk_ctx *c, const void *buf, size_t bytes) {
    if (!c || !buf) return fail(c ? SK_EINVAL : SK_ESTATE, "null argument");
    CkptHeader h;
    if (bytes < sizeof(h)) return fail(SK_EINVAL, "checkpoint too small");
    memcpy(&h, buf, sizeof(h));
    if (h.magic != kCkptMagic || h.arena_bytes != c->arena_bytes || h.M != c->M || h.nz != c->nz ||
        h.nl != c->nl || h.world != c->world || h.rank != c->rank || h.method != c->method || h.full != c->full ||
        bytes < sizeof(h) + h.arena_bytes)
        return fail(SK_EINVAL, "checkpoint does not match this context (operator/parameters/placement)");
    CK(cudaSetDevice(c->device));
    CK(cudaStreamSynchronize(c->stream));
    // the shard tables hold this process's peer mappings: keep them across the restore
    std::vector<char> keep_r, keep_t;
    const size_t tab = sizeof(cplx *) * 3 * c->world;
    if (c->world > 1) {
        keep_r.resize(tab);
        keep_t.resize(tab);
        CK(cudaMemcpy(keep_r.data(), c->kp.shard_r, tab, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(keep_t.data(), c->kp.shard_t, tab, cudaMemcpyDeviceToHost));
    }
    CK(cudaMemcpyAsync(c->arena, (const char *)buf + sizeof(h), c->arena_bytes, cudaMemcpyHostToDevice, c->stream));
    if (c->world > 1) {
        CK(cudaMemcpyAsync((void *)c->kp.shard_r, keep_r.data(), tab, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync((void *)c->kp.shard_t, keep_t.data(), tab, cudaMemcpyHostToDevice, c->stream));
    }
    if (c->kp.split_ahi && c->kp.left_re) {   // the restored arena's left vector decides (kflag[1])
        uint32_t any_imag = 1;
        CK(cudaMemcpyAsync(&any_imag, c->kp.kflag + 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        c->kp.left_real = any_imag ? 0 : 1;
    }
    CK(cudaStreamSynchronize(c->stream));
    c->pending_host = false;   // the checkpoint was taken after a finish
    int rc;
    if ((rc = read_state(c)) != SK_OK) return rc;
    c->host_started = c->st_host->n_started;
    return SK_OK;
}

int sk_ipc_handle(sk_ctx *c, void *out64) {
    if (!c || !out64) return fail(c ? SK_EINVAL : SK_ESTATE, "null argument");
    cudaIpcMemHandle_t h;
    CK(cudaSetDevice(c->device));
    CK(cudaIpcGetMemHandle(&h, c->arena));
    memcpy(out64, &h, sizeof(h));
    return SK_OK;
}

int sk_nccl_unique_id(void *out128) {
    if (!out128) return fail(SK_EINVAL, "null argument");
    if (!nccl().ok) return fail(SK_ENCCL, "libnccl.so.2 not loadable");
    ncclUniqueId id;
    NK(nccl().getUniqueId(&id));
    memcpy(out128, &id, sizeof(id));
    return SK_OK;
}

// One-rank communicator on `device`: the dlopen'ed NCCL entry points, ncclCommInitRank, and the
// all-reduce the iteration uses (ncclDouble / ncclSum on a user stream) — once directly and once
// replayed from a captured CUDA graph (sk_run captures the iteration).  out1 / out2 receive the
// two results (with one rank: the input).
int sk_nccl_selftest(int32_t device, int64_t n, const double *in_host, double *out1_host, double *out2_host) {
    if (n < 1 || !in_host || !out1_host || !out2_host) return fail(SK_EINVAL, "null argument / n < 1");
    if (!nccl().ok) return fail(SK_ENCCL, "libnccl.so.2 not loadable");
    CK(cudaSetDevice(device));
    ncclUniqueId id;
    NK(nccl().getUniqueId(&id));
    ncclComm_t comm = nullptr;
    NK(nccl().commInitRank(&comm, 1, id, 0));
    cudaStream_t s = nullptr;
    double *d = nullptr;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    int rc = SK_OK;
    auto step = [&](cudaError_t e, const char *what) {
        if (rc == SK_OK && e != cudaSuccess) rc = fail(SK_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    };
    auto nstep = [&](ncclResult_t e, const char *what) {
        if (rc == SK_OK && e != ncclSuccess) rc = fail(SK_ENCCL, std::string(what) + ": " + nccl().getErrorString(e));
    };
    step(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    step(cudaMalloc(&d, 3 * sizeof(double) * n), "malloc");
    if (rc == SK_OK) {
        step(cudaMemcpyAsync(d, in_host, sizeof(double) * n, cudaMemcpyHostToDevice, s), "h2d");
        nstep(nccl().allReduce(d, d + n, (size_t)n, ncclDouble, ncclSum, comm, s), "ncclAllReduce");
        step(cudaStreamSynchronize(s), "sync");
    }
    if (rc == SK_OK) {
        step(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "begin capture");
        nstep(nccl().allReduce(d, d + 2 * n, (size_t)n, ncclDouble, ncclSum, comm, s), "ncclAllReduce (captured)");
        const cudaError_t e = cudaStreamEndCapture(s, &g);
        step(e, "end capture");
        if (rc == SK_OK) step(cudaGraphInstantiate(&ge, g, 0), "instantiate");
        if (rc == SK_OK) step(cudaGraphLaunch(ge, s), "graph launch");
        if (rc == SK_OK) step(cudaStreamSynchronize(s), "sync");
    }
    if (rc == SK_OK) {
        step(cudaMemcpy(out1_host, d + n, sizeof(double) * n, cudaMemcpyDeviceToHost), "d2h");
        step(cudaMemcpy(out2_host, d + 2 * n, sizeof(double) * n, cudaMemcpyDeviceToHost), "d2h");
    }
    if (ge) cudaGraphExecDestroy(ge);
    if (g) cudaGraphDestroy(g);
    if (d) cudaFree(d);
    if (s) cudaStreamDestroy(s);
    nccl().commDestroy(comm);
    return rc;
}

static int map_peers(sk_ctx *c, const void *handles) {
    CK(cudaSetDevice(c->device));
    std::vector<char *> bases(c->world);
    c->peer_bases.assign(c->world, nullptr);
    for (int g = 0; g < c->world; ++g) {
        if (g == c->rank) { bases[g] = (char *)c->arena; continue; }
        cudaIpcMemHandle_t h;
        memcpy(&h, (const char *)handles + 64 * g, sizeof(h));
        void *p = nullptr;
        CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        c->peer_bases[g] = p;
        bases[g] = (char *)p;
    }
    return write_shard_tables(c, bases);
}

int sk_connect(sk_ctx *c, const void *handles, const void *nccl_id) {
    if (!c || !handles || !nccl_id) return fail(c ? SK_EINVAL : SK_ESTATE, "null argument");
    if (c->world == 1 || c->group || c->connected) return fail(SK_ESTATE, "not an unconnected NCCL-mode context");
    if (!nccl().ok) return fail(SK_ENCCL, "libnccl.so.2 not loadable");
    int rc;
    if ((rc = map_peers(c, handles)) != SK_OK) return rc;
    ncclUniqueId id;
    memcpy(&id, nccl_id, sizeof(id));
    NK(nccl().commInitRank(&c->comm, c->world, id, c->rank));
    if ((rc = nccl_allreduce(c, c->kp.uloc, c->kp.usum, 2 + c->nl)) != SK_OK) return rc;
    return finish_init(c);
}

int sk_connect_host(sk_ctx *c, const void *handles, sk_allreduce_fn fn, void *user) {
    if (!c || !handles || !fn) return fail(c ? SK_EINVAL : SK_ESTATE, "null argument");
    if (c->world == 1 || c->group || c->connected) return fail(SK_ESTATE, "not an unconnected multi-rank context");
    int rc;
    if ((rc = map_peers(c, handles)) != SK_OK) return rc;
    if (cudaMallocHost((void **)&c->host_stage, sizeof(double) * 4 * (2 + c->nl)) != cudaSuccess)
        return fail(SK_ENOMEM, "cudaMallocHost (all-reduce staging)");
    c->host_ar = fn;
    c->host_ar_user = user;
    if ((rc = nccl_allreduce(c, c->kp.uloc, c->kp.usum, 2 + c->nl)) != SK_OK) return rc;
    return finish_init(c);
}

int sk_group_create(sk_group **out, int32_t world, int32_t device) {
    if (!out || world < 1 || world > sk::kMaxWorld) return fail(SK_EINVAL, "group size");
    sk_group *g = new (std::nothrow) sk_group();
    if (!g) return fail(SK_ENOMEM, "host allocation");
    g->world = world;
    g->device = device;
    g->members.assign(world, nullptr);
    if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete g;
        return fail(SK_ECUDA, "group stream");
    }
    *out = g;
    return SK_OK;
}

int sk_group_destroy(sk_group **pg) {
    if (!pg || !*pg) return fail(SK_ESTATE, "null group");
    sk_group *g = *pg;
    for (sk_ctx *m : g->members)
        if (m) return fail(SK_ESTATE, "finalize every member context first");
    cudaStreamSynchronize(g->stream);
    cudaStreamDestroy(g->stream);
    delete g;
    *pg = nullptr;
    return SK_OK;
}

int sk_group_connect(sk_group *g) {
    if (!g) return fail(SK_ESTATE, "null group");
    if (g->connected) return fail(SK_ESTATE, "group already connected");
    for (sk_ctx *m : g->members)
        if (!m) return fail(SK_ESTATE, "every rank of the group must be initialised first");
    std::vector<char *> bases(g->world);
    for (int r = 0; r < g->world; ++r) bases[r] = (char *)g->members[r]->arena;
    int rc;
    for (sk_ctx *m : g->members)
        if ((rc = write_shard_tables(m, bases)) != SK_OK) return rc;
    if ((rc = group_allreduce(g, true)) != SK_OK) return rc;
    for (sk_ctx *m : g->members)
        if ((rc = finish_init(m)) != SK_OK) return rc;
    g->connected = true;
    return SK_OK;
}

int sk_group_update(sk_group *g, int32_t *status) {
    if (!g || !g->connected) return fail(SK_ESTATE, "group not connected");
    CK(cudaSetDevice(g->device));
    int rc;
    for (sk_ctx *m : g->members)
        if ((rc = enqueue_finish(m)) != SK_OK) return rc;
    if ((rc = group_iteration(g)) != SK_OK) return rc;
    for (sk_ctx *m : g->members)
        if ((rc = enqueue_finish(m)) != SK_OK) return rc;
    if ((rc = read_state(g->members[0])) != SK_OK) return rc;
    if (status) *status = g->members[0]->st_host->status;
    return SK_OK;
}

int sk_group_run(sk_group *g, int64_t max_iters, int32_t *status) {
    if (!g || !g->connected) return fail(SK_ESTATE, "group not connected");
    CK(cudaSetDevice(g->device));
    int rc;
    if ((rc = read_state(g->members[0])) != SK_OK) return rc;
    int64_t done = 0;
    while (done < max_iters && g->members[0]->st_host->status == SK_ITERATING) {
        const int64_t chunk = max_iters - done < 64 ? max_iters - done : 64;
        for (int64_t i = 0; i < chunk; ++i)
            if ((rc = group_iteration(g)) != SK_OK) return rc;
        done += chunk;
        for (sk_ctx *m : g->members)
            if ((rc = enqueue_finish(m)) != SK_OK) return rc;
        if ((rc = read_state(g->members[0])) != SK_OK) return rc;
    }
    if (status) *status = g->members[0]->st_host->status;
    return SK_OK;
}

int sk_update(sk_ctx *c, int32_t *status) {
    if (!c) return fail(SK_ESTATE, "null context");
    if (c->op.kind == SK_OP_RC) return fail(SK_ESTATE, "SK_OP_RC context: use sk_update_rc");
    CK(cudaSetDevice(c->device));
    int rc;
    if ((rc = enqueue_finish(c)) != SK_OK) return rc;
    if ((rc = enqueue_iteration(c, nullptr, nullptr)) != SK_OK) return rc;
    if ((rc = enqueue_finish(c)) != SK_OK) return rc;
    if ((rc = read_state(c)) != SK_OK) return rc;
    if (status) *status = c->st_host->status;
    return SK_OK;
}

int sk_update_rc(sk_ctx *c, const sk_cplx *q, const sk_cplx *qt, int32_t *status) {
    if (!c) return fail(SK_ESTATE, "null context");
    if (!q || (c->method == SK_BICG && !qt)) return fail(SK_EINVAL, "q (and qt for BiCG) required");
    if (c->kp.split_ahi)   // its update adds H_B r itself (the library's own operator)
        return fail(SK_EUNSUPPORTED, "sk_update_rc on a bond-split Heisenberg context (SHIFTK_HEIS_SPLIT=0 disables the split)");
    CK(cudaSetDevice(c->device));
    int rc;
    if ((rc = enqueue_finish(c)) != SK_OK) return rc;
    if ((rc = enqueue_iteration(c, (const cplx *)q, (const cplx *)qt)) != SK_OK) return rc;
    if ((rc = enqueue_finish(c)) != SK_OK) return rc;
    if ((rc = read_state(c)) != SK_OK) return rc;
    if (status) *status = c->st_host->status;
    return SK_OK;
}

int sk_get_seed_vectors(sk_ctx *c, const sk_cplx **r, const sk_cplx **rt) {
    if (!c) return fail(SK_ESTATE, "null context");
    int rc;
    if ((rc = enqueue_finish(c)) != SK_OK) return rc;
    if ((rc = read_state(c)) != SK_OK) return rc;
    const int64_t i = c->st_host->n_started % 3;
    if (r) *r = (const sk_cplx *)c->kp.r[i];
    if (rt) *rt = c->method == SK_BICG ? (const sk_cplx *)c->kp.t[i] : nullptr;
    return SK_OK;
}

static int capture_graph(sk_ctx *c, int iters) {
    cudaGraphExec_t &slot = iters == 1 ? c->graph1 : c->graph;
    if (iters == 1 && c->graph1) return SK_OK;
    if (iters != 1 && c->graph && c->graph_iters == iters) return SK_OK;
    if (slot) {
        cudaGraphExecDestroy(slot);
        slot = nullptr;
    }
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    const int64_t hs = c->host_started;
    const bool ph = c->pending_host;
    int rc = SK_OK;
    c->capturing = true;
    for (int i = 0; i < iters && rc == SK_OK; ++i) rc = enqueue_iteration(c, nullptr, nullptr);
    c->capturing = false;
    cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    c->host_started = hs;
    c->pending_host = ph;
    if (rc != SK_OK) return rc;
    CK(e);
    e = cudaGraphInstantiate(&slot, g, 0);
    cudaGraphDestroy(g);
    CK(e);
    if (iters != 1) c->graph_iters = iters;
    return SK_OK;
}

// Enqueue `iters` iterations: full graph chunks, then single iterations.
// single1: iterations left over below a chunk go through a cached one-iteration graph (the
// repeated single-step sk_enqueue of a timing loop) instead of direct launches (sk_run, whose
// remainders are rare and should not pay a second capture).
static int enqueue_iters(sk_ctx *c, int64_t iters, int chunk, bool single1 = false) {
    int rc;
    if (c->profiling || c->host_ar) chunk = 1;   // individual launches (events; host collectives)
    if (iters >= chunk && chunk > 1) {
        if ((rc = capture_graph(c, chunk)) != SK_OK) return rc;
    }
    // kernels per iteration (+ the seed kernel with several ranks; + the extra column-block passes)
    const int kpi = (c->world > 1 ? 3 : 2) + (c->kp.csr_nblk >= 2 ? c->kp.csr_nblk - 1 : 0);
    while (iters >= chunk && chunk > 1) {
        CK(cudaGraphLaunch(c->graph, c->stream));
        c->launches += kpi * chunk;
        c->host_started += chunk;
        c->pending_host = true;
        iters -= chunk;
    }
    if (single1 && iters > 0 && !c->profiling && c->world == 1) {   // a one-iteration graph
        if ((rc = capture_graph(c, 1)) != SK_OK) return rc;
        for (; iters > 0; --iters) {
            CK(cudaGraphLaunch(c->graph1, c->stream));
            c->launches += kpi;
            c->host_started += 1;
            c->pending_host = true;
        }
    }
    while (iters-- > 0)
        if ((rc = enqueue_iteration(c, nullptr, nullptr)) != SK_OK) return rc;
    return SK_OK;
}

int sk_run(sk_ctx *c, int64_t max_iters, int32_t poll_every, int32_t *status) {
    if (!c) return fail(SK_ESTATE, "null context");
    if (c->op.kind == SK_OP_RC) return fail(SK_ESTATE, "SK_OP_RC context: use sk_update_rc");
    if (max_iters < 0) return fail(SK_EINVAL, "max_iters < 0");
    CK(cudaSetDevice(c->device));
    if (poll_every <= 0) poll_every = 64;
    const int chunk = poll_every < 16 ? poll_every : 16;
    int rc;
    if ((rc = read_state(c)) != SK_OK) return rc;
    int64_t left = max_iters;
    while (left > 0 && c->st_host->status == SK_ITERATING) {
        const int64_t now = left < poll_every ? left : poll_every;
        if ((rc = enqueue_iters(c, now, chunk)) != SK_OK) return rc;
        left -= now;
        // status visible after the next finish: copy asynchronously (finish pending iteration)
        if ((rc = enqueue_finish(c)) != SK_OK) return rc;
        if ((rc = read_state(c)) != SK_OK) return rc;
    }
    if (status) *status = c->st_host->status;
    return SK_OK;
}

int sk_enqueue(sk_ctx *c, int64_t iters) {
    if (!c) return fail(SK_ESTATE, "null context");
    if (c->op.kind == SK_OP_RC) return fail(SK_ESTATE, "SK_OP_RC context: use sk_update_rc");
    if (iters < 0) return fail(SK_EINVAL, "iters < 0");
    CK(cudaSetDevice(c->device));
    return enqueue_iters(c, iters, 16, /*single1=*/true);
}

int sk_get_residual(sk_ctx *c, double *res) {
    if (!c || !res) return fail(c ? SK_EINVAL : SK_ESTATE, "null argument");
    int rc;
    if ((rc = enqueue_finish(c)) != SK_OK) return rc;
    CK(cudaMemcpyAsync(res, c->kp.res, sizeof(double) * c->nz, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return SK_OK;
}

int sk_get_projection(sk_ctx *c, sk_cplx *y) {
    if (!c || !y) return fail(c ? SK_EINVAL : SK_ESTATE, "null argument");
    int rc;
    if ((rc = enqueue_finish(c)) != SK_OK) return rc;
    CK(cudaMemcpyAsync(y, c->kp.y, sizeof(cplx) * c->nz * c->nl, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return SK_OK;
}

int sk_get_solution(sk_ctx *c, int64_t k, const sk_cplx **x) {
    if (!c || !x) return fail(c ? SK_EINVAL : SK_ESTATE, "null argument");
    if (!c->full) return fail(SK_ESTATE, "context was created without full_x");
    if (k < 0 || k >= c->nz) return fail(SK_EINVAL, "shift index out of range");
    int rc;
    if ((rc = enqueue_finish(c)) != SK_OK) return rc;
    CK(cudaStreamSynchronize(c->stream));
    *x = (const sk_cplx *)(c->kp.x + k * c->M);
    return SK_OK;
}

int sk_copy_solution(sk_ctx *c, int64_t k, sk_cplx *dst, int32_t dst_mem) {
    if (!c || !dst) return fail(c ? SK_EINVAL : SK_ESTATE, "null argument");
    if (!c->full) return fail(SK_ESTATE, "context was created without full_x");
    if (k < 0 || k >= c->nz) return fail(SK_EINVAL, "shift index out of range");
    int rc;
    if ((rc = enqueue_finish(c)) != SK_OK) return rc;
    CK(cudaMemcpyAsync(dst, c->kp.x + k * c->M, sizeof(cplx) * c->M,
                       dst_mem == SK_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return SK_OK;
}

int sk_get_shift_state(sk_ctx *c, sk_cplx *pi, uint8_t *active, int64_t *retired_at) {
    if (!c) return fail(SK_ESTATE, "null context");
    int rc;
    if ((rc = enqueue_finish(c)) != SK_OK) return rc;
    if ((rc = read_state(c)) != SK_OK) return rc;
    const int64_t n = c->st_host->n;
    std::vector<cplx> cur(c->nz), frozen(c->nz);
    std::vector<uint8_t> act(c->nz);
    std::vector<int64_t> ret(c->nz);
    CK(cudaMemcpyAsync(cur.data(), c->kp.pibuf + (size_t)(n % 3) * c->nz, sizeof(cplx) * c->nz,
                       cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(frozen.data(), c->kp.pi_frozen, sizeof(cplx) * c->nz, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(act.data(), c->kp.active, c->nz, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(ret.data(), c->kp.retired_at, sizeof(int64_t) * c->nz, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int k = 0; k < c->nz; ++k) {
        const cplx bs = c->st_host->bscale[n % 3];   // lazy buffer scale (seed switches)
        const cplx v = act[k] ? mk(cur[k].x * bs.x - cur[k].y * bs.y, cur[k].x * bs.y + cur[k].y * bs.x)
                              : frozen[k];   // retired shifts report pi at retirement
        if (pi) pi[k] = {v.x, v.y};
        if (active) active[k] = act[k];
        if (retired_at) retired_at[k] = ret[k];
    }
    return SK_OK;
}

int sk_get_coefficients(sk_ctx *c, sk_coeffs *o) {
    if (!c || !o) return fail(c ? SK_EINVAL : SK_ESTATE, "null argument");
    int rc;
    if ((rc = enqueue_finish(c)) != SK_OK) return rc;
    if ((rc = read_state(c)) != SK_OK) return rc;
    const DevState &h = *c->st_host;
    o->iterations = h.n;
    o->seed_index = h.seed;
    o->switches = h.nswitch;
    o->spmv_count = h.nspmv;
    o->n_active = h.n_active;
    o->status = h.status;
    o->reserved = 0;
    o->z_seed = {h.zs.x, h.zs.y};
    o->alpha = {h.alpha_prev.x, h.alpha_prev.y};
    o->rho = {h.rho_prev.x, h.rho_prev.y};
    o->beta = {h.beta.x, h.beta.y};
    o->seed_residual = h.nu;
    return SK_OK;
}

int sk_profile_enable(sk_ctx *c, int32_t on) {
    if (!c) return fail(SK_ESTATE, "null context");
    c->profiling = on != 0;
    return SK_OK;
}

int sk_get_profile(sk_ctx *c, sk_profile *o, int32_t reset) {
    if (!c || !o) return fail(c ? SK_EINVAL : SK_ESTATE, "null argument");
    CK(cudaSetDevice(c->device));
    CK(cudaStreamSynchronize(c->stream));
    // events come in groups of 3 per iteration: [spmv (+finish, +seed)] [update (+shift step)]
    const size_t groups = c->ev_used / 3;
    for (size_t i = 0; i < groups; ++i) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, c->ev_pool[3 * i], c->ev_pool[3 * i + 1]));
        c->prof_ms[0] += ms;
        CK(cudaEventElapsedTime(&ms, c->ev_pool[3 * i + 1], c->ev_pool[3 * i + 2]));
        c->prof_ms[2] += ms;
    }
    c->prof_iters += (int64_t)groups;
    c->ev_used = 0;
    o->iterations = c->prof_iters;
    o->launches = c->launches;
    o->ms_spmv = c->prof_ms[0];
    o->ms_scalar = c->prof_ms[1];
    o->ms_update = c->prof_ms[2];
    if (reset) {
        c->prof_iters = 0;
        c->prof_ms[0] = c->prof_ms[1] = c->prof_ms[2] = 0;
    }
    return SK_OK;
}

int sk_get_info(sk_ctx *c, sk_info *o) {
    if (!c || !o) return fail(c ? SK_EINVAL : SK_ESTATE, "null argument");
    o->split_ahi = c->kp.split_ahi;
    o->spmv_ctas = c->kp.nblk_spmv;
    o->update_ctas = c->kp.nblk_upd;
    o->shift_agents = c->kp.n_agents;
    o->arena_bytes = (int64_t)c->arena_bytes;
    o->split_fuse = c->kp.split_fuse;
    o->left_real = c->kp.left_real;
    o->csr_col_blocks = c->kp.csr_nblk;
    o->csr_block_shift = c->kp.csr_nblk ? c->kp.csr_bshift : 0;
    return SK_OK;
}

int sk_debug_timestamps(sk_ctx *c, int64_t *out16) {
    if (!c || !out16) return fail(c ? SK_EINVAL : SK_ESTATE, "null argument");
    if (!c->kp.dbg_ts) return fail(SK_ESTATE, "set SHIFTK_DEBUG_TS before sk_init");
    CK(cudaSetDevice(c->device));
    CK(cudaMemcpyAsync(out16, c->kp.dbg_ts, sizeof(int64_t) * 16, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return SK_OK;
}

int sk_finalize(sk_ctx **pc) {
    if (!pc || !*pc) return fail(SK_ESTATE, "sk_finalize on a null / finalized context");
    destroy(*pc);
    *pc = nullptr;
    return SK_OK;
}

int sk_apply_operator(const sk_operator *H, const sk_cplx *r, sk_cplx *q, void *stream) {
    if (!H || !r || !q) return fail(SK_EINVAL, "null argument");
    sk::SpmvArgs a{};
    a.st = nullptr;
    a.r[0] = (const cplx *)r;
    a.q = (cplx *)q;
    a.part_w = nullptr;
    a.bicg = 0;
    cudaStream_t s = (cudaStream_t)stream;
    if (H->kind == SK_OP_HEISENBERG || H->kind == SK_OP_HEISENBERG_SZ) {
        // work queue of the streaming / sector kernels: one zeroed pair per device, rewound by
        // the kernel itself (stand-alone calls on one device must not run concurrently)
        static unsigned long long *work[sk::kMaxWorld] = {};
        int dev = 0;
        CK(cudaGetDevice(&dev));
        if (dev < 0 || dev >= sk::kMaxWorld) return fail(SK_EINVAL, "device ordinal");
        if (!work[dev]) {
            CK(cudaMalloc(&work[dev], 2 * sizeof(unsigned long long)));
            CK(cudaMemset(work[dev], 0, 2 * sizeof(unsigned long long)));
        }
        a.work = work[dev];
    }
    if (H->kind == SK_OP_HEISENBERG) {
        if (H->L < 1 || H->L > 34 || H->M != (int64_t(1) << H->L)) return fail(SK_EINVAL, "L/M");
        a.M = H->M;
        CK(sk::launch_heisenberg(a, KParams{}, H->L, H->J, s));
    } else if (H->kind == SK_OP_HEISENBERG_SZ) {
        if (H->L < 1 || H->L > 34 || H->n_up < 0 || H->n_up > H->L || H->M < 1)
            return fail(SK_EINVAL, "L/n_up/M");
        int64_t dim = 1;   // C(L, n_up): the kernel writes every sector row, so M must be it
        for (int j = 1; j <= H->n_up; ++j) dim = dim * (H->L - H->n_up + j) / j;
        if (H->M != dim) return fail(SK_EINVAL, "Heisenberg sector: need M = C(L, n_up)");
        a.M = H->M;
        CK(sk::launch_heisenberg_sz(a, KParams{}, H->L, H->n_up, H->J, s));
    } else if (H->kind == SK_OP_CSR_REAL || H->kind == SK_OP_CSR_CPLX) {
        const int64_t M = H->M_local > 0 ? H->M_local : H->M;
        if (!H->row_ptr || !H->col || !H->val || M < 1) return fail(SK_EINVAL, "CSR");
        a.M = M;
        CK(sk::launch_csr(a, KParams{}, H->row_ptr, H->col, H->val, H->kind == SK_OP_CSR_CPLX,
                          double(H->nnz) / double(M), s));
    } else {
        return fail(SK_EINVAL, "operator kind");
    }
    return SK_OK;
}

}  // extern "C"
