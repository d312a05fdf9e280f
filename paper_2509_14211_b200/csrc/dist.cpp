// dist.cpp -- 1-D row partition across GPUs: one process per GPU, NCCL over
// NVLink/NVSwitch for the exchange.  torch.distributed only broadcasts the 128-byte unique id.
//
// Per sweep every rank runs the fused kernel on its contiguous block of AT's rows, then
//   * allgather-v of the scaled ranks y (grouped ncclBroadcast, one root per block: blocks are
//     unequal because the cut balances BYTES, not rows), and
//   * exact allreduce of the delta / dangling mass: the fixed-point limbs of each rank's
//     reduction slot are summed as int64 (ncclSum), so the global scalar does not depend on the
//     order in which NCCL combines ranks (deterministic across P).
// NCCL is dlopen'ed on first use ("libnccl.so.2": the copy torch already loaded, else the
// system one) so the library loads on hosts without NCCL.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "nbg_internal.hpp"

namespace nbg {

struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi &nccl() {
    static NcclApi api;
    if (api.h) return api;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) fail(NBG_PANIC, "NCCL not found (libnccl.so.2)");
#define NBG_SYM(name)                                                     \
    api.name = (decltype(api.name))dlsym(h, "nccl" #name);                \
    if (!api.name) fail(NBG_PANIC, "NCCL symbol missing: nccl" #name);
    NBG_SYM(GetUniqueId)
    NBG_SYM(CommInitRank)
    NBG_SYM(CommDestroy)
    NBG_SYM(Broadcast)
    NBG_SYM(AllReduce)
    NBG_SYM(AllGather)
    NBG_SYM(GroupStart)
    NBG_SYM(GroupEnd)
    NBG_SYM(GetErrorString)
#undef NBG_SYM
    api.h = h;
    return api;
}

#define NBG_NCCL(x)                                                                            \
    do {                                                                                       \
        ncclResult_t r_ = (x);                                                                 \
        if (r_ != ncclSuccess) fail(NBG_PANIC, std::string("NCCL: ") + nccl().GetErrorString(r_) + " in " #x); \
    } while (0)

Dist::~Dist() {
    if (!peersets.empty()) cudaDeviceSynchronize();   // no kernel may still store into the buffers
    for (auto &kv : peersets) {
        for (void *p : kv.second.opened) cudaIpcCloseMemHandle(p);
        for (void *p : kv.second.own)
            if (p) cudaFree(p);
    }
    if (comm) nccl().CommDestroy((ncclComm_t)comm);
}

// In-process transport for tests (nbg_dist_init_loopback): P contexts driven by P host threads on
// one GPU.  A collective = sync own stream, host barrier, each rank READS the other ranks' buffers
// with its own copies / sum kernels (same process, same device), sync, barrier.  No kernel ever
// waits on another rank's kernel (the synchronisation is on the host).
struct LoopGroup {
    int P = 1;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long long gen = 0;
    std::vector<const void *> ptr;
    std::vector<std::vector<const unsigned long long *>> slots;
    std::vector<void *> pw;   // peer mode setup: each rank's two exchange buffers
    explicit LoopGroup(int p) : P(p), ptr(p, nullptr), slots(p), pw(2 * p, nullptr) {}
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const long long g = gen;
        if (++arrived == P) {
            arrived = 0;
            gen++;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

static void loop_allreduce_i32(Ctx &c, Dist &D, int *d, long long n) {
    LoopGroup &G = *D.loop;
    NBG_CUDA(cudaStreamSynchronize(c.stream));
    G.ptr[D.rank] = d;
    G.barrier();
    BufP tmp = alloc_buf(c, (size_t)std::max(n, 1ll) * 4);
    std::vector<const int *> src(G.P);
    for (int q = 0; q < G.P; q++) src[q] = (const int *)G.ptr[q];
    gpu_sum_i32(c, n, G.P, src.data(), (int *)tmp->d);
    NBG_CUDA(cudaStreamSynchronize(c.stream));
    G.barrier();
    if (n > 0) NBG_CUDA(cudaMemcpyAsync(d, tmp->d, (size_t)n * 4, cudaMemcpyDeviceToDevice, c.stream));
    NBG_CUDA(cudaStreamSynchronize(c.stream));
}

static void loop_exchange(Ctx &c, Dist &D, char *W, size_t ws, const std::vector<int64_t> &off, const std::vector<int64_t> &cnt,
                          const std::vector<const unsigned long long *> &sin, const std::vector<unsigned long long *> &sout) {
    LoopGroup &G = *D.loop;
    NBG_CUDA(cudaStreamSynchronize(c.stream));
    G.ptr[D.rank] = W;
    G.slots[D.rank] = sin;
    G.barrier();
    for (int q = 0; q < G.P; q++)
        if (q != D.rank && cnt[q] > 0)
            NBG_CUDA(cudaMemcpyAsync(W + off[q] * ws, (const char *)G.ptr[q] + off[q] * ws, (size_t)cnt[q] * ws,
                                     cudaMemcpyDeviceToDevice, c.stream));
    for (size_t i = 0; i < sout.size(); i++) {
        std::vector<const unsigned long long *> src(G.P);
        for (int q = 0; q < G.P; q++) src[q] = G.slots[q][i];
        gpu_sum_slots(c, G.P, src.data(), sout[i]);
    }
    NBG_CUDA(cudaStreamSynchronize(c.stream));
    G.barrier();
}

static ncclComm_t comm_of(Dist &d) { return (ncclComm_t)d.comm; }

// Peer mode (nbg_dist_set_exchange): the ping-pong pair of exchange buffers of (ncols_g, ws) on this
// rank and every peer's, set up collectively on first use.  Buffers come from cudaMalloc (CUDA IPC
// needs them outside the stream-ordered pool).  Under NCCL the IPC handles are all-gathered once and
// opened with lazy peer access (NVLink/NVSwitch P2P); under loopback the ranks share one device and
// exchange plain pointers at a host barrier.
static Dist::PeerSet &peer_set(Ctx &c, Dist &D, int64_t ncols_g, size_t ws) {
    auto key = std::make_pair(ncols_g, ws);
    auto it = D.peersets.find(key);
    if (it != D.peersets.end()) return it->second;
    Dist::PeerSet S;
    S.bytes = (size_t)std::max<int64_t>(ncols_g, 1) * ws + 64;
    for (int b = 0; b < 2; b++) {
        NBG_CUDA(cudaMalloc(&S.own[b], S.bytes));
        S.peer[b].assign(D.nranks, nullptr);
        S.peer[b][D.rank] = S.own[b];
    }
    if (D.nranks > 1 && D.loop) {
        LoopGroup &G = *D.loop;
        G.pw[2 * D.rank] = S.own[0];
        G.pw[2 * D.rank + 1] = S.own[1];
        G.barrier();
        for (int q = 0; q < D.nranks; q++)
            for (int b = 0; b < 2; b++) S.peer[b][q] = G.pw[2 * q + b];
        G.barrier();
    } else if (D.nranks > 1) {
        const size_t hs = sizeof(cudaIpcMemHandle_t);
        std::vector<cudaIpcMemHandle_t> h(2 * (size_t)D.nranks);
        for (int b = 0; b < 2; b++) NBG_CUDA(cudaIpcGetMemHandle(&h[2 * D.rank + b], S.own[b]));
        BufP hb = alloc_buf(c, 2 * hs * D.nranks);
        char *mine = (char *)hb->d + 2 * hs * D.rank;
        NBG_CUDA(cudaMemcpyAsync(mine, &h[2 * D.rank], 2 * hs, cudaMemcpyHostToDevice, c.stream));
        NBG_NCCL(nccl().AllGather(mine, hb->d, 2 * hs, ncclUint8, comm_of(D), c.stream));
        NBG_CUDA(cudaMemcpyAsync(h.data(), hb->d, 2 * hs * D.nranks, cudaMemcpyDeviceToHost, c.stream));
        NBG_CUDA(cudaStreamSynchronize(c.stream));
        for (int q = 0; q < D.nranks; q++)
            for (int b = 0; b < 2; b++) {
                if (q == D.rank) continue;
                void *p = nullptr;
                NBG_CUDA(cudaIpcOpenMemHandle(&p, h[2 * q + b], cudaIpcMemLazyEnablePeerAccess));
                S.opened.push_back(p);
                S.peer[b][q] = p;
            }
    }
    return D.peersets.emplace(key, std::move(S)).first->second;
}

}  // namespace nbg

using namespace nbg;

static nbg_status to_status(nbg_ctx *ctx, const Error &e) {
    if (ctx) ctx->last_error = e.msg;
    return e.st;
}

// exact allreduce of an exact-accumulator slot: words 0-9 (limbs) and 10 (non-finite counts) are
// integers (one int64 sum, rank-order independent); word 12 (fp64 sum of out-of-window terms) is
// summed in fp64.  Callers may wrap several of these in one NCCL group.
static void xacc_allreduce(nbg_ctx *ctx, Dist &D, const unsigned long long *src, unsigned long long *dst) {
    NBG_NCCL(nccl().AllReduce(src, dst, 11, ncclInt64, ncclSum, comm_of(D), ctx->stream));
    NBG_NCCL(nccl().AllReduce(src + 12, dst + 12, 1, ncclFloat64, ncclSum, comm_of(D), ctx->stream));
}

static NodeP new_full_leaf(nbg_ctx *ctx, int type, int64_t n, BufP buf) {
    auto y = std::make_shared<Node>();
    y->op = Op::LEAF;
    y->type = type;
    y->n = n;
    y->uid = ctx->new_id();
    y->mat = true;
    y->kind = VKind::FULL;
    y->buf = std::move(buf);
    return y;
}

extern "C" {

nbg_status nbg_partition_rows(const int64_t *rowptr, int64_t n, int nparts, int64_t bytes_per_row, int64_t *cuts) {
    if (!rowptr || !cuts) return NBG_NULL_POINTER;
    if (n < 0 || nparts < 1 || bytes_per_row < 0) return NBG_INVALID_VALUE;
    // cost(i) = 4*len(i) + 8 + bytes_per_row  (colidx + rowptr + the per-row vector traffic)
    const __int128 total = (__int128)4 * (rowptr[n] - rowptr[0]) + (__int128)(8 + bytes_per_row) * n;
    // cut k goes to the row boundary nearest to k/nparts of the total cost
    cuts[0] = 0;
    int k = 1;
    __int128 prefix = 0;
    for (int64_t i = 0; i < n && k < nparts; i++) {
        const __int128 nxt = prefix + (__int128)4 * (rowptr[i + 1] - rowptr[i]) + 8 + bytes_per_row;
        while (k < nparts && nxt * nparts >= total * k) {
            const __int128 t = total * k;
            cuts[k++] = (t - prefix * nparts <= nxt * nparts - t) ? i : i + 1;
        }
        prefix = nxt;
    }
    while (k < nparts) cuts[k++] = n;
    cuts[nparts] = n;
    return NBG_SUCCESS;
}

nbg_status nbg_dist_unique_id(void *id128) {
    if (!id128) return NBG_NULL_POINTER;
    try {
        ncclUniqueId id;
        NBG_NCCL(nccl().GetUniqueId(&id));
        memcpy(id128, &id, sizeof id);
    } catch (const Error &e) {
        return e.st;
    }
    return NBG_SUCCESS;
}

nbg_status nbg_dist_init(nbg_ctx *ctx, int rank, int nranks, const void *id128) {
    if (!ctx || !id128) return NBG_NULL_POINTER;
    if (nranks < 1 || rank < 0 || rank >= nranks) return NBG_INVALID_VALUE;
    try {
        auto d = std::make_unique<Dist>();
        d->rank = rank;
        d->nranks = nranks;
        ncclUniqueId id;
        memcpy(&id, id128, sizeof id);
        NBG_CUDA(cudaSetDevice(ctx->device));
        ncclComm_t cm = nullptr;
        NBG_NCCL(nccl().CommInitRank(&cm, nranks, id, rank));
        d->comm = cm;
        ctx->dist = std::move(d);
    } catch (const Error &e) {
        return to_status(ctx, e);
    }
    return NBG_SUCCESS;
}

nbg_status nbg_dist_init_loopback(nbg_ctx **ctxs, int nranks) {
    if (!ctxs) return NBG_NULL_POINTER;
    if (nranks < 1 || nranks > 64) return NBG_INVALID_VALUE;
    for (int q = 0; q < nranks; q++)
        if (!ctxs[q]) return NBG_NULL_POINTER;
    auto G = std::make_shared<LoopGroup>(nranks);
    for (int q = 0; q < nranks; q++) {
        auto d = std::make_unique<Dist>();
        d->rank = q;
        d->nranks = nranks;
        d->loop = G;
        ctxs[q]->dist = std::move(d);
    }
    return NBG_SUCCESS;
}

nbg_status nbg_dist_set_exchange(nbg_ctx *ctx, int mode) {
    if (!ctx) return NBG_NULL_POINTER;
    if (!ctx->dist || (mode != NBG_DIST_EXCHANGE_COLLECTIVE && mode != NBG_DIST_EXCHANGE_PEER)) return NBG_INVALID_VALUE;
    if (mode == NBG_DIST_EXCHANGE_PEER && ctx->dist->nranks > MAX_PEER) return NBG_INVALID_VALUE;
    ctx->dist->xmode = mode;
    return NBG_SUCCESS;
}

nbg_status nbg_matrix_row_block(nbg_ctx *ctx, nbg_matrix *B, nbg_matrix A, int64_t lo, int64_t hi) {
    if (!ctx || !B || !A) return NBG_NULL_POINTER;
    if (A->ctx != ctx) return NBG_INVALID_OBJECT;
    const Mat &M = *A->m;
    if (lo < 0 || hi < lo || hi > M.nrows) return NBG_INVALID_VALUE;
    try {
        int64_t p0 = 0, p1 = 0;
        NBG_CUDA(cudaMemcpyAsync(&p0, (const long long *)M.rowptr->d + lo, 8, cudaMemcpyDeviceToHost, ctx->stream));
        NBG_CUDA(cudaMemcpyAsync(&p1, (const long long *)M.rowptr->d + hi, 8, cudaMemcpyDeviceToHost, ctx->stream));
        NBG_CUDA(cudaStreamSynchronize(ctx->stream));
        auto S = std::make_shared<Mat>();
        S->ctx = ctx;
        S->id = ctx->new_id();
        S->nrows = hi - lo;
        S->ncols = M.ncols;
        S->nnz = p1 - p0;
        S->type = M.type;
        S->iso = M.iso;
        S->rowptr = alloc_buf(*ctx, (size_t)(hi - lo + 1) * 8);
        gpu_rebase_rowptr(*ctx, hi - lo + 1, (const long long *)M.rowptr->d + lo, p0, (long long *)S->rowptr->d);
        S->colidx = alloc_buf(*ctx, (size_t)std::max<int64_t>(S->nnz, 1) * 4);
        if (S->nnz)
            NBG_CUDA(cudaMemcpyAsync(S->colidx->d, (const int *)M.colidx->d + p0, (size_t)S->nnz * 4, cudaMemcpyDeviceToDevice,
                                     ctx->stream));
        if (M.vals) {
            size_t w = type_size(M.type);
            S->vals = alloc_buf(*ctx, (size_t)std::max<int64_t>(S->nnz, 1) * w);
            if (S->nnz)
                NBG_CUDA(cudaMemcpyAsync(S->vals->d, (const char *)M.vals->d + p0 * w, (size_t)S->nnz * w, cudaMemcpyDeviceToDevice,
                                         ctx->stream));
        }
        NBG_CUDA(cudaStreamSynchronize(ctx->stream));
        *B = new nbg_matrix_s{ctx, S};
    } catch (const Error &e) {
        return to_status(ctx, e);
    }
    return NBG_SUCCESS;
}

nbg_status nbg_vector_allgather(nbg_ctx *ctx, nbg_vector *w, nbg_vector u, const int64_t *cuts) {
    if (!ctx || !w || !u || !cuts) return NBG_NULL_POINTER;
    if (u->ctx != ctx) return NBG_INVALID_OBJECT;
    if (!ctx->dist) return NBG_INVALID_VALUE;
    if (ctx->dist->loop) return NBG_NOT_IMPLEMENTED;   // NCCL groups only (see nbg_vector_allgather_reduce)
    try {
        Dist &D = *ctx->dist;
        NodeP x = u->node;
        if (x->n != cuts[D.rank + 1] - cuts[D.rank]) return NBG_DIMENSION_MISMATCH;
        if (!x->mat) materialize(*ctx, {x});
        if (x->kind == VKind::EMPTY) return NBG_NOT_IMPLEMENTED;
        ensure_full(*ctx, x);
        const int64_t n = cuts[D.nranks];
        const size_t ws = type_size(x->type);
        auto y = std::make_shared<Node>();
        y->op = Op::LEAF;
        y->type = x->type;
        y->n = n;
        y->uid = ctx->new_id();
        y->mat = true;
        y->kind = VKind::FULL;
        y->buf = alloc_buf(*ctx, (size_t)n * ws);
        const void *src = x->kind == VKind::ISO ? x->full_cache->d : x->buf->d;
        char *dst = (char *)y->buf->d;
        if (x->n) NBG_CUDA(cudaMemcpyAsync(dst + cuts[D.rank] * ws, src, (size_t)x->n * ws, cudaMemcpyDeviceToDevice, ctx->stream));
        ncclDataType_t dt = ws == 8 ? ncclInt64 : (ws == 4 ? ncclInt32 : ncclUint8);
        cudaEvent_t ev0;
        timing_begin(*ctx, "comm", &ev0);
        NBG_NCCL(nccl().GroupStart());
        for (int q = 0; q < D.nranks; q++) {
            size_t cnt = (size_t)(cuts[q + 1] - cuts[q]);
            if (cnt == 0) continue;
            NBG_NCCL(nccl().Broadcast(dst + cuts[q] * ws, dst + cuts[q] * ws, cnt, dt, q, comm_of(D), ctx->stream));
        }
        NBG_NCCL(nccl().GroupEnd());
        timing_end(*ctx, "comm", ev0);
        auto *h = new nbg_vector_s{ctx, y};
        y->user_refs++;
        *w = h;
    } catch (const Error &e) {
        return to_status(ctx, e);
    }
    return NBG_SUCCESS;
}

nbg_status nbg_scalar_allreduce(nbg_ctx *ctx, nbg_scalar *out, nbg_scalar s) {
    if (!ctx || !out || !s) return NBG_NULL_POINTER;
    if (s->ctx != ctx) return NBG_INVALID_OBJECT;
    if (!ctx->dist) return NBG_INVALID_VALUE;
    if (ctx->dist->loop) return NBG_NOT_IMPLEMENTED;
    try {
        Dist &D = *ctx->dist;
        NodeP x = s->node;
        if (!x->mat) materialize(*ctx, {x});
        if (!x->mat) {   // a pending scalar op: evaluate on the host (needs its operand)
            double v = scalar_read(*ctx, x);
            x->mat = true;
            x->sfmt = SFmt::HOST;
            x->hval = v;
            x->a.reset();
        }
        auto y = std::make_shared<Node>();
        y->op = Op::LEAF;
        y->scalar = true;
        y->type = x->type;
        y->uid = ctx->new_id();
        y->mat = true;
        y->slot = alloc_slot(*ctx);
        if (x->sfmt == SFmt::HOST) {
            // a host value: contribute it as exact limbs via a tiny upload, then sum
            // (rank-order independent like every other PLUS combine)
            if (!is_float(x->type)) fail(NBG_NOT_IMPLEMENTED, "allreduce of a host integer scalar");
            unsigned long long limbs[SLOT_U64] = {0};
            host_xacc_add(limbs, x->hval);
            SlotP tmp = alloc_slot(*ctx);
            NBG_CUDA(cudaMemcpyAsync(tmp->dptr(), limbs, sizeof limbs, cudaMemcpyHostToDevice, ctx->stream));
            NBG_CUDA(cudaStreamSynchronize(ctx->stream));
            xacc_allreduce(ctx, D, tmp->dptr(), y->slot->dptr());
            y->sfmt = SFmt::XACC;
        } else if (x->sfmt == SFmt::XACC) {
            xacc_allreduce(ctx, D, x->slot->dptr(), y->slot->dptr());
            y->sfmt = SFmt::XACC;
        } else if (x->sfmt == SFmt::I64) {
            NBG_NCCL(nccl().AllReduce(x->slot->dptr() + 11, y->slot->dptr() + 11, 1, ncclInt64, ncclSum, comm_of(D), ctx->stream));
            y->sfmt = SFmt::I64;
        } else {
            NBG_NCCL(nccl().AllReduce(x->slot->dptr() + 11, y->slot->dptr() + 11, 1, ncclUint64, ncclMax, comm_of(D), ctx->stream));
            y->sfmt = x->sfmt;
        }
        mark_readable(*ctx, y->slot, record_prod_event(*ctx));   // a later get() waits only on this collective
        auto *h = new nbg_scalar_s{ctx, y};
        y->user_refs++;
        *out = h;
    } catch (const Error &e) {
        return to_status(ctx, e);
    }
    return NBG_SUCCESS;
}


// ---------------------------------------------------------------- round-2 data plane

nbg_status nbg_dist_exchange_plan(const int64_t *cuts, int nranks, int64_t ncols_g, int64_t *offsets, int64_t *counts) {
    if (!cuts || !offsets || !counts) return NBG_NULL_POINTER;
    if (nranks < 1 || ncols_g < 0) return NBG_INVALID_VALUE;
    for (int q = 0; q < nranks; q++) {
        if (cuts[q + 1] < cuts[q] || cuts[q] < 0) return NBG_INVALID_VALUE;
        const int64_t a = std::min(cuts[q], ncols_g), b = std::min(cuts[q + 1], ncols_g);
        offsets[q] = a;
        counts[q] = b - a;
    }
    return NBG_SUCCESS;
}

nbg_status nbg_xacc_encode(const double *terms, int64_t n, uint64_t *slot) {
    if ((!terms && n > 0) || !slot) return NBG_NULL_POINTER;
    if (n < 0) return NBG_INVALID_VALUE;
    unsigned long long L[SLOT_U64] = {0};
    for (int64_t i = 0; i < n; i++) host_xacc_add(L, terms[i]);
    memcpy(slot, L, sizeof L);
    return NBG_SUCCESS;
}

nbg_status nbg_xacc_decode(const uint64_t *slot, double *value) {
    if (!slot || !value) return NBG_NULL_POINTER;
    *value = xacc_to_double((const unsigned long long *)slot);
    return NBG_SUCCESS;
}

nbg_status nbg_scalar_export_slot(nbg_ctx *ctx, nbg_scalar s, uint64_t *slot) {
    if (!ctx || !s || !slot) return NBG_NULL_POINTER;
    if (s->ctx != ctx) return NBG_INVALID_OBJECT;
    try {
        NodeP x = s->node;
        if (!x->mat) materialize(*ctx, {x});
        if (!x->mat || x->sfmt != SFmt::XACC || !x->slot) return NBG_INVALID_OBJECT;
        NBG_CUDA(cudaMemcpyAsync(slot, x->slot->dptr(), SLOT_U64 * 8, cudaMemcpyDeviceToHost, ctx->stream));
        NBG_CUDA(cudaStreamSynchronize(ctx->stream));
        if (ctx->latched != NBG_SUCCESS) return ctx->latched;
    } catch (const Error &e) {
        return to_status(ctx, e);
    }
    return NBG_SUCCESS;
}

nbg_status nbg_dist_graph_from_generator(nbg_ctx *ctx, const nbg_graphgen *g, int64_t bytes_per_row, nbg_matrix *AT_blk,
                                         nbg_vector *deg_blk, int64_t *cuts, int64_t *ncols_g) {
    if (!ctx || !g || !AT_blk || !deg_blk || !cuts || !ncols_g) return NBG_NULL_POINTER;
    if (g->kind != NBG_GRAPH_RMAT && g->kind != NBG_GRAPH_ER) return NBG_INVALID_VALUE;
    if (g->scale < 1 || g->scale > 30 || g->edge_factor < 1 || bytes_per_row < 0) return NBG_INVALID_VALUE;
    try {
        const int rank = ctx->dist ? ctx->dist->rank : 0, P = ctx->dist ? ctx->dist->nranks : 1;
        if (P > 64) return NBG_NOT_IMPLEMENTED;
        auto ar = [&](int *d, long long cnt) {
            if (ctx->dist->loop) loop_allreduce_i32(*ctx, *ctx->dist, d, cnt);
            else NBG_NCCL(nccl().AllReduce(d, d, (size_t)cnt, ncclInt32, ncclSum, comm_of(*ctx->dist), ctx->stream));
        };
        DistGraph G = gpu_dist_graph(*ctx, *g, rank, P, (long long)bytes_per_row, ar);
        for (int q = 0; q <= P; q++) cuts[q] = G.cuts[q];
        *ncols_g = G.ncols_g;
        const int64_t nb = G.cuts[rank + 1] - G.cuts[rank];
        *AT_blk = new nbg_matrix_s{ctx, G.blk};
        NodeP d = new_full_leaf(ctx, NBG_INT32, nb, G.deg_blk);
        d->user_refs++;
        *deg_blk = new nbg_vector_s{ctx, d};
        if (!ctx->dist_maps) ctx->dist_maps = std::make_shared<std::map<std::pair<int64_t, int64_t>, BufP>>();
    } catch (const Error &e) {
        return to_status(ctx, e);
    }
    return NBG_SUCCESS;
}

nbg_status nbg_vector_allgather_reduce(nbg_ctx *ctx, nbg_vector *w, nbg_vector u_blk, const int64_t *cuts, int64_t ncols_g,
                                       int nscal, const nbg_scalar *s_in, nbg_scalar *s_out) {
    if (!ctx || !w || !u_blk || !cuts || (nscal > 0 && (!s_in || !s_out))) return NBG_NULL_POINTER;
    if (u_blk->ctx != ctx) return NBG_INVALID_OBJECT;
    if (nscal < 0 || nscal > 8 || ncols_g < 0) return NBG_INVALID_VALUE;
    try {
        const int rank = ctx->dist ? ctx->dist->rank : 0, P = ctx->dist ? ctx->dist->nranks : 1;
        if (ncols_g > cuts[P]) return NBG_INVALID_VALUE;
        NodeP x = u_blk->node;
        const int64_t c0 = cuts[rank], nb = cuts[rank + 1] - cuts[rank];
        if (x->n != nb) return NBG_DIMENSION_MISMATCH;
        if (x->scalar || structured_kind(x->kind)) return NBG_NOT_IMPLEMENTED;
        std::vector<NodeP> sin;
        for (int i = 0; i < nscal; i++) {
            if (!s_in[i] || s_in[i]->ctx != ctx) return NBG_INVALID_OBJECT;
            sin.push_back(s_in[i]->node);
        }
        const size_t ws = type_size(x->type);
        const bool peer = ctx->dist && ctx->dist->xmode == NBG_DIST_EXCHANGE_PEER;
        BufP W;
        std::vector<void *> peers;   // peer mode: every rank's buffer for this exchange (own included)
        if (peer) {
            Dist::PeerSet &S = peer_set(*ctx, *ctx->dist, ncols_g, ws);
            const int b = S.parity;
            S.parity ^= 1;
            W = std::make_shared<Buf>();   // a fresh buffer identity (memo keys) over the recycled memory
            W->ctx = ctx;
            W->id = ctx->new_id();
            W->d = S.own[b];
            W->bytes = S.bytes;
            W->owned = false;
            peers = S.peer[b];
        } else {
            W = alloc_buf(*ctx, (size_t)std::max<int64_t>(ncols_g, 1) * ws + 64);
        }
        // ---- this rank's block, written by the producing kernel straight into W[c0 + i] (i < ncols_g - c0)
        if (!ctx->dist_maps) ctx->dist_maps = std::make_shared<std::map<std::pair<int64_t, int64_t>, BufP>>();
        auto key = std::make_pair(c0, nb);
        BufP &map = (*ctx->dist_maps)[key];
        if (!map) {
            map = alloc_buf(*ctx, (size_t)std::max<int64_t>(nb, 1) * 4);
            gpu_offset_map(*ctx, nb, c0, ncols_g, (int *)map->d);
        }
        std::vector<NodeP> roots;
        if (!x->mat) {
            // the map is affine (gpu_offset_map): the fused kernel stores to W[c0 + i], i < ncols_g - c0
            ctx->out_targets[x.get()] = Ctx::OutTarget{W, (const int *)map->d, peers, c0, std::max<int64_t>(0, std::min(nb, ncols_g - c0))};
            roots.push_back(x);
        }
        for (const NodeP &sn : sin)
            if (!sn->mat) roots.push_back(sn);
        try {
            if (!roots.empty()) materialize(*ctx, roots);
        } catch (...) {
            ctx->out_targets.erase(x.get());
            throw;
        }
        ctx->out_targets.erase(x.get());
        if (x->mat) {   // already materialised (or iso): copy its block into place
            if (x->kind == VKind::EMPTY) return NBG_NOT_IMPLEMENTED;
            ensure_full(*ctx, x);
            const void *src = x->kind == VKind::ISO ? x->full_cache->d : x->buf->d;
            const int64_t cnt = std::max<int64_t>(0, std::min(nb, ncols_g - c0));
            if (cnt > 0) {
                if (!peer) peers.assign(1, W->d);
                for (void *dst : peers)   // peer mode: into every rank's buffer (P2P copies)
                    NBG_CUDA(cudaMemcpyAsync((char *)dst + c0 * ws, src, (size_t)cnt * ws, cudaMemcpyDeviceToDevice, ctx->stream));
            }
        }
        std::vector<NodeP> sout;
        for (const NodeP &sn : sin) {
            if (!sn->mat) {   // a pending scalar op: evaluate on the host
                double v = scalar_read(*ctx, sn);
                sn->mat = true;
                sn->sfmt = SFmt::HOST;
                sn->hval = v;
                sn->a.reset();
            }
            if (sn->sfmt != SFmt::XACC && P > 1) return NBG_NOT_IMPLEMENTED;   // float PLUS reductions only
            auto y = std::make_shared<Node>();
            y->op = Op::LEAF;
            y->scalar = true;
            y->type = sn->type;
            y->uid = ctx->new_id();
            y->mat = true;
            if (P == 1) {
                y->sfmt = sn->sfmt;
                y->slot = sn->slot;
                y->hval = sn->hval;
            } else {
                y->sfmt = SFmt::XACC;
                y->slot = alloc_slot(*ctx);
            }
            sout.push_back(y);
        }
        // ---- one NCCL group: the P blocks broadcast in place + the exact scalar sums
        if (P > 1 && ctx->dist->loop) {
            std::vector<int64_t> off(P), cnt(P);
            nbg_dist_exchange_plan(cuts, P, ncols_g, off.data(), cnt.data());
            if (peer) std::fill(cnt.begin(), cnt.end(), 0);   // data already in place: barrier + sums only
            std::vector<const unsigned long long *> si;
            std::vector<unsigned long long *> so;
            for (size_t i = 0; i < sin.size(); i++) {
                si.push_back(sin[i]->slot->dptr());
                so.push_back(sout[i]->slot->dptr());
            }
            loop_exchange(*ctx, *ctx->dist, (char *)W->d, ws, off, cnt, si, so);
        } else if (P > 1) {
            Dist &D = *ctx->dist;
            std::vector<int64_t> off(P), cnt(P);
            nbg_dist_exchange_plan(cuts, P, ncols_g, off.data(), cnt.data());
            ncclDataType_t dt = ws == 8 ? ncclInt64 : (ws == 4 ? ncclInt32 : ncclUint8);
            char *dst = (char *)W->d;
            cudaEvent_t ev0;
            timing_begin(*ctx, "comm", &ev0);
            SlotP bar;
            NBG_NCCL(nccl().GroupStart());
            for (int q = 0; q < P && !peer; q++)
                if (cnt[q] > 0)
                    NBG_NCCL(nccl().Broadcast(dst + off[q] * ws, dst + off[q] * ws, (size_t)cnt[q], dt, q, comm_of(D), ctx->stream));
            for (size_t i = 0; i < sin.size(); i++) xacc_allreduce(ctx, D, sin[i]->slot->dptr(), sout[i]->slot->dptr());
            if (peer && sin.empty()) {   // the peer stores need a cross-rank barrier: a one-word allreduce
                bar = alloc_slot(*ctx);
                NBG_NCCL(nccl().AllReduce(bar->dptr(), bar->dptr(), 1, ncclInt64, ncclSum, comm_of(D), ctx->stream));
            }
            NBG_NCCL(nccl().GroupEnd());
            timing_end(*ctx, "comm", ev0);
        }
        ProdEvP pe;
        for (size_t i = 0; i < sout.size(); i++) {
            if (sout[i]->slot && P > 1) {
                if (!pe) pe = record_prod_event(*ctx);
                mark_readable(*ctx, sout[i]->slot, pe);
            }
            sout[i]->user_refs++;
            s_out[i] = new nbg_scalar_s{ctx, sout[i]};
        }
        NodeP y = new_full_leaf(ctx, x->type, ncols_g, W);
        y->user_refs++;
        *w = new nbg_vector_s{ctx, y};
    } catch (const Error &e) {
        return to_status(ctx, e);
    }
    return NBG_SUCCESS;
}

}  // extern "C"
