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

#include <cstring>
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
    if (comm) nccl().CommDestroy((ncclComm_t)comm);
}

static ncclComm_t comm_of(Dist &d) { return (ncclComm_t)d.comm; }

}  // namespace nbg

using namespace nbg;

static nbg_status to_status(nbg_ctx *ctx, const Error &e) {
    if (ctx) ctx->last_error = e.msg;
    return e.st;
}

// exact allreduce of an exact-accumulator slot: the limbs are integers (sum, rank-order
// independent), the flag word is OR-ed (split / max / join: NCCL has no bitwise OR), and the fp64
// sum of out-of-window terms is summed in fp64
static void xacc_allreduce(nbg_ctx *ctx, Dist &D, const unsigned long long *src, unsigned long long *dst) {
    NBG_NCCL(nccl().AllReduce(src, dst, 10, ncclInt64, ncclSum, comm_of(D), ctx->stream));
    SlotP f3 = alloc_slot(*ctx), g3 = alloc_slot(*ctx);
    gpu_flags_split(*ctx, src, f3->dptr());
    NBG_NCCL(nccl().AllReduce(f3->dptr(), g3->dptr(), 3, ncclUint64, ncclMax, comm_of(D), ctx->stream));
    gpu_flags_join(*ctx, g3->dptr(), dst);
    NBG_NCCL(nccl().AllReduce(src + 12, dst + 12, 1, ncclFloat64, ncclSum, comm_of(D), ctx->stream));
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
        issue_readback(*ctx, *y->slot);   // a later get() waits only on this collective
        auto *h = new nbg_scalar_s{ctx, y};
        y->user_refs++;
        *out = h;
    } catch (const Error &e) {
        return to_status(ctx, e);
    }
    return NBG_SUCCESS;
}

}  // extern "C"
