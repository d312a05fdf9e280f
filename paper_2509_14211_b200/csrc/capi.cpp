// capi.cpp -- the C ABI (include/nbg.h): argument validation and DAG recording.
//
// Nonblocking mode: an operation validates its arguments and records a node; the
// only eager work is folding on operands whose values are already known on the host (iso
// vectors, host scalars, empty vectors) -- a DAG-preserving rewrite that keeps
// iso values "accessed only once".  Blocking mode: the same node is materialised
// and the stream synchronised before the call returns.
#include <cmath>
#include <cstdio>
#include <new>

#include <cstring>
#include <vector>
#include <string>
#include <cctype>
#include <execinfo.h>
#include <signal.h>
#include <unistd.h>

#include "nbg_internal.hpp"

using namespace nbg;

static nbg_status latch(nbg_ctx *ctx, nbg_status st, const std::string &msg) {
    if (ctx) {
        ctx->last_error = msg;
        if (st == NBG_PANIC || st == NBG_OUT_OF_MEMORY) ctx->latched = st;
    }
    return st;
}

#define API_BEGIN try {
#define API_END(ctx)                                                   \
    }                                                                  \
    catch (const nbg::Error &e) { return latch(ctx, e.st, e.msg); }    \
    catch (const std::bad_alloc &) { return latch(ctx, NBG_OUT_OF_MEMORY, "host allocation failed"); } \
    catch (...) { return latch(ctx, NBG_PANIC, "unknown exception"); } \
    return NBG_SUCCESS;

#define CHECK(cond, st, msg) \
    do {                     \
        if (!(cond)) fail(st, msg); \
    } while (0)

static const int64_t MAXDIM = 2147483647ll;

static void check_ctx(nbg_ctx *ctx) {
    if (!ctx) fail(NBG_NULL_POINTER, "ctx is NULL");
}
static void check_vec(nbg_ctx *ctx, nbg_vector v) {
    CHECK(v != nullptr, NBG_NULL_POINTER, "vector handle is NULL");
    CHECK(v->ctx == ctx, NBG_INVALID_OBJECT, "vector belongs to another context");
}
static void check_scal(nbg_ctx *ctx, nbg_scalar s) {
    CHECK(s != nullptr, NBG_NULL_POINTER, "scalar handle is NULL");
    CHECK(s->ctx == ctx, NBG_INVALID_OBJECT, "scalar belongs to another context");
}
static void check_mat(nbg_ctx *ctx, nbg_matrix A) {
    CHECK(A != nullptr, NBG_NULL_POINTER, "matrix handle is NULL");
    CHECK(A->ctx == ctx, NBG_INVALID_OBJECT, "matrix belongs to another context");
}
static void check_type(int t) { CHECK(valid_type(t), NBG_INVALID_VALUE, "invalid nbg_type"); }
static bool is_user(int code) { return code >= NBG_USER_OP_BASE; }
static void check_unop(const nbg_unop &op) {
    if (is_user(op.code)) {
        const UserOp *u = user_op(op.code);
        CHECK(u && u->arity == 1, NBG_INVALID_VALUE, "invalid unop code (not a defined unary operator)");
        return;
    }
    CHECK(op.code >= NBG_IDENTITY && op.code <= NBG_ISZERO, NBG_INVALID_VALUE, "invalid unop code");
}
static void check_binop(const nbg_binop &op) {
    if (is_user(op.code)) {
        const UserOp *u = user_op(op.code);
        CHECK(u && u->arity == 2, NBG_INVALID_VALUE, "invalid binop code (not a defined binary operator)");
        return;
    }
    CHECK(op.code >= NBG_PLUS && op.code <= NBG_MAX_DIVX_C, NBG_INVALID_VALUE, "invalid binop code");
}
static void check_monoid(int m) { CHECK(m == NBG_PLUS || m == NBG_MIN || m == NBG_MAX, NBG_INVALID_VALUE, "invalid monoid"); }

static NodeP mk(Ctx &c, Op op, int type, int64_t n, bool scalar) {
    auto x = std::make_shared<Node>();
    x->op = op;
    x->type = type;
    x->n = scalar ? 0 : n;
    x->scalar = scalar;
    x->uid = c.new_id();
    return x;
}

static NodeP leaf_empty(Ctx &c, int type, int64_t n) {
    NodeP x = mk(c, Op::LEAF, type, n, false);
    x->mat = true;
    x->kind = VKind::EMPTY;
    return x;
}
static NodeP leaf_iso(Ctx &c, int type, int64_t n, double v) {
    NodeP x = mk(c, Op::LEAF, type, n, false);
    x->mat = true;
    x->kind = VKind::ISO;
    x->iso = host_round(type, v);
    return x;
}
static NodeP leaf_host_scalar(Ctx &c, int type, double v) {
    NodeP x = mk(c, Op::LEAF, type, 0, true);
    x->mat = true;
    x->sfmt = SFmt::HOST;
    x->hval = host_round(type, v);
    return x;
}

static bool is_empty(const NodeP &x) { return x->mat && !x->scalar && x->kind == VKind::EMPTY; }
static bool is_iso(const NodeP &x) { return x->mat && !x->scalar && x->kind == VKind::ISO; }
static bool is_host_scalar(const NodeP &x) { return x->mat && x->scalar && x->sfmt == SFmt::HOST; }

static NodeP rec_apply(Ctx &c, int type, const nbg_unop &op, const NodeP &u) {
    if (is_empty(u)) return leaf_empty(c, type, u->n);
    if (is_iso(u) && !is_user(op.code)) return leaf_iso(c, type, u->n, host_unop(op.code, type, u->iso, op.c0, op.c1));
    NodeP x = mk(c, Op::APPLY, type, u->n, false);
    x->code = op.code;
    x->c0 = op.c0;
    x->c1 = op.c1;
    x->a = u;
    return x;
}

static NodeP rec_binary(Ctx &c, Op op, int type, const nbg_binop &bo, const NodeP &u, const NodeP &v) {
    if (op == Op::EMULT) {
        if (is_empty(u) || is_empty(v)) return leaf_empty(c, type, u->n);
    } else if (op == Op::EADD) {
        if (is_empty(u) && is_empty(v)) return leaf_empty(c, type, u->n);
        nbg_unop id{NBG_IDENTITY, 0.0, 0.0};
        if (is_empty(u)) return rec_apply(c, type, id, v);
        if (is_empty(v)) return rec_apply(c, type, id, u);
    }
    if (is_iso(u) && is_iso(v) && !is_user(bo.code)) return leaf_iso(c, type, u->n, host_binop(bo.code, type, u->iso, v->iso, bo.c0));
    NodeP x = mk(c, op, type, u->n, false);
    x->code = bo.code;
    x->c0 = bo.c0;
    x->a = u;
    x->b = v;
    return x;
}

static NodeP rec_bind2nd(Ctx &c, int type, const nbg_binop &bo, const NodeP &u, const NodeP &s) {
    if (is_empty(u)) return leaf_empty(c, type, u->n);
    if (is_iso(u) && is_host_scalar(s) && !is_user(bo.code))
        return leaf_iso(c, type, u->n, host_binop(bo.code, type, u->iso, s->hval, bo.c0));
    NodeP x = mk(c, Op::BIND2ND, type, u->n, false);
    x->code = bo.code;
    x->c0 = bo.c0;
    x->a = u;
    x->b = s;
    return x;
}

double nbg::monoid_identity(int monoid, int type) {
    if (monoid == NBG_PLUS) return 0.0;
    if (is_float(type)) return monoid == NBG_MIN ? INFINITY : -INFINITY;
    if (type == NBG_INT32) return monoid == NBG_MIN ? 2147483647.0 : -2147483648.0;
    if (type == NBG_BOOL) return monoid == NBG_MIN ? 1.0 : 0.0;
    return monoid == NBG_MIN ? 9.2233720368547758e18 : -9.2233720368547758e18;
}

static NodeP rec_mxv(Ctx &c, int type, const nbg_semiring &sr, const MatP &A, const NodeP &u) {
    if (is_empty(u)) return leaf_iso(c, type, A->nrows, monoid_identity(sr.add, type));
    NodeP x = mk(c, Op::MXV, type, A->nrows, false);
    x->add = sr.add;
    x->mul = sr.mul;
    x->c0 = sr.mul_c0;
    x->A = A;
    x->a = u;
    return x;
}

static NodeP rec_reduce(Ctx &c, int type, int monoid, const NodeP &u) {
    if (is_empty(u) || u->n == 0) return leaf_host_scalar(c, type, monoid_identity(monoid, type));
    if (is_iso(u)) {
        double term = host_round(type, u->iso);
        if (monoid != NBG_PLUS) return leaf_host_scalar(c, type, term);
        if (is_float(type)) return leaf_host_scalar(c, type, (double)u->n * term);
        return leaf_host_scalar(c, type, (double)((long long)u->n * (long long)term));
    }
    NodeP x = mk(c, Op::REDUCE, type, 0, true);
    x->code = monoid;
    x->a = u;
    return x;
}

static NodeP rec_sapply(Ctx &c, int type, const nbg_unop &op, const NodeP &s) {
    if (is_host_scalar(s)) return leaf_host_scalar(c, type, host_unop(op.code, type, s->hval, op.c0, op.c1));
    NodeP x = mk(c, Op::SAPPLY, type, 0, true);
    x->code = op.code;
    x->c0 = op.c0;
    x->c1 = op.c1;
    x->a = s;
    return x;
}

// every node a user handle points to is registered (weakly) for nbg_wait_all
static void register_user_node(nbg_ctx *ctx, const NodeP &x) {
    if (x->mat) return;
    auto &v = ctx->user_nodes;
    if (v.size() >= 64 && v.size() >= 2 * ctx->user_nodes_live) {   // drop dead / materialised entries
        size_t k = 0;
        for (auto &w : v) {
            NodeP n = w.lock();
            if (n && !n->mat && n->user_refs > 0) v[k++] = w;
        }
        v.resize(k);
        ctx->user_nodes_live = k;
    }
    v.push_back(x);
    ctx->user_nodes_live++;
}
static nbg_vector new_vhandle(nbg_ctx *ctx, const NodeP &x) {
    auto *h = new nbg_vector_s{ctx, x};
    x->user_refs++;
    register_user_node(ctx, x);
    return h;
}
static nbg_scalar new_shandle(nbg_ctx *ctx, const NodeP &x) {
    auto *h = new nbg_scalar_s{ctx, x};
    x->user_refs++;
    register_user_node(ctx, x);
    return h;
}

// blocking mode: complete the operation before returning
static void blocking_finish(nbg_ctx *ctx, const NodeP &x) {
    if (ctx->mode != NBG_BLOCKING) return;
    if (x->scalar && !x->mat && x->op == Op::SAPPLY) {
        double v = scalar_read(*ctx, x);
        x->mat = true;
        x->sfmt = SFmt::HOST;
        x->hval = v;
        x->a.reset();
        return;
    }
    if (!x->mat) materialize(*ctx, {x});
    NBG_CUDA(cudaStreamSynchronize(ctx->stream));
}

// NBG_SEGV_TRACE=1: print the native stack on SIGSEGV (debug aid for host crashes on GPU boxes
// without a debugger; addresses resolve with addr2line against libnbg.so)
static void segv_trace(int sig) {
    void *fr[64];
    const int k = backtrace(fr, 64);
    const char msg[] = "[nbg] fatal signal, native stack:\n";
    ssize_t w = write(2, msg, sizeof msg - 1);
    (void)w;
    backtrace_symbols_fd(fr, k, 2);
    signal(sig, SIG_DFL);
    raise(sig);
}

extern "C" {

// ---------------------------------------------------------------- context

nbg_status nbg_init(nbg_ctx **out, const nbg_config *cfg) {
    nbg_ctx *ctx = nullptr;
    API_BEGIN
    CHECK(out && cfg, NBG_NULL_POINTER, "nbg_init: NULL argument");
    {
        static bool armed = false;
        const char *e = getenv("NBG_SEGV_TRACE");
        if (!armed && e && e[0] == '1') {
            static char altstack[1 << 16];
            stack_t ss{};
            ss.ss_sp = altstack;
            ss.ss_size = sizeof altstack;
            sigaltstack(&ss, nullptr);
            struct sigaction sa{};
            sa.sa_handler = segv_trace;
            sa.sa_flags = SA_ONSTACK;
            sigaction(SIGSEGV, &sa, nullptr);
            armed = true;
        }
    }
    CHECK(cfg->mode == NBG_BLOCKING || cfg->mode == NBG_NONBLOCKING, NBG_INVALID_VALUE, "nbg_init: bad mode");
    CHECK((cfg->flags & ~NBG_FLAG_DETERMINISTIC) == 0, NBG_INVALID_VALUE, "nbg_init: unknown flag bits");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) fail(NBG_PANIC, "nbg_init: no CUDA device");
    CHECK(cfg->device >= 0 && cfg->device < ndev, NBG_INVALID_VALUE, "nbg_init: bad device");
    NBG_CUDA(cudaSetDevice(cfg->device));
    ctx = new nbg_ctx();
    ctx->mode = cfg->mode;
    ctx->device = cfg->device;
    if (cfg->stream) {
        ctx->stream = (cudaStream_t)cfg->stream;
    } else {
        NBG_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        ctx->own_stream = true;
    }
    NBG_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, cfg->device));
    // side stream of the scalar readbacks (issue_readback), on the context's device
    NBG_CUDA(cudaStreamCreateWithFlags(&ctx->rb_stream, cudaStreamNonBlocking));
    NBG_CUDA(cudaEventCreateWithFlags(&ctx->rb_dep, cudaEventDisableTiming));
    cudaMemPool_t pool;
    NBG_CUDA(cudaDeviceGetDefaultMemPool(&pool, cfg->device));
    uint64_t thr = UINT64_MAX;
    NBG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    *out = ctx;
    ctx = nullptr;
    }
    catch (const nbg::Error &e) { delete ctx; return e.st; }
    catch (...) { delete ctx; return NBG_PANIC; }
    return NBG_SUCCESS;
}

nbg_status nbg_finalize(nbg_ctx *ctx) {
    if (!ctx) return NBG_NULL_POINTER;
    delete ctx;
    return NBG_SUCCESS;
}

nbg_status nbg_last_error(nbg_ctx *ctx, char *buf, size_t len) {
    if (!ctx || !buf) return NBG_NULL_POINTER;
    if (len == 0) return NBG_INVALID_VALUE;
    snprintf(buf, len, "%s", ctx->last_error.c_str());
    return NBG_SUCCESS;
}

nbg_status nbg_guard_selftest(nbg_ctx *ctx) {
    API_BEGIN
    check_ctx(ctx);
    if (!guard_enabled()) return NBG_NOT_IMPLEMENTED;
    BufP b = alloc_buf(*ctx, 1000);
    NBG_CUDA(cudaMemsetAsync((char *)b->d + 1000, 0, 1, ctx->stream));   // one byte past the end
    std::string err;
    try {
        guard_check(*ctx, "nbg_guard_selftest");
    } catch (const Error &e) {
        err = e.msg;
    }
    // repair the zone so the buffer's release does not report it again (the context stays usable)
    NBG_CUDA(cudaMemsetAsync((char *)b->d + 1000, 0xA5, 1, ctx->stream));
    if (err.empty()) return NBG_SUCCESS;   // not detected: the caller's test fails on this status
    ctx->last_error = err;
    return NBG_PANIC;
    API_END(ctx)
}

nbg_status nbg_sync(nbg_ctx *ctx) {
    API_BEGIN
    check_ctx(ctx);
    NBG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->rb_stream) NBG_CUDA(cudaStreamSynchronize(ctx->rb_stream));   // scalar readbacks (side stream)
    guard_check(*ctx, "nbg_sync");
    if (ctx->latched != NBG_SUCCESS) return ctx->latched;
    API_END(ctx)
}

nbg_status nbg_get_stats(nbg_ctx *ctx, nbg_stats *out) {
    if (!ctx || !out) return NBG_NULL_POINTER;
    *out = ctx->stats;
    return NBG_SUCCESS;
}

nbg_status nbg_reset_stats(nbg_ctx *ctx) {
    if (!ctx) return NBG_NULL_POINTER;
    ctx->stats = nbg_stats{};
    return NBG_SUCCESS;
}

nbg_status nbg_set_timing(nbg_ctx *ctx, int enable) {
    API_BEGIN
    check_ctx(ctx);
    timing_collect(*ctx);
    ctx->tclass.clear();
    ctx->timing = enable != 0;
    API_END(ctx)
}

nbg_status nbg_get_timing(nbg_ctx *ctx, const char *cls, double *total_ms, int64_t *launches) {
    API_BEGIN
    check_ctx(ctx);
    CHECK(cls && total_ms && launches, NBG_NULL_POINTER, "nbg_get_timing: NULL argument");
    timing_collect(*ctx);
    auto it = ctx->tclass.find(cls);
    *total_ms = it == ctx->tclass.end() ? 0.0 : it->second.ms;
    *launches = it == ctx->tclass.end() ? 0 : it->second.launches;
    API_END(ctx)
}

// ---------------------------------------------------------------- matrices

// sync = false: the caller synchronises the stream before it returns (several host copies then
// queue back to back instead of one round trip each), and on every error path (HostCopiesDone)
static BufP upload(Ctx &c, const void *p, size_t bytes, int space, int own, bool sync = true) {
    if (bytes == 0) return alloc_buf(c, 0);
    // borrowed device memory is used in place when 16-byte aligned (vector loads); else copied
    if (space == NBG_DEVICE && own == NBG_BORROW && ((uintptr_t)p % 16) == 0) return borrow_buf(c, const_cast<void *>(p), bytes);
    BufP b = alloc_buf(c, bytes);
    NBG_CUDA(cudaMemcpyAsync(b->d, p, bytes, space == NBG_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, c.stream));
    if (space == NBG_HOST && sync) NBG_CUDA(cudaStreamSynchronize(c.stream));   // caller may reuse its buffer
    return b;
}

// the caller's host buffers may be reused once the call returns, error or not (the side stream
// carries the overlapped column-index upload of nbg_matrix_from_csr)
struct HostCopiesDone {
    Ctx &c;
    ~HostCopiesDone() {
        cudaStreamSynchronize(c.stream);
        if (c.rb_stream) cudaStreamSynchronize(c.rb_stream);
    }
};

// Eager ingestion of a large host CSR without values (NBG_EAGER_PLAN=0 turns it off): the SpMV plan's
// structure (row pointers only: groups, skew, tasks, and the row-binned bins / slices / task lists)
// is built while the column indices travel over PCIe on a side stream; the column-dependent fill
// (relabel, padded indices, slice fill) follows the copy.  C4: upload 5.8 ms + plan 3.4 ms at the
// first solve -> ingestion ≈ 7.x ms with the plan done (DESIGN.md §7 "e2e").
static bool eager_plan_wanted(int64_t nrows, int64_t nnz, const void *vals, int space) {
    const char *e = getenv("NBG_EAGER_PLAN");
    if (e && e[0] == '0') return false;
    return space == NBG_HOST && !vals && nrows > 0 && nnz >= (1ll << 19);
}

nbg_status nbg_matrix_from_csr(nbg_ctx *ctx, nbg_matrix *A, int64_t nrows, int64_t ncols, int64_t nnz,
                               const int64_t *rowptr, const int32_t *colidx, const void *vals, int type, double iso,
                               int space, int own) {
    API_BEGIN
    check_ctx(ctx);
    CHECK(A && rowptr && (colidx || nnz == 0), NBG_NULL_POINTER, "nbg_matrix_from_csr: NULL argument");
    CHECK(nrows >= 0 && ncols >= 0 && nrows <= MAXDIM && ncols <= MAXDIM && nnz >= 0, NBG_INVALID_VALUE,
          "nbg_matrix_from_csr: bad dimensions");
    CHECK(space == NBG_HOST || space == NBG_DEVICE, NBG_INVALID_VALUE, "bad space");
    CHECK(own == NBG_COPY || own == NBG_BORROW, NBG_INVALID_VALUE, "bad ownership");
    CHECK(!(space == NBG_HOST && own == NBG_BORROW), NBG_INVALID_VALUE, "host memory cannot be borrowed");
    check_type(type);
    auto M = std::make_shared<Mat>();
    M->ctx = ctx;
    M->id = ctx->new_id();
    M->nrows = nrows;
    M->ncols = ncols;
    M->nnz = nnz;
    M->type = type;
    M->iso = host_round(type, iso);
    HostCopiesDone done_{*ctx};
    if (eager_plan_wanted(nrows, nnz, vals, space)) {
        Ctx &c = *ctx;
        M->rowptr = upload(c, rowptr, (size_t)(nrows + 1) * 8, space, own, false);
        // the structure is built from the row pointers: validate them first
        int bad = gpu_validate_csr(c, nrows, ncols, nnz, (const long long *)M->rowptr->d, nullptr);
        if (bad & 1) fail(NBG_INVALID_VALUE, "rowptr must start at 0, end at nnz and be non-decreasing");
        M->colidx = alloc_buf(c, (size_t)nnz * 4);
        cudaEvent_t ev[2] = {nullptr, nullptr};
        NBG_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
        NBG_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
        struct EvGuard { cudaEvent_t *e; ~EvGuard() { cudaEventDestroy(e[0]); cudaEventDestroy(e[1]); } } evg{ev};
        NBG_CUDA(cudaEventRecord(ev[0], c.stream));            // the buffer's allocation, in stream order
        NBG_CUDA(cudaStreamWaitEvent(c.rb_stream, ev[0], 0));
        NBG_CUDA(cudaMemcpyAsync(M->colidx->d, colidx, (size_t)nnz * 4, cudaMemcpyHostToDevice, c.rb_stream));
        NBG_CUDA(cudaEventRecord(ev[1], c.rb_stream));
        gpu_build_spmv_plan(c, *M, 1);
        if (!M->plan->low_skew) gpu_rb_plan(c, *M, false);
        NBG_CUDA(cudaStreamWaitEvent(c.stream, ev[1], 0));
        bad = gpu_validate_csr(c, nrows, ncols, nnz, nullptr, (const int *)M->colidx->d);
        if (bad & 2) fail(NBG_INDEX_OUT_OF_BOUNDS, "column index out of range");
        gpu_build_spmv_plan(c, *M, 2);
        if (M->plan->rb) gpu_rb_fill(c, *M);
        *A = new nbg_matrix_s{ctx, M};
        return NBG_SUCCESS;
    }
    M->rowptr = upload(*ctx, rowptr, (size_t)(nrows + 1) * 8, space, own, false);
    M->colidx = upload(*ctx, colidx, (size_t)nnz * 4, space, own, false);
    if (vals) M->vals = upload(*ctx, vals, (size_t)nnz * type_size(type), space, own, false);
    // structural validation on the device: row pointers and column range
    int bad = gpu_validate_csr(*ctx, nrows, ncols, nnz, (const long long *)M->rowptr->d, (const int *)M->colidx->d);
    if (bad & 1) fail(NBG_INVALID_VALUE, "rowptr must start at 0, end at nnz and be non-decreasing");
    if (bad & 2) fail(NBG_INDEX_OUT_OF_BOUNDS, "column index out of range");
    *A = new nbg_matrix_s{ctx, M};
    API_END(ctx)
}

static nbg_vector deg_vector(nbg_ctx *ctx, int64_t n, const BufP &deg) {
    NodeP x = mk(*ctx, Op::LEAF, NBG_INT32, n, false);
    x->mat = true;
    x->kind = VKind::FULL;
    x->buf = deg;
    return new_vhandle(ctx, x);
}

nbg_status nbg_matrix_from_edges(nbg_ctx *ctx, nbg_matrix *AT, nbg_vector *deg, int64_t n, int64_t m,
                                 const int32_t *src, const int32_t *dst, int space) {
    API_BEGIN
    check_ctx(ctx);
    CHECK(AT && ((src && dst) || m == 0), NBG_NULL_POINTER, "nbg_matrix_from_edges: NULL argument");
    CHECK(n >= 0 && n <= MAXDIM && m >= 0, NBG_INVALID_VALUE, "nbg_matrix_from_edges: bad sizes");
    CHECK(space == NBG_HOST || space == NBG_DEVICE, NBG_INVALID_VALUE, "bad space");
    BufP ds, dd;
    const int32_t *s = src, *d = dst;
    HostCopiesDone done_{*ctx};
    if (space == NBG_HOST && m > 0) {
        ds = upload(*ctx, src, (size_t)m * 4, NBG_HOST, NBG_COPY, false);
        dd = upload(*ctx, dst, (size_t)m * 4, NBG_HOST, NBG_COPY, false);
        s = (const int32_t *)ds->d;
        d = (const int32_t *)dd->d;
    }
    BufP degb;
    MatP M = gpu_build_csr(*ctx, n, m, s, d, &degb);
    *AT = new nbg_matrix_s{ctx, M};
    if (deg) *deg = deg_vector(ctx, n, degb);
    API_END(ctx)
}

// ---- Matrix Market (coordinate) reader: a buffered hand-rolled parser (fscanf is too slow for
// billion-entry files); produces the edge list for gpu_build_csr
static bool mtx_read(const char *path, int64_t *n_out, std::vector<int32_t> &src, std::vector<int32_t> &dst, std::string &err) {
    FILE *f = fopen(path, "rb");
    if (!f) { err = std::string("cannot open ") + path; return false; }
    std::vector<char> buf(1 << 22);
    size_t len = 0, pos = 0;
    bool eof = false;
    auto fill = [&]() {
        if (pos > 0) { memmove(buf.data(), buf.data() + pos, len - pos); len -= pos; pos = 0; }
        if (!eof) {
            size_t r = fread(buf.data() + len, 1, buf.size() - len, f);
            if (r == 0) eof = true;
            len += r;
        }
    };
    auto getline = [&](std::string &line) -> bool {
        for (;;) {
            for (size_t k = pos; k < len; k++)
                if (buf[k] == '\n') { line.assign(buf.data() + pos, k - pos); pos = k + 1; return true; }
            if (eof) {
                if (pos < len) { line.assign(buf.data() + pos, len - pos); pos = len; return true; }
                return false;
            }
            if (len - pos == buf.size()) buf.resize(buf.size() * 2);
            fill();
        }
    };
    std::string line;
    bool ok = getline(line);
    if (!ok || line.compare(0, 14, "%%MatrixMarket") != 0) { fclose(f); err = "missing %%MatrixMarket header"; return false; }
    std::string lower = line;
    for (char &ch : lower) ch = (char)tolower(ch);
    if (lower.find(" matrix ") == std::string::npos || lower.find("coordinate") == std::string::npos) { fclose(f); err = "only 'matrix coordinate' files are supported"; return false; }
    if (lower.find("complex") != std::string::npos || lower.find("hermitian") != std::string::npos || lower.find("skew") != std::string::npos) {
        fclose(f); err = "complex / hermitian / skew-symmetric files are not supported"; return false;
    }
    const bool pattern = lower.find("pattern") != std::string::npos;
    const bool symmetric = lower.find("symmetric") != std::string::npos;
    long long M = -1, N = -1, NZ = -1;
    while (getline(line)) {
        size_t k = line.find_first_not_of(" \t\r");
        if (k == std::string::npos || line[k] == '%') continue;
        if (sscanf(line.c_str(), "%lld %lld %lld", &M, &N, &NZ) != 3) { fclose(f); err = "malformed size line"; return false; }
        break;
    }
    if (M < 0 || N < 0 || NZ < 0) { fclose(f); err = "missing size line"; return false; }
    const int64_t n = std::max(M, N);
    if (n > MAXDIM) { fclose(f); err = "dimension exceeds int32 indices"; return false; }
    src.reserve((size_t)NZ * (symmetric ? 2 : 1));
    dst.reserve((size_t)NZ * (symmetric ? 2 : 1));
    long long got = 0;
    while (got < NZ && getline(line)) {
        const char *c = line.c_str();
        while (*c == ' ' || *c == '\t') c++;
        if (*c == '\0' || *c == '\r' || *c == '%') continue;
        char *e1 = nullptr, *e2 = nullptr;
        long long i = strtoll(c, &e1, 10);
        long long j = strtoll(e1, &e2, 10);
        if (e1 == c || e2 == e1) { fclose(f); err = "malformed entry line " + std::to_string(got + 1); return false; }
        if (!pattern) {
            char *e3 = nullptr;
            (void)strtod(e2, &e3);
            if (e3 == e2) { fclose(f); err = "missing value on entry line " + std::to_string(got + 1); return false; }
        }
        if (i < 1 || i > M || j < 1 || j > N) { fclose(f); err = "index out of range on entry line " + std::to_string(got + 1); return false; }
        src.push_back((int32_t)(i - 1));
        dst.push_back((int32_t)(j - 1));
        if (symmetric && i != j) { src.push_back((int32_t)(j - 1)); dst.push_back((int32_t)(i - 1)); }
        got++;
    }
    fclose(f);
    if (got != NZ) { err = "file ends after " + std::to_string(got) + " of " + std::to_string(NZ) + " entries"; return false; }
    *n_out = n;
    return true;
}

nbg_status nbg_matrix_from_mtx(nbg_ctx *ctx, nbg_matrix *AT, nbg_vector *deg, const char *path) {
    API_BEGIN
    check_ctx(ctx);
    CHECK(AT && path, NBG_NULL_POINTER, "nbg_matrix_from_mtx: NULL argument");
    std::vector<int32_t> src, dst;
    int64_t n = 0;
    std::string err;
    if (!mtx_read(path, &n, src, dst, err)) {
        const bool oob = err.find("out of range") != std::string::npos;
        fail(oob ? NBG_INDEX_OUT_OF_BOUNDS : NBG_INVALID_VALUE, "nbg_matrix_from_mtx: " + err);
    }
    const int64_t m = (int64_t)src.size();
    BufP ds, dd;
    if (m > 0) {
        ds = upload(*ctx, src.data(), (size_t)m * 4, NBG_HOST, NBG_COPY);
        dd = upload(*ctx, dst.data(), (size_t)m * 4, NBG_HOST, NBG_COPY);
    }
    BufP degb;
    MatP M = gpu_build_csr(*ctx, n, m, m ? (const int32_t *)ds->d : nullptr, m ? (const int32_t *)dd->d : nullptr, &degb);
    NBG_CUDA(cudaStreamSynchronize(ctx->stream));     // the host edge vectors go out of scope
    *AT = new nbg_matrix_s{ctx, M};
    if (deg) *deg = deg_vector(ctx, n, degb);
    API_END(ctx)
}

static void check_gen(const nbg_graphgen *g) {
    CHECK(g != nullptr, NBG_NULL_POINTER, "graphgen is NULL");
    CHECK(g->kind == NBG_GRAPH_RMAT || g->kind == NBG_GRAPH_ER, NBG_INVALID_VALUE, "bad graph kind");
    CHECK(g->scale >= 1 && g->scale <= 30, NBG_INVALID_VALUE, "scale must be in [1, 30]");
    CHECK(g->edge_factor >= 0 && g->edge_factor <= 256, NBG_INVALID_VALUE, "bad edge factor");
}

nbg_status nbg_graph_edges(nbg_ctx *ctx, const nbg_graphgen *g, int32_t *src, int32_t *dst, int space) {
    API_BEGIN
    check_ctx(ctx);
    check_gen(g);
    CHECK(src && dst, NBG_NULL_POINTER, "nbg_graph_edges: NULL output");
    int64_t m = (int64_t)g->edge_factor << g->scale;
    if (space == NBG_DEVICE) {
        gpu_graph_edges(*ctx, *g, src, dst);
        NBG_CUDA(cudaStreamSynchronize(ctx->stream));
    } else {
        BufP s = alloc_buf(*ctx, (size_t)std::max<int64_t>(m, 1) * 4), d = alloc_buf(*ctx, (size_t)std::max<int64_t>(m, 1) * 4);
        gpu_graph_edges(*ctx, *g, (int32_t *)s->d, (int32_t *)d->d);
        NBG_CUDA(cudaMemcpyAsync(src, s->d, (size_t)m * 4, cudaMemcpyDeviceToHost, ctx->stream));
        NBG_CUDA(cudaMemcpyAsync(dst, d->d, (size_t)m * 4, cudaMemcpyDeviceToHost, ctx->stream));
        NBG_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    API_END(ctx)
}

nbg_status nbg_matrix_from_generator(nbg_ctx *ctx, nbg_matrix *AT, nbg_vector *deg, const nbg_graphgen *g) {
    API_BEGIN
    check_ctx(ctx);
    check_gen(g);
    CHECK(AT != nullptr, NBG_NULL_POINTER, "nbg_matrix_from_generator: NULL output");
    int64_t n = 1ll << g->scale;
    int64_t m = (int64_t)g->edge_factor << g->scale;
    MatP M;
    BufP degb;
    {
        BufP s = alloc_buf(*ctx, (size_t)std::max<int64_t>(m, 1) * 4), d = alloc_buf(*ctx, (size_t)std::max<int64_t>(m, 1) * 4);
        gpu_graph_edges(*ctx, *g, (int32_t *)s->d, (int32_t *)d->d);
        M = gpu_build_csr(*ctx, n, m, (const int32_t *)s->d, (const int32_t *)d->d, &degb);
    }
    *AT = new nbg_matrix_s{ctx, M};
    if (deg) *deg = deg_vector(ctx, n, degb);
    API_END(ctx)
}

nbg_status nbg_matrix_nrows(nbg_ctx *ctx, nbg_matrix A, int64_t *out) {
    API_BEGIN check_ctx(ctx); check_mat(ctx, A); CHECK(out, NBG_NULL_POINTER, "NULL out"); *out = A->m->nrows;
    API_END(ctx)
}
nbg_status nbg_matrix_ncols(nbg_ctx *ctx, nbg_matrix A, int64_t *out) {
    API_BEGIN check_ctx(ctx); check_mat(ctx, A); CHECK(out, NBG_NULL_POINTER, "NULL out"); *out = A->m->ncols;
    API_END(ctx)
}
nbg_status nbg_matrix_nnz(nbg_ctx *ctx, nbg_matrix A, int64_t *out) {
    API_BEGIN check_ctx(ctx); check_mat(ctx, A); CHECK(out, NBG_NULL_POINTER, "NULL out"); *out = A->m->nnz;
    API_END(ctx)
}

nbg_status nbg_matrix_export_csr(nbg_ctx *ctx, nbg_matrix A, int64_t *rowptr, int32_t *colidx, int space) {
    API_BEGIN
    check_ctx(ctx);
    check_mat(ctx, A);
    CHECK(rowptr && (colidx || A->m->nnz == 0), NBG_NULL_POINTER, "nbg_matrix_export_csr: NULL output");
    cudaMemcpyKind k = space == NBG_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    NBG_CUDA(cudaMemcpyAsync(rowptr, A->m->rowptr->d, (size_t)(A->m->nrows + 1) * 8, k, ctx->stream));
    if (A->m->nnz) NBG_CUDA(cudaMemcpyAsync(colidx, A->m->colidx->d, (size_t)A->m->nnz * 4, k, ctx->stream));
    NBG_CUDA(cudaStreamSynchronize(ctx->stream));
    API_END(ctx)
}

nbg_status nbg_matrix_free(nbg_ctx *ctx, nbg_matrix A) {
    API_BEGIN
    check_ctx(ctx);
    check_mat(ctx, A);
    delete A;
    API_END(ctx)
}

// ---------------------------------------------------------------- vectors

nbg_status nbg_vector_new(nbg_ctx *ctx, nbg_vector *v, int type, int64_t n) {
    API_BEGIN
    check_ctx(ctx);
    CHECK(v, NBG_NULL_POINTER, "NULL out");
    check_type(type);
    CHECK(n >= 0 && n <= MAXDIM, NBG_INVALID_VALUE, "vector length out of range");
    *v = new_vhandle(ctx, leaf_empty(*ctx, type, n));
    API_END(ctx)
}

nbg_status nbg_vector_new_const(nbg_ctx *ctx, nbg_vector *v, int type, int64_t n, double value) {
    API_BEGIN
    check_ctx(ctx);
    CHECK(v, NBG_NULL_POINTER, "NULL out");
    check_type(type);
    CHECK(n >= 0 && n <= MAXDIM, NBG_INVALID_VALUE, "vector length out of range");
    *v = new_vhandle(ctx, leaf_iso(*ctx, type, n, value));
    API_END(ctx)
}

nbg_status nbg_vector_from_dense(nbg_ctx *ctx, nbg_vector *v, int type, int64_t n, const void *data, int space, int own) {
    API_BEGIN
    check_ctx(ctx);
    CHECK(v && (data || n == 0), NBG_NULL_POINTER, "NULL argument");
    check_type(type);
    CHECK(n >= 0 && n <= MAXDIM, NBG_INVALID_VALUE, "vector length out of range");
    CHECK(space == NBG_HOST || space == NBG_DEVICE, NBG_INVALID_VALUE, "bad space");
    CHECK(own == NBG_COPY || own == NBG_BORROW, NBG_INVALID_VALUE, "bad ownership");
    CHECK(!(space == NBG_HOST && own == NBG_BORROW), NBG_INVALID_VALUE, "host memory cannot be borrowed");
    NodeP x = mk(*ctx, Op::LEAF, type, n, false);
    x->mat = true;
    x->kind = VKind::FULL;
    x->buf = upload(*ctx, data, (size_t)n * type_size(type), space, own);
    *v = new_vhandle(ctx, x);
    API_END(ctx)
}

nbg_status nbg_vector_export_dense(nbg_ctx *ctx, nbg_vector v, void *out, int space) {
    API_BEGIN
    check_ctx(ctx);
    check_vec(ctx, v);
    NodeP x = v->node;
    CHECK(out || x->n == 0, NBG_NULL_POINTER, "NULL out");
    if (!x->mat) materialize(*ctx, {x});
    if (x->kind == VKind::EMPTY) fail(NBG_INVALID_OBJECT, "export of an empty vector");
    if (structured_kind(x->kind)) fail(NBG_INVALID_OBJECT, "vector is not full (sparse / bitset): use nbg_vector_export_sparse");
    size_t bytes = (size_t)x->n * type_size(x->type);
    if (bytes == 0) return NBG_SUCCESS;
    if (x->kind == VKind::ISO) {
        if (space == NBG_HOST) {
            NBG_CUDA(cudaStreamSynchronize(ctx->stream));
            for (int64_t i = 0; i < x->n; i++) {
                switch (x->type) {
                    case NBG_BOOL: ((unsigned char *)out)[i] = x->iso != 0.0; break;
                    case NBG_INT32: ((int32_t *)out)[i] = (int32_t)x->iso; break;
                    case NBG_INT64: ((int64_t *)out)[i] = (int64_t)x->iso; break;
                    case NBG_FP32: ((float *)out)[i] = (float)x->iso; break;
                    case NBG_FP64: ((double *)out)[i] = x->iso; break;
                }
            }
        } else {
            gpu_fill_iso(*ctx, out, x->type, x->n, x->iso);
            NBG_CUDA(cudaStreamSynchronize(ctx->stream));
        }
        return NBG_SUCCESS;
    }
    NBG_CUDA(cudaMemcpyAsync(out, x->buf->d, bytes, space == NBG_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                             ctx->stream));
    NBG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->latched != NBG_SUCCESS) return ctx->latched;
    API_END(ctx)
}

nbg_status nbg_vector_size(nbg_ctx *ctx, nbg_vector v, int64_t *n) {
    API_BEGIN check_ctx(ctx); check_vec(ctx, v); CHECK(n, NBG_NULL_POINTER, "NULL out"); *n = v->node->n;
    API_END(ctx)
}
nbg_status nbg_vector_type(nbg_ctx *ctx, nbg_vector v, int *t) {
    API_BEGIN check_ctx(ctx); check_vec(ctx, v); CHECK(t, NBG_NULL_POINTER, "NULL out"); *t = v->node->type;
    API_END(ctx)
}
nbg_status nbg_vector_nvals(nbg_ctx *ctx, nbg_vector v, int64_t *nv) {
    API_BEGIN
    check_ctx(ctx);
    check_vec(ctx, v);
    CHECK(nv, NBG_NULL_POINTER, "NULL out");
    const NodeP &x = v->node;
    if (!x->mat && needs_structured(x)) materialize(*ctx, {x});
    if (x->mat && x->kind == VKind::EMPTY) *nv = 0;
    else if (x->mat && structured_kind(x->kind)) *nv = x->nvals;
    else *nv = x->n;
    API_END(ctx)
}
nbg_status nbg_vector_is_materialized(nbg_ctx *ctx, nbg_vector v, int *out) {
    API_BEGIN check_ctx(ctx); check_vec(ctx, v); CHECK(out, NBG_NULL_POINTER, "NULL out"); *out = v->node->mat ? 1 : 0;
    API_END(ctx)
}
nbg_status nbg_vector_device_ptr(nbg_ctx *ctx, nbg_vector v, void **ptr) {
    API_BEGIN
    check_ctx(ctx);
    check_vec(ctx, v);
    CHECK(ptr, NBG_NULL_POINTER, "NULL out");
    NodeP x = v->node;
    if (!x->mat) materialize(*ctx, {x});
    if (x->kind == VKind::EMPTY) fail(NBG_INVALID_OBJECT, "empty vector has no values");
    if (structured_kind(x->kind)) fail(NBG_INVALID_OBJECT, "vector is not full (sparse / bitset)");
    if (x->kind == VKind::ISO) {
        ensure_full(*ctx, x);
        *ptr = x->full_cache->d;
    } else {
        *ptr = x->buf->d;
    }
    API_END(ctx)
}

// ---------------------------------------------------------------- sparse / bitset vectors (NEXT-3)

nbg_status nbg_vector_from_sparse(nbg_ctx *ctx, nbg_vector *v, int type, int64_t n, int64_t nvals, const int32_t *indices,
                                  const void *values, int space) {
    API_BEGIN
    check_ctx(ctx);
    CHECK(v && ((indices && values) || nvals == 0), NBG_NULL_POINTER, "nbg_vector_from_sparse: NULL argument");
    CHECK(n >= 0 && n <= MAXDIM && nvals >= 0 && nvals <= n, NBG_INVALID_VALUE, "nbg_vector_from_sparse: bad sizes");
    CHECK(space == NBG_HOST || space == NBG_DEVICE, NBG_INVALID_VALUE, "bad space");
    check_type(type);
    NodeP x = mk(*ctx, Op::LEAF, type, n, false);
    x->mat = true;
    if (nvals == 0) {
        x->kind = VKind::EMPTY;
    } else {
        x->idx = upload(*ctx, indices, (size_t)nvals * 4, space, NBG_COPY);
        x->buf = upload(*ctx, values, (size_t)nvals * type_size(type), space, NBG_COPY);
        const int bad = gpu_check_sparse(*ctx, n, nvals, (const int32_t *)x->idx->d);
        if (bad == 2) fail(NBG_INDEX_OUT_OF_BOUNDS, "nbg_vector_from_sparse: index outside [0, n)");
        if (bad == 1) fail(NBG_INVALID_VALUE, "nbg_vector_from_sparse: indices must be strictly ascending");
        x->nvals = nvals;
        if (nvals == n) {
            x->kind = VKind::FULL;   // every entry present: the dense representation
            x->idx.reset();
        } else {
            x->kind = VKind::SPARSE;
        }
    }
    *v = new_vhandle(ctx, x);
    API_END(ctx)
}

nbg_status nbg_vector_export_sparse(nbg_ctx *ctx, nbg_vector v, int64_t *nvals, int32_t *indices, void *values, int space) {
    API_BEGIN
    check_ctx(ctx);
    check_vec(ctx, v);
    CHECK(nvals, NBG_NULL_POINTER, "NULL nvals");
    CHECK(space == NBG_HOST || space == NBG_DEVICE, NBG_INVALID_VALUE, "bad space");
    NodeP x = v->node;
    if (!x->mat) materialize(*ctx, {x});
    const int64_t nv = x->kind == VKind::EMPTY ? 0 : (structured_kind(x->kind) ? x->nvals : x->n);
    if (!indices && !values) {
        *nvals = nv;
        NBG_CUDA(cudaStreamSynchronize(ctx->stream));
        return ctx->latched;
    }
    CHECK(indices && values, NBG_NULL_POINTER, "nbg_vector_export_sparse: indices and values are both required");
    CHECK(*nvals >= nv, NBG_INVALID_VALUE, "nbg_vector_export_sparse: *nvals smaller than the number of entries");
    *nvals = nv;
    if (nv == 0) return NBG_SUCCESS;
    const cudaMemcpyKind dir = space == NBG_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    const size_t w = type_size(x->type);
    BufP idx = x->idx, vals = x->buf, keep_i, keep_v;
    if (x->kind == VKind::BITSET) {
        gpu_bitset_to_sparse(*ctx, x->n, (const uint32_t *)x->bits->d, x->buf->d, x->type, &keep_i, &keep_v);
        idx = keep_i;
        vals = keep_v;
    } else if (x->kind == VKind::FULL || x->kind == VKind::ISO) {
        BufP bits = alloc_buf(*ctx, (size_t)((x->n + 31) / 32) * 4);
        gpu_bitset_full(*ctx, x->n, (uint32_t *)bits->d);
        const void *dense;
        if (x->kind == VKind::ISO) {
            ensure_full(*ctx, x);
            dense = x->full_cache->d;
        } else {
            dense = x->buf->d;
        }
        gpu_bitset_to_sparse(*ctx, x->n, (const uint32_t *)bits->d, dense, x->type, &keep_i, &keep_v);
        idx = keep_i;
        vals = keep_v;
    }
    NBG_CUDA(cudaMemcpyAsync(indices, idx->d, (size_t)nv * 4, dir, ctx->stream));
    NBG_CUDA(cudaMemcpyAsync(values, vals->d, (size_t)nv * w, dir, ctx->stream));
    NBG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->latched != NBG_SUCCESS) return ctx->latched;
    API_END(ctx)
}

nbg_status nbg_vector_format(nbg_ctx *ctx, nbg_vector v, int *format) {
    API_BEGIN
    check_ctx(ctx);
    check_vec(ctx, v);
    CHECK(format, NBG_NULL_POINTER, "NULL out");
    NodeP x = v->node;
    if (!x->mat) materialize(*ctx, {x});
    switch (x->kind) {
        case VKind::FULL: *format = NBG_FORMAT_FULL; break;
        case VKind::ISO: *format = NBG_FORMAT_ISO; break;
        case VKind::SPARSE: *format = NBG_FORMAT_SPARSE; break;
        case VKind::BITSET: *format = NBG_FORMAT_BITSET; break;
        default: *format = NBG_FORMAT_EMPTY;
    }
    API_END(ctx)
}

nbg_status nbg_vector_estimated_fill(nbg_ctx *ctx, nbg_vector v, double *fill) {
    API_BEGIN
    check_ctx(ctx);
    check_vec(ctx, v);
    CHECK(fill, NBG_NULL_POINTER, "NULL out");
    *fill = estimated_fill(v->node.get());
    API_END(ctx)
}

nbg_status nbg_vector_free(nbg_ctx *ctx, nbg_vector v) {
    API_BEGIN
    check_ctx(ctx);
    check_vec(ctx, v);
    v->node->user_refs--;
    delete v;
    API_END(ctx)
}

// ---------------------------------------------------------------- scalars

nbg_status nbg_scalar_new(nbg_ctx *ctx, nbg_scalar *s, int type, double value) {
    API_BEGIN
    check_ctx(ctx);
    CHECK(s, NBG_NULL_POINTER, "NULL out");
    check_type(type);
    *s = new_shandle(ctx, leaf_host_scalar(*ctx, type, value));
    API_END(ctx)
}

nbg_status nbg_scalar_get(nbg_ctx *ctx, nbg_scalar s, double *value) {
    API_BEGIN
    check_ctx(ctx);
    check_scal(ctx, s);
    CHECK(value, NBG_NULL_POINTER, "NULL out");
    *value = scalar_read(*ctx, s->node);
    if (ctx->latched != NBG_SUCCESS) return ctx->latched;
    API_END(ctx)
}

nbg_status nbg_scalar_free(nbg_ctx *ctx, nbg_scalar s) {
    API_BEGIN
    check_ctx(ctx);
    check_scal(ctx, s);
    s->node->user_refs--;
    delete s;
    API_END(ctx)
}

// ---------------------------------------------------------------- operations

nbg_status nbg_apply(nbg_ctx *ctx, nbg_vector *w, int type, nbg_unop op, nbg_vector u) {
    API_BEGIN
    check_ctx(ctx);
    CHECK(w, NBG_NULL_POINTER, "NULL out");
    check_vec(ctx, u);
    check_type(type);
    check_unop(op);
    NodeP x = rec_apply(*ctx, type, op, u->node);
    blocking_finish(ctx, x);
    *w = new_vhandle(ctx, x);
    API_END(ctx)
}

nbg_status nbg_convert(nbg_ctx *ctx, nbg_vector *w, int type, nbg_vector u) {
    return nbg_apply(ctx, w, type, nbg_unop{NBG_IDENTITY, 0.0, 0.0}, u);
}

nbg_status nbg_apply_bind2nd(nbg_ctx *ctx, nbg_vector *w, int type, nbg_binop op, nbg_vector u, nbg_scalar s) {
    API_BEGIN
    check_ctx(ctx);
    CHECK(w, NBG_NULL_POINTER, "NULL out");
    check_vec(ctx, u);
    check_scal(ctx, s);
    check_type(type);
    check_binop(op);
    NodeP x = rec_bind2nd(*ctx, type, op, u->node, s->node);
    blocking_finish(ctx, x);
    *w = new_vhandle(ctx, x);
    API_END(ctx)
}

static nbg_status ewise(nbg_ctx *ctx, nbg_vector *w, int type, nbg_binop op, nbg_vector u, nbg_vector v, Op kind) {
    API_BEGIN
    check_ctx(ctx);
    CHECK(w, NBG_NULL_POINTER, "NULL out");
    check_vec(ctx, u);
    check_vec(ctx, v);
    check_type(type);
    check_binop(op);
    CHECK(u->node->n == v->node->n, NBG_DIMENSION_MISMATCH, "operand lengths differ");
    NodeP x = rec_binary(*ctx, kind, type, op, u->node, v->node);
    blocking_finish(ctx, x);
    *w = new_vhandle(ctx, x);
    API_END(ctx)
}

nbg_status nbg_ewise_mult(nbg_ctx *ctx, nbg_vector *w, int type, nbg_binop op, nbg_vector u, nbg_vector v) {
    return ewise(ctx, w, type, op, u, v, Op::EMULT);
}
nbg_status nbg_ewise_add(nbg_ctx *ctx, nbg_vector *w, int type, nbg_binop op, nbg_vector u, nbg_vector v) {
    return ewise(ctx, w, type, op, u, v, Op::EADD);
}

nbg_status nbg_mxv(nbg_ctx *ctx, nbg_vector *w, int type, nbg_semiring sr, nbg_matrix A, nbg_vector u) {
    API_BEGIN
    check_ctx(ctx);
    CHECK(w, NBG_NULL_POINTER, "NULL out");
    check_mat(ctx, A);
    check_vec(ctx, u);
    check_type(type);
    check_monoid(sr.add);
    check_binop(nbg_binop{sr.mul, sr.mul_c0});
    CHECK(A->m->ncols == u->node->n, NBG_DIMENSION_MISMATCH, "mxv: A.ncols != len(u)");
    NodeP x = rec_mxv(*ctx, type, sr, A->m, u->node);
    blocking_finish(ctx, x);
    *w = new_vhandle(ctx, x);
    API_END(ctx)
}

nbg_status nbg_reduce(nbg_ctx *ctx, nbg_scalar *s, int type, int monoid, nbg_vector u) {
    API_BEGIN
    check_ctx(ctx);
    CHECK(s, NBG_NULL_POINTER, "NULL out");
    check_vec(ctx, u);
    check_type(type);
    check_monoid(monoid);
    NodeP x = rec_reduce(*ctx, type, monoid, u->node);
    blocking_finish(ctx, x);
    *s = new_shandle(ctx, x);
    API_END(ctx)
}

nbg_status nbg_scalar_apply(nbg_ctx *ctx, nbg_scalar *out, int type, nbg_unop op, nbg_scalar s) {
    API_BEGIN
    check_ctx(ctx);
    CHECK(out, NBG_NULL_POINTER, "NULL out");
    check_scal(ctx, s);
    check_type(type);
    check_unop(op);
    // scalar ops are evaluated on the host where they are read: a user operator (device source) is
    // only usable on vectors and in semirings
    CHECK(!is_user(op.code), NBG_NOT_IMPLEMENTED, "user-defined operators apply to vectors, not host-evaluated scalars");
    NodeP x = rec_sapply(*ctx, type, op, s->node);
    blocking_finish(ctx, x);
    *out = new_shandle(ctx, x);
    API_END(ctx)
}

nbg_status nbg_vector_wait(nbg_ctx *ctx, nbg_vector v) {
    API_BEGIN
    check_ctx(ctx);
    check_vec(ctx, v);
    if (!v->node->mat) materialize(*ctx, {v->node});
    if (ctx->latched != NBG_SUCCESS) return ctx->latched;
    API_END(ctx)
}

nbg_status nbg_wait_all(nbg_ctx *ctx) {
    API_BEGIN
    check_ctx(ctx);
    std::vector<NodeP> roots;
    size_t k = 0;
    for (auto &w : ctx->user_nodes) {
        NodeP n = w.lock();
        if (!n || n->mat || n->user_refs <= 0) continue;
        ctx->user_nodes[k++] = w;
        roots.push_back(n);
    }
    ctx->user_nodes.resize(k);
    ctx->user_nodes_live = k;
    if (!roots.empty()) materialize(*ctx, roots);
    if (ctx->latched != NBG_SUCCESS) return ctx->latched;
    API_END(ctx)
}

nbg_status nbg_scalar_wait(nbg_ctx *ctx, nbg_scalar s) {
    API_BEGIN
    check_ctx(ctx);
    check_scal(ctx, s);
    if (!s->node->mat) materialize(*ctx, {s->node});
    if (ctx->latched != NBG_SUCCESS) return ctx->latched;
    API_END(ctx)
}

}  // extern "C"
