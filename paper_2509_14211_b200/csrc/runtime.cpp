// runtime.cpp -- device memory, scalar slots, events, timing, host-side arithmetic helpers.
#include <cmath>
#include <cstdio>
#include <cstring>

#include "nbg_internal.hpp"

namespace nbg {

void fail(nbg_status st, const std::string &msg) { throw Error{st, msg}; }

void cuda_fail(cudaError_t e, const char *what, const char *file, int line) {
    char buf[512];
    snprintf(buf, sizeof buf, "CUDA error %d (%s) in %s at %s:%d", (int)e, cudaGetErrorString(e), what, file, line);
    nbg_status st = (e == cudaErrorMemoryAllocation) ? NBG_OUT_OF_MEMORY : NBG_PANIC;
    throw Error{st, buf};
}

double now_ns() {
    return (double)std::chrono::duration_cast<std::chrono::nanoseconds>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

uint64_t hash_str(const std::string &s) {   // FNV-1a 64
    uint64_t h = 1469598103934665603ull;
    for (unsigned char ch : s) {
        h ^= ch;
        h *= 1099511628211ull;
    }
    return h;
}

// ---------------------------------------------------------------- buffers

static constexpr size_t POOL_MAX_BUF = 64ull << 20, POOL_MAX_TOTAL = 512ull << 20;

static bool pool_enabled() {
    static int v = -1;
    if (v < 0) { const char *e = getenv("NBG_NO_POOL"); v = (e && e[0] == '1') ? 0 : 1; }
    return v == 1;
}

// ---------------------------------------------------------------- guard mode (NBG_GUARD=1)
// compute-sanitizer is closed on the GPU pool, so out-of-bounds WRITES are caught by red zones:
// every pool buffer gets GUARD_BYTES of 0xA5 after its end; after every generated-kernel launch and
// every materialisation the red zones of all live buffers are checked on the device (one kernel),
// and a buffer's zone is checked again when it is freed.  Test-only (synchronises every launch).
static constexpr size_t GUARD_BYTES = 256;
bool guard_enabled() {
    static int v = -1;
    if (v < 0) { const char *e = getenv("NBG_GUARD"); v = (e && e[0] == '1') ? 1 : 0; }
    return v == 1;
}

void guard_check(Ctx &c, const char *where) {
    if (!guard_enabled()) return;
    if (!c.guard_msg.empty()) fail(NBG_PANIC, c.guard_msg);
    if (c.guard_live.empty()) return;
    std::vector<const unsigned char *> zones;
    zones.reserve(c.guard_live.size());
    for (auto &kv : c.guard_live) zones.push_back((const unsigned char *)kv.first + kv.second);
    const int bad = gpu_guard_scan(c, zones.data(), (int)zones.size(), GUARD_BYTES);
    if (bad >= 0) {
        char msg[256];
        auto it = c.guard_live.begin();
        std::advance(it, bad);
        snprintf(msg, sizeof msg, "guard: red zone after a %zu-byte buffer at %p overwritten (detected after %s)", it->second,
                 it->first, where);
        fail(NBG_PANIC, msg);
    }
}

Buf::~Buf() {
    if (!(owned && d && ctx)) return;
    if (guard_enabled() && bytes) {
        if (ctx->guard_live.count(d) && !ctx->closing) {
            const unsigned char *z = (const unsigned char *)d + bytes;
            if (gpu_guard_scan(*ctx, &z, 1, GUARD_BYTES) >= 0) {   // reported by the next guard_check
                char msg[160];
                snprintf(msg, sizeof msg, "guard: red zone after a %zu-byte buffer overwritten (detected at free)", bytes);
                fprintf(stderr, "[nbg] %s\n", msg);
                if (ctx->guard_msg.empty()) ctx->guard_msg = msg;
            }
        }
        ctx->guard_live.erase(d);
    }
    if (pool_enabled() && !ctx->closing && bytes <= POOL_MAX_BUF && ctx->pooled_bytes + bytes <= POOL_MAX_TOTAL) {
        ctx->buf_pool[bytes].push_back(d);
        ctx->pooled_bytes += bytes;
    } else {
        cudaFreeAsync(d, ctx->stream);
    }
}

BufP alloc_buf(Ctx &c, size_t bytes) {
    auto b = std::make_shared<Buf>();
    b->ctx = &c;
    b->id = c.new_id();
    b->bytes = bytes;
    b->owned = true;
    if (bytes) {
        auto it = c.buf_pool.find(bytes);
        if (it != c.buf_pool.end() && !it->second.empty()) {
            b->d = it->second.back();
            it->second.pop_back();
            c.pooled_bytes -= bytes;
        } else {
            NBG_CUDA(cudaMallocAsync(&b->d, bytes + (guard_enabled() ? GUARD_BYTES : 0), c.stream));
        }
        if (guard_enabled()) {
            NBG_CUDA(cudaMemsetAsync((char *)b->d + bytes, 0xA5, GUARD_BYTES, c.stream));
            c.guard_live[b->d] = bytes;
        }
    }
    return b;
}

BufP borrow_buf(Ctx &c, void *d, size_t bytes) {
    auto b = std::make_shared<Buf>();
    b->ctx = &c;
    b->id = c.new_id();
    b->bytes = bytes;
    b->d = d;
    b->owned = false;
    return b;
}

// ---------------------------------------------------------------- scalar slots

Slab::~Slab() {
    if (ctx->rb_stream) cudaStreamSynchronize(ctx->rb_stream);   // readbacks of its slots are done
    if (d) cudaFreeAsync(d, ctx->stream);
    if (h) {
        // the host mirror may still be the target of a queued copy
        cudaStreamSynchronize(ctx->stream);
        cudaFreeHost(h);
    }
}

Slot::~Slot() {
    if (ev && slab) put_event(*slab->ctx, ev);
}

SlotP alloc_slot(Ctx &c) {
    if (!c.cur_slab || c.cur_slab->used >= SLAB_SLOTS) {
        auto s = std::make_shared<Slab>();
        s->ctx = &c;
        size_t bytes = (size_t)SLAB_SLOTS * SLOT_U64 * sizeof(unsigned long long);
        NBG_CUDA(cudaMallocAsync((void **)&s->d, bytes, c.stream));
        NBG_CUDA(cudaMemsetAsync(s->d, 0, bytes, c.stream));
        NBG_CUDA(cudaMallocHost((void **)&s->h, bytes));
        c.cur_slab = s;
    }
    auto sl = std::make_shared<Slot>();
    sl->slab = c.cur_slab;
    sl->idx = c.cur_slab->used++;
    sl->id = c.new_id();
    return sl;
}

cudaEvent_t get_event(Ctx &c) {
    if (!c.event_pool.empty()) {
        cudaEvent_t e = c.event_pool.back();
        c.event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    NBG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return e;
}

void put_event(Ctx &c, cudaEvent_t e) { c.event_pool.push_back(e); }

// The D2H copy of a slot's mirror runs on a side stream ordered after the producing kernel: on the
// context stream the copy sat between consecutive sweep kernels and cost ≈ 13 µs of device time per
// sweep (copy-engine handoff before and after the 2 µs copy).
ProdEv::~ProdEv() {
    if (ctx && e) put_event(*ctx, e);
}

ProdEvP record_prod_event(Ctx &c) {
    auto p = std::make_shared<ProdEv>();
    p->e = get_event(c);
    p->ctx = &c;
    NBG_CUDA(cudaEventRecord(p->e, c.stream));
    return p;
}

void mark_readable(Ctx &c, const SlotP &s, const ProdEvP &pe) {
    if (s->rb_issued) return;
    s->pev = pe;
    c.deferred.push_back(s);
    if (c.deferred.size() > 256) {   // drop the entries of freed or already copied slots
        std::deque<std::weak_ptr<Slot>> keep;
        for (auto &w : c.deferred) {
            auto q = w.lock();
            if (q && !q->rb_issued) keep.push_back(w);
        }
        c.deferred.swap(keep);
    }
}

// The D2H copy of a readable slot is issued when the host first reads it, on the side stream and
// ordered after the slot's producer only (a speculated later launch is not waited for).  It covers,
// in one copy per slab, every pending readable slot produced up to this one -- or all pending ones
// when the newest producer has already finished (the end of a fixed-count loop reads its deltas in
// one copy) -- so a scalar produced each sweep costs one event record at launch and nothing more
// unless it is read.
void issue_readback(Ctx &c, Slot &s) {
    if (s.rb_issued) return;
    if (!s.pev) {
        NBG_CUDA(cudaEventRecord(c.rb_dep, c.stream));
        NBG_CUDA(cudaStreamWaitEvent(c.rb_stream, c.rb_dep, 0));
        NBG_CUDA(cudaMemcpyAsync(s.hptr(), s.dptr(), SLOT_U64 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c.rb_stream));
        if (!s.ev) s.ev = get_event(c);
        NBG_CUDA(cudaEventRecord(s.ev, c.rb_stream));
        s.rb_issued = true;
        return;
    }
    SlotP newest;
    for (auto it = c.deferred.rbegin(); it != c.deferred.rend() && !newest; ++it) {
        auto q = it->lock();
        if (q && !q->rb_issued && q->pev) newest = q;
    }
    const bool all = newest && newest.get() != &s && cudaEventQuery(newest->pev->e) == cudaSuccess;
    std::vector<SlotP> set;
    for (auto &w : c.deferred) {
        auto q = w.lock();
        if (!q || q->rb_issued || !q->pev) continue;
        set.push_back(q);
        if (!all && q.get() == &s) break;
    }
    if (set.empty() || (!all && set.back().get() != &s)) fail(NBG_PANIC, "readback: slot not in the deferred list");
    NBG_CUDA(cudaStreamWaitEvent(c.rb_stream, set.back()->pev->e, 0));
    std::map<Slab *, std::pair<int, int>> rng;   // per slab: lowest and highest slot index
    for (const SlotP &q : set) {
        auto it = rng.find(q->slab.get());
        if (it == rng.end()) rng[q->slab.get()] = {q->idx, q->idx};
        else it->second = {std::min(it->second.first, q->idx), std::max(it->second.second, q->idx)};
    }
    for (auto &kv : rng) {
        const size_t off = (size_t)kv.second.first * SLOT_U64, cnt = (size_t)(kv.second.second - kv.second.first + 1) * SLOT_U64;
        NBG_CUDA(cudaMemcpyAsync(kv.first->h + off, kv.first->d + off, cnt * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                 c.rb_stream));
    }
    auto ce = std::make_shared<ProdEv>();
    ce->ctx = &c;
    ce->e = get_event(c);
    NBG_CUDA(cudaEventRecord(ce->e, c.rb_stream));
    for (const SlotP &q : set) {
        q->cev = ce;
        q->rb_issued = true;
        q->pev.reset();
    }
    while (!c.deferred.empty()) {
        auto f = c.deferred.front().lock();
        if (f && !f->rb_issued) break;
        c.deferred.pop_front();
    }
}

// ---------------------------------------------------------------- exact accumulator decode (host)
// Same arithmetic as nbg_xacc_value in jit/prelude.cuh: carry-normalise the 10 limbs of signed
// 32-bit pieces into an 11-word two's complement integer (LSB 2^-160), then round to nearest even.
static double xacc_window(const unsigned long long *L);

double xacc_to_double(const unsigned long long *L) {
    const unsigned long long flags = L[10];   // counts: NaN bits 0-20, +inf 21-41, -inf 42-62 (prelude.cuh)
    const unsigned long long nan = flags & 0x1FFFFFull, pinf = (flags >> 21) & 0x1FFFFFull, ninf = (flags >> 42) & 0x1FFFFFull;
    if (nan || (pinf && ninf)) return NAN;
    if (pinf) return INFINITY;
    if (ninf) return -INFINITY;
    double extra;                       // fp64 sum of the terms outside the exact window
    memcpy(&extra, &L[12], 8);
    return xacc_window(L) + extra;
}

static double xacc_window(const unsigned long long *L) {
    uint32_t w[11];
    long long carry = 0;
    for (int k = 0; k < 10; k++) {
        long long v = (long long)L[k] + carry;
        w[k] = (uint32_t)(v & 0xffffffffll);
        carry = v >> 32;
    }
    w[10] = (uint32_t)carry;
    bool neg = carry < 0;
    if (neg) {
        uint32_t cr = 1;
        for (int k = 0; k < 11; k++) {
            unsigned long long t = (unsigned long long)(uint32_t)(~w[k]) + cr;
            w[k] = (uint32_t)t;
            cr = (uint32_t)(t >> 32);
        }
    }
    int h = -1;
    for (int k = 10; k >= 0; k--)
        if (w[k]) { h = k; break; }
    if (h < 0) return 0.0;
    // word-level extraction of the top 64 bits (same arithmetic as prelude.cuh)
    const uint32_t wh = w[h], wm = h >= 1 ? w[h - 1] : 0u, wl = h >= 2 ? w[h - 2] : 0u;
    bool sticky = false;
    for (int k = 0; k < h - 2; k++)
        if (w[k]) sticky = true;
    const int tb = 31 - __builtin_clz(wh);
    const int sh = 31 - tb;
    const unsigned long long hi64 = ((unsigned long long)wh << 32) | (unsigned long long)wm;
    unsigned long long top = sh ? ((hi64 << sh) | ((unsigned long long)wl >> (32 - sh))) : hi64;
    const unsigned long long lowmask = sh ? ((1ull << (32 - sh)) - 1ull) : 0xffffffffull;
    if ((unsigned long long)wl & lowmask) sticky = true;
    const int g = h * 32 + tb;
    unsigned long long mant = top >> 11;
    unsigned long long rb = top & 0x7ffull;
    if (rb & 0x3ffull) sticky = true;
    int lsb = g - 52;
    if ((rb & 0x400ull) && (sticky || (mant & 1ull))) {
        mant += 1;
        if (mant == (1ull << 53)) { mant >>= 1; lsb += 1; }
    }
    double v = std::ldexp((double)mant, lsb - 160);
    return neg ? -v : v;
}

// host twin of nbg_xacc_add (prelude.cuh): add one double into the limbs
void host_xacc_add(unsigned long long *acc, double d) {
    if (d == 0.0) return;
    long long bits;
    memcpy(&bits, &d, 8);
    int e = (int)((bits >> 52) & 0x7ff);
    if (e == 0x7ff) {   // counted like the device's nbg_xacc_add (one per term)
        acc[10] += ((bits & 0xFFFFFFFFFFFFFll) != 0) ? 1ull : (bits < 0 ? (1ull << 42) : (1ull << 21));
        return;
    }
    unsigned long long m = (unsigned long long)bits & 0xFFFFFFFFFFFFFull;
    int ex;
    if (e == 0) ex = -1074; else { m |= (1ull << 52); ex = e - 1075; }
    int pos = ex + 160;
    if (pos > 235 || pos + 52 < 0) {     // outside the window [2^-160, 2^128): fp64 in acc[12]
        double e12;
        memcpy(&e12, &acc[12], 8);
        e12 += d;
        memcpy(&acc[12], &e12, 8);
        return;
    }
    if (pos < 0) {                       // straddles the low edge: keep the bits >= 2^-160
        m >>= -pos;
        pos = 0;
        if (m == 0) return;
    }
    int k = pos >> 5, sh = pos & 31;
    unsigned long long lo = m << sh;
    unsigned long long hi = sh ? (m >> (64 - sh)) : 0ull;
    unsigned long long p0 = lo & 0xffffffffull, p1 = lo >> 32, p2 = hi;
    if (bits < 0) { p0 = (unsigned long long)(-(long long)p0); p1 = (unsigned long long)(-(long long)p1); p2 = (unsigned long long)(-(long long)p2); }
    acc[k] += p0;
    acc[k + 1] += p1;
    acc[k + 2] += p2;
}

static double fkey_dec(unsigned long long k) {
    long long b = (k & 0x8000000000000000ull) ? (long long)(k & 0x7fffffffffffffffull) : (long long)(~k);
    double d;
    memcpy(&d, &b, 8);
    return d;
}

double slot_value(const unsigned long long *s, SFmt fmt) {
    switch (fmt) {
        case SFmt::XACC: return xacc_to_double(s);
        case SFmt::I64: return (double)(long long)s[11];
        case SFmt::FMAX: return s[11] ? fkey_dec(s[11]) : -INFINITY;
        case SFmt::FMIN: return s[11] ? fkey_dec(~s[11]) : INFINITY;
        case SFmt::IMAX: return s[11] ? (double)(long long)(s[11] ^ 0x8000000000000000ull) : -9.2233720368547758e18;
        case SFmt::IMIN: return s[11] ? (double)(long long)(~s[11] ^ 0x8000000000000000ull) : 9.2233720368547758e18;
        default: return 0.0;
    }
}

// ---------------------------------------------------------------- timing

// timing events are recycled (creating two events per launch cost ≈ 2 µs of host time per wait)
static cudaEvent_t get_timing_event(Ctx &c) {
    if (!c.timing_pool.empty()) {
        cudaEvent_t e = c.timing_pool.back();
        c.timing_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    NBG_CUDA(cudaEventCreate(&e));
    return e;
}

void timing_begin(Ctx &c, const char *cls, cudaEvent_t *ev0) {
    *ev0 = nullptr;
    if (!c.timing) return;
    *ev0 = get_timing_event(c);
    NBG_CUDA(cudaEventRecord(*ev0, c.stream));
    (void)cls;
}

void timing_end(Ctx &c, const char *cls, cudaEvent_t ev0) {
    if (!c.timing || !ev0) return;
    cudaEvent_t ev1 = get_timing_event(c);
    NBG_CUDA(cudaEventRecord(ev1, c.stream));
    c.tclass[cls].pending.push_back({ev0, ev1});
}

void timing_collect(Ctx &c) {
    for (auto &kv : c.tclass) {
        for (auto &pr : kv.second.pending) {
            NBG_CUDA(cudaEventSynchronize(pr.second));
            float ms = 0.f;
            NBG_CUDA(cudaEventElapsedTime(&ms, pr.first, pr.second));
            kv.second.ms += ms;
            kv.second.launches++;
            c.timing_pool.push_back(pr.first);
            c.timing_pool.push_back(pr.second);
        }
        kv.second.pending.clear();
    }
}

// ---------------------------------------------------------------- host arithmetic
// Used for eager folding of iso operands and for host-side scalar ops.  Compiled with
// -ffp-contract=off: each line is one IEEE round-to-nearest operation in the operator's type,
// identical to the device code generated for the same operator.

template <class C>
static C h_div(C a, C b) {
    if constexpr (std::is_floating_point<C>::value) return a / b;
    else return b == 0 ? (C)0 : a / b;
}
template <class C>
static C h_abs(C a) {
    if constexpr (std::is_floating_point<C>::value) return std::fabs(a);
    else return a < 0 ? -a : a;
}
template <class C>
static C h_min(C a, C b) {
    if constexpr (std::is_floating_point<C>::value) return std::fmin(a, b);
    else return a < b ? a : b;
}
template <class C>
static C h_max(C a, C b) {
    if constexpr (std::is_floating_point<C>::value) return std::fmax(a, b);
    else return a > b ? a : b;
}

template <class C>
static C h_unop(int code, C x, C k0, C k1) {
    switch (code) {
        case NBG_IDENTITY: return x;
        case NBG_AINV: return -x;
        case NBG_ABS: return h_abs(x);
        case NBG_MINV: return h_div((C)1, x);
        case NBG_ADD_C: return x + k0;
        case NBG_MUL_C: return x * k0;
        case NBG_AXPB: { C t = k0 * x; return t + k1; }
        case NBG_ABS_SUB_C: return h_abs(x - k0);
        case NBG_RECIP_SCALED: return x != (C)0 ? h_div(k0, x) : (C)0;
        case NBG_ISZERO: return x == (C)0 ? (C)1 : (C)0;
    }
    fail(NBG_INVALID_VALUE, "unknown unop code");
}

template <class C>
static C h_binop(int code, C x, C y, C k0) {
    switch (code) {
        case NBG_PLUS: return x + y;
        case NBG_MINUS: return x - y;
        case NBG_TIMES: return x * y;
        case NBG_DIV: return h_div(x, y);
        case NBG_MIN: return h_min(x, y);
        case NBG_MAX: return h_max(x, y);
        case NBG_FIRST: return x;
        case NBG_SECOND: return y;
        case NBG_ABSDIFF: return h_abs(x - y);
        case NBG_MAX_DIVX_C: return h_max(h_div(x, k0), y);
    }
    fail(NBG_INVALID_VALUE, "unknown binop code");
}

// values travel as double; a double holding a value of type t converts exactly back to t
double host_round(int t, double v) {
    switch (t) {
        case NBG_BOOL: return v != 0.0 ? 1.0 : 0.0;
        // saturating (an out-of-range double -> integer conversion is undefined; the monoid
        // identities INT_MAX / INT64_MAX arrive here as the nearest doubles)
        case NBG_INT32: return v >= 2147483647.0 ? 2147483647.0 : (v <= -2147483648.0 ? -2147483648.0 : (double)(int)v);
        case NBG_INT64:
            return v >= 9223372036854775807.0 ? 9223372036854775807.0
                                              : (v <= -9223372036854775808.0 ? -9223372036854775808.0 : (double)(long long)v);
        case NBG_FP32: return (double)(float)v;
        default: return v;
    }
}

double host_unop(int code, int t, double x, double c0, double c1) {
    switch (t) {
        case NBG_FP32: return (double)h_unop<float>(code, (float)x, (float)c0, (float)c1);
        case NBG_FP64: return h_unop<double>(code, x, c0, c1);
        case NBG_INT32: return (double)h_unop<int>(code, (int)x, (int)c0, (int)c1);
        case NBG_INT64: return (double)h_unop<long long>(code, (long long)x, (long long)c0, (long long)c1);
        case NBG_BOOL: return h_unop<long long>(code, (long long)x, (long long)c0, (long long)c1) != 0 ? 1.0 : 0.0;
    }
    fail(NBG_INVALID_VALUE, "bad type");
}

double host_binop(int code, int t, double x, double y, double c0) {
    switch (t) {
        case NBG_FP32: return (double)h_binop<float>(code, (float)x, (float)y, (float)c0);
        case NBG_FP64: return h_binop<double>(code, x, y, c0);
        case NBG_INT32: return (double)h_binop<int>(code, (int)x, (int)y, (int)c0);
        case NBG_INT64: return (double)h_binop<long long>(code, (long long)x, (long long)y, (long long)c0);
        case NBG_BOOL: return h_binop<long long>(code, (long long)x, (long long)y, (long long)c0) != 0 ? 1.0 : 0.0;
    }
    fail(NBG_INVALID_VALUE, "bad type");
}

Kernel::~Kernel() {
    if (lib) cudaLibraryUnload(lib);
}

Ctx::~Ctx() {
    if (stream) cudaStreamSynchronize(stream);
    // every member that holds device buffers is released here, while the stream and the pool
    // still exist (members are destroyed only after this body, i.e. after the stream)
    out_targets.clear();
    dist_maps.reset();
    user_nodes.clear();
    memo.clear();
    hints.clear();
    plans.clear();
    cur_slab.reset();
    closing = true;
    for (auto &kv : buf_pool)
        for (void *p : kv.second) cudaFreeAsync(p, stream);
    buf_pool.clear();
    if (stream) cudaStreamSynchronize(stream);
    for (auto e : event_pool) cudaEventDestroy(e);
    for (auto e : timing_pool) cudaEventDestroy(e);
    if (l2_limit_set) {
        // the stream is idle here: release this context's persisting lines and put the device's
        // set-aside back to what it was before this context raised it
        int prev_dev = -1;
        if (cudaGetDevice(&prev_dev) == cudaSuccess) {
            if (prev_dev != device) cudaSetDevice(device);
            if (l2_win_base) cudaCtxResetPersistingL2Cache();
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, l2_limit_prev);
            if (prev_dev != device) cudaSetDevice(prev_dev);
        }
        cudaGetLastError();
    }
    if (rb_stream) {
        cudaStreamSynchronize(rb_stream);
        cudaStreamDestroy(rb_stream);
        cudaEventDestroy(rb_dep);
        rb_stream = nullptr;
    }
    for (auto &kv : tclass)
        for (auto &pr : kv.second.pending) {
            cudaEventDestroy(pr.first);
            cudaEventDestroy(pr.second);
        }
    if (own_stream && stream) cudaStreamDestroy(stream);
}

}  // namespace nbg
