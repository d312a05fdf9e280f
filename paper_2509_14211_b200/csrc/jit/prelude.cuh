// prelude.cuh -- device-side support code prepended to every generated kernel (NVRTC source).
// Self-contained: no #include, so NVRTC needs no header search path on the GPU box.
// Compiled with --fmad=false (no FMA contraction), IEEE division, no FTZ: every operator is one
// round-to-nearest operation in its type, the rounding points DESIGN.md "parity" relies on.

typedef unsigned long long u64;

#define NBG_MAX_IN 16
#define NBG_MAX_OUT 8
#define NBG_MAX_IMM 32
#define NBG_MAX_SIN 8
#define NBG_MAX_RED 8

// Mirror of nbg::KArgs (nbg_internal.hpp): same member order and types.
struct KArgs {
    long long n;
    const void *in[NBG_MAX_IN];
    void *out[NBG_MAX_OUT];
    double imm[NBG_MAX_IMM];
    const u64 *sin[NBG_MAX_SIN];
    u64 *racc[NBG_MAX_RED];
    const long long *rowptr;
    const int *colidx;
    const void *aval;
    const void *x;
    const int *tiles;
    const int *chunks;
    const int *longs;
    int *counters;
    double *partials;
    long long ntiles, nchunks;
    long long row_offset;
    const int *oscat[NBG_MAX_OUT];
    long long hc;
    long long nnz;
    const int *tblk;
    const int *cta;
    const int *pslot;
    const long long *rowslot;
    void *part;
    long long S;
    long long ncols_g;
};

// ------------------------------------------------------------------ operators in type T
__device__ __forceinline__ float nbg_min(float a, float b) { return fminf(a, b); }
__device__ __forceinline__ double nbg_min(double a, double b) { return fmin(a, b); }
__device__ __forceinline__ int nbg_min(int a, int b) { return a < b ? a : b; }
__device__ __forceinline__ long long nbg_min(long long a, long long b) { return a < b ? a : b; }
__device__ __forceinline__ float nbg_max(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ double nbg_max(double a, double b) { return fmax(a, b); }
__device__ __forceinline__ int nbg_max(int a, int b) { return a > b ? a : b; }
__device__ __forceinline__ long long nbg_max(long long a, long long b) { return a > b ? a : b; }
__device__ __forceinline__ float nbg_div(float a, float b) { return a / b; }
__device__ __forceinline__ double nbg_div(double a, double b) { return a / b; }
__device__ __forceinline__ int nbg_div(int a, int b) { return b == 0 ? 0 : a / b; }
__device__ __forceinline__ long long nbg_div(long long a, long long b) { return b == 0 ? 0 : a / b; }
__device__ __forceinline__ float nbg_abs(float a) { return fabsf(a); }
__device__ __forceinline__ double nbg_abs(double a) { return fabs(a); }
__device__ __forceinline__ int nbg_abs(int a) { return a < 0 ? -a : a; }
__device__ __forceinline__ long long nbg_abs(long long a) { return a < 0 ? -a : a; }

// ------------------------------------------------------------------ exact accumulator
// A reduction's cross-block combine: 10 limbs of 32-bit pieces (LSB weight 2^-160) added with
// 64-bit atomics.  Integer addition is associative, so the combined value does not depend on
// the order in which thread blocks finish (deterministic).
// Word 10 of a global slot COUNTS non-finite contributions (NaN in bits 0-20, +inf in 21-41,
// -inf in 42-62; each block / direct term adds at most one per kind), so slots of several ranks
// combine by one integer sum as well.  Per-warp local accumulators keep OR bits (1 NaN, 2 +inf,
// 4 -inf) in word 10; nbg_xacc_flag_counts converts them when they are flushed.
__device__ __forceinline__ u64 nbg_xacc_flag_counts(u64 f) {
    return ((f & 1ull) ? 1ull : 0ull) + ((f & 2ull) ? (1ull << 21) : 0ull) + ((f & 4ull) ? (1ull << 42) : 0ull);
}
__device__ void nbg_xacc_add(u64 *acc, double d) {
    if (d == 0.0) return;
    long long bits = __double_as_longlong(d);
    int e = (int)((bits >> 52) & 0x7ff);
    if (e == 0x7ff) {
        u64 f = ((bits & 0xFFFFFFFFFFFFFull) != 0) ? 1ull : (bits < 0 ? 4ull : 2ull);
        atomicAdd(&acc[10], nbg_xacc_flag_counts(f));
        return;
    }
    u64 m = (u64)bits & 0xFFFFFFFFFFFFFull;
    int ex;
    if (e == 0) ex = -1074; else { m |= (1ull << 52); ex = e - 1075; }
    int pos = ex + 160;
    // terms outside the window [2^-160, 2^128) are summed in fp64 in acc[12] (arrival order); a
    // term straddling the low edge keeps its bits >= 2^-160 (an error < 2^-160, deterministic)
    if (pos > 235 || pos + 52 < 0) { atomicAdd((double *)&acc[12], d); return; }
    if (pos < 0) { m >>= -pos; pos = 0; if (m == 0) return; }
    int k = pos >> 5, sh = pos & 31;
    u64 lo = m << sh;
    u64 hi = sh ? (m >> (64 - sh)) : 0ull;
    u64 p0 = lo & 0xffffffffull, p1 = lo >> 32, p2 = hi;
    if (bits < 0) { p0 = (u64)(-(long long)p0); p1 = (u64)(-(long long)p1); p2 = (u64)(-(long long)p2); }
    if (p0) atomicAdd(&acc[k], p0);
    if (p1) atomicAdd(&acc[k + 1], p1);
    if (p2) atomicAdd(&acc[k + 2], p2);
}

// the same exact add into limbs the caller owns exclusively (shared memory of one warp): no atomics;
// the caller's block has 12 words (11: fp64 sum of out-of-window terms)
__device__ void nbg_xacc_add_local(u64 *acc, double d) {
    if (d == 0.0) return;
    long long bits = __double_as_longlong(d);
    int e = (int)((bits >> 52) & 0x7ff);
    if (e == 0x7ff) {
        acc[10] |= ((bits & 0xFFFFFFFFFFFFFull) != 0) ? 1ull : (bits < 0 ? 4ull : 2ull);
        return;
    }
    u64 m = (u64)bits & 0xFFFFFFFFFFFFFull;
    int ex;
    if (e == 0) ex = -1074; else { m |= (1ull << 52); ex = e - 1075; }
    int pos = ex + 160;
    // outside the window: the caller's acc[11] holds their fp64 sum (flushed into acc[12])
    if (pos > 235 || pos + 52 < 0) { acc[11] = __double_as_longlong(__longlong_as_double(acc[11]) + d); return; }
    if (pos < 0) { m >>= -pos; pos = 0; if (m == 0) return; }
    int k = pos >> 5, sh = pos & 31;
    u64 lo = m << sh;
    u64 hi = sh ? (m >> (64 - sh)) : 0ull;
    u64 p0 = lo & 0xffffffffull, p1 = lo >> 32, p2 = hi;
    if (bits < 0) { p0 = (u64)(-(long long)p0); p1 = (u64)(-(long long)p1); p2 = (u64)(-(long long)p2); }
    acc[k] += p0;
    acc[k + 1] += p1;
    acc[k + 2] += p2;
}

__device__ double nbg_xacc_window(const u64 *L);
__device__ double nbg_xacc_value(const u64 *L) {
    const u64 flags = L[10];
    const u64 nan = flags & 0x1FFFFFull, pinf = (flags >> 21) & 0x1FFFFFull, ninf = (flags >> 42) & 0x1FFFFFull;
    if (nan || (pinf && ninf)) return __longlong_as_double(0x7ff8000000000000ll);
    if (pinf) return __longlong_as_double(0x7ff0000000000000ll);
    if (ninf) return __longlong_as_double((long long)0xfff0000000000000ull);
    const double extra = __longlong_as_double((long long)L[12]);   // out-of-window terms
    return nbg_xacc_window(L) + extra;
}

__device__ double nbg_xacc_window(const u64 *L) {
    unsigned w[11];
    long long carry = 0;
    #pragma unroll
    for (int k = 0; k < 10; k++) {
        long long v = (long long)L[k] + carry;
        w[k] = (unsigned)(v & 0xffffffffll);
        carry = v >> 32;
    }
    w[10] = (unsigned)carry;
    bool neg = carry < 0;
    if (neg) {
        unsigned c = 1;
        #pragma unroll
        for (int k = 0; k < 11; k++) { unsigned long long t = (unsigned long long)(~w[k]) + c; w[k] = (unsigned)t; c = (unsigned)(t >> 32); }
    }
    // word-level extraction of the top 64 bits (no bit loops): top word h, its top bit tb
    int h = -1;
    #pragma unroll
    for (int k = 10; k >= 0; k--) if (h < 0 && w[k]) h = k;
    if (h < 0) return 0.0;
    unsigned wh = 0, wm = 0, wl = 0;
    bool sticky = false;
    #pragma unroll
    for (int k = 0; k < 11; k++) {
        if (k == h) wh = w[k];
        else if (k == h - 1) wm = w[k];
        else if (k == h - 2) wl = w[k];
        else if (k < h - 2 && w[k]) sticky = true;
    }
    const int tb = 31 - __clz(wh);                   // top set bit inside wh
    const int sh = 31 - tb;                          // left shift that puts it at bit 63
    const u64 hi64 = ((u64)wh << 32) | (u64)wm;
    u64 top = sh ? ((hi64 << sh) | ((u64)wl >> (32 - sh))) : hi64;
    const u64 lowmask = sh ? ((1ull << (32 - sh)) - 1ull) : 0xffffffffull;
    if ((u64)wl & lowmask) sticky = true;
    const int g = h * 32 + tb;
    u64 mant = top >> 11;
    u64 rb = top & 0x7ffull;
    if (rb & 0x3ffull) sticky = true;
    int lsb = g - 52;
    if ((rb & 0x400ull) && (sticky || (mant & 1ull))) {
        mant += 1;
        if (mant == (1ull << 53)) { mant >>= 1; lsb += 1; }
    }
    double v = ldexp((double)mant, lsb - 160);
    return neg ? -v : v;
}

// order-preserving keys for MIN / MAX combines (0 = no value yet)
__device__ __forceinline__ u64 nbg_fkey(double x) {
    long long b = __double_as_longlong(x);
    return b < 0 ? ~(u64)b : ((u64)b | 0x8000000000000000ull);
}
__device__ __forceinline__ double nbg_fkey_dec(u64 k) {
    long long b = (k & 0x8000000000000000ull) ? (long long)(k & 0x7fffffffffffffffull) : (long long)(~k);
    return __longlong_as_double(b);
}
__device__ __forceinline__ u64 nbg_ikey(long long x) { return (u64)x ^ 0x8000000000000000ull; }

__device__ double nbg_sval(const u64 *s, int fmt) {
    switch (fmt) {
        case 1: return nbg_xacc_value(s);
        case 2: return (double)(long long)s[11];
        case 3: return s[11] ? nbg_fkey_dec(s[11]) : -__longlong_as_double(0x7ff0000000000000ll);
        case 4: return s[11] ? nbg_fkey_dec(~s[11]) : __longlong_as_double(0x7ff0000000000000ll);
        case 5: return s[11] ? (double)(long long)(s[11] ^ 0x8000000000000000ull) : -9.2233720368547758e18;
        case 6: return s[11] ? (double)(long long)(~s[11] ^ 0x8000000000000000ull) : 9.2233720368547758e18;
    }
    return 0.0;
}
__device__ long long nbg_sval_i(const u64 *s, int fmt) {
    switch (fmt) {
        case 2: return (long long)s[11];
        case 5: return s[11] ? (long long)(s[11] ^ 0x8000000000000000ull) : (long long)0x8000000000000000ull;
        case 6: return s[11] ? (long long)(~s[11] ^ 0x8000000000000000ull) : 0x7fffffffffffffffll;
    }
    return (long long)nbg_sval(s, fmt);
}

// ------------------------------------------------------------------ deterministic block combines
// Fixed shuffle-down tree inside a warp, then warp partials summed in warp order by thread 0.
__device__ __forceinline__ double nbg_warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ long long nbg_warp_sum(long long v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double nbg_warp_min(double v) {
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double nbg_warp_max(double v) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ long long nbg_warp_min(long long v) {
    for (int o = 16; o > 0; o >>= 1) { long long u = __shfl_down_sync(0xffffffffu, v, o); v = u < v ? u : v; }
    return v;
}
__device__ __forceinline__ long long nbg_warp_max(long long v) {
    for (int o = 16; o > 0; o >>= 1) { long long u = __shfl_down_sync(0xffffffffu, v, o); v = u > v ? u : v; }
    return v;
}

// Block-level finish of one reduction; every thread calls it (contains __syncthreads).
// kind: 0 = float PLUS (xacc), 1 = int PLUS, 2 = float MAX, 3 = float MIN, 4 = int MAX, 5 = int MIN
__device__ void nbg_block_finish_f(double v, int kind, u64 *acc, double *sh) {
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double r = kind == 0 ? nbg_warp_sum(v) : (kind == 2 ? nbg_warp_max(v) : nbg_warp_min(v));
    __syncthreads();
    if (lane == 0) sh[w] = r;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = sh[0];
        for (int i = 1; i < nw; i++) t = kind == 0 ? t + sh[i] : (kind == 2 ? fmax(t, sh[i]) : fmin(t, sh[i]));
        if (kind == 0) nbg_xacc_add(acc, t);
        else if (kind == 2) { if (!(t == -__longlong_as_double(0x7ff0000000000000ll))) atomicMax(&acc[11], nbg_fkey(t)); }
        else { if (!(t == __longlong_as_double(0x7ff0000000000000ll))) atomicMax(&acc[11], ~nbg_fkey(t)); }
    }
}
__device__ void nbg_block_finish_i(long long v, int kind, u64 *acc, double *sh) {
    long long *shl = (long long *)sh;
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    long long r = kind == 1 ? nbg_warp_sum(v) : (kind == 4 ? nbg_warp_max(v) : nbg_warp_min(v));
    __syncthreads();
    if (lane == 0) shl[w] = r;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = shl[0];
        for (int i = 1; i < nw; i++) t = kind == 1 ? t + shl[i] : (kind == 4 ? (t > shl[i] ? t : shl[i]) : (t < shl[i] ? t : shl[i]));
        if (kind == 1) atomicAdd(&acc[11], (u64)t);
        else if (kind == 4) { if (t != (long long)0x8000000000000000ull) atomicMax(&acc[11], nbg_ikey(t)); }
        else { if (t != 0x7fffffffffffffffll) atomicMax(&acc[11], ~nbg_ikey(t)); }
    }
}

// loads that bypass / hint the caches
__device__ __forceinline__ int nbg_ld_stream(const int *p) { return __ldcs(p); }

// ------------------------------------------------------------------ SpMV gathers
// x[c] from the shared-memory hot-column cache when c < hc, else from global memory cached in L2
// only (ld.global.cg); both loads are predicated (no divergent branch per element).  The
// caller passes c >= 0 (padding positions are clamped to 0 and masked out afterwards).
__device__ __forceinline__ unsigned nbg_gx32(unsigned sbase, const void *X, int c, int hc) {
    unsigned r;
    asm("{ .reg .pred p; setp.lt.s32 p, %1, %2; @p ld.shared.b32 %0, [%3]; @!p ld.global.cg.b32 %0, [%4]; }"
        : "=r"(r) : "r"(c), "r"(hc), "r"(sbase + 4u * (unsigned)(c < hc ? c : 0)), "l"((const unsigned *)X + c));
    return r;
}
// the same through the read-only path with L1 allocation (matrices whose gathered vector does not
// stay L2-resident keep the L1 hits)
__device__ __forceinline__ unsigned nbg_gx32nc(unsigned sbase, const void *X, int c, int hc) {
    unsigned r;
    asm("{ .reg .pred p; setp.lt.s32 p, %1, %2; @p ld.shared.b32 %0, [%3]; @!p ld.global.nc.b32 %0, [%4]; }"
        : "=r"(r) : "r"(c), "r"(hc), "r"(sbase + 4u * (unsigned)(c < hc ? c : 0)), "l"((const unsigned *)X + c));
    return r;
}
__device__ __forceinline__ unsigned long long nbg_gx64nc(unsigned sbase, const void *X, int c, int hc) {
    unsigned long long r;
    asm("{ .reg .pred p; setp.lt.s32 p, %1, %2; @p ld.shared.b64 %0, [%3]; @!p ld.global.nc.b64 %0, [%4]; }"
        : "=l"(r) : "r"(c), "r"(hc), "r"(sbase + 8u * (unsigned)(c < hc ? c : 0)), "l"((const unsigned long long *)X + c));
    return r;
}
__device__ __forceinline__ unsigned long long nbg_gx64(unsigned sbase, const void *X, int c, int hc) {
    unsigned long long r;
    asm("{ .reg .pred p; setp.lt.s32 p, %1, %2; @p ld.shared.b64 %0, [%3]; @!p ld.global.cg.b64 %0, [%4]; }"
        : "=l"(r) : "r"(c), "r"(hc), "r"(sbase + 8u * (unsigned)(c < hc ? c : 0)), "l"((const unsigned long long *)X + c));
    return r;
}
