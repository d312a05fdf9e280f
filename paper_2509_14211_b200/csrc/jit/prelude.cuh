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
    void *peer[8];
    int npeer;
    const int *rb_tasks;
    const int *rb_sell;
    const int *rb_srow;
    const int *rb_swid;
    const int *rb_lrows;
    const unsigned *rb_mask;
    void *rb_tot;
    unsigned *rb_bar;
    long long rb_ntasks;
    long long ooff[NBG_MAX_OUT], olim[NBG_MAX_OUT];
    unsigned long long *rb_done;
    const int *rb_gcnt;
    long long rb_ngrp, rb_gsize;
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

// ------------------------------------------------------------------ per-thread exact accumulator
// For PLUS reductions of fp64 terms (DESIGN.md §4 "P9"): a thread accumulates its terms EXACTLY in
// a 128-bit two's-complement fixed-point integer V (value V * 2^L).  The anchor L is a multiple of
// 32 chosen from the exponent of the thread's first term (its LSB lands 8..39 bits above L); a
// term whose LSB lies more than 44 bits above L flushes V (exactly) into the block's limbs and
// re-anchors; a term below the window goes to the block's limbs directly (exact).  |V| < 2^121 for
// < 2^24 terms per thread, so V never overflows and 32 of them can be summed.  At the end the
// lanes of a warp that share the anchor add their V with an exact 128-bit shuffle tree and one lane
// flushes (no contention).  Every path is exact: the block's value is the exact sum of its terms
// whatever the grouping, so the fused and the per-op kernels give the same bits.  Block limbs
// `loc` use the global slot convention (nbg_xacc_add: 0-9 limbs, 10 non-finite counts, 12 fp64 sum
// of out-of-window terms), live in shared memory, are zeroed before a __syncthreads.
struct nbg_xt { unsigned __int128 v; int L; int init; };
// 64-bit add into shared memory from two native 32-bit atomics (the 64-bit form is a CAS loop on
// this part): low half first, its carry added to the high half with the value's high word.  The
// pair is not atomic as a unit but every carry is counted, so the final value is exact.
__device__ __forceinline__ void nbg_smem_add64(u64 *p, u64 v) {
    unsigned *w = (unsigned *)p;
    const unsigned lo = (unsigned)v, hi = (unsigned)(v >> 32);
    const unsigned old = atomicAdd(w, lo);
    const unsigned c = (old + lo < old) ? 1u : 0u;
    if (hi + c) atomicAdd(w + 1, hi + c);
}
// the exact add of one term into shared block limbs (nbg_xacc_add's arithmetic, smem atomics)
__device__ void nbg_xacc_add_smem(u64 *acc, double d) {
    if (d == 0.0) return;
    long long bits = __double_as_longlong(d);
    int e = (int)((bits >> 52) & 0x7ff);
    if (e == 0x7ff) {
        nbg_smem_add64(&acc[10], nbg_xacc_flag_counts(((bits & 0xFFFFFFFFFFFFFull) != 0) ? 1ull : (bits < 0 ? 4ull : 2ull)));
        return;
    }
    u64 m = (u64)bits & 0xFFFFFFFFFFFFFull;
    int ex;
    if (e == 0) ex = -1074; else { m |= (1ull << 52); ex = e - 1075; }
    int pos = ex + 160;
    if (pos > 235 || pos + 52 < 0) { atomicAdd((double *)&acc[12], d); return; }
    if (pos < 0) { m >>= -pos; pos = 0; if (m == 0) return; }
    int k = pos >> 5, sh = pos & 31;
    u64 lo = m << sh;
    u64 hi = sh ? (m >> (64 - sh)) : 0ull;
    u64 p0 = lo & 0xffffffffull, p1 = lo >> 32, p2 = hi;
    if (bits < 0) { p0 = (u64)(-(long long)p0); p1 = (u64)(-(long long)p1); p2 = (u64)(-(long long)p2); }
    if (p0) nbg_smem_add64(&acc[k], p0);
    if (p1) nbg_smem_add64(&acc[k + 1], p1);
    if (p2) nbg_smem_add64(&acc[k + 2], p2);
}
__device__ __forceinline__ nbg_xt nbg_xt_zero() { nbg_xt a; a.v = 0; a.L = 0; a.init = 0; return a; }
// V * 2^L into the block limbs (by value: the caller's accumulator stays in registers)
__device__ __noinline__ void nbg_xt_flush_v(unsigned __int128 v, int L, u64 *loc) {
    if (v == 0) return;
    const bool neg = (long long)(v >> 64) < 0;
    const unsigned __int128 mag = neg ? (unsigned __int128)0 - v : v;
    const int pos = L + 160;
    const int hb = (mag >> 64) ? 127 - __clzll((long long)(u64)(mag >> 64)) : 63 - __clzll((long long)(u64)mag);
    if (pos < 0 || pos + hb >= 319) {
        // outside the limb window (wider than any PageRank value): fp64, arrival order
        const double dv = ((double)(u64)(mag >> 64) * 18446744073709551616.0 + (double)(u64)mag) * ldexp(1.0, L);
        atomicAdd((double *)&loc[12], neg ? -dv : dv);
    } else {
        const int k0 = pos >> 5, sh = pos & 31;
        const unsigned __int128 lo = mag << sh;
        const u64 pc[5] = {(u64)lo & 0xffffffffull, (u64)(lo >> 32) & 0xffffffffull, (u64)(lo >> 64) & 0xffffffffull,
                           (u64)(lo >> 96) & 0xffffffffull, sh ? (u64)(mag >> (128 - sh)) : 0ull};
        for (int i = 0; i < 5; i++)
            if (pc[i] && k0 + i <= 9) nbg_smem_add64(&loc[k0 + i], neg ? (u64)(-(long long)pc[i]) : pc[i]);
    }
}
__device__ __forceinline__ int nbg_xt_anchor(int ex) { return ((ex - 8) & ~31) - 0; }
// everything but the common case (first term, re-anchor, below the window, non-finite, subnormal)
__device__ __noinline__ nbg_xt nbg_xt_slow(nbg_xt a, double d, u64 *loc) {
    if (d == 0.0) return a;
    const long long bits = __double_as_longlong(d);
    const int e = (int)((bits >> 52) & 0x7ff);
    if (e == 0x7ff) { nbg_xacc_add_smem(loc, d); return a; }   // non-finite: counted in the block limbs
    u64 m = (u64)bits & 0xFFFFFFFFFFFFFull;
    int ex;
    if (e == 0) ex = -1074; else { m |= (1ull << 52); ex = e - 1075; }
    if (!a.init) { a.L = nbg_xt_anchor(ex); a.init = 1; }
    int sh = ex - a.L;
    if (sh < 0) { nbg_xacc_add_smem(loc, d); return a; }     // far below the window: exact, straight to the block
    if (sh > 44) { nbg_xt_flush_v(a.v, a.L, loc); a.v = 0; a.L = nbg_xt_anchor(ex); sh = ex - a.L; }
    const unsigned __int128 t = ((unsigned __int128)m) << sh;
    a.v = bits < 0 ? a.v - t : a.v + t;
    return a;
}
// the common case inline: a normal term whose LSB lies in the anchored window
__device__ __forceinline__ void nbg_xt_add(nbg_xt &a, double d, u64 *loc) {
    const long long bits = __double_as_longlong(d);
    const int e = (int)((bits >> 52) & 0x7ff);
    const int sh = e - 1075 - a.L;
    if (a.init && (unsigned)(e - 1) < 0x7feu && (unsigned)sh <= 44u) {
        const u64 m = ((u64)bits & 0xFFFFFFFFFFFFFull) | (1ull << 52);
        const u64 lo = m << sh, hi = sh ? (m >> (64 - sh)) : 0ull;
        const unsigned __int128 t = ((unsigned __int128)hi << 64) | lo;
        a.v = bits < 0 ? a.v - t : a.v + t;
    } else if (d != 0.0) {
        a = nbg_xt_slow(a, d, loc);
    }
}
// block finish of one exact reduction (every thread calls it; contains __syncthreads): lanes that
// share lane 0's anchor sum their V exactly (128-bit shuffle tree) and lane 0 flushes it; the
// others (a different anchor) flush their own
__device__ void nbg_block_finish_xt(const nbg_xt a, u64 *loc, u64 *acc) {
    const int lane = threadIdx.x & 31;
    const int L0 = __shfl_sync(0xffffffffu, a.init ? a.L : 0x7fffffff, 0);
    const bool same = a.init && a.L == L0;
    const unsigned own = __ballot_sync(0xffffffffu, a.init && !same);
    if (own & (1u << lane)) nbg_xt_flush_v(a.v, a.L, loc);
    u64 lo = same ? (u64)a.v : 0ull, hi = same ? (u64)(a.v >> 64) : 0ull;
    for (int d = 16; d >= 1; d >>= 1) {
        const u64 l2 = __shfl_down_sync(0xffffffffu, lo, d), h2 = __shfl_down_sync(0xffffffffu, hi, d);
        const u64 s = lo + l2;
        hi = hi + h2 + (s < l2 ? 1ull : 0ull);
        lo = s;
    }
    if (lane == 0 && L0 != 0x7fffffff) nbg_xt_flush_v(((unsigned __int128)hi << 64) | lo, L0, loc);
    __syncthreads();
    const int k = threadIdx.x;
    if (k <= 10) { if (loc[k]) atomicAdd(&acc[k], loc[k]); }
    else if (k == 12) { const double dd = __longlong_as_double((long long)loc[12]); if (dd != 0.0) atomicAdd((double *)&acc[12], dd); }
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

// Grid-wide barrier of a persistent kernel whose CTAs are all resident (one per SM, grid <= SMs):
// bar[0] counts arrivals, bar[1] is the generation.  The generation is read before arriving, the
// last arriver resets the count (and `reset`, a counter every CTA is done with) and releases the
// next generation; the others spin on it.  Writes
// before the barrier (any CTA) are visible to reads after it (fences on both sides, __syncthreads).
__device__ __forceinline__ void nbg_grid_sync(unsigned *bar, unsigned *reset = nullptr) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned gen;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(gen) : "l"(bar + 1) : "memory");
        __threadfence();
        const unsigned old = atomicAdd(bar, 1u);
        if (old == gridDim.x - 1) {
            atomicExch(bar, 0u);
            if (reset) atomicExch(reset, 0u);   // a counter every CTA is done with (the next launch starts from 0)
            __threadfence();
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(bar + 1) : "memory");
        } else {
            unsigned cur;
            for (;;) {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 1) : "memory");
                if (cur != gen) break;
                __nanosleep(64);
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// bulk prefetch of [p, p + bytes) into L2 (TMA engine, fire and forget); p 16-byte aligned
__device__ __forceinline__ void nbg_prefetch_l2(const void *p, long long bytes) {
    bytes &= ~15ll;
    for (long long o = 0; o < bytes; o += (1ll << 20)) {
        const unsigned b = (unsigned)((bytes - o) < (1ll << 20) ? (bytes - o) : (1ll << 20));
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"((const char *)p + o), "r"(b) : "memory");
    }
}

__device__ __forceinline__ int nbg_ld_stream(const int *p) { return __ldcs(p); }

// ------------------------------------------------------------------ TMA bulk copies + mbarriers
// (ewise TMA skeleton, codegen.cpp gen_ewise): one thread arms a stage's mbarrier with the byte
// count and issues 1-D bulk copies global -> shared that complete on it; consumers wait on the
// stage's phase parity.
__device__ __forceinline__ unsigned nbg_smem_addr(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void nbg_mbar_init(u64 *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(nbg_smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void nbg_mbar_expect_tx(u64 *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(nbg_smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void nbg_mbar_wait(u64 *bar, unsigned parity) {
    asm volatile("{\n .reg .pred p_;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p_, [%0], %1;\n @!p_ bra W_%=;\n}"
                 :: "r"(nbg_smem_addr(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void nbg_bulk_g2s(void *dst, const void *src, unsigned bytes, u64 *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(nbg_smem_addr(dst)), "l"(src), "r"(bytes), "r"(nbg_smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void nbg_fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

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
__device__ __forceinline__ unsigned nbg_gx32el(unsigned sbase, const void *X, int c, int hc) {
    unsigned r;
    asm("{ .reg .pred p; setp.lt.s32 p, %1, %2; @p ld.shared.b32 %0, [%3]; @!p ld.global.nc.L1::evict_last.b32 %0, [%4]; }"
        : "=r"(r) : "r"(c), "r"(hc), "r"(sbase + 4u * (unsigned)(c < hc ? c : 0)), "l"((const unsigned *)X + c));
    return r;
}
__device__ __forceinline__ unsigned long long nbg_gx64el(unsigned sbase, const void *X, int c, int hc) {
    unsigned long long r;
    asm("{ .reg .pred p; setp.lt.s32 p, %1, %2; @p ld.shared.b64 %0, [%3]; @!p ld.global.nc.L1::evict_last.b64 %0, [%4]; }"
        : "=l"(r) : "r"(c), "r"(hc), "r"(sbase + 8u * (unsigned)(c < hc ? c : 0)), "l"((const unsigned long long *)X + c));
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
