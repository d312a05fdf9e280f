p='paper_2509_14211_b200/csrc/jit/prelude.cuh'; s=open(p).read()
a=s.index("__device__ double nbg_xacc_value(const u64 *L) {")
b=s.index("// order-preserving keys for MIN / MAX combines")
new='''__device__ double nbg_xacc_value(const u64 *L) {
    u64 flags = L[10];
    if (flags & 9ull) return __longlong_as_double(0x7ff8000000000000ll);
    if ((flags & 6ull) == 6ull) return __longlong_as_double(0x7ff8000000000000ll);
    if (flags & 2ull) return __longlong_as_double(0x7ff0000000000000ll);
    if (flags & 4ull) return __longlong_as_double((long long)0xfff0000000000000ull);
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

'''
s=s[:a]+new+s[b:]
open(p,'w').write(s)

p='paper_2509_14211_b200/csrc/runtime.cpp'; s=open(p).read()
a=s.index("    int h = -1;\n    for (int k = 10; k >= 0; k--)\n        if (w[k]) { h = k; break; }")
b=s.index("    double v = std::ldexp((double)mant, lsb - 160);")
new='''    int h = -1;
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
'''
s=s[:a]+new+s[b:]
open(p,'w').write(s)
