// micro v9: CSR with rows padded to 4-entry groups (sentinel 0 = zero column); each lane owns one group (one row)
// per 128-entry step; segmented warp scan keyed by row; tiles <= 32 rows; dynamic batches of tiles per warp.
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ float gx(unsigned s_base, const float* X, int c, int hc) {
  float r;
  asm volatile("{ .reg .pred p; setp.lt.s32 p, %1, %2; @p ld.shared.f32 %0, [%3]; @!p ld.global.nc.f32 %0, [%4]; }"
               : "=f"(r) : "r"(c), "r"(hc), "r"(s_base + 4u * (unsigned)(c < hc ? c : 0)), "l"(X + c));
  return r;
}

template <int NT, int BATCH>
__global__ void __launch_bounds__(NT, 1) sp9(long long ntiles, long long nchunks, const int2* __restrict__ tiles,
    const int4* __restrict__ chunks, const int4* __restrict__ longs, int* __restrict__ counters, double* __restrict__ partials,
    const long long* __restrict__ grp,      // per row: first group index (padded CSR, 4 entries per group), grp[n] = ngroups
    const int4* __restrict__ cg,            // groups of 4 gather indices (sentinel 0)
    const float* __restrict__ X, int hc,
    const float* __restrict__ t, const float* __restrict__ dinv, const int* __restrict__ gpos, float c, float* __restrict__ r, float* __restrict__ ynext,
    double* __restrict__ dsum, int* __restrict__ ctr, int mode) {
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) unsigned char dyn[];
  float* s_hot = (float*)dyn;
  const unsigned s_base = (unsigned)__cvta_generic_to_shared(s_hot);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* s_racc = (double*)(dyn + ((hc * 4 + 15) & ~15)) + warp * 32;
  for (int k = threadIdx.x; k < hc; k += NT) s_hot[k] = __ldg(X + k);
  __syncthreads();
  double d = 0.0;
  // long-row chunks: chunk = group range [g0, g0 + cnt)
  for (;;) {
    long long it = 0;
    if (lane == 0) it = atomicAdd(ctr, 1);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= nchunks) break;
    const int4 ch = chunks[it];
    const long long g0 = ((long long)(unsigned)ch.z << 32) | (long long)(unsigned)ch.y;
    const int cnt = ch.w;
    double acc = 0.0;
    for (int b = 0; b < cnt; b += 128) {
      int4 q[4];
#pragma unroll
      for (int v = 0; v < 4; v++) { const int gi = b + lane + 32 * v; q[v] = gi < cnt ? __ldcs(cg + g0 + gi) : make_int4(0, 0, 0, 0); }
      float f[16];
#pragma unroll
      for (int v = 0; v < 4; v++) { f[4*v] = gx(s_base, X, q[v].x, hc); f[4*v+1] = gx(s_base, X, q[v].y, hc); f[4*v+2] = gx(s_base, X, q[v].z, hc); f[4*v+3] = gx(s_base, X, q[v].w, hc); }
#pragma unroll
      for (int k = 0; k < 16; k++) acc += (double)f[k];
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      partials[it] = acc;
      __threadfence();
      const int4 lr = longs[ch.x];
      const int tk = atomicAdd(&counters[ch.x], 1);
      if (tk == lr.z - 1) {
        __threadfence();
        double s = 0.0;
        for (int j = 0; j < lr.z; j++) s += *(volatile double*)(partials + lr.y + j);
        counters[ch.x] = 0;
        const long long i = lr.x;
        const float ri = (float)s + c;
        r[i] = ri; d += fabs((double)ri - (double)t[i]);
        const int gp = gpos[i]; if (gp > 0) ynext[gp] = ri * dinv[i];
      }
    }
  }
  // row tiles in batches
  for (;;) {
    long long t0 = 0;
    if (lane == 0) t0 = atomicAdd(ctr + 1, BATCH);
    t0 = __shfl_sync(0xffffffffu, t0, 0);
    if (t0 >= ntiles) break;
    const long long t1 = min(t0 + BATCH, ntiles);
    for (long long tt = t0; tt < t1; ++tt) {
      const int2 T = tiles[tt];
      const int R = T.y - T.x;
      const bool valid = lane < R;
      const long long i = (long long)T.x + lane;
      float tv = 0.f, dv = 0.f; int gp = -1;
      if (valid) { tv = t[i]; dv = dinv[i]; gp = gpos[i]; }
      const long long gs = grp[T.x + min(lane, R)];                    // my row's first group (lane R: end)
      const long long gnext = __shfl_down_sync(0xffffffffu, gs, 1);
      const long long ge = (lane == 31) ? grp[T.x + min(32, R)] : gnext;
      const long long G0 = __shfl_sync(0xffffffffu, gs, 0);
      const long long G1 = __shfl_sync(0xffffffffu, (lane == 31) ? ge : gs, R < 32 ? R : 31);
      const bool nonempty = valid && ge > gs;
      const unsigned nem = __ballot_sync(0xffffffffu, nonempty);
      const int nbits = __popc(nem);
      const int rgs = (int)(gs - G0);                                   // my row's first group (tile-relative)
      const int rge = (int)(ge - G0) - 1;                               // my row's last group
      double carry = 0.0;
      int nstarted = 0;                                                 // nonempty rows started before the step
      const int NG = (int)(G1 - G0);
      int4 q = (lane < NG) ? __ldcs(cg + G0 + lane) : make_int4(0, 0, 0, 0);
      for (int b = 0; b < NG; b += 32) {
        float f0, f1, f2, f3;
        if (mode & 2) { f0 = (float)q.x; f1 = (float)q.y; f2 = (float)q.z; f3 = (float)q.w; }
        else { f0 = gx(s_base, X, q.x, hc); f1 = gx(s_base, X, q.y, hc); f2 = gx(s_base, X, q.z, hc); f3 = gx(s_base, X, q.w, hc); }
        if (b + 32 < NG) q = (b + 32 + lane < NG) ? __ldcs(cg + G0 + b + 32 + lane) : make_int4(0, 0, 0, 0);
        if (mode & 1) { carry += ((double)f0 + (double)f1) + ((double)f2 + (double)f3); continue; }
        const int os = rgs - b, oe = rge - b;
        const unsigned M = __reduce_or_sync(0xffffffffu, (nonempty && os >= 0 && os < 32) ? (1u << os) : 0u);
        const unsigned Eb = __reduce_or_sync(0xffffffffu, (nonempty && oe >= 0 && oe < 32) ? (1u << oe) : 0u);
        double S = ((double)f0 + (double)f1) + ((double)f2 + (double)f3);
        if (lane == 0 && !(M & 1u)) S += carry;
        bool F = ((M >> lane) & 1u) || lane == 0;
#pragma unroll
        for (int dd = 1; dd < 32; dd <<= 1) {
          const double Sy = __shfl_up_sync(0xffffffffu, S, dd);
          const bool Fy = __shfl_up_sync(0xffffffffu, F, dd);
          if (lane >= dd && !F) { S += Sy; F = Fy; }
        }
        if ((Eb >> lane) & 1u) {
          const int rk = nstarted + __popc(M & ((2u << lane) - 1u)) - 1;
          s_racc[rk] = S;
        }
        const double S31 = __shfl_sync(0xffffffffu, S, 31);
        carry = ((Eb >> 31) & 1u) ? 0.0 : S31;
        nstarted += __popc(M);
      }
      if (mode & 1) { if (lane == 0) s_racc[0] = carry; }
      __syncwarp();
      if (valid) {
        const int rk = __popc(nem & ((1u << lane) - 1u));
        const double acc = nonempty ? s_racc[rk] : 0.0;
        const float ri = (float)acc + c;
        r[i] = ri; d += fabs((double)ri - (double)tv);
        if (gp > 0) ynext[gp] = ri * dv;
      }
      __syncwarp();
    }
  }
  for (int o = 16; o; o >>= 1) d += __shfl_down_sync(0xffffffffu, d, o);
  if (lane == 0) atomicAdd(dsum, d);
}

extern "C" int sp9_run(int mode, int batch, long long ntiles, long long nchunks, const void* tiles, const void* chunks, const void* longs, int* counters, double* partials,
    const long long* grp, const void* cg, const float* X, int hc, const float* t, const float* dinv, const int* gpos, float c,
    float* r, float* ynext, double* dsum, int* ctr) {
  cudaMemsetAsync(ctr, 0, 8);
  int smem = ((hc * 4 + 15) & ~15) + 32 * 32 * 8;
#define GO(B_) if (batch == B_) { cudaFuncSetAttribute(sp9<1024, B_>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
  sp9<1024, B_><<<148, 1024, smem>>>(ntiles, nchunks, (const int2*)tiles, (const int4*)chunks, (const int4*)longs, counters, partials, grp, (const int4*)cg, X, hc, t, dinv, gpos, c, r, ynext, dsum, ctr, mode); \
  return (int)cudaGetLastError(); }
  GO(1) GO(4) GO(16)
#undef GO
  return -1;
}
