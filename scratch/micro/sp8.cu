// micro prototype v8: E entries per lane per step (4*NV), 32-bit tile-relative positions, smem row-start map,
// per-lane segmented sums + one segmented warp scan per step, contiguous tile ranges per warp with prefetch.
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ float gx(unsigned s_base, const float* X, int c, int hc) {
  float r;
  asm volatile("{ .reg .pred p; setp.lt.s32 p, %1, %2; @p ld.shared.f32 %0, [%3]; @!p ld.global.nc.f32 %0, [%4]; }"
               : "=f"(r) : "r"(c), "r"(hc), "r"(s_base + 4u * (unsigned)(c < hc ? c : 0)), "l"(X + c));
  return r;
}

template <int NT, int NV>
__global__ void __launch_bounds__(NT, 1) sp8(long long nchunks, const int* __restrict__ wt, const int2* __restrict__ tiles, const longlong2* __restrict__ tnz,
    const int4* __restrict__ chunks, const int4* __restrict__ longs, int* __restrict__ counters, double* __restrict__ partials,
    const long long* __restrict__ rowptr, const int* __restrict__ colidx, const float* __restrict__ X, int hc,
    const float* __restrict__ t, const float* __restrict__ dinv, const int* __restrict__ gpos, float c, float* __restrict__ r, float* __restrict__ ynext,
    double* __restrict__ dsum, int* __restrict__ ctr) {
  constexpr int E = 4 * NV, STEP = 32 * E, NW = NT / 32;
  extern __shared__ __align__(16) unsigned char dyn[];
  float* s_hot = (float*)dyn;
  const unsigned s_base = (unsigned)__cvta_generic_to_shared(s_hot);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* wbase = dyn + ((hc * 4 + 15) & ~15) + warp * (256 + STEP + STEP / 8);
  double* s_racc = (double*)wbase;                         // [32]
  unsigned char* s_rof = wbase + 256;                      // [STEP] row (lane) starting at a position
  unsigned* s_fl = (unsigned*)(wbase + 256 + STEP);        // [STEP/32] start bitmap
  for (int k = threadIdx.x; k < hc; k += NT) s_hot[k] = __ldg(X + k);
  for (int k = lane; k < STEP / 32; k += 32) s_fl[k] = 0u;
  __syncthreads();
  double d = 0.0;
  for (;;) {
    long long it = 0;
    if (lane == 0) it = atomicAdd(ctr, 1);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= nchunks) break;
    const int4 ch = chunks[it];
    const long long pb = ((long long)(unsigned)ch.z << 32) | (long long)(unsigned)ch.y;
    const int len = ch.w;
    const int* cp = colidx + (pb & ~3ll);
    const int sh = (int)(pb & 3);
    double acc = 0.0;
    for (int b = 0; b < len + sh; b += 512) {
      int4 q[4];
#pragma unroll
      for (int v = 0; v < 4; v++) { const int P0 = b + 4 * (lane + 32 * v); q[v] = (P0 < len + sh) ? __ldcs((const int4*)(cp + P0)) : make_int4(0, 0, 0, 0); }
      float f[16];
#pragma unroll
      for (int v = 0; v < 4; v++) { f[4*v] = gx(s_base, X, q[v].x, hc); f[4*v+1] = gx(s_base, X, q[v].y, hc); f[4*v+2] = gx(s_base, X, q[v].z, hc); f[4*v+3] = gx(s_base, X, q[v].w, hc); }
#pragma unroll
      for (int v = 0; v < 4; v++)
#pragma unroll
        for (int k = 0; k < 4; k++) { const int P = b + 4 * (lane + 32 * v) + k - sh; if (P >= 0 && P < len) acc += (double)f[4 * v + k]; }
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
        const int gp = gpos[i]; if (gp >= 0) ynext[gp] = ri * dinv[i];
      }
    }
  }
  const int gw = blockIdx.x * NW + warp;
  const int ta = wt[gw], tb = wt[gw + 1];
  if (ta < tb) {
    int2 T0 = tiles[ta]; longlong2 Z0 = tnz[ta];
    long long rs = __ldg(rowptr + T0.x + min(lane, T0.y - T0.x));
    long long rl = __ldg(rowptr + T0.x + min(32, T0.y - T0.x));
    float tv = 0.f, dv = 0.f; int gp = -1;
    if (lane < T0.y - T0.x) { tv = t[T0.x + lane]; dv = dinv[T0.x + lane]; gp = gpos[T0.x + lane]; }
    int4 q[NV];
    {
      const long long a0 = Z0.x & ~3ll; const int n0 = (int)(Z0.y - a0);
#pragma unroll
      for (int v = 0; v < NV; v++) { const int P0 = 4 * (lane * NV + v); q[v] = (P0 < n0) ? __ldcs((const int4*)(colidx + a0 + P0)) : make_int4(0, 0, 0, 0); }
    }
    for (int tt = ta; tt < tb; ++tt) {
      const bool hasn = tt + 1 < tb;
      const int2 T1 = hasn ? tiles[tt + 1] : make_int2(0, 0);
      const longlong2 Z1 = hasn ? tnz[tt + 1] : make_longlong2(0, 0);
      const int R = T0.y - T0.x;
      const long long a0 = Z0.x & ~3ll;
      const int sh = (int)(Z0.x - a0);             // positions are relative to a0; valid range [sh, n0)
      const int n0 = (int)(Z0.y - a0);
      const bool valid = lane < R;
      const long long rnext = __shfl_down_sync(0xffffffffu, rs, 1);
      const long long re_ = (lane == 31) ? rl : rnext;
      const bool starts = valid && re_ > rs;
      const int rpos = (int)(rs - a0);             // my row's start (relative)
      s_racc[lane] = 0.0;
      double carry = 0.0;
      int crow = -1;
      int b = 0;
      do {
        float f[E];
#pragma unroll
        for (int v = 0; v < NV; v++) { f[4*v] = gx(s_base, X, q[v].x, hc); f[4*v+1] = gx(s_base, X, q[v].y, hc); f[4*v+2] = gx(s_base, X, q[v].z, hc); f[4*v+3] = gx(s_base, X, q[v].w, hc); }
        // mark row starts of this step
        const int off = rpos - b;
        if (starts && off >= 0 && off < STEP) { s_rof[off] = (unsigned char)lane; atomicOr(&s_fl[off >> 5], 1u << (off & 31)); }
        // prefetch next step
        if (b + STEP < n0) {
#pragma unroll
          for (int v = 0; v < NV; v++) { const int P0 = b + STEP + 4 * (lane * NV + v); q[v] = (P0 < n0) ? __ldcs((const int4*)(colidx + a0 + P0)) : make_int4(0, 0, 0, 0); }
        } else if (hasn) {
          const long long a1 = Z1.x & ~3ll; const int n1 = (int)(Z1.y - a1);
#pragma unroll
          for (int v = 0; v < NV; v++) { const int P0 = 4 * (lane * NV + v); q[v] = (P0 < n1) ? __ldcs((const int4*)(colidx + a1 + P0)) : make_int4(0, 0, 0, 0); }
        }
        __syncwarp();
        // my E flags: positions [E lane, E lane + E)
        const unsigned fw = s_fl[(E * lane) >> 5];
        const unsigned myflags = (E == 32) ? fw : ((fw >> ((E * lane) & 31)) & ((1u << E) - 1u));
        // valid mask of my positions
        const int p0 = b + E * lane;
        double h = 0.0, cur = 0.0;
        int curow = -1;
#pragma unroll
        for (int k = 0; k < E; k++) {
          if ((myflags >> k) & 1u) {
            if (curow >= 0) s_racc[curow] = cur;
            curow = s_rof[E * lane + k];
            cur = 0.0;
          }
          const int P = p0 + k;
          const double m = (P >= sh && P < n0) ? (double)f[k] : 0.0;
          if (curow >= 0) cur += m; else h += m;
        }
        __syncwarp();
        if (lane < STEP / 32) s_fl[lane] = 0u;
        const bool hf = myflags != 0;
        double S = hf ? cur : h;
        if (lane == 0 && !hf) S += carry;
        int key = hf ? curow : (lane == 0 ? crow : -1);   // -1 = no segment head here (continue)
        bool F = hf || lane == 0;
#pragma unroll
        for (int dd = 1; dd < 32; dd <<= 1) {
          const double Sy = __shfl_up_sync(0xffffffffu, S, dd);
          const int ky = __shfl_up_sync(0xffffffffu, (key & 0xff) | (F ? 0x100 : 0), dd);
          if (lane >= dd && !F) { S = Sy + S; F = (ky & 0x100) != 0; key = ((ky & 0xff) == 0xff) ? -1 : (ky & 0xff); }
        }
        double Sl = __shfl_up_sync(0xffffffffu, S, 1);
        int kl = __shfl_up_sync(0xffffffffu, key, 1);
        if (lane == 0) { Sl = carry; kl = crow; }
        if (hf && kl >= 0) s_racc[kl] = Sl + h;
        carry = __shfl_sync(0xffffffffu, S, 31);
        crow = __shfl_sync(0xffffffffu, key, 31);
        b += STEP;
      } while (b < n0);
      if (lane == 0 && crow >= 0) s_racc[crow] = carry;
      long long rs1 = 0, rl1 = 0; float tv1 = 0.f, dv1 = 0.f; int gp1 = -1;
      if (hasn) {
        rs1 = __ldg(rowptr + T1.x + min(lane, T1.y - T1.x));
        rl1 = __ldg(rowptr + T1.x + min(32, T1.y - T1.x));
        if (lane < T1.y - T1.x) { tv1 = t[T1.x + lane]; dv1 = dinv[T1.x + lane]; gp1 = gpos[T1.x + lane]; }
      }
      __syncwarp();
      if (valid) {
        const double acc = s_racc[lane];
        const float ri = (float)acc + c;
        r[T0.x + lane] = ri; d += fabs((double)ri - (double)tv);
        if (gp >= 0) ynext[gp] = ri * dv;
      }
      __syncwarp();
      T0 = T1; Z0 = Z1; rs = rs1; rl = rl1; tv = tv1; dv = dv1; gp = gp1;
    }
  }
  for (int o = 16; o; o >>= 1) d += __shfl_down_sync(0xffffffffu, d, o);
  if (lane == 0) atomicAdd(dsum, d);
}

extern "C" int sp8_run(int nt, int nv, long long nchunks, const int* wt, const void* tiles, const void* tnz, const void* chunks, const void* longs, int* counters, double* partials,
    const long long* rowptr, const int* colidx, const float* X, int hc, const float* t, const float* dinv, const int* gpos, float c,
    float* r, float* ynext, double* dsum, int* ctr) {
  cudaMemsetAsync(ctr, 0, 4);
#define GO(NT_, NV_) if (nt == NT_ && nv == NV_) { constexpr int STEP = 32 * 4 * NV_; int smem = ((hc * 4 + 15) & ~15) + (NT_ / 32) * (256 + STEP + STEP / 8); \
  cudaFuncSetAttribute(sp8<NT_, NV_>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
  sp8<NT_, NV_><<<148, NT_, smem>>>(nchunks, wt, (const int2*)tiles, (const longlong2*)tnz, (const int4*)chunks, (const int4*)longs, counters, partials, rowptr, colidx, X, hc, t, dinv, gpos, c, r, ynext, dsum, ctr); \
  return (int)cudaGetLastError(); }
  GO(1024, 1) GO(1024, 2) GO(512, 2) GO(512, 4)
#undef GO
  return -1;
}
