// micro prototype v7: each warp streams a contiguous range of row tiles; next step's indices and next tile's header,
// row starts and epilogue inputs are prefetched one step / one tile ahead.
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ float gx(const float* s_hot, const float* X, int c, int hc) {
  float r;
  asm volatile("{ .reg .pred p; setp.lt.s32 p, %1, %2; @p ld.shared.f32 %0, [%3]; @!p ld.global.nc.f32 %0, [%4]; }"
               : "=f"(r) : "r"(c), "r"(hc), "r"((unsigned)__cvta_generic_to_shared(s_hot) + 4u * (unsigned)(c < hc ? c : 0)), "l"(X + c));
  return r;
}
__device__ __forceinline__ int4 ldidx(const int* colidx, long long P0, long long pe) {
  return (P0 < pe) ? __ldcs((const int4*)(colidx + P0)) : make_int4(0, 0, 0, 0);
}

struct TileH { long long ps, pe; int rb, R; };

__global__ void __launch_bounds__(1024, 1) sp7(long long nchunks, const int* __restrict__ wt, const int2* __restrict__ tiles, const longlong2* __restrict__ tnz,
    const int4* __restrict__ chunks, const int4* __restrict__ longs, int* __restrict__ counters, double* __restrict__ partials,
    const long long* __restrict__ rowptr, const int* __restrict__ colidx, const float* __restrict__ X, int hc,
    const float* __restrict__ t, const float* __restrict__ dinv, const int* __restrict__ gpos, float c, float* __restrict__ r, float* __restrict__ ynext,
    double* __restrict__ dsum, int* __restrict__ ctr) {
  extern __shared__ __align__(16) unsigned char dyn[];
  float* s_hot = (float*)dyn;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* s_racc = (double*)(dyn + ((hc * 4 + 15) & ~15)) + warp * 32;
  for (int k = threadIdx.x; k < hc; k += blockDim.x) s_hot[k] = __ldg(X + k);
  __syncthreads();
  double d = 0.0;
  // ---- long-row chunks (global queue)
  for (;;) {
    long long it = 0;
    if (lane == 0) it = atomicAdd(ctr, 1);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= nchunks) break;
    const int4 ch = chunks[it];
    const long long pb = ((long long)(unsigned)ch.z << 32) | (long long)(unsigned)ch.y;
    const long long pe = pb + ch.w;
    double acc = 0.0;
    for (long long base = pb & ~3ll; base < pe; base += 512) {
      int4 q[4];
#pragma unroll
      for (int v = 0; v < 4; v++) q[v] = ldidx(colidx, base + 4 * (lane + 32 * v), pe);
      float f[16];
#pragma unroll
      for (int v = 0; v < 4; v++) { f[4*v] = gx(s_hot, X, q[v].x, hc); f[4*v+1] = gx(s_hot, X, q[v].y, hc); f[4*v+2] = gx(s_hot, X, q[v].z, hc); f[4*v+3] = gx(s_hot, X, q[v].w, hc); }
#pragma unroll
      for (int v = 0; v < 4; v++)
#pragma unroll
        for (int k = 0; k < 4; k++) { const long long P = base + 4 * (lane + 32 * v) + k; if (P >= pb && P < pe) acc += (double)f[4 * v + k]; }
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
  // ---- my contiguous tile range
  const int gw = blockIdx.x * 32 + warp;
  const int ta = wt[gw], tb = wt[gw + 1];
  if (ta < tb) {
    // current tile header + per-lane data
    int2 T0 = tiles[ta]; longlong2 Z0 = tnz[ta];
    long long rs = __ldg(rowptr + T0.x + min(lane, T0.y - T0.x));
    long long rlast = __ldg(rowptr + T0.x + min(32, T0.y - T0.x));
    float tv = 0.f, dv = 0.f; int gp = -1;
    if (lane < T0.y - T0.x) { tv = t[T0.x + lane]; dv = dinv[T0.x + lane]; gp = gpos[T0.x + lane]; }
    long long base = Z0.x & ~3ll;
    int4 q = ldidx(colidx, base + 4 * lane, Z0.y);
    for (int tt = ta; tt < tb; ++tt) {
      // prefetch next tile header
      const bool hasn = tt + 1 < tb;
      int2 T1 = hasn ? tiles[tt + 1] : make_int2(0, 0);
      longlong2 Z1 = hasn ? tnz[tt + 1] : make_longlong2(0, 0);
      const int R = T0.y - T0.x;
      const long long ps = Z0.x, pe = Z0.y;
      const bool valid = lane < R;
      const long long rnext = __shfl_down_sync(0xffffffffu, rs, 1);
      const long long re_ = (lane == 31) ? rlast : rnext;
      const bool starts = valid && re_ > rs;
      const unsigned smask = __ballot_sync(0xffffffffu, starts);
      s_racc[lane] = 0.0;
      double carry = 0.0;
      int crow = -1;
      for (; base < pe; base += 128) {
        // gathers of this step
        float f[4] = {gx(s_hot, X, q.x, hc), gx(s_hot, X, q.y, hc), gx(s_hot, X, q.z, hc), gx(s_hot, X, q.w, hc)};
        // prefetch next step (this tile or the next tile's first step)
        if (base + 128 < pe) q = ldidx(colidx, base + 128 + 4 * lane, pe);
        else if (hasn) q = ldidx(colidx, (Z1.x & ~3ll) + 4 * lane, Z1.y);
        // row-start flags (4 per lane): 4 words of 8 lanes
        const long long off = rs - base;
        const bool in = starts && off >= 0 && off < 128;
        const int tl_ = in ? (int)(off >> 2) : -1, bp = in ? (int)(off & 3) : 0;
        unsigned myflags = 0;
#pragma unroll
        for (int w = 0; w < 4; w++) {
          const unsigned val = (in && (tl_ >> 3) == w) ? (1u << ((tl_ & 7) * 4 + bp)) : 0u;
          const unsigned M = __reduce_or_sync(0xffffffffu, val);
          if ((lane >> 3) == w) myflags = (M >> ((lane & 7) * 4)) & 15u;
        }
        const int cnt = __popc(myflags);
        int incl = cnt;
#pragma unroll
        for (int dd = 1; dd < 32; dd <<= 1) { const int y = __shfl_up_sync(0xffffffffu, incl, dd); if (lane >= dd) incl += y; }
        const unsigned before = __ballot_sync(0xffffffffu, starts && rs < base);
        int fk = __popc(before) + incl - cnt;
        double h = 0.0, cur = 0.0;
        int curow = -1;
#pragma unroll
        for (int k = 0; k < 4; k++) {
          const long long P = base + 4 * lane + k;
          if ((myflags >> k) & 1u) {
            if (curow >= 0) s_racc[curow] = cur;
            curow = __fns(smask, 0, fk + 1);
            ++fk;
            cur = 0.0;
          }
          if (P >= ps && P < pe) { const double m = (double)f[k]; if (curow >= 0) cur += m; else h += m; }
        }
        const bool hf = myflags != 0;
        double S = hf ? cur : h;
        if (lane == 0 && !hf) S += carry;
        bool F = hf || lane == 0;
        int rid = hf ? curow : (lane == 0 ? crow : -1);
#pragma unroll
        for (int dd = 1; dd < 32; dd <<= 1) {
          const double Sy = __shfl_up_sync(0xffffffffu, S, dd);
          const bool Fy = __shfl_up_sync(0xffffffffu, F, dd);
          const int ry = __shfl_up_sync(0xffffffffu, rid, dd);
          if (lane >= dd && !F) { S = Sy + S; F = Fy; rid = ry; }
        }
        double Sl = __shfl_up_sync(0xffffffffu, S, 1);
        int rl = __shfl_up_sync(0xffffffffu, rid, 1);
        if (lane == 0) { Sl = carry; rl = crow; }
        if (hf && rl >= 0) s_racc[rl] = Sl + h;
        carry = __shfl_sync(0xffffffffu, S, 31);
        crow = __shfl_sync(0xffffffffu, rid, 31);
      }
      if (lane == 0 && crow >= 0) s_racc[crow] = carry;
      // prefetch next tile's row starts / epilogue inputs before the epilogue of this one
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
      T0 = T1; Z0 = Z1; rs = rs1; rlast = rl1; tv = tv1; dv = dv1; gp = gp1;
      base = Z0.x & ~3ll;
    }
  }
  for (int o = 16; o; o >>= 1) d += __shfl_down_sync(0xffffffffu, d, o);
  if (lane == 0) atomicAdd(dsum, d);
}

extern "C" int sp7_run(long long nchunks, const int* wt, const void* tiles, const void* tnz, const void* chunks, const void* longs, int* counters, double* partials,
    const long long* rowptr, const int* colidx, const float* X, int hc, const float* t, const float* dinv, const int* gpos, float c,
    float* r, float* ynext, double* dsum, int* ctr) {
  int smem = ((hc * 4 + 15) & ~15) + 32 * 32 * 8;
  cudaMemsetAsync(ctr, 0, 4);
  cudaFuncSetAttribute(sp7, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  sp7<<<148, 1024, smem>>>(nchunks, wt, (const int2*)tiles, (const longlong2*)tnz, (const int4*)chunks, (const int4*)longs, counters, partials, rowptr, colidx, X, hc, t, dinv, gpos, c, r, ynext, dsum, ctr);
  return (int)cudaGetLastError();
}
