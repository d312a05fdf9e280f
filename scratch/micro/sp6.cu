// micro prototype of SpMV skeleton v6 (row tasks of <= 32 rows / <= 2048 nnz, 256-entry steps,
// REDUX row-start flags, prefetched indices, predicated hot/cold gathers; chunk tasks for long rows)
#include <cuda_runtime.h>
#include <cstdint>
typedef unsigned long long u64;

__device__ __forceinline__ float gx(const float* s_hot, const float* X, int c, int hc) {
  float r;
  asm volatile("{ .reg .pred p; setp.lt.s32 p, %1, %2; @p ld.shared.f32 %0, [%3]; @!p ld.global.nc.f32 %0, [%4]; }"
               : "=f"(r) : "r"(c), "r"(hc), "r"((unsigned)__cvta_generic_to_shared(s_hot) + 4u * (unsigned)(c < hc ? c : 0)), "l"(X + c));
  return r;
}

template <int E>   // entries per lane per step (multiple of 4)
__global__ void __launch_bounds__(1024, 1) sp6(long long ntasks, long long nchunks, const int2* __restrict__ tiles, const int4* __restrict__ chunks,
    const int4* __restrict__ longs, int* __restrict__ counters, double* __restrict__ partials,
    const long long* __restrict__ rowptr, const int* __restrict__ colidx, long long nnz, const float* __restrict__ X, int hc,
    const float* __restrict__ t, const float* __restrict__ dinv, const int* __restrict__ gpos, float c, float* __restrict__ r, float* __restrict__ ynext,
    double* __restrict__ dsum, int* __restrict__ ctr) {
  extern __shared__ __align__(16) unsigned char dyn[];
  float* s_hot = (float*)dyn;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* s_racc = (double*)(dyn + ((hc * 4 + 15) & ~15)) + warp * 32;
  for (int k = threadIdx.x; k < hc; k += blockDim.x) s_hot[k] = __ldg(X + k);
  __syncthreads();
  constexpr int STEP = 32 * E, NV = E / 4;
  double d = 0.0;
  const long long items = nchunks + ntasks;
  for (;;) {
    long long it = 0;
    if (lane == 0) it = atomicAdd(ctr, 1);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= items) break;
    if (it < nchunks) {
      const int4 ch = chunks[it];
      const long long pb = ((long long)(unsigned)ch.z << 32) | (long long)(unsigned)ch.y;
      const long long pe = pb + ch.w;
      double acc = 0.0;
      for (long long base = pb & ~3ll; base < pe; base += STEP) {
        int4 q[NV];
#pragma unroll
        for (int v = 0; v < NV; v++) { const long long P0 = base + 4 * (lane + 32 * v); q[v] = (P0 < pe) ? __ldcs((const int4*)(colidx + P0)) : make_int4(0, 0, 0, 0); }
        float f[E];
#pragma unroll
        for (int v = 0; v < NV; v++) { f[4*v] = gx(s_hot, X, q[v].x, hc); f[4*v+1] = gx(s_hot, X, q[v].y, hc); f[4*v+2] = gx(s_hot, X, q[v].z, hc); f[4*v+3] = gx(s_hot, X, q[v].w, hc); }
#pragma unroll
        for (int v = 0; v < NV; v++)
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
      continue;
    }
    // ---- row task
    const int2 tl = tiles[it - nchunks];
    const int R = tl.y - tl.x;
    const long long i = (long long)tl.x + lane;
    const bool valid = lane < R;
    // epilogue inputs, issued early
    float tv = 0.f, dv = 0.f; int gp = -1;
    if (valid) { tv = t[i]; dv = dinv[i]; gp = gpos[i]; }
    const long long rs = __ldg(rowptr + tl.x + (lane < R ? lane : R));
    const long long rnext = __shfl_down_sync(0xffffffffu, rs, 1);
    const long long re_ = (lane == 31) ? __ldg(rowptr + tl.x + (R < 32 ? R : 32)) : rnext;
    const long long ps = __shfl_sync(0xffffffffu, rs, 0);
    const long long pe = __shfl_sync(0xffffffffu, (lane == 31) ? re_ : rs, R < 32 ? R : 31);
    const bool starts = valid && re_ > rs;         // nonempty row j starts at rs
    s_racc[lane] = 0.0;
    __syncwarp();
    double carry = 0.0;
    int crow = -1;
    long long base = ps & ~3ll;
    int4 q[NV];
#pragma unroll
    for (int v = 0; v < NV; v++) { const long long P0 = base + 4 * (lane * NV + v); q[v] = (P0 < pe) ? __ldcs((const int4*)(colidx + P0)) : make_int4(0, 0, 0, 0); }
    for (; base < pe; base += STEP) {
      // gathers for this step
      float f[E];
#pragma unroll
      for (int v = 0; v < NV; v++) { f[4*v] = gx(s_hot, X, q[v].x, hc); f[4*v+1] = gx(s_hot, X, q[v].y, hc); f[4*v+2] = gx(s_hot, X, q[v].z, hc); f[4*v+3] = gx(s_hot, X, q[v].w, hc); }
      // prefetch next step's indices
#pragma unroll
      for (int v = 0; v < NV; v++) { const long long P0 = base + STEP + 4 * (lane * NV + v); q[v] = (P0 < pe) ? __ldcs((const int4*)(colidx + P0)) : make_int4(0, 0, 0, 0); }
      // row-start flags of this step: lane l owns positions [base + E l, base + E l + E)
      const long long off = rs - base;
      const bool in = starts && off >= 0 && off < STEP;
      const int tl_ = in ? (int)(off / E) : -1, bp = in ? (int)(off % E) : 0;
      unsigned myflags = 0;
      // word w holds lanes with (target lane % (32/E)) ... generic: E bits per lane, 32/E lanes per word
      constexpr int LPW = 32 / E;                 // lanes per 32-bit word
#pragma unroll
      for (int w = 0; w < 32 / LPW; w++) {
        const unsigned val = (in && tl_ / LPW == w) ? (1u << ((tl_ % LPW) * E + bp)) : 0u;
        const unsigned M = __reduce_or_sync(0xffffffffu, val);
        if (lane / LPW == w) myflags = (M >> ((lane % LPW) * E)) & ((E == 32) ? 0xffffffffu : ((1u << E) - 1));
      }
      // row index of my first flag: rows started before my first position within this step + rows before the step
      // count flags in lanes < lane via warp inclusive scan of popc
      int cnt = __popc(myflags);
      int incl = cnt;
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) { const int y = __shfl_up_sync(0xffffffffu, incl, dd); if (lane >= dd) incl += y; }
      const int excl = incl - cnt;
      // row index (task-local) of the k-th flag overall = index of the row start; rows are numbered by their start order
      // among NONEMPTY rows -> map via the owner lanes: rank r -> lane j with the r-th start. Build with ballot of 'starts'
      const unsigned smask = __ballot_sync(0xffffffffu, starts);
      // rows that started before this step: popc(smask & lanes with rs < base)
      const unsigned before = __ballot_sync(0xffffffffu, starts && rs < base);
      const int nbefore = __popc(before);
      // lane-sequential segments
      double h = 0.0, cur = 0.0;
      int curow = -1;
      int fk = nbefore + excl;           // rank (among nonempty rows) of my next flag
#pragma unroll
      for (int k = 0; k < E; k++) {
        const long long P = base + (long long)lane * E + k;
        if ((myflags >> k) & 1u) {
          if (curow >= 0) s_racc[curow] = cur;
          curow = __fns(smask, 0, fk + 1);     // lane index of the (fk)-th set bit
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
    __syncwarp();
    if (valid) {
      const double acc = s_racc[lane];
      const float ri = (float)acc + c;
      r[i] = ri; d += fabs((double)ri - (double)tv);
      if (gp >= 0) ynext[gp] = ri * dv;
    }
    __syncwarp();
  }
  for (int o = 16; o; o >>= 1) d += __shfl_down_sync(0xffffffffu, d, o);
  if (lane == 0) atomicAdd(dsum, d);
}

extern "C" int sp6_run(int E, long long ntasks, long long nchunks, const void* tiles, const void* chunks, const void* longs, int* counters, double* partials,
    const long long* rowptr, const int* colidx, long long nnz, const float* X, int hc, const float* t, const float* dinv, const int* gpos, float c,
    float* r, float* ynext, double* dsum, int* ctr) {
  int smem = ((hc * 4 + 15) & ~15) + 32 * 32 * 8;
  cudaMemsetAsync(ctr, 0, 4);
#define GO(E_) if (E == E_) { cudaFuncSetAttribute(sp6<E_>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
  sp6<E_><<<148, 1024, smem>>>(ntasks, nchunks, (const int2*)tiles, (const int4*)chunks, (const int4*)longs, counters, partials, rowptr, colidx, nnz, X, hc, t, dinv, gpos, c, r, ynext, dsum, ctr); return (int)cudaGetLastError(); }
  GO(4) GO(8) GO(16)
#undef GO
  return -1;
}
