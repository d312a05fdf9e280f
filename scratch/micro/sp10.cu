// micro v10: per-warp flattened stream.  Each warp owns a contiguous range of 32-row blocks; the
// short-row groups of that range are one contiguous stream (long rows live in a separate chunk
// array), consumed 32 groups per step with indices prefetched two steps ahead and gathers one
// step ahead.  Nonempty row starts flow through a per-warp smem queue; completed row sums go to a
// per-warp smem ring; a block's epilogue runs (lane j -> row 32 k + j) once all its rows are done,
// its inputs staged by cp.async when the block entered the queue.
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ float gx(unsigned s_base, const float* X, int c, int hc) {
  float r;
  asm("{ .reg .pred p; setp.lt.s32 p, %1, %2; @p ld.shared.f32 %0, [%3]; @!p ld.global.nc.f32 %0, [%4]; }"
      : "=f"(r) : "r"(c), "r"(hc), "r"(s_base + 4u * (unsigned)(c < hc ? c : 0)), "l"(X + c));
  return r;
}
__device__ __forceinline__ void cpa4(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"((unsigned)__cvta_generic_to_shared(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

constexpr int QN = 128;   // nonempty-start queue (per warp)
constexpr int RN = 128;   // row-sum ring (per warp)
constexpr int EB = 4;     // epilogue-input blocks in flight (per warp)

struct WarpSmem {
  int qs[QN];
  double racc[RN];
  float et[EB][32], ed[EB][32];
  int eg[EB][32];
};

template <int NT>
__global__ void __launch_bounds__(NT, 1) sp10(long long nchunks, const int4* __restrict__ chunks, const int4* __restrict__ longs,
    int* __restrict__ counters, double* __restrict__ partials, const int4* __restrict__ cgl,       // long-row groups
    const int* __restrict__ wk,                  // per warp: first row block (wk[w] .. wk[w+1])
    const long long* __restrict__ grps,          // short-stream start group per row (n + 1)
    const uint2* __restrict__ binfo,             // per block: {nonempty mask, long mask}
    const int4* __restrict__ cgs,                // short stream
    long long n, const float* __restrict__ X, int hc,
    const float* __restrict__ t, const float* __restrict__ dinv, const int* __restrict__ gpos, float c, float* __restrict__ r, float* __restrict__ ynext,
    double* __restrict__ dsum, int* __restrict__ ctr) {
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) unsigned char dyn[];
  float* s_hot = (float*)dyn;
  const unsigned s_base = (unsigned)__cvta_generic_to_shared(s_hot);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpSmem& W = ((WarpSmem*)(dyn + ((hc * 4 + 15) & ~15)))[warp];
  for (int k = threadIdx.x; k < hc; k += NT) s_hot[k] = __ldg(X + k);
  __syncthreads();
  double d = 0.0;
  // ---- long-row chunks (global queue, lean loop)
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
      for (int v = 0; v < 4; v++) { const int gi = b + lane + 32 * v; q[v] = gi < cnt ? __ldcs(cgl + g0 + gi) : make_int4(-1, -1, -1, -1); }
#pragma unroll
      for (int v = 0; v < 4; v++) {
        const float f0 = gx(s_base, X, max(q[v].x, 0), hc), f1 = gx(s_base, X, max(q[v].y, 0), hc), f2 = gx(s_base, X, max(q[v].z, 0), hc), f3 = gx(s_base, X, max(q[v].w, 0), hc);
        acc += (q[v].x >= 0 ? (double)f0 : 0.0) + (q[v].y >= 0 ? (double)f1 : 0.0) + (q[v].z >= 0 ? (double)f2 : 0.0) + (q[v].w >= 0 ? (double)f3 : 0.0);
      }
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
  // ---- my block range
  const int gw = blockIdx.x * NW + warp;
  const int kb = wk[gw], ke = wk[gw + 1];
  if (kb < ke) {
    const long long S0 = grps[32LL * kb];
    const int NS = (int)(grps[min(32LL * ke, n)] - S0);        // groups in my stream
    // starts queue (blocks ks..: nonempty row starts) and epilogue staging (blocks kf .. kf + EB)
    int ks = kb;                 // next block whose starts get queued
    int kf = kb;                 // next block to flush (epilogue)
    int qt = 0;                  // queue tail (nonempty rows queued)
    int qh = 0;                  // queue head (nonempty rows started)
    int rank_f = 0;              // rank of the first nonempty row of block kf
    long long pst = grps[min(32LL * ks + lane, n)];
    unsigned pnm = binfo[ks].x;
    auto append = [&]() {
      if ((pnm >> lane) & 1u) W.qs[(qt + __popc(pnm & ((1u << lane) - 1u))) % QN] = (int)(pst - S0);
      qt += __popc(pnm);
      ++ks;
      if (ks < ke) { pst = grps[min(32LL * ks + lane, n)]; pnm = binfo[ks].x; }
    };
    auto stage = [&](int k) {
      const long long i = 32LL * k + lane;
      const int slot = k % EB;
      if (i < n) { cpa4(&W.et[slot][lane], t + i); cpa4(&W.ed[slot][lane], dinv + i); cpa4(&W.eg[slot][lane], gpos + i); }
      cpa_commit();
    };
    for (int k = kb; k < ke && k < kb + EB; k++) stage(k);
    while (ks < ke && qt - qh < 64) append();
    __syncwarp();
    int4 q0 = lane < NS ? __ldcs(cgs + S0 + lane) : make_int4(-1, -1, -1, -1);
    int4 q1 = 32 + lane < NS ? __ldcs(cgs + S0 + 32 + lane) : make_int4(-1, -1, -1, -1);
    int4 q2 = 64 + lane < NS ? __ldcs(cgs + S0 + 64 + lane) : make_int4(-1, -1, -1, -1);
    float f0 = gx(s_base, X, max(q0.x, 0), hc), f1 = gx(s_base, X, max(q0.y, 0), hc), f2 = gx(s_base, X, max(q0.z, 0), hc), f3 = gx(s_base, X, max(q0.w, 0), hc);
    double carry = 0.0;
    for (int b = 0; b < NS; b += 32) {
      const int4 qc = q0;
      const float c0 = f0, c1 = f1, c2 = f2, c3 = f3;
      q0 = q1; q1 = q2;
      q2 = (b + 96 + lane < NS) ? __ldcs(cgs + S0 + b + 96 + lane) : make_int4(-1, -1, -1, -1);
      if (b + 32 < NS) { f0 = gx(s_base, X, max(q0.x, 0), hc); f1 = gx(s_base, X, max(q0.y, 0), hc); f2 = gx(s_base, X, max(q0.z, 0), hc); f3 = gx(s_base, X, max(q0.w, 0), hc); }
      double S = (qc.x >= 0 ? (double)c0 : 0.0) + (qc.y >= 0 ? (double)c1 : 0.0) + (qc.z >= 0 ? (double)c2 : 0.0) + (qc.w >= 0 ? (double)c3 : 0.0);
      // starts in [b, b + 32): queue entries qh + lane (at most 32 starts per step)
      unsigned ms = 0u;
      if (qh + lane < qt) { const int o = W.qs[(qh + lane) % QN] - b; if (o < 32) ms = 1u << o; }
      const unsigned M = __reduce_or_sync(0xffffffffu, ms);
      if (lane == 0 && (M & 1u) && qh > 0) W.racc[(qh - 1) % RN] = carry;
      if (lane == 0 && !(M & 1u)) S += carry;
      bool F = ((M >> lane) & 1u) || lane == 0;
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
        const double Sy = __shfl_up_sync(0xffffffffu, S, dd);
        const bool Fy = __shfl_up_sync(0xffffffffu, F, dd);
        if (lane >= dd && !F) { S += Sy; F = Fy; }
      }
      const double Sp = __shfl_up_sync(0xffffffffu, S, 1);
      if (lane > 0 && ((M >> lane) & 1u)) W.racc[(qh + __popc(M & ((1u << lane) - 1u)) - 1) % RN] = Sp;
      carry = __shfl_sync(0xffffffffu, S, 31);
      qh += __popc(M);
      const bool last = b + 32 >= NS;
      if (last && lane == 0 && qh > 0) W.racc[(qh - 1) % RN] = carry;
      const int done = last ? qh : qh - 1;          // nonempty rows complete
      __syncwarp();
      // flush blocks whose nonempty rows are all complete
      while (kf < ks) {
        const uint2 bi = binfo[kf];
        const int cnt = __popc(bi.x);
        if (rank_f + cnt > done) break;
        cpa_wait_all();
        __syncwarp();
        const long long i = 32LL * kf + lane;
        if (i < n && !((bi.y >> lane) & 1u)) {
          const int slot = kf % EB;
          const double acc = ((bi.x >> lane) & 1u) ? W.racc[(rank_f + __popc(bi.x & ((1u << lane) - 1u))) % RN] : 0.0;
          const float ri = (float)acc + c;
          r[i] = ri; d += fabs((double)ri - (double)W.et[slot][lane]);
          const int gp = W.eg[slot][lane]; if (gp > 0) ynext[gp] = ri * W.ed[slot][lane];
        }
        __syncwarp();
        if (kf + EB < ke) stage(kf + EB);
        rank_f += cnt; ++kf;
      }
      while (ks < ke && qt - qh < 64) append();
      __syncwarp();
    }
    // blocks without any stream (all-empty tail)
    while (kf < ke) {
      while (ks < ke && ks <= kf) append();
      cpa_wait_all();
      __syncwarp();
      const uint2 bi = binfo[kf];
      const long long i = 32LL * kf + lane;
      if (i < n && !((bi.y >> lane) & 1u)) {
        const int slot = kf % EB;
        const double acc = ((bi.x >> lane) & 1u) ? W.racc[(rank_f + __popc(bi.x & ((1u << lane) - 1u))) % RN] : 0.0;
        const float ri = (float)acc + c;
        r[i] = ri; d += fabs((double)ri - (double)W.et[slot][lane]);
        const int gp = W.eg[slot][lane]; if (gp > 0) ynext[gp] = ri * W.ed[slot][lane];
      }
      __syncwarp();
      if (kf + EB < ke) stage(kf + EB);
      rank_f += __popc(bi.x); ++kf;
    }
  }
  for (int o = 16; o; o >>= 1) d += __shfl_down_sync(0xffffffffu, d, o);
  if (lane == 0) atomicAdd(dsum, d);
}

extern "C" int sp10_run(int nt, long long nchunks, const void* chunks, const void* longs, int* counters, double* partials, const void* cgl,
    const int* wk, const long long* grps, const void* binfo, const void* cgs, long long n, const float* X, int hc,
    const float* t, const float* dinv, const int* gpos, float c, float* r, float* ynext, double* dsum, int* ctr) {
  cudaMemsetAsync(ctr, 0, 4);
  const int smem = ((hc * 4 + 15) & ~15) + (nt / 32) * (int)sizeof(WarpSmem);
#define GO(NT_) if (nt == NT_) { cudaFuncSetAttribute(sp10<NT_>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
  sp10<NT_><<<148, NT_, smem>>>(nchunks, (const int4*)chunks, (const int4*)longs, counters, partials, (const int4*)cgl, wk, grps, (const uint2*)binfo, (const int4*)cgs, n, X, hc, t, dinv, gpos, c, r, ynext, dsum, ctr); \
  return (int)cudaGetLastError(); }
  GO(1024) GO(768) GO(512)
#undef GO
  return -1;
}
