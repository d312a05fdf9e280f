// micro: SELL-P-pow2 SpMV (rows in P order = length-descending; power-of-two lane groups per row;
// [slice][k][lane] index layout with sentinel 0 -> zero column; xor-tree per group; long rows as chunks)
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ float gx(unsigned s_base, const float* X, int c, int hc) {
  float r;
  asm volatile("{ .reg .pred p; setp.lt.s32 p, %1, %2; @p ld.shared.f32 %0, [%3]; @!p ld.global.nc.f32 %0, [%4]; }"
               : "=f"(r) : "r"(c), "r"(hc), "r"(s_base + 4u * (unsigned)(c < hc ? c : 0)), "l"(X + c));
  return r;
}

template <int NT, int U>
__global__ void __launch_bounds__(NT, 1) sellp(int nslices, const int* __restrict__ wt, const longlong4* __restrict__ hdr, const int* __restrict__ idx,
    long long nlong, long long nchunks, const int4* __restrict__ chunks, const int4* __restrict__ longs, int* __restrict__ counters, double* __restrict__ partials,
    const long long* __restrict__ rowptr, const int* __restrict__ colidx1,      // CSR with +1 gather indices (long rows)
    const float* __restrict__ X, int hc, long long n, long long nempty0,
    const float* __restrict__ tP, const float* __restrict__ dP, const int* __restrict__ gP, float c, float* __restrict__ rP, float* __restrict__ ynext,
    double* __restrict__ dsum, int* __restrict__ ctr) {
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) float s_hot[];
  const unsigned s_base = (unsigned)__cvta_generic_to_shared(s_hot);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < hc; k += NT) s_hot[k] = __ldg(X + k);
  __syncthreads();
  double d = 0.0;
  // long-row chunks
  for (;;) {
    long long it = 0;
    if (lane == 0) it = atomicAdd(ctr, 1);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= nchunks) break;
    const int4 ch = chunks[it];
    const long long pb = ((long long)(unsigned)ch.z << 32) | (long long)(unsigned)ch.y;
    const int len = ch.w;
    const int* cp = colidx1 + (pb & ~3ll);
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
        rP[i] = ri; d += fabs((double)ri - (double)tP[i]);
        const int gp = gP[i]; if (gp > 0) ynext[gp] = ri * dP[i];
      }
    }
  }
  // slices
  const int gw = blockIdx.x * NW + warp;
  const int sa = wt[gw], sb = wt[gw + 1];
  longlong4 hn = (sa < sb) ? hdr[sa] : make_longlong4(0, 0, 0, 0);
  for (int s = sa; s < sb; ++s) {
    const longlong4 h = hn;
    if (s + 1 < sb) hn = hdr[s + 1];
    const long long off = h.x, base = h.y;
    const int L = (int)(h.z & 0xffff), R = (int)(h.z >> 16), lg = (int)(h.w & 0xff), nr = (int)(h.w >> 8);
    const int* ip = idx + off + lane;
    if (lg == 0) {
      // R rows per lane (row r of lane = P-row base + 32 r + lane), R * L <= 16 entries
      const int RL = R * L;
      float tv[8], dv[8]; int gp[8];
#pragma unroll
      for (int r = 0; r < 8; r++) {
        const int q = 32 * r + lane;
        tv[r] = 0.f; dv[r] = 0.f; gp[r] = -1;
        if (r < R && q < nr) { tv[r] = tP[base + q]; dv[r] = dP[base + q]; gp[r] = gP[base + q]; }
      }
      int cc[16];
#pragma unroll
      for (int e = 0; e < 16; e++) cc[e] = (e < RL) ? __ldcs(ip + 32 * e) : 0;
      float f[16];
#pragma unroll
      for (int e = 0; e < 16; e++) f[e] = gx(s_base, X, cc[e], hc);
      double acc = 0.0;
      int r = 0, k = 0;
#pragma unroll
      for (int e = 0; e < 16; e++) {
        if (e < RL) {
          acc += (double)f[e];
          if (++k == L) {
            const int q = 32 * r + lane;
            if (q < nr) {
              float t_ = tv[0], d_ = dv[0]; int g_ = gp[0];
#pragma unroll
              for (int z = 1; z < 8; z++) if (r == z) { t_ = tv[z]; d_ = dv[z]; g_ = gp[z]; }
              const float ri = (float)acc + c;
              rP[base + q] = ri; d += fabs((double)ri - (double)t_);
              if (g_ > 0) ynext[g_] = ri * d_;
            }
            acc = 0.0; k = 0; ++r;
          }
        }
      }
    } else {
      const int gsz = 1 << lg;
      const int slot = lane >> lg;
      const bool leader = (lane & (gsz - 1)) == 0 && slot < nr;
      const long long i = base + slot;
      float tv = 0.f, dv = 0.f; int gp = -1;
      if (leader) { tv = tP[i]; dv = dP[i]; gp = gP[i]; }
      double acc = 0.0;
      for (int k0 = 0; k0 < L; k0 += U) {
        int cc[U];
#pragma unroll
        for (int u = 0; u < U; u++) cc[u] = (k0 + u < L) ? __ldcs(ip + 32 * (k0 + u)) : 0;
        float f[U];
#pragma unroll
        for (int u = 0; u < U; u++) f[u] = gx(s_base, X, cc[u], hc);
#pragma unroll
        for (int u = 0; u < U; u++) acc += (double)f[u];
      }
      for (int o = 1; o < 32; o <<= 1)
        if (o < gsz) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (leader) {
        const float ri = (float)acc + c;
        rP[i] = ri; d += fabs((double)ri - (double)tv);
        if (gp > 0) ynext[gp] = ri * dv;
      }
    }
  }
  // empty tail [nempty0, n): acc = 0
  for (long long i = nempty0 + (long long)blockIdx.x * NT + threadIdx.x; i < n; i += (long long)gridDim.x * NT) {
    const float ri = c;
    rP[i] = ri; d += fabs((double)ri - (double)tP[i]);
    const int gp = gP[i]; if (gp > 0) ynext[gp] = ri * dP[i];
  }
  for (int o = 16; o; o >>= 1) d += __shfl_down_sync(0xffffffffu, d, o);
  if (lane == 0) atomicAdd(dsum, d);
}

extern "C" int sellp_run(int U, int nslices, const int* wt, const void* hdr, const int* idx, long long nlong, long long nchunks, const void* chunks, const void* longs,
    int* counters, double* partials, const long long* rowptr, const int* colidx1, const float* X, int hc, long long n, long long nempty0,
    const float* tP, const float* dP, const int* gP, float c, float* rP, float* ynext, double* dsum, int* ctr) {
  cudaMemsetAsync(ctr, 0, 4);
  int smem = hc * 4;
#define GO(U_) if (U == U_) { cudaFuncSetAttribute(sellp<1024, U_>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
  sellp<1024, U_><<<148, 1024, smem>>>(nslices, wt, (const longlong4*)hdr, idx, nlong, nchunks, (const int4*)chunks, (const int4*)longs, counters, partials, rowptr, colidx1, X, hc, n, nempty0, tP, dP, gP, c, rP, ynext, dsum, ctr); \
  return (int)cudaGetLastError(); }
  GO(4) GO(8) GO(16)
#undef GO
  return -1;
}
