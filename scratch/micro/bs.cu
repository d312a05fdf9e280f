// micro-benchmark of the two-phase block-SELL SpMV (phase 1: per column-block partial sums from
// shared memory; phase 2: per-row combine of partials + PageRank-like epilogue).
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// work: per CTA c, slices [cs[c], cs[c+1]); slice q: block sb[q], lcol offset so[q] (in entries), len sl[q]
// per lane-entry j of slice q: slot sslot[32q+j], length slen[32q+j]
template <int NT>
__global__ void __launch_bounds__(NT, 1) p1(const int* __restrict__ cs, const int* __restrict__ sb, const long long* __restrict__ so,
    const int* __restrict__ sl, const int* __restrict__ sslot, const unsigned short* __restrict__ slen,
    const unsigned short* __restrict__ lcol, const float* __restrict__ x, int SB, int ncols, double* __restrict__ part) {
  extern __shared__ __align__(16) float xs[];
  __shared__ int s_q;
  const int q0 = cs[blockIdx.x], q1 = cs[blockIdx.x + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int S = 1 << SB;
  int q = q0;
  while (q < q1) {
    const int b = sb[q];
    int qe = q;  // slices of this block in my range
    // find end of block b within [q, q1)
    {
      // binary search on sb (sorted ascending)
      int lo = q, hi = q1;
      while (lo < hi) { int mid = (lo + hi) >> 1; if (sb[mid] <= b) lo = mid + 1; else hi = mid; }
      qe = lo;
    }
    __syncthreads();
    const int c0 = b * S;
    const int cn = min(S, ncols - c0);
    for (int k = threadIdx.x * 4; k < cn; k += NT * 4) {
      if (k + 3 < cn) { float4 v = __ldg((const float4*)(x + c0 + k)); *(float4*)(xs + k) = v; }
      else for (int u = k; u < cn; u++) xs[u] = __ldg(x + c0 + u);
    }
    __syncthreads();
    for (int qq = q + warp; qq < qe; qq += NT / 32) {
      const long long off = so[qq];
      const int L = sl[qq];
      const int my = slen[32 * qq + lane];
      const unsigned short* lp = lcol + off + lane;
      double acc = 0.0;
      int k = 0;
      for (; k + 4 <= L; k += 4) {
        unsigned short c0_ = __ldcs(lp + 32 * k), c1_ = __ldcs(lp + 32 * (k + 1)), c2_ = __ldcs(lp + 32 * (k + 2)), c3_ = __ldcs(lp + 32 * (k + 3));
        float v0 = xs[c0_], v1 = xs[c1_], v2 = xs[c2_], v3 = xs[c3_];
        if (k < my) acc += (double)v0;
        if (k + 1 < my) acc += (double)v1;
        if (k + 2 < my) acc += (double)v2;
        if (k + 3 < my) acc += (double)v3;
      }
      for (; k < L; k++) { unsigned short c_ = __ldcs(lp + 32 * k); float v = xs[c_]; if (k < my) acc += (double)v; }
      const int s = sslot[32 * qq + lane];
      if (s >= 0) part[s] = acc;
    }
    q = qe;
  }
}

// phase 2: thread per row
__global__ void __launch_bounds__(256) p2(long long n, const int* __restrict__ rslot, const double* __restrict__ part,
    const float* __restrict__ t, const float* __restrict__ dinv, const int* __restrict__ gpos, float c,
    float* __restrict__ r, float* __restrict__ ynext, double* __restrict__ dsum) {
  double d = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int s0 = rslot[i], s1 = rslot[i + 1];
    double acc = 0.0;
    for (int s = s0; s < s1; s++) acc += part[s];
    const float ri = (float)acc + c;
    r[i] = ri;
    d += fabs((double)ri - (double)t[i]);
    const int gp = gpos[i];
    if (gp >= 0) ynext[gp] = ri * dinv[i];
  }
  for (int o = 16; o; o >>= 1) d += __shfl_down_sync(0xffffffffu, d, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(dsum, d);
}

extern "C" {
int bs_p1(int nt, int grid, const int* cs, const int* sb, const long long* so, const int* sl, const int* sslot, const unsigned short* slen,
          const unsigned short* lcol, const float* x, int SB, int ncols, double* part) {
  int smem = (1 << SB) * 4;
  if (nt == 1024) {
    cudaFuncSetAttribute(p1<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    p1<1024><<<grid, 1024, smem>>>(cs, sb, so, sl, sslot, slen, lcol, x, SB, ncols, part);
  } else {
    cudaFuncSetAttribute(p1<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    p1<512><<<grid, 512, smem>>>(cs, sb, so, sl, sslot, slen, lcol, x, SB, ncols, part);
  }
  return (int)cudaGetLastError();
}
int bs_p2(int grid, long long n, const int* rslot, const double* part, const float* t, const float* dinv, const int* gpos, float c,
          float* r, float* ynext, double* dsum) {
  p2<<<grid, 256>>>(n, rslot, part, t, dinv, gpos, c, r, ynext, dsum);
  return (int)cudaGetLastError();
}
}

// ---------------- v2
template <int NT, int L>
__global__ void __launch_bounds__(NT, 1) p1v2(const int* __restrict__ cs, const int* __restrict__ sblk, const int* __restrict__ hdr,
    const int* __restrict__ pslot, const uint4* __restrict__ lcol, const float* __restrict__ x, int SB, int ncols, double* __restrict__ part) {
  extern __shared__ __align__(16) float xs[];
  const int q0 = cs[blockIdx.x], q1 = cs[blockIdx.x + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int S = 1 << SB;
  int q = q0;
  while (q < q1) {
    const int b = sblk[q];
    int lo = q, hi = q1;
    while (lo < hi) { int mid = (lo + hi) >> 1; if (sblk[mid] <= b) lo = mid + 1; else hi = mid; }
    const int qe = lo;
    __syncthreads();
    const int c0 = b * S;
    const int cn = min(S, ncols - c0);
    for (int k = threadIdx.x * 4; k < cn; k += NT * 4) {
      if (k + 3 < cn) { float4 v = __ldg((const float4*)(x + c0 + k)); *(float4*)(xs + k) = v; }
      else for (int u = k; u < cn; u++) xs[u] = __ldg(x + c0 + u);
    }
    __syncthreads();
    for (int s = q + warp; s < qe; s += NT / 32) {
      const uint4* lp = lcol + (long long)s * (L / 8) * 32 + lane;
      uint4 w[L / 8];
#pragma unroll
      for (int v = 0; v < L / 8; v++) w[v] = __ldcs(lp + v * 32);
      int pi = hdr[32 * s + lane];
      int nslot = pslot[pi];
      double acc = 0.0;
#pragma unroll
      for (int v = 0; v < L / 8; v++) {
        const unsigned ww[4] = {w[v].x, w[v].y, w[v].z, w[v].w};
#pragma unroll
        for (int h = 0; h < 8; h++) {
          const unsigned e = (ww[h >> 1] >> ((h & 1) * 16)) & 0xffffu;
          acc += (double)xs[e & 0x7fffu];
          if (e & 0x8000u) { part[nslot] = acc; acc = 0.0; ++pi; nslot = pslot[pi]; }
        }
      }
    }
    q = qe;
  }
}

// phase 2 v2: warp per 32 rows, slots staged in smem
template <int K>
__global__ void __launch_bounds__(256) p2v2(long long n, const int* __restrict__ rslot, const double* __restrict__ part,
    const float* __restrict__ t, const float* __restrict__ dinv, const int* __restrict__ gpos, float c,
    float* __restrict__ r, float* __restrict__ ynext, double* __restrict__ dsum) {
  __shared__ double buf[8][32 * K];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double d = 0.0;
  const long long ngroups = (n + 31) / 32;
  for (long long gi = (long long)blockIdx.x * 8 + warp; gi < ngroups; gi += (long long)gridDim.x * 8) {
    const long long i = gi * 32 + lane;
    const bool valid = i < n;
    const int s0 = valid ? rslot[i] : 0;
    const int s1 = valid ? rslot[i + 1] : 0;
    const int S0 = __shfl_sync(0xffffffffu, s0, 0);
    const int lastv = (int)min((long long)31, n - 1 - gi * 32);
    const int S1 = __shfl_sync(0xffffffffu, s1, lastv);
    double acc = 0.0;
    if (S1 - S0 <= 32 * K) {
#pragma unroll
      for (int m = 0; m < K; m++) { const int s = S0 + m * 32 + lane; if (s < S1) buf[warp][m * 32 + lane] = part[s]; }
      __syncwarp();
      for (int s = s0; s < s1; s++) acc += buf[warp][s - S0];
      __syncwarp();
    } else {
      for (int s = s0; s < s1; s++) acc += part[s];
    }
    if (valid) {
      const float ri = (float)acc + c;
      r[i] = ri;
      d += fabs((double)ri - (double)t[i]);
      const int gp = gpos[i];
      if (gp >= 0) ynext[gp] = ri * dinv[i];
    }
  }
  for (int o = 16; o; o >>= 1) d += __shfl_down_sync(0xffffffffu, d, o);
  if (lane == 0) atomicAdd(dsum, d);
}

extern "C" {
int bs_p1v2(int nt, int L, int grid, const int* cs, const int* sblk, const int* hdr, const int* pslot, const void* lcol,
            const float* x, int SB, int ncols, double* part) {
  int smem = (1 << SB) * 4;
#define GO(NT_, L_) if (nt == NT_ && L == L_) { cudaFuncSetAttribute(p1v2<NT_, L_>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
    p1v2<NT_, L_><<<grid, NT_, smem>>>(cs, sblk, hdr, pslot, (const uint4*)lcol, x, SB, ncols, part); return (int)cudaGetLastError(); }
  GO(1024, 32) GO(1024, 64) GO(512, 64) GO(1024, 128)
#undef GO
  return -1;
}
int bs_p2v2(int K, int grid, long long n, const int* rslot, const double* part, const float* t, const float* dinv, const int* gpos, float c,
            float* r, float* ynext, double* dsum) {
  if (K == 4) p2v2<4><<<grid, 256>>>(n, rslot, part, t, dinv, gpos, c, r, ynext, dsum);
  else p2v2<8><<<grid, 256>>>(n, rslot, part, t, dinv, gpos, c, r, ynext, dsum);
  return (int)cudaGetLastError();
}
}

// ---------------- v3
template <int NT, int L>
__global__ void __launch_bounds__(NT, 1) p1v3(const int* __restrict__ cs, const int* __restrict__ sblk, const int* __restrict__ hdr,
    const uint4* __restrict__ lcol, const float* __restrict__ x, int SB, int ncols, double* __restrict__ part) {
  extern __shared__ __align__(16) float xs[];
  const int q0 = cs[blockIdx.x], q1 = cs[blockIdx.x + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int S = 1 << SB;
  int q = q0;
  while (q < q1) {
    const int b = sblk[q];
    int lo = q, hi = q1;
    while (lo < hi) { int mid = (lo + hi) >> 1; if (sblk[mid] <= b) lo = mid + 1; else hi = mid; }
    const int qe = lo;
    __syncthreads();
    const int c0 = b * S;
    const int cn = min(S, ncols - c0);
    for (int k = threadIdx.x * 4; k < cn; k += NT * 4) {
      if (k + 3 < cn) { float4 v = __ldg((const float4*)(x + c0 + k)); *(float4*)(xs + k) = v; }
      else for (int u = k; u < cn; u++) xs[u] = __ldg(x + c0 + u);
    }
    __syncthreads();
    for (int s = q + warp; s < qe; s += NT / 32) {
      const uint4* lp = lcol + (long long)s * (L / 8) * 32 + lane;
      uint4 w[L / 8];
#pragma unroll
      for (int v = 0; v < L / 8; v++) w[v] = __ldcs(lp + v * 32);
      double* pp = part + hdr[32 * s + lane];
      double acc = 0.0;
#pragma unroll
      for (int v = 0; v < L / 8; v++) {
        const unsigned ww[4] = {w[v].x, w[v].y, w[v].z, w[v].w};
#pragma unroll
        for (int h = 0; h < 8; h++) {
          const unsigned e = (ww[h >> 1] >> ((h & 1) * 16)) & 0xffffu;
          acc += (double)xs[e & 0x7fffu];
          if (e & 0x8000u) { *pp++ = acc; acc = 0.0; }
        }
      }
    }
    q = qe;
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) p2v3(long long n, int ntiles, int nb, const int* __restrict__ tiles, const int* __restrict__ rstart,
    const int* __restrict__ pre, const int* __restrict__ rslot, const unsigned short* __restrict__ qidx, const double* __restrict__ part,
    const float* __restrict__ t, const float* __restrict__ dinv, const int* __restrict__ gpos, float c,
    float* __restrict__ r, float* __restrict__ ynext, double* __restrict__ dsum) {
  extern __shared__ __align__(16) double spart[];
  __shared__ int spre[130], sst[130];
  double d = 0.0;
  for (int tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    const int R0 = tiles[tl], R1 = tiles[tl + 1];
    for (int k = threadIdx.x; k <= nb; k += NT) { spre[k] = pre[tl * (nb + 1) + k]; if (k < nb) sst[k] = rstart[tl * nb + k]; }
    __syncthreads();
    const int P = spre[nb];
    for (int k = threadIdx.x; k < P; k += NT) {
      int lo = 0, hi = nb;   // largest b with spre[b] <= k
      while (hi - lo > 1) { int mid = (lo + hi) >> 1; if (spre[mid] <= k) lo = mid; else hi = mid; }
      spart[k] = part[sst[lo] + k - spre[lo]];
    }
    __syncthreads();
    const long long i = R0 + threadIdx.x;
    if (i < R1) {
      const int s0 = rslot[i], s1 = rslot[i + 1];
      double acc = 0.0;
      int s = s0;
      for (; s + 4 <= s1; s += 4) {
        const unsigned short a0 = qidx[s], a1 = qidx[s + 1], a2 = qidx[s + 2], a3 = qidx[s + 3];
        acc += spart[a0]; acc += spart[a1]; acc += spart[a2]; acc += spart[a3];
      }
      for (; s < s1; s++) acc += spart[qidx[s]];
      const float ri = (float)acc + c;
      r[i] = ri;
      d += fabs((double)ri - (double)t[i]);
      const int gp = gpos[i];
      if (gp >= 0) ynext[gp] = ri * dinv[i];
    }
    __syncthreads();
  }
  for (int o = 16; o; o >>= 1) d += __shfl_down_sync(0xffffffffu, d, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(dsum, d);
}

extern "C" {
int bs_p1v3(int nt, int L, int grid, const int* cs, const int* sblk, const int* hdr, const void* lcol,
            const float* x, int SB, int ncols, double* part) {
  int smem = (1 << SB) * 4;
#define GO(NT_, L_) if (nt == NT_ && L == L_) { cudaFuncSetAttribute(p1v3<NT_, L_>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
    p1v3<NT_, L_><<<grid, NT_, smem>>>(cs, sblk, hdr, (const uint4*)lcol, x, SB, ncols, part); return (int)cudaGetLastError(); }
  GO(1024, 32) GO(1024, 64) GO(512, 64) GO(1024, 128)
#undef GO
  return -1;
}
int bs_p2v3(int nt, int grid, int pmax, long long n, int ntiles, int nb, const int* tiles, const int* rstart, const int* pre, const int* rslot,
            const unsigned short* qidx, const double* part, const float* t, const float* dinv, const int* gpos, float c,
            float* r, float* ynext, double* dsum) {
  int smem = pmax * 8;
#define GO(NT_) if (nt == NT_) { cudaFuncSetAttribute(p2v3<NT_>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
    p2v3<NT_><<<grid, NT_, smem>>>(n, ntiles, nb, tiles, rstart, pre, rslot, qidx, part, t, dinv, gpos, c, r, ynext, dsum); return (int)cudaGetLastError(); }
  GO(1024) GO(512) GO(256)
#undef GO
  return -1;
}
}

// ---------------- v4: variable slices, pieces staged in smem and written coalesced
template <int NT, int L, int C>
__global__ void __launch_bounds__(NT, 1) p1v4(const int* __restrict__ cs, const int* __restrict__ sblk, const int* __restrict__ soff,
    const int* __restrict__ snv, const int* __restrict__ hdr, const uint4* __restrict__ lcol, const float* __restrict__ x, int SB, int ncols,
    double* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char dyn[];
  float* xs = (float*)dyn;
  const int S = 1 << SB;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* pb = (double*)(dyn + S * 4) + warp * C;
  const int q0 = cs[blockIdx.x], q1 = cs[blockIdx.x + 1];
  int q = q0;
  while (q < q1) {
    const int b = sblk[q];
    int lo = q, hi = q1;
    while (lo < hi) { int mid = (lo + hi) >> 1; if (sblk[mid] <= b) lo = mid + 1; else hi = mid; }
    const int qe = lo;
    __syncthreads();
    const int c0 = b * S;
    const int cn = min(S, ncols - c0);
    for (int k = threadIdx.x * 4; k < cn; k += NT * 4) {
      if (k + 3 < cn) { float4 v = __ldg((const float4*)(x + c0 + k)); *(float4*)(xs + k) = v; }
      else for (int u = k; u < cn; u++) xs[u] = __ldg(x + c0 + u);
    }
    __syncthreads();
    for (int s = q + warp; s < qe; s += NT / 32) {
      const int nv = snv[s];
      const uint4* lp = lcol + (long long)soff[s] + lane;
      uint4 w[L / 8];
#pragma unroll
      for (int v = 0; v < L / 8; v++) if (v < nv) w[v] = __ldcs(lp + v * 32);
      const int h0 = hdr[32 * s];
      const int hl = hdr[32 * s + lane];
      const int hn = hdr[32 * s + 32];
      int pi = hl - h0;
      double acc = 0.0;
#pragma unroll
      for (int v = 0; v < L / 8; v++) {
        if (v < nv) {
          const unsigned ww[4] = {w[v].x, w[v].y, w[v].z, w[v].w};
          float f[8];
#pragma unroll
          for (int h = 0; h < 8; h++) f[h] = xs[(ww[h >> 1] >> ((h & 1) * 16)) & 0x7fffu];
#pragma unroll
          for (int h = 0; h < 8; h++) {
            acc += (double)f[h];
            if ((ww[h >> 1] >> ((h & 1) * 16)) & 0x8000u) { pb[pi++] = acc; acc = 0.0; }
          }
        }
      }
      __syncwarp();
      const int np_ = hn - h0;
      for (int k = lane; k < np_; k += 32) part[h0 + k] = pb[k];
      __syncwarp();
    }
    q = qe;
  }
}

__global__ void __launch_bounds__(256) p2v4(long long n, const int* __restrict__ rslot, const int* __restrict__ gidx, const double* __restrict__ part,
    const float* __restrict__ t, const float* __restrict__ dinv, const int* __restrict__ gpos, float c,
    float* __restrict__ r, float* __restrict__ ynext, double* __restrict__ dsum) {
  double d = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int s0 = rslot[i], s1 = rslot[i + 1];
    const float ti = t[i], di = dinv[i];
    const int gp = gpos[i];
    double acc = 0.0;
    int s = s0;
    for (; s + 4 <= s1; s += 4) {
      const int a0 = gidx[s], a1 = gidx[s + 1], a2 = gidx[s + 2], a3 = gidx[s + 3];
      const double v0 = part[a0], v1 = part[a1], v2 = part[a2], v3 = part[a3];
      acc += v0; acc += v1; acc += v2; acc += v3;
    }
    for (; s < s1; s++) acc += part[gidx[s]];
    const float ri = (float)acc + c;
    r[i] = ri;
    d += fabs((double)ri - (double)ti);
    if (gp >= 0) ynext[gp] = ri * di;
  }
  for (int o = 16; o; o >>= 1) d += __shfl_down_sync(0xffffffffu, d, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(dsum, d);
}

extern "C" {
int bs_p1v4(int nt, int L, int C, int grid, const int* cs, const int* sblk, const int* soff, const int* snv, const int* hdr, const void* lcol,
            const float* x, int SB, int ncols, double* part) {
  int smem = (1 << SB) * 4 + (nt / 32) * C * 8;
#define GO(NT_, L_, C_) if (nt == NT_ && L == L_ && C == C_) { cudaFuncSetAttribute(p1v4<NT_, L_, C_>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
    p1v4<NT_, L_, C_><<<grid, NT_, smem>>>(cs, sblk, soff, snv, hdr, (const uint4*)lcol, x, SB, ncols, part); return (int)cudaGetLastError(); }
  GO(1024, 64, 256) GO(1024, 32, 256) GO(512, 64, 512) GO(1024, 64, 128)
#undef GO
  return -1;
}
int bs_p2v4(int grid, long long n, const int* rslot, const int* gidx, const double* part, const float* t, const float* dinv, const int* gpos, float c,
            float* r, float* ynext, double* dsum) {
  p2v4<<<grid, 256>>>(n, rslot, gidx, part, t, dinv, gpos, c, r, ynext, dsum);
  return (int)cudaGetLastError();
}
}

// ---------------- p2 v5: row data + qidx range + runs staged with independent loads
template <int NT, int PMAX>
__global__ void __launch_bounds__(NT) p2v5(int ntiles, int nb, const int4* __restrict__ tinfo, const int* __restrict__ rstart,
    const int* __restrict__ pre, const int* __restrict__ rslot, const unsigned short* __restrict__ qidx, const double* __restrict__ part,
    const float* __restrict__ t, const float* __restrict__ dinv, const int* __restrict__ gpos, float c,
    float* __restrict__ r, float* __restrict__ ynext, double* __restrict__ dsum) {
  __shared__ double spart[PMAX];
  __shared__ unsigned short sq[PMAX];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = NT / 32;
  double d = 0.0;
  for (int tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    const int4 ti = tinfo[tl];     // R0, R1, S0, S1
    const int i = ti.x + threadIdx.x;
    const bool valid = i < ti.y;
    int s0 = 0, s1 = 0, gp = -1; float tv = 0.f, dv = 0.f;
    if (valid) { s0 = rslot[i]; s1 = rslot[i + 1]; tv = t[i]; dv = dinv[i]; gp = gpos[i]; }
    // qidx range
    const int nS = ti.w - ti.z;
    for (int k = threadIdx.x; k < nS; k += NT) sq[k] = qidx[ti.z + k];
    // runs: warp w handles runs w, w + NW, ...
    for (int b0 = warp; b0 < nb; b0 += NW) {
      const int st = rstart[tl * nb + b0];
      const int p0 = pre[tl * (nb + 1) + b0], p1 = pre[tl * (nb + 1) + b0 + 1];
      for (int k = lane; k < p1 - p0; k += 32) spart[p0 + k] = part[st + k];
    }
    __syncthreads();
    if (valid) {
      double acc = 0.0;
      for (int s = s0; s < s1; s++) acc += spart[sq[s - ti.z]];
      const float ri = (float)acc + c;
      r[i] = ri;
      d += fabs((double)ri - (double)tv);
      if (gp >= 0) ynext[gp] = ri * dv;
    }
    __syncthreads();
  }
  for (int o = 16; o; o >>= 1) d += __shfl_down_sync(0xffffffffu, d, o);
  if (lane == 0) atomicAdd(dsum, d);
}
extern "C" int bs_p2v5(int grid, int ntiles, int nb, const void* tinfo, const int* rstart, const int* pre, const int* rslot,
            const unsigned short* qidx, const double* part, const float* t, const float* dinv, const int* gpos, float c,
            float* r, float* ynext, double* dsum) {
  p2v5<512, 3072><<<grid, 512>>>(ntiles, nb, (const int4*)tinfo, rstart, pre, rslot, qidx, part, t, dinv, gpos, c, r, ynext, dsum);
  return (int)cudaGetLastError();
}

// ---------------- v4: variable slices, pieces staged in smem and written coalesced
template <int NT, int L, int C>
__global__ void __launch_bounds__(NT, 1) p1v6(const int* __restrict__ cs, const int* __restrict__ sblk, const int* __restrict__ soff,
    const int* __restrict__ snv, const int* __restrict__ hdr, const uint4* __restrict__ lcol, const float* __restrict__ x, int SB, int ncols,
    double* __restrict__ part, int mode) {
  extern __shared__ __align__(16) unsigned char dyn[];
  float* xs = (float*)dyn;
  const int S = 1 << SB;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* pb = (double*)(dyn + S * 4) + warp * C;
  const int q0 = cs[blockIdx.x], q1 = cs[blockIdx.x + 1];
  int q = q0;
  while (q < q1) {
    const int b = sblk[q];
    int lo = q, hi = q1;
    while (lo < hi) { int mid = (lo + hi) >> 1; if (sblk[mid] <= b) lo = mid + 1; else hi = mid; }
    const int qe = lo;
    __syncthreads();
    const int c0 = b * S;
    const int cn = min(S, ncols - c0);
    for (int k = threadIdx.x * 4; k < cn; k += NT * 4) {
      if (k + 3 < cn) { float4 v = __ldg((const float4*)(x + c0 + k)); *(float4*)(xs + k) = v; }
      else for (int u = k; u < cn; u++) xs[u] = __ldg(x + c0 + u);
    }
    __syncthreads();
    for (int s = q + warp; s < qe; s += NT / 32) {
      const int nv = snv[s];
      const uint4* lp = lcol + (long long)soff[s] + lane;
      uint4 w[L / 8];
#pragma unroll
      for (int v = 0; v < L / 8; v++) if (v < nv) w[v] = __ldcs(lp + v * 32);
      const int h0 = hdr[32 * s];
      const int hl = hdr[32 * s + lane];
      const int hn = hdr[32 * s + 32];
      int pi = hl - h0;
      double acc = 0.0;
#pragma unroll
      for (int v = 0; v < L / 8; v++) {
        if (v < nv) {
          const unsigned ww[4] = {w[v].x, w[v].y, w[v].z, w[v].w};
          float f[8];
#pragma unroll
          for (int h = 0; h < 8; h++) f[h] = (mode & 2) ? (float)((ww[h >> 1] >> ((h & 1) * 16)) & 0x7fffu) : xs[(ww[h >> 1] >> ((h & 1) * 16)) & 0x7fffu];
#pragma unroll
          for (int h = 0; h < 8; h++) {
            acc += (double)f[h];
            if (!(mode & 1) && ((ww[h >> 1] >> ((h & 1) * 16)) & 0x8000u)) { pb[pi++] = acc; acc = 0.0; }
          }
        }
      }
      __syncwarp();
      const int np_ = hn - h0;
      if (mode & 1) { if (lane == 0) part[h0] = acc; } else for (int k = lane; k < np_; k += 32) part[h0 + k] = pb[k];
      __syncwarp();
    }
    q = qe;
  }
}


extern "C" int bs_p1v6(int mode, int grid, const int* cs, const int* sblk, const int* soff, const int* snv, const int* hdr, const void* lcol,
            const float* x, int SB, int ncols, double* part) {
  int smem = (1 << SB) * 4 + 32 * 256 * 8;
  cudaFuncSetAttribute(p1v6<1024, 64, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  p1v6<1024, 64, 256><<<grid, 1024, smem>>>(cs, sblk, soff, snv, hdr, (const uint4*)lcol, x, SB, ncols, part, mode); return (int)cudaGetLastError();
}

// ---------------- v7: lane-per-piece SELL, per-warp cp.async ring over the warp's contiguous lcol stream
__device__ __forceinline__ void cpa16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }

template <int NT, int NS>
__global__ void __launch_bounds__(NT, 1) p1v7(const int* __restrict__ cs, const int* __restrict__ sblk, const int* __restrict__ soff,
    const int* __restrict__ sL, const unsigned short* __restrict__ lcol, const float* __restrict__ x, int S, int ncols, double* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char dyn[];
  constexpr int NW = NT / 32;
  constexpr int CH = 512;                                    // bytes per ring stage (32 lanes x 16 B) = 8 k-rows
  float* xs = (float*)dyn;                                   // [S + 1], xs[S] = 0 sentinel
  unsigned char* ring_all = dyn + ((S + 1) * 4 + 15) / 16 * 16;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* ring = ring_all + warp * NS * CH;
  const int q0 = cs[blockIdx.x], q1 = cs[blockIdx.x + 1];
  int q = q0;
  while (q < q1) {
    const int b = sblk[q];
    int lo = q, hi = q1;
    while (lo < hi) { int mid = (lo + hi) >> 1; if (sblk[mid] <= b) lo = mid + 1; else hi = mid; }
    const int qe = lo;
    __syncthreads();
    const int c0 = b * S;
    const int cn = min(S, ncols - c0);
    for (int k = threadIdx.x; k < cn; k += NT) xs[k] = __ldg(x + c0 + k);
    if (threadIdx.x == 0) xs[S] = 0.f;
    // warp sub-range balanced by entries: split [soff[q], soff[qe]) evenly
    const long long E0 = soff[q], E1 = (qe < q1 || true) ? (long long)soff[qe - 1] + 32LL * sL[qe - 1] : 0;
    const long long ea = E0 + (E1 - E0) * warp / NW, eb = E0 + (E1 - E0) * (warp + 1) / NW;
    // first slice with soff >= ea, first slice with soff >= eb
    int sa, sb;
    { int l = q, h = qe; while (l < h) { int m = (l + h) >> 1; if (soff[m] < ea) l = m + 1; else h = m; } sa = l; }
    { int l = q, h = qe; while (l < h) { int m = (l + h) >> 1; if (soff[m] < eb) l = m + 1; else h = m; } sb = l; }
    if (warp == NW - 1) sb = qe;
    __syncthreads();
    if (sa < sb) {
      const long long B0 = 2LL * soff[sa];                   // stream bytes [B0, B1)
      const long long B1 = 2LL * ((long long)soff[sb - 1] + 32LL * sL[sb - 1]);
      const unsigned char* gs = (const unsigned char*)lcol;
      // prologue: stages 0..NS-1
#pragma unroll
      for (int i = 0; i < NS; i++) {
        const long long gb = B0 + (long long)i * CH + 16 * lane;
        if (gb < B1) cpa16(ring + i * CH + 16 * lane, gs + gb);
        cpa_commit();
      }
      long long rr = 0;                                      // k-rows consumed (64 B each)
      int s = sa;
      int L = sL[s];
      int k = 0;
      double acc = 0.0;
      const long long nrows = (B1 - B0) / 64;
      while (rr < nrows) {
        if ((rr & 7) == 0) {                                  // entering stage (rr / 8)
          cpa_wait<NS - 1>();
          __syncwarp();
        }
        const unsigned short* rowp = (const unsigned short*)(ring + ((rr >> 3) % NS) * CH + (rr & 7) * 64);
        // process up to the end of this stage or slice, 1 k-row per step
        const unsigned short c = rowp[lane];
        acc += (double)xs[c];
        ++rr; ++k;
        if (k == L) {
          part[32LL * s + lane] = acc; acc = 0.0; ++s; k = 0;
          if (s < sb) L = sL[s];
        }
        if ((rr & 7) == 0) {                                  // finished a stage: refill it with stage + NS
          __syncwarp();
          const long long st = (rr >> 3) - 1 + NS;
          const long long gb = B0 + st * CH + 16 * lane;
          if (gb < B1) cpa16(ring + ((st % NS) * CH) + 16 * lane, gs + gb);
          cpa_commit();
        }
      }
      cpa_wait<0>();
    }
    q = qe;
  }
}
extern "C" int bs_p1v7(int grid, const int* cs, const int* sblk, const int* soff, const int* sL, const void* lcol,
            const float* x, int S, int ncols, double* part) {
  const int NS = 4;
  int smem = ((S + 1) * 4 + 15) / 16 * 16 + 32 * NS * 512;
  cudaFuncSetAttribute(p1v7<1024, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  p1v7<1024, NS><<<grid, 1024, smem>>>(cs, sblk, soff, sL, (const unsigned short*)lcol, x, S, ncols, part); return (int)cudaGetLastError();
}

// p2 v7: runs table (start, len) per (tile, block), prefetched per tile
template <int NT, int PMAX>
__global__ void __launch_bounds__(NT) p2v7(int ntiles, int nb, const int4* __restrict__ tinfo, const int2* __restrict__ runs,
    const int* __restrict__ pre, const int* __restrict__ rslot, const unsigned short* __restrict__ qidx, const double* __restrict__ part,
    const float* __restrict__ t, const float* __restrict__ dinv, const int* __restrict__ gpos, float c,
    float* __restrict__ r, float* __restrict__ ynext, double* __restrict__ dsum) {
  __shared__ double spart[PMAX];
  __shared__ unsigned short sq[PMAX];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = NT / 32;
  double d = 0.0;
  for (int tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    const int4 ti = tinfo[tl];
    const int i = ti.x + threadIdx.x;
    const bool valid = i < ti.y;
    int s0 = 0, s1 = 0, gp = -1; float tv = 0.f, dv = 0.f;
    if (valid) { s0 = rslot[i]; s1 = rslot[i + 1]; tv = t[i]; dv = dinv[i]; gp = gpos[i]; }
    const int nS = ti.w - ti.z;
    for (int k = threadIdx.x; k < nS; k += NT) sq[k] = qidx[ti.z + k];
    // runs: lane l of warp w owns run w + NW * (l) ... one run per lane
    for (int b0 = warp * 32 + lane; b0 < nb; b0 += NT) { }
    {
      // each warp copies runs b = warp, warp + NW, ...; run descriptor fetched by all lanes (broadcast)
      for (int b = warp; b < nb; b += NW) {
        const int2 ru = runs[tl * nb + b];
        const int p0 = pre[tl * (nb + 1) + b];
        for (int k = lane; k < ru.y; k += 32) spart[p0 + k] = part[ru.x + k];
      }
    }
    __syncthreads();
    if (valid) {
      double acc = 0.0;
      for (int s = s0; s < s1; s++) acc += spart[sq[s - ti.z]];
      const float ri = (float)acc + c;
      r[i] = ri;
      d += fabs((double)ri - (double)tv);
      if (gp >= 0) ynext[gp] = ri * dv;
    }
    __syncthreads();
  }
  for (int o = 16; o; o >>= 1) d += __shfl_down_sync(0xffffffffu, d, o);
  if (lane == 0) atomicAdd(dsum, d);
}
extern "C" int bs_p2v7(int grid, int ntiles, int nb, const void* tinfo, const void* runs, const int* pre, const int* rslot,
            const unsigned short* qidx, const double* part, const float* t, const float* dinv, const int* gpos, float c,
            float* r, float* ynext, double* dsum) {
  p2v7<512, 3072><<<grid, 512>>>(ntiles, nb, (const int4*)tinfo, (const int2*)runs, pre, rslot, qidx, part, t, dinv, gpos, c, r, ynext, dsum);
  return (int)cudaGetLastError();
}

// ---------------- v8: single pass, rows globally sorted by length (P order), SELL [slice][k][lane], hot cache in smem
template <int NT, int U>
__global__ void __launch_bounds__(NT, 1) sp8(int nslices, const int* __restrict__ soff, const int* __restrict__ sL, const unsigned* __restrict__ idx,
    const float* __restrict__ xg, int hc, const float* __restrict__ tP, const float* __restrict__ dP, const int* __restrict__ gP, float c,
    float* __restrict__ rP, float* __restrict__ ynext, double* __restrict__ dsum, int* __restrict__ ctr) {
  extern __shared__ __align__(16) float s_hot[];
  const int lane = threadIdx.x & 31;
  for (int k = threadIdx.x; k < hc; k += NT) s_hot[k] = xg[k];
  __syncthreads();
  double d = 0.0;
  for (;;) {
    int s = 0;
    if (lane == 0) s = atomicAdd(ctr, 1);
    s = __shfl_sync(0xffffffffu, s, 0);
    if (s >= nslices) break;
    const int L = sL[s];
    const long long off = soff[s];
    const long long i = 32LL * s + lane;
    const float tv = tP[i], dv = dP[i];
    const int gp = gP[i];
    double acc = 0.0;
    const unsigned* ip = idx + off + lane;
    for (int k0 = 0; k0 < L; k0 += U) {
      unsigned cc[U];
#pragma unroll
      for (int u = 0; u < U; u++) cc[u] = (k0 + u < L) ? __ldcs(ip + 32LL * (k0 + u)) : 0u;
      float f[U];
#pragma unroll
      for (int u = 0; u < U; u++) f[u] = cc[u] < (unsigned)hc ? s_hot[cc[u]] : __ldg(xg + cc[u]);
#pragma unroll
      for (int u = 0; u < U; u++) acc += (double)f[u];
    }
    const float ri = (float)acc + c;
    rP[i] = ri;
    d += fabs((double)ri - (double)tv);
    if (gp > 0) ynext[gp] = ri * dv;
  }
  for (int o = 16; o; o >>= 1) d += __shfl_down_sync(0xffffffffu, d, o);
  if (lane == 0) atomicAdd(dsum, d);
}
extern "C" int bs_sp8(int U, int grid, int nslices, const int* soff, const int* sL, const unsigned* idx, const float* xg, int hc,
    const float* tP, const float* dP, const int* gP, float c, float* rP, float* ynext, double* dsum, int* ctr) {
  int smem = hc * 4;
  cudaMemsetAsync(ctr, 0, 4);
#define GO(U_) if (U == U_) { cudaFuncSetAttribute(sp8<1024, U_>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
  sp8<1024, U_><<<grid, 1024, smem>>>(nslices, soff, sL, idx, xg, hc, tP, dP, gP, c, rP, ynext, dsum, ctr); return (int)cudaGetLastError(); }
  GO(4) GO(8) GO(16)
#undef GO
  return -1;
}
