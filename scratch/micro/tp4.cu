// micro: two-phase v4.  Phase 1: column blocks in shared memory, adaptive slices of 32 lane chunks
// (u16 local column | pair-end flag), lane-local split + one segmented scan per slice, pieces staged
// in shared memory and flushed to their tile-major position pos2[].  Phase 2: per tile the pieces are
// one contiguous range (staged with qidx), per-row sums, epilogue.
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ void cpa4(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"((unsigned)__cvta_generic_to_shared(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

constexpr int PMAXS = 384;

template <int NT>
__global__ void __launch_bounds__(NT, 1) p1(const int* __restrict__ cta, const int* __restrict__ sl_blk, const int* __restrict__ sl_off,
    const int* __restrict__ sl_Ls, const int* __restrict__ spbase, const uint4* __restrict__ lcol, const int* __restrict__ pos2,
    const float* __restrict__ X, int S, int ncols, double* __restrict__ part, long long* dbg) {
  constexpr int NW = NT / 32;
  const long long t0_ = clock64(); int nblk_ = 0;
  extern __shared__ __align__(16) unsigned char dyn[];
  float* xs = (float*)dyn;
  __shared__ int s_ctr;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* pbuf = (double*)(dyn + S * 4) + warp * PMAXS;
  int* pidx = (int*)(dyn + S * 4 + NW * PMAXS * 8) + warp * PMAXS;
  int q = cta[blockIdx.x];
  const int q1 = cta[blockIdx.x + 1];
  while (q < q1) {
    ++nblk_;
    const int blk = sl_blk[q];
    int lo = q, hi = q1;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (sl_blk[mid] <= blk) lo = mid + 1; else hi = mid; }
    const int qe = lo;
    __syncthreads();
    if (threadIdx.x == 0) s_ctr = q;
    {
      const long long c0 = (long long)blk * S;
      const int cn = (int)min((long long)S, ncols - c0);
      const float4* src = (const float4*)(X + c0);
      const int nv = cn >> 2;
      for (int v = threadIdx.x; v < nv; v += NT) ((float4*)xs)[v] = __ldg(src + v);
      for (int j = (nv << 2) + threadIdx.x; j < cn; j += NT) xs[j] = X[c0 + j];
    }
    __syncthreads();
    int sn = 0;
    if (lane == 0) sn = atomicAdd(&s_ctr, 1);
    sn = __shfl_sync(0xffffffffu, sn, 0);
    int offn = 0, Lsn = 0, pbn = 0, pen = 0;
    if (sn < qe) { offn = sl_off[sn]; Lsn = sl_Ls[sn]; pbn = spbase[sn]; pen = spbase[sn + 1]; }
    for (;;) {
      const int s = sn;
      if (s >= qe) break;
      const int off = offn, Ls = Lsn, pb = pbn, npc = pen - pbn;
      // claim + prefetch the next slice's header
      if (lane == 0) sn = atomicAdd(&s_ctr, 1);
      sn = __shfl_sync(0xffffffffu, sn, 0);
      if (sn < qe) { offn = sl_off[sn]; Lsn = sl_Ls[sn]; pbn = spbase[sn]; pen = spbase[sn + 1]; }
      // piece destinations (async) and the slice's entries
      for (int k = lane; k < npc; k += 32) cpa4(pidx + k, pos2 + pb + k);
      cpa_commit();
      const uint4* lp = lcol + (off >> 3) + lane;
      uint4 w[4];
#pragma unroll
      for (int v = 0; v < 4; v++) w[v] = (v < (Ls >> 3)) ? __ldcs(lp + 32 * v) : make_uint4(0, 0, 0, 0);
      int cnt = 0;
#pragma unroll
      for (int v = 0; v < 4; v++) cnt += __popc((w[v].x | (w[v].y >> 1) & 0) & 0) ;   // placeholder (replaced below)
      // flags are bit 15 of each u16: count them
      cnt = 0;
#pragma unroll
      for (int v = 0; v < 4; v++) cnt += __popc(w[v].x & 0x80008000u) + __popc(w[v].y & 0x80008000u) + __popc(w[v].z & 0x80008000u) + __popc(w[v].w & 0x80008000u);
      int incl = cnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) { const int y = __shfl_up_sync(0xffffffffu, incl, d); if (lane >= d) incl += y; }
      const int o = incl - cnt;                    // rank of my first piece in the slice
      // lane-local: head (up to and incl. the first flag), inner pieces, tail
      double h = 0.0, cur = 0.0;
      bool seen = false;
      int m = 0;
#pragma unroll
      for (int v = 0; v < 4; v++) {
        if (v < (Ls >> 3)) {
          const unsigned ww[4] = {w[v].x, w[v].y, w[v].z, w[v].w};
          float f[8];
#pragma unroll
          for (int hh = 0; hh < 8; hh++) f[hh] = xs[(ww[hh >> 1] >> ((hh & 1) * 16)) & 0x3fffu];
#pragma unroll
          for (int hh = 0; hh < 8; hh++) {
            const bool fl = (ww[hh >> 1] >> ((hh & 1) * 16 + 15)) & 1u;
            cur += (double)f[hh];
            if (fl) {
              if (!seen) { h = cur; seen = true; } else pbuf[o + m] = cur;
              ++m; cur = 0.0;
            }
          }
        }
      }
      // segmented scan: lanes with a flag start a new segment with their tail
      double Sv = cur;                              // tail (or the whole lane if no flag)
      bool F = seen;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double Sy = __shfl_up_sync(0xffffffffu, Sv, d);
        const bool Fy = __shfl_up_sync(0xffffffffu, F, d);
        if (lane >= d && !F) { Sv += Sy; F = Fy; }
      }
      double A = __shfl_up_sync(0xffffffffu, Sv, 1);
      if (lane == 0) A = 0.0;
      if (seen) pbuf[o] = A + h;
      cpa_wait_all();
      __syncwarp();
      for (int k = lane; k < npc; k += 32) part[pidx[k]] = pbuf[k];
      __syncwarp();
    }
    q = qe;
  }
  __syncthreads();
  if (threadIdx.x == 0 && dbg) { dbg[4 * blockIdx.x] = clock64() - t0_; dbg[4 * blockIdx.x + 1] = nblk_; dbg[4 * blockIdx.x + 2] = q1 - cta[blockIdx.x]; dbg[4 * blockIdx.x + 3] = sl_blk[cta[blockIdx.x]]; }
}

template <int NT, int PM2>
__global__ void __launch_bounds__(NT) p2(int ntiles, const int4* __restrict__ tinfo, const int* __restrict__ rslot,
    const unsigned short* __restrict__ qidx, const double* __restrict__ part, const float* __restrict__ t, const float* __restrict__ dinv,
    const int* __restrict__ gpos, float c, float* __restrict__ r, float* __restrict__ ynext, double* __restrict__ dsum) {
  constexpr int NW = NT / 32;
  __shared__ double sv[NW][PM2];
  __shared__ unsigned short sq[NW][PM2];
  __shared__ int s_ctr;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_ctr = 0;
  __syncthreads();
  double d = 0.0;
  int ln = 0;
  if (lane == 0) ln = atomicAdd(&s_ctr, 1);
  ln = __shfl_sync(0xffffffffu, ln, 0);
  int tn = blockIdx.x + ln * gridDim.x;
  int4 hn = tn < ntiles ? tinfo[tn] : make_int4(0, 0, 0, 0);
  for (;;) {
    const int tt = tn;
    if (tt >= ntiles) break;
    const int4 h = hn;
    if (lane == 0) ln = atomicAdd(&s_ctr, 1);
    ln = __shfl_sync(0xffffffffu, ln, 0);
    tn = blockIdx.x + ln * gridDim.x;
    if (tn < ntiles) hn = tinfo[tn];
    const int np = h.w - h.z;
    for (int k = lane; k < np; k += 32) { sv[warp][k] = part[h.z + k]; sq[warp][k] = qidx[h.z + k]; }
    int s0[4], s1[4]; float tv[4], dv[4]; int gp[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int i = h.x + lane + 32 * q;
      const bool ok = i < h.y;
      s0[q] = ok ? rslot[i] : 0; s1[q] = ok ? rslot[i + 1] : 0;
      tv[q] = ok ? t[i] : 0.f; dv[q] = ok ? dinv[i] : 0.f; gp[q] = ok ? gpos[i] : -1;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int i = h.x + lane + 32 * q;
      if (i < h.y) {
        double acc = 0.0;
        for (int s = s0[q]; s < s1[q]; s++) acc += sv[warp][sq[warp][s - h.z]];
        const float ri = (float)acc + c;
        r[i] = ri; d += fabs((double)ri - (double)tv[q]);
        if (gp[q] >= 0) ynext[gp[q]] = ri * dv[q];
      }
    }
    __syncwarp();
  }
  for (int o = 16; o; o >>= 1) d += __shfl_down_sync(0xffffffffu, d, o);
  if (lane == 0) atomicAdd(dsum, d);
}

extern "C" int tp4_p1(int nt, const int* cta, const int* sl_blk, const int* sl_off, const int* sl_Ls, const int* spbase, const void* lcol,
                      const int* pos2, const float* X, int S, int ncols, double* part, long long* dbg) {
  const int smem = S * 4 + (nt / 32) * PMAXS * 12;
#define GO(NT_) if (nt == NT_) { cudaFuncSetAttribute(p1<NT_>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
  p1<NT_><<<148, NT_, smem>>>(cta, sl_blk, sl_off, sl_Ls, spbase, (const uint4*)lcol, pos2, X, S, ncols, part, dbg); return (int)cudaGetLastError(); }
  GO(768) GO(512) GO(1024)
#undef GO
  return -1;
}
extern "C" int tp4_p2(int grid, int ntiles, const void* tinfo, const int* rslot, const unsigned short* qidx, const double* part,
                      const float* t, const float* dinv, const int* gpos, float c, float* r, float* ynext, double* dsum) {
  p2<256, 512><<<grid, 256>>>(ntiles, (const int4*)tinfo, rslot, qidx, part, t, dinv, gpos, c, r, ynext, dsum);
  return (int)cudaGetLastError();
}
