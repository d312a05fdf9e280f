// micro-benchmark: gather throughput from L2 / local smem / cluster DSMEM on the relabelled C4 colidx
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa(unsigned a, unsigned r) { unsigned o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ float ld_dsm(unsigned a) { float v; asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a)); return v; }
__device__ __forceinline__ unsigned cta_rank() { unsigned r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void cluster_sync() { asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }

__device__ __forceinline__ float ld_na(const float* p) { float v; asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p)); return v; }
__device__ __forceinline__ float ld_el(const float* p) { float v; asm volatile("ld.global.nc.L1::evict_last.f32 %0, [%1];" : "=f"(v) : "l"(p)); return v; }
__device__ __forceinline__ float ld_ef(const float* p) { float v; asm volatile("ld.global.nc.L1::evict_first.f32 %0, [%1];" : "=f"(v) : "l"(p)); return v; }
// MODE 0: L2 only; 1: local smem hot [0,hc); 2: cluster DSMEM hot [0,hc) interleaved c % CS
template <int MODE, int CS>
__global__ void __launch_bounds__(1024, 1) gsum(const int* __restrict__ ci, long long nnz, const float* __restrict__ x, int hc, float* out) {
  extern __shared__ float s_hot[];
  unsigned me = 0;
  if (MODE == 1) { for (int k = threadIdx.x; k < hc; k += blockDim.x) s_hot[k] = x[k]; __syncthreads(); }
  if (MODE == 2) {
    me = cta_rank();
    int per = (hc + CS - 1) / CS;
    for (int k = threadIdx.x; k < per; k += blockDim.x) { long long c = (long long)k * CS + me; s_hot[k] = c < hc ? x[c] : 0.f; }
    cluster_sync();
  }
  const unsigned base = smem_u32(s_hot);
  unsigned rb[CS];
  if (MODE == 2) {
#pragma unroll
    for (int r = 0; r < CS; r++) rb[r] = mapa(base, r);
  }
  float acc = 0.f;
  long long nv = nnz >> 2;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (long long)gridDim.x * blockDim.x) {
    int4 c = __ldcs((const int4*)ci + v);
    int cc[4] = {c.x, c.y, c.z, c.w};
    float a[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      if (MODE == 0) a[k] = __ldg(x + cc[k]);
      else if (MODE == 3) a[k] = cc[k] < hc ? ld_el(x + cc[k]) : ld_na(x + cc[k]);
      else if (MODE == 4) a[k] = cc[k] < hc ? ld_el(x + cc[k]) : ld_ef(x + cc[k]);
      else if (MODE == 5) { const float* p = x + cc[k]; a[k] = cc[k] < hc ? ld_el(p) : ld_na(p); }
      else if (MODE == 1) a[k] = cc[k] < hc ? s_hot[cc[k]] : __ldg(x + cc[k]);
      else {
        if (cc[k] < hc) {
          unsigned r = (unsigned)cc[k] % CS, off = (unsigned)cc[k] / CS;
          unsigned rbase = rb[0];
#pragma unroll
          for (int q = 1; q < CS; q++) if (r == q) rbase = rb[q];
          a[k] = ld_dsm(rbase + off * 4);
        } else a[k] = __ldg(x + cc[k]);
      }
    }
    acc += a[0] + a[1] + a[2] + a[3];
  }
  out[(long long)blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (MODE == 2) cluster_sync();
}

// raw smem random gather rate: idx from a hash, no global traffic
__global__ void __launch_bounds__(1024, 1) smem_rand(int hc, int iters, float* out) {
  extern __shared__ float s_hot[];
  for (int k = threadIdx.x; k < hc; k += blockDim.x) s_hot[k] = (float)k;
  __syncthreads();
  unsigned h = threadIdx.x * 2654435761u + blockIdx.x * 97u;
  float acc = 0.f;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 4; k++) { h = h * 1664525u + 1013904223u; acc += s_hot[(h >> 8) % hc]; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
template <int CS>
__global__ void __launch_bounds__(1024, 1) dsm_rand(int per, int iters, float* out) {
  extern __shared__ float s_hot[];
  for (int k = threadIdx.x; k < per; k += blockDim.x) s_hot[k] = (float)k;
  cluster_sync();
  const unsigned base = smem_u32(s_hot);
  unsigned h = threadIdx.x * 2654435761u + blockIdx.x * 97u;
  float acc = 0.f;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 4; k++) { h = h * 1664525u + 1013904223u; unsigned r = (h >> 4) % CS; unsigned off = (h >> 8) % per; acc += ld_dsm(mapa(base, r) + off * 4); }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  cluster_sync();
}

template <class K>
static int launch(K kern, int clusters, int cs, int smem, void** args) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (cs > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(clusters * cs); cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  return (int)cudaLaunchKernelExC(&cfg, (const void*)kern, args);
}
template <class K>
static int max_clusters(K kern, int cs, int smem) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (cs > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs); cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  int n = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (const void*)kern, &cfg);
  if (e != cudaSuccess) return -(int)e;
  return n;
}

extern "C" {
// mode 0/1/2, cs in {1,2,4,8,16}; returns max active clusters (query) or launches
int mg_maxclusters(int mode, int cs, int smem) {
  switch (mode * 100 + cs) {
    case 1: return max_clusters(gsum<0,1>, 1, smem);
    case 101: return max_clusters(gsum<1,1>, 1, smem);
    case 301: return max_clusters(gsum<3,1>, 1, smem);
    case 401: return max_clusters(gsum<4,1>, 1, smem);
    case 202: return max_clusters(gsum<2,2>, 2, smem);
    case 204: return max_clusters(gsum<2,4>, 4, smem);
    case 208: return max_clusters(gsum<2,8>, 8, smem);
    case 216: return max_clusters(gsum<2,16>, 16, smem);
  }
  return -999;
}
int mg_run(int mode, int cs, int clusters, const int* ci, long long nnz, const float* x, int hc, float* out, int smem) {
  void* args[] = {(void*)&ci, (void*)&nnz, (void*)&x, (void*)&hc, (void*)&out};
  switch (mode * 100 + cs) {
    case 1: return launch(gsum<0,1>, clusters, 1, smem, args);
    case 101: return launch(gsum<1,1>, clusters, 1, smem, args);
    case 301: return launch(gsum<3,1>, clusters, 1, smem, args);
    case 401: return launch(gsum<4,1>, clusters, 1, smem, args);
    case 202: return launch(gsum<2,2>, clusters, 2, smem, args);
    case 204: return launch(gsum<2,4>, clusters, 4, smem, args);
    case 208: return launch(gsum<2,8>, clusters, 8, smem, args);
    case 216: return launch(gsum<2,16>, clusters, 16, smem, args);
  }
  return -999;
}
int mg_rand(int cs, int clusters, int per, int iters, float* out) {
  int smem = per * 4;
  void* args[] = {(void*)&per, (void*)&iters, (void*)&out};
  switch (cs) {
    case 1: return launch(smem_rand, clusters, 1, smem, args);
    case 2: return launch(dsm_rand<2>, clusters, 2, smem, args);
    case 4: return launch(dsm_rand<4>, clusters, 4, smem, args);
    case 8: return launch(dsm_rand<8>, clusters, 8, smem, args);
    case 16: return launch(dsm_rand<16>, clusters, 16, smem, args);
  }
  return -999;
}
}

// pipelined gather-only: each thread handles V int4 per iteration; next iteration's indices prefetched
template <int V, bool PRED>
__global__ void __launch_bounds__(1024, 1) gpipe(const int* __restrict__ ci, long long nnz, const float* __restrict__ x, int hc, float* out) {
  extern __shared__ float s_hot[];
  for (int k = threadIdx.x; k < hc; k += blockDim.x) s_hot[k] = x[k];
  __syncthreads();
  float acc = 0.f;
  const long long nv = nnz >> 2;
  const long long stride = (long long)gridDim.x * blockDim.x * V;
  long long v = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * V;
  int4 c[V];
#pragma unroll
  for (int j = 0; j < V; j++) c[j] = (v + j < nv) ? __ldcs((const int4*)ci + v + j) : make_int4(0, 0, 0, 0);
  for (; v < nv; v += stride) {
    int4 cn[V];
#pragma unroll
    for (int j = 0; j < V; j++) cn[j] = (v + stride + j < nv) ? __ldcs((const int4*)ci + v + stride + j) : make_int4(0, 0, 0, 0);
    float a[4 * V];
#pragma unroll
    for (int j = 0; j < V; j++) {
      const int cc[4] = {c[j].x, c[j].y, c[j].z, c[j].w};
#pragma unroll
      for (int k = 0; k < 4; k++) {
        if (PRED) {
          float r;
          asm volatile("{ .reg .pred p; setp.lt.s32 p, %1, %2; @p ld.shared.f32 %0, [%3]; @!p ld.global.nc.f32 %0, [%4]; }"
                       : "=f"(r) : "r"(cc[k]), "r"(hc), "r"((unsigned)__cvta_generic_to_shared(s_hot + (cc[k] < hc ? cc[k] : 0))), "l"(x + cc[k]));
          a[4 * j + k] = r;
        } else a[4 * j + k] = cc[k] < hc ? s_hot[cc[k]] : __ldg(x + cc[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < 4 * V; k++) acc += a[k];
#pragma unroll
    for (int j = 0; j < V; j++) c[j] = cn[j];
  }
  out[(long long)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
extern "C" int mg_pipe(int V, int pred, const int* ci, long long nnz, const float* x, int hc, float* out) {
  int smem = hc * 4;
#define GO(V_, P_) if (V == V_ && pred == P_) { cudaFuncSetAttribute(gpipe<V_, P_>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
   gpipe<V_, P_><<<148, 1024, smem>>>(ci, nnz, x, hc, out); return (int)cudaGetLastError(); }
  GO(1, false) GO(2, false) GO(4, false) GO(1, true) GO(2, true) GO(4, true)
#undef GO
  return -1;
}

// texture-path gathers: cold columns through tex1Dfetch (TEX pipe) vs ld.global.nc (LSU pipe)
template <int MODE>
__global__ void __launch_bounds__(1024, 1) gtex(const int* __restrict__ ci, long long nnz, const float* __restrict__ x, cudaTextureObject_t tx, int hc, float* out) {
  extern __shared__ float s_hot[];
  for (int k = threadIdx.x; k < hc; k += blockDim.x) s_hot[k] = x[k];
  __syncthreads();
  float acc = 0.f;
  const long long nv = nnz >> 2;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (long long)gridDim.x * blockDim.x) {
    const int4 c = __ldcs((const int4*)ci + v);
    const int cc[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
    for (int k = 0; k < 4; k++) {
      float a;
      if (cc[k] < hc) a = s_hot[cc[k]];
      else if (MODE == 0) a = __ldg(x + cc[k]);
      else if (MODE == 1) a = tex1Dfetch<float>(tx, cc[k]);
      else a = (k & 1) ? tex1Dfetch<float>(tx, cc[k]) : __ldg(x + cc[k]);
      acc += a;
    }
  }
  out[(long long)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
extern "C" int mg_tex(int mode, const int* ci, long long nnz, const float* x, long long n, int hc, float* out) {
  cudaResourceDesc rd = {}; rd.resType = cudaResourceTypeLinear; rd.res.linear.devPtr = (void*)x;
  rd.res.linear.desc = cudaCreateChannelDesc<float>(); rd.res.linear.sizeInBytes = n * 4;
  cudaTextureDesc td = {}; td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tx = 0; cudaCreateTextureObject(&tx, &rd, &td, nullptr);
  int smem = hc * 4;
#define GO(M_) if (mode == M_) { cudaFuncSetAttribute(gtex<M_>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); gtex<M_><<<148, 1024, smem>>>(ci, nnz, x, tx, hc, out); }
  GO(0) GO(1) GO(2)
#undef GO
  int e = (int)cudaGetLastError();
  cudaDeviceSynchronize(); cudaDestroyTextureObject(tx);
  return e;
}
