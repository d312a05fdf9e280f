import sys, os; sys.path.insert(0,'.')
import torch, numpy as np
from torch.utils.cpp_extension import load_inline
from paper_2509_14211_b200 import nbg
torch.cuda.set_device(0)
src = r'''
#include <torch/extension.h>
template <int MODE>
__global__ void __launch_bounds__(1024, 1) gsum(const int* __restrict__ ci, long long nnz, const float* __restrict__ x, int hc, float* out) {
  extern __shared__ float s_hot[];
  if (MODE == 1) { for (int k = threadIdx.x; k < hc; k += blockDim.x) s_hot[k] = x[k]; __syncthreads(); }
  float acc = 0.f;
  long long nv = nnz >> 2;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (long long)gridDim.x * blockDim.x) {
    int4 c = __ldcs((const int4*)ci + v);
    float a0, a1, a2, a3;
    if (MODE == 1) {
      a0 = c.x < hc ? s_hot[c.x] : __ldg(x + c.x); a1 = c.y < hc ? s_hot[c.y] : __ldg(x + c.y);
      a2 = c.z < hc ? s_hot[c.z] : __ldg(x + c.z); a3 = c.w < hc ? s_hot[c.w] : __ldg(x + c.w);
    } else if (MODE == 2) {
      const float* p0 = c.x < hc ? s_hot + c.x : x + c.x; const float* p1 = c.y < hc ? s_hot + c.y : x + c.y;
      const float* p2 = c.z < hc ? s_hot + c.z : x + c.z; const float* p3 = c.w < hc ? s_hot + c.w : x + c.w;
      a0 = *p0; a1 = *p1; a2 = *p2; a3 = *p3;
    } else { a0 = __ldg(x + c.x); a1 = __ldg(x + c.y); a2 = __ldg(x + c.z); a3 = __ldg(x + c.w); }
    acc += a0 + a1 + a2 + a3;
  }
  out[(long long)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
torch::Tensor run(torch::Tensor ci, torch::Tensor x, int hc, int mode, int blocks, int threads) {
  auto out = torch::empty({blocks * threads}, x.options());
  int smem = (mode == 1 || mode == 2) ? hc * 4 : 0;
  if (mode == 1) { cudaFuncSetAttribute(gsum<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    gsum<1><<<blocks, threads, smem>>>(ci.data_ptr<int>(), ci.numel(), x.data_ptr<float>(), hc, out.data_ptr<float>()); }
  else if (mode == 2) { cudaFuncSetAttribute(gsum<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    gsum<2><<<blocks, threads, smem>>>(ci.data_ptr<int>(), ci.numel(), x.data_ptr<float>(), hc, out.data_ptr<float>()); }
  else gsum<0><<<blocks, threads, 0>>>(ci.data_ptr<int>(), ci.numel(), x.data_ptr<float>(), hc, out.data_ptr<float>());
  return out;
}
'''
m = load_inline("gmicro", cpp_sources="torch::Tensor run(torch::Tensor ci, torch::Tensor x, int hc, int mode, int blocks, int threads);",
                cuda_sources=src, functions=["run"], extra_cuda_cflags=["-O3", "-gencode", "arch=compute_100a,code=sm_100a"], verbose=False)
c = nbg.nbg_init(nbg.NONBLOCKING, 0)
A, deg = nbg.nbg_matrix_from_generator(c, nbg.GRAPH_RMAT, 22, 16, 1)
rp, ci = nbg.nbg_matrix_export_csr(c, A)
d = nbg.nbg_vector_export_dense(c, deg)
n = rp.shape[0]-1
ci_t = torch.from_numpy(ci).cuda()
order = np.argsort(-d.astype(np.int64), kind='stable'); perm = np.empty(n, np.int64); perm[order] = np.arange(n)
cig = torch.from_numpy(perm[ci].astype(np.int32)).cuda()
x = torch.rand(n, device='cuda')
def t(ci_, hc, mode, blocks, threads, reps=10):
    for _ in range(2): m.run(ci_, x, hc, mode, blocks, threads)
    torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): m.run(ci_, x, hc, mode, blocks, threads)
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)/reps*1000
print("natural, no cache, 148x1024:", t(ci_t, 0, 0, 148, 1024))
print("natural, no cache, 296x1024 (2/SM):", t(ci_t, 0, 0, 296, 1024))
print("natural, no cache, 148*8 x 256:", t(ci_t, 0, 0, 148*8, 256))
print("relabel, no cache, 148*8 x256:", t(cig, 0, 0, 148*8, 256))
print("relabel, no cache, 296x1024:", t(cig, 0, 0, 296, 1024))
for hc in (16384, 32768, 51200):
    print("relabel, hot", hc, "branch:", t(cig, hc, 1, 148, 1024), " generic:", t(cig, hc, 2, 148, 1024))
print("colidx stream only (hc=n via generic? no) -> mode1 hc=0:", t(cig, 0, 1, 148, 1024))
