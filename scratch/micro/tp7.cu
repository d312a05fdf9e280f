// Micro-benchmark: two-phase SpMV v7 (flagged u16 stream, fixed 2048-entry warp ranges).
// Phase 1: per column block (S columns of x in shared memory), stream of u16 entries
//   (bit 15 = last entry of a piece; low 15 bits = block-local column, 0x7fff = pad -> xs[pad] = 0).
//   Every 2048-entry warp range ends with a flag, so ranges are independent; the k-th flag of the
//   stream closes piece k: P[k] = sum of the piece's gathered values.
// Phase 2: row i = sum of P over its pieces (rowpieces[rp2[i] .. rp2[i+1])) -> y[i].
#include <cuda_runtime.h>
#include <stdint.h>

#define WR 2048

template <typename ACC, int NT>
__global__ void __launch_bounds__(NT, 1) k_p1(const uint4 *__restrict__ E, const float *__restrict__ X,
                                               const int *__restrict__ wblk, const int *__restrict__ cta,
                                               const long long *__restrict__ pbase, ACC *__restrict__ P, int S,
                                               long long ncols) {
    extern __shared__ __align__(16) float xs[];
    __shared__ int s_ctr;
    const int lane = threadIdx.x & 31;
    const int q1 = cta[blockIdx.x + 1];
    int q = cta[blockIdx.x];
    while (q < q1) {
        const int blk = wblk[q];
        int qe = q + 1;
        while (qe < q1 && wblk[qe] == blk) qe++;
        __syncthreads();
        if (threadIdx.x == 0) s_ctr = q;
        {
            const long long c0 = (long long)blk * S;
            const int cn = (int)((ncols - c0) < S ? (ncols - c0) : S);
            // 16-byte loads, 4 in flight per thread (c0 * 4 is 16-byte aligned when S % 4 == 0; else scalar)
            const bool al = ((c0 & 3) == 0);
            const int nv = al ? (cn >> 2) : 0;
            const uint4 *s4 = (const uint4 *)(X + c0);
            for (int v = threadIdx.x; v < nv; v += 4 * NT) {
                uint4 r[4];
#pragma unroll
                for (int k = 0; k < 4; k++) if (v + k * NT < nv) r[k] = __ldg(s4 + v + k * NT);
#pragma unroll
                for (int k = 0; k < 4; k++) if (v + k * NT < nv) ((uint4 *)xs)[v + k * NT] = r[k];
            }
            for (int j = 4 * nv + threadIdx.x; j < 32768; j += NT) xs[j] = (j < cn) ? __ldg(X + c0 + j) : 0.0f;
        }
        __syncthreads();
        for (;;) {
            int t = 0;
            if (lane == 0) t = atomicAdd(&s_ctr, 1);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t >= qe) break;
            const uint4 *src = E + (long long)t * (WR / 8) + lane;
            uint4 w[8];
#pragma unroll
            for (int s = 0; s < 8; s++) w[s] = __ldcs(src + 32 * s);
            long long ob = pbase[t];
            ACC carry = 0;
#pragma unroll
            for (int s = 0; s < 8; s++) {
                const unsigned u[4] = {w[s].x, w[s].y, w[s].z, w[s].w};
                const int nf = __popc(u[0] & 0x80008000u) + __popc(u[1] & 0x80008000u) + __popc(u[2] & 0x80008000u) +
                               __popc(u[3] & 0x80008000u);
                // exclusive prefix of flag counts over lanes
                int inc = nf;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, inc, d);
                    if (lane >= d) inc += y;
                }
                const int tot = __shfl_sync(0xffffffffu, inc, 31);
                long long o = ob + inc - nf;      // ordinal of this lane's first flag
                ACC a = 0, head = 0;
                bool hf = false;
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    const unsigned e = (u[j >> 1] >> (16 * (j & 1))) & 0xffffu;
                    a += (ACC)xs[e & 0x7fffu];
                    if (e & 0x8000u) {
                        if (hf) { P[o] = a; o++; } else { head = a; hf = true; o++; }
                        a = 0;
                    }
                }
                // carry-in for the lane's first piece: segmented scan of tails
                ACC S_ = a;
                if (lane == 0 && !hf) S_ += carry;
                const unsigned H = __ballot_sync(0xffffffffu, hf) | 1u;
                const int seg = 31 - __clz(H & ((2u << lane) - 1u));
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const ACC y = __shfl_up_sync(0xffffffffu, S_, d);
                    if (lane - d >= seg) S_ += y;
                }
                ACC cin = __shfl_up_sync(0xffffffffu, S_, 1);
                if (lane == 0) cin = carry;
                if (hf) P[ob + inc - nf] = cin + head;
                carry = __shfl_sync(0xffffffffu, S_, 31);
                ob += tot;
            }
        }
        q = qe;
    }
}

template <typename ACC>
__global__ void k_p2(long long n, const long long *__restrict__ rp2, const int *__restrict__ rpc,
                     const ACC *__restrict__ P, float *__restrict__ y) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long s0 = rp2[i], s1 = rp2[i + 1];
        double acc = 0;
        for (long long s = s0; s < s1; s++) acc += (double)P[rpc[s]];
        y[i] = (float)acc;
    }
}

extern "C" int tp7_p1(int reps, int accd, int nt, const void *E, const void *X, const void *wblk, const void *cta, int ncta,
                      const void *pbase, void *P, int S, long long ncols) {
    const int smem = 32768 * 4;
    static bool init = false;
    if (!init) {
        init = true;
        cudaFuncSetAttribute(k_p1<double, 768>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_p1<double, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_p1<float, 768>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_p1<float, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    }
    for (int r = 0; r < reps; r++)
    if (accd) {
        if (nt == 768) {
            // cudaFuncSetAttribute(k_p1<double, 768>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            k_p1<double, 768><<<ncta, 768, smem>>>((const uint4 *)E, (const float *)X, (const int *)wblk, (const int *)cta,
                                                    (const long long *)pbase, (double *)P, S, ncols);
        } else {
            // cudaFuncSetAttribute(k_p1<double, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            k_p1<double, 1024><<<ncta, 1024, smem>>>((const uint4 *)E, (const float *)X, (const int *)wblk, (const int *)cta,
                                                      (const long long *)pbase, (double *)P, S, ncols);
        }
    } else {
        if (nt == 768) {
            // cudaFuncSetAttribute(k_p1<float, 768>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            k_p1<float, 768><<<ncta, 768, smem>>>((const uint4 *)E, (const float *)X, (const int *)wblk, (const int *)cta,
                                                   (const long long *)pbase, (float *)P, S, ncols);
        } else {
            // cudaFuncSetAttribute(k_p1<float, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            k_p1<float, 1024><<<ncta, 1024, smem>>>((const uint4 *)E, (const float *)X, (const int *)wblk, (const int *)cta,
                                                     (const long long *)pbase, (float *)P, S, ncols);
        }
    }
    return (int)cudaGetLastError();
}

extern "C" int tp7_p2(int accd, long long n, const void *rp2, const void *rpc, const void *P, void *y) {
    if (accd)
        k_p2<double><<<148 * 8, 256>>>(n, (const long long *)rp2, (const int *)rpc, (const double *)P, (float *)y);
    else
        k_p2<float><<<148 * 8, 256>>>(n, (const long long *)rp2, (const int *)rpc, (const float *)P, (float *)y);
    return (int)cudaGetLastError();
}

// ---- v3: lane-contiguous runs of 64 entries (forced flag at each run end), no cross-lane work.
// Physical layout per 2048-entry range: uint4 k of lane l at (range * 256 + k * 32 + l).
template <typename ACC, int NT>
__global__ void __launch_bounds__(NT, 1) k_p1c(const uint4 *__restrict__ E, const float *__restrict__ X,
                                                const int *__restrict__ wblk, const int *__restrict__ cta,
                                                const int *__restrict__ lbase, float *__restrict__ P, int S,
                                                long long ncols, unsigned long long *tim) {
    extern __shared__ __align__(16) float xs[];
    __shared__ int s_ctr;
    const int lane = threadIdx.x & 31;
    unsigned long long t_start, t_slice = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    const int q1 = cta[blockIdx.x + 1];
    int q = cta[blockIdx.x];
    const unsigned sb = (unsigned)__cvta_generic_to_shared(xs);
    while (q < q1) {
        const int blk = wblk[q];
        int qe = q + 1;
        while (qe < q1 && wblk[qe] == blk) qe++;
        __syncthreads();
        if (threadIdx.x == 0) s_ctr = q;
        {
            const long long c0 = (long long)blk * S;
            const int cn = (int)((ncols - c0) < S ? (ncols - c0) : S);
            const bool al = ((c0 & 3) == 0);
            const int nv = al ? (cn >> 2) : 0;
            const uint4 *s4 = (const uint4 *)(X + c0);
            for (int v = threadIdx.x; v < nv; v += 4 * NT) {
                uint4 r[4];
#pragma unroll
                for (int k = 0; k < 4; k++) if (v + k * NT < nv) r[k] = __ldg(s4 + v + k * NT);
#pragma unroll
                for (int k = 0; k < 4; k++) if (v + k * NT < nv) ((uint4 *)xs)[v + k * NT] = r[k];
            }
            for (int j = 4 * nv + threadIdx.x; j < 32768; j += NT) xs[j] = (j < cn) ? __ldg(X + c0 + j) : 0.0f;
        }
        __syncthreads();
        if (tim && threadIdx.x == 0) { unsigned long long t1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1)); t_slice += t1 - t_start; }
        for (;;) {
            int t = 0;
            if (lane == 0) t = atomicAdd(&s_ctr, 1);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t >= qe) break;
            const uint4 *src = E + (long long)t * 256 + lane;
            uint4 w[8];
#pragma unroll
            for (int k = 0; k < 8; k++) w[k] = __ldcs(src + 32 * k);
            int o = __ldcs(lbase + (long long)t * 32 + lane);
            ACC r = 0;
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const unsigned u[4] = {w[k].x, w[k].y, w[k].z, w[k].w};
#pragma unroll
                for (int h = 0; h < 8; h++) {
                    const unsigned a = (h & 1) ? ((u[h >> 1] >> 14) & 0x1fffcu) : ((u[h >> 1] << 2) & 0x1fffcu);
                    float v;
                    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(sb + a));
                    r += (ACC)v;
                    const bool f = (u[h >> 1] >> (16 * (h & 1) + 15)) & 1u;
                    if (f) P[o] = (float)r;
                    o += f ? 1 : 0;
                    r = f ? (ACC)0 : r;
                }
            }
        }
        q = qe;
    }
    if (tim) {
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t2; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
            unsigned smid; asm("mov.u32 %0, %%smid;" : "=r"(smid));
            tim[4 * blockIdx.x] = t_start; tim[4 * blockIdx.x + 1] = t2; tim[4 * blockIdx.x + 2] = t_slice; tim[4 * blockIdx.x + 3] = smid;
        }
    }
}

extern "C" int tp7_p1c(int reps, int nt, const void *E, const void *X, const void *wblk, const void *cta, int ncta,
                       const void *lbase, void *P, int S, long long ncols, void *tim) {
    const int smem = 32768 * 4;
    static bool init = false;
    if (!init) {
        init = true;
        cudaFuncSetAttribute(k_p1c<float, 768>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_p1c<float, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_p1c<float, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    }
    for (int r = 0; r < reps; r++) {
        if (nt == 768)
            k_p1c<float, 768><<<ncta, 768, smem>>>((const uint4 *)E, (const float *)X, (const int *)wblk, (const int *)cta,
                                                    (const int *)lbase, (float *)P, S, ncols, (unsigned long long *)tim);
        else if (nt == 512)
            k_p1c<float, 512><<<ncta, 512, smem>>>((const uint4 *)E, (const float *)X, (const int *)wblk, (const int *)cta,
                                                    (const int *)lbase, (float *)P, S, ncols, (unsigned long long *)tim);
        else
            k_p1c<float, 1024><<<ncta, 1024, smem>>>((const uint4 *)E, (const float *)X, (const int *)wblk, (const int *)cta,
                                                      (const int *)lbase, (float *)P, S, ncols, (unsigned long long *)tim);
    }
    return (int)cudaGetLastError();
}
