// Micro-benchmark tp11: two-phase SpMV with the dense and the cold part running CONCURRENTLY on
// every SM (different warps of one CTA), pieces written in ordinal order (no slot scatter), and a
// combine kernel per 32-row tile driven by per-tile segment offsets.
//   K_A: warps [0, WD): dense ranges (1024 u16 entries, lane runs of 32, block slice of x in shared
//        memory loaded by TMA, named barrier 1 among the dense warps for slice switches);
//        warps [WD, 32): cold ranges (512 int32 gather indices, lane runs of 16, x from L2).
//        Every lane run ends with a flag; the k-th flag of the stream closes piece k.  Pieces are
//        staged per warp in shared memory and written coalesced at their ordinals.
//   K_B: warp per tile of 32 rows; lane b < NSEG walks segment b's pieces of the tile (ordinals
//        off[b][t] .. off[b][t+1], row-in-tile in prow8) into tab[row][b]; lane j then sums its row
//        over the segments in order -> y (deterministic).
#include <cuda_runtime.h>
#include <stdint.h>

#define STG_CAP 384

__device__ __forceinline__ void mbar_init(unsigned a, int cnt) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(cnt)); }
__device__ __forceinline__ void mbar_expect(unsigned a, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void *src, unsigned bytes, unsigned mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src),
                 "r"(bytes), "r"(mbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned a, unsigned ph) {
    asm volatile("{ .reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W_%=; }" ::"r"(a), "r"(ph)
                 : "memory");
}
__device__ __forceinline__ void bar_dense(int nthreads) { asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory"); }

template <bool DENSE>
__device__ __forceinline__ void run4(const uint4 (&w)[4], unsigned sb, const float *__restrict__ X, int o, float *P, bool staged,
                                     unsigned sdst) {
    float r = 0.f;
    if (DENSE) {
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const unsigned u[4] = {w[k].x, w[k].y, w[k].z, w[k].w};
#pragma unroll
            for (int h = 0; h < 8; h++) {
                const unsigned a = (h & 1) ? ((u[h >> 1] >> 14) & 0x1fffcu) : ((u[h >> 1] << 2) & 0x1fffcu);
                float v;
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(sb + a));
                r += v;
                const bool f = (u[h >> 1] >> (16 * (h & 1) + 15)) & 1u;
                if (f) {
                    if (staged) asm volatile("st.shared.f32 [%0], %1;" ::"r"(sdst + 4u * (unsigned)o), "f"(r) : "memory");
                    else P[o] = r;
                }
                o += f ? 1 : 0;
                r = f ? 0.f : r;
            }
        }
    } else {
        float g[16];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const unsigned u[4] = {w[k].x, w[k].y, w[k].z, w[k].w};
#pragma unroll
            for (int h = 0; h < 4; h++) g[4 * k + h] = __ldg(X + (u[h] & 0x7fffffffu));
        }
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const unsigned u[4] = {w[k].x, w[k].y, w[k].z, w[k].w};
#pragma unroll
            for (int h = 0; h < 4; h++) {
                r += g[4 * k + h];
                const bool f = u[h] >> 31;
                if (f) {
                    if (staged) asm volatile("st.shared.f32 [%0], %1;" ::"r"(sdst + 4u * (unsigned)o), "f"(r) : "memory");
                    else P[o] = r;
                }
                o += f ? 1 : 0;
                r = f ? 0.f : r;
            }
        }
    }
}

template <int WD>
__global__ void __launch_bounds__(1024, 1) k_a(const uint4 *__restrict__ E, const uint4 *__restrict__ C, const float *__restrict__ X,
                                                const int *__restrict__ rblk, const int *__restrict__ bnext, const int *__restrict__ cta,
                                                const int *__restrict__ ccta, const int *__restrict__ lbase, float *__restrict__ P, int S,
                                                long long ncols, int ndr) {
    extern __shared__ __align__(128) unsigned char dyn[];
    float *xs = (float *)dyn;
    float *stg = (float *)(dyn + 32768 * 4);
    __shared__ __align__(8) unsigned long long mbar;
    __shared__ int s_ctr, s_cctr;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(xs);
    const unsigned sstg = (unsigned)__cvta_generic_to_shared(stg + warp * STG_CAP);
    const unsigned smb = (unsigned)__cvta_generic_to_shared(&mbar);
    if (threadIdx.x == 0) {
        mbar_init(smb, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        xs[32767] = 0.f;
        s_cctr = ndr + ccta[blockIdx.x];
    }
    __syncthreads();
    if (warp < WD) {
        // ---- dense warps: segments of one column block each, slice switch under barrier 1
        unsigned phase = 0;
        const int q1 = cta[blockIdx.x + 1];
        int q = cta[blockIdx.x];
        while (q < q1) {
            const int qe = min(q1, bnext[q]);
            bar_dense(WD * 32);
            if (threadIdx.x == 0) {
                s_ctr = q;
                const long long c0 = (long long)rblk[q] * S;
                const int cn = (int)((ncols - c0) < S ? (ncols - c0) : S);
                const unsigned bytes = (unsigned)(cn * 4 + 15) & ~15u;
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect(smb, bytes);
                for (unsigned off = 0; off < bytes; off += 32768u)
                    bulk_g2s(sb + off, (const char *)(X + c0) + off, bytes - off < 32768u ? bytes - off : 32768u, smb);
            }
            bar_dense(WD * 32);
            mbar_wait(smb, phase);
            phase ^= 1u;
            for (;;) {
                int t = 0;
                if (lane == 0) t = atomicAdd(&s_ctr, 1);
                t = __shfl_sync(0xffffffffu, t, 0);
                if (t >= qe) break;
                uint4 w[4];
#pragma unroll
                for (int k = 0; k < 4; k++) w[k] = __ldcs(E + (long long)t * 128 + 32 * k + lane);
                const int o = __ldcs(lbase + (long long)t * 32 + lane);
                const int oe = __ldcs(lbase + (long long)t * 32 + 32);
                const int ob = __shfl_sync(0xffffffffu, o, 0);
                const int cnt = oe - ob;
                const bool staged = cnt <= STG_CAP;
                run4<true>(w, sb, X, staged ? o - ob : o, P, staged, sstg);
                if (staged) {
                    __syncwarp();
                    for (int j = lane; j < cnt; j += 32) P[ob + j] = stg[warp * STG_CAP + j];
                    __syncwarp();
                }
            }
            q = qe;
        }
    } else {
        // ---- cold warps: the CTA's cold span, claimed range by range
        const int q1 = ndr + ccta[blockIdx.x + 1];
        for (;;) {
            int t = 0;
            if (lane == 0) t = atomicAdd(&s_cctr, 1);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t >= q1) break;
            uint4 w[4];
#pragma unroll
            for (int k = 0; k < 4; k++) w[k] = __ldcs(C + (long long)(t - ndr) * 128 + 32 * k + lane);
            const int o = __ldcs(lbase + (long long)t * 32 + lane);
            const int oe = __ldcs(lbase + (long long)t * 32 + 32);
            const int ob = __shfl_sync(0xffffffffu, o, 0);
            const int cnt = oe - ob;
            const bool staged = cnt <= STG_CAP;
            run4<false>(w, sb, X, staged ? o - ob : o, P, staged, sstg);
            if (staged) {
                __syncwarp();
                for (int j = lane; j < cnt; j += 32) P[ob + j] = stg[warp * STG_CAP + j];
                __syncwarp();
            }
        }
    }
}

// K_B: NSEG segments (<= 32); off is [NSEG][ntiles + 1]
__global__ void __launch_bounds__(256) k_b(long long n, int nseg, long long ntiles, const int *__restrict__ off,
                                           const unsigned char *__restrict__ prow8, const float *__restrict__ P, float *__restrict__ y) {
    __shared__ float tab[8][32][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long t = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ntiles; t += nw) {
        for (int b = 0; b < nseg; b++) tab[w][lane][b] = 0.f;
        __syncwarp();
        if (lane < nseg) {
            const int o0 = off[(long long)lane * (ntiles + 1) + t], o1 = off[(long long)lane * (ntiles + 1) + t + 1];
            int p = o0;
            for (; p + 4 <= o1; p += 4) {
                const float v0 = P[p], v1 = P[p + 1], v2 = P[p + 2], v3 = P[p + 3];
                const int r0 = prow8[p], r1 = prow8[p + 1], r2 = prow8[p + 2], r3 = prow8[p + 3];
                tab[w][r0][lane] += v0;
                tab[w][r1][lane] += v1;
                tab[w][r2][lane] += v2;
                tab[w][r3][lane] += v3;
            }
            for (; p < o1; p++) tab[w][prow8[p]][lane] += P[p];
        }
        __syncwarp();
        const long long i = t * 32 + lane;
        if (i < n) {
            double acc = 0.0;
            for (int b = 0; b < nseg; b++) acc += (double)tab[w][lane][b];
            y[i] = (float)acc;
        }
        __syncwarp();
    }
}

extern "C" int tp11_a(int reps, int wd, const void *E, const void *C, const void *X, const void *rblk, const void *bnext, const void *cta,
                      const void *ccta, int ncta, const void *lbase, void *P, int S, long long ncols, int ndr) {
    const int smem = 32768 * 4 + 32 * STG_CAP * 4;
    static bool init = false;
    if (!init) {
        init = true;
        cudaFuncSetAttribute(k_a<24>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_a<20>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_a<28>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_a<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    }
    for (int r = 0; r < reps; r++) {
#define L(WD_)                                                                                                                        \
    k_a<WD_><<<ncta, 1024, smem>>>((const uint4 *)E, (const uint4 *)C, (const float *)X, (const int *)rblk, (const int *)bnext,       \
                                   (const int *)cta, (const int *)ccta, (const int *)lbase, (float *)P, S, ncols, ndr)
        if (wd == 24) L(24);
        else if (wd == 20) L(20);
        else if (wd == 28) L(28);
        else L(16);
#undef L
    }
    return (int)cudaGetLastError();
}

extern "C" int tp11_b(int reps, long long n, int nseg, long long ntiles, const void *off, const void *prow8, const void *P, void *y) {
    for (int r = 0; r < reps; r++)
        k_b<<<148 * 8, 256>>>(n, nseg, ntiles, (const int *)off, (const unsigned char *)prow8, (const float *)P, (float *)y);
    return (int)cudaGetLastError();
}
