// 2D-staged SpMV design study v5 (plan: p5d_plan.py): v4's staged tiles for the warm columns, plus a
// per-panel cold phase gathering the remaining columns straight from L2.
// (v4 notes:)  One CTA of 1024 threads per SM walks a static
// sequence of tiles (its panels' tiles, panel after panel).  A ring of P5D_NS slots stages tiles
// ahead with cp.async (sector ids prefetched one tile earlier); per tile the warps claim items in
// LPT order (slices: one lane per short pair; pieces: lane-strided groups of 8 + xor tree;
// sub-pieces: partials, the last arriver of a combine sums them in order); fp64 accumulators in
// shared memory; after a panel's last tile, the PageRank epilogue over its rows.
#include <cstdint>
#include <cuda_runtime.h>

#ifndef P5D_SMAX
#define P5D_SMAX 768
#endif
#ifndef P5D_BLOB
#define P5D_BLOB 16384
#endif
#ifndef P5D_NRMAX
#define P5D_NRMAX 8192
#endif
#ifndef P5D_PMAX
#define P5D_PMAX 256
#endif
#ifndef P5D_CMAX
#define P5D_CMAX 64
#endif
#ifndef P5D_MAXSEQ
#define P5D_MAXSEQ 256
#endif
#ifndef P5D_NT
#define P5D_NT 1024
#endif
#ifndef P5D_NS
#define P5D_NS 3
#endif

#define S8 (P5D_SMAX * 8)
#define XBYTES ((S8 + 8) * 4)
#define SLOT_BYTES (XBYTES + P5D_BLOB)

struct Args {
    const float *x;
    const int *secs;
    const uint4 *blob;
    const int *tiles;        // int[8]: blob16, n16, sec_off, nsec, nitems, ncomb, comb_off (u16), panel
    const int *panels;       // int[8]: grp_begin, grp_end, tile_begin, tile_end, nr
    const int *seqrec;       // per sequence entry int[8]: blob16, n16, sec_off, nsec, nitems, comb_off, panel | last << 30, tile (-1: none)
    const int *seqoff;       // [grid + 1]
    const int4 *citems;      // cold items: piece {off, len, slot|cmb, -1|pslot}; slice {off, L | 1 << 30, rows_off, 0}
    const int4 *ccomb;       // cold combines {slot, pfirst, count, 0}
    const unsigned *cidx;    // cold gather-layout indices
    const unsigned short *crows;
    const unsigned *gmask;
    const int *gbase;
    const float *t, *dinv;
    const int *perm;
    float *r, *y;
    double *red;
    long long n;
    float c;
};

__device__ __forceinline__ void cp16(unsigned dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ float lds_f(unsigned a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}

extern "C" __global__ void __launch_bounds__(P5D_NT, 1024 / P5D_NT) k_p5d(const Args a) {
    extern __shared__ __align__(16) unsigned char sm[];
    double *ACC = (double *)sm;
    double *PART = ACC + P5D_NRMAX;
    unsigned char *RING = (unsigned char *)(PART + P5D_PMAX);
    __shared__ int s_item[P5D_NS];
    __shared__ int s_tick[P5D_NS][P5D_CMAX];
    __shared__ int4 s_rec[P5D_MAXSEQ][2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned ring_s = (unsigned)__cvta_generic_to_shared(RING);
    const int k0 = a.seqoff[blockIdx.x], k1 = a.seqoff[blockIdx.x + 1];
    for (int k = tid; k < 2 * (k1 - k0); k += P5D_NT) ((int4 *)s_rec)[k] = ((const int4 *)a.seqrec)[2 * k0 + k];
    for (int k = tid; k < P5D_NRMAX; k += P5D_NT) ACC[k] = 0.0;
    for (int s = 0; s < P5D_NS; s++)
        if (tid < 8) ((float *)(RING + s * SLOT_BYTES))[S8 + tid] = 0.f;
    __syncthreads();
    // issue sequence entry kk (relative) into its slot; `id` = this thread's sector id (prefetched)
    auto issue = [&](int kk, int id) {
        const int sl = kk % P5D_NS;
        const int4 q0 = s_rec[kk][0];
        const unsigned dst = ring_s + sl * SLOT_BYTES;
        if (tid < q0.w) {
            const float *src = a.x + 8ll * id;
            cp16(dst + tid * 32, src);
            cp16(dst + tid * 32 + 16, src + 4);
        }
#if P5D_SMAX > P5D_NT
#error "P5D_SMAX must be <= P5D_NT"
#endif
        for (int c = tid; c < q0.y; c += P5D_NT) cp16(dst + XBYTES + c * 16, a.blob + q0.x + c);
        if (tid == 0) s_item[sl] = 0;
        if (tid < P5D_CMAX) s_tick[sl][tid] = 0;
        cp_commit();
    };
    auto load_id = [&](int kk) -> int {
        if (kk >= k1 - k0) return 0;
        const int4 q0 = s_rec[kk][0];
        return tid < q0.w ? __ldg(a.secs + q0.z + tid) : 0;
    };
    const int nk = k1 - k0;
    for (int j = 0; j < P5D_NS - 1; j++) {
        if (j < nk) issue(j, load_id(j));
        else cp_commit();
    }
    // sector ids for entries NS-1, NS, NS+1 in flight (used two iterations after their load)
    int id0 = load_id(P5D_NS - 1), id1 = load_id(P5D_NS), id2 = load_id(P5D_NS + 1);
    double dl = 0.0, dsum = 0.0;
    for (int k = 0; k < nk; k++) {
        if (k + P5D_NS - 1 < nk) issue(k + P5D_NS - 1, id0);
        else cp_commit();
        id0 = id1; id1 = id2; id2 = load_id(k + P5D_NS + 2);
        cp_wait<P5D_NS - 1>();
        __syncthreads();
        const int4 r0 = s_rec[k][0], r1 = s_rec[k][1];
        const int fl = r1.z;
        const int sl = k % P5D_NS;
        if (r1.w >= 0) {
            const int ni = r1.x, coff = r1.y;
            const unsigned xs = ring_s + sl * SLOT_BYTES;
            const unsigned short *H16 = (const unsigned short *)(RING + sl * SLOT_BYTES + XBYTES);
            (void)r0;
            for (;;) {
                int i = 0;
                if (lane == 0) i = atomicAdd(&s_item[sl], 1);
                i = __shfl_sync(0xffffffffu, i, 0);
                if (i >= ni) break;
                const uint2 rq = *(const uint2 *)(H16 + 4 * i);
                const int off8 = rq.x & 0xffff, ln = rq.x >> 16, ia = rq.y & 0xffff, ic = rq.y >> 16;
                if (ln & 0x8000) {
                    const int L = ln & 0x7fff;
                    const int row = H16[ia + lane];
                    const unsigned short *e = H16 + off8 * 8 + lane;
                    double s = 0.0;
                    int kq = 0;
                    for (; kq + 4 <= L; kq += 4) {
                        const float v0 = lds_f(xs + e[(kq + 0) * 32] * 4), v1 = lds_f(xs + e[(kq + 1) * 32] * 4);
                        const float v2 = lds_f(xs + e[(kq + 2) * 32] * 4), v3 = lds_f(xs + e[(kq + 3) * 32] * 4);
                        s += (double)v0; s += (double)v1; s += (double)v2; s += (double)v3;
                    }
                    for (; kq < L; kq++) s += (double)lds_f(xs + e[kq * 32] * 4);
                    if (row != 0xffff) ACC[row] += s;
                } else {
                    double s = 0.0;
                    for (int j = lane; j < ln; j += 32) {
                        const uint4 e = ((const uint4 *)H16)[off8 + j];
                        const float v0 = lds_f(xs + (e.x & 0xffff) * 4), v1 = lds_f(xs + (e.x >> 16) * 4);
                        const float v2 = lds_f(xs + (e.y & 0xffff) * 4), v3 = lds_f(xs + (e.y >> 16) * 4);
                        const float v4 = lds_f(xs + (e.z & 0xffff) * 4), v5 = lds_f(xs + (e.z >> 16) * 4);
                        const float v6 = lds_f(xs + (e.w & 0xffff) * 4), v7 = lds_f(xs + (e.w >> 16) * 4);
                        s += (double)v0; s += (double)v1; s += (double)v2; s += (double)v3;
                        s += (double)v4; s += (double)v5; s += (double)v6; s += (double)v7;
                    }
#pragma unroll
                    for (int d = 16; d >= 1; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
                    if (lane == 0) {
                        if (ic == 0xffff) {
                            ACC[ia] += s;
                        } else {
                            PART[ic] = s;
                            __threadfence_block();
                            const int cnt = H16[coff + 4 * ia + 2];
                            if (atomicAdd(&s_tick[sl][ia], 1) == cnt - 1) {
                                __threadfence_block();
                                const int row = H16[coff + 4 * ia], f = H16[coff + 4 * ia + 1];
                                double u = *(volatile double *)&PART[f];
                                for (int j = 1; j < cnt; j++) u += *(volatile double *)&PART[f + j];
                                ACC[row] += u;
                            }
                        }
                    }
                }
            }
        }
        else if (r1.w == -2) {
            // cold phase: items gathered from L2
            const int i0 = r0.x, c0 = r0.z, ni = r1.x;
            const float *X = a.x;
            for (;;) {
                int i = 0;
                if (lane == 0) i = atomicAdd(&s_item[sl], 1);
                i = __shfl_sync(0xffffffffu, i, 0);
                if (i >= ni) break;
                const int4 rq = __ldg(a.citems + i0 + i);
                if (rq.y & (1 << 30)) {
                    const int L = rq.y & ((1 << 30) - 1);
                    const int row = __ldg(a.crows + rq.z + lane);
                    const unsigned *e = a.cidx + rq.x + lane;
                    double s = 0.0;
                    int kq = 0;
                    for (; kq + 4 <= L; kq += 4) {
                        const unsigned i0_ = __ldcs(e + (kq + 0) * 32), i1_ = __ldcs(e + (kq + 1) * 32);
                        const unsigned i2_ = __ldcs(e + (kq + 2) * 32), i3_ = __ldcs(e + (kq + 3) * 32);
                        const float v0 = __ldcg(X + i0_), v1 = __ldcg(X + i1_), v2 = __ldcg(X + i2_), v3 = __ldcg(X + i3_);
                        s += (double)v0; s += (double)v1; s += (double)v2; s += (double)v3;
                    }
                    for (; kq < L; kq++) s += (double)__ldcg(X + __ldcs(e + kq * 32));
                    if (row != 0xffff) ACC[row] += s;
                } else {
                    const int n4 = (rq.y + 3) >> 2;
                    const uint4 *e4 = (const uint4 *)(a.cidx + rq.x);
                    double s = 0.0;
                    int j = lane;
                    for (; j + 32 < n4; j += 64) {
                        const uint4 qa = __ldcs(e4 + j), qb = __ldcs(e4 + j + 32);
                        const float v0 = __ldcg(X + qa.x), v1 = __ldcg(X + qa.y), v2 = __ldcg(X + qa.z), v3 = __ldcg(X + qa.w);
                        const float v4 = __ldcg(X + qb.x), v5 = __ldcg(X + qb.y), v6 = __ldcg(X + qb.z), v7 = __ldcg(X + qb.w);
                        s += (double)v0; s += (double)v1; s += (double)v2; s += (double)v3;
                        s += (double)v4; s += (double)v5; s += (double)v6; s += (double)v7;
                    }
                    for (; j < n4; j += 32) {
                        const uint4 qa = __ldcs(e4 + j);
                        const float v0 = __ldcg(X + qa.x), v1 = __ldcg(X + qa.y), v2 = __ldcg(X + qa.z), v3 = __ldcg(X + qa.w);
                        s += (double)v0; s += (double)v1; s += (double)v2; s += (double)v3;
                    }
#pragma unroll
                    for (int d = 16; d >= 1; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
                    if (lane == 0) {
                        if (rq.w < 0) {
                            ACC[rq.z] += s;
                        } else {
                            PART[rq.w] = s;
                            __threadfence_block();
                            const int4 cb = __ldg(a.ccomb + c0 + rq.z);
                            if (atomicAdd(&s_tick[sl][rq.z], 1) == cb.z - 1) {
                                __threadfence_block();
                                double u = *(volatile double *)&PART[cb.y];
                                for (int q = 1; q < cb.z; q++) u += *(volatile double *)&PART[cb.y + q];
                                ACC[cb.x] += u;
                            }
                        }
                    }
                }
            }
        }
        __syncthreads();
        if (fl >> 30) {
            const int p = fl & ((1 << 29) - 1);
            const int4 pr = ((const int4 *)a.panels)[2 * p];
            const int nr = a.panels[8 * p + 4];
            // 4 groups per warp per trip: all loads first
            for (int gq = pr.x + warp; gq < pr.y; gq += 4 * (P5D_NT / 32)) {
                unsigned m[4]; int gb[4]; float tv[4], dv[4]; int pm[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int grp = gq + (P5D_NT / 32) * u;
                    const long long i = (long long)grp * 32 + lane;
                    const bool ok = grp < pr.y && i < a.n;
                    m[u] = grp < pr.y ? __ldg(a.gmask + grp) : 0u;
                    gb[u] = grp < pr.y ? __ldg(a.gbase + grp) : 0;
                    tv[u] = ok ? __ldg(a.t + i) : 0.f;
                    dv[u] = ok ? __ldg(a.dinv + i) : 0.f;
                    pm[u] = ok ? __ldg(a.perm + i) : -1;
                }
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int grp = gq + (P5D_NT / 32) * u;
                    const long long i = (long long)grp * 32 + lane;
                    if (grp < pr.y && i < a.n) {
                        const double acc = ((m[u] >> lane) & 1u) ? ACC[gb[u] + __popc(m[u] & ((1u << lane) - 1u))] : 0.0;
                        const float r = (float)acc + a.c;
                        a.r[i] = r;
                        dl += fabs((double)r - (double)tv[u]);
                        if (dv[u] == 0.f) dsum += (double)r;
                        if (pm[u] >= 0) a.y[pm[u]] = r * dv[u];
                    }
                }
            }
            __syncthreads();
            for (int q = tid; q < nr; q += P5D_NT) ACC[q] = 0.0;
            __syncthreads();
        }
    }
    cp_wait<0>();
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        dl += __shfl_xor_sync(0xffffffffu, dl, d);
        dsum += __shfl_xor_sync(0xffffffffu, dsum, d);
    }
    if (lane == 0) {
        atomicAdd(&a.red[0], dl);
        atomicAdd(&a.red[1], dsum);
    }
}

extern "C" int p5d_smem() { return (P5D_NRMAX + P5D_PMAX) * 8 + P5D_NS * SLOT_BYTES; }

extern "C" int p5d_launch(const Args *a, int grid, cudaStream_t st) {
    static bool init = false;
    const int smem = p5d_smem();
    if (!init) {
        cudaFuncSetAttribute(k_p5d, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        init = true;
    }
    k_p5d<<<grid, P5D_NT, smem, st>>>(*a);
    return (int)cudaGetLastError();
}
