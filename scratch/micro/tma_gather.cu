// can Blackwell's TMA gather (cp.async.bulk.tensor.2d ... tile::gather4)
// take the SpMV's random cold gathers off the LSU / L1TEX data pipe?  x is an L2-resident
// [R][8] fp32 tensor (8 MB, C4's gathered vector); M random rows are fetched
//   (a) by the LSU: one 4-byte ld.global.cg per index (the SpMV's cold gather), and
//   (b) by TMA gather4: one elected thread per producer warp issues gather4s (4 rows x 32 B each)
//       into a shared-memory ring of stages completing on mbarriers; consumer threads read the
//       element they need from shared memory.
// Reports G rows per second for each and checks the gathered sums against a host reference.
// Every mbarrier wait is bounded (a missing completion sets an error flag instead of hanging).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

// 8 independent gathers in flight per thread (the SpMV's depth), index loads coalesced
__global__ void k_lsu(const float *X, const int *idx, long long M, double *out) {
    double s = 0.0;
    const long long T = (long long)gridDim.x * blockDim.x;
    for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < M; i0 += 8 * T) {
        float v[8];
        #pragma unroll
        for (int u = 0; u < 8; u++) {
            const long long i = i0 + u * T;
            v[u] = 0.f;
            if (i < M) asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v[u]) : "l"(X + (long long)idx[i] * 8 + (i & 7)));
        }
        #pragma unroll
        for (int u = 0; u < 8; u++) s += v[u];
    }
    for (int d = 16; d; d >>= 1) s += __shfl_down_sync(0xffffffffu, s, d);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, s);   // one atomic per warp (a per-thread one serialises)
}

__device__ __forceinline__ unsigned sa(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

// NP producer warps (lane 0 issues), NC consumer warps; per producer: NST stages of G gather4s
template <int NP, int NST, int G>
__global__ void __launch_bounds__(32 * (NP + 8)) k_tma(const __grid_constant__ CUtensorMap tm, const int *idx, long long M, double *out, int *err) {
    extern __shared__ __align__(128) float sm[];                 // [NP][NST][G*4 rows][8]
    __shared__ __align__(8) unsigned long long full[NP][NST], empty[NP][NST];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int NC = 8;                                             // consumer warps
    if (threadIdx.x == 0) {
        for (int p = 0; p < NP; p++)
            for (int s = 0; s < NST; s++) {
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&full[p][s])));
                asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(sa(&empty[p][s])), "r"(NC / NP));
            }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    const long long per_step = (long long)G * 4;                  // rows per stage
    const long long nsteps = M / per_step;
    // producer p handles steps p, p + NP, ... of this CTA's share; consumer warps c serve producer c % NP
    const long long cta_steps0 = blockIdx.x, cta_stride = gridDim.x;
    if (warp < NP) {
        // the producer warp loads its stage's 4 G indices coalesced (G*4/32 per lane), then lane 0
        // issues the G gather4s with the row ids taken from the lanes by shuffles
        static_assert((G * 4) % 32 == 0, "whole index words per lane");
        constexpr int K = G * 4 / 32;
        const int p = warp;
        int it = 0;
        for (long long st = cta_steps0 + (long long)p * cta_stride; st < nsteps; st += (long long)NP * cta_stride, it++) {
            const int s = it % NST;
            int rid[K];
            #pragma unroll
            for (int k = 0; k < K; k++) rid[k] = idx[st * per_step + k * 32 + lane];
            if (lane == 0 && it >= NST) {
                const unsigned ph = ((it / NST) & 1) ^ 1;           // wait for the consumers to free the stage
                unsigned done = 0; long long spins = 0;
                while (!done) {
                    asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0, 1, 0, q; }"
                                 : "=r"(done) : "r"(sa(&empty[p][s])), "r"(ph));
                    if (++spins > (1ll << 22)) { atomicExch(err, 1); break; }
                }
            }
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&full[p][s])), "r"(G * 4 * 32));
            float *dst = sm + ((size_t)(p * NST + s) * G * 4) * 8;
            #pragma unroll
            for (int g = 0; g < G; g++) {
                const int k = (4 * g) / 32, l0 = (4 * g) % 32;
                const int r0 = __shfl_sync(0xffffffffu, rid[k], l0), r1 = __shfl_sync(0xffffffffu, rid[k], l0 + 1);
                const int r2 = __shfl_sync(0xffffffffu, rid[k], l0 + 2), r3 = __shfl_sync(0xffffffffu, rid[k], l0 + 3);
                if (lane == 0)
                    asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                                 :: "r"(sa(dst + g * 32)), "l"(&tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(sa(&full[p][s]))
                                 : "memory");
            }
        }
        return;
    }
    // consumers
    const int c = warp - NP, p = c % NP;
    double acc = 0.0;
    int it = 0;
    for (long long st = cta_steps0 + (long long)p * cta_stride; st < nsteps; st += (long long)NP * cta_stride, it++) {
        const int s = it % NST;
        unsigned done = 0; long long spins = 0;
        while (!done) {
            asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0, 1, 0, q; }"
                         : "=r"(done) : "r"(sa(&full[p][s])), "r"((unsigned)((it / NST) & 1)));
            if (++spins > (1ll << 22)) { atomicExch(err, 2); return; }
        }
        // the consumers of producer p split its rows: consumer j of NC/NP takes rows j, j + NC/NP, ...
        const int j = c / NP, nj = NC / NP;
        const float *src = sm + ((size_t)(p * NST + s) * G * 4) * 8;
        for (int r = j * 32 + lane; r < G * 4; r += nj * 32) {
            const long long i = st * per_step + r;
            acc += src[r * 8 + (i & 7)];
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(sa(&empty[p][s])) : "memory");
    }
    for (int d = 16; d; d >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, d);
    if (lane == 0) atomicAdd(out, acc);
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                             const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int NP, int NST, int G>
int run_tma(const CUtensorMap &tm, const int *d_idx, long long M, double *d_out, int *d_err, double ref, int sms, int ctas_per_sm) {
    static_assert(8 % NP == 0, "the 8 consumer warps are split evenly over the producers");
    const size_t smem = (size_t)NP * NST * G * 4 * 8 * sizeof(float);
    auto k = k_tma<NP, NST, G>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = sms * ctas_per_sm, block = 32 * (NP + 8);
    float best = 1e30f;
    for (int rep = 0; rep < 6; rep++) {
        CK(cudaMemset(d_out, 0, 8));
        CK(cudaMemset(d_err, 0, 4));
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        k<<<grid, block, smem>>>(tm, d_idx, M, d_out, d_err);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        CK(cudaGetLastError());
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep) best = ms < best ? ms : best;
        int err; double got;
        CK(cudaMemcpy(&err, d_err, 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&got, d_out, 8, cudaMemcpyDeviceToHost));
        if (err || (rep == 0 && (got - ref) * (got - ref) > 1e-6 * ref * ref)) {
            printf("TMA NP=%d NST=%d G=%d: %s (sum %.6f ref %.6f)\n", NP, NST, G, err ? "bounded wait expired" : "WRONG", got, ref);
            return 1;
        }
    }
    const long long rows = (M / (G * 4)) * (G * 4);
    printf("TMA gather4  producers/CTA %d stages %d gather4s/stage %d, %d CTAs/SM, smem %zu KB: %.3f ms  %.1f G rows/s\n", NP, NST, G,
           ctas_per_sm, smem / 1024, best, rows / (best * 1e-3) / 1e9);
    return 0;
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const long long R = 1 << 18, M = 1ll << 25;
    std::vector<float> hx(R * 8);
    for (long long i = 0; i < R * 8; i++) hx[i] = (float)((i * 2654435761ull) % 1000) * 1e-3f;
    std::vector<int> hi(M);
    unsigned long long z = 12345;
    for (long long i = 0; i < M; i++) { z = z * 6364136223846793005ull + 1442695040888963407ull; hi[i] = (int)((z >> 33) % R); }
    double ref = 0.0;
    for (long long i = 0; i < M; i++) ref += hx[(long long)hi[i] * 8 + (i & 7)];
    float *d_x; int *d_idx, *d_err; double *d_out;
    CK(cudaMalloc(&d_x, R * 8 * 4)); CK(cudaMalloc(&d_idx, M * 4)); CK(cudaMalloc(&d_out, 8)); CK(cudaMalloc(&d_err, 4));
    CK(cudaMemcpy(d_x, hx.data(), R * 8 * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_idx, hi.data(), M * 4, cudaMemcpyHostToDevice));
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    // (a) LSU
    {
        float best = 1e30f;
        for (int rep = 0; rep < 6; rep++) {
            CK(cudaMemset(d_out, 0, 8));
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            k_lsu<<<sms * 8, 256>>>(d_x, d_idx, M, d_out);
            cudaEventRecord(b); CK(cudaEventSynchronize(b));
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep) best = ms < best ? ms : best;
            double got; CK(cudaMemcpy(&got, d_out, 8, cudaMemcpyDeviceToHost));
            if (rep == 0 && (got - ref) * (got - ref) > 1e-6 * ref * ref) { printf("LSU WRONG\n"); return 1; }
        }
        printf("LSU ld.global.cg 4 B gathers: %.3f ms  %.1f G rows/s (incl. the 4-byte index stream)\n", best, M / (best * 1e-3) / 1e9);
    }
    // (b) TMA gather4
    void *fn = nullptr; cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    CUtensorMap tm;
    cuuint64_t gdim[2] = {8, (cuuint64_t)R}, gstr[1] = {32};
    cuuint32_t box[2] = {8, 1}, es[2] = {1, 1};
    CUresult r = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d_x, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("cuTensorMapEncodeTiled failed %d\n", (int)r); return 1; }
    int bad = 0;
    bad |= run_tma<1, 8, 16>(tm, d_idx, M, d_out, d_err, ref, sms, 2);
    bad |= run_tma<2, 8, 16>(tm, d_idx, M, d_out, d_err, ref, sms, 2);
    bad |= run_tma<4, 8, 16>(tm, d_idx, M, d_out, d_err, ref, sms, 2);
    bad |= run_tma<4, 8, 32>(tm, d_idx, M, d_out, d_err, ref, sms, 1);
    bad |= run_tma<8, 4, 16>(tm, d_idx, M, d_out, d_err, ref, sms, 2);
    bad |= run_tma<8, 8, 8>(tm, d_idx, M, d_out, d_err, ref, sms, 3);
    bad |= run_tma<8, 4, 8>(tm, d_idx, M, d_out, d_err, ref, sms, 4);
    bad |= run_tma<4, 8, 8>(tm, d_idx, M, d_out, d_err, ref, sms, 4);
    printf(bad ? "SOME_FAILED\n" : "ALL_OK\n");
    return 0;
}
