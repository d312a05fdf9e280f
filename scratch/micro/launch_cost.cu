// host cost of one launch vs kernel-parameter size and dynamic shared memory (C1 host path)
#include <cstdio>
#include <chrono>
#include <cuda_runtime.h>
template <int N> struct P { long long v[N]; };
template <int N> __global__ void k(P<N> p) { if (p.v[0] == 12345 && threadIdx.x == 0) printf("x"); }
__global__ void kd(P<128> p) { extern __shared__ char sm[]; if (p.v[0] == 12345) sm[threadIdx.x] = 1; }
template <class F> double time_launch(F f, cudaStream_t s) {
    for (int i = 0; i < 200; i++) f();
    cudaStreamSynchronize(s);
    auto t0 = std::chrono::high_resolution_clock::now();
    for (int i = 0; i < 2000; i++) f();
    auto t1 = std::chrono::high_resolution_clock::now();
    cudaStreamSynchronize(s);
    return std::chrono::duration<double, std::micro>(t1 - t0).count() / 2000;
}
int main() {
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    P<1> p1{}; P<16> p16{}; P<128> p128{}; P<512> p512{};
    printf("8 B params   : %.2f us\n", time_launch([&] { k<1><<<2, 768, 0, s>>>(p1); }, s));
    printf("128 B params : %.2f us\n", time_launch([&] { k<16><<<2, 768, 0, s>>>(p16); }, s));
    printf("1 KB params  : %.2f us\n", time_launch([&] { k<128><<<2, 768, 0, s>>>(p128); }, s));
    printf("4 KB params  : %.2f us\n", time_launch([&] { k<512><<<2, 768, 0, s>>>(p512); }, s));
    cudaFuncSetAttribute(kd, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    printf("1 KB + 197 KB smem : %.2f us\n", time_launch([&] { kd<<<2, 768, 197 * 1024, s>>>(p128); }, s));
    printf("1 KB + 197 KB smem, 148 CTAs : %.2f us\n", time_launch([&] { kd<<<148, 768, 197 * 1024, s>>>(p128); }, s));
    cudaEvent_t e; cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    printf("event record : %.2f us\n", time_launch([&] { cudaEventRecord(e, s); }, s));
    return 0;
}
