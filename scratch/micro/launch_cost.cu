// host cost of one launch: small vs ~850-byte parameter struct, with / without two event records
#include <cstdio>
#include <chrono>
struct Big { long long v[108]; };
__global__ void ks(long long a) { if (a == -1) printf("x"); }
__global__ void kb(const Big b) { if (b.v[0] == -1) printf("x"); }
int main() {
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    Big b{}; cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int mode = 0; mode < 4; mode++) {
        for (int rep = 0; rep < 2; rep++) {
            cudaStreamSynchronize(s);
            auto t0 = std::chrono::steady_clock::now();
            const int N = 2000;
            for (int i = 0; i < N; i++) {
                if (mode & 2) cudaEventRecord(e0, s);
                if (mode & 1) { void *p[] = {&b}; cudaLaunchKernel((const void *)kb, dim3(1), dim3(32), p, 0, s); }
                else { long long a = i; void *p[] = {&a}; cudaLaunchKernel((const void *)ks, dim3(1), dim3(32), p, 0, s); }
                if (mode & 2) cudaEventRecord(e1, s);
                if ((i & 63) == 63) cudaStreamSynchronize(s);   // keep the queue short
            }
            cudaStreamSynchronize(s);
            auto t1 = std::chrono::steady_clock::now();
            if (rep) printf("params %s events %s: %.2f us per launch\n", (mode & 1) ? "864 B" : "8 B", (mode & 2) ? "2" : "0",
                            std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
        }
    }
    return 0;
}
