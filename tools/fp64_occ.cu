// Microbenchmark: FP64 DFMA throughput vs warps/SM and independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void k(long iters, double b, double c, double* sink) {
    double a[C];
#pragma unroll
    for (int i = 0; i < C; ++i) a[i] = threadIdx.x * 1e-9 + i;
    for (long it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < C; ++i) a[i] = fma(a[i], b, c);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < C; ++i) s += a[i];
    if (s == 1234.5) sink[0] = s;
}
template <int C>
void run(int warps_per_sm, int sms) {
    double* sink; cudaMalloc(&sink, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    long iters = 200000 / C * 16;
    int blocks = sms * warps_per_sm;
    k<C><<<blocks, 32>>>(iters / 10, 0.999, 1e-7, sink);
    cudaEventRecord(e0);
    k<C><<<blocks, 32>>>(iters, 0.999, 1e-7, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double tf = 2.0 * C * iters * blocks * 32 / (ms * 1e-3) / 1e12;
    printf("chains=%2d warps/SM=%2d  %.1f TF/s\n", C, warps_per_sm, tf);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {4, 8, 12, 16, 32}) { run<8>(w, sms); run<16>(w, sms); run<32>(w, sms); run<54>(w, sms); }
    return 0;
}
