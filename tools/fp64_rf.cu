// Microbenchmark: DFMA throughput with 1, 2 or 3 distinct register source operands.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(long iters, double* io) {
    double a[16], x[16], y[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) { a[i] = io[threadIdx.x + i]; x[i] = io[64 + i + threadIdx.x]; y[i] = io[128 + i]; }
    for (long it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (MODE == 0) a[i] = fma(a[i], 0.999, 1e-7);          // 1 reg operand
            if (MODE == 1) a[i] = fma(x[0], a[i], y[0]);             // shared x,y (reuse)
            if (MODE == 2) a[i] = fma(x[i], y[i], a[i]);             // 3 distinct regs
            if (MODE == 3) a[i] = fma(x[i & 7], y[i >> 3], a[i]);    // partial reuse
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = x[i] * 1.0000001;  // keep x live/varying (DMUL)
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i];
    if (s == 1234.5) io[0] = s;
}
template <int MODE>
void run(int wpsm, int sms, double* io) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    long iters = 20000; int blocks = sms * wpsm;
    k<MODE><<<blocks, 32>>>(iters / 10, io);
    cudaEventRecord(e0); k<MODE><<<blocks, 32>>>(iters, io); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double tf = 2.0 * 16 * iters * blocks * 32 / (ms * 1e-3) / 1e12;   // counts only the 16 FMAs
    printf("mode=%d warps/SM=%2d  %.1f TF/s (fma only; +16 DMUL per iter)\n", MODE, wpsm, tf);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* io; cudaMalloc(&io, 4096 * 8); cudaMemset(io, 0, 4096 * 8);
    for (int w : {8, 16}) { run<0>(w, sms, io); run<1>(w, sms, io); run<2>(w, sms, io); run<3>(w, sms, io); }
    return 0;
}
