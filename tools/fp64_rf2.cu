// DFMA issue cost vs operand sharing (register-file bandwidth), no other instructions in the loop.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE, int NA>
__global__ void k(long iters, double* io) {
    double acc[NA], x[NA], y[NA];
#pragma unroll
    for (int i = 0; i < NA; ++i) { acc[i] = io[threadIdx.x + i]; x[i] = io[64 + i] + threadIdx.x; y[i] = io[128 + i] + i; }
    for (long it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NA; ++i) {
            if (MODE == 0) acc[i] = fma(x[0], y[0], acc[i]);
            if (MODE == 1) acc[i] = fma(x[i], y[0], acc[i]);
            if (MODE == 2) acc[i] = fma(x[i], y[i], acc[i]);
            if (MODE == 3) acc[i] = fma(x[i % 6], y[i / 6], acc[i]);   // spread-like: 6 w0 x 9 pbc
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NA; ++i) s += acc[i];
    if (s == 1234.5) io[0] = s;
}
template <int MODE, int NA>
void run(int wpsm, int sms, double* io) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    long iters = 20000 * 16 / NA; int blocks = sms * wpsm;
    k<MODE, NA><<<blocks, 32>>>(iters / 10, io);
    cudaEventRecord(e0); k<MODE, NA><<<blocks, 32>>>(iters, io); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double tf = 2.0 * NA * iters * blocks * 32 / (ms * 1e-3) / 1e12;
    printf("mode=%d NA=%d warps/SM=%2d  %.1f TF/s (%.0f%%)\n", MODE, NA, wpsm, tf, 100 * tf / 36.7);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* io; cudaMalloc(&io, 4096 * 8); cudaMemset(io, 0, 4096 * 8);
    for (int w : {8}) { run<0, 16>(w, sms, io); run<1, 16>(w, sms, io); run<2, 16>(w, sms, io); run<3, 54>(w, sms, io); run<2, 54>(w, sms, io); run<1, 54>(w, sms, io);}
    return 0;
}
