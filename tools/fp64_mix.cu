// Are FP64 DMMA (mma.sync m8n8k4) and DFMA separate pipes?  Run them alone and interleaved.
#include <cstdio>
#include <cuda_runtime.h>
template <int NF, int NM>
__global__ void k(long iters, double* io) {
    double f[16];
    double acc[4][2];
#pragma unroll
    for (int i = 0; i < 16; ++i) f[i] = io[threadIdx.x] + i;
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0;
    const double a = io[1] + threadIdx.x, b = io[2];
    for (long it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < NF; ++r)
#pragma unroll
            for (int i = 0; i < 16; ++i) f[i] = fma(f[i], 0.999, 1e-7);
#pragma unroll
        for (int r = 0; r < NM; ++r)
#pragma unroll
            for (int i = 0; i < 4; ++i)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += f[i];
#pragma unroll
    for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1];
    if (s == 1234.5) io[0] = s;
}
template <int NF, int NM>
void run(int wpsm, int sms, double* io) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    long iters = 4000; int blocks = sms * wpsm;
    k<NF, NM><<<blocks, 32>>>(iters / 10, io);
    cudaEventRecord(e0); k<NF, NM><<<blocks, 32>>>(iters, io); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl_f = 2.0 * 16 * NF * iters * blocks * 32, fl_m = 2.0 * 256 * 4 * NM * iters * blocks;
    printf("NF=%d NM=%d warps/SM=%2d  dfma %.1f + dmma %.1f = %.1f TF/s  (%.3f ms)\n", NF, NM, wpsm,
           fl_f / (ms * 1e-3) / 1e12, fl_m / (ms * 1e-3) / 1e12, (fl_f + fl_m) / (ms * 1e-3) / 1e12, ms);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* io; cudaMalloc(&io, 4096 * 8); cudaMemset(io, 0, 4096 * 8);
    for (int w : {8, 16}) { run<8, 0>(w, sms, io); run<0, 8>(w, sms, io); run<8, 8>(w, sms, io); run<8, 4>(w, sms, io); run<4, 8>(w, sms, io); }
    return 0;
}
