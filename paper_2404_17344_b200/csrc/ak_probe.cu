// FP64 throughput probes: the roofline denominator for the compute-bound
// spread/interp kernels (MEASURED_PEAKS.json carries HBM and bf16 only).
#include <cuda_runtime.h>
#include <string>
#include "../../include/addkern_b200.h"


// 16 independent DFMA chains per thread.
__global__ void __launch_bounds__(256) k_probe_dfma(int64_t iters, double b, double c, double* sink) {
    double a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-9 + i;
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i];
    if (s == 1234.5) sink[0] = s;
}

// FP64 tensor-core probe: mma.sync m8n8k4 f64, 4 independent accumulators per warp.
__global__ void __launch_bounds__(256) k_probe_dmma(int64_t iters, double b0, double* sink) {
    double acc[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0.0;
    const double a = threadIdx.x * 1e-9 + 1.0;
    const double b = b0;
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[i][0]), "+d"(acc[i][1])
                         : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1];
    if (s == 1234.5) sink[0] = s;
}

static int probe(int kind, int64_t iters, void* stream, double* tflops) {
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* sink = nullptr;
    if (cudaMalloc(&sink, 8) != cudaSuccess) return AK_ERR_ALLOC;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 8, threads = 256;
    // warm-up
    if (kind == 0) k_probe_dfma<<<blocks, threads, 0, st>>>(iters / 10 + 1, 0.999999, 1e-7, sink);
    else k_probe_dmma<<<blocks, threads, 0, st>>>(iters / 10 + 1, 0.999999, sink);
    cudaEventRecord(e0, st);
    if (kind == 0) k_probe_dfma<<<blocks, threads, 0, st>>>(iters, 0.999999, 1e-7, sink);
    else k_probe_dmma<<<blocks, threads, 0, st>>>(iters, 0.999999, sink);
    cudaEventRecord(e1, st);
    cudaError_t err = cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    if (err != cudaSuccess) return AK_ERR_CUDA;
    double flops;
    if (kind == 0) flops = 2.0 * 16.0 * (double)iters * blocks * threads;
    else flops = 2.0 * 8 * 8 * 4 * 4.0 * (double)iters * blocks * (threads / 32);
    *tflops = flops / (ms * 1e-3) / 1e12;
    return AK_OK;
}

extern "C" int ak_probe_fp64(int64_t iters, void* stream, double* tflops) { return probe(0, iters, stream, tflops); }
extern "C" int ak_probe_dmma(int64_t iters, void* stream, double* tflops) { return probe(1, iters, stream, tflops); }
