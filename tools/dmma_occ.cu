// FP64 tensor-core (mma.sync m8n8k4) throughput vs warps per SM, and the interp
// group pattern (54 DMMA + 48-FMA quad contraction + 2 shuffles) vs warps per SM.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__global__ void k_pure(long iters, double* io) {
    double C[18][2];
    for (int t = 0; t < 18; ++t) C[t][0] = C[t][1] = 0;
    const double a = io[1] + threadIdx.x, b = io[2];
    for (long it = 0; it < iters; ++it)
#pragma unroll
        for (int t = 0; t < 18; ++t) dmma(C[t][0], C[t][1], a, b);
    double s = 0;
    for (int t = 0; t < 18; ++t) s += C[t][0] + C[t][1];
    if (s == 1234.5) io[0] = s;
}
__global__ void k_group(long iters, double* io) {
    double gf[18][3];
    for (int t = 0; t < 18; ++t) for (int k = 0; k < 3; ++k) gf[t][k] = io[threadIdx.x + t + k];
    double w[15];
    for (int i = 0; i < 15; ++i) w[i] = io[40 + i];
    double out = 0;
    for (long it = 0; it < iters; ++it) {
        double af[3] = {w[0] + it, w[1], w[2]};
        double C[18][2];
#pragma unroll
        for (int t = 0; t < 18; ++t) C[t][0] = C[t][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < 3; ++ks)
#pragma unroll
            for (int t = 0; t < 18; ++t) dmma(C[t][0], C[t][1], af[ks], gf[t][ks]);
        double acc[4] = {0, 0, 0, 0};
#pragma unroll
        for (int a = 0; a < 12; ++a) {
            double sa = w[12] * C[(3 * a) >> 1][(3 * a) & 1];
#pragma unroll
            for (int bb = 1; bb < 3; ++bb) { const int i = 3 * a + bb; sa = fma(w[12 + bb], C[i >> 1][i & 1], sa); }
            acc[a & 3] = fma(w[a], sa, acc[a & 3]);
        }
        double v = (acc[0] + acc[1]) + (acc[2] + acc[3]);
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        out += v;
    }
    if (out == 1234.5) io[0] = out;
}
// same group pattern, A fragment and contraction weights loaded from shared memory
// per group exactly like k_interp3c (row of 36 doubles per point)
__global__ void k_group_smem(long iters, double* io) {
    __shared__ __align__(16) double wrow[32][36];
    for (int i = threadIdx.x; i < 32 * 36; i += 32) (&wrow[0][0])[i] = io[i % 64] + 1e-3 * i;
    __syncwarp();
    double gf[18][3];
    for (int t = 0; t < 18; ++t) for (int k = 0; k < 3; ++k) gf[t][k] = io[threadIdx.x + t + k];
    const int lane = threadIdx.x, pj = lane >> 2, q = lane & 3;
    double out = 0;
    for (long it = 0; it < iters; ++it) {
        const double* w = wrow[(8 * (it & 3)) + pj];
        double af[3];
#pragma unroll
        for (int ks = 0; ks < 3; ++ks) af[ks] = w[24 + 4 * ks + q];
        double C[18][2];
#pragma unroll
        for (int t = 0; t < 18; ++t) C[t][0] = C[t][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < 3; ++ks)
#pragma unroll
            for (int t = 0; t < 18; ++t) dmma(C[t][0], C[t][1], af[ks], gf[t][ks]);
        double s[3];
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) s[bb] = w[0] * C[bb >> 1][bb & 1];
#pragma unroll
        for (int a = 1; a < 12; ++a) {
            const double w0a = w[a];
#pragma unroll
            for (int bb = 0; bb < 3; ++bb) { const int i = 3 * a + bb; s[bb] = fma(w0a, C[i >> 1][i & 1], s[bb]); }
        }
        const double* w1 = w + 12 + 3 * q;
        double v = fma(w1[2], s[2], fma(w1[1], s[1], w1[0] * s[0]));
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        out += v;
    }
    if (out == 1234.5) io[0] = out;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* io; cudaMalloc(&io, 8192 * 8); cudaMemset(io, 0, 8192 * 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int w : {4, 8, 12, 16, 24, 32}) {
        long iters = 2000; int blocks = sms * w; float ms;
        k_pure<<<blocks, 32>>>(iters / 10, io);
        cudaEventRecord(e0); k_pure<<<blocks, 32>>>(iters, io); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double tf = 2.0 * 256 * 18 * iters * blocks / (ms * 1e-3) / 1e12;
        k_group<<<blocks, 32>>>(iters / 10, io);
        cudaEventRecord(e0); k_group<<<blocks, 32>>>(iters / 3, io); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms2; cudaEventElapsedTime(&ms2, e0, e1);
        // useful: 8 points x 1728 FMA per group
        double tf2 = 2.0 * 8 * 1728 * (iters / 3) * blocks / (ms2 * 1e-3) / 1e12;
        k_group_smem<<<blocks, 32>>>(iters / 10, io);
        cudaEventRecord(e0); k_group_smem<<<blocks, 32>>>(iters / 3, io); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms3; cudaEventElapsedTime(&ms3, e0, e1);
        double tf3 = 2.0 * 8 * 1728 * (iters / 3) * blocks / (ms3 * 1e-3) / 1e12;
        printf("warps/SM=%2d  pure DMMA %.1f TF/s   interp group %.1f TF/s (useful), smem operands %.1f\n", w, tf, tf2, tf3);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
