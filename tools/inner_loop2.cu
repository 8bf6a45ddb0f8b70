// Variants of the spread inner loop, plus DFMA/DMUL dependent-chain latency.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2404_17344_b200/csrc/ak_q3.cuh"
using namespace ak;

__global__ void lat(long iters, double* io, int mode) {
    double x = io[threadIdx.x], y = io[1];
    long long t0 = clock64();
    if (mode == 0) for (long i = 0; i < iters; ++i) x = fma(x, y, 1e-9);
    else for (long i = 0; i < iters; ++i) x = x * y;
    long long t1 = clock64();
    if (threadIdx.x == 0) io[100 + mode] = (double)(t1 - t0) / iters;
    if (x == 1234.5) io[0] = x;
}

// V=0: reference (LDS weights + DMUL products); V=1: products precomputed in smem (no DMUL);
// V=2: weights in registers (no LDS), DMUL products; V=3: a-outer loop order
template <int V>
__global__ void __launch_bounds__(32, 8) k(long iters, double* io) {
    constexpr int T = 12, P0 = 6, P1 = 3, P2 = 3;
    __shared__ __align__(16) double wst[32][48];
    const int lane = threadIdx.x, g0 = lane >> 4, g1 = (lane >> 2) & 3, g2 = lane & 3;
    for (int i = lane; i < 32 * 48; i += 32) (&wst[0][0])[i] = io[i % 64] + 1e-3 * i;
    __syncwarp();
    double acc[P0][P1][P2];
    for (int a = 0; a < P0; ++a) for (int b = 0; b < P1; ++b) for (int c = 0; c < P2; ++c) acc[a][b][c] = 0;
    double r0[P0], r1[P1], r2[P2];
    load_w<T>(r0, r1, r2, &wst[3][0], g0, g1, g2);
    for (long it = 0; it < iters; ++it) {
#pragma unroll 2
        for (int j = 0; j < 32; ++j) {
            if (V == 0) {
                double a0[P0], a1[P1], a2[P2];
                load_w<T>(a0, a1, a2, &wst[j][0], g0, g1, g2);
                spread_fma(acc, a0, a1, a2);
            } else if (V == 1) {
                double a0[P0], p[P1 * P2];
                const double* row = &wst[j][0];
                for (int a = 0; a < P0; ++a) a0[a] = row[g0 * P0 + a];
                for (int q = 0; q < 9; ++q) p[q] = row[12 + (g1 * 4 + g2) + q];
                for (int b = 0; b < P1; ++b) for (int c = 0; c < P2; ++c) for (int a = 0; a < P0; ++a)
                    acc[a][b][c] = fma(a0[a], p[b * 3 + c], acc[a][b][c]);
            } else if (V == 2) {
                r0[j % P0] += 1e-12;
                spread_fma(acc, r0, r1, r2);
            } else {
                double a0[P0], a1[P1], a2[P2];
                load_w<T>(a0, a1, a2, &wst[j][0], g0, g1, g2);
                double p[P1][P2];
                for (int b = 0; b < P1; ++b) for (int c = 0; c < P2; ++c) p[b][c] = a1[b] * a2[c];
                for (int a = 0; a < P0; ++a) for (int b = 0; b < P1; ++b) for (int c = 0; c < P2; ++c)
                    acc[a][b][c] = fma(a0[a], p[b][c], acc[a][b][c]);
            }
        }
    }
    double s = 0;
    for (int a = 0; a < P0; ++a) for (int b = 0; b < P1; ++b) for (int c = 0; c < P2; ++c) s += acc[a][b][c];
    if (s == 1234.5) io[0] = s;
}
template <int V>
void run(int wpsm, int sms, double* io) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    long iters = 2000; int blocks = sms * wpsm;
    k<V><<<blocks, 32>>>(iters / 10, io);
    cudaEventRecord(e0); k<V><<<blocks, 32>>>(iters, io); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 1728 * 32 * iters * blocks;
    printf("variant=%d warps/SM=%2d  %.1f TF/s algorithmic (%.0f%%)\n", V, wpsm, fl / (ms * 1e-3) / 1e12, 100 * fl / (ms * 1e-3) / 1e12 / 36.7);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* io; cudaMalloc(&io, 4096 * 8); cudaMemset(io, 0, 4096 * 8);
    double h[2];
    for (int m = 0; m < 2; ++m) { lat<<<1, 32>>>(100000, io, m); }
    cudaMemcpy(h, io + 100, 16, cudaMemcpyDeviceToHost);
    printf("latency: DFMA %.1f cycles, DMUL %.1f cycles\n", h[0], h[1]);
    for (int w : {8, 16}) { run<0>(w, sms, io); run<1>(w, sms, io); run<2>(w, sms, io); run<3>(w, sms, io); }
    return 0;
}
