// Spread inner loop: the k_spread3c form (6 w0 + 3 w1 + 3 w2 loads, 9 DMUL products,
// 54 DFMA per lane per point) vs the w1 (x) w2 products precomputed per point in
// shared memory (6 w0 + 9 product loads, no DMUL: 11% fewer FP64-pipe instructions,
// 25% more shared loads).  9 warps per SM (the real kernel's occupancy).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2404_17344_b200/csrc/ak_q3.cuh"
using namespace ak;
constexpr int T = 12, P0 = 6, P1 = 3, P2 = 3;

template <int V>
__global__ void __launch_bounds__(32, 9) k(long iters, double* io) {
    constexpr int RW = V == 0 ? 36 : 12 + 144;
    constexpr int NB = 16;
    __shared__ __align__(16) double wbuf[NB][RW];
    const int lane = threadIdx.x, g0 = lane >> 4, g1 = (lane >> 2) & 3, g2 = lane & 3;
    for (int i = lane; i < NB * RW; i += 32) (&wbuf[0][0])[i] = io[i % 64] + 1e-3 * i;
    __syncwarp();
    double acc[P0][P1][P2];
#pragma unroll
    for (int a = 0; a < P0; ++a)
#pragma unroll
        for (int b = 0; b < P1; ++b)
#pragma unroll
            for (int c = 0; c < P2; ++c) acc[a][b][c] = 0;
    for (long it = 0; it < iters; ++it) {
#pragma unroll 2
        for (int j = 0; j < NB; ++j) {
            const double* row = wbuf[j];
            double w0[P0];
#pragma unroll
            for (int a = 0; a < P0; ++a) w0[a] = row[g0 * P0 + a];
            if (V == 0) {
                double w1[P1], w2[P2];
#pragma unroll
                for (int b = 0; b < P1; ++b) w1[b] = row[T + g1 * P1 + b];
#pragma unroll
                for (int c = 0; c < P2; ++c) w2[c] = row[2 * T + g2 * P2 + c];
                spread_fma(acc, w0, w1, w2);
            } else {
#pragma unroll
                for (int b = 0; b < P1; ++b)
#pragma unroll
                    for (int c = 0; c < P2; ++c) {
                        const double p = row[T + (g1 * P1 + b) * T + g2 * P2 + c];
#pragma unroll
                        for (int a = 0; a < P0; ++a) acc[a][b][c] = fma(w0[a], p, acc[a][b][c]);
                    }
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int a = 0; a < P0; ++a)
#pragma unroll
        for (int b = 0; b < P1; ++b)
#pragma unroll
            for (int c = 0; c < P2; ++c) s += acc[a][b][c];
    if (s == 1234.5) io[0] = s;
}
template <int V>
void run(int wpsm, int sms, double* io) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    long iters = 2000;
    int blocks = sms * wpsm;
    k<V><<<blocks, 32>>>(iters / 10, io);
    cudaEventRecord(e0);
    k<V><<<blocks, 32>>>(iters, io);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 1728 * 16 * iters * blocks;
    printf("variant=%d warps/SM=%d  %.1f TF/s algorithmic (%.0f%% of 36.7)\n", V, wpsm, fl / (ms * 1e-3) / 1e12,
           100 * fl / (ms * 1e-3) / 1e12 / 36.7);
}
int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* io;
    cudaMalloc(&io, 4096 * 8);
    cudaMemset(io, 0, 4096 * 8);
    for (int w : {8, 9}) {
        run<0>(w, sms, io);
        run<1>(w, sms, io);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
