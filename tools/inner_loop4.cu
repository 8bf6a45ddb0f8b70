// Spread inner loop exactly as k_spread3c (rows of 36 doubles, load_w / spread_fma,
// 2-point ping-pong) vs FMA-order variants, 8 and 12 warps/SM.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2404_17344_b200/csrc/ak_q3.cuh"
using namespace ak;
constexpr int T = 12, P0 = 6, P1 = 3, P2 = 3, RW = 36;

template <int V>
__device__ __forceinline__ void fmas(double (&acc)[P0][P1][P2], const double (&w0)[P0], const double (&w1)[P1],
                                     const double (&w2)[P2]) {
    if (V == 0) {
        spread_fma(acc, w0, w1, w2);
    } else {
        double p[P1][P2];
#pragma unroll
        for (int b = 0; b < P1; ++b)
#pragma unroll
            for (int c = 0; c < P2; ++c) p[b][c] = w1[b] * w2[c];
#pragma unroll
        for (int a = 0; a < P0; ++a)
#pragma unroll
            for (int b = 0; b < P1; ++b)
#pragma unroll
                for (int c = 0; c < P2; ++c) acc[a][b][c] = fma(w0[a], p[b][c], acc[a][b][c]);
    }
}

template <int V>
__global__ void __launch_bounds__(32, 8) k(long iters, double* io) {
    __shared__ __align__(128) double wbuf[32][RW];
    const int lane = threadIdx.x, g0 = lane >> 4, g1 = (lane >> 2) & 3, g2 = lane & 3;
    for (int i = lane; i < 32 * RW; i += 32) (&wbuf[0][0])[i] = io[i % 64] + 1e-3 * i;
    __syncwarp();
    double acc[P0][P1][P2];
    for (int a = 0; a < P0; ++a) for (int b = 0; b < P1; ++b) for (int c = 0; c < P2; ++c) acc[a][b][c] = 0;
    const int nb = 32;
    if (V == 2) {
        // no shared-memory loads: two register weight sets, made opaque every point so the
        // w1*w2 products are recomputed (same FP64 instruction mix as the real loop)
        double a0[P0], a1[P1], a2[P2], b0[P0], b1[P1], b2[P2];
        load_w<T>(a0, a1, a2, &wbuf[0][0], g0, g1, g2);
        load_w<T>(b0, b1, b2, &wbuf[1][0], g0, g1, g2);
        for (long it = 0; it < iters; ++it) {
            for (int j = 0; j < nb; j += 2) {
#pragma unroll
                for (int i = 0; i < P1; ++i) asm volatile("" : "+d"(a1[i]), "+d"(a2[i]));
                spread_fma(acc, a0, a1, a2);
#pragma unroll
                for (int i = 0; i < P1; ++i) asm volatile("" : "+d"(b1[i]), "+d"(b2[i]));
                spread_fma(acc, b0, b1, b2);
            }
        }
    } else
    for (long it = 0; it < iters; ++it) {
        double a0[P0], a1[P1], a2[P2], b0[P0], b1[P1], b2[P2];
        load_w<T>(a0, a1, a2, &wbuf[0][0], g0, g1, g2);
        int j = 0;
        for (; j + 1 < nb; j += 2) {
            load_w<T>(b0, b1, b2, &wbuf[j + 1][0], g0, g1, g2);
            fmas<V>(acc, a0, a1, a2);
            load_w<T>(a0, a1, a2, &wbuf[j + 2 < nb ? j + 2 : j + 1][0], g0, g1, g2);
            fmas<V>(acc, b0, b1, b2);
        }
    }
    double s = 0;
    for (int a = 0; a < P0; ++a) for (int b = 0; b < P1; ++b) for (int c = 0; c < P2; ++c) s += acc[a][b][c];
    if (s == 1234.5) io[0] = s;
}
template <int V>
void run(int wpsm, int sms, double* io) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    long iters = 1000; int blocks = sms * wpsm;
    k<V><<<blocks, 32>>>(iters / 10, io);
    cudaEventRecord(e0); k<V><<<blocks, 32>>>(iters, io); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 1728 * 32 * iters * blocks;
    printf("variant=%d warps/SM=%2d  %.1f TF/s algorithmic (%.0f%%)\n", V, wpsm, fl / (ms * 1e-3) / 1e12, 100 * fl / (ms * 1e-3) / 1e12 / 36.7);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* io; cudaMalloc(&io, 4096 * 8); cudaMemset(io, 0, 4096 * 8);
    for (int w : {8, 16}) { run<0>(w, sms, io); run<1>(w, sms, io); run<2>(w, sms, io); }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
