// Ceiling of the q=3 spread inner loop: register-tiled FMAs with weights from shared memory.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2404_17344_b200/csrc/ak_q3.cuh"
using namespace ak;
template <int PAD_KB>
__global__ void __launch_bounds__(32, 8) k(long iters, double* io) {
    constexpr int T = 12, P0 = 6, P1 = 3, P2 = 3;
    __shared__ __align__(16) double wst[32][38];
    __shared__ double pad[PAD_KB * 128];
    const int lane = threadIdx.x, g0 = lane >> 4, g1 = (lane >> 2) & 3, g2 = lane & 3;
    for (int i = lane; i < 32 * 38; i += 32) (&wst[0][0])[i] = io[i % 64] + 1e-3 * i;
    pad[lane] = 0; __syncwarp();
    double acc[P0][P1][P2];
    for (int a = 0; a < P0; ++a) for (int b = 0; b < P1; ++b) for (int c = 0; c < P2; ++c) acc[a][b][c] = 0;
    for (long it = 0; it < iters; ++it) {
        double a0[P0], a1[P1], a2[P2], b0[P0], b1[P1], b2[P2];
        load_w<T>(a0, a1, a2, &wst[0][0], g0, g1, g2);
        for (int j = 0; j < 32; j += 2) {
            load_w<T>(b0, b1, b2, &wst[j + 1][0], g0, g1, g2);
            spread_fma(acc, a0, a1, a2);
            load_w<T>(a0, a1, a2, &wst[(j + 2) & 31][0], g0, g1, g2);
            spread_fma(acc, b0, b1, b2);
        }
    }
    double s = pad[lane];
    for (int a = 0; a < P0; ++a) for (int b = 0; b < P1; ++b) for (int c = 0; c < P2; ++c) s += acc[a][b][c];
    if (s == 1234.5) io[0] = s;
}
template <int PAD>
void run(int wpsm, int sms, double* io) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    long iters = 2000; int blocks = sms * wpsm;
    k<PAD><<<blocks, 32>>>(iters / 10, io);
    cudaEventRecord(e0); k<PAD><<<blocks, 32>>>(iters, io); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 1728 * 32 * iters * blocks;   // algorithmic: 1728 FMA per point, 32 points per iter
    printf("pad=%dKB warps/SM(launched)=%2d  %.1f TF/s algorithmic (%.0f%% of 36.7)\n", PAD, wpsm, fl / (ms * 1e-3) / 1e12,
           100 * fl / (ms * 1e-3) / 1e12 / 36.7);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* io; cudaMalloc(&io, 4096 * 8); cudaMemset(io, 0, 4096 * 8);
    for (int w : {4, 8, 16}) { run<1>(w, sms, io); }
    run<20>(8, sms, io);
    return 0;
}
