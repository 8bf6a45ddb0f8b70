// Spread inner-loop variants: load width / count, 2-point interleave.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2404_17344_b200/csrc/ak_q3.cuh"
using namespace ak;
// row layout for V4/V6: w0[12] | w1 groups of 4 (3 used) x4 | w2 groups of 4 x4  -> 44 doubles (+pad 4) = 48
template <int V>
__global__ void __launch_bounds__(32, 8) k(long iters, double* io) {
    constexpr int T = 12, P0 = 6, P1 = 3, P2 = 3;
    __shared__ __align__(16) double wst[32][48];
    const int lane = threadIdx.x, g0 = lane >> 4, g1 = (lane >> 2) & 3, g2 = lane & 3;
    for (int i = lane; i < 32 * 48; i += 32) (&wst[0][0])[i] = io[i % 64] + 1e-3 * i;
    __syncwarp();
    double acc[P0][P1][P2];
    for (int a = 0; a < P0; ++a) for (int b = 0; b < P1; ++b) for (int c = 0; c < P2; ++c) acc[a][b][c] = 0;
    for (long it = 0; it < iters; ++it) {
        if (V == 4) {
#pragma unroll 2
            for (int j = 0; j < 32; ++j) {
                const double2* row = reinterpret_cast<const double2*>(&wst[j][0]);
                double w0[6], w1[4], w2[4];
                for (int q = 0; q < 3; ++q) { double2 t = row[g0 * 3 + q]; w0[2 * q] = t.x; w0[2 * q + 1] = t.y; }
                for (int q = 0; q < 2; ++q) { double2 t = row[6 + g1 * 2 + q]; w1[2 * q] = t.x; w1[2 * q + 1] = t.y; }
                for (int q = 0; q < 2; ++q) { double2 t = row[14 + g2 * 2 + q]; w2[2 * q] = t.x; w2[2 * q + 1] = t.y; }
                for (int b = 0; b < P1; ++b) for (int c = 0; c < P2; ++c) {
                    const double p = w1[b] * w2[c];
                    for (int a = 0; a < P0; ++a) acc[a][b][c] = fma(w0[a], p, acc[a][b][c]);
                }
            }
        } else {
            // V6: two points per step, FMAs interleaved (acc += x0*p0 + ... two fma chains)
            for (int j = 0; j < 32; j += 2) {
                const double2* r0 = reinterpret_cast<const double2*>(&wst[j][0]);
                const double2* r1 = reinterpret_cast<const double2*>(&wst[j + 1][0]);
                double u0[6], u1[4], u2[4], v0[6], v1[4], v2[4];
                for (int q = 0; q < 3; ++q) { double2 t = r0[g0 * 3 + q]; u0[2 * q] = t.x; u0[2 * q + 1] = t.y; t = r1[g0 * 3 + q]; v0[2 * q] = t.x; v0[2 * q + 1] = t.y; }
                for (int q = 0; q < 2; ++q) { double2 t = r0[6 + g1 * 2 + q]; u1[2 * q] = t.x; u1[2 * q + 1] = t.y; t = r1[6 + g1 * 2 + q]; v1[2 * q] = t.x; v1[2 * q + 1] = t.y; }
                for (int q = 0; q < 2; ++q) { double2 t = r0[14 + g2 * 2 + q]; u2[2 * q] = t.x; u2[2 * q + 1] = t.y; t = r1[14 + g2 * 2 + q]; v2[2 * q] = t.x; v2[2 * q + 1] = t.y; }
                for (int b = 0; b < P1; ++b) for (int c = 0; c < P2; ++c) {
                    const double p = u1[b] * u2[c], pv = v1[b] * v2[c];
                    for (int a = 0; a < P0; ++a) acc[a][b][c] = fma(v0[a], pv, fma(u0[a], p, acc[a][b][c]));
                }
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
    for (int w : {8, 16}) { run<4>(w, sms, io); run<6>(w, sms, io); }
    return 0;
}
