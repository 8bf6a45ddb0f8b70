// q = 2 kernels for single-cell work items on the FP64 tensor cores (T = 12).
//
// A 2-D footprint is a 12 x 12 tile; per cell both directions are small GEMMs
// over the cell's points j (weights w0_j, w1_j from the plan-time table, rows of
// 24 doubles: [w0 | w1]):
//   spread : G[a][b] += sum_j (v_j w0_j[a]) w1_j[b]      M = a, N = b, K = points
//            4 DMMA (m8n8k4: 2 row tiles x 2 column tiles, 16 x 16 padded) per 4
//            points; C (8 doubles per lane) is flushed with RED.F64 at the end.
//   interp : U[j][a] = sum_b w1_j[b] G[a][b]           M = points, N = a, K = b
//            6 DMMA (2 column tiles x 3 k-steps) per 8 points; the columns are
//            permuted so lane quad q holds a in {3q, 3q+1, 3q+2}, and
//            out_j = sum_a w0_j[a] U[j][a] is 3 FMAs + a 2-step quad shuffle.
// Compared with the lane-per-point kernels (ak_kernels.cuh) this removes the
// per-point window polynomials (~180 FP64 ops, more than the 144 useful FMAs)
// and almost all instruction issue: the tensor pipe does the contraction.
// Padding costs 25% (interp) / 44% (spread) of the DMMA slots.
#pragma once
#include "ak_q3m.cuh"

namespace ak {

template <int B>
__global__ void __launch_bounds__(32, 16)
k_spread2c(const CellIdx* __restrict__ ci, const double* __restrict__ W, const int64_t* __restrict__ wshift,
           const WorkItem* __restrict__ items, const double* __restrict__ V, Strides vs,
           double* __restrict__ grids, const int64_t* __restrict__ canon_off, int nrhs, int n)
{
    constexpr int T = 12;
    constexpr int RW = 2 * T;
    static_assert(B % 4 == 0 && B <= 32, "batch");

    __shared__ __align__(128) double wbuf[2][B][RW];
    __shared__ __align__(16) CellIdx cib[3][B];
    __shared__ double vb[2][B];
    __shared__ __align__(8) uint64_t bar[2];

    // the RHS index runs fastest: the nrhs CTAs of one item share its weight rows in L2
    const WorkItem it = items[blockIdx.x / nrhs];
    const int r = blockIdx.x % nrhs;
    const int lane = threadIdx.x;
    const double* __restrict__ Vr = V + (int64_t)r * vs.rs;
    const int nbatch = (it.count + B - 1) / B;
    const double* __restrict__ Wit = W + (int64_t)(it.start - wshift[it.window]) * RW;
    const CellIdx* __restrict__ CIit = ci + (it.start - wshift[it.window]);

    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncwarp();
    if (lane == 0) tma_load_1d(&wbuf[0][0][0], Wit, (unsigned)(min(B, it.count) * RW * 8), &bar[0]);
    if (lane < min(B, it.count)) cp_async8(&cib[0][lane], CIit + lane);
    if (nbatch > 1 && lane < min(B, it.count - B)) cp_async8(&cib[1][lane], CIit + B + lane);
    cp_async_commit();
    cp_async_wait_all();
    __syncwarp();
    if (lane < min(B, it.count)) cp_async8(&vb[0][lane], Vr + (int64_t)cib[0][lane].idx * vs.is);
    cp_async_commit();

    const int rn = lane >> 2, kq = lane & 3;
    double C[2][2][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) C[mt][nt][0] = C[mt][nt][1] = 0.0;

    for (int bi = 0; bi < nbatch; ++bi) {
        const int s = bi & 1;
        const int off = bi * B;
        const int nb = min(B, it.count - off);
        cp_async_wait_all();
        mbar_wait(&bar[s], (bi >> 1) & 1);
        __syncwarp();
        if (bi + 1 < nbatch) {
            const int nb1 = min(B, it.count - off - B);
            if (lane == 0) {
                fence_proxy_async();
                tma_load_1d(&wbuf[s ^ 1][0][0], Wit + (int64_t)(off + B) * RW, (unsigned)(nb1 * RW * 8), &bar[s ^ 1]);
            }
            if (lane < nb1) cp_async8(&vb[s ^ 1][lane], Vr + (int64_t)cib[(bi + 1) % 3][lane].idx * vs.is);
        }
        if (bi + 2 < nbatch && lane < min(B, it.count - off - 2 * B))
            cp_async8(&cib[(bi + 2) % 3][lane], CIit + off + 2 * B + lane);
        cp_async_commit();
#pragma unroll 4
        for (int k0 = 0; k0 < nb; k0 += 4) {
            const int j = k0 + kq;
            const bool valid = j < nb;
            const double* w = wbuf[s][valid ? j : 0];
            const double v = valid ? vb[s][j] : 0.0;    // zero rows pad the last k-step
            const double a0 = v * w[rn];
            const double a1 = rn < 4 ? v * w[8 + rn] : 0.0;
            const double b0 = w[T + rn];
            const double b1 = rn < 4 ? w[T + 8 + rn] : 0.0;
            dmma_8x8x4(C[0][0][0], C[0][0][1], a0, b0);
            dmma_8x8x4(C[0][1][0], C[0][1][1], a0, b1);
            dmma_8x8x4(C[1][0][0], C[1][0][1], a1, b0);
            dmma_8x8x4(C[1][1][0], C[1][1][1], a1, b1);
        }
    }

    // lane holds G[a = rn + 8 mt][b = 2 kq + e + 8 nt]
    const int c0 = it.sc & 1023, c1 = (it.sc >> 10) & 1023;
    double* __restrict__ g = grids + (int64_t)nrhs * canon_off[it.window] + (int64_t)r * n * n;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
        const int a = rn + 8 * mt;
        if (a >= T) continue;
        double* row = g + (int64_t)wrap(c0 - (T / 2 - 1) + a, n) * n;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int b = 2 * kq + e + 8 * nt;
                if (b < T) red_add(row + wrap(c1 - (T / 2 - 1) + b, n), C[mt][nt][e]);
            }
    }
}

template <int B>
__global__ void __launch_bounds__(32, 16)
k_interp2c(const CellIdx* __restrict__ ci, const double* __restrict__ W, const int64_t* __restrict__ wshift,
           const WorkItem* __restrict__ items, const double* __restrict__ grids,
           const int64_t* __restrict__ canon_off, int nrhs, int n, const double* __restrict__ scale,
           double* __restrict__ out, Strides os, int atomic_out, int64_t wstride)
{
    constexpr int T = 12;
    constexpr int RW = 2 * T;
    static_assert(B % 8 == 0 && B <= 32, "batch");

    __shared__ __align__(128) double wbuf[2][B][RW];
    __shared__ __align__(16) CellIdx cib[2][B];
    __shared__ __align__(8) uint64_t bar[2];

    // the RHS index runs fastest: the nrhs CTAs of one item share its weight rows in L2
    const WorkItem it = items[blockIdx.x / nrhs];
    const int r = blockIdx.x % nrhs;
    const int lane = threadIdx.x;
    const int nbatch = (it.count + B - 1) / B;
    const double* __restrict__ Wit = W + (int64_t)(it.start - wshift[it.window]) * RW;
    const CellIdx* __restrict__ CIit = ci + (it.start - wshift[it.window]);

    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncwarp();
    if (lane == 0) tma_load_1d(&wbuf[0][0][0], Wit, (unsigned)(min(B, it.count) * RW * 8), &bar[0]);
    if (lane < min(B, it.count)) cp_async8(&cib[0][lane], CIit + lane);
    cp_async_commit();

    // B fragments: column n = lane/4 of tile t is a = 3 (n >> 1) + 2 t + (n & 1) (invalid: 2t + (n&1) = 3),
    // row k = lane%4 of k-step ks is b = 4 ks + k
    double gf[2][3];
    {
        const int c0 = it.sc & 1023, c1 = (it.sc >> 10) & 1023;
        const double* __restrict__ g = grids + (int64_t)nrhs * canon_off[it.window] + (int64_t)r * n * n;
        const int nn = lane >> 2, kk = lane & 3;
        int z[3];
#pragma unroll
        for (int ks = 0; ks < 3; ++ks) z[ks] = wrap(c1 - (T / 2 - 1) + 4 * ks + kk, n);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int i = 2 * t + (nn & 1);
            const int a = 3 * (nn >> 1) + i;
            const double* row = g + (int64_t)wrap(c0 - (T / 2 - 1) + (i < 3 ? a : 0), n) * n;
#pragma unroll
            for (int ks = 0; ks < 3; ++ks) gf[t][ks] = i < 3 ? __ldg(row + z[ks]) : 0.0;
        }
    }
    const double sc = scale[it.window];
    double* __restrict__ o = out + (int64_t)it.window * wstride + (int64_t)r * os.rs;
    const int pj = lane >> 2, q = lane & 3;

    for (int bi = 0; bi < nbatch; ++bi) {
        const int s = bi & 1;
        const int off = bi * B;
        const int nb = min(B, it.count - off);
        cp_async_wait_all();
        mbar_wait(&bar[s], (bi >> 1) & 1);
        __syncwarp();
        if (bi + 1 < nbatch) {
            const int nb1 = min(B, it.count - off - B);
            if (lane == 0) {
                fence_proxy_async();
                tma_load_1d(&wbuf[s ^ 1][0][0], Wit + (int64_t)(off + B) * RW, (unsigned)(nb1 * RW * 8), &bar[s ^ 1]);
            }
            if (lane < nb1) cp_async8(&cib[s ^ 1][lane], CIit + off + B + lane);
        }
        cp_async_commit();
#pragma unroll 2
        for (int k0 = 0; k0 < nb; k0 += 8) {
            const int cnt = min(8, nb - k0);
            const bool valid = pj < cnt;
            const double* w = wbuf[s][k0 + (valid ? pj : 0)];
            double C[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
            for (int ks = 0; ks < 3; ++ks) {
                const double af = valid ? w[T + 4 * ks + q] : 0.0;
                dmma_8x8x4(C[0][0], C[0][1], af, gf[0][ks]);
                dmma_8x8x4(C[1][0], C[1][1], af, gf[1][ks]);
            }
            // lane (pj, q) holds U[pj][3q + i], i = 2t + e (i = 3 is padding)
            double v = w[3 * q] * C[0][0];
            v = fma(w[3 * q + 1], C[0][1], v);
            v = fma(w[3 * q + 2], C[1][0], v);
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            if (q == 0 && valid) {
                double* dst = o + (int64_t)cib[s][k0 + pj].idx * os.is;
                if (atomic_out) red_add(dst, sc * v);
                else *dst = sc * v;
            }
        }
    }
}

}  // namespace ak
