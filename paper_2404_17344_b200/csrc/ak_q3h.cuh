// q = 3 single-cell spread of one right-hand side, split between the FP64 tensor
// cores and the FP64 FMA pipe (dense 3-D windows: config 4).
//
// For one cell and one RHS the spread (nufft.py:231-254) is the GEMM
//   G[a][(b, c)] += sum_j (w0_j[a]) (v_j w1_j[b] w2_j[c])      M = 12, N = 144, K = points.
// mma.sync m8n8k4 tiles M in 8s, so rows a = 0..7 go to the tensor cores (one m-tile,
// no padding) and the 4 rows a = 8..11 are done with DFMAs on the same B operand
// values the lane already holds for the DMMA:
//   CTA = 2 warps = one (item, RHS) unit; warp h owns the columns b in [6h, 6h + 6)
//   (72 columns = 9 n-tiles).  Lane group g = lane / 4 owns a 3 x 3 block of them
//   (b = 6h + 3 (g / 4) + jb, c = 3 (g % 4) + jc, tile j = 3 jb + jc), lane kk = lane % 4
//   is the point of the k-step: its 9 B values v w1[b] w2[c] (3 + 9 DMUL) feed 9 DMMA
//   (rows a < 8, A = w0[lane / 4]) and 36 DFMA (rows a = 8..11 of its own point into
//   per-lane accumulators, summed over the 4 lanes of a group at the flush).
// FP64 pipe slots per 4 points and warp: 9 DMMA (= 72 DFMA slots) + 36 DFMA + 12 DMUL
// = 120 for 108 useful: 90%, against 54 DFMA + 12 DMUL per point and lane (82%) for
// the register-tiled DFMA kernel (k_spread3c), whose one-RHS output rows would pad
// 12 -> 16 on the tensor cores alone (70%).
#pragma once
#include "ak_q3r.cuh"

namespace ak {

// CTAs (2 warps) per SM the register allocation must allow (5: <= 168 registers, the
// per-SMSP register file at 10 warps/SM); points per staged batch.  Final: 1.374 ms per
// config-4 launch (0.686 of the FP64 peak).  Measured on config 4 (B200,
// tools/gpu_var.sh), with 32-point batches and unroll 2: 5 CTAs 1.432 ms, 4 CTAs (198
// registers) 1.529, 6 CTAs 1.459;
// 64-point batches 1.445; 3 warps per CTA (2 b values per lane group, 128 registers,
// 15 warps/SM) 1.631; operands of the next k-step loaded ahead in registers: 1.605
// (spills at 168 registers) / 1.619 (198 registers, 8 warps/SM); rows 8..11 kept
// XOR-rotated per lane (acc2[j] = row 8 + (j ^ kk): a select-free reduce-scatter, but
// lane-dependent w0 loads in the loop): 1.470; rows 8..11 summed through shared memory
// instead of shuffles (one more CTA barrier per item): 1.400 vs 1.371.
#ifndef AK_SPREAD3H_MINB
#define AK_SPREAD3H_MINB 5
#endif
#ifndef AK_SPREAD3H_BATCH
#define AK_SPREAD3H_BATCH 48
#endif
#ifndef AK_SPREAD3H_UNROLL
#define AK_SPREAD3H_UNROLL 1
#endif
#ifndef AK_SPREAD3H_WARPS
#define AK_SPREAD3H_WARPS 2
#endif
template <int B, int WC>
__global__ void __launch_bounds__(32 * WC, AK_SPREAD3H_MINB)
k_spread3h(const CellIdx* __restrict__ ci, const double* __restrict__ W, const int64_t* __restrict__ wshift,
           const WorkItem* __restrict__ items, const double* __restrict__ V, Strides vs,
           double* __restrict__ grids, const int64_t* __restrict__ canon_off, int nrhs, int n)
{
    constexpr int T = 12, RW = 3 * T;
    constexpr int NB = 6 / WC, NT = 3 * NB;   // b values per lane group, n-tiles per warp
    constexpr int NTH = 32 * WC;
    static_assert(WC == 2 || WC == 3, "2 or 3 warps");
    static_assert(B % 4 == 0 && B <= NTH, "batch");
    __shared__ Spread3cSmem<B> sm;
    auto& wbuf = sm.wbuf;
    auto& vb = sm.vb;
    auto& bar = sm.bar;
    auto& cib = sm.cib;

    const WorkItem it = items[blockIdx.x / nrhs];
    const int r = blockIdx.x % nrhs;            // RHS fastest: the R CTAs of an item share its rows in L2
    const int tid = threadIdx.x, h = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, kk = lane & 3;
    const double* __restrict__ Vr = V + (int64_t)r * vs.rs;
    const int nbatch = (it.count + B - 1) / B;
    const double* __restrict__ Wit = W + (int64_t)(it.start - wshift[it.window]) * RW;
    const CellIdx* __restrict__ CIit = ci + (it.start - wshift[it.window]);

    // rows past a batch's end hold finite weights (zeroed here, then earlier batches)
    // and zero RHS values, so the k-step loop needs no bounds checks
    // (only rows no batch of this item fills: buffer 0 past the item's count, buffer 1
    // past count - B when it is used; later batches leave finite earlier rows behind)
    {
        const int z0 = min(B, it.count), z1 = it.count > B ? min(B, it.count - B) : B;
        for (int e = tid; e < (B - z0) * RW; e += NTH) wbuf[0][z0 + e / RW][e % RW] = 0.0;
        for (int e = tid; e < (B - z1) * RW; e += NTH) wbuf[1][z1 + e / RW][e % RW] = 0.0;
    }
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) tma_load_1d(&wbuf[0][0][0], Wit, (unsigned)(min(B, it.count) * RW * 8), &bar[0]);
    if (tid < min(B, it.count)) cp_async8(&cib[0][tid], CIit + tid);
    if (nbatch > 1 && tid < min(B, it.count - B)) cp_async8(&cib[1][tid], CIit + B + tid);
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    if (tid < min(B, it.count)) cp_async8(&vb[0][tid], Vr + (int64_t)cib[0][tid].idx * vs.is);
    else if (tid < B) vb[0][tid] = 0.0;
    cp_async_commit();

    // this lane's weight offsets: w1 at b0 .. b0 + NB - 1, w2 at c0 .. c0 + 2 (row layout w0 | w1 | w2)
    const int b0 = T + 2 * NB * h + NB * (g >> 2), c0 = 2 * T + 3 * (g & 3);
    double acc[NT][2], acc2[4][NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) {
        acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
        for (int a = 0; a < 4; ++a) acc2[a][j] = 0.0;
    }

    for (int bi = 0; bi < nbatch; ++bi) {
        const int s = bi & 1;
        const int off = bi * B;
        const int nb = min(B, it.count - off);
        cp_async_wait_all();
        mbar_wait(&bar[s], (bi >> 1) & 1);
        __syncthreads();
        if (bi + 1 < nbatch) {
            const int nb1 = min(B, it.count - off - B);
            if (tid == 0) {
                fence_proxy_async();
                tma_load_1d(&wbuf[s ^ 1][0][0], Wit + (int64_t)(off + B) * RW, (unsigned)(nb1 * RW * 8), &bar[s ^ 1]);
            }
            if (tid < nb1) cp_async8(&vb[s ^ 1][tid], Vr + (int64_t)cib[(bi + 1) % 3][tid].idx * vs.is);
            else if (tid < B) vb[s ^ 1][tid] = 0.0;
        }
        if (bi + 2 < nbatch && tid < min(B, it.count - off - 2 * B))
            cp_async8(&cib[(bi + 2) % 3][tid], CIit + off + 2 * B + tid);
        cp_async_commit();
        AK_UNROLL(AK_SPREAD3H_UNROLL)
        for (int k0 = 0; k0 < nb; k0 += 4) {
            const int j = k0 + kk;   // < B; rows past nb contribute zero (v = 0)
            const double* w = wbuf[s][j];
            const double v = vb[s][j];
            double vw1[NB], w2[3], w0h[4], bf[NT];
#pragma unroll
            for (int x = 0; x < NB; ++x) vw1[x] = v * w[b0 + x];
#pragma unroll
            for (int x = 0; x < 3; ++x) w2[x] = w[c0 + x];
#pragma unroll
            for (int a = 0; a < 4; ++a) w0h[a] = w[8 + a];
            const double af = w[g];
#pragma unroll
            for (int t = 0; t < NT; ++t) bf[t] = vw1[t / 3] * w2[t % 3];
#pragma unroll
            for (int t = 0; t < NT; ++t) dmma_8x8x4(acc[t][0], acc[t][1], af, bf[t]);
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int t = 0; t < NT; ++t) acc2[a][t] = fma(w0h[a], bf[t], acc2[a][t]);
        }
    }

    // flush.  DMMA tiles: lane holds D[a = g][col 2 kk + e] of tile t, i.e. column block
    // g' = 2 kk + e: (b, c) = (6h + 3 (g' / 4) + t / 3, 3 (g' % 4) + t % 3).
    // DFMA rows: summed over the group's 4 lanes; lane kk adds row a = 8 + kk.
    const int cc0 = it.sc & 1023, cc1 = (it.sc >> 10) & 1023, cc2 = (it.sc >> 20) & 1023;
    const int o0 = cc0 - (T / 2 - 1), o1 = cc1 - (T / 2 - 1), o2 = cc2 - (T / 2 - 1);
    double* __restrict__ gr = grids + (int64_t)nrhs * canon_off[it.window] + (int64_t)r * n * n * n;
    const bool inside = o0 >= 0 && o0 + T <= n && o1 >= 0 && o1 + T <= n && o2 >= 0 && o2 + T <= n;
    auto X = [&](int o, int i) { return inside ? o + i : wrap(o + i, n); };
    const int64_t nn = (int64_t)n * n;
    auto flush9 = [&](int a, int gg, const double (&v)[NT]) {
        double* plane = gr + (int64_t)X(o0, a) * nn;
        int xb[NB], xc[3];
#pragma unroll
        for (int x = 0; x < NB; ++x) xb[x] = X(o1, 2 * NB * h + NB * (gg >> 2) + x) * n;
#pragma unroll
        for (int x = 0; x < 3; ++x) xc[x] = X(o2, 3 * (gg & 3) + x);
#pragma unroll
        for (int t = 0; t < NT; ++t) red_add(plane + xb[t / 3] + xc[t % 3], v[t]);
    };
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        double v[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) v[t] = acc[t][e];
        flush9(g, 2 * kk + e, v);
    }
    // rows 8..11: reduce-scatter over the group's 4 lanes (lane kk ends with row 8 + kk)
    const bool hi2 = (kk & 2) != 0, hi1 = (kk & 1) != 0;
    double keep[2][NT], mine[NT];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const double send = hi2 ? acc2[x][t] : acc2[2 + x][t];
            keep[x][t] = (hi2 ? acc2[2 + x][t] : acc2[x][t]) + __shfl_xor_sync(0xffffffffu, send, 2);
        }
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        const double send = hi1 ? keep[0][t] : keep[1][t];
        mine[t] = (hi1 ? keep[1][t] : keep[0][t]) + __shfl_xor_sync(0xffffffffu, send, 1);
    }
    flush9(8 + kk, g, mine);
}

}  // namespace ak
