// q = 3 single-cell spread for pairs of right-hand sides on the FP64 tensor cores.
//
// For one cell and two RHS r in {0, 1} the spread (nufft.py:231-254, one grid per
// RHS) is the GEMM
//   G[(r, a)][(b, c)] += sum_j (v_rj w0_j[a]) (w1_j[b] w2_j[c])     M = 24, N = 144, K = points
// whose output rows (r, a) tile the m8n8k4 fragments exactly (24 = 3 x 8), and whose
// B operand (the w1 (x) w2 products) is shared by both RHS.  With one RHS the rows
// would be a alone (12 -> padded to 16) and the DFMA register tile (k_spread3c) wins;
// with two, 27 DMMA per lane per 4 points carry the work at ~95% useful FP64 slots
// (products and v w0 factors included) against ~82% for the DFMA tile.
// CTA = 2 warps = one (item, RHS pair); warp w owns n-tiles 9w .. 9w + 8 (all 3
// m-tiles: 54 accumulator doubles per lane, as the DFMA tile).  Weight rows are
// double-buffered by TMA bulk copies as in k_spread3c; the 2 x B RHS values are
// gathered by cp.async.
#pragma once
#include "ak_q3c.cuh"

// k-step loop unroll (config 5: unroll 2 43.92 ms, 1 43.43) and points per batch
#ifndef AK_SPREAD3R_UNROLL
#define AK_SPREAD3R_UNROLL 1
#endif
#ifndef AK_SPREAD3R_BATCH
#define AK_SPREAD3R_BATCH 48   // config 5: 32 -> 43.43 ms, 48 -> 43.14, 64 -> 44.58
#endif

namespace ak {

template <int B>
struct alignas(128) Spread3rSmem {
    double wbuf[2][B][36];
    double vb[2][2][B];
    CellIdx cib[3][B];
    uint64_t bar[2];
};

// CTAs per SM (2 warps each): 5 -> 167 registers, 10 warps/SM: config 5 spread
// 48.03 -> 43.95 ms; 4 (190 registers): 48.03; 6 (157): 57.8 (tools/gpu_var_cfg.sh)
#ifndef AK_SPREAD3R_MINB
#define AK_SPREAD3R_MINB 5
#endif
template <int B>
__global__ void __launch_bounds__(64, AK_SPREAD3R_MINB)
k_spread3r(const CellIdx* __restrict__ ci, const double* __restrict__ W, const int64_t* __restrict__ wshift,
           const WorkItem* __restrict__ items, const double* __restrict__ V, Strides vs,
           double* __restrict__ grids, const int64_t* __restrict__ canon_off, int nrhs, int n)
{
    constexpr int T = 12, RW = 3 * T, NT = 9;   // n-tiles per warp
    static_assert(B % 4 == 0 && B <= 64, "batch");
    __shared__ Spread3rSmem<B> sm;
    auto& wbuf = sm.wbuf;
    auto& vb = sm.vb;
    auto& cib = sm.cib;
    auto& bar = sm.bar;

    const int npair = nrhs / 2;
    const WorkItem it = items[blockIdx.x / npair];
    const int pr = blockIdx.x % npair;          // RHS pair (fastest: pairs of an item share its rows in L2)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int lr = lane >> 2, kk = lane & 3;
    const double* __restrict__ V0 = V + (int64_t)(2 * pr) * vs.rs;
    const int nbatch = (it.count + B - 1) / B;
    const double* __restrict__ Wit = W + (int64_t)(it.start - wshift[it.window]) * RW;
    const CellIdx* __restrict__ CIit = ci + (it.start - wshift[it.window]);

    // rows past a batch's end hold finite weights (zeroed here, then earlier batches)
    // and zero RHS values, so the k-step loop needs no bounds checks
    // (only rows no batch of this item fills: buffer 0 past the item's count, buffer 1
    // past count - B when it is used; later batches leave finite earlier rows behind)
    {
        const int z0 = min(B, it.count), z1 = it.count > B ? min(B, it.count - B) : B;
        for (int e = tid; e < (B - z0) * RW; e += 64) wbuf[0][z0 + e / RW][e % RW] = 0.0;
        for (int e = tid; e < (B - z1) * RW; e += 64) wbuf[1][z1 + e / RW][e % RW] = 0.0;
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
    for (int e = tid; e < 2 * B; e += 64) {
        const int r = e / B, j = e - r * B;
        if (j < min(B, it.count)) cp_async8(&vb[0][r][j], V0 + (int64_t)r * vs.rs + (int64_t)cib[0][j].idx * vs.is);
        else vb[0][r][j] = 0.0;
    }
    cp_async_commit();

    // fragment coordinates: A rows (r, a) of m-tile i, B columns (b, c) of n-tile t
    int ar[3], aa[3], bb[NT], bc[NT];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const int row = 8 * i + lr;
        ar[i] = row / T;
        aa[i] = row - ar[i] * T;
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        const int col = 8 * (NT * warp + t) + lr;
        bb[t] = col / T;
        bc[t] = col - bb[t] * T;
    }
    double acc[3][NT][2];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int t = 0; t < NT; ++t) acc[i][t][0] = acc[i][t][1] = 0.0;

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
            for (int e = tid; e < 2 * B; e += 64) {
                const int r = e / B, j = e - r * B;
                if (j < nb1) cp_async8(&vb[s ^ 1][r][j], V0 + (int64_t)r * vs.rs + (int64_t)cib[(bi + 1) % 3][j].idx * vs.is);
                else vb[s ^ 1][r][j] = 0.0;
            }
        }
        if (bi + 2 < nbatch && tid < min(B, it.count - off - 2 * B))
            cp_async8(&cib[(bi + 2) % 3][tid], CIit + off + 2 * B + tid);
        cp_async_commit();
AK_UNROLL(AK_SPREAD3R_UNROLL)
        for (int k0 = 0; k0 < nb; k0 += 4) {
            const int j = k0 + kk;   // < B; rows past nb contribute zero (v = 0)
            const double* w = wbuf[s][j];
            double af[3], bf[NT];
#pragma unroll
            for (int i = 0; i < 3; ++i) af[i] = vb[s][ar[i]][j] * w[aa[i]];
#pragma unroll
            for (int t = 0; t < NT; ++t) bf[t] = w[T + bb[t]] * w[2 * T + bc[t]];
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int t = 0; t < NT; ++t) dmma_8x8x4(acc[i][t][0], acc[i][t][1], af[i], bf[t]);
        }
    }

    // flush: lane holds C[row = 8 i + lr][col = 8 tile + 2 kk + e] -> grid of RHS 2 pr + r
    const int c0 = it.sc & 1023, c1 = (it.sc >> 10) & 1023, c2 = (it.sc >> 20) & 1023;
    const int o0 = c0 - (T / 2 - 1), o1 = c1 - (T / 2 - 1), o2 = c2 - (T / 2 - 1);
    const int64_t n3 = (int64_t)n * n * n;
    double* __restrict__ g0 = grids + (int64_t)nrhs * canon_off[it.window] + (int64_t)(2 * pr) * n3;
    const bool inside = o0 >= 0 && o0 + T <= n && o1 >= 0 && o1 + T <= n && o2 >= 0 && o2 + T <= n;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        double* gr = g0 + ar[i] * n3;
        const int x0 = inside ? o0 + aa[i] : wrap(o0 + aa[i], n);
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = 8 * (NT * warp + t) + 2 * kk + e;
                const int b = col / T, c = col - (col / T) * T;
                const int x1 = inside ? o1 + b : wrap(o1 + b, n);
                const int x2 = inside ? o2 + c : wrap(o2 + c, n);
                red_add(gr + ((int64_t)x0 * n + x1) * n + x2, acc[i][t][e]);
            }
    }
}

}  // namespace ak
