// q = 2 single-cell kernels for many right-hand sides (RHS-minor data), T = 12.
//
// The per-RHS kernels (ak_q2c.cuh) run one CTA per (cell item, RHS): every RHS
// re-streams the item's weight rows (192 B per point) from L2, waits on its own
// TMA barriers and scatters 8-byte values into separate lines.  Here one CTA
// takes a cell item for 8 x NW right-hand sides: the NW warps share the
// double-buffered weight rows (one TMA stream per item), warp w owns RHS
// r0 + 8w .. r0 + 8w + 7, and the RHS values / results of a batch move between
// HBM and shared memory as whole lines (a point's RHS are contiguous).
// The per-RHS math is that of ak_q2c.cuh:
//   spread : G_r[a][b] += sum_j (v_rj w0_j[a]) w1_j[b]  -- 4 DMMA per 4 points per RHS,
//            the B operand (w1) shared by the warp's 8 RHS;
//   interp : U_r[j][a] = sum_b w1_j[b] G_r[a][b]        -- 6 DMMA per 8 points per RHS,
//            the A operand (w1 of the 8 points) shared; out = sum_a w0_j[a] U_r[j][a].
#pragma once
#include "ak_q2c.cuh"

namespace ak {

constexpr int Q2R_RPW = 8;   // right-hand sides per warp

template <int B, int NW>
struct alignas(128) Q2rSmem {
    double wbuf[2][B][24];
    double xb[2][B][Q2R_RPW * NW];   // spread: RHS values; interp: results
    CellIdx cib[3][B];
    uint64_t bar[2];
};

template <int B, int NW>
__global__ void __launch_bounds__(32 * NW, 12 / NW)
k_interp2r(const CellIdx* __restrict__ ci, const double* __restrict__ W, const int64_t* __restrict__ wshift,
           const WorkItem* __restrict__ items, const double* __restrict__ grids,
           const int64_t* __restrict__ canon_off, int nrhs, int n, const double* __restrict__ scale,
           double* __restrict__ out, Strides os, int atomic_out, int64_t wstride)
{
    constexpr int T = 12, RW = 2 * T, RPC = Q2R_RPW * NW;
    static_assert(B % 8 == 0 && B <= 32, "batch");
    __shared__ Q2rSmem<B, NW> sm;
    auto& wbuf = sm.wbuf;
    auto& ob = sm.xb;
    auto& cib = sm.cib;
    auto& bar = sm.bar;

    const WorkItem it = items[blockIdx.x];
    const int r0 = blockIdx.y * RPC;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nr = min(RPC, nrhs - r0);            // RHS of this CTA
    const int nbatch = (it.count + B - 1) / B;
    const double* __restrict__ Wit = W + (int64_t)(it.start - wshift[it.window]) * RW;
    const CellIdx* __restrict__ CIit = ci + (it.start - wshift[it.window]);

    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (tid == 0) tma_load_1d(&wbuf[0][0][0], Wit, (unsigned)(min(B, it.count) * RW * 8), &bar[0]);
    if (tid < min(B, it.count)) cp_async8(&cib[0][tid], CIit + tid);
    cp_async_commit();

    // B fragments of the warp's 8 footprints (mapping of k_interp2c)
    double gf[Q2R_RPW][2][3];
    {
        const int c0 = it.sc & 1023, c1 = (it.sc >> 10) & 1023;
        const int nn = lane >> 2, kk = lane & 3;
        int z[3];
#pragma unroll
        for (int ks = 0; ks < 3; ++ks) z[ks] = wrap(c1 - (T / 2 - 1) + 4 * ks + kk, n);
        int64_t rowoff[2];
        bool ok[2];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int i = 2 * t + (nn & 1);
            const int a = 3 * (nn >> 1) + i;
            ok[t] = i < 3;
            rowoff[t] = (int64_t)wrap(c0 - (T / 2 - 1) + (ok[t] ? a : 0), n) * n;
        }
        const int64_t n2 = (int64_t)n * n;
        const double* __restrict__ g0 = grids + (int64_t)nrhs * canon_off[it.window];
#pragma unroll
        for (int rr = 0; rr < Q2R_RPW; ++rr) {
            const int r = r0 + warp * Q2R_RPW + rr;
            const double* __restrict__ g = g0 + (int64_t)min(r, nrhs - 1) * n2;
#pragma unroll
            for (int t = 0; t < 2; ++t)
#pragma unroll
                for (int ks = 0; ks < 3; ++ks)
                    gf[rr][t][ks] = (ok[t] && r < nrhs) ? __ldg(g + rowoff[t] + z[ks]) : 0.0;
        }
    }
    const double sc = scale[it.window];
    double* __restrict__ o = out + (int64_t)it.window * wstride + (int64_t)r0 * os.rs;
    const int pj = lane >> 2, q = lane & 3;

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
            if (tid < nb1) cp_async8(&cib[(bi + 1) % 3][tid], CIit + off + B + tid);
        }
        cp_async_commit();
        for (int k0 = 0; k0 < nb; k0 += 8) {
            const int cnt = min(8, nb - k0);
            const bool valid = pj < cnt;
            const double* w = wbuf[s][k0 + (valid ? pj : 0)];
            double af[3];
#pragma unroll
            for (int ks = 0; ks < 3; ++ks) af[ks] = valid ? w[T + 4 * ks + q] : 0.0;
            const double w0a = w[3 * q], w0b = w[3 * q + 1], w0c = w[3 * q + 2];
#pragma unroll
            for (int rr = 0; rr < Q2R_RPW; ++rr) {
                double C[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
                for (int ks = 0; ks < 3; ++ks) {
                    dmma_8x8x4(C[0][0], C[0][1], af[ks], gf[rr][0][ks]);
                    dmma_8x8x4(C[1][0], C[1][1], af[ks], gf[rr][1][ks]);
                }
                double v = fma(w0c, C[1][0], fma(w0b, C[0][1], w0a * C[0][0]));
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                if (q == 0 && valid) ob[s][k0 + pj][warp * Q2R_RPW + rr] = sc * v;
            }
        }
        __syncthreads();
        // results of the batch: a point's nr values are contiguous (RHS-minor)
        for (int e = tid; e < nb * RPC; e += 32 * NW) {
            const int j = e / RPC, rr = e - j * RPC;
            if (rr < nr) {
                double* dst = o + (int64_t)cib[bi % 3][j].idx * os.is + (int64_t)rr * os.rs;
                if (atomic_out) red_add(dst, ob[s][j][rr]);
                else *dst = ob[s][j][rr];
            }
        }
    }
}

template <int B, int NW>
__global__ void __launch_bounds__(32 * NW, 12 / NW)
k_spread2r(const CellIdx* __restrict__ ci, const double* __restrict__ W, const int64_t* __restrict__ wshift,
           const WorkItem* __restrict__ items, const double* __restrict__ V, Strides vs,
           double* __restrict__ grids, const int64_t* __restrict__ canon_off, int nrhs, int n)
{
    constexpr int T = 12, RW = 2 * T, RPC = Q2R_RPW * NW;
    static_assert(B % 4 == 0 && B <= 32, "batch");
    __shared__ Q2rSmem<B, NW> sm;
    auto& wbuf = sm.wbuf;
    auto& vb = sm.xb;
    auto& cib = sm.cib;
    auto& bar = sm.bar;

    const WorkItem it = items[blockIdx.x];
    const int r0 = blockIdx.y * RPC;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nr = min(RPC, nrhs - r0);
    const int nbatch = (it.count + B - 1) / B;
    const double* __restrict__ Wit = W + (int64_t)(it.start - wshift[it.window]) * RW;
    const CellIdx* __restrict__ CIit = ci + (it.start - wshift[it.window]);
    const double* __restrict__ V0 = V + (int64_t)r0 * vs.rs;

    // RHS values of a batch (j < cnt points, the CTA's RPC RHS) by cp.async, zero padded
    auto gather = [&](int slot, int cslot, int cnt) {
        for (int e = tid; e < B * RPC; e += 32 * NW) {
            const int j = e / RPC, rr = e - j * RPC;
            if (j < cnt && rr < nr) cp_async8(&vb[slot][j][rr], V0 + (int64_t)cib[cslot][j].idx * vs.is + (int64_t)rr * vs.rs);
            else vb[slot][j][rr] = 0.0;
        }
    };

    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (tid == 0) tma_load_1d(&wbuf[0][0][0], Wit, (unsigned)(min(B, it.count) * RW * 8), &bar[0]);
    if (tid < min(B, it.count)) cp_async8(&cib[0][tid], CIit + tid);
    if (nbatch > 1 && tid < min(B, it.count - B)) cp_async8(&cib[1][tid], CIit + B + tid);
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    gather(0, 0, min(B, it.count));
    cp_async_commit();

    const int rn = lane >> 2, kq = lane & 3;
    double C[Q2R_RPW][2][2][2];
#pragma unroll
    for (int rr = 0; rr < Q2R_RPW; ++rr)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) C[rr][mt][nt][0] = C[rr][mt][nt][1] = 0.0;

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
            gather(s ^ 1, (bi + 1) % 3, nb1);
        }
        if (bi + 2 < nbatch && tid < min(B, it.count - off - 2 * B))
            cp_async8(&cib[(bi + 2) % 3][tid], CIit + off + 2 * B + tid);
        cp_async_commit();
#pragma unroll 2
        for (int k0 = 0; k0 < nb; k0 += 4) {
            const int j = k0 + kq;                       // rows past nb hold zero RHS values
            const double* w = wbuf[s][j < nb ? j : 0];
            const double x0 = w[rn], x1 = rn < 4 ? w[8 + rn] : 0.0;
            const double b0 = w[T + rn];
            const double b1 = rn < 4 ? w[T + 8 + rn] : 0.0;
            const double* vr = &vb[s][j][warp * Q2R_RPW];
#pragma unroll
            for (int rr = 0; rr < Q2R_RPW; ++rr) {
                const double v = vr[rr];
                const double a0 = v * x0, a1 = v * x1;
                dmma_8x8x4(C[rr][0][0][0], C[rr][0][0][1], a0, b0);
                dmma_8x8x4(C[rr][0][1][0], C[rr][0][1][1], a0, b1);
                dmma_8x8x4(C[rr][1][0][0], C[rr][1][0][1], a1, b0);
                dmma_8x8x4(C[rr][1][1][0], C[rr][1][1][1], a1, b1);
            }
        }
    }

    // lane holds G_r[a = rn + 8 mt][b = 2 kq + e + 8 nt] for its warp's 8 RHS
    const int c0 = it.sc & 1023, c1 = (it.sc >> 10) & 1023;
    const int64_t n2 = (int64_t)n * n;
#pragma unroll
    for (int rr = 0; rr < Q2R_RPW; ++rr) {
        const int r = r0 + warp * Q2R_RPW + rr;
        if (r >= nrhs) break;
        double* __restrict__ g = grids + (int64_t)nrhs * canon_off[it.window] + (int64_t)r * n2;
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
                    if (b < T) red_add(row + wrap(c1 - (T / 2 - 1) + b, n), C[rr][mt][nt][e]);
                }
        }
    }
}

}  // namespace ak
