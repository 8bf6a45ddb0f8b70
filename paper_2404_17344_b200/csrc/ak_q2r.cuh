// q = 2 single-cell kernels for many right-hand sides (RHS-minor data), T = 12.
//
// The per-RHS kernels (ak_q2c.cuh) run one CTA per (cell item, RHS): every RHS
// re-streams the item's weight rows (192 B per point) from L2, waits on its own
// TMA barriers and scatters 8-byte values into separate lines.  Here one CTA
// takes a cell item for 8 x NW right-hand sides: the NW warps share the
// double-buffered weight rows (one TMA stream per item), warp w owns RHS
// r0 + 8w .. r0 + 8w + 7, and the RHS values / results of a batch move between
// HBM and shared memory as whole lines (a point's RHS are contiguous).
// The math runs on RHS pairs (as the 3-D RHS-pair spread, ak_q3r.cuh), so the
// 12-wide tap axis that ak_q2c.cuh pads to 16 tiles exactly as 2 x 12 = 24:
//   spread : G_r[a][b] += sum_j (v_rj w0_j[a]) w1_j[b]; rows (r, a) of the pair = 3
//            m-tiles, columns b = 2 n-tiles (16, padded), K = points: 6 DMMA per 4
//            points per pair (8 for two single-RHS products), B (w1) shared by the pairs;
//   interp : U[j][(r, a)] = sum_b w1_j[b] G_r[a][b]; columns (r, a) of the pair = 3
//            n-tiles (no padding), K = b = 3 k-steps: 9 DMMA per 8 points per pair
//            (12 single-RHS); the columns are permuted so lane quad q holds
//            r = q >> 1, a = 6 (q & 1) + 0..5: out = 6 FMA + one quad shuffle.
#pragma once
#include "ak_q2c.cuh"

#ifndef AK_SPREAD2R_UNROLL
#define AK_SPREAD2R_UNROLL 2
#endif

namespace ak {

constexpr int Q2R_RPW = 8;   // right-hand sides per warp

// warps per SM the register allocation must allow: 16 (<= 128 registers): config-5
// interp 1.422 -> 1.347 ms per launch, spread 1.839 -> 1.819 ms; 12 (166 registers) before
// points per staged batch of the interpolation / spread (config 5: interpolation 16 / 24 /
// 32 -> 2.762 / 2.712 / 2.692 ms per step, spread 16 / 24 / 32 -> 1.875 / 1.842 / 1.818)
#ifndef AK_Q2R_INTERP_BATCH
#define AK_Q2R_INTERP_BATCH 32
#endif
#ifndef AK_Q2R_SPREAD_BATCH
#define AK_Q2R_SPREAD_BATCH 32
#endif
#ifndef AK_Q2R_MINW
#define AK_Q2R_MINW 16
#endif

template <int B, int NW>
struct alignas(128) Q2rSmem {
    double wbuf[2][B][24];
    double xb[2][B][Q2R_RPW * NW];   // spread: RHS values; interp: results
    CellIdx cib[3][B];
    uint64_t bar[2];
};

template <int B, int NW>
__global__ void __launch_bounds__(32 * NW, AK_Q2R_MINW / NW)
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

    // B fragments of the warp's 4 RHS pairs: lane (k = lane % 4, n = lane / 4) of n-tile t
    // holds G_r[a][b] with r = pair + (n >> 2), a = 6 ((n >> 1) & 1) + 2 t + (n & 1),
    // b = 4 ks + k (columns permuted: lane quad q of C holds r = q >> 1, a = 6 (q & 1) + 0..5)
    constexpr int NP = Q2R_RPW / 2;
    double gf[NP][3][3];
    {
        const int c0 = it.sc & 1023, c1 = (it.sc >> 10) & 1023;
        const int nn = lane >> 2, kk = lane & 3;
        const int rl = nn >> 2, ah = 6 * ((nn >> 1) & 1), ae = nn & 1;
        int z[3];
#pragma unroll
        for (int ks = 0; ks < 3; ++ks) z[ks] = wrap(c1 - (T / 2 - 1) + 4 * ks + kk, n);
        int64_t rowoff[3];
#pragma unroll
        for (int t = 0; t < 3; ++t) rowoff[t] = (int64_t)wrap(c0 - (T / 2 - 1) + ah + 2 * t + ae, n) * n;
        const int64_t n2 = (int64_t)n * n;
        const double* __restrict__ g0 = grids + (int64_t)nrhs * canon_off[it.window];
#pragma unroll
        for (int pr = 0; pr < NP; ++pr) {
            const int r = r0 + warp * Q2R_RPW + 2 * pr + rl;
            const double* __restrict__ g = g0 + (int64_t)min(r, nrhs - 1) * n2;
#pragma unroll
            for (int t = 0; t < 3; ++t)
#pragma unroll
                for (int ks = 0; ks < 3; ++ks) gf[pr][t][ks] = r < nrhs ? __ldg(g + rowoff[t] + z[ks]) : 0.0;
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
            double w0[6];
#pragma unroll
            for (int i = 0; i < 6; ++i) w0[i] = w[6 * (q & 1) + i];
#pragma unroll
            for (int pr = 0; pr < NP; ++pr) {
                double C[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
                for (int ks = 0; ks < 3; ++ks)
#pragma unroll
                    for (int t = 0; t < 3; ++t) dmma_8x8x4(C[t][0], C[t][1], af[ks], gf[pr][t][ks]);
                // lane (pj, q): columns a = 6 (q & 1) + 2 t + e of RHS 2 pr + (q >> 1)
                double v = w0[0] * C[0][0];
                v = fma(w0[1], C[0][1], v);
                v = fma(w0[2], C[1][0], v);
                v = fma(w0[3], C[1][1], v);
                v = fma(w0[4], C[2][0], v);
                v = fma(w0[5], C[2][1], v);
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                if ((q & 1) == 0 && valid) ob[s][k0 + pj][warp * Q2R_RPW + 2 * pr + (q >> 1)] = sc * v;
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
__global__ void __launch_bounds__(32 * NW, AK_Q2R_MINW / NW)
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

    // A fragments: row (r, a) = divmod(8 mt + lane / 4, 12) of the pair, k = lane % 4;
    // B: k = lane % 4, column b = 8 nt + lane / 4 (b >= 12 padding)
    constexpr int NP = Q2R_RPW / 2;
    const int rn = lane >> 2, kq = lane & 3;
    int ar[3], aa[3];
#pragma unroll
    for (int mt = 0; mt < 3; ++mt) {
        const int row = 8 * mt + rn;
        ar[mt] = row / T;
        aa[mt] = row - ar[mt] * T;
    }
    double C[NP][3][2][2];
#pragma unroll
    for (int pr = 0; pr < NP; ++pr)
#pragma unroll
        for (int mt = 0; mt < 3; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) C[pr][mt][nt][0] = C[pr][mt][nt][1] = 0.0;

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
AK_UNROLL(AK_SPREAD2R_UNROLL)
        for (int k0 = 0; k0 < nb; k0 += 4) {
            const int j = k0 + kq;                       // rows past nb hold zero RHS values
            const double* w = wbuf[s][j < nb ? j : 0];
            double x[3];
#pragma unroll
            for (int mt = 0; mt < 3; ++mt) x[mt] = w[aa[mt]];
            const double b0 = w[T + rn];
            const double b1 = rn < 4 ? w[T + 8 + rn] : 0.0;
            const double* vr = &vb[s][j][warp * Q2R_RPW];
#pragma unroll
            for (int pr = 0; pr < NP; ++pr) {
#pragma unroll
                for (int mt = 0; mt < 3; ++mt) {
                    const double a = vr[2 * pr + ar[mt]] * x[mt];
                    dmma_8x8x4(C[pr][mt][0][0], C[pr][mt][0][1], a, b0);
                    dmma_8x8x4(C[pr][mt][1][0], C[pr][mt][1][1], a, b1);
                }
            }
        }
    }

    // lane holds G_r[a][b] for (r, a) = divmod(8 mt + lane / 4, 12) of each pair,
    // b = 8 nt + 2 (lane % 4) + e
    const int c0 = it.sc & 1023, c1 = (it.sc >> 10) & 1023;
    const int64_t n2 = (int64_t)n * n;
#pragma unroll
    for (int pr = 0; pr < NP; ++pr)
#pragma unroll
        for (int mt = 0; mt < 3; ++mt) {
            const int r = r0 + warp * Q2R_RPW + 2 * pr + ar[mt];
            if (r >= nrhs) continue;
            double* row = grids + (int64_t)nrhs * canon_off[it.window] + (int64_t)r * n2 +
                          (int64_t)wrap(c0 - (T / 2 - 1) + aa[mt], n) * n;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int b = 2 * kq + e + 8 * nt;
                    if (b < T) red_add(row + wrap(c1 - (T / 2 - 1) + b, n), C[pr][mt][nt][e]);
                }
        }
}

}  // namespace ak
