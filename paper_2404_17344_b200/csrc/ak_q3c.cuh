// q = 3 kernels for single-cell work items (supercell edge S = 1).
//
// When cells are densely populated (config 4: 395 points per occupied cell on
// average) every work item can be one cell (or a chunk of one): the warp's
// register tile IS the item's footprint, so there is no shared region tile, no
// cell-run bookkeeping, no shared-memory flushes:
//   spread : register-tiled FMAs over all points of the item, then 54 RED.F64
//            per lane straight from registers to the grid;
//   interp : the footprint fragments are loaded once per item from the grid
//            (L2) and every batch is processed in groups of 8 points on the
//            FP64 tensor cores (ak_q3m.cuh).
// Shared memory shrinks to the double-buffered weight rows, which allows more
// warps per SM.  The plan picks these kernels when the mean occupancy of the
// occupied cells is high (ak_lib.cu: geom_build).
#pragma once
#include "ak_q3m.cuh"

// group loop of the single-cell interpolation: not unrolled (config 4: unroll 2 / 4
// 1.266 / 1.257 vs 1.255 ms; config 5 +1.4% / +0.6%).  Each group's tail (w1 . s,
// quad shuffles, output: ~30% of the stall samples) finished inside the next group's
// DMMA stream: 1.306 ms (176-byte spill at 168 registers), 1.374 at 200 registers,
// 1.423 at 184 -- the other warps already cover it.  Unmasked groups over zero-
// initialised weight buffers (as the spreads): 1.231 -> 1.270 ms, config 5 +3.3%.
#ifndef AK_INTERP3C_UNROLL
#define AK_INTERP3C_UNROLL 1
#endif
#ifndef AK_INTERP3C_BATCH
#define AK_INTERP3C_BATCH 16   // weight rows per batch: config 4 interp 32 -> 1.255 ms, 24 -> 1.236, 16 -> 1.231, 8 -> 1.363; config 5 -0.9% at 16
#endif

namespace ak {

// Register cap of the single-cell spread (config 4, B200, tools/gpu_var.sh): 196 registers
// under __maxnreg__(208), no spills: 1.523 ms; cap 224 (212 used): 1.541; 192: 1.557;
// 240 (__launch_bounds__(32, 8)): 1.569.  A single weight set in registers (no
// double buffering) allows 168 registers but loses: 1.594 ms.
#ifndef AK_SPREAD3C_BOUNDS
#define AK_SPREAD3C_BOUNDS __maxnreg__(208)
#endif
template <int B>
struct alignas(128) Spread3cSmem {
    double wbuf[2][B][36];
    CellIdx cib[3][B];
    double vb[2][B];
    uint64_t bar[2];
};

// One (item, RHS) unit of the single-cell spread (the body of k_spread3c).  A = active
// taps on axis 0: 12, or 10 for a zero-padded 10-tap window (cutoff 5: the lane tile
// skips the zero taps 0 and 11, 5 x 3 x 3 instead of 6 x 3 x 3 accumulators).
template <int B, int A = 12>
__device__ __forceinline__ void spread3c_unit(Spread3cSmem<B>& sm, int unit, const CellIdx* __restrict__ ci, const double* __restrict__ W, const int64_t* __restrict__ wshift,
           const WorkItem* __restrict__ items, const double* __restrict__ V, Strides vs,
           double* __restrict__ grids, const int64_t* __restrict__ canon_off, int nrhs, int n)
{
    constexpr int T = 12;
    using LN = Q3Lanes<T>;
    constexpr int P0 = A / 2, P1 = LN::P1, P2 = LN::P2, AO = (T - A) / 2;
    constexpr int RW = 3 * T;
    static_assert(B <= 32, "batch");

    auto& wbuf = sm.wbuf;
    auto& cib = sm.cib;
    auto& vb = sm.vb;
    auto& bar = sm.bar;

    // the RHS index runs fastest: the nrhs CTAs of one item share its weight rows in L2
    const WorkItem it = items[unit / nrhs];
    const int r = unit % nrhs;
    const int lane = threadIdx.x;
    const int g0 = lane >> 4, g1 = (lane >> 2) & 3, g2 = lane & 3;
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

    double acc[P0][P1][P2];
#pragma unroll
    for (int a = 0; a < P0; ++a)
#pragma unroll
        for (int b = 0; b < P1; ++b)
#pragma unroll
            for (int c = 0; c < P2; ++c) acc[a][b][c] = 0.0;

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
        __syncwarp();
        // v folded into the per-point products in the FMA loop (3 DMUL per point and
        // lane) instead of a per-batch staging pass over the w0 rows
        double a0[P0], a1[P1], a2[P2], b0[P0], b1[P1], b2[P2], av, bv;
        auto load = [&](double (&w0)[P0], double (&w1)[P1], double (&w2)[P2], const double* row) {
#pragma unroll
            for (int a = 0; a < P0; ++a) w0[a] = row[AO + g0 * P0 + a];
#pragma unroll
            for (int b = 0; b < P1; ++b) w1[b] = row[T + g1 * P1 + b];
#pragma unroll
            for (int c = 0; c < P2; ++c) w2[c] = row[2 * T + g2 * P2 + c];
        };
        load(a0, a1, a2, &wbuf[s][0][0]);
        av = vb[s][0];
        int j = 0;
        for (; j + 1 < nb; j += 2) {
            load(b0, b1, b2, &wbuf[s][j + 1][0]);
            bv = vb[s][j + 1];
            spread_fma_v(acc, a0, a1, a2, av);
            const int jn = j + 2 < nb ? j + 2 : j + 1;
            load(a0, a1, a2, &wbuf[s][jn][0]);
            av = vb[s][jn];
            spread_fma_v(acc, b0, b1, b2, bv);
        }
        if (j < nb) spread_fma_v(acc, a0, a1, a2, av);
        __syncwarp();
    }

    const int c0 = it.sc & 1023, c1 = (it.sc >> 10) & 1023, c2 = (it.sc >> 20) & 1023;
    double* __restrict__ g = grids + (int64_t)nrhs * canon_off[it.window] + (int64_t)r * n * n * n;
    const int o0 = c0 - (T / 2 - 1), o1 = c1 - (T / 2 - 1), o2 = c2 - (T / 2 - 1);
    if (o0 >= 0 && o0 + T <= n && o1 >= 0 && o1 + T <= n && o2 >= 0 && o2 + T <= n) {
        // footprint inside the grid (no periodic wrap): one base pointer, constant strides
        const int64_t nn = (int64_t)n * n;
        double* __restrict__ base = g + (int64_t)(o0 + AO + g0 * P0) * nn + (int64_t)(o1 + g1 * P1) * n + o2 + g2 * P2;
#pragma unroll
        for (int a = 0; a < P0; ++a)
#pragma unroll
            for (int b = 0; b < P1; ++b)
#pragma unroll
                for (int c = 0; c < P2; ++c) red_add(base + a * nn + b * n + c, acc[a][b][c]);
        return;
    }
    {
        // flush the register tile straight to the grid (a shared-memory staged, row-
        // coalesced flush measured 3% slower on B200)
        int x0[P0], x1[P1], x2[P2];
#pragma unroll
        for (int a = 0; a < P0; ++a) x0[a] = wrap(c0 - (T / 2 - 1) + AO + g0 * P0 + a, n);
#pragma unroll
        for (int b = 0; b < P1; ++b) x1[b] = wrap(c1 - (T / 2 - 1) + g1 * P1 + b, n);
#pragma unroll
        for (int c = 0; c < P2; ++c) x2[c] = wrap(c2 - (T / 2 - 1) + g2 * P2 + c, n);
#pragma unroll
        for (int a = 0; a < P0; ++a) {
            double* plane = g + (int64_t)x0[a] * n * n;
#pragma unroll
            for (int b = 0; b < P1; ++b) {
                double* row = plane + x1[b] * n;
#pragma unroll
                for (int c = 0; c < P2; ++c) red_add(row + x2[c], acc[a][b][c]);
            }
        }
    }
}

template <int B, int A = 12>
__global__ void AK_SPREAD3C_BOUNDS
k_spread3c(const CellIdx* __restrict__ ci, const double* __restrict__ W, const int64_t* __restrict__ wshift,
           const WorkItem* __restrict__ items, const double* __restrict__ V, Strides vs,
           double* __restrict__ grids, const int64_t* __restrict__ canon_off, int nrhs, int n)
{
    __shared__ Spread3cSmem<B> sm;
    spread3c_unit<B, A>(sm, blockIdx.x, ci, W, wshift, items, V, vs, grids, canon_off, nrhs, n);
}

// B fragments of a cell's 12^3 footprint straight from the grid g (one RHS of one
// window), in the permuted layout of fragment_offsets: lane (n = lane/4, kk = lane%4)
// of tile t holds G[a][b][c] with pair i = 2t + (n & 1), a = AO + i/3,
// b = 3 (n >> 1) + i % 3, c = 4 ks + kk.  A = active taps on axis 0 (12, or 10).
template <int A>
__device__ __forceinline__ void load_footprint(double (&gf)[3 * A / 2][3], const double* __restrict__ g, int sc,
                                               int n, int lane)
{
    constexpr int T = 12, NT = 3 * A / 2, AO = (T - A) / 2;
    const int c0 = sc & 1023, c1 = (sc >> 10) & 1023, c2 = (sc >> 20) & 1023;
    const int nn = lane >> 2, kk = lane & 3;
    const int qq = nn >> 1, e = nn & 1;
    const int o0 = c0 - (T / 2 - 1), o1 = c1 - (T / 2 - 1), o2 = c2 - (T / 2 - 1);
    if (o0 >= 0 && o0 + T <= n && o1 >= 0 && o1 + T <= n && o2 >= 0 && o2 + T <= n) {
        // footprint inside the grid: lane base + per-tile (a, b) plane/row offsets
        const int64_t n2 = (int64_t)n * n;
        const double* __restrict__ base = g + (int64_t)(o0 + AO) * n2 + (int64_t)(o1 + 3 * qq) * n + o2 + kk;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            // pair i = 2t + e: a = i / 3, b = i % 3 (selected per lane parity e)
            const int i0 = 2 * t, i1 = 2 * t + 1;
            const int64_t off0 = (i0 / 3) * n2 + (i0 % 3) * n, off1 = (i1 / 3) * n2 + (i1 % 3) * n;
            const double* row = base + (e ? off1 : off0);
#pragma unroll
            for (int ks = 0; ks < 3; ++ks) gf[t][ks] = __ldg(row + 4 * ks);
        }
        return;
    }
    int z[3];
#pragma unroll
    for (int ks = 0; ks < 3; ++ks) z[ks] = wrap(c2 - (T / 2 - 1) + 4 * ks + kk, n);
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        const int i = 2 * t + e;
        const int a = AO + i / 3, b = 3 * qq + i % 3;
        const int64_t rowb = ((int64_t)wrap(c0 - (T / 2 - 1) + a, n) * n + wrap(c1 - (T / 2 - 1) + b, n)) * n;
#pragma unroll
        for (int ks = 0; ks < 3; ++ks) gf[t][ks] = __ldg(g + rowb + z[ks]);
    }
}

template <int B>
struct alignas(128) Interp3cSmem {
    double wbuf[2][B][36];
    CellIdx cib[2][B];
    uint64_t bar[2];
};

// One (item, RHS) unit of the single-cell interpolation (the body of k_interp3c);
// A as for spread3c_unit (10: 15 fragment tiles instead of 18).
template <int B, int A = 12>
__device__ __forceinline__ void interp3c_unit(Interp3cSmem<B>& sm, int unit, const CellIdx* __restrict__ ci, const double* __restrict__ W, const int64_t* __restrict__ wshift,
           const WorkItem* __restrict__ items, const double* __restrict__ grids,
           const int64_t* __restrict__ canon_off, int nrhs, int n, const double* __restrict__ scale,
           double* __restrict__ out, Strides os, int atomic_out, int64_t wstride)
{
    constexpr int T = 12;
    constexpr int RW = 3 * T;
    static_assert(B % 8 == 0 && B <= 32, "batch");

    auto& wbuf = sm.wbuf;
    auto& cib = sm.cib;
    auto& bar = sm.bar;

    // the RHS index runs fastest: the nrhs CTAs of one item share its weight rows in L2
    const WorkItem it = items[unit / nrhs];
    const int r = unit % nrhs;
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

    constexpr int NT = 3 * A / 2;
    double gf[NT][3];
    load_footprint<A>(gf, grids + (int64_t)nrhs * canon_off[it.window] + (int64_t)r * n * n * n, it.sc, n, lane);
    const double sc = scale[it.window];
    double* __restrict__ o = out + (int64_t)it.window * wstride + (int64_t)r * os.rs;

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
        AK_UNROLL(AK_INTERP3C_UNROLL)
        for (int k0 = 0; k0 < nb; k0 += 8) {
            const int cnt = min(8, nb - k0);
            double v = interp_group_mma<RW, A>(gf, wbuf[s], k0, cnt, lane);
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            const int pj = lane >> 2;
            if ((lane & 3) == 0 && pj < cnt) {
                double* dst = o + (int64_t)cib[s][k0 + pj].idx * os.is;
                if (atomic_out) red_add(dst, sc * v);
                else *dst = sc * v;
            }
        }
    }
}

// Register cap (B200, tools/gpu_var_both.sh): 168 registers -> 12 warps/SM by registers
// (11 by shared memory): config 4 1.329 -> 1.256 ms, config 5 97.5 -> 91.4 ms per two
// launches; 184 / 200 / 224 registers: no gain; 160 / 152 / 144: 1.266 / 1.272 / 1.273 ms.
// (A two-set variant sharing the weight rows between K and dK/dl needed 255 registers
// plus spills and gained 0.1% on config 5 at the old cap: removed.)
#ifndef AK_INTERP3C_BOUNDS
#define AK_INTERP3C_BOUNDS __maxnreg__(168)
#endif
template <int B, int A = 12>
__global__ void AK_INTERP3C_BOUNDS
k_interp3c(const CellIdx* __restrict__ ci, const double* __restrict__ W, const int64_t* __restrict__ wshift,
           const WorkItem* __restrict__ items, const double* __restrict__ grids,
           const int64_t* __restrict__ canon_off, int nrhs, int n, const double* __restrict__ scale,
           double* __restrict__ out, Strides os, int atomic_out, int64_t wstride)
{
    __shared__ Interp3cSmem<B> sm;
    interp3c_unit<B, A>(sm, blockIdx.x, ci, W, wshift, items, grids, canon_off, nrhs, n, scale, out, os, atomic_out,
                     wstride);
}

}  // namespace ak
