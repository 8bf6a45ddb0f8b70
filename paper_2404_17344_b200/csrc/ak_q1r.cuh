// q = 1 spread / interpolation for R >= 8 right-hand sides (RHS-minor data).
//
// A 1-D window has 12 taps per point: per point and RHS the gridding work is 12
// FMAs, so with R right-hand sides the kernels are bound by moving the R values
// of each point (one cache line at R = 16 in the RHS-minor layout), not by FP64.
// One warp = a part of a work item (a chunk of <= 2048 bin-sorted points of a
// 16-cell supercell) x one chunk of RC right-hand sides; per batch of 32 points
// each lane evaluates the 12 window weights of one point (they serve all RC RHS),
// and within one cell the products are small GEMMs on the FP64 tensor cores
// (below).  RHS values are gathered / results scattered as whole lines.
// Replaces the lane-per-point kernels (ak_kernels.cuh) for R >= 8 RHS-minor
// products: those recompute the weights per RHS and touch one 8-byte value per
// point per CTA.  Round 2 first ran these products as per-lane DFMA chains (lanes
// = 2 point streams x 16 RHS): issue-bound at ~760 warp instructions per batch,
// config 5 spread 0.374 / interpolation 0.782 ms per step; the DMMA form: 0.271 / 0.698.
#pragma once
#include "ak_common.cuh"
#include "ak_q3m.cuh"   // dmma_8x8x4

namespace ak {

// Launch-time split of a work item into contiguous point ranges (one warp each): a
// q = 1 item holds up to 2048 points of one 16-cell supercell, and a warp per item
// leaves too few warps in flight to cover the gather latency.  The spread splits less:
// every part adds its cell-run accumulators to the same few grid values (RED
// contention).  Config 5 (B200, DFMA lane kernels): spread 2 parts 0.377 ms, 4: 0.484,
// 8: 0.865; interpolation 4 parts 0.392 ms per launch, 2: 0.397, 8: 0.404.  DMMA kernels:
// interpolation 4 parts 0.698 ms per step, 2: 0.722; 24 instead of 16 warps per SM
// (AK_Q1_MINB): spread 0.271 -> 0.289, interpolation 0.698 -> 0.703.
#ifndef AK_Q1_SPLIT_SPREAD
#define AK_Q1_SPLIT_SPREAD 2
#endif
#ifndef AK_Q1_SPLIT_INTERP
#define AK_Q1_SPLIT_INTERP 4
#endif
#ifndef AK_Q1_MINB
#define AK_Q1_MINB 16
#endif
__device__ __forceinline__ void q1_range(const WorkItem& it, int part, int parts, int& beg, int& end) {
    beg = it.start + (int)((int64_t)it.count * part / parts);
    end = it.start + (int)((int64_t)it.count * (part + 1) / parts);
}

// weights, local cell offset and row of the batch's points (one point per lane,
// already in registers: the next batch's records are loaded before this one is used)
template <int T>
__device__ __forceinline__ void q1_stage(const Point& p, bool valid, int sc0, int lane, const ak_window_fn& wf,
                                         double (*wst)[T], int* lst, int* ist)
{
    if (valid) {
        double w[T];
        window_weights<T>(wf, p.s[0], w);
#pragma unroll
        for (int a = 0; a < T; ++a) wst[lane][a] = w[a];
        lst[lane] = cell_axis(p.cell, 0) - sc0 * 16;
        AK_DCHECK(lst[lane] >= 0 && lst[lane] < 16);
        ist[lane] = p.idx;
    }
}

// In the q = 1 windows of the BASELINE workloads a cell holds thousands of points
// (config 5: 1M points per window over 64 cells), so a warp changes cell a few
// times per work item: the kernels keep no shared region tile -- the interpolation
// loads a new cell's grid values straight from L2, the spread adds its
// accumulators to the grid with REDs at a cell change.  Batches whose points all
// lie in the current cell (almost all) take an unrolled path with no cell tests.
//
// FP64 tensor-core formulation (mma.sync m8n8k4 f64).  Within one cell the q = 1
// products are small GEMMs over (points x taps x RHS):
//   interp : out[j][r] = sum_a w_j[a] G_r[cell + a]   A = weights (8 points x 4 taps),
//            B = the cell's grid values (4 taps x 8 RHS, registers while the cell
//            lasts), C = 8 points x 8 RHS: 3 DMMA per 8 points per 8 RHS;
//   spread : G_r[cell + a] += sum_j v_j[r] w_j[a]    A = RHS values (8 RHS x 4 points),
//            B = weights (4 points x 8 taps; 12 taps padded to 16), C = 8 RHS x 16 taps
//            accumulated over the cell run: 2 DMMA per 4 points per 8 RHS.
// Per 32-point batch a warp issues 12 NT (interp) / 16 MT (spread) DMMA instead of
// 12 x 32 x RC / 32 DFMA and the same number of shared-memory weight reads; each
// lane evaluates the 12 window weights of one point.  Groups that span a cell
// boundary run once per distinct cell with the other rows masked to zero.
// ncu (config 5): spread 1.25 GB DRAM in 0.277 ms; per-window interpolation 1.22 GB in
// 0.270 ms; the summed interpolation (RED into the [N][16] output lines that every
// window adds to: one read-modify-write of 512 MB per window) 2.2 GB in 0.420 ms.
template <int T, int RC>
__global__ void __launch_bounds__(32, AK_Q1_MINB)
k_interp1r(const Point* __restrict__ pts, const WorkItem* __restrict__ items, const double* __restrict__ grids,
           const int64_t* __restrict__ canon_off, int nrhs, int n, const ak_window_fn wf,
           const double* __restrict__ scale, double* __restrict__ out, Strides os, int atomic_out, int64_t wstride)
{
    static_assert(T == 12 && RC % 8 == 0, "12 taps, RHS chunks of 8");
    constexpr int NT = RC / 8;   // RHS n-tiles per warp
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int OS = RC % 16 ? RC : RC + 8;   // staged result row stride
    __shared__ __align__(16) double wst[32][T];
    __shared__ __align__(16) double ob[32][OS];
    __shared__ int lst[32], ist[32];

    const WorkItem it = items[blockIdx.x / AK_Q1_SPLIT_INTERP];
    int beg, end;
    q1_range(it, blockIdx.x % AK_Q1_SPLIT_INTERP, AK_Q1_SPLIT_INTERP, beg, end);
    const int r0 = blockIdx.y * RC;
    const int lane = threadIdx.x, pj = lane >> 2, q = lane & 3;
    const int sc0 = it.sc & 1023;
    const int o0 = sc0 * 16 - (T / 2 - 1);
    Point pn;
    if (lane < end - beg) pn = pts[beg + lane];
    const double* __restrict__ g0 = grids + (int64_t)nrhs * canon_off[it.window];
    const double sc = scale[it.window];
    double* __restrict__ o = out + (int64_t)it.window * wstride + (int64_t)r0 * os.rs;

    // B fragments of the current cell: lane (k = q, n = pj) of n-tile nt, k-step ks holds
    // G_r[cell + 4 ks + q], r = r0 + 8 nt + pj
    int cur = -1;
    double gb[NT][3];
    auto load_cell = [&](int c) {
        cur = c;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const int r = r0 + 8 * nt + pj;
            const double* __restrict__ g = g0 + (int64_t)min(r, nrhs - 1) * n;
#pragma unroll
            for (int ks = 0; ks < 3; ++ks) gb[nt][ks] = r < nrhs ? __ldg(g + wrap(o0 + c + 4 * ks + q, n)) : 0.0;
        }
    };
    // C row pj = point j, columns 2 q + e of n-tile nt = RHS r0 + 8 nt + 2 q + e: staged in
    // shared memory (16-B stores, rows padded so a quarter warp hits distinct banks) and
    // written out with the lanes along a point's RHS, so every store / RED instruction
    // covers whole lines (from the fragment layout a RED would touch 8 lines x 2 sectors)
    auto stage = [&](int j, const double (&C)[NT][2]) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
            *reinterpret_cast<double2*>(&ob[j][8 * nt + 2 * q]) = make_double2(sc * C[nt][0], sc * C[nt][1]);
    };
    const int nr = min(RC, nrhs - r0);
    for (int base = beg; base < end; base += 32) {
        const int nb = min(32, end - base);
        const Point p = pn;
        if (lane < end - base - 32) pn = pts[base + 32 + lane];
        __syncwarp();
        q1_stage<T>(p, lane < nb, sc0, lane, wf, wst, lst, ist);
        __syncwarp();
        if (__all_sync(FULL, lane >= nb || lst[lane] == cur)) {
            // the whole batch in the current cell: 4 m-tiles x 3 k-steps x NT independent DMMA
            double C[4][NT][2];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                double af[3];
#pragma unroll
                for (int ks = 0; ks < 3; ++ks) af[ks] = wst[8 * mt + pj][4 * ks + q];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    C[mt][nt][0] = C[mt][nt][1] = 0.0;
#pragma unroll
                    for (int ks = 0; ks < 3; ++ks) dmma_8x8x4(C[mt][nt][0], C[mt][nt][1], af[ks], gb[nt][ks]);
                }
            }
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) stage(8 * mt + pj, C[mt]);
        } else {
            // a cell boundary inside the batch: each 8-point group once per distinct cell
#pragma unroll 1
            for (int mt = 0; 8 * mt < nb; ++mt) {
                const int j = 8 * mt + pj;
                const int myc = j < nb ? lst[j] : -1;
                bool done = j >= nb;
                double C[NT][2];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) C[nt][0] = C[nt][1] = 0.0;
                for (;;) {
                    const unsigned pending = __ballot_sync(FULL, !done);
                    if (!pending) break;
                    const int c = __shfl_sync(FULL, myc, __ffs(pending) - 1);
                    if (c != cur) load_cell(c);
                    const bool mine = !done && myc == c;
                    double af[3];
#pragma unroll
                    for (int ks = 0; ks < 3; ++ks) af[ks] = mine ? wst[j][4 * ks + q] : 0.0;
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                        for (int ks = 0; ks < 3; ++ks) dmma_8x8x4(C[nt][0], C[nt][1], af[ks], gb[nt][ks]);
                    done = done || mine;
                }
                stage(j, C);
            }
        }
        __syncwarp();
#pragma unroll 4
        for (int e = lane; e < nb * RC; e += 32) {
            const int j = e / RC, rr = e - j * RC;
            if (rr < nr) {
                double* dst = o + (int64_t)ist[j] * os.is + (int64_t)rr * os.rs;
                if (atomic_out) red_add(dst, ob[j][rr]);
                else *dst = ob[j][rr];
            }
        }
        __syncwarp();
    }
}

template <int T, int RC>
__global__ void __launch_bounds__(32, AK_Q1_MINB)
k_spread1r(const Point* __restrict__ pts, const WorkItem* __restrict__ items, const double* __restrict__ V,
           Strides vs, double* __restrict__ grids, const int64_t* __restrict__ canon_off, int nrhs, int n,
           const ak_window_fn wf)
{
    static_assert(T == 12 && RC % 8 == 0, "12 taps, RHS chunks of 8");
    constexpr int MT = RC / 8;   // RHS m-tiles per warp
    constexpr unsigned FULL = 0xffffffffu;
    __shared__ __align__(16) double wst[32][T];
    __shared__ double vst[32][RC];
    __shared__ int lst[32];

    const WorkItem it = items[blockIdx.x / AK_Q1_SPLIT_SPREAD];
    int beg, end;
    q1_range(it, blockIdx.x % AK_Q1_SPLIT_SPREAD, AK_Q1_SPLIT_SPREAD, beg, end);
    const int r0 = blockIdx.y * RC;
    const int lane = threadIdx.x, pj = lane >> 2, q = lane & 3;
    const int sc0 = it.sc & 1023;
    const int o0 = sc0 * 16 - (T / 2 - 1);
    Point pn;
    if (lane < end - beg) pn = pts[beg + lane];
    const double* __restrict__ V0 = V + (int64_t)r0 * vs.rs;
    double* __restrict__ g0 = grids + (int64_t)nrhs * canon_off[it.window];
    // rows past a short batch's end keep finite weights (their RHS values are zero)
#pragma unroll
    for (int a = 0; a < T; ++a) wst[lane][a] = 0.0;

    // C of m-tile mt, n-tile nt: row pj = RHS r0 + 8 mt + pj, columns 2 q + e = tap 8 nt + 2 q + e
    int cur = -1;
    double C[MT][2][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) C[mt][nt][0] = C[mt][nt][1] = 0.0;
    auto flush = [&]() {
        if (cur >= 0) {
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                const int r = r0 + 8 * mt + pj;
                if (r < nrhs) {
                    double* __restrict__ g = g0 + (int64_t)r * n;
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int a = 8 * nt + 2 * q + e;
                            if (a < T) red_add(g + wrap(o0 + cur + a, n), C[mt][nt][e]);
                        }
                }
            }
        }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) C[mt][nt][0] = C[mt][nt][1] = 0.0;
    };
    for (int base = beg; base < end; base += 32) {
        const int nb = min(32, end - base);
        const Point p = pn;
        if (lane < end - base - 32) pn = pts[base + 32 + lane];
        // A fragments of the batch: lane (row pj, col q) of k-step ks, m-tile mt holds the
        // value of point 4 ks + q for RHS r0 + 8 mt + pj (a point's RHS values are one line)
        double vv[8][MT];
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            const int j = 4 * ks + q;
            const int idx = __shfl_sync(FULL, p.idx, j);
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
                vv[ks][mt] = (j < nb && r0 + 8 * mt + pj < nrhs)
                                 ? __ldg(V0 + (int64_t)idx * vs.is + (int64_t)(8 * mt + pj) * vs.rs)
                                 : 0.0;
        }
        __syncwarp();
        if (lane < nb) {
            double w[T];
            window_weights<T>(wf, p.s[0], w);
#pragma unroll
            for (int a = 0; a < T; ++a) wst[lane][a] = w[a];
            lst[lane] = cell_axis(p.cell, 0) - sc0 * 16;
            AK_DCHECK(lst[lane] >= 0 && lst[lane] < 16);
        }
        __syncwarp();
        if (__all_sync(FULL, lane >= nb || lst[lane] == cur)) {
            // B: lane (k = q, n = pj) holds tap 8 nt + pj of point 4 ks + q (taps >= 12: 0)
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const double b0 = wst[4 * ks + q][pj];
                const double b1 = pj < 4 ? wst[4 * ks + q][8 + pj] : 0.0;
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    dmma_8x8x4(C[mt][0][0], C[mt][0][1], vv[ks][mt], b0);
                    dmma_8x8x4(C[mt][1][0], C[mt][1][1], vv[ks][mt], b1);
                }
            }
            continue;
        }
        // a cell boundary inside the batch: each 4-point k-step once per distinct cell
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) vst[4 * ks + q][8 * mt + pj] = vv[ks][mt];
        __syncwarp();
#pragma unroll 1
        for (int ks = 0; 4 * ks < nb; ++ks) {
            const int j = 4 * ks + q;
            const int myc = j < nb ? lst[j] : -1;
            bool done = j >= nb;
            for (;;) {
                const unsigned pending = __ballot_sync(FULL, !done);
                if (!pending) break;
                const int c = __shfl_sync(FULL, myc, __ffs(pending) - 1);
                if (c != cur) {
                    flush();
                    cur = c;
                }
                const bool mine = !done && myc == c;
                const double b0 = mine ? wst[j][pj] : 0.0;
                const double b1 = (mine && pj < 4) ? wst[j][8 + pj] : 0.0;
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    const double a = vst[j][8 * mt + pj];
                    dmma_8x8x4(C[mt][0][0], C[mt][0][1], a, b0);
                    dmma_8x8x4(C[mt][1][0], C[mt][1][1], a, b1);
                }
                done = done || mine;
            }
        }
        __syncwarp();
    }
    flush();
}

}  // namespace ak
