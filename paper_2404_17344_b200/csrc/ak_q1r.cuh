// q = 1 spread / interpolation with the RHS index across the lanes (RHS-minor data).
//
// A 1-D window has 12 taps per point: per point and RHS the gridding work is 12
// FMAs, so with R right-hand sides the kernels are bound by moving the R values
// of each point (one cache line at R = 16 in the RHS-minor layout), not by FP64.
// One warp = a part of a work item (a chunk of <= 2048 bin-sorted points of a
// 16-cell supercell) x one chunk of RC right-hand sides:
//   lanes = SP point streams x RC RHS lanes (SP = 32 / RC);
//   per batch of 32 points each lane evaluates the 12 window weights of one
//   point (the weights serve all RC RHS) and the warp gathers / scatters the
//   points' RHS values as whole lines (lane = RHS within a point: coalesced);
//   interp: a stream keeps its current cell's 12 grid values per RHS lane in
//           registers and contracts them with each point's weights;
//   spread: a stream accumulates a cell run in registers (12 per lane) and adds
//           them to the grid (RED) when the cell changes.
// Replaces the lane-per-point kernels (ak_kernels.cuh) for R >= 8 RHS-minor
// products: those recompute the weights per RHS and touch one 8-byte value per
// point per CTA.
#pragma once
#include "ak_common.cuh"

namespace ak {

template <int RC>
struct Q1Lanes {
    static constexpr int SP = 32 / RC;   // point streams per warp
};

// Launch-time split of a work item into contiguous point ranges (one warp each): a
// q = 1 item holds up to 2048 points of one 16-cell supercell, and a warp per item
// leaves too few warps in flight to cover the gather latency.  The spread splits less:
// every part adds its cell-run accumulators to the same few grid values (RED
// contention).  Config 5 (B200): spread 2 parts 0.377 ms, 4: 0.484, 8: 0.865;
// interpolation 4 parts 0.392 ms per launch, 2: 0.397, 8: 0.404.
#ifndef AK_Q1_SPLIT_SPREAD
#define AK_Q1_SPLIT_SPREAD 2
#endif
#ifndef AK_Q1_SPLIT_INTERP
#define AK_Q1_SPLIT_INTERP 4
#endif
#ifndef AK_Q1_MINB
#define AK_Q1_MINB 16
#endif
// RHS values gathered one batch ahead (records two ahead) instead of at the batch start:
// config 5 spread 0.378 -> 0.391 ms (16 CTAs/SM, 12-byte spill) / 0.373 ms (12 CTAs/SM).
// ncu (k_spread1r, config 5): issue-bound, not gather-latency-bound -- 46.7% issue
// active, FP64 pipe 33%, 760 warp instructions per 32-point batch of which 84 DFMA
// evaluate the 12 window weights and ~350 load their coefficients / form gather
// addresses; DRAM 1.25 GB per launch (3.1 TB/s).
#ifndef AK_Q1_VPREFETCH
#define AK_Q1_VPREFETCH 0
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
// (config 5: 1M points per window over 64 cells), so a stream changes cell a few
// times per work item: the kernels keep no shared region tile -- the interpolation
// loads a new cell's 12 grid values per RHS lane straight from L2, the spread adds
// its register accumulators to the grid with 12 REDs per lane at a cell change.
// Batches whose points all lie in the stream's current cell (almost all) take an
// unrolled path: independent FMA chains across points, no per-point cell test.

template <int T, int RC>
__global__ void __launch_bounds__(32, AK_Q1_MINB)
k_interp1r(const Point* __restrict__ pts, const WorkItem* __restrict__ items, const double* __restrict__ grids,
           const int64_t* __restrict__ canon_off, int nrhs, int n, const ak_window_fn wf,
           const double* __restrict__ scale, double* __restrict__ out, Strides os, int atomic_out, int64_t wstride)
{
    constexpr int SP = Q1Lanes<RC>::SP, PPS = 32 / SP;   // point streams, points per stream per batch
    __shared__ __align__(16) double wst[32][T];
    __shared__ int lst[32], ist[32];

    const WorkItem it = items[blockIdx.x / AK_Q1_SPLIT_INTERP];
    int beg, end;
    q1_range(it, blockIdx.x % AK_Q1_SPLIT_INTERP, AK_Q1_SPLIT_INTERP, beg, end);
    const int r0 = blockIdx.y * RC;
    const int lane = threadIdx.x, rl = lane % RC, sp = lane / RC;
    const bool ract = r0 + rl < nrhs;
    const int sc0 = it.sc & 1023;
    const int o0 = sc0 * 16 - (T / 2 - 1);
    Point pn;
    if (lane < end - beg) pn = pts[beg + lane];
    const double* __restrict__ g =
        grids + (int64_t)nrhs * canon_off[it.window] + (int64_t)(ract ? r0 + rl : r0) * n;
    const double sc = scale[it.window];
    double* __restrict__ o = out + (int64_t)it.window * wstride + (int64_t)(r0 + rl) * os.rs;
    int cur = -1;
    double tv[T];
#define AK_Q1_LOAD_CELL(L)                                                        \
    do {                                                                          \
        cur = (L);                                                                \
        _Pragma("unroll") for (int a = 0; a < T; ++a) tv[a] = ract ? __ldg(g + wrap(o0 + cur + a, n)) : 0.0; \
    } while (0)
    for (int base = beg; base < end; base += 32) {
        const int nb = min(32, end - base);
        const Point p = pn;
        if (lane < end - base - 32) pn = pts[base + 32 + lane];
        __syncwarp();
        q1_stage<T>(p, lane < nb, sc0, lane, wf, wst, lst, ist);
        __syncwarp();
        // every point of the batch in the warp's current cell (both streams)?
        const bool same = __all_sync(0xffffffffu, lane >= nb || lst[lane] == cur);
        if (same && nb == 32) {
            constexpr int H = PPS > 8 ? 8 : PPS;   // points per pass (independent FMA chains)
#pragma unroll
            for (int k0 = 0; k0 < PPS; k0 += H) {
                double acc[H];
#pragma unroll
                for (int k = 0; k < H; ++k) acc[k] = 0.0;
#pragma unroll
                for (int a = 0; a < T; ++a)
#pragma unroll
                    for (int k = 0; k < H; ++k) acc[k] = fma(wst[sp + SP * (k0 + k)][a], tv[a], acc[k]);
#pragma unroll
                for (int k = 0; k < H; ++k) {
                    double* dst = o + (int64_t)ist[sp + SP * (k0 + k)] * os.is;
                    if (ract) {
                        if (atomic_out) red_add(dst, sc * acc[k]);
                        else *dst = sc * acc[k];
                    }
                }
            }
            continue;
        }
#pragma unroll 1
        for (int j = sp; j < nb; j += SP) {
            const int l = lst[j];
            if (l != cur) AK_Q1_LOAD_CELL(l);
            double acc = 0.0;
#pragma unroll
            for (int a = 0; a < T; ++a) acc = fma(wst[j][a], tv[a], acc);
            if (ract) {
                double* dst = o + (int64_t)ist[j] * os.is;
                if (atomic_out) red_add(dst, sc * acc);
                else *dst = sc * acc;
            }
        }
        // both streams continue in the cell of the batch's last point
        if (cur != lst[nb - 1]) AK_Q1_LOAD_CELL(lst[nb - 1]);
    }
#undef AK_Q1_LOAD_CELL
}

template <int T, int RC>
__global__ void __launch_bounds__(32, AK_Q1_MINB)
k_spread1r(const Point* __restrict__ pts, const WorkItem* __restrict__ items, const double* __restrict__ V,
           Strides vs, double* __restrict__ grids, const int64_t* __restrict__ canon_off, int nrhs, int n,
           const ak_window_fn wf)
{
    constexpr int SP = Q1Lanes<RC>::SP, PPS = 32 / SP;
    __shared__ __align__(16) double wst[32][T];
    __shared__ double vst[32][RC];
    __shared__ int lst[32];

    const WorkItem it = items[blockIdx.x / AK_Q1_SPLIT_SPREAD];
    int beg, end;
    q1_range(it, blockIdx.x % AK_Q1_SPLIT_SPREAD, AK_Q1_SPLIT_SPREAD, beg, end);
    const int r0 = blockIdx.y * RC;
    const int lane = threadIdx.x, rl = lane % RC, sp = lane / RC;
    const bool ract = r0 + rl < nrhs;
    const int sc0 = it.sc & 1023;
    const int o0 = sc0 * 16 - (T / 2 - 1);
    Point pn;
    if (lane < end - beg) pn = pts[beg + lane];
    const double* __restrict__ Vr = V + (int64_t)(r0 + rl) * vs.rs;
    double* __restrict__ g = grids + (int64_t)nrhs * canon_off[it.window] + (int64_t)(r0 + rl) * n;

    int cur = -1;
    double acc[T];
#pragma unroll
    for (int a = 0; a < T; ++a) acc[a] = 0.0;
    auto flush = [&]() {
        if (cur >= 0 && ract) {
#pragma unroll
            for (int a = 0; a < T; ++a) red_add(g + wrap(o0 + cur + a, n), acc[a]);
        }
#pragma unroll
        for (int a = 0; a < T; ++a) acc[a] = 0.0;
    };
    // the stream's RHS values of a batch (point j = sp + SP k, RHS r0 + rl); a stream's RC
    // lanes read one line per point
    auto gather = [&](double (&vv)[PPS], const Point& q, int nb) {
#pragma unroll
        for (int k = 0; k < PPS; ++k) {
            const int j = sp + SP * k;
            const int idx = __shfl_sync(0xffffffffu, q.idx, j);
            vv[k] = (j < nb && ract) ? __ldg(Vr + (int64_t)idx * vs.is) : 0.0;
        }
    };
#if AK_Q1_VPREFETCH
    // records two batches ahead, RHS values one batch ahead (the gather latency overlaps
    // a whole batch instead of the weight evaluation alone)
    Point pn2;
    if (lane < end - beg - 32) pn2 = pts[beg + 32 + lane];
    double vn[PPS];
    gather(vn, pn, min(32, end - beg));
#endif
    for (int base = beg; base < end; base += 32) {
        const int nb = min(32, end - base);
        const Point p = pn;
        double vv[PPS];
#if AK_Q1_VPREFETCH
#pragma unroll
        for (int k = 0; k < PPS; ++k) vv[k] = vn[k];
        pn = pn2;
        if (lane < end - base - 64) pn2 = pts[base + 64 + lane];
        if (base + 32 < end) gather(vn, pn, min(32, end - base - 32));
#else
        if (lane < end - base - 32) pn = pts[base + 32 + lane];
        gather(vv, p, nb);
#endif
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
        const bool same = __all_sync(0xffffffffu, lane >= nb || lst[lane] == cur);
        if (same) {
            // rows past nb hold v = 0
#pragma unroll
            for (int k = 0; k < PPS; ++k) {
                const int j = min(sp + SP * k, nb - 1);
#pragma unroll
                for (int a = 0; a < T; ++a) acc[a] = fma(wst[j][a], vv[k], acc[a]);
            }
            continue;
        }
        // a cell boundary inside the batch: point by point
#pragma unroll
        for (int k = 0; k < PPS; ++k) vst[sp + SP * k][rl] = vv[k];
        __syncwarp();
#pragma unroll 1
        for (int j = sp; j < nb; j += SP) {
            const int l = lst[j];
            if (l != cur) {
                flush();
                cur = l;
            }
            const double v = vst[j][rl];
#pragma unroll
            for (int a = 0; a < T; ++a) acc[a] = fma(wst[j][a], v, acc[a]);
        }
        __syncwarp();
    }
    flush();
}

}  // namespace ak
