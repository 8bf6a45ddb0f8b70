// q = 3 spread / interpolation kernels (the hot kernels of every 3-D window).
//
// Same decomposition as ak_kernels.cuh (one warp = one work item = at most
// `chunk` points of one S^3-cell supercell; (S+T-1)^3 shared region tile;
// T^3 footprint of the current cell held in registers, 2 x 4 x 4 lanes with
// (T/2) x (T/4) x (T/4) taps each), tuned for latency hiding at the ~8 warps
// per SM the 108-double register tile allows:
//  - the next batch's point records (and, for spread, the gathered RHS
//    values) are loaded while the current batch is processed;
//  - the next point's window weights are fetched from the staging buffer
//    into registers while the current point's FMAs issue;
//  - the staging rows are padded to 3T+2 doubles (2-way instead of 8-way
//    shared-memory bank conflicts on the staging stores).
#pragma once
#include "ak_common.cuh"

namespace ak {

template <int T>
struct Q3Lanes {
    static constexpr int P0 = T / 2, P1 = T / 4, P2 = T / 4;
    static constexpr int WS = 3 * T + 2;  // padded staging row
};

__device__ __forceinline__ Point load_point(const Point* __restrict__ p) {
    const double2* q = reinterpret_cast<const double2*>(p);
    const double2 a = __ldg(q);
    const double2 b = __ldg(q + 1);
    Point r;
    r.s[0] = a.x;
    r.s[1] = a.y;
    r.s[2] = b.x;
    const int2 ci = *reinterpret_cast<const int2*>(&b.y);
    r.cell = ci.x;
    r.idx = ci.y;
    return r;
}

// Grid index of region-tile element i (R^3 tile at origin o0,o1,o2), wrapped
// periodically.  For n >= 16 every coordinate lies in [-n, 2n) (S <= 4,
// T <= 16), so one conditional add/subtract replaces the modulo.
template <int R>
__device__ __forceinline__ int64_t region_index(int i, int o0, int o1, int o2, int n) {
    const int i2 = i % R, i1 = (i / R) % R, i0 = i / (R * R);
    int x = o0 + i0, y = o1 + i1, z = o2 + i2;
    if (n >= 16) {
        x += x < 0 ? n : (x >= n ? -n : 0);
        y += y < 0 ? n : (y >= n ? -n : 0);
        z += z < 0 ? n : (z >= n ? -n : 0);
    } else {
        x = wrap(x, n);
        y = wrap(y, n);
        z = wrap(z, n);
    }
    return ((int64_t)x * n + y) * n + z;
}

// Load this lane's slice of one point's weights from its staging row.
template <int T, int P0, int P1, int P2>
__device__ __forceinline__ void load_w(double (&w0)[P0], double (&w1)[P1], double (&w2)[P2],
                                       const double* __restrict__ row, int g0, int g1, int g2)
{
#pragma unroll
    for (int a = 0; a < P0; ++a) w0[a] = row[g0 * P0 + a];
#pragma unroll
    for (int b = 0; b < P1; ++b) w1[b] = row[T + g1 * P1 + b];
#pragma unroll
    for (int c = 0; c < P2; ++c) w2[c] = row[2 * T + g2 * P2 + c];
}

// acc[a][b][c] += (v w0[a]) * (w1[b] w2[c]) for this lane's footprint slice.
template <int P0, int P1, int P2>
__device__ __forceinline__ void spread_fma(double (&acc)[P0][P1][P2], const double (&w0)[P0],
                                           const double (&w1)[P1], const double (&w2)[P2])
{
#pragma unroll
    for (int b = 0; b < P1; ++b)
#pragma unroll
        for (int c = 0; c < P2; ++c) {
            const double pbc = w1[b] * w2[c];
#pragma unroll
            for (int a = 0; a < P0; ++a) acc[a][b][c] = fma(w0[a], pbc, acc[a][b][c]);
        }
}

template <int T, int S>
__global__ void __launch_bounds__(32, 8)
k_spread3(const Point* __restrict__ pts, const WorkItem* __restrict__ items,
          const double* __restrict__ V, Strides vs,
          double* __restrict__ grids, const int64_t* __restrict__ canon_off, int nrhs,
          int n, const ak_window_fn wf)
{
    using LN = Q3Lanes<T>;
    constexpr int P0 = LN::P0, P1 = LN::P1, P2 = LN::P2, WS = LN::WS;
    constexpr int R = S + T - 1;
    constexpr int TILE = R * R * R;

    __shared__ double tile[TILE];
    __shared__ __align__(16) double wst[32][WS];
    __shared__ int cst[32];

    const WorkItem it = items[blockIdx.x / nrhs];   // RHS index fastest
    const int r = blockIdx.x % nrhs;
    const int lane = threadIdx.x;
    const int g0 = lane >> 4, g1 = (lane >> 2) & 3, g2 = lane & 3;
    const int sc0 = it.sc & 1023, sc1 = (it.sc >> 10) & 1023, sc2 = (it.sc >> 20) & 1023;
    const double* __restrict__ Vr = V + (int64_t)r * vs.rs;
    const int end = it.start + it.count;

    for (int i = lane; i < TILE; i += 32) tile[i] = 0.0;

    double acc[P0][P1][P2];
#pragma unroll
    for (int a = 0; a < P0; ++a)
#pragma unroll
        for (int b = 0; b < P1; ++b)
#pragma unroll
            for (int c = 0; c < P2; ++c) acc[a][b][c] = 0.0;
    int cur = -1;

    auto flush = [&](int cell) {
        const int l0 = cell & 255, l1 = (cell >> 8) & 255, l2 = (cell >> 16) & 255;
#pragma unroll
        for (int a = 0; a < P0; ++a)
#pragma unroll
            for (int b = 0; b < P1; ++b)
#pragma unroll
                for (int c = 0; c < P2; ++c) {
                    double* t = &tile[((l0 + g0 * P0 + a) * R + (l1 + g1 * P1 + b)) * R + (l2 + g2 * P2 + c)];
                    *t += acc[a][b][c];
                    acc[a][b][c] = 0.0;
                }
        __syncwarp();
    };

    // batch prefetch registers
    Point pn;
    double vn = 0.0;
    if (lane < min(32, end - it.start)) {
        pn = load_point(pts + it.start + lane);
        vn = __ldg(Vr + (int64_t)pn.idx * vs.is);
    }
    for (int base = it.start; base < end; base += 32) {
        const int nb = min(32, end - base);
        const Point p = pn;
        const double val = vn;
        const int nbase = base + 32;
        const bool more = lane < min(32, end - nbase);
        if (more) pn = load_point(pts + nbase + lane);
        __syncwarp();
        if (lane < nb) {
            double w[T];
            window_weights<T>(wf, p.s[0], w);
#pragma unroll
            for (int a = 0; a < T; ++a) wst[lane][a] = val * w[a];
            window_weights<T>(wf, p.s[1], w);
#pragma unroll
            for (int a = 0; a < T; ++a) wst[lane][T + a] = w[a];
            window_weights<T>(wf, p.s[2], w);
#pragma unroll
            for (int a = 0; a < T; ++a) wst[lane][2 * T + a] = w[a];
            cst[lane] = (cell_axis(p.cell, 0) - sc0 * S) | ((cell_axis(p.cell, 1) - sc1 * S) << 8) |
                        ((cell_axis(p.cell, 2) - sc2 * S) << 16);
        }
        if (more) vn = __ldg(Vr + (int64_t)pn.idx * vs.is);
        __syncwarp();

        // bit k set <=> point k starts a new cell run (register-only test in the loop)
        const int mycell = lane < nb ? cst[lane] : -2;
        const int prev = __shfl_up_sync(0xffffffffu, mycell, 1);
        const unsigned chg = __ballot_sync(0xffffffffu, lane < nb && (lane == 0 ? mycell != cur : mycell != prev));

        // Cell runs: the FMA loop of a run has no cell test; weights of the next
        // point are loaded (register set B) before the FMAs of the current one (A).
        for (int k = 0; k < nb;) {
            if ((chg >> k) & 1u) {
                if (cur >= 0) flush(cur);
                cur = cst[k];
            }
            const unsigned later = k < 31 ? chg & ~((2u << k) - 1u) : 0u;
            const int kend = later ? min(__ffs(later) - 1, nb) : nb;
            double a0[P0], a1[P1], a2[P2], b0[P0], b1[P1], b2[P2];
            load_w<T>(a0, a1, a2, &wst[k][0], g0, g1, g2);
            int j = k;
            for (; j + 1 < kend; j += 2) {
                load_w<T>(b0, b1, b2, &wst[j + 1][0], g0, g1, g2);
                spread_fma(acc, a0, a1, a2);
                load_w<T>(a0, a1, a2, &wst[j + 2 < kend ? j + 2 : j + 1][0], g0, g1, g2);
                spread_fma(acc, b0, b1, b2);
            }
            if (j < kend) spread_fma(acc, a0, a1, a2);
            k = kend;
        }
    }
    if (cur >= 0) flush(cur);
    __syncwarp();

    double* __restrict__ g = grids + (int64_t)nrhs * canon_off[it.window] + (int64_t)r * n * n * n;
    const int o0 = sc0 * S - (T / 2 - 1);
    const int o1 = sc1 * S - (T / 2 - 1);
    const int o2 = sc2 * S - (T / 2 - 1);
    for (int i = lane; i < TILE; i += 32) {
        const double val = tile[i];
        if (val != 0.0) red_add(g + region_index<R>(i, o0, o1, o2, n), val);
    }
}

// Partial dot product of one point's weights (staging row) with this lane's
// footprint slice: sum_{a,b,c} w0[a] w1[b] w2[c] tv[a][b][c].
template <int P0, int P1, int P2>
__device__ __forceinline__ double footprint_dot(const double (&tv)[P0][P1][P2], const double* wrow,
                                                int g0, int g1, int g2)
{
    constexpr int T = 2 * P0;
    double w0[P0], w1[P1], w2[P2];
#pragma unroll
    for (int a = 0; a < P0; ++a) w0[a] = wrow[g0 * P0 + a];
#pragma unroll
    for (int b = 0; b < P1; ++b) w1[b] = wrow[T + g1 * P1 + b];
#pragma unroll
    for (int c = 0; c < P2; ++c) w2[c] = wrow[2 * T + g2 * P2 + c];
    double accb = 0.0;
#pragma unroll
    for (int b = 0; b < P1; ++b) {
        double accc = 0.0;
#pragma unroll
        for (int c = 0; c < P2; ++c) {
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < P0; ++a) s = fma(w0[a], tv[a][b][c], s);
            accc = fma(w2[c], s, accc);
        }
        accb = fma(w1[b], accc, accb);
    }
    return accb;
}

template <int T, int S>
__global__ void __launch_bounds__(32, 8)
k_interp3(const Point* __restrict__ pts, const WorkItem* __restrict__ items,
          const double* __restrict__ grids, const int64_t* __restrict__ canon_off, int nrhs,
          int n, const ak_window_fn wf, const double* __restrict__ scale,
          double* __restrict__ out, Strides os, int atomic_out, int64_t wstride)
{
    using LN = Q3Lanes<T>;
    constexpr int P0 = LN::P0, P1 = LN::P1, P2 = LN::P2, WS = LN::WS;
    constexpr int R = S + T - 1;
    constexpr int TILE = R * R * R;

    __shared__ double tile[TILE];
    __shared__ __align__(16) double wst[32][WS];
    __shared__ int cst[32];
    __shared__ int ist[32];

    const WorkItem it = items[blockIdx.x / nrhs];   // RHS index fastest
    const int r = blockIdx.x % nrhs;
    const int lane = threadIdx.x;
    const int g0 = lane >> 4, g1 = (lane >> 2) & 3, g2 = lane & 3;
    const int sc0 = it.sc & 1023, sc1 = (it.sc >> 10) & 1023, sc2 = (it.sc >> 20) & 1023;
    const int end = it.start + it.count;

    Point pn;
    if (lane < min(32, end - it.start)) pn = load_point(pts + it.start + lane);

    {
        const double* __restrict__ g = grids + (int64_t)nrhs * canon_off[it.window] + (int64_t)r * n * n * n;
        const int o0 = sc0 * S - (T / 2 - 1);
        const int o1 = sc1 * S - (T / 2 - 1);
        const int o2 = sc2 * S - (T / 2 - 1);
        for (int i = lane; i < TILE; i += 32) cp_async8(&tile[i], g + region_index<R>(i, o0, o1, o2, n));
        cp_async_commit();
        cp_async_wait_all();
        __syncwarp();
    }
    const double sc = scale[it.window];
    double* __restrict__ o = out + (int64_t)it.window * wstride + (int64_t)r * os.rs;

    double tv[P0][P1][P2];
    int cur = -1;

    for (int base = it.start; base < end; base += 32) {
        const int nb = min(32, end - base);
        const Point p = pn;
        const int nbase = base + 32;
        if (lane < min(32, end - nbase)) pn = load_point(pts + nbase + lane);
        __syncwarp();
        if (lane < nb) {
            double w[T];
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
                window_weights<T>(wf, p.s[ax], w);
#pragma unroll
                for (int a = 0; a < T; ++a) wst[lane][ax * T + a] = w[a];
            }
            cst[lane] = (cell_axis(p.cell, 0) - sc0 * S) | ((cell_axis(p.cell, 1) - sc1 * S) << 8) |
                        ((cell_axis(p.cell, 2) - sc2 * S) << 16);
            ist[lane] = p.idx;
        }
        __syncwarp();

        const int mycell = lane < nb ? cst[lane] : -2;
        const int prev = __shfl_up_sync(0xffffffffu, mycell, 1);
        const unsigned chg = __ballot_sync(0xffffffffu, lane < nb && (lane == 0 ? mycell != cur : mycell != prev));

        for (int grp = 0; grp < nb; grp += 8) {
            double part[8];
            if (grp + 8 <= nb && ((chg >> grp) & 0xffu) == 0u) {
                // fast path: 8 points of the current cell, straight-line code
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    part[kk] = footprint_dot<P0, P1, P2>(tv, &wst[grp + kk][0], g0, g1, g2);
            } else {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const int k = grp + kk;
                    part[kk] = 0.0;
                    if (k < nb) {
                        if ((chg >> k) & 1u) {
                            cur = cst[k];
                            const int l0 = cur & 255, l1 = (cur >> 8) & 255, l2 = (cur >> 16) & 255;
#pragma unroll
                            for (int a = 0; a < P0; ++a)
#pragma unroll
                                for (int b = 0; b < P1; ++b)
#pragma unroll
                                    for (int c = 0; c < P2; ++c)
                                        tv[a][b][c] = tile[((l0 + g0 * P0 + a) * R + (l1 + g1 * P1 + b)) * R +
                                                           (l2 + g2 * P2 + c)];
                        }
                        part[kk] = footprint_dot<P0, P1, P2>(tv, &wst[k][0], g0, g1, g2);
                    }
                }
            }
            // Transposed reduction: lane ends with the warp sum of part[lane & 7].
            const bool hi4 = lane & 4;
            double q4[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const double send = hi4 ? part[j] : part[j + 4];
                const double keep = hi4 ? part[j + 4] : part[j];
                q4[j] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
            }
            const bool hi2 = lane & 2;
            double q2[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const double send = hi2 ? q4[j] : q4[j + 2];
                const double keep = hi2 ? q4[j + 2] : q4[j];
                q2[j] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
            }
            const bool hi1 = lane & 1;
            const double send = hi1 ? q2[0] : q2[1];
            double v = (hi1 ? q2[1] : q2[0]) + __shfl_xor_sync(0xffffffffu, send, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 8);
            v += __shfl_xor_sync(0xffffffffu, v, 16);
            if (lane < 8 && grp + lane < nb) {
                double* dst = o + (int64_t)ist[grp + lane] * os.is;
                if (atomic_out) red_add(dst, sc * v);
                else *dst = sc * v;
            }
        }
    }
}

}  // namespace ak
