// Spread / interpolation kernels (sm_100a, FP64 CUDA cores).
//
// Replaces the numba loops _spread_q / _interp_q of the reference
// (/root/reference/pkg/src/addkern/nufft.py:197-320).
//
// Work decomposition: points of each window are bin-sorted by
// (supercell, cell).  One CTA = one warp = one WorkItem, i.e. at most `chunk`
// points of one supercell (S^q cells).  The CTA owns a shared-memory tile of
// the (S+T-1)^q grid region the supercell's footprints touch:
//   spread : register-tiled accumulation of each cell run (all points of a
//            cell share one T^q footprint), flushed into the shared tile at
//            every cell change, and the tile flushed once to the global grid
//            with RED.F64 (one atomic per touched grid value per item instead
//            of T^q per point);
//   interp : the region is loaded once into shared memory, each cell's T^q
//            footprint is held in registers while its points are evaluated,
//            and partial dot products are combined with a transposed warp
//            reduction (8 points per reduction).
// The lane layout splits the T^q footprint over the 32 lanes (G0 x G1 x G2
// lane groups per axis); for q < 3 the warp holds 32/L "slots" that process
// several points of the same cell per step.
#pragma once
#include "ak_common.cuh"
#include "ak_q3.cuh"

namespace ak {

// Lane layout of the T^q footprint: G0 x G1 x G2 lane groups per axis.
//   q = 3: 2 x 4 x 4 lanes (T=12: 6 x 3 x 3 taps per lane), one point per step
//   q = 2: 4 x 4 lanes (T=12: 3 x 3 taps per lane), two points (slots) per step
//   q = 1: 4 lanes (T=12: 3 taps per lane), eight points per step
template <int Q> struct Layout;
template <> struct Layout<3> { static constexpr int G0 = 2, G1 = 4, G2 = 4; };
template <> struct Layout<2> { static constexpr int G0 = 4, G1 = 4, G2 = 1; };
template <> struct Layout<1> { static constexpr int G0 = 4, G1 = 1, G2 = 1; };

template <int Q> __host__ __device__ constexpr int ipow(int b) { return Q == 1 ? b : (Q == 2 ? b * b : b * b * b); }

// ---------------------------------------------------------------------------
// Spread: sum_j v_j prod_a phi(t_ja - i_a) onto the grid (real arithmetic).
// grid(w, r) = grids + nrhs * canon_off[w] + r * n^Q  (canonical layout, see ak_lib.cu)
template <int Q, int T>
__global__ void __launch_bounds__(32)
k_spread_tile(const Point* __restrict__ pts, const WorkItem* __restrict__ items,
              const double* __restrict__ V, Strides vs,
              double* __restrict__ grids, const int64_t* __restrict__ canon_off, int nrhs,
              int n, const ak_window_fn wf)
{
    using LY = Layout<Q>;
    constexpr int S = SuperCell<Q>::S;
    constexpr int R = S + T - 1;
    constexpr int TILE = ipow<Q>(R);
    constexpr int G0 = LY::G0, G1 = LY::G1, G2 = LY::G2;
    constexpr int L = G0 * G1 * G2;
    constexpr int SLOTS = 32 / L;
    constexpr int P0 = T / G0;
    constexpr int P1 = Q >= 2 ? T / G1 : 1;
    constexpr int P2 = Q >= 3 ? T / G2 : 1;
    constexpr int WROW = Q * T;

    __shared__ double tile[TILE];
    __shared__ __align__(16) double wst[32][WROW];
    __shared__ int cst[32];

    // the RHS index runs fastest: the nrhs CTAs of one item share its point records in L2
    const WorkItem it = items[blockIdx.x / nrhs];
    const int r = blockIdx.x % nrhs;
    const int lane = threadIdx.x;
    const int slot = lane / L;
    const int rl = lane % L;
    const int g0 = rl / (G1 * G2);
    const int g1 = (rl / G2) % G1;
    const int g2 = rl % G2;
    const int sc0 = it.sc & 1023, sc1 = (it.sc >> 10) & 1023, sc2 = (it.sc >> 20) & 1023;

    for (int i = lane; i < TILE; i += 32) tile[i] = 0.0;

    double acc[P0][P1][P2];
#pragma unroll
    for (int a = 0; a < P0; ++a)
#pragma unroll
        for (int b = 0; b < P1; ++b)
#pragma unroll
            for (int c = 0; c < P2; ++c) acc[a][b][c] = 0.0;

    int cur = -1;
    const double* __restrict__ Vr = V + (int64_t)r * vs.rs;
    const int end = it.start + it.count;

    auto flush = [&](int cell) {
        if (SLOTS > 1) {
#pragma unroll
            for (int off = L; off < 32; off <<= 1)
#pragma unroll
                for (int a = 0; a < P0; ++a)
#pragma unroll
                    for (int b = 0; b < P1; ++b)
#pragma unroll
                        for (int c = 0; c < P2; ++c)
                            acc[a][b][c] += __shfl_xor_sync(0xffffffffu, acc[a][b][c], off);
        }
        if (slot == 0) {
            const int l0 = cell & 255, l1 = (cell >> 8) & 255, l2 = (cell >> 16) & 255;
#pragma unroll
            for (int a = 0; a < P0; ++a)
#pragma unroll
                for (int b = 0; b < P1; ++b)
#pragma unroll
                    for (int c = 0; c < P2; ++c) {
                        int ti;
                        if (Q == 3) ti = ((l0 + g0 * P0 + a) * R + (l1 + g1 * P1 + b)) * R + (l2 + g2 * P2 + c);
                        else if (Q == 2) ti = (l0 + g0 * P0 + a) * R + (l1 + g1 * P1 + b);
                        else ti = l0 + g0 * P0 + a;
                        tile[ti] += acc[a][b][c];
                    }
        }
#pragma unroll
        for (int a = 0; a < P0; ++a)
#pragma unroll
            for (int b = 0; b < P1; ++b)
#pragma unroll
                for (int c = 0; c < P2; ++c) acc[a][b][c] = 0.0;
        __syncwarp();
    };

    for (int base = it.start; base < end; base += 32) {
        const int nb = min(32, end - base);
        __syncwarp();
        if (lane < nb) {
            const Point p = pts[base + lane];
            const double val = Vr[(int64_t)p.idx * vs.is];
            double w[T];
            window_weights<T>(wf, p.s[0], w);
#pragma unroll
            for (int a = 0; a < T; ++a) wst[lane][a] = val * w[a];
            if (Q >= 2) {
                window_weights<T>(wf, p.s[1], w);
#pragma unroll
                for (int a = 0; a < T; ++a) wst[lane][T + a] = w[a];
            }
            if (Q >= 3) {
                window_weights<T>(wf, p.s[2], w);
#pragma unroll
                for (int a = 0; a < T; ++a) wst[lane][2 * T + a] = w[a];
            }
            const int l0 = cell_axis(p.cell, 0) - sc0 * S;
            const int l1 = Q >= 2 ? cell_axis(p.cell, 1) - sc1 * S : 0;
            const int l2 = Q >= 3 ? cell_axis(p.cell, 2) - sc2 * S : 0;
            AK_DCHECK(l0 >= 0 && l0 < S && l1 >= 0 && l1 < S && l2 >= 0 && l2 < S);
            cst[lane] = l0 | (l1 << 8) | (l2 << 16);
        }
        __syncwarp();
        for (int k = 0; k < nb;) {
            const int cell = cst[k];
            if (cell != cur) {
                if (cur >= 0) flush(cur);
                cur = cell;
            }
            const int kk = k + slot;
            const bool act = (kk < nb) && (cst[kk < 32 ? kk : 31] == cell);
            const int src = act ? kk : k;
            double w0[P0], w1[P1], w2[P2];
#pragma unroll
            for (int a = 0; a < P0; ++a) w0[a] = act ? wst[src][g0 * P0 + a] : 0.0;
#pragma unroll
            for (int b = 0; b < P1; ++b) w1[b] = Q >= 2 ? wst[src][T + g1 * P1 + b] : 1.0;
#pragma unroll
            for (int c = 0; c < P2; ++c) w2[c] = Q >= 3 ? wst[src][2 * T + g2 * P2 + c] : 1.0;
#pragma unroll
            for (int b = 0; b < P1; ++b)
#pragma unroll
                for (int c = 0; c < P2; ++c) {
                    const double pbc = (Q >= 3) ? w1[b] * w2[c] : w1[b];
#pragma unroll
                    for (int a = 0; a < P0; ++a) acc[a][b][c] = fma(w0[a], pbc, acc[a][b][c]);
                }
            if (SLOTS == 1) {
                k += 1;
            } else {
                const unsigned bal = __ballot_sync(0xffffffffu, act && rl == 0);
                k += __popc(bal);
            }
        }
    }
    if (cur >= 0) flush(cur);
    __syncwarp();

    double* __restrict__ g = grids + (int64_t)nrhs * canon_off[it.window] + (int64_t)r * ipow<Q>(n);
    const int o0 = sc0 * S - (T / 2 - 1);
    const int o1 = sc1 * S - (T / 2 - 1);
    const int o2 = sc2 * S - (T / 2 - 1);
    for (int i = lane; i < TILE; i += 32) {
        const double val = tile[i];
        if (val != 0.0) {
            int64_t gi;
            if (Q == 3) {
                const int i2 = i % R, i1 = (i / R) % R, i0 = i / (R * R);
                gi = ((int64_t)wrap(o0 + i0, n) * n + wrap(o1 + i1, n)) * n + wrap(o2 + i2, n);
            } else if (Q == 2) {
                const int i1 = i % R, i0 = i / R;
                gi = (int64_t)wrap(o0 + i0, n) * n + wrap(o1 + i1, n);
            } else {
                gi = wrap(o0 + i, n);
            }
            red_add(g + gi, val);
        }
    }
}

// ---------------------------------------------------------------------------
// Load the (S+T-1)^Q grid region of a supercell into shared memory.
template <int Q, int T>
__device__ __forceinline__ void load_region(double* tile, const double* __restrict__ g, int n,
                                            int sc0, int sc1, int sc2, int lane)
{
    constexpr int S = SuperCell<Q>::S;
    constexpr int R = S + T - 1;
    constexpr int TILE = ipow<Q>(R);
    const int o0 = sc0 * S - (T / 2 - 1);
    const int o1 = sc1 * S - (T / 2 - 1);
    const int o2 = sc2 * S - (T / 2 - 1);
    for (int i = lane; i < TILE; i += 32) {
        int64_t gi;
        if (Q == 3) {
            const int i2 = i % R, i1 = (i / R) % R, i0 = i / (R * R);
            gi = ((int64_t)wrap(o0 + i0, n) * n + wrap(o1 + i1, n)) * n + wrap(o2 + i2, n);
        } else if (Q == 2) {
            const int i1 = i % R, i0 = i / R;
            gi = (int64_t)wrap(o0 + i0, n) * n + wrap(o1 + i1, n);
        } else {
            gi = wrap(o0 + i, n);
        }
        cp_async8(&tile[i], g + gi);
    }
    cp_async_commit();
    cp_async_wait_all();
}

__device__ __forceinline__ void store_out(double* __restrict__ out, int atomic_out, double v) {
    if (atomic_out) red_add(out, v);
    else *out = v;
}

// Interp for q <= 2 (any T <= 16): one lane per point, footprint read from the
// shared region tile.
template <int Q, int T>
__global__ void __launch_bounds__(32)
k_interp_lane(const Point* __restrict__ pts, const WorkItem* __restrict__ items,
              const double* __restrict__ grids, const int64_t* __restrict__ canon_off, int nrhs,
              int n, const ak_window_fn wf, const double* __restrict__ scale,
              double* __restrict__ out, Strides os, int atomic_out, int64_t wstride)
{
    constexpr int S = SuperCell<Q>::S;
    constexpr int R = S + T - 1;
    constexpr int TILE = ipow<Q>(R);
    __shared__ double tile[TILE];

    const WorkItem it = items[blockIdx.x / nrhs];
    const int r = blockIdx.x % nrhs;
    const int lane = threadIdx.x;
    const int sc0 = it.sc & 1023, sc1 = (it.sc >> 10) & 1023;
    const double* __restrict__ g = grids + (int64_t)nrhs * canon_off[it.window] + (int64_t)r * ipow<Q>(n);
    load_region<Q, T>(tile, g, n, sc0, sc1, 0, lane);
    __syncwarp();
    const double sc = scale[it.window];
    double* __restrict__ o = out + (int64_t)it.window * wstride + (int64_t)r * os.rs;
    const int end = it.start + it.count;
    for (int j = it.start + lane; j < end; j += 32) {
        const Point p = pts[j];
        double w0[T], w1[T];
        window_weights<T>(wf, p.s[0], w0);
        const int l0 = cell_axis(p.cell, 0) - sc0 * S;
        AK_DCHECK(l0 >= 0 && l0 < S);
        double acc = 0.0;
        if (Q == 1) {
#pragma unroll
            for (int a = 0; a < T; ++a) acc = fma(w0[a], tile[l0 + a], acc);
        } else {
            window_weights<T>(wf, p.s[1], w1);
            const int l1 = cell_axis(p.cell, 1) - sc1 * S;
#pragma unroll
            for (int a = 0; a < T; ++a) {
                double s = 0.0;
                const double* row = tile + (l0 + a) * R + l1;
#pragma unroll
                for (int b = 0; b < T; ++b) s = fma(w1[b], row[b], s);
                acc = fma(w0[a], s, acc);
            }
        }
        store_out(o + (int64_t)p.idx * os.is, atomic_out, sc * acc);
    }
}

// ---------------------------------------------------------------------------
// Generic (any q, any taps <= 16) kernels: one thread per point, direct global
// atomics / loads.  Used for non-default cutoffs; correctness reference for
// the tiled kernels in the GPU tests.  Launched per window w (points p0..p0+np).
__global__ void k_spread_generic(const Point* __restrict__ pts, int64_t p0, int64_t np, int q,
                                 const double* __restrict__ V, Strides vs,
                                 double* __restrict__ g_w /* window w, rhs 0 */, int n,
                                 const ak_window_fn wf);
__global__ void k_interp_generic(const Point* __restrict__ pts, int64_t p0, int64_t np, int q,
                                 const double* __restrict__ g_w, int n, const ak_window_fn wf,
                                 const double* __restrict__ scale, int w,
                                 double* __restrict__ out_w /* rhs 0 */, Strides os, int sum_windows);

}  // namespace ak
