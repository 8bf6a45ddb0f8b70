// q = 3 spread / interpolation with plan-time window weights ("cached" mode).
//
// The window weights of a 3-D window depend only on the nodes, so the plan
// tabulates them once (k_weights: q*T doubles per point, in bin-sorted
// order, with the same per-tap polynomial the on-the-fly kernels use) and
// the per-product kernels stream them instead of re-evaluating 36 window
// polynomials per point per pass.  That removes ~12% of the FP64 work and the
// latency-bound polynomial phase from every pass, at the price of 288 B of
// HBM traffic per point per pass (~2 TB/s at the kernels' rate: the FP64 pipe
// stays the bound).
//
// Pipeline per work item (one warp), batches of B points:
//   - weight rows of batch b+1 arrive by a TMA bulk copy (cp.async.bulk,
//     mbarrier completion) into the other half of a double buffer while batch
//     b is processed;
//   - (cell, row) records of batch b+2 and the gathered RHS values of batch
//     b+1 arrive by cp.async;
//   - spread multiplies the batch's axis-0 weights by the RHS values in shared
//     memory (element-parallel, conflict-free), then runs the same register-
//     tiled cell-run FMA loop as ak_q3.cuh.
#pragma once
#include "ak_common.cuh"
#include "ak_q3.cuh"

namespace ak {

struct alignas(8) CellIdx {
    int32_t cell;
    int32_t idx;
};


__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "AK_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra AK_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// One elected lane: arm the barrier with `bytes` and start the bulk copy.
__device__ __forceinline__ void tma_load_1d(void* smem, const void* gmem, unsigned bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(smem)),
        "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Plan time: weight rows (axis-major: w0[0..T), w1[0..T), w2[0..T)) and
// (cell, row) records of the points of 2-D / 3-D windows, compact per-window layout.
template <int Q, int T>
__global__ void __launch_bounds__(128) k_weights(const Point* __restrict__ pts, int64_t np, const ak_window_fn wf,
                                                double* __restrict__ W, CellIdx* __restrict__ CI)
{
    // 128 points per block: weights evaluated per thread (unrolled polynomials) into
    // shared memory, then the block's contiguous [128][Q T] slice is stored coalesced.
    __shared__ double st[128 * Q * T];
    const int64_t p0 = (int64_t)blockIdx.x * 128;
    const int64_t j = p0 + threadIdx.x;
    if (j < np) {
        const Point p = pts[j];
        double w[T];
#pragma unroll
        for (int ax = 0; ax < Q; ++ax) {
            window_weights<T>(wf, p.s[ax], w);
#pragma unroll
            for (int a = 0; a < T; ++a) st[threadIdx.x * Q * T + ax * T + a] = w[a];
        }
        CI[j] = CellIdx{p.cell, p.idx};
    }
    __syncthreads();
    const int64_t cnt = (np - p0 < 128 ? np - p0 : 128) * Q * T;
    for (int64_t e = threadIdx.x; e < cnt; e += 128) W[p0 * Q * T + e] = st[e];
}

// acc += v * w0 (x) w1 (x) w2 with v folded into the w1 factor in registers
// (3 extra DMUL per point and lane instead of a per-batch scaling pass).
template <int P0, int P1, int P2>
__device__ __forceinline__ void spread_fma_v(double (&acc)[P0][P1][P2], const double (&w0)[P0],
                                             const double (&w1)[P1], const double (&w2)[P2], double v)
{
    double vw1[P1];
#pragma unroll
    for (int b = 0; b < P1; ++b) vw1[b] = v * w1[b];
#pragma unroll
    for (int b = 0; b < P1; ++b)
#pragma unroll
        for (int c = 0; c < P2; ++c) {
            const double pbc = vw1[b] * w2[c];
#pragma unroll
            for (int a = 0; a < P0; ++a) acc[a][b][c] = fma(w0[a], pbc, acc[a][b][c]);
        }
}

// Wrapped grid index of each region-tile coordinate per axis, in shared memory.
template <int R>
__device__ __forceinline__ void region_axes(int (*widx)[R], int o0, int o1, int o2, int n, int tid, int nthreads) {
    for (int t = tid; t < 3 * R; t += nthreads) {
        const int a = t / R, k = t - a * R;
        const int o = a == 0 ? o0 : (a == 1 ? o1 : o2);
        widx[a][k] = wrap(o + k, n);
    }
}

// Visit the R^3 region tile plane by plane: a warp pass covers 32 / R whole rows
// (lane = row-in-pass x element); each lane keeps its rows' grid offsets in
// registers, so per element the work is one add, and the unrolled row loop keeps
// the elements of a plane independent (ILP for the REDs / cp.asyncs).  Warps of
// a multi-warp CTA take interleaved planes.  f(tile index, grid index).
// Measured on sparse data (config 3, ~15 points per cell): the element-wise loop
// with three constant divisions per element was a quarter of the spread time.
// Region tile layouts: element (i0, i1, i2) at i0 * S0 + i1 * S1 + i2 * S2.
template <int S0, int S1, int S2, int SIZE>
struct TileLayout {
    static constexpr int size = SIZE;
    __host__ __device__ static constexpr int at(int i0, int i1, int i2) { return i0 * S0 + i1 * S1 + i2 * S2; }
};
template <int R>
using DenseTile = TileLayout<R * R, R, 1, R * R * R>;

template <int R, typename F, typename L = DenseTile<R>>
__device__ __forceinline__ void for_region_rows(const int (*widx)[R], int n, int tid, int nthreads, F&& f, L = L{}) {
    static_assert(R <= 32, "region row must fit a warp");
    constexpr int RPP = 32 / R;                 // rows per warp pass
    constexpr int RPL = (R + RPP - 1) / RPP;    // rows per lane per plane
    const int lane = tid & 31;
    const int sub = lane / R, k = lane - sub * R;
    if (sub >= RPP) return;
    const int z = widx[2][k];
    int64_t rowoff[RPL];
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
        const int i1 = sub + RPP * t;
        rowoff[t] = (int64_t)widx[1][i1 < R ? i1 : 0] * n + z;
    }
    for (int i0 = tid >> 5; i0 < R; i0 += nthreads >> 5) {
        const int64_t pl = (int64_t)widx[0][i0] * n * n;
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
            const int i1 = sub + RPP * t;
            AK_DCHECK(i1 >= R || (pl + rowoff[t] >= 0 && pl + rowoff[t] < (int64_t)n * n * n));
            if (i1 < R) f(L::at(i0, i1, k), pl + rowoff[t]);
        }
    }
}

// Shared region tile of the sparse spread.  A cell-run flush adds the lane tiles
// (6 x 3 x 3 per lane: lane (g0, g1, g2) at axis offsets 6 g0, 3 g1, 3 g2) into the
// region with one 8-byte load + store per element; a half-warp's 16 addresses must
// fall on 16 different bank pairs.  In the dense 13^3 layout every flush access is
// 2-way conflicted (3 g1 * 13 + 3 g2 collides mod 16); with axis 2 innermost, axis 0
// at stride 13 and axis 1 at stride 172 (2236 elements, +2%) all 54 are conflict-free
// (exhaustive search over axis orders and paddings: tools/bank_search.py).  Config 3
// (B200): spread 0.862 -> 0.746 ms per launch.
#ifndef AK_SPREAD3W_PAD
#define AK_SPREAD3W_PAD 1
#endif
template <int R>
struct Spread3wTile {
#if AK_SPREAD3W_PAD
    static_assert(R <= 13, "padded layout holds regions up to 13^3");
    using L = TileLayout<13, 172, 1, 13 * 172>;
#else
    using L = DenseTile<R>;
#endif
};

// points per staged weight batch of the sparse (supercell) 3-D kernels
#ifndef AK_SPARSE_BATCH
#define AK_SPARSE_BATCH 16
#endif
#ifndef AK_SPREAD3W_BOUNDS
#define AK_SPREAD3W_BOUNDS __launch_bounds__(32, 8)
#endif
template <int T, int S, int B>
__global__ void AK_SPREAD3W_BOUNDS
k_spread3w(const CellIdx* __restrict__ ci, const double* __restrict__ W, const int64_t* __restrict__ wshift,
           const WorkItem* __restrict__ items, const double* __restrict__ V, Strides vs,
           double* __restrict__ grids, const int64_t* __restrict__ canon_off, int nrhs, int n)
{
    using LN = Q3Lanes<T>;
    constexpr int P0 = LN::P0, P1 = LN::P1, P2 = LN::P2;
    constexpr int RW = 3 * T;
    constexpr int R = S + T - 1;
    using TL = typename Spread3wTile<R>::L;
    constexpr int TILE = TL::size;
    static_assert(B <= 32, "batch must fit the change mask");

    __shared__ double tile[TILE];
    __shared__ __align__(128) double wbuf[2][B][RW];
    __shared__ __align__(16) CellIdx cib[3][B];
    __shared__ double vb[2][B];
    __shared__ int cst[B];
    __shared__ int widx[3][R];
    __shared__ __align__(8) uint64_t bar[2];

    // the RHS index runs fastest: the nrhs CTAs of one item share its weight rows in L2
    const WorkItem it = items[blockIdx.x / nrhs];
    const int r = blockIdx.x % nrhs;
    const int lane = threadIdx.x;
    const int g0 = lane >> 4, g1 = (lane >> 2) & 3, g2 = lane & 3;
    const int sc0 = it.sc & 1023, sc1 = (it.sc >> 10) & 1023, sc2 = (it.sc >> 20) & 1023;
    const double* __restrict__ Vr = V + (int64_t)r * vs.rs;
    const int end = it.start + it.count;
    const int nbatch = (it.count + B - 1) / B;
    const double* __restrict__ Wit = W + (int64_t)(it.start - wshift[it.window]) * RW;
    const CellIdx* __restrict__ CIit = ci + (it.start - wshift[it.window]);

    for (int i = lane; i < TILE; i += 32) tile[i] = 0.0;
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
    int cur = -1;

    auto flush = [&](int cell) {
        const int l0 = cell & 255, l1 = (cell >> 8) & 255, l2 = (cell >> 16) & 255;
#pragma unroll
        for (int a = 0; a < P0; ++a)
#pragma unroll
            for (int b = 0; b < P1; ++b)
#pragma unroll
                for (int c = 0; c < P2; ++c) {
                    double* t = &tile[TL::at(l0 + g0 * P0 + a, l1 + g1 * P1 + b, l2 + g2 * P2 + c)];
                    *t += acc[a][b][c];
                    acc[a][b][c] = 0.0;
                }
        __syncwarp();
    };

    for (int bi = 0; bi < nbatch; ++bi) {
        const int s = bi & 1;
        const int off = bi * B;  // offset of this batch within the item
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
        {
            // axis-0 weights times the RHS value, element-parallel over the batch
            constexpr int PER = (B * T + 31) / 32;  // elements of the batch's w0 block per lane
            double x[PER], y[PER];
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const int e = lane + 32 * i;
                const int row = e / T;
                if (row < nb) {
                    x[i] = wbuf[s][row][e - row * T];
                    y[i] = vb[s][row];
                }
            }
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const int e = lane + 32 * i;
                const int row = e / T;
                if (row < nb) wbuf[s][row][e - row * T] = x[i] * y[i];
            }
        }
        if (lane < nb) {
            const int c = cib[bi % 3][lane].cell;
            AK_DCHECK(cell_axis(c, 0) - sc0 * S >= 0 && cell_axis(c, 0) - sc0 * S < S &&
                      cell_axis(c, 1) - sc1 * S >= 0 && cell_axis(c, 1) - sc1 * S < S &&
                      cell_axis(c, 2) - sc2 * S >= 0 && cell_axis(c, 2) - sc2 * S < S);
            cst[lane] = (cell_axis(c, 0) - sc0 * S) | ((cell_axis(c, 1) - sc1 * S) << 8) |
                        ((cell_axis(c, 2) - sc2 * S) << 16);
        }
        __syncwarp();
        const int mycell = lane < nb ? cst[lane] : -2;
        const int prev = __shfl_up_sync(0xffffffffu, mycell, 1);
        const unsigned chg = __ballot_sync(0xffffffffu, lane < nb && (lane == 0 ? mycell != cur : mycell != prev));
        for (int k = 0; k < nb;) {
            if ((chg >> k) & 1u) {
                if (cur >= 0) flush(cur);
                cur = cst[k];
            }
            const unsigned later = k < 31 ? chg & ~((2u << k) - 1u) : 0u;
            const int kend = later ? min(__ffs(later) - 1, nb) : nb;
            double a0[P0], a1[P1], a2[P2], b0[P0], b1[P1], b2[P2];
            load_w<T>(a0, a1, a2, &wbuf[s][k][0], g0, g1, g2);
            int j = k;
            for (; j + 1 < kend; j += 2) {
                load_w<T>(b0, b1, b2, &wbuf[s][j + 1][0], g0, g1, g2);
                spread_fma(acc, a0, a1, a2);
                const int jn = j + 2 < kend ? j + 2 : j + 1;
                load_w<T>(a0, a1, a2, &wbuf[s][jn][0], g0, g1, g2);
                spread_fma(acc, b0, b1, b2);
            }
            if (j < kend) spread_fma(acc, a0, a1, a2);
            k = kend;
        }
    }
    if (cur >= 0) flush(cur);
    __syncwarp();

    double* __restrict__ g = grids + (int64_t)nrhs * canon_off[it.window] + (int64_t)r * n * n * n;
    region_axes<R>(widx, sc0 * S - (T / 2 - 1), sc1 * S - (T / 2 - 1), sc2 * S - (T / 2 - 1), n, lane, 32);
    __syncwarp();
    for_region_rows<R>(
        widx, n, lane, 32,
        [&](int i, int64_t gi) {
            const double val = tile[i];
            if (val != 0.0) red_add(g + gi, val);
        },
        TL{});
    (void)end;
}

}  // namespace ak
