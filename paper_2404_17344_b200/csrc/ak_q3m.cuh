// q = 3 interpolation on the FP64 tensor cores (mma.sync m8n8k4 f64), T = 12.
//
// For the points of one cell the interpolation is a small GEMM followed by two
// cheap contractions:
//   U[j, (a,b)] = sum_c w2_j[c] G[a,b,c]          (8 points x 144 pairs, K = 12 = 3 k-steps)
//   out_j       = sum_a w0_j[a] sum_b w1_j[b] U[j, (a,b)]
// The first stage (1728 FMA per point, 90% of the work) runs as 54 DMMA per 8
// points: A = w2 of the 8 points (row-major 8x4 fragment), B = the cell's
// footprint G (col-major 4x8 fragments, held in registers while the cell
// lasts, 54 doubles per lane), C = U (18 tiles, 36 doubles per lane).  The
// B columns are permuted so that lane quad q (lane % 4) holds exactly the
// pairs (a, b) with b in {3q, 3q+1, 3q+2}, which makes the second stage a
// compile-time-indexed 39-op contraction per lane followed by a 2-step quad
// shuffle.  DMMA and DFMA share the FP64 datapath (37 TF/s either way on
// B200), so the gain is not peak rate but issue pressure: ~135 instructions
// per 8 points per lane instead of ~700, and 1884 instead of 2144 FP64 slots
// per point.  Partially filled groups (run ends) are padded with zero rows.
#pragma once
#include "ak_q3w.cuh"

namespace ak {

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// One group of up to 8 points (rows k0 .. k0+cnt-1 of the staged batch), all in the
// cell whose fragments are in gf.  Returns this lane's quad-partial for point
// k0 + lane/4 (summed over the quad by the caller).  A = active taps on axis 0
// (12, or 10 for a zero-padded 10-tap window: taps 1..10, 15 instead of 18 tiles).
template <int RW, int A = 12>
__device__ __forceinline__ double interp_group_mma(const double (&gf)[3 * A / 2][3], const double (*wrow)[RW],
                                                   int k0, int cnt, int lane)
{
    constexpr int NT = 3 * A / 2, AO = (12 - A) / 2;
    const int pj = lane >> 2, q = lane & 3;
    const bool valid = pj < cnt;
    const double* w = wrow[k0 + (valid ? pj : 0)];
    double af[3];
#pragma unroll
    for (int ks = 0; ks < 3; ++ks) af[ks] = valid ? w[24 + 4 * ks + q] : 0.0;
    double C[NT][2];
#pragma unroll
    for (int t = 0; t < NT; ++t) C[t][0] = C[t][1] = 0.0;
    // k-step outer: NT independent accumulators between dependent DMMAs
#pragma unroll
    for (int ks = 0; ks < 3; ++ks)
#pragma unroll
        for (int t = 0; t < NT; ++t) dmma_8x8x4(C[t][0], C[t][1], af[ks], gf[t][ks]);
    // lane (pj, q) holds U[pj][(a, b)] for a = AO + i/3, b = 3q + i%3, i = 2t + e:
    // out = sum_b w1[b] (sum_a w0[a] U[a][b]) -- 3 chains of A FMAs, then 3 more
    // (2 / 3 interleaved partial sums per b: config 4 interp 1.231 -> 1.287 / 1.302 ms)
    double s[3];
#pragma unroll
    for (int bb = 0; bb < 3; ++bb) s[bb] = w[AO] * C[bb >> 1][bb & 1];
#pragma unroll
    for (int a = 1; a < A; ++a) {
        const double w0a = w[AO + a];
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) {
            const int i = 3 * a + bb;
            s[bb] = fma(w0a, C[i >> 1][i & 1], s[bb]);
        }
    }
    const double* w1 = w + 12 + 3 * q;
    const double v = fma(w1[2], s[2], fma(w1[1], s[1], w1[0] * s[0]));
    return valid ? v : 0.0;
}

// Per-lane tile offsets of the 18 permuted B-fragment columns: column n = lane/4 of
// tile t is pair i = 2t + (n & 1) of quad n >> 1, i.e. a = i / 3, b = 3 (n >> 1) + i % 3;
// row kk = lane % 4 of k-step ks is c = 4 ks + kk.
template <int R>
__device__ __forceinline__ void fragment_offsets(int (&off)[18], int lane) {
    const int n = lane >> 2, kk = lane & 3;
    const int qq = n >> 1, e = n & 1;
#pragma unroll
    for (int t = 0; t < 18; ++t) {
        const int i = 2 * t + e;
        off[t] = ((i / 3) * R + 3 * qq + i % 3) * R + kk;
    }
}

// Region tile of the sparse interpolation and its B-fragment columns.  Lane column n
// = lane / 4 of tile t is (a, b) = (t / 3 + 6 (n & 1), 3 (n >> 1) + t % 3) -- lane quad q
// = n >> 1 still owns b = 3q .. 3q+2 (the contraction below), but the two columns of a
// lane pair are 6 apart in a, and the tile keeps a innermost: element (a, b, c) at
// a + 13 b + 172 c.  Then the 16 addresses of every half-warp fragment load fall on 16
// different bank pairs (tools/bank_search.py: 108 wavefronts per 54 loads, the
// minimum; the dense 13^3 tile with the pairs (i / 3, i % 3), i = 2t + (n & 1), of
// interp_group_mma costs 216 -- ncu: 38% of the shared wavefronts were conflicts).
// Measured on config 3 (B200): shared wavefronts per launch 105 M -> 83 M, kernel time
// unchanged within 0.2% (1.358 vs 1.356 ms per step for the dense layout with the same
// pairing, AK_INTERP3M_PAD=0): the DMMA group stream, not shared memory, bounds it.
#ifndef AK_INTERP3M_PAD
#define AK_INTERP3M_PAD 1
#endif
template <int R>
struct Interp3mTile {
#if AK_INTERP3M_PAD
    using L = typename std::conditional<R == 13, TileLayout<1, 13, 172, 12 + 12 * 13 + 12 * 172 + 1>,
                                        TileLayout<1, R, R * R, R * R * R>>::type;
#else
    using L = DenseTile<R>;
#endif
};
template <class L>
__device__ __forceinline__ void fragment_offsets_s(int (&off)[18], int lane) {
    const int n = lane >> 2, kk = lane & 3;
#pragma unroll
    for (int t = 0; t < 18; ++t) off[t] = L::at(t / 3 + 6 * (n & 1), 3 * (n >> 1) + t % 3, kk);
}

// G consecutive 8-point groups of one cell run (rows k0 + 8 g + pj, cnt[g] valid rows
// each) against the same footprint: the B fragments are read from the region tile
// once per run segment instead of once per group.  The 18 column tiles run in three
// chunks of six (tiles 6 ch .. 6 ch + 5: a in {2ch, 2ch+1, 2ch+6, 2ch+7}, lane quad q
// owning b = 3q .. 3q+2 as above): per chunk each group's 6 accumulator tiles are
// contracted over a right away, so a lane holds 18 fragments + 12 accumulators
// instead of 36 accumulators.
template <class L, int RW, int G>
__device__ __forceinline__ void interp_groups_mma_s(const double* cb, const int (&off)[18], const double (*wrow)[RW],
                                                    int k0, const int (&cnt)[G], int lane, double (&v)[G])
{
    constexpr int CS = L::at(0, 0, 1);   // stride of c in the tile
    const int pj = lane >> 2, q = lane & 3;
    const double* w[G];
    double af[G][3], s[G][3];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const bool valid = pj < cnt[g];
        w[g] = wrow[k0 + 8 * g + (valid ? pj : 0)];
#pragma unroll
        for (int ks = 0; ks < 3; ++ks) af[g][ks] = valid ? w[g][24 + 4 * ks + q] : 0.0;
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) s[g][bb] = 0.0;
    }
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        double B[6][3];
#pragma unroll
        for (int tt = 0; tt < 6; ++tt)
#pragma unroll
            for (int ks = 0; ks < 3; ++ks) B[tt][ks] = cb[off[6 * ch + tt] + 4 * ks * CS];
        // every group's DMMAs first, then the contractions (no DMMA -> DFMA latency wait
        // between them when G = 2)
        double C[G][6][2];
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
            for (int tt = 0; tt < 6; ++tt) C[g][tt][0] = C[g][tt][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < 3; ++ks)
#pragma unroll
            for (int g = 0; g < G; ++g)
#pragma unroll
                for (int tt = 0; tt < 6; ++tt) dmma_8x8x4(C[g][tt][0], C[g][tt][1], af[g][ks], B[tt][ks]);
#pragma unroll
        for (int g = 0; g < G; ++g)
            // column e of tile 6 ch + tt: a = 2 ch + tt / 3 + 6 e, b = 3 q + tt % 3
#pragma unroll
            for (int tt = 0; tt < 6; ++tt)
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    s[g][tt % 3] = fma(w[g][2 * ch + tt / 3 + 6 * e], C[g][tt][e], s[g][tt % 3]);
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const double* w1 = w[g] + 12 + 3 * q;
        const double r = fma(w1[2], s[g][2], fma(w1[1], s[g][1], w1[0] * s[g][0]));
        v[g] = pj < cnt[g] ? r : 0.0;
    }
}

// Multi-cell (supercell) work items: the item's (S+11)^3 grid region is staged in
// shared memory once, and the 8-point groups of a cell run read their B fragments
// from it inside the DMMA loop (no per-cell register copy of the footprint).
// NW (1 or 2) warps share the region tile (read only); each takes a contiguous part
// of the item (split at a cell boundary) and walks it in batches of at most B points
// with its own double-buffered weight rows and barriers (the tile is 17.6 KB at
// S = 2: one warp per CTA leaves shared memory, not registers, as the occupancy
// limit).  Batches end at their last cell-run start when more points follow, so a
// run is never cut by a batch boundary except after 16 of its points: a run of L
// points takes ceil(L / 8) groups.  (Fixed 16-point batches cut ~40% of the runs;
// at ~12 points per cell the groups were 67% full instead of 78%.)
template <int S, int B, int NW>
#ifndef AK_INTERP3M_MINW
#define AK_INTERP3M_MINW 10   // warps per SM the register allocation must allow
#endif
__global__ void __launch_bounds__(32 * NW, AK_INTERP3M_MINW / NW)
k_interp3m(const CellIdx* __restrict__ ci, const double* __restrict__ W, const int64_t* __restrict__ wshift,
           const WorkItem* __restrict__ items, const double* __restrict__ grids,
           const int64_t* __restrict__ canon_off, int nrhs, int n, const double* __restrict__ scale,
           double* __restrict__ out, Strides os, int atomic_out, int64_t wstride)
{
    constexpr int T = 12;
    constexpr int RW = 3 * T;
    constexpr int R = S + T - 1;
    using TL = typename Interp3mTile<R>::L;
    constexpr int TILE = TL::size;
    static_assert(B % 16 == 0 && B <= 32, "batch: multiple of 16, at most 32");
    static_assert(NW == 1 || NW == 2, "one or two warps per item");
    constexpr unsigned FULL = 0xffffffffu;

    __shared__ double tile[TILE];
    __shared__ __align__(128) double wbuf_all[NW][2][B][RW];
    __shared__ __align__(16) CellIdx cib_all[NW][2][B];
    __shared__ int cst_all[NW][B];
    __shared__ int widx[3][R];
    __shared__ __align__(8) uint64_t bar_all[NW][2];

    // the RHS index runs fastest: the nrhs CTAs of one item share its weight rows in L2
    const WorkItem it = items[blockIdx.x / nrhs];
    const int r = blockIdx.x % nrhs;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    double (*wbuf)[B][RW] = wbuf_all[warp];
    CellIdx (*cib)[B] = cib_all[warp];
    int* cst = cst_all[warp];
    uint64_t* bar = bar_all[warp];
    const int sc0 = it.sc & 1023, sc1 = (it.sc >> 10) & 1023, sc2 = (it.sc >> 20) & 1023;
    const double* __restrict__ Wit = W + (int64_t)(it.start - wshift[it.window]) * RW;
    const CellIdx* __restrict__ CIit = ci + (it.start - wshift[it.window]);

    // this warp's points [off, wend): two warps split the item at the first cell-run
    // start at or after its middle (within 32 points; else at the middle)
    int off = 0, wend = it.count;
    if (NW == 2) {
        const int mid = it.count / 2, j = mid + lane;
        const bool bd = j > 0 && j < it.count && CIit[j].cell != CIit[j - 1].cell;
        const unsigned m = __ballot_sync(FULL, bd);
        const int split = m ? mid + __ffs(m) - 1 : mid;
        off = warp ? split : 0;
        wend = warp ? it.count : split;
    }

    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncwarp();
    if (off < wend) {
        const int cnt = min(B, wend - off);
        if (lane == 0) tma_load_1d(&wbuf[0][0][0], Wit + (int64_t)off * RW, (unsigned)(cnt * RW * 8), &bar[0]);
        if (lane < cnt) cp_async8(&cib[0][lane], CIit + off + lane);
    }
    {
        const double* __restrict__ g = grids + (int64_t)nrhs * canon_off[it.window] + (int64_t)r * n * n * n;
        region_axes<R>(widx, sc0 * S - (T / 2 - 1), sc1 * S - (T / 2 - 1), sc2 * S - (T / 2 - 1), n, threadIdx.x,
                       32 * NW);
        if (NW > 1) __syncthreads();
        else __syncwarp();
        for_region_rows<R>(widx, n, threadIdx.x, 32 * NW, [&](int i, int64_t gi) { cp_async8(&tile[i], g + gi); },
                           TL{});
    }
    cp_async_commit();
    cp_async_wait_all();
    if (NW > 1) __syncthreads();
    else __syncwarp();
    const double sc = scale[it.window];
    double* __restrict__ o = out + (int64_t)it.window * wstride + (int64_t)r * os.rs;

    int foff[18];
    fragment_offsets_s<TL>(foff, lane);
    const double* cb = tile;
    int cur = -1;
    const int pj = lane >> 2;

    for (int u = 0; off < wend; ++u) {
        const int s = u & 1;
        const int nb = min(B, wend - off);
        cp_async_wait_all();
        mbar_wait(&bar[s], (u >> 1) & 1);
        __syncwarp();
        if (lane < nb) {
            const int c = cib[s][lane].cell;
            AK_DCHECK(cell_axis(c, 0) - sc0 * S >= 0 && cell_axis(c, 0) - sc0 * S < S &&
                      cell_axis(c, 1) - sc1 * S >= 0 && cell_axis(c, 1) - sc1 * S < S &&
                      cell_axis(c, 2) - sc2 * S >= 0 && cell_axis(c, 2) - sc2 * S < S);
            cst[lane] = (cell_axis(c, 0) - sc0 * S) | ((cell_axis(c, 1) - sc1 * S) << 8) |
                        ((cell_axis(c, 2) - sc2 * S) << 16);
        }
        __syncwarp();
        const int mycell = lane < nb ? cst[lane] : -2;
        const int prev = __shfl_up_sync(FULL, mycell, 1);
        // run starts inside the batch; the batch's last (possibly unfinished) run moves
        // to the next batch when more points follow
        const unsigned inner = __ballot_sync(FULL, lane > 0 && lane < nb && mycell != prev);
        const int take = (off + nb < wend && inner) ? 31 - __clz(inner) : nb;
        const int next = off + take;
        if (next < wend) {
            const int nb1 = min(B, wend - next);
            if (lane == 0) {
                fence_proxy_async();
                tma_load_1d(&wbuf[s ^ 1][0][0], Wit + (int64_t)next * RW, (unsigned)(nb1 * RW * 8), &bar[s ^ 1]);
            }
            if (lane < nb1) cp_async8(&cib[s ^ 1][lane], CIit + next + lane);
        }
        cp_async_commit();
        const unsigned chg = __ballot_sync(FULL, lane < take && (lane == 0 ? mycell != cur : mycell != prev));
        for (int k = 0; k < take;) {
            if ((chg >> k) & 1u) {
                cur = cst[k];
                cb = tile + TL::at(cur & 255, (cur >> 8) & 255, (cur >> 16) & 255);
            }
            const unsigned later = k < 31 ? chg & ~((2u << k) - 1u) : 0u;
            const int kend = later ? min(__ffs(later) - 1, take) : take;
            // two groups per pass while the run has more than 8 points left
            for (int k0 = k; k0 < kend; k0 += 16) {
                const int c0 = min(8, kend - k0), c1 = min(8, kend - k0 - 8);
                auto emit = [&](int g, int cnt, double v) {
                    v += __shfl_xor_sync(FULL, v, 1);
                    v += __shfl_xor_sync(FULL, v, 2);
                    if ((lane & 3) == 0 && pj < cnt) {
                        double* dst = o + (int64_t)cib[s][k0 + 8 * g + pj].idx * os.is;
                        if (atomic_out) red_add(dst, sc * v);
                        else *dst = sc * v;
                    }
                };
                if (c1 > 0) {
                    const int cnt[2] = {c0, c1};
                    double v[2];
                    interp_groups_mma_s<TL, RW, 2>(cb, foff, wbuf[s], k0, cnt, lane, v);
                    emit(0, c0, v[0]);
                    emit(1, c1, v[1]);
                } else {
                    const int cnt[1] = {c0};
                    double v[1];
                    interp_groups_mma_s<TL, RW, 1>(cb, foff, wbuf[s], k0, cnt, lane, v);
                    emit(0, c0, v[0]);
                }
            }
            k = kend;
        }
        off = next;
    }
}

}  // namespace ak
