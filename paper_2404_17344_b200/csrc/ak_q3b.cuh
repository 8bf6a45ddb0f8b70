// q = 3 spread of 8 right-hand sides per CTA over supercell items, on the FP64 tensor
// cores (sparse 3-D windows, RHS-minor data).
//
// A supercell item (2^3 cells, ~15 points per occupied cell in config 3) spreads into
// a 13^3 region.  Per RHS chunk of 8 the region update is one GEMM over the item's
// points, whatever cell each point is in:
//   G[(r, a')][(b', c')] += sum_j (v_jr w0'_j[a']) (w1'_j[b'] w2'_j[c'])
//   rows (r, a') = 8 x 13 = 104 = 13 m-tiles, columns (b', c') = 169 -> 22 n-tiles,
//   K = the item's points in k-steps of 4,
// where w'_j[x'] = w_j[x' - u_j] is the point's 12-tap weight row shifted by its cell
// offset u_j in {0, 1} inside the supercell (zero outside).  Rows and columns waste
// (12/13)^3 x 169/176 = 24% of the MACs on the footprint shifts, but nothing else:
// the k-steps run across cell boundaries (no per-cell-run flush, no partially filled
// groups), and the 8 RHS share every B fragment.  The DFMA kernel this replaces
// (k_spread3w, one RHS per warp) flushes its register tile into a shared region tile
// at every cell change: config 3 spread 0.745 ms there, 0.687 ms here.
// CTA = 4 warps, one (item, RHS chunk, column part): part p of 3 holds n-tiles
// [22p/3, 22(p+1)/3), warp w of them w and w + 4 and all 13 m-tiles (at most 52
// accumulator doubles per lane), so several CTAs share an SM and one's prologue /
// flush overlaps another's DMMA stream; the item's accumulators are added to the
// grids with RED.F64 at the end.  Per batch of B points the
// weight rows arrive by a TMA bulk copy (double-buffered), the (cell, row) records
// and the 8 RHS values of each point by cp.async, and the CTA writes the A operand
// (v_jr w0'_j[a'], 104 values per point) to shared memory once for all warps.
#pragma once
#include "ak_q3r.cuh"

#ifndef AK_SPREAD3B_UNROLL
#define AK_SPREAD3B_UNROLL 2
#endif

namespace ak {

// warps per CTA and CTAs (column parts) per (item, RHS chunk)
// (config 3, B200: 6 warps x 2 parts 0.687 ms, 4 x 3 0.654 (default), 5 x 3 0.861,
// 3 x 4 0.851, one CTA of 11 warps per item 0.852; with 4 x 3: 32-point batches
// 0.661, 40 0.662, 64 0.752)
#ifndef AK_SPREAD3B_WARPS
#define AK_SPREAD3B_WARPS 4
#endif
#ifndef AK_SPREAD3B_PARTS
#define AK_SPREAD3B_PARTS 3
#endif
constexpr int Q3B_WARPS = AK_SPREAD3B_WARPS;
constexpr int Q3B_PARTS = AK_SPREAD3B_PARTS;
static_assert(2 * Q3B_WARPS * Q3B_PARTS >= 22, "22 n-tiles, at most two per warp");
#ifndef AK_SPREAD3B_BATCH
#define AK_SPREAD3B_BATCH 48       // points per staged batch (config 3: 32 -> 0.734 ms, 48 -> 0.687, 64 -> 0.693)
#endif
constexpr int Q3B_LDA = 108;   // A row stride (doubles): fragment loads (k = lane % 4 rows) conflict-free

template <int B>
struct alignas(128) Spread3bSmem {
    double wbuf[2][B][36];
    double A[B][Q3B_LDA];
    double vb[2][B][8];
    CellIdx cib[3][B];
    uint64_t bar[2];
};

template <int B>
inline size_t spread3b_smem() { return sizeof(Spread3bSmem<B>); }

template <int B>
__global__ void __launch_bounds__(32 * Q3B_WARPS, 12 / Q3B_WARPS)
k_spread3b(const CellIdx* __restrict__ ci, const double* __restrict__ W, const int64_t* __restrict__ wshift,
           const WorkItem* __restrict__ items, const double* __restrict__ V, Strides vs,
           double* __restrict__ grids, const int64_t* __restrict__ canon_off, int nrhs, int n)
{
    constexpr int T = 12, RW = 3 * T, S = 2, RG = S + T - 1;   // region edge 13
    constexpr int MT = RG;                                     // 13 m-tiles: rows (r, a') = 8 x 13
    constexpr int NCOL = RG * RG;                              // 169 columns (b', c')
    constexpr int NTH = 32 * Q3B_WARPS;
    static_assert(B % 4 == 0 && B <= NTH, "batch");
    extern __shared__ __align__(128) unsigned char q3b_raw[];
    auto& sm = *reinterpret_cast<Spread3bSmem<B>*>(q3b_raw);
    auto& wbuf = sm.wbuf;
    auto& vb = sm.vb;
    auto& cib = sm.cib;
    auto& bar = sm.bar;

    const int nch = nrhs / 8;
    const WorkItem it = items[blockIdx.x / (Q3B_PARTS * nch)];
    const int rc = (blockIdx.x / Q3B_PARTS) % nch;   // RHS chunk and column part run fastest: the CTAs
    const int part = blockIdx.x % Q3B_PARTS;         // of an item share its weight rows in L2
    const int pbeg = 22 * part / Q3B_PARTS, pcnt = 22 * (part + 1) / Q3B_PARTS - pbeg;   // n-tiles
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int lr = lane >> 2, kk = lane & 3;
    const double* __restrict__ V0 = V + (int64_t)(8 * rc) * vs.rs;
    const int nbatch = (it.count + B - 1) / B;
    const double* __restrict__ Wit = W + (int64_t)(it.start - wshift[it.window]) * RW;
    const CellIdx* __restrict__ CIit = ci + (it.start - wshift[it.window]);
    const int sc0 = it.sc & 1023, sc1 = (it.sc >> 10) & 1023, sc2 = (it.sc >> 20) & 1023;

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
    for (int e = tid; e < 8 * min(B, it.count); e += NTH) {
        const int j = e >> 3, r = e & 7;
        cp_async8(&vb[0][j][r], V0 + (int64_t)r * vs.rs + (int64_t)cib[0][j].idx * vs.is);
    }
    cp_async_commit();

    // this lane's B-fragment columns: n-tile pbeg + warp + W t, column 8 nt + lr -> (b', c')
    int bcol[2], ccol[2];
    bool cok[2];
    const bool one = warp < pcnt, two = warp + Q3B_WARPS < pcnt;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const int col = 8 * (pbeg + warp + Q3B_WARPS * t) + lr;
        cok[t] = col < NCOL && (t == 0 ? one : two);
        bcol[t] = col / RG;
        ccol[t] = col - bcol[t] * RG;
    }
    double acc[MT][2][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int t = 0; t < 2; ++t) acc[i][t][0] = acc[i][t][1] = 0.0;

    for (int bi = 0; bi < nbatch; ++bi) {
        const int s = bi & 1;
        const int off = bi * B;
        const int nb = min(B, it.count - off);
        const CellIdx* cb = cib[bi % 3];
        cp_async_wait_all();
        mbar_wait(&bar[s], (bi >> 1) & 1);
        __syncthreads();   // batch bi visible; every warp is done with batch bi - 1 (A, wbuf[s ^ 1], vb[s ^ 1])
        if (bi + 1 < nbatch) {
            const int nb1 = min(B, it.count - off - B);
            if (tid == 0) {
                fence_proxy_async();
                tma_load_1d(&wbuf[s ^ 1][0][0], Wit + (int64_t)(off + B) * RW, (unsigned)(nb1 * RW * 8), &bar[s ^ 1]);
            }
            for (int e = tid; e < 8 * nb1; e += NTH) {
                const int j = e >> 3, r = e & 7;
                cp_async8(&vb[s ^ 1][j][r], V0 + (int64_t)r * vs.rs + (int64_t)cib[(bi + 1) % 3][j].idx * vs.is);
            }
        }
        if (bi + 2 < nbatch && tid < min(B, it.count - off - 2 * B))
            cp_async8(&cib[(bi + 2) % 3][tid], CIit + off + 2 * B + tid);
        cp_async_commit();
        // A operand of the batch: A[j][(r, a')] = v_jr w0_j[a' - u0_j] (zero outside the
        // footprint and for rows past nb); one thread per (point, RHS)
        for (int e = tid; e < B * 8; e += NTH) {
            const int j = e >> 3, r = e & 7;
            double* dst = &sm.A[j][r * RG];
            if (j < nb) {
                const int u0 = cell_axis(cb[j].cell, 0) - sc0 * S;
                AK_DCHECK(u0 >= 0 && u0 < S);
                const double v = vb[s][j][r];
                const double* w0 = wbuf[s][j];
                dst[0] = u0 ? 0.0 : v * w0[0];
#pragma unroll
                for (int a = 1; a < T; ++a) dst[a] = v * w0[u0 ? a - 1 : a];
                dst[T] = u0 ? v * w0[T - 1] : 0.0;
            } else {
#pragma unroll
                for (int a = 0; a < RG; ++a) dst[a] = 0.0;
            }
        }
        __syncthreads();
AK_UNROLL(AK_SPREAD3B_UNROLL)
        for (int k0 = 0; k0 < nb; k0 += 4) {
            const int j = k0 + kk;
            const bool valid = j < nb;
            const int jj = valid ? j : 0;
            const double* w = wbuf[s][jj];
            const int cell = cb[jj].cell;
            const int u1 = cell_axis(cell, 1) - sc1 * S, u2 = cell_axis(cell, 2) - sc2 * S;
            AK_DCHECK(!valid || (u1 >= 0 && u1 < S && u2 >= 0 && u2 < S));
            double bf[2];
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const int ib = bcol[t] - u1, ic = ccol[t] - u2;
                const bool on = valid && cok[t] && (unsigned)ib < (unsigned)T && (unsigned)ic < (unsigned)T;
                const double p = w[T + (on ? ib : 0)] * w[2 * T + (on ? ic : 0)];
                bf[t] = on ? p : 0.0;
            }
            double af[MT];
#pragma unroll
            for (int i = 0; i < MT; ++i) af[i] = sm.A[j < B ? j : 0][8 * i + lr];
#pragma unroll
            for (int i = 0; i < MT; ++i) dmma_8x8x4(acc[i][0][0], acc[i][0][1], af[i], bf[0]);
            if (two) {
#pragma unroll
                for (int i = 0; i < MT; ++i) dmma_8x8x4(acc[i][1][0], acc[i][1][1], af[i], bf[1]);
            }
        }
    }

    // flush: lane holds C[row = 8 i + lr][col = 8 nt + 2 kk + e] -> region (r, a', b', c')
    const int o0 = sc0 * S - (T / 2 - 1), o1 = sc1 * S - (T / 2 - 1), o2 = sc2 * S - (T / 2 - 1);
    const int64_t n3 = (int64_t)n * n * n;
    double* __restrict__ g0 = grids + (int64_t)nrhs * canon_off[it.window] + (int64_t)(8 * rc) * n3;
    int coff[2][2];
    bool ok[2][2];
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int col = 8 * (pbeg + warp + Q3B_WARPS * t) + 2 * kk + e;
            ok[t][e] = col < NCOL && (t == 0 ? one : two);
            const int b = ok[t][e] ? col / RG : 0, c = ok[t][e] ? col - (col / RG) * RG : 0;
            coff[t][e] = wrap(o1 + b, n) * n + wrap(o2 + c, n);
        }
    // rows: (r, a') = (row / 13, row % 13), row = 8 i + lr, walked incrementally
    int r = lr / RG, ap = lr - (lr / RG) * RG;
    const int64_t nn = (int64_t)n * n;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
        double* gp = g0 + r * n3 + wrap(o0 + ap, n) * nn;
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int e = 0; e < 2; ++e)
                if (ok[t][e]) red_add(gp + coff[t][e], acc[i][t][e]);
        ap += 8;
        if (ap >= RG) {
            ap -= RG;
            ++r;
        }
    }
}

}  // namespace ak
