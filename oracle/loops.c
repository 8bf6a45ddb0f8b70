/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.  Never linked into, or called by, the
 * product (paper_2404_17344_b200/).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs use it, as the checker or
 * as the timed CPU baseline.
 *
 * Serial C restatement of the reference's numba gridding loops
 * (/root/reference/pkg/src/addkern/nufft.py:197-320): complex128 values and
 * grids (interleaved re/im doubles), per-axis wrapped first-tap indices and
 * per-point tap weights exactly as prepare_points produces them
 * (nufft.py:169-191), row-major grid with the last axis fastest, and the
 * same loop nesting / accumulation order, so results agree with the
 * reference to rounding.
 *
 * One deliberate difference: the reference wraps a tap index with a single
 * `if (i >= n) i -= n` (nufft.py:204-206 and the other loops), which indexes
 * out of bounds when the grid is smaller than the window (n < 2*cutoff, e.g.
 * m <= 4 at cutoff 6) -- undefined behaviour in the numba kernels.  Here the
 * wrap is a loop (full periodic wrap), identical whenever the reference is
 * defined; the CUDA kernels wrap the same way.
 */
#include <stdint.h>

/* _spread_1/2/3 (nufft.py:197-254): grid += values_j * prod_a w_a[j, tap_a] */
void oracle_spread(int q, int64_t N, int T, int64_t n,
                   const int64_t* first,   /* [q][N] */
                   const double* w,        /* [q][N][T] */
                   const double* values,   /* [N][2] complex */
                   double* grid)           /* [n^q][2] complex, accumulated */
{
    const int64_t* f0 = first;
    const int64_t* f1 = first + N;
    const int64_t* f2 = first + 2 * N;
    const double* w0 = w;
    const double* w1 = w + N * T;
    const double* w2 = w + 2 * N * T;
    for (int64_t j = 0; j < N; ++j) {
        const double vr = values[2 * j], vi = values[2 * j + 1];
        for (int a = 0; a < T; ++a) {
            int64_t ia = f0[j] + a;
            while (ia >= n) ia -= n;
            const double ar = vr * w0[j * T + a], ai = vi * w0[j * T + a];
            if (q == 1) {
                grid[2 * ia] += ar;
                grid[2 * ia + 1] += ai;
                continue;
            }
            const int64_t plane = ia * n;
            for (int b = 0; b < T; ++b) {
                int64_t ib = f1[j] + b;
                while (ib >= n) ib -= n;
                const double br = ar * w1[j * T + b], bi = ai * w1[j * T + b];
                if (q == 2) {
                    grid[2 * (plane + ib)] += br;
                    grid[2 * (plane + ib) + 1] += bi;
                    continue;
                }
                const int64_t row = (plane + ib) * n;
                for (int c = 0; c < T; ++c) {
                    int64_t ic = f2[j] + c;
                    while (ic >= n) ic -= n;
                    grid[2 * (row + ic)] += br * w2[j * T + c];
                    grid[2 * (row + ic) + 1] += bi * w2[j * T + c];
                }
            }
        }
    }
}

/* _interp_1/2/3 (nufft.py:257-320): out_j = sum_a w0 sum_b w1 sum_c w2 grid (nested partial sums) */
void oracle_interp(int q, int64_t N, int T, int64_t n,
                   const int64_t* first, const double* w,
                   const double* grid,     /* [n^q][2] */
                   double* out)            /* [N][2], overwritten */
{
    const int64_t* f0 = first;
    const int64_t* f1 = first + N;
    const int64_t* f2 = first + 2 * N;
    const double* w0 = w;
    const double* w1 = w + N * T;
    const double* w2 = w + 2 * N * T;
    for (int64_t j = 0; j < N; ++j) {
        double accr = 0.0, acci = 0.0;
        for (int a = 0; a < T; ++a) {
            int64_t ia = f0[j] + a;
            while (ia >= n) ia -= n;
            double sar, sai;
            if (q == 1) {
                sar = grid[2 * ia];
                sai = grid[2 * ia + 1];
            } else {
                const int64_t plane = ia * n;
                sar = 0.0;
                sai = 0.0;
                for (int b = 0; b < T; ++b) {
                    int64_t ib = f1[j] + b;
                    while (ib >= n) ib -= n;
                    double sbr, sbi;
                    if (q == 2) {
                        sbr = grid[2 * (plane + ib)];
                        sbi = grid[2 * (plane + ib) + 1];
                    } else {
                        const int64_t row = (plane + ib) * n;
                        sbr = 0.0;
                        sbi = 0.0;
                        for (int c = 0; c < T; ++c) {
                            int64_t ic = f2[j] + c;
                            while (ic >= n) ic -= n;
                            sbr += grid[2 * (row + ic)] * w2[j * T + c];
                            sbi += grid[2 * (row + ic) + 1] * w2[j * T + c];
                        }
                    }
                    sar += sbr * w1[j * T + b];
                    sai += sbi * w1[j * T + b];
                }
            }
            accr += sar * w0[j * T + a];
            acci += sai * w0[j * T + a];
        }
        out[2 * j] = accr;
        out[2 * j + 1] = acci;
    }
}
