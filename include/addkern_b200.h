/*
 * addkern_b200.h -- C ABI of the B200 (sm_100a) NFFT fast-summation path.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `addkern` (arXiv 2404.17344).  The reference runs it in-process as numba
 * kernels called from numpy code; the entry points below replace, one for
 * one, the pieces of that path (citations are /root/reference/pkg/src/addkern):
 *
 *   ak_geom_create     prepare_points            nufft.py:169-191
 *                      (called per window by build_plan, fastsum.py:128-130)
 *   ak_spread          _spread_1/_spread_2/_spread_3 nufft.py:197-254
 *   ak_interp          _interp_1/_interp_2/_interp_3 nufft.py:257-320
 *   ak_op_apply        the per-window loop of fast_matvec fastsum.py:150-160
 *                      (type-1 NUFFT nufft.py:346-365 -> coefficient multiply
 *                      fastsum.py:159 -> type-2 NUFFT nufft.py:368-394, summed
 *                      over windows and scaled, fastsum.py:136-138)
 *   ak_type1_band      fftn + band + deconvolution of nufft_type1 (nufft.py:362-365)
 *   ak_type2_grid      deconvolution + zero-pad + ifftn of nufft_type2 (nufft.py:379-383)
 *   ak_dense_apply     dense_matvec / dense_cross_matvec / dense_matrix (kernels.py:92-170)
 *   ak_cg_step         the body of one cg_solve iteration after the product (solver.py:63-77)
 *   ak_cg_step_batched the same for the grid search's cells in lockstep (solver.py:157-198)
 *
 * Conventions
 *  - All array pointers are DEVICE pointers owned by the caller unless noted.
 *    Scalars and small descriptor arrays are host memory and are copied.
 *  - `stream` is a cudaStream_t passed as void*; NULL means the legacy stream.
 *    Every call is stream-ordered and asynchronous unless documented.
 *  - Return value: AK_OK (0) or a negative AK_ERR_* code.  Nothing throws
 *    across the ABI; ak_last_error() returns a thread-local message.
 *  - Handles are immutable after creation (ak_op owns mutable workspace: use
 *    one ak_op per concurrent stream).
 *  - Arithmetic is IEEE float64 throughout (real arithmetic: for real inputs
 *    the reference's complex pipeline has an exactly zero imaginary part up to
 *    rounding, fastsum.py:141-147).
 */
#ifndef ADDKERN_B200_H
#define ADDKERN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AK_OK              0
#define AK_ERR_INVALID    -1   /* bad argument (maps to ValueError)                  */
#define AK_ERR_CUDA       -2   /* CUDA runtime error                                  */
#define AK_ERR_DOMAIN     -3   /* point outside [-1/2,1/2) (PointOutOfDomainError)    */
#define AK_ERR_ALLOC      -4   /* device allocation failed                            */
#define AK_ERR_CUFFT      -5   /* cuFFT error                                         */
#define AK_ERR_UNSUPPORTED -6  /* configuration has no kernel (e.g. taps > 16)        */

#define AK_MAX_TAPS   16
#define AK_MAX_PAIRS   8
#define AK_NCOEF       7       /* coefficients per even/odd window polynomial (degree 13) */

/*
 * Separable window function (Kaiser-Bessel or Gaussian, nufft.py:125-131)
 * tabulated as one polynomial per tap in s = 2*frac - 1, frac = t - floor(t),
 * t = (x + 1/2) * n.  Tap a (0 <= a < taps) sits at offset z_a = frac + cutoff-1-a
 * (nufft.py:185-187).  Because the window is even, taps a and taps-1-a share
 * one even/odd split:  w_a = E_a(s^2) + s*O_a(s^2),  w_{taps-1-a} = E_a - s*O_a.
 * Coefficients are stored highest power first.
 */
typedef struct ak_window_fn {
    int32_t taps;                              /* 2*cutoff, even, 4..16 */
    int32_t ncoef;                             /* must equal AK_NCOEF    */
    double  ce[AK_MAX_PAIRS][AK_NCOEF];        /* even parts             */
    double  co[AK_MAX_PAIRS][AK_NCOEF];        /* odd parts              */
} ak_window_fn;

/* Opaque handles */
typedef struct ak_geom ak_geom;  /* bin-sorted points of P windows (replaces SpreadGeometry, nufft.py:160-166) */
typedef struct ak_op   ak_op;    /* workspace + cuFFT plans for one (geometry, R, C) apply shape */

const char* ak_last_error(void);
const char* ak_version(void);

/* Number of kernel launches issued by this library since load (evidence counter). */
int64_t ak_launch_count(void);

/*
 * ak_geom_create -- bin-sort the points of every window (replaces prepare_points).
 *   n         oversampled grid size per axis (NufftPlan.n, nufft.py:108)
 *   P         number of windows
 *   q         host int[P]: window lengths (1..3)
 *   cols      host int[P*3]: 0-based feature columns of each window (row-major, unused slots ignored)
 *   X         device double[N*ld]: row-major feature matrix (Dataset.features)
 *   wf        host window polynomial table (copied)
 * Checks every coordinate lies in [-1/2, 1/2) (nufft.py:180-181) -> AK_ERR_DOMAIN.
 * Synchronises `stream` (plan time).
 */
int ak_geom_create(int32_t n, int32_t P, const int32_t* q, const int32_t* cols,
                   const double* X, int64_t N, int64_t ld,
                   const ak_window_fn* wf, void* stream, ak_geom** out);

/*
 * ak_geom_create_masked -- ak_geom_create with a row subset per window (no
 * reference counterpart: the multi-GPU cell-slab layout, distributed.py
 * CellShardedPlan).  Window w spreads from / interpolates to only the rows r with
 * masks[w*N + r] != 0; the other rows contribute nothing and receive nothing
 * (outputs stay row-indexed over all N rows).
 *   masks     device uint8[P*N]
 *   rows_in   host int64[P]: number of nonzero mask entries per window
 */
int ak_geom_create_masked(int32_t n, int32_t P, const int32_t* q, const int32_t* cols,
                          const double* X, int64_t N, int64_t ld,
                          const uint8_t* masks, const int64_t* rows_in,
                          const ak_window_fn* wf, void* stream, ak_geom** out);
/*
 * Plan-time kernel selection.  The library never reads the process environment:
 * every choice below is made at ak_geom_create from the data (cell occupancy,
 * memory) and can be pinned explicitly with ak_geom_create_ex (tests force each
 * code path this way; the defaults are the measured-best heuristics).
 */
typedef struct ak_tuning {
    int32_t weight_tables;      /* 1: plan-time tap-weight tables when taps == 12 (default; falls
                                    back to per-pass window polynomials when they do not fit);
                                    0: always per-pass polynomials                                   */
    int32_t cell_items3;        /* 3-D work items: 0 auto (occupancy thresholds below), 1 single
                                    cells, 2 supercells of 2^3 cells                                  */
    double  dense_cells3;       /* auto: single-cell 3-D spread items from this many points per
                                    occupied cell (default 300)                                      */
    double  dense_cells3_interp;/* auto: single-cell 3-D interpolation items from this many (64)     */
    int32_t cell_items2;        /* 2-D work items: 0 auto, 1 single cells (tensor-core kernels),
                                    8 supercells of 8^2 cells (lane kernels)                         */
    double  dense_cells2;       /* auto: single-cell 2-D items from this many points per cell (2)    */
    int32_t chunk3;             /* maximum points per 3-D work item: 0 auto, else 64..65536          */
    int32_t rhs_pair_spread;    /* 1: even RHS counts of dense 3-D windows spread in RHS pairs on
                                    the FP64 tensor cores (default); 0: one RHS per CTA (DFMA)       */
    int32_t fused_fft3;         /* 1: band-pruned fused 3-D transforms for (n, m) = (64, 32) /
                                    (32, 16) (default); 0: cuFFT + band multiply                     */
    int32_t generic_kernels;    /* 1: one-thread-per-point kernels for every window (cross-check)    */
    int32_t sparse_warps;       /* warps sharing a supercell item's region tile in the 3-D sparse
                                    (multi-cell) interpolation: 1 or 2 (default 2; the spread keeps
                                    one warp per item: two warps flushing cell runs into one tile
                                    need shared-memory atomics, measured 2.3x slower on config 3)    */
    int32_t tc_spread3;         /* 3-D spread on the FP64 tensor cores where the DFMA kernels are the
                                    alternative: bit 0 single-RHS dense cells (rows a < 8 by DMMA,
                                    a = 8..11 by DFMA), bit 1 supercell items with 8 RHS per CTA
                                    (RHS-minor data, R % 8 == 0); default 3 (both)                   */
} ak_tuning;

/* Fill *t with the defaults ak_geom_create uses. */
void ak_tuning_default(ak_tuning* t);

/* ak_geom_create_masked with explicit tuning (masks / rows_in may be NULL: all rows). */
int ak_geom_create_ex(int32_t n, int32_t P, const int32_t* q, const int32_t* cols,
                      const double* X, int64_t N, int64_t ld,
                      const uint8_t* masks, const int64_t* rows_in,
                      const ak_window_fn* wf, const ak_tuning* tuning, void* stream, ak_geom** out);

/* The plan's kernel choices, for diagnostics: a short text such as
 * "q3: spread cells, interp cells, weights table; q2: cells; q1: supercells 16". */
const char* ak_geom_describe(const ak_geom* g);

int     ak_geom_destroy(ak_geom* g);
int64_t ak_geom_num_points(const ak_geom* g);
int32_t ak_geom_num_windows(const ak_geom* g);
int64_t ak_geom_num_items(const ak_geom* g);   /* work items (supercell chunks) over all windows */

/* Grid elements (doubles) of one RHS of window w: n^q[w]. */
int64_t ak_geom_grid_elems(const ak_geom* g, int32_t w);
/* Canonical grid layout used by every entry point: windows ordered by
 * decreasing q (stable), the R grids of window w consecutive:
 *   grid(w, r) = grids + R * ak_geom_canon_offset(g, w) + r * n^q[w]
 * ak_geom_canon_total(g) = sum_w n^q[w]  (total doubles for R = 1). */
int64_t ak_geom_canon_offset(const ak_geom* g, int32_t w);
int64_t ak_geom_canon_total(const ak_geom* g);
/* Occupied box of 3-D window w (diagnostics; no reference counterpart): box[2a] = lo,
 * box[2a+1] = L per axis a -- the cyclic grid-index range [lo, lo + L) mod n that holds
 * every footprint of the window's points (L a multiple of 16, or n).  The fused 3-D
 * transforms of ak_op_apply work on this box only.  Other windows: lo = 0, L = n. */
int ak_geom_box(const ak_geom* g, int32_t w, int32_t* box6);

/*
 * ak_spread -- real-valued spreading of R right-hand sides onto per-window grids
 * (replaces _spread_q, nufft.py:197-254; accumulates (+=), like the reference).
 *   V        device double[R][ldv], RHS r value of original row i at V[r*ldv + i]
 *   grids    device double[R * canon_total], canonical layout (above)
 */
int ak_spread(const ak_geom* g, const double* V, int32_t R, int64_t ldv,
              double* grids, void* stream);

/*
 * ak_interp -- interpolation from per-window real grids (canonical layout)
 * back to the points (replaces _interp_q, nufft.py:257-320), scaled:
 *   sum_windows=1: out[r*ldo + i] += scale[w] * interp(window w, grid r)(row i)
 *   sum_windows=0: out[w*wstride + r*ldo + i] = scale[w] * ...
 *   scale    device double[P]
 */
int ak_interp(const ak_geom* g, const double* grids, int32_t R,
              const double* scale, double* out, int64_t ldo, int32_t sum_windows,
              int64_t wstride, void* stream);

/*
 * Fast-summation operator: one spread per (window, RHS) serves C coefficient
 * sets (K, dK/dl, ...).  H is the real band multiplier per (set, window):
 *   H = Re(c_hat_k) / prod_a psi_hat(k_a/n)^2 on the band I_m (FFT order,
 *   last axis k >= 0 only: compact shape m^(q-1) * (m/2)),
 * i.e. coefficient multiply (fastsum.py:159) fused with both deconvolutions
 * (nufft.py:336-343, the (-1)^k signs cancel).
 *   spread_geom / interp_geom may differ (fast_cross_matvec, fastsum.py:180-191)
 *   but must have identical windows (n, q).
 */
int ak_op_create(const ak_geom* spread_geom, const ak_geom* interp_geom,
                 int32_t m, int32_t R, int32_t C, void* stream, ak_op** out);
int ak_op_destroy(ak_op* op);

/* ak_op_apply flags */
#define AK_APPLY_ACCUMULATE   1  /* add to the outputs instead of overwriting them            */
#define AK_APPLY_SPREAD_ONLY  2  /* zero the op's grids, spread V, return (no FFT / interp)    */
#define AK_APPLY_FROM_GRIDS   4  /* skip the spread: transform + interpolate the op's grids    */
#define AK_APPLY_H_PER_RHS    8  /* C == 1 and H holds R*P multipliers: RHS r of window w uses
                                    H[r*P + w] (R different kernels in lockstep, e.g. the cells
                                    of a length-scale grid search over one geometry)            */
#define AK_APPLY_SPECTRUM_ONLY 16 /* spread, forward FFT, pack the band of the half spectra into
                                    the op's band buffer (ak_op_band), return                   */
#define AK_APPLY_FROM_SPECTRUM 32 /* skip spread + forward FFT: unpack the band buffer, then
                                    multiply, inverse FFT, interpolate                           */

/* The op's spread grids (canonical layout, R right-hand sides): the exchange
 * buffer of point-sharded multi-GPU products (spread locally, all-reduce the
 * grids, then ak_op_apply(..., AK_APPLY_FROM_GRIDS)). */
int ak_op_grids(ak_op* op, double** grids, int64_t* count);
/* The op's compact band spectra (doubles = 2 * complex count): R * sum_w m^(q-1) * m/2
 * complex values, 8x smaller than the grids at sigma = 2 -- the exchange buffer of
 * point-sharded products with AK_APPLY_SPECTRUM_ONLY / AK_APPLY_FROM_SPECTRUM. */
int ak_op_band(ak_op* op, double** band, int64_t* count);

#define AK_APPLY_RHS_MINOR    64 /* V and the outputs are row-major with the RHS index fastest:
                                    V[i*ldv + r], summed out[i*ldo + r], per-window
                                    out[(w*N + i)*ldo + r] (ldv, ldo >= R).  A point's R values
                                    share one cache line: the layout the kernels gather / scatter
                                    in full sectors (the default RHS-major layout is V[r*ldv + i]) */

/*
 *   V          device double[R][ldv]  (AK_APPLY_RHS_MINOR: double[N][ldv])
 *   H          DEVICE array [C*P] of device pointers to compact band multipliers
 *              (set c, window w at index c*P + w)
 *   scale      device double[C*P] per (set, window) operator scale (fastsum.py:136-138)
 *   outs       host array [C] of device output pointers;
 *              sum_windows[c]=1: out[c] is double[R][ldo] summed over windows
 *              sum_windows[c]=0: out[c] is double[P][R][ldo] (per-window products)
 *   flags      AK_APPLY_* bits; without AK_APPLY_ACCUMULATE the outputs are
 *              overwritten (zeroed first)
 */
int ak_op_apply(ak_op* op, const double* V, int64_t ldv,
                const double* const* H, const double* scale,
                double* const* outs, int64_t ldo, const int32_t* sum_windows,
                int32_t flags, void* stream);

/*
 * Complex NUFFT building blocks (nufft_type1 / nufft_type2 API parity).
 * ak_type1_band: real grids gre, gim (n^q each, the spread of Re/Im weights)
 *   -> S (m^q complex interleaved, FFT order) = deconv * band(fftn(gre + i gim))
 * ak_type2_grid: coefficients c (m^q complex interleaved) -> real grids
 *   gre, gim = Re/Im of ifftn(pad(deconv * c)) * n^q
 *   deconv  device double[3][m]: per-axis (-1)^k / psi_hat(k/n) (nufft.py:149-157)
 */
int ak_type1_band(int32_t q, int32_t n, int32_t m, const double* gre, const double* gim,
                  const double* deconv, double* S, void* stream);
int ak_type2_grid(int32_t q, int32_t n, int32_t m, const double* c,
                  const double* deconv, double* gre, double* gim, void* stream);

/*
 * Exact dense products (the reference's dense oracle, kernels.py:92-170):
 *   matrix == NULL: out[i] = scale * sum_w sum_j kappa(r^2_w(i,j)) v[j]   (i < Na, j < Nb)
 *   matrix != NULL: matrix[i*Nb + j] = scale * sum_w kappa(r^2_w(i,j))   (dense_matrix; P <= 64)
 * r^2_w over the window's columns in ascending order (kernels.py:92-98).
 *   Xa, Xb  device row-major feature matrices (eval / train rows; same pointer for K v)
 *   q, cols host window lengths and 0-based columns (as ak_geom_create)
 */
#define AK_FAMILY_GAUSS         0
#define AK_FAMILY_DER_GAUSS     1
#define AK_FAMILY_MATERN12      2
#define AK_FAMILY_DER_MATERN12  3
int ak_dense_apply(int32_t family, double ell, double scale, int32_t P, const int32_t* q,
                   const int32_t* cols, const double* Xa, int64_t Na, int64_t lda,
                   const double* Xb, int64_t Nb, int64_t ldb, const double* v,
                   double* out, double* matrix, void* stream);

/*
 * One conjugate-gradient iteration of the reference's cg_solve (solver.py:63-77), given
 * the product Kp = K p the caller has just computed (fast_matvec(plan, p), ak_op_apply):
 *   Ap = Kp + beta p;  pAp = p . Ap;  alpha = rs / pAp;  x += alpha p;  r -= alpha Ap;
 *   rs_new = r . r;  p = r + (rs_new / rs) p unless sqrt(rs_new) <= threshold;  rs = rs_new.
 * Every scalar lives in `state` on the device, and the step does nothing once
 * state[AK_CG_ACTIVE] is 0, so a captured graph (product + step) can be replayed
 * several times between host reads: iterations past convergence or past a breakdown
 * leave x, the iteration count and the history untouched.
 *   x, r, p  CG vectors of n doubles, updated in place
 *   state    AK_CG_STATE doubles, initialised by the caller:
 *            [AK_CG_RS] r . r, [AK_CG_ACTIVE] 1, [AK_CG_ITERATIONS] 0,
 *            [AK_CG_BREAKDOWN_AT] 0 (set to the iteration at which p^T A p <= 0, the
 *            reference's CgBreakdownError, with the value in [AK_CG_BREAKDOWN_PAP]),
 *            [AK_CG_THRESHOLD] tol * ||y||
 *   hist     hist[it] = r . r after iteration it, for it < cap (the callback values)
 *   work     AK_CG_WORK doubles of scratch (partial sums; deterministic two-level dots)
 * Elementwise arithmetic is unfused (numpy's multiply-then-add).
 */
#define AK_CG_RS             0
#define AK_CG_ACTIVE         1
#define AK_CG_ITERATIONS     2
#define AK_CG_BREAKDOWN_AT   3
#define AK_CG_BREAKDOWN_PAP  4
#define AK_CG_THRESHOLD      5
#define AK_CG_STATE          8
#define AK_CG_WORK           2048
int ak_cg_step(const double* Kp, double beta, double* x, double* r, double* p, int64_t n,
               double* state, double* hist, int64_t cap, double* work, void* stream);

/*
 * The same step for independent systems (A_s + beta_s I) x_s = y_s in lockstep -- the KRR
 * grid search runs one system per (ell, beta) cell where the reference's grid_search
 * (solver.py:157-198) calls cg_solve cell by cell.  Kp holds B product rows ("slots") of
 * n doubles; slot b updates system slot_sys[b] (NULL: slot b is system b; -1: a padding
 * row, skipped), whose vectors are rows of X, R, P ([S][n]), whose scalars are
 * state[slot_sys[b]][AK_CG_STATE] and whose ridge is betas[slot_sys[b]] (device array).
 * Systems that have ended are skipped, so converged cells may stay in the batch until the
 * caller next reads the states and compacts it.
 *   hist  NULL, or [S][cap] residual histories
 *   work  B * AK_CG_WORK doubles
 */
int ak_cg_step_batched(const double* Kp, const int32_t* slot_sys, int32_t B, const double* betas,
                       double* X, double* R, double* P, int64_t n, double* state, double* hist,
                       int64_t cap, double* work, void* stream);

/*
 * Per-kernel device timing (diagnostics; off by default, no cost when off).
 * While enabled, every kernel the library launches is bracketed by a pair of
 * CUDA events on its stream; ak_prof_report synchronises the device and returns
 * one line per kernel name: "name<TAB>launches<TAB>total_ms" (the buffer holds
 * at most `cap` bytes; the return value is the length needed).
 */
int ak_prof_enable(int32_t on);
int ak_prof_reset(void);
int64_t ak_prof_report(char* buf, int64_t cap);

/* FP64 FMA throughput probe (roofline denominator; MEASURED_PEAKS.json has no FP64 entry).
 * Runs `iters` dependent-chain-free DFMA loops on all SMs; returns achieved TFLOP/s. */
int ak_probe_fp64(int64_t iters, void* stream, double* tflops);
/* Same for FP64 tensor-core mma.sync.m8n8k4 (design probe, not on the hot path). */
int ak_probe_dmma(int64_t iters, void* stream, double* tflops);

#ifdef __cplusplus
}
#endif
#endif /* ADDKERN_B200_H */
