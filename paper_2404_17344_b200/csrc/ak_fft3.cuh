// Band-pruned, multiplier-fused transform stage for 3-D windows, on the FP64 tensor
// cores.
//
// The reference (nufft.py:362-365, 379-383, fastsum.py:159) takes the full n^3 FFT of
// each grid, keeps the band of m modes per axis, multiplies by the kernel's
// coefficients and the window deconvolution (one real multiplier H per band entry; the
// (-1)^k signs cancel), zero-pads and takes the full inverse FFT.  Only the band (m of
// n frequencies per axis, m/2 along the real axis) is ever used, so these kernels
// compute exactly the band, as DFT-matrix products on the FP64 tensor cores
// (mma.sync m8n8k4, operands in shared memory):
//   fwd12 : per plane x0 of a grid:  real P[x1][x2] -> B[x0][k1][k2]
//           S1  A[x1][(k2,re|im)] = P . T1                (M n,  N m,    K n)
//           S2  [Bre; Bim] = [[Wr, -Wi], [Wi, Wr]] . [Are; Aim]   (M 2m, N m/2, K 2n)
//   fwd0  : per (k1, grid) slab:     B[.][k1][.] -> S[k0][k1][k2], the compact band
//           spectrum (multi-GPU exchange buffer, layout of k_band_pack)  (M 2m, N m/2, K 2n)
//   inv0  : per (k1, grid) slab:     H * S -> C[x0][k1][k2]   (multiplier fused; M 2n, N m/2, K 2m)
//   inv12 : per plane x0:            C[x0] -> D[x1][k2] (M 2n, N m/2, K 2m)
//           -> real g[x1][x2] = sum_k2 c_k2 Re(D e^{+i w k2 x2}) = [Dre | Dim] . T3  (M n, N n, K m)
// Frequencies: band index b in [0, m) is k = b (b < m/2) or b - m; w = 2 pi / n.
// Along the real axis k2 runs over [0, m/2) with c_0 = 1, c_k2 = 2 otherwise, which is
// cuFFT's Z2D on the Hermitian-consistent band (H even, forward input real).
// Every stage is a 131K-MAC GEMM per plane/slab at n = 64, m = 32 (512 DMMA) over the
// whole grid; the kernels work on each window's occupied box (GridBox below), so the
// x sums / outputs shrink to the box: config 3 transforms 0.264 -> 0.121 ms per step,
// config 4 2.874 -> 2.844 ms per product (B200).
#pragma once
#include "ak_common.cuh"

#ifndef AK_FFT3_KC
#define AK_FFT3_KC 4
#endif

namespace ak {

#ifndef AK_FFT3_ALIAS
#define AK_FFT3_ALIAS 1
#endif
#ifndef AK_FFT3_THREADS
#define AK_FFT3_THREADS 128
#endif
#ifndef AK_FFT3_MINB
#define AK_FFT3_MINB 6
#endif
constexpr int FFT3_THREADS = AK_FFT3_THREADS;

// row strides (doubles) that keep the m8n8k4 fragment loads conflict-free:
// A operands (8 rows x 4 k) want ld = 4 (mod 16), B operands (4 k x 8 cols) ld = 8 (mod 16)
__host__ __device__ constexpr int fft3_ldA(int cols) { return cols + ((4 - cols) % 16 + 16) % 16; }
__host__ __device__ constexpr int fft3_ldB(int cols) { return cols + ((8 - cols) % 16 + 16) % 16; }

__device__ __forceinline__ void dmma_884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// C[M][N] = sum_k A(r, k) B(k, c) over the CTA's warps; each warp takes blocks of
// TM x TN 8x8 output tiles.  a(r, k) / b(k, c) fetch operand elements (shared memory),
// st(r, c, v) consumes each result.  M % (8 TM) == N % (8 TN) == K % 4 == 0.
template <int TM, int TN, class FA, class FB, class FS>
__device__ __forceinline__ void cta_gemm(int M, int N, int K, FA a, FB b, FS st)
{
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int mt = M / (8 * TM), nt = N / (8 * TN);
    const int lr = lane >> 2, lk = lane & 3;
    for (int blk = warp; blk < mt * nt; blk += nw) {
        const int r0 = (blk / nt) * 8 * TM, c0 = (blk % nt) * 8 * TN;
        double acc[TM][TN][2];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        // fragments of KC k-steps are fetched together (one load latency per KC steps)
        constexpr int KC = AK_FFT3_KC;
        int k = 0;
        for (; k + 4 * KC <= K; k += 4 * KC) {
            double af[KC][TM], bf[KC][TN];
#pragma unroll
            for (int s = 0; s < KC; ++s) {
#pragma unroll
                for (int i = 0; i < TM; ++i) af[s][i] = a(r0 + 8 * i + lr, k + 4 * s + lk);
#pragma unroll
                for (int j = 0; j < TN; ++j) bf[s][j] = b(k + 4 * s + lk, c0 + 8 * j + lr);
            }
#pragma unroll
            for (int s = 0; s < KC; ++s)
#pragma unroll
                for (int i = 0; i < TM; ++i)
#pragma unroll
                    for (int j = 0; j < TN; ++j) dmma_884(acc[i][j][0], acc[i][j][1], af[s][i], bf[s][j]);
        }
        for (; k < K; k += 4) {
            double af[TM], bf[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) af[i] = a(r0 + 8 * i + lr, k + lk);
#pragma unroll
            for (int j = 0; j < TN; ++j) bf[j] = b(k + lk, c0 + 8 * j + lr);
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) dmma_884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) {
                st(r0 + 8 * i + lr, c0 + 8 * j + 2 * lk, acc[i][j][0]);
                st(r0 + 8 * i + lr, c0 + 8 * j + 2 * lk + 1, acc[i][j][1]);
            }
    }
}

// As cta_gemm<2, 2>, but every warp keeps its (at most NB) result blocks in registers
// and the CTA synchronises before any store: the output may overwrite the operands.
template <int NB, class FA, class FB, class FS>
__device__ __forceinline__ void cta_gemm_hold(int M, int N, int K, FA a, FB b, FS st)
{
    constexpr int TM = 2, TN = 2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int mt = M / (8 * TM), nt = N / (8 * TN);
    const int lr = lane >> 2, lk = lane & 3;
    double acc[NB][TM][TN][2];
#pragma unroll
    for (int q = 0; q < NB; ++q) {
        const int blk = warp + q * nw;
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) acc[q][i][j][0] = acc[q][i][j][1] = 0.0;
        if (blk >= mt * nt) continue;
        const int r0 = (blk / nt) * 8 * TM, c0 = (blk % nt) * 8 * TN;
        for (int k = 0; k < K; k += 4) {
            double af[TM], bf[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) af[i] = a(r0 + 8 * i + lr, k + lk);
#pragma unroll
            for (int j = 0; j < TN; ++j) bf[j] = b(k + lk, c0 + 8 * j + lr);
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) dmma_884(acc[q][i][j][0], acc[q][i][j][1], af[i], bf[j]);
        }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NB; ++q) {
        const int blk = warp + q * nw;
        if (blk >= mt * nt) continue;
        const int r0 = (blk / nt) * 8 * TM, c0 = (blk % nt) * 8 * TN;
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) {
                st(r0 + 8 * i + lr, c0 + 8 * j + 2 * lk, acc[q][i][j][0]);
                st(r0 + 8 * i + lr, c0 + 8 * j + 2 * lk + 1, acc[q][i][j][1]);
            }
    }
}

// 2 x 2 tiles per warp when the shape allows it and still feeds every warp, else smaller
template <class FA, class FB, class FS>
__device__ __forceinline__ void cta_gemm_auto(int M, int N, int K, FA a, FB b, FS st)
{
    const int nw = blockDim.x >> 5;
    if (M % 16 == 0 && N % 16 == 0 && (M / 16) * (N / 16) >= nw) cta_gemm<2, 2>(M, N, K, a, b, st);
    else if (N % 16 == 0 && (M / 8) * (N / 16) >= nw) cta_gemm<1, 2>(M, N, K, a, b, st);
    else if (M % 16 == 0 && (M / 16) * (N / 8) >= nw) cta_gemm<2, 1>(M, N, K, a, b, st);
    else cta_gemm<1, 1>(M, N, K, a, b, st);
}

// Twiddle tables (one device buffer per operator, built on the host), w = 2 pi / n,
// f(b) the frequency of band index b:
//   T1 [n][m]    T1[x][2k] = cos(w k x), T1[x][2k+1] = -sin(w k x)       (k < m/2)
//   T3 [m][n]    T3[k2][x] = c cos(w k2 x), T3[m/2 + k2][x] = -c sin(w k2 x)
//   FW [2m][2n]  [[FR, -FI], [FI, FR]] with FR + i FI = e^{-i w f(b) x}   (forward band DFT)
//   IW [2n][2m]  [[IR, -II], [II, IR]] with IR + i II = e^{+i w f(b) x}   (inverse)
struct Fft3Tables {
    const double *T1, *T3, *FW, *IW;
};

// Occupied box of grid b (ak_geom::box of its window; nullptr: the whole grid).  Box
// index i of axis a is grid index x(a, i) = lo_a + i (mod n); L_a is a multiple of 16.
// Outside the box a spread grid is zero and an interpolation never reads, so the
// forward stages contract only over box indices and the inverse stages produce only
// box outputs: at config-3/4 data (points in a 30^3 corner of the 64^3 grid, L = 32)
// fwd12 / inv12 do 1/8 and fwd0 / inv0 1/2 of the full-grid work.
template <int n>
struct GridBox {
    int lo[3], L[3];
    __device__ __forceinline__ GridBox(const int* __restrict__ box, const int* __restrict__ gwin, int64_t b, int R) {
        if (box) {
            const int* bx = box + 6 * gwin[b / R];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                lo[a] = __ldg(bx + 2 * a);
                L[a] = __ldg(bx + 2 * a + 1);
            }
        } else {
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                lo[a] = 0;
                L[a] = n;
            }
        }
    }
    __device__ __forceinline__ int x(int a, int i) const {
        const int v = lo[a] + i;
        return v >= n ? v - n : v;
    }
    // column of a [..][2n] table / row of a [2n][..] table for split-complex box index
    // k in [0, 2 L_a): real part at x, imaginary part at n + x
    __device__ __forceinline__ int x2(int a, int k) const { return k < L[a] ? x(a, k) : n + x(a, k - L[a]); }
};

// plane copy global -> shared with 16-byte loads (cols even, ld even)
__device__ __forceinline__ void fft3_copy2(double* dst, int ld, const double* __restrict__ src, int rows, int cols) {
    const int c2 = cols / 2;
    const double2* __restrict__ s2 = reinterpret_cast<const double2*>(src);
    for (int e = threadIdx.x; e < rows * c2; e += blockDim.x) {
        const int r = e / c2, c = e - r * c2;
        *reinterpret_cast<double2*>(dst + r * ld + 2 * c) = __ldg(s2 + e);
    }
}

// box plane copy global -> shared: P[i1][j2] = src[x1(i1)][x2(j2)] (16-byte loads when
// the axis-2 range is contiguous and even-aligned)
template <int n>
__device__ __forceinline__ void fft3_copy_box(double* dst, int ld, const double* __restrict__ src, const GridBox<n>& bx) {
    const int L1 = bx.L[1], L2 = bx.L[2], lo2 = bx.lo[2];
    if (lo2 + L2 <= n && (lo2 & 1) == 0) {
        const int c2 = L2 / 2;
        for (int e = threadIdx.x; e < L1 * c2; e += blockDim.x) {
            const int r = e / c2, c = e - r * c2;
            *reinterpret_cast<double2*>(dst + r * ld + 2 * c) =
                __ldg(reinterpret_cast<const double2*>(src + bx.x(1, r) * n + lo2) + c);
        }
    } else {
        for (int e = threadIdx.x; e < L1 * L2; e += blockDim.x) {
            const int r = e / L2, c = e - r * L2;
            dst[r * ld + c] = __ldg(src + bx.x(1, r) * n + bx.x(2, c));
        }
    }
}

// fbuf (per grid, per box plane i0 of axis 0): split complex [2][m][mh] doubles
// fwd12: grids [nb][n][n][n] real -> fbuf [nb][L0 (i0)][2][m(b1)][mh]
template <int n, int m>
__global__ void __launch_bounds__(FFT3_THREADS, AK_FFT3_MINB)
k_fft3_fwd12(const double* __restrict__ grids, double* __restrict__ fbuf, Fft3Tables tb,
             const int* __restrict__ box, const int* __restrict__ gwin, int R)
{
    extern __shared__ __align__(16) double sm[];
    const int mh = m / 2, i0 = blockIdx.x;
    const int64_t b = blockIdx.y;
    const GridBox<n> bx(box, gwin, b, R);
    if (i0 >= bx.L[0]) return;
    const int L1 = bx.L[1], L2 = bx.L[2];
    const int ldP = fft3_ldA(n), ldX = fft3_ldB(mh);
    double* P = sm;                       // [L1][ldP]     (S1 A)
#if AK_FFT3_ALIAS
    double* X = sm;                       // [2 L1][ldX]   (S1 out over P, S2 B)
#else
    double* X = P + n * ldP;
#endif
    fft3_copy_box<n>(P, ldP, grids + (b * n + bx.x(0, i0)) * n * n, bx);
    __syncthreads();
    const double* __restrict__ T1 = tb.T1;
    auto s1a = [&](int r, int k) { return P[r * ldP + k]; };
    auto s1b = [&](int k, int c) { return __ldg(T1 + bx.x(2, k) * m + c); };
    auto s1s = [&](int r, int c, double v) { X[((c & 1) * L1 + r) * ldX + (c >> 1)] = v; };
#if AK_FFT3_ALIAS
    constexpr int NW = FFT3_THREADS / 32, NBLK = (n / 16) * (m / 16);
    constexpr int NB = (NBLK + NW - 1) / NW;   // S1 blocks per warp (2 x 2 tiles each)
    static_assert(n % 16 == 0 && m % 16 == 0, "S1 tiling");
    cta_gemm_hold<NB>(L1, m, L2, s1a, s1b, s1s);
#else
    cta_gemm_auto(L1, m, L2, s1a, s1b, s1s);
#endif
    __syncthreads();
    double* __restrict__ dst = fbuf + (b * n + i0) * 2 * m * mh;
    const double* __restrict__ FW = tb.FW;
    cta_gemm_auto(
        2 * m, mh, 2 * L1, [&](int r, int k) { return __ldg(FW + r * 2 * n + bx.x2(1, k)); },
        [&](int k, int c) { return X[k * ldX + c]; }, [&](int r, int c, double v) { dst[r * mh + c] = v; });
}

// fwd0: fbuf [nb][L0 (i0)][2][m(b1)][mh] -> band [nb][m(b0)][m(b1)][mh] complex
template <int n, int m>
__global__ void __launch_bounds__(FFT3_THREADS, AK_FFT3_MINB)
k_fft3_fwd0(const double* __restrict__ fbuf, double* __restrict__ band, Fft3Tables tb,
            const int* __restrict__ box, const int* __restrict__ gwin, int R)
{
    extern __shared__ __align__(16) double sm[];
    const int mh = m / 2, b1 = blockIdx.x;
    const int64_t b = blockIdx.y;
    const GridBox<n> bx(box, gwin, b, R);
    const int L0 = bx.L[0];
    const int ldX = fft3_ldB(mh);
    double* X = sm;                       // [2 L0 (re i0 | im i0)][ldX]
    const int h2 = mh / 2;
    for (int e = threadIdx.x; e < 2 * L0 * h2; e += blockDim.x) {
        const int row = e / h2, c = e - row * h2;     // row = ri * L0 + i0
        const int ri = row >= L0, i0 = row - ri * L0;
        *reinterpret_cast<double2*>(X + row * ldX + 2 * c) =
            __ldg(reinterpret_cast<const double2*>(fbuf + (((b * n + i0) * 2 + ri) * m + b1) * mh) + c);
    }
    __syncthreads();
    double* __restrict__ dst = band + b * 2 * (int64_t)m * m * mh;
    const double* __restrict__ FW = tb.FW;
    cta_gemm_auto(
        2 * m, mh, 2 * L0, [&](int r, int k) { return __ldg(FW + r * 2 * n + bx.x2(0, k)); },
        [&](int k, int c) { return X[k * ldX + c]; },
        [&](int r, int c, double v) {
            const int ro = r >= m, b0 = r - ro * m;
            dst[2 * (((int64_t)b0 * m + b1) * mh + c) + ro] = v;
        });
}

// inv0: H * band -> fbuf [nb][L0 (i0)][2][m(b1)][mh]; the multiplier of grid b is
// H[hsel][(b0 m + b1) mh + k2] with hsel as in k_band_multiply
template <int n, int m>
__global__ void __launch_bounds__(FFT3_THREADS, AK_FFT3_MINB)
k_fft3_inv0(const double* __restrict__ band, double* __restrict__ fbuf, Fft3Tables tb, int R,
            const int* __restrict__ gwin, const double* const* __restrict__ H, int hbase, int P, int per_rhs,
            const int* __restrict__ box)
{
    extern __shared__ __align__(16) double sm[];
    const int mh = m / 2, b1 = blockIdx.x;
    const int64_t b = blockIdx.y;
    const GridBox<n> bx(box, gwin, b, R);
    const int L0 = bx.L[0];
    const int ldY = fft3_ldB(mh);
    double* Y = sm;                       // [2m (re b0 | im b0)][ldY]
    const int w = gwin[b / R];
    const double* __restrict__ h = H[per_rhs ? (int)(b % R) * P + w : hbase + w];
    const double2* __restrict__ src = reinterpret_cast<const double2*>(band + b * 2 * (int64_t)m * m * mh);
    for (int e = threadIdx.x; e < m * mh; e += blockDim.x) {
        const int b0 = e / mh, k2 = e - b0 * mh;
        const int64_t ci = ((int64_t)b0 * m + b1) * mh + k2;
        const double hv = __ldg(h + ci);
        const double2 v = __ldg(src + ci);
        Y[b0 * ldY + k2] = hv * v.x;
        Y[(m + b0) * ldY + k2] = hv * v.y;
    }
    __syncthreads();
    const double* __restrict__ IW = tb.IW;
    cta_gemm_auto(
        2 * L0, mh, 2 * m, [&](int r, int k) { return __ldg(IW + bx.x2(0, r) * 2 * m + k); },
        [&](int k, int c) { return Y[k * ldY + c]; },
        [&](int r, int c, double v) {
            const int ro = r >= L0, i0 = r - ro * L0;
            fbuf[(((b * n + i0) * 2 + ro) * m + b1) * mh + c] = v;
        });
}

// inv12: fbuf [nb][L0 (i0)][2][m][mh] -> the box of grids [nb][n][n][n] real (one block
// per (i0, grid)); grid values outside the box are not written
template <int n, int m>
__global__ void __launch_bounds__(FFT3_THREADS, AK_FFT3_MINB)
k_fft3_inv12(const double* __restrict__ fbuf, double* __restrict__ out, Fft3Tables tb,
             const int* __restrict__ box, const int* __restrict__ gwin, int R)
{
    extern __shared__ __align__(16) double sm[];
    const int mh = m / 2, i0 = blockIdx.x;
    const int64_t b = blockIdx.y;
    const GridBox<n> bx(box, gwin, b, R);
    if (i0 >= bx.L[0]) return;
    const int L1 = bx.L[1], L2 = bx.L[2];
    const int ldC = fft3_ldB(mh), ldD = fft3_ldA(mh);
    double* C = sm;                       // [2m][ldC]  (I1 B)
    double* D = C + 2 * m * ldC;          // [2 L1][ldD]  (I1 out, I2 A)
    fft3_copy2(C, ldC, fbuf + (b * n + i0) * 2 * m * mh, 2 * m, mh);
    __syncthreads();
    const double* __restrict__ IW = tb.IW;
    cta_gemm_auto(
        2 * L1, mh, 2 * m, [&](int r, int k) { return __ldg(IW + bx.x2(1, r) * 2 * m + k); },
        [&](int k, int c) { return C[k * ldC + c]; }, [&](int r, int c, double v) { D[r * ldD + c] = v; });
    __syncthreads();
    double* __restrict__ dst = out + (b * n + bx.x(0, i0)) * n * n;
    const double* __restrict__ T3 = tb.T3;
    cta_gemm_auto(
        L1, L2, m,
        [&](int r, int k) {
            const int ri = k >= mh;
            return D[(ri * L1 + r) * ldD + k - ri * mh];
        },
        [&](int k, int c) { return __ldg(T3 + k * n + bx.x(2, c)); },
        [&](int r, int c, double v) { dst[bx.x(1, r) * n + bx.x(2, c)] = v; });
}

// dynamic shared memory (bytes) of each kernel
inline size_t fft3_smem_fwd12(int n, int m) {
#if AK_FFT3_ALIAS
    return sizeof(double) * std::max((size_t)n * fft3_ldA(n), (size_t)2 * n * fft3_ldB(m / 2));
#else
    return sizeof(double) * ((size_t)n * fft3_ldA(n) + (size_t)2 * n * fft3_ldB(m / 2));
#endif
}
inline size_t fft3_smem_fwd0(int n, int m) { return sizeof(double) * (size_t)2 * n * fft3_ldB(m / 2); }
inline size_t fft3_smem_inv0(int n, int m) { return sizeof(double) * (size_t)2 * m * fft3_ldB(m / 2); }
inline size_t fft3_smem_inv12(int n, int m) {
    return sizeof(double) * ((size_t)2 * m * fft3_ldB(m / 2) + (size_t)2 * n * fft3_ldA(m / 2));
}
inline size_t fft3_smem_max(int n, int m) {
    return std::max(std::max(fft3_smem_fwd12(n, m), fft3_smem_fwd0(n, m)),
                    std::max(fft3_smem_inv0(n, m), fft3_smem_inv12(n, m)));
}

// Host: the twiddle tables for (n, m) in one buffer, order T1, T3, FW, IW (10 n m doubles).
inline std::vector<double> fft3_host_tables(int n, int m) {
    const int mh = m / 2;
    std::vector<long double> c(n), s(n);
    for (int j = 0; j < n; ++j) {
        const long double a = 2.0L * 3.14159265358979323846264338327950288L * j / n;
        c[j] = cosl(a);
        s[j] = sinl(a);
    }
    auto f = [&](int bi) { return bi < mh ? bi : bi - m + n; };
    std::vector<double> t((size_t)10 * n * m);
    double* T1 = t.data();
    double* T3 = T1 + (size_t)n * m;
    double* FW = T3 + (size_t)n * m;          // [2m][2n]
    double* IW = FW + (size_t)4 * n * m;      // [2n][2m]
    for (int x = 0; x < n; ++x)
        for (int k = 0; k < mh; ++k) {
            const int j = (int)((int64_t)k * x % n);
            T1[x * m + 2 * k] = (double)c[j];
            T1[x * m + 2 * k + 1] = (double)-s[j];
            const double w = k == 0 ? 1.0 : 2.0;
            T3[k * n + x] = w * (double)c[j];
            T3[(mh + k) * n + x] = -w * (double)s[j];
        }
    for (int bi = 0; bi < m; ++bi)
        for (int x = 0; x < n; ++x) {
            const int j = (int)((int64_t)f(bi) * x % n);
            const double cr = (double)c[j], sn = (double)s[j];
            // forward e^{-i..} = cr - i sn: FR = cr, FI = -sn; inverse e^{+i..}: IR = cr, II = sn
            FW[bi * 2 * n + x] = cr;                 // [re out][re in] =  FR
            FW[bi * 2 * n + n + x] = sn;             // [re out][im in] = -FI
            FW[(m + bi) * 2 * n + x] = -sn;          // [im out][re in] =  FI
            FW[(m + bi) * 2 * n + n + x] = cr;       // [im out][im in] =  FR
            IW[x * 2 * m + bi] = cr;                 // [re out][re in] =  IR
            IW[x * 2 * m + m + bi] = -sn;            // [re out][im in] = -II
            IW[(n + x) * 2 * m + bi] = sn;           // [im out][re in] =  II
            IW[(n + x) * 2 * m + m + bi] = cr;       // [im out][im in] =  IR
        }
    return t;
}

}  // namespace ak
