// Exact dense additive-kernel products on the GPU (K5).
//
// Replaces the reference's dense oracle path (kernels.py:92-170):
//   out_i = scale * sum_w sum_j kappa_w(r^2_w(i, j)) v_j
// with r^2 accumulated per window column in ascending column order
// (_window_sqdist, kernels.py:92-98), for N up to DENSE_ROW_LIMIT.  FP64;
// O(P * Na * Nb) work, one thread per output row, the other side's
// coordinates and v staged through shared memory in tiles.
#include <cuda_runtime.h>
#include <stdint.h>


#include "../../include/addkern_b200.h"

namespace {

constexpr int TILE = 128;
constexpr int MAXW = 64;  // windows per launch (the host splits larger sets)

struct DenseWindows {
    int32_t P;
    int32_t q[MAXW];
    int32_t col[MAXW][3];
};

__device__ __forceinline__ double profile(int family, double inv2l2, double invl, double r2) {
    switch (family) {
        case AK_FAMILY_GAUSS: return exp(-r2 * inv2l2);
        case AK_FAMILY_DER_GAUSS: {
            const double t = r2 * inv2l2;
            return t * exp(-t);
        }
        case AK_FAMILY_MATERN12: return exp(-sqrt(r2) * invl);
        default: {
            const double t = sqrt(r2) * invl;
            return t * exp(-t);
        }
    }
}

// matrix == nullptr: out[i] = scale * sum_j K(i,j) v[j]; otherwise matrix[i*Nb + j] = scale * K(i,j).
__global__ void __launch_bounds__(TILE)
k_dense(int family, double ell, double scale, const DenseWindows wins, const double* __restrict__ Xa, int64_t Na,
        int64_t lda, const double* __restrict__ Xb, int64_t Nb, int64_t ldb, const double* __restrict__ v,
        double* __restrict__ out, double* __restrict__ matrix, int accumulate)
{
    __shared__ double xb[8 * 3][TILE];
    __shared__ double vb[TILE];
    const int64_t i = (int64_t)blockIdx.x * TILE + threadIdx.x;
    const double inv2l2 = 1.0 / (2.0 * ell * ell);
    const double invl = 1.0 / ell;
    double acc = 0.0;
    // windows in groups of 8 (shared-memory staging of up to 24 coordinate columns)
    for (int w0 = 0; w0 < wins.P; w0 += 8) {
        const int nw = min(8, wins.P - w0);
        double xa[8][3];
#pragma unroll
        for (int w = 0; w < 8; ++w)
#pragma unroll
            for (int a = 0; a < 3; ++a)
                xa[w][a] = (i < Na && w < nw && a < wins.q[w0 + w]) ? Xa[i * lda + wins.col[w0 + w][a]] : 0.0;
        for (int64_t j0 = 0; j0 < Nb; j0 += TILE) {
            __syncthreads();
            const int64_t jj = j0 + threadIdx.x;
            if (jj < Nb) {
                for (int w = 0; w < nw; ++w)
                    for (int a = 0; a < wins.q[w0 + w]; ++a) xb[w * 3 + a][threadIdx.x] = Xb[jj * ldb + wins.col[w0 + w][a]];
                vb[threadIdx.x] = v ? v[jj] : 0.0;
            }
            __syncthreads();
            if (i >= Na) continue;
            const int nj = (int)(Nb - j0 < TILE ? Nb - j0 : TILE);
            for (int j = 0; j < nj; ++j) {
                double k = 0.0;
#pragma unroll
                for (int w = 0; w < 8; ++w) {
                    if (w < nw) {
                        double r2 = 0.0;
#pragma unroll
                        for (int a = 0; a < 3; ++a) {
                            if (a < wins.q[w0 + w]) {
                                const double d = xa[w][a] - xb[w * 3 + a][j];
                                r2 += d * d;
                            }
                        }
                        k += profile(family, inv2l2, invl, r2);
                    }
                }
                if (matrix) {
                    double* m = matrix + i * Nb + j0 + j;
                    *m = (w0 == 0 ? 0.0 : *m) + k;
                } else {
                    acc = fma(k, vb[j], acc);
                }
            }
        }
    }
    if (i < Na) {
        if (matrix) {
            for (int64_t j = 0; j < Nb; ++j) matrix[i * Nb + j] *= scale;
        } else {
            out[i] = (accumulate ? out[i] : 0.0) + scale * acc;
        }
    }
}

}  // namespace

int ak_internal_fail(int code, const char* msg);
void ak_internal_count(int n);

extern "C" int ak_dense_apply(int32_t family, double ell, double scale, int32_t P, const int32_t* q,
                              const int32_t* cols, const double* Xa, int64_t Na, int64_t lda, const double* Xb,
                              int64_t Nb, int64_t ldb, const double* v, double* out, double* matrix, void* stream)
{
    if (family < AK_FAMILY_GAUSS || family > AK_FAMILY_DER_MATERN12 || !(ell > 0) || P < 1 || !q || !cols ||
        Na < 0 || Nb < 0 || (!matrix && (!v || !out)))
        return ak_internal_fail(AK_ERR_INVALID, "bad dense arguments");
    if (Na == 0) return AK_OK;
    cudaStream_t st = (cudaStream_t)stream;
    for (int w0 = 0; w0 < P; w0 += MAXW) {
        DenseWindows dw{};
        dw.P = P - w0 < MAXW ? P - w0 : MAXW;
        for (int w = 0; w < dw.P; ++w) {
            dw.q[w] = q[w0 + w];
            if (dw.q[w] < 1 || dw.q[w] > 3) return ak_internal_fail(AK_ERR_INVALID, "window length must be 1..3");
            for (int a = 0; a < 3; ++a) dw.col[w][a] = cols[3 * (w0 + w) + a];
        }
        const int accumulate = w0 > 0 ? 1 : 0;
        if (matrix && w0 > 0) return ak_internal_fail(AK_ERR_UNSUPPORTED, "dense matrix: at most 64 windows");
        k_dense<<<(unsigned)((Na + TILE - 1) / TILE), TILE, 0, st>>>(family, ell, scale, dw, Xa, Na, lda, Xb, Nb, ldb,
                                                                     v, out, matrix, accumulate);
        ak_internal_count(1);
        if (cudaGetLastError() != cudaSuccess) return ak_internal_fail(AK_ERR_CUDA, "dense kernel launch failed");
    }
    return AK_OK;
}
