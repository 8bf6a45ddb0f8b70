// One conjugate-gradient iteration of the reference's cg_solve (solver.py:63-77) as
// four small kernels that keep every scalar on the device, so a captured CUDA graph
// (product + this step) can be replayed several times between host reads.
//
//   Ap = K p + beta p;  pAp = p . Ap                      (k_cg_dot)
//   alpha = rs / pAp;  x += alpha p;  r -= alpha Ap;  rs_new = r . r   (k_cg_update)
//   p = r + (rs_new / rs) p   unless converged                         (k_cg_direction)
//   state: iteration count, rs, history, convergence / breakdown flags (k_cg_state)
//
// The iteration is predicated on state[AK_CG_ACTIVE]: once the residual test
// sqrt(rs_new) <= tol ||y|| passes, or p^T A p <= 0 (CgBreakdownError in the
// reference), further replays change nothing, so the host may run a few iterations
// past the end and still read exactly the reference's result and iteration count.
// Elementwise arithmetic is unfused (multiply, then add: numpy's order); the two dot
// products are deterministic two-level sums (per-block partials, re-reduced in a fixed
// order by every block that needs the value).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/addkern_b200.h"

namespace {

constexpr int TB = 256;
constexpr int MAXB = AK_CG_WORK / 2;   // partial sums per dot product

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double warp_part[TB / 32];
    __shared__ double total;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    __syncthreads();   // a previous call's readers of `total` are done
    if ((threadIdx.x & 31) == 0) warp_part[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < TB / 32; ++w) s += warp_part[w];
        total = s;
    }
    __syncthreads();
    return total;
}

// sum of nb partials, the same order in every block
__device__ __forceinline__ double reduce_partials(const double* __restrict__ part, int nb) {
    double v = 0.0;
    for (int i = threadIdx.x; i < nb; i += TB) v += part[i];
    return block_sum(v);
}

__global__ void __launch_bounds__(TB)
k_cg_dot(const double* __restrict__ Kp, const double* __restrict__ p, double beta, int64_t n,
         const double* __restrict__ state, double* __restrict__ part)
{
    if (state[AK_CG_ACTIVE] == 0.0) return;
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * TB + threadIdx.x; i < n; i += (int64_t)gridDim.x * TB) {
        const double ap = __dadd_rn(Kp[i], __dmul_rn(beta, p[i]));
        acc = __dadd_rn(acc, __dmul_rn(p[i], ap));
    }
    acc = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(TB)
k_cg_update(const double* __restrict__ Kp, const double* __restrict__ p, double beta, int64_t n,
            const double* __restrict__ state, double* __restrict__ x, double* __restrict__ r,
            const double* __restrict__ part, double* __restrict__ part2)
{
    if (state[AK_CG_ACTIVE] == 0.0) return;
    const double pAp = reduce_partials(part, gridDim.x);
    if (!(pAp > 0.0)) return;
    const double alpha = state[AK_CG_RS] / pAp;
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * TB + threadIdx.x; i < n; i += (int64_t)gridDim.x * TB) {
        const double pi = p[i];
        const double ap = __dadd_rn(Kp[i], __dmul_rn(beta, pi));
        x[i] = __dadd_rn(x[i], __dmul_rn(alpha, pi));
        const double ri = __dsub_rn(r[i], __dmul_rn(alpha, ap));
        r[i] = ri;
        acc = __dadd_rn(acc, __dmul_rn(ri, ri));
    }
    acc = block_sum(acc);
    if (threadIdx.x == 0) part2[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(TB)
k_cg_direction(const double* __restrict__ r, double* __restrict__ p, int64_t n, const double* __restrict__ state,
               const double* __restrict__ part, const double* __restrict__ part2)
{
    if (state[AK_CG_ACTIVE] == 0.0) return;
    const double pAp = reduce_partials(part, gridDim.x);
    if (!(pAp > 0.0)) return;
    const double rs_new = reduce_partials(part2, gridDim.x);
    if (sqrt(rs_new) <= state[AK_CG_THRESHOLD]) return;   // converged: the reference returns before updating p
    const double c = rs_new / state[AK_CG_RS];
    for (int64_t i = (int64_t)blockIdx.x * TB + threadIdx.x; i < n; i += (int64_t)gridDim.x * TB)
        p[i] = __dadd_rn(r[i], __dmul_rn(c, p[i]));
}

__global__ void __launch_bounds__(TB)
k_cg_state(double* __restrict__ state, double* __restrict__ hist, int64_t cap, const double* __restrict__ part,
           const double* __restrict__ part2, int nb)
{
    if (state[AK_CG_ACTIVE] == 0.0) return;
    const double pAp = reduce_partials(part, nb);
    const double rs_new = pAp > 0.0 ? reduce_partials(part2, nb) : 0.0;
    if (threadIdx.x != 0) return;
    const int64_t it = (int64_t)state[AK_CG_ITERATIONS] + 1;
    if (!(pAp > 0.0)) {
        state[AK_CG_BREAKDOWN_AT] = (double)it;
        state[AK_CG_BREAKDOWN_PAP] = pAp;
        state[AK_CG_ACTIVE] = 0.0;
        return;
    }
    state[AK_CG_ITERATIONS] = (double)it;
    if (it < cap) hist[it] = rs_new;
    if (sqrt(rs_new) <= state[AK_CG_THRESHOLD]) state[AK_CG_ACTIVE] = 0.0;
    state[AK_CG_RS] = rs_new;
}

}  // namespace

int ak_internal_fail(int code, const char* msg);
void ak_internal_count(int n);

extern "C" int ak_cg_step(const double* Kp, double beta, double* x, double* r, double* p, int64_t n, double* state,
                          double* hist, int64_t cap, double* work, void* stream)
{
    if (!Kp || !x || !r || !p || !state || !hist || !work || n < 1 || cap < 1)
        return ak_internal_fail(AK_ERR_INVALID, "bad CG step arguments");
    cudaStream_t st = (cudaStream_t)stream;
    int64_t want = (n + 4 * TB - 1) / (4 * TB);
    const int nb = (int)(want < 1 ? 1 : (want > MAXB ? MAXB : want));
    double* part = work;
    double* part2 = work + MAXB;
    k_cg_dot<<<nb, TB, 0, st>>>(Kp, p, beta, n, state, part);
    k_cg_update<<<nb, TB, 0, st>>>(Kp, p, beta, n, state, x, r, part, part2);
    k_cg_direction<<<nb, TB, 0, st>>>(r, p, n, state, part, part2);
    k_cg_state<<<1, TB, 0, st>>>(state, hist, cap, part, part2, nb);
    ak_internal_count(4);
    if (cudaGetLastError() != cudaSuccess) return ak_internal_fail(AK_ERR_CUDA, "CG step launch failed");
    return AK_OK;
}
