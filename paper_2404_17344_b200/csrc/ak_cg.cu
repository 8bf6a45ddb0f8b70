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
//
// Batched form (ak_cg_step_batched): B product rows ("slots") of independent systems
// in lockstep, blockIdx.y = slot, slot_sys[slot] = the system whose vectors, state and
// beta the slot updates (-1: a padding row) -- the lockstep CG of the KRR grid search
// (one system per (ell, beta) cell), whose converged cells leave the product batch.
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

// slot -> system; false when the slot is padding or its system is no longer active
struct Batch {
    const int32_t* slot_sys;   // nullptr: slot == system
    const double* betas;       // nullptr: `beta` for every system
    double beta;
    int64_t n, cap;
};

__device__ __forceinline__ bool slot_system(const Batch& b, const double* state, int& sys, double& beta) {
    sys = b.slot_sys ? b.slot_sys[blockIdx.y] : (int)blockIdx.y;
    if (sys < 0 || state[(int64_t)sys * AK_CG_STATE + AK_CG_ACTIVE] == 0.0) return false;
    beta = b.betas ? b.betas[sys] : b.beta;
    return true;
}

__global__ void __launch_bounds__(TB)
k_cg_dot(const double* __restrict__ Kp, const double* __restrict__ p, Batch b,
         const double* __restrict__ state, double* __restrict__ part)
{
    int sys;
    double beta;
    if (!slot_system(b, state, sys, beta)) return;
    const int64_t n = b.n;
    Kp += (int64_t)blockIdx.y * n;
    p += (int64_t)sys * n;
    part += (int64_t)blockIdx.y * AK_CG_WORK;
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * TB + threadIdx.x; i < n; i += (int64_t)gridDim.x * TB) {
        const double ap = __dadd_rn(Kp[i], __dmul_rn(beta, p[i]));
        acc = __dadd_rn(acc, __dmul_rn(p[i], ap));
    }
    acc = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(TB)
k_cg_update(const double* __restrict__ Kp, const double* __restrict__ p, Batch b,
            const double* __restrict__ state, double* __restrict__ x, double* __restrict__ r,
            const double* __restrict__ part, double* __restrict__ part2)
{
    int sys;
    double beta;
    if (!slot_system(b, state, sys, beta)) return;
    const int64_t n = b.n;
    Kp += (int64_t)blockIdx.y * n;
    p += (int64_t)sys * n;
    x += (int64_t)sys * n;
    r += (int64_t)sys * n;
    state += (int64_t)sys * AK_CG_STATE;
    part += (int64_t)blockIdx.y * AK_CG_WORK;
    part2 += (int64_t)blockIdx.y * AK_CG_WORK;
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
k_cg_direction(const double* __restrict__ r, double* __restrict__ p, Batch b, const double* __restrict__ state,
               const double* __restrict__ part, const double* __restrict__ part2)
{
    int sys;
    double beta;
    if (!slot_system(b, state, sys, beta)) return;
    const int64_t n = b.n;
    p += (int64_t)sys * n;
    r += (int64_t)sys * n;
    state += (int64_t)sys * AK_CG_STATE;
    part += (int64_t)blockIdx.y * AK_CG_WORK;
    part2 += (int64_t)blockIdx.y * AK_CG_WORK;
    const double pAp = reduce_partials(part, gridDim.x);
    if (!(pAp > 0.0)) return;
    const double rs_new = reduce_partials(part2, gridDim.x);
    if (sqrt(rs_new) <= state[AK_CG_THRESHOLD]) return;   // converged: the reference returns before updating p
    const double c = rs_new / state[AK_CG_RS];
    for (int64_t i = (int64_t)blockIdx.x * TB + threadIdx.x; i < n; i += (int64_t)gridDim.x * TB)
        p[i] = __dadd_rn(r[i], __dmul_rn(c, p[i]));
}

__global__ void __launch_bounds__(TB)
k_cg_state(double* __restrict__ state, double* __restrict__ hist, Batch b, const double* __restrict__ part,
           const double* __restrict__ part2, int nb)
{
    int sys;
    double beta;
    if (!slot_system(b, state, sys, beta)) return;
    const int64_t cap = b.cap;
    state += (int64_t)sys * AK_CG_STATE;
    if (hist) hist += (int64_t)sys * cap;
    part += (int64_t)blockIdx.y * AK_CG_WORK;
    part2 += (int64_t)blockIdx.y * AK_CG_WORK;
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
    if (hist && it < cap) hist[it] = rs_new;
    if (sqrt(rs_new) <= state[AK_CG_THRESHOLD]) state[AK_CG_ACTIVE] = 0.0;
    state[AK_CG_RS] = rs_new;
}

}  // namespace

int ak_internal_fail(int code, const char* msg);
void ak_internal_count(int n);

static int cg_launch(const double* Kp, const Batch& b, int B, double* x, double* r, double* p, double* state,
                     double* hist, double* work, cudaStream_t st)
{
    int64_t want = (b.n + 4 * TB - 1) / (4 * TB);
    const int nb = (int)(want < 1 ? 1 : (want > MAXB ? MAXB : want));
    double* part = work;
    double* part2 = work + MAXB;
    const dim3 grid((unsigned)nb, (unsigned)B);
    k_cg_dot<<<grid, TB, 0, st>>>(Kp, p, b, state, part);
    k_cg_update<<<grid, TB, 0, st>>>(Kp, p, b, state, x, r, part, part2);
    k_cg_direction<<<grid, TB, 0, st>>>(r, p, b, state, part, part2);
    k_cg_state<<<dim3(1, (unsigned)B), TB, 0, st>>>(state, hist, b, part, part2, nb);
    ak_internal_count(4);
    if (cudaGetLastError() != cudaSuccess) return ak_internal_fail(AK_ERR_CUDA, "CG step launch failed");
    return AK_OK;
}

extern "C" int ak_cg_step(const double* Kp, double beta, double* x, double* r, double* p, int64_t n, double* state,
                          double* hist, int64_t cap, double* work, void* stream)
{
    if (!Kp || !x || !r || !p || !state || !hist || !work || n < 1 || cap < 1)
        return ak_internal_fail(AK_ERR_INVALID, "bad CG step arguments");
    const Batch b{nullptr, nullptr, beta, n, cap};
    return cg_launch(Kp, b, 1, x, r, p, state, hist, work, (cudaStream_t)stream);
}

extern "C" int ak_cg_step_batched(const double* Kp, const int32_t* slot_sys, int32_t B, const double* betas,
                                  double* X, double* R, double* P, int64_t n, double* state, double* hist,
                                  int64_t cap, double* work, void* stream)
{
    if (!Kp || !betas || !X || !R || !P || !state || !work || n < 1 || B < 1 || B > 65535 || (hist && cap < 1))
        return ak_internal_fail(AK_ERR_INVALID, "bad batched CG step arguments");
    const Batch b{slot_sys, betas, 0.0, n, cap};
    return cg_launch(Kp, b, B, X, R, P, state, hist, work, (cudaStream_t)stream);
}
