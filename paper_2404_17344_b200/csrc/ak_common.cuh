// Shared device-side definitions for the B200 fast-summation kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/addkern_b200.h"

#define AK_PRAGMA(x) _Pragma(#x)
#define AK_UNROLL(n) AK_PRAGMA(unroll n)

namespace ak {

// One bin-sorted point of one window (32 B, two 16-B vector loads).
//   s[a]  = 2*frac_a - 1, frac_a = t_a - floor(t_a), t_a = (x_a + 1/2) * n
//   cell  = packed floor(t) mod n, 10 bits per axis (axis 0 lowest)
//   idx   = original row
struct alignas(16) Point {
    double s[3];
    int32_t cell;
    int32_t idx;
};

// A chunk of at most `chunk` points of one supercell of one window.
struct alignas(16) WorkItem {
    int32_t window;
    int32_t sc;      // packed supercell coordinates, 10 bits per axis
    int32_t start;   // global index into the sorted point array
    int32_t count;
};

// Supercell edge (cells per axis) per window length.  A CTA accumulates one
// supercell chunk into a (S+T-1)^q shared tile before flushing to HBM/L2.
// (q = 3 uses a runtime edge of 2..4, see ak_geom::sedge and ak_q3.cuh.)
template <int Q> struct SuperCell;
template <> struct SuperCell<2> { static constexpr int S = 8; };
template <> struct SuperCell<1> { static constexpr int S = 16; };


// Element (r, i) of an RHS-indexed array (right-hand sides V or outputs) lives at
// base + r * rs + i * is: RHS-major (rs = ld, is = 1) or RHS-minor (rs = 1, is = ld),
// AK_APPLY_RHS_MINOR.  With RHS-minor data the R CTAs of a work item (the RHS index
// runs fastest in every launch) gather / scatter the R values of a point from one
// cache line instead of R separate sectors.
struct Strides {
    int64_t rs, is;
};

__device__ __forceinline__ int cell_axis(int32_t packed, int a) { return (packed >> (10 * a)) & 1023; }

// Window weights of one axis: w[a] for the T taps of a point with polynomial
// variable s (see ak_window_fn in the public header).
template <int T>
__device__ __forceinline__ void window_weights(const ak_window_fn& wf, double s, double* w) {
    const double s2 = s * s;
#pragma unroll
    for (int a = 0; a < T / 2; ++a) {
        double e = wf.ce[a][0];
        double o = wf.co[a][0];
#pragma unroll
        for (int k = 1; k < AK_NCOEF; ++k) {
            e = fma(e, s2, wf.ce[a][k]);
            o = fma(o, s2, wf.co[a][k]);
        }
        w[a] = fma(s, o, e);
        w[T - 1 - a] = fma(-s, o, e);
    }
}

// Runtime-taps variant used by the generic kernels.
__device__ __forceinline__ double window_weight_rt(const ak_window_fn& wf, double s, int a) {
    const int T = wf.taps;
    const bool mirror = a >= T / 2;
    const int p = mirror ? T - 1 - a : a;
    const double s2 = s * s;
    double e = wf.ce[p][0], o = wf.co[p][0];
#pragma unroll
    for (int k = 1; k < AK_NCOEF; ++k) {
        e = fma(e, s2, wf.ce[p][k]);
        o = fma(o, s2, wf.co[p][k]);
    }
    return mirror ? fma(-s, o, e) : fma(s, o, e);
}

// Checked builds (-DAK_CHECKED, tools/checked_build.py): device-side invariant checks
// that trap with a message; compiled out of the product library.
#ifdef AK_CHECKED
#define AK_DCHECK(cond)                                                                           \
    do {                                                                                          \
        if (!(cond)) {                                                                            \
            printf("AK_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                           \
            __trap();                                                                             \
        }                                                                                         \
    } while (0)
#else
#define AK_DCHECK(cond) \
    do {                \
    } while (0)
#endif

// Periodic grid index.  Every index the kernels form (footprints and supercell
// regions: S <= 16, T <= 16) lies in [-7, n + 22], so for n >= 32 one conditional
// add/subtract suffices (a few integer ops instead of a ~20-instruction integer
// division); n is warp-uniform, the branch does not diverge.
__device__ __forceinline__ int wrap(int i, int n) {
    int r;
    if (n >= 32) {
        AK_DCHECK(i >= -n && i < 2 * n);
        i += i < 0 ? n : 0;
        r = i >= n ? i - n : i;
    } else {
        i %= n;
        r = i < 0 ? i + n : i;
    }
    AK_DCHECK(r >= 0 && r < n);
    return r;
}

// cp.async (LDGSTS): global -> shared without a register round trip.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ void red_add(double* p, double v) {
    atomicAdd(p, v);  // compiles to RED.E.ADD.F64 when the result is unused
}

}  // namespace ak
