// km_common.cuh -- shared device types of the FastPAM SWAP library (sm_100a).
//
// Layout in HBM:
//   D        borrowed slab, row-major, d(x_o, x_c) = D[o*ld + (c - col_begin)]
//   MC[k][n] medoid columns, MC[j][o] = d(x_o, m_j)            (gathered once per swap)
//   near/sec/dn/ds[n]  nearest/second cache (Alg.3)
//   RowInfo[n]  rows sorted by nearest slot: {o, slot, dn, ds}   (16 B, one per row)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <limits.h>
#include <float.h>
#include <assert.h>

// Device-side index checks of the checked build (libkmedoids_checked.so,
// -DKM_DEVICE_ASSERTS; compute-sanitizer is not available on this pool):
// a violated check traps the kernel (cudaErrorAssert).  No code in the
// product build.
#ifdef KM_DEVICE_ASSERTS
#define KM_ASSERT(c) assert(c)
#else
#define KM_ASSERT(c) ((void)0)
#endif

namespace km {

template <typename T> struct Acc;
template <> struct Acc<uint32_t> {
    using type = long long;                    // exact int64 sums (int path)
    static constexpr bool is_float = false;
    __host__ __device__ static constexpr long long maxv() { return LLONG_MAX; }
};
template <> struct Acc<float> {
    using type = double;                       // fp64 sums of f32 values (float path)
    static constexpr bool is_float = true;
    __host__ __device__ static constexpr double maxv() { return DBL_MAX; }
};

template <typename T> __host__ __device__ inline T dmax();
template <> __host__ __device__ inline uint32_t dmax<uint32_t>() { return 0xffffffffu; }
template <> __host__ __device__ inline float dmax<float>() { return FLT_MAX; }

// One row of the slot-sorted stream order.
template <typename T> struct alignas(16) RowInfo {
    int32_t o;      // object (row of D)
    int32_t slot;   // nearest(o)
    T dn;           // d_nearest(o)
    T ds;           // d_second(o)
};

// Candidate record; ordered lexicographically by (v, slot, c) (reading R1).
template <typename A> struct alignas(16) Rec {
    A v;
    int32_t slot;
    int32_t c;
};

template <typename A> __host__ __device__ inline A amax();
template <> __host__ __device__ inline long long amax<long long>() { return LLONG_MAX; }
template <> __host__ __device__ inline double amax<double>() { return DBL_MAX; }

template <typename A> __host__ __device__ inline Rec<A> rec_none() {
    Rec<A> r;
    r.v = amax<A>();
    r.slot = INT_MAX;
    r.c = INT_MAX;
    return r;
}

template <typename A> __host__ __device__ inline bool rec_less(const Rec<A>& a, const Rec<A>& b) {
    if (a.v != b.v) return a.v < b.v;
    if (a.slot != b.slot) return a.slot < b.slot;
    return a.c < b.c;
}

// Decision of one SWAP / BUILD step (device resident, mirrored to pinned host).
template <typename A> struct alignas(16) Decision {
    A dtd;           // dTD* of the chosen swap (or BUILD gain)
    int32_t slot;    // slot i*
    int32_t c;       // candidate x_c* (global index)
    int32_t apply;   // 1 if the step is applied
    int32_t old_m;   // medoid that left slot i*
    int32_t iters;   // passes so far
    int32_t swaps;   // swaps so far
    int32_t done;    // FastPAM1: a pass found no improving swap; later passes are no-ops
};

// One FastPAM1 iteration's outcome, written by the post kernel into a pinned
// host ring (slot = launch sequence number % ring size), so the host can keep
// iterations queued ahead of the one whose outcome it reads.
template <typename A> struct alignas(16) IterMirror {
    Decision<A> d;
    A td;
    int32_t seq;
    int32_t noop;    // queued behind a converged pass: nothing ran
};

// Row parts of the SWAP / BUILD streams: part q of P covers slot-sorted
// positions [part_lo(q), part_lo(q + 1)).  The sizes tilt linearly from
// (1 + a) n/P (first part) to (1 - a) n/P (last), a = c_part_skew / 16:
// blocks are dispatched part-major, so the last wave of a bandwidth-bound
// stream holds its smallest CTAs and the tail in which SMs fall idle is
// shorter.  a = 0 gives the uniform split q*n/P.
// c_part_skew >= 16 selects the power shape g(x) = 1 - (1 - x)^(1 + skew/16)
// (sizes ~ (1 - x)^(skew/16): steeper still; measurement option).
__constant__ int c_part_skew;
__device__ __forceinline__ int64_t part_lo(int q, int64_t n, int P) {
    const int64_t a = c_part_skew, PP = P;
    if (a >= 16) {
        if (q >= P) return n;
        const double r = (double)(P - q) / (double)P;
        const int64_t v = (int64_t)((double)n * (1.0 - pow(r, 1.0 + (double)a / 16.0)));
        return v < 0 ? 0 : (v > n ? n : v);
    }
    return (int64_t)q * n * ((16 + a) * PP - a * q) / (16 * PP * PP);
}
__device__ __forceinline__ int64_t part_lo_uniform(int q, int64_t n, int P) { return (int64_t)q * n / P; }

}  // namespace km
