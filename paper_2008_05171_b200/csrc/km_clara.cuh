// km_clara.cuh -- FastCLARA from points (P:414-419,
// P:1109-1129): no n x n matrix is ever formed.
//
//   k_subdist_exact   the s x s dissimilarity matrix of one sample, computed
//                     from the sample's points by the definitions (L2: fp64
//                     sum of squared differences in dimension order, every
//                     operation rounded on its own, sqrt, rounded to f32;
//                     L1: int64 sum of |differences|, stored as uint32), so
//                     the sub-problem equals the one the oracle builds;
//   k_td_points       TD over ALL n objects of the sample's medoids (Eq.
//                     eqn:td) with each object's distance to every medoid
//                     recomputed from the points the same way (reading C2),
//                     per-block sums in a fixed tree, optional assignment;
//   k_sum_partials    the block sums in block order (deterministic).
// Work: s^2 d for the sub-matrix, n k d for the TD pass -- O(n k d) instead
// of the O(n^2) of a materialised matrix.
#pragma once
#include "km_kernels.cuh"

namespace km {

template <typename T> struct PointOf;
template <> struct PointOf<float> { using type = float; };        // L2: float coordinates
template <> struct PointOf<uint32_t> { using type = int32_t; };   // L1: integer coordinates

template <typename T>
__device__ __forceinline__ T point_dist(const typename PointOf<T>::type* a, const typename PointOf<T>::type* b,
                                        int d);

template <>
__device__ __forceinline__ float point_dist<float>(const float* a, const float* b, int d) {
    double s = 0.0;
    for (int t = 0; t < d; ++t) {
        const double u = (double)a[t] - (double)b[t];
        s = __dadd_rn(s, __dmul_rn(u, u));
    }
    return __double2float_rn(sqrt(s));
}

template <>
__device__ __forceinline__ uint32_t point_dist<uint32_t>(const int32_t* a, const int32_t* b, int d) {
    long long s = 0;
    for (int t = 0; t < d; ++t) {
        const long long u = (long long)a[t] - (long long)b[t];
        s += u < 0 ? -u : u;
    }
    return (uint32_t)s;
}

// out[a * lds + b] = d(x_{S[a]}, x_{S[b]}); 32 x 8 threads per 32 x 32 tile,
// the tile's 2 x 32 rows of points staged in shared memory (d <= CLARA_MAXD)
constexpr int CLARA_MAXD = 128;
template <typename T>
__global__ void __launch_bounds__(256)
k_subdist_exact(const typename PointOf<T>::type* __restrict__ X, int d, const int* __restrict__ idx, int s,
                T* __restrict__ out, int64_t lds) {
    using P = typename PointOf<T>::type;
    extern __shared__ __align__(16) unsigned char cl_smem[];
    P* ra = reinterpret_cast<P*>(cl_smem);              // 32 rows (a side)
    P* rb = ra + 32 * d;                                // 32 rows (b side)
    const int a0 = blockIdx.y * 32, b0 = blockIdx.x * 32;
    for (int e = threadIdx.x; e < 32 * d; e += blockDim.x) {
        const int r = e / d, t = e - r * d;
        KM_ASSERT(a0 + r >= s || idx[a0 + r] >= 0);
        ra[e] = (a0 + r < s) ? X[(int64_t)idx[a0 + r] * d + t] : (P)0;
        rb[e] = (b0 + r < s) ? X[(int64_t)idx[b0 + r] * d + t] : (P)0;
    }
    __syncthreads();
    const int bx = threadIdx.x & 31, ay = threadIdx.x >> 5;
    for (int r = ay; r < 32; r += 8) {
        const int a = a0 + r, b = b0 + bx;
        if (a < s && b < s) out[(int64_t)a * lds + b] = point_dist<T>(ra + r * d, rb + bx * d, d);
    }
}

// TD over all objects: each thread one object; the medoid points are staged
// in shared memory in chunks.  The smallest slot wins ties (reading R2).
template <typename T, typename A>
__global__ void __launch_bounds__(256)
k_td_points(const typename PointOf<T>::type* __restrict__ X, int n, int d, const int* __restrict__ M, int k,
            int kc, A* __restrict__ partials, int* __restrict__ asg) {
    using P = typename PointOf<T>::type;
    extern __shared__ __align__(16) unsigned char cl_smem[];
    P* mp = reinterpret_cast<P*>(cl_smem);              // kc medoid rows
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    T best = dmax<T>();
    int bj = -1;
    for (int j0 = 0; j0 < k; j0 += kc) {
        const int m = min(kc, k - j0);
        __syncthreads();
        for (int e = threadIdx.x; e < m * d; e += blockDim.x) {
            const int r = e / d, t = e - r * d;
            mp[e] = X[(int64_t)M[j0 + r] * d + t];
        }
        __syncthreads();
        if (o < n) {
            const P* xo = X + (int64_t)o * d;
            for (int j = 0; j < m; ++j) {
                const T v = point_dist<T>(xo, mp + j * d, d);
                if (bj < 0 || v < best) { best = v; bj = j0 + j; }
            }
        }
    }
    if (o < n && asg) asg[o] = bj;
    // fixed-order block sum of the per-object minima
    __shared__ A wsum[8];
    A v = (o < n) ? (A)best : (A)0;
#pragma unroll
    for (int x = 16; x >= 1; x >>= 1) v += __shfl_xor_sync(FULL, v, x);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        A t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += wsum[w];
        partials[blockIdx.x] = t;
    }
}

template <typename A>
__global__ void k_sum_partials(const A* __restrict__ partials, int nb, A* __restrict__ out) {
    // one warp: lane-strided sums in block order, then a fixed shuffle tree
    A v = 0;
    for (int b = threadIdx.x; b < nb; b += 32) v += partials[b];
#pragma unroll
    for (int x = 16; x >= 1; x >>= 1) v += __shfl_xor_sync(FULL, v, x);
    if (threadIdx.x == 0) *out = v;
}

}  // namespace km
