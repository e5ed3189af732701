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
//   k_sum_partials    the block sums in block order (deterministic);
//   k_map_sample_medoids  a sample's local medoids -> object indices;
//   k_td_cols         the TD of a sample's medoids over a resident D
//                     (kmedoids_clara).
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

// Row stride of a staged point tile: odd, so lanes reading coordinate t of
// 32 different rows hit 32 different banks.
__host__ __device__ inline int clara_row_stride(int d) { return d | 1; }

// out[a * lds + b] = d(x_{S[a]}, x_{S[b]}); 32 x 8 threads per 32 x 32 tile,
// the tile's 2 x 32 rows of points staged in shared memory (d <= CLARA_MAXD),
// rows `clara_row_stride(d)` apart
constexpr int CLARA_MAXD = 128;
template <typename T>
__global__ void __launch_bounds__(256)
k_subdist_exact(const typename PointOf<T>::type* __restrict__ X, int d, const int* __restrict__ idx, int s,
                T* __restrict__ out, int64_t lds) {
    using P = typename PointOf<T>::type;
    extern __shared__ __align__(16) unsigned char cl_smem[];
    const int rs = clara_row_stride(d);
    P* ra = reinterpret_cast<P*>(cl_smem);              // 32 rows (a side)
    P* rb = ra + 32 * rs;                               // 32 rows (b side)
    const int a0 = blockIdx.y * 32, b0 = blockIdx.x * 32;
    for (int e = threadIdx.x; e < 32 * d; e += blockDim.x) {
        const int r = e / d, t = e - r * d;
        KM_ASSERT(a0 + r >= s || idx[a0 + r] >= 0);
        ra[r * rs + t] = (a0 + r < s) ? X[(int64_t)idx[a0 + r] * d + t] : (P)0;
        rb[r * rs + t] = (b0 + r < s) ? X[(int64_t)idx[b0 + r] * d + t] : (P)0;
    }
    __syncthreads();
    const int bx = threadIdx.x & 31, ay = threadIdx.x >> 5;
    for (int r = ay; r < 32; r += 8) {
        const int a = a0 + r, b = b0 + bx;
        if (a < s && b < s) out[(int64_t)a * lds + b] = point_dist<T>(ra + r * rs, rb + bx * rs, d);
    }
}

// Widened coordinate type of the definitions (L2: fp64, L1: int64), one term
// of the sum and the final rounding -- the arithmetic of point_dist, split so
// several medoids can be accumulated side by side.
template <typename T> struct PointWide;
template <> struct PointWide<float> {
    using type = double;
    static __device__ __forceinline__ double term(double s, double u) { return __dadd_rn(s, __dmul_rn(u, u)); }
    static __device__ __forceinline__ float fin(double s) { return __double2float_rn(sqrt(s)); }
};
template <> struct PointWide<uint32_t> {
    using type = long long;
    static __device__ __forceinline__ long long term(long long s, long long u) { return s + (u < 0 ? -u : u); }
    static __device__ __forceinline__ uint32_t fin(long long s) { return (uint32_t)s; }
};

// TD over all objects: each thread one object.  The block's TDP_THREADS
// object rows are staged once, transposed (coordinate t of object r at
// xs[t * (TDP_THREADS + 1) + r]: conflict-free for the staging writes and
// the per-thread reads -- round 2's first version read every coordinate of
// its object from global memory per medoid, 32 distinct lines per warp
// load: 1.76 ms at C4); the medoid points are staged widened (fp64 / int64)
// in chunks of kc rows (broadcast reads), and every thread accumulates
// TDP_MU medoids side by side (independent chains, one coordinate load and
// conversion per TDP_MU terms).  Each distance is the definition's sum in
// dimension order, as point_dist.  The smallest slot wins ties (reading R2).
constexpr int TDP_THREADS = 128;
constexpr int TDP_MU = 4;
template <typename T>
__host__ inline size_t td_points_xs_bytes(int d) {
    return ((size_t)d * (TDP_THREADS + 1) * sizeof(typename PointOf<T>::type) + 15) / 16 * 16;
}
template <typename T>
__host__ inline size_t td_points_smem(int d, int kc) {
    return td_points_xs_bytes<T>(d) + (size_t)kc * d * sizeof(typename PointWide<T>::type);
}
template <typename T, typename A>
__global__ void __launch_bounds__(TDP_THREADS)
k_td_points(const typename PointOf<T>::type* __restrict__ X, int n, int d, const int* __restrict__ M, int k,
            int kc, A* __restrict__ partials, int* __restrict__ asg) {
    using P = typename PointOf<T>::type;
    using PW = PointWide<T>;
    using W = typename PW::type;
    extern __shared__ __align__(16) unsigned char cl_smem[];
    constexpr int XS = TDP_THREADS + 1;
    P* xs = reinterpret_cast<P*>(cl_smem);              // [d][XS] the block's objects
    W* mw = reinterpret_cast<W*>(cl_smem + ((size_t)d * XS * sizeof(P) + 15) / 16 * 16);   // kc medoid rows
    const int o0 = blockIdx.x * TDP_THREADS;
    const int o = o0 + threadIdx.x;
    for (int e = threadIdx.x; e < TDP_THREADS * d; e += blockDim.x) {
        const int r = e / d, t = e - r * d;             // consecutive e: one row, coalesced
        xs[t * XS + r] = (o0 + r < n) ? X[(int64_t)(o0 + r) * d + t] : (P)0;
    }
    const P* xo = xs + threadIdx.x;
    T best = dmax<T>();
    int bj = -1;
    for (int j0 = 0; j0 < k; j0 += kc) {
        const int m = min(kc, k - j0);
        __syncthreads();
        for (int e = threadIdx.x; e < m * d; e += blockDim.x) {
            const int r = e / d, t = e - r * d;
            mw[e] = (W)X[(int64_t)M[j0 + r] * d + t];
        }
        __syncthreads();
        if (o < n) {
            for (int j = 0; j < m; j += TDP_MU) {
                const W* mr[TDP_MU];
                W sacc[TDP_MU];
#pragma unroll
                for (int i = 0; i < TDP_MU; ++i) { mr[i] = mw + (size_t)min(j + i, m - 1) * d; sacc[i] = 0; }
                for (int t = 0; t < d; ++t) {
                    const W x = (W)xo[t * XS];
#pragma unroll
                    for (int i = 0; i < TDP_MU; ++i) sacc[i] = PW::term(sacc[i], x - mr[i][t]);
                }
#pragma unroll
                for (int i = 0; i < TDP_MU; ++i) {
                    if (j + i >= m) break;
                    const T v = PW::fin(sacc[i]);
                    if (bj < 0 || v < best) { best = v; bj = j0 + j + i; }
                }
            }
        }
    }
    if (o < n && asg) asg[o] = bj;
    // fixed-order block sum of the per-object minima
    __shared__ A wsum[TDP_THREADS / 32];
    A v = (o < n) ? (A)best : (A)0;
#pragma unroll
    for (int x = 16; x >= 1; x >>= 1) v += __shfl_xor_sync(FULL, v, x);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        A t = 0;
        for (int w = 0; w < TDP_THREADS / 32; ++w) t += wsum[w];
        partials[blockIdx.x] = t;
    }
}

// TD over all objects of a resident slab-free D (kmedoids_clara): thread per
// object, min over the k medoid columns of its row (M staged in shared
// memory), per-block sums in the fixed tree of k_td_points.
template <typename T, typename A>
__global__ void __launch_bounds__(256)
k_td_cols(const T* __restrict__ D, int64_t ld, int n, const int* __restrict__ M, int k, A* __restrict__ partials) {
    extern __shared__ int tc_m[];
    for (int i = threadIdx.x; i < k; i += blockDim.x) tc_m[i] = M[i];
    __syncthreads();
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    T best = dmax<T>();
    if (o < n) {
        const T* row = D + (int64_t)o * ld;
        for (int j = 0; j < k; ++j) {
            const T v = __ldg(&row[tc_m[j]]);
            best = v < best ? v : best;
        }
    }
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

// Global indices of a sample's medoids, out[i] = idx[M[i]] (the sample
// handle's local medoids mapped through the sample; one block).
__global__ void k_map_sample_medoids(const int* __restrict__ M, const int* __restrict__ idx, int k,
                                     int* __restrict__ out) {
    for (int i = threadIdx.x; i < k; i += blockDim.x) out[i] = idx[M[i]];
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
