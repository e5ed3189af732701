// km_init.cuh -- NEXT-4 initialisations.
// Random numbers are inputs drawn by the caller (the same for the oracle).
//
//   k_init_weighted  distance-weighted seeding (k-means++ adapted to arbitrary
//                    dissimilarities; reading I1):
//                    seed i is the first object whose running sum of
//                    w(o) = min_j d(x_o, m_j) exceeds u_i * W.
//   k_init_lab       LAB, Linear Approximative BUILD (reading
//                    I2): BUILD's choice restricted to a subsample of
//                    s = 10 + ceil(sqrt(n)) non-medoids per step.
// Both are sequential over the k steps and O(n) (weighted) / O(s^2 + n)
// (LAB) per step -- small next to one SWAP pass -- and run as ONE block of
// 1024 threads that loops over the steps (no launch or grid sync per step).
#pragma once
#include "km_kernels.cuh"

namespace km {

constexpr int INIT_THREADS = 1024;

template <typename A>
__device__ __forceinline__ A init_block_sum_prefix(A v, A* sh, A* total) {
    // exclusive prefix over threads in thread order; sh: INIT_THREADS entries
    sh[threadIdx.x] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        A run = 0;
        for (int t = 0; t < (int)blockDim.x; ++t) { const A x = sh[t]; sh[t] = run; run += x; }
        *total = run;
    }
    __syncthreads();
    return sh[threadIdx.x];
}

// w: n entries of scratch (D's type), ismed: n flags (zero on entry).
template <typename T, typename A>
__global__ void __launch_bounds__(INIT_THREADS)
k_init_weighted(const T* __restrict__ D, int64_t ld, int n, int k, const double* __restrict__ u,
                int* __restrict__ M, T* __restrict__ w, int* __restrict__ ismed) {
    __shared__ A sh[INIT_THREADS];
    __shared__ A s_total;
    __shared__ int s_pick;
    const int tid = threadIdx.x;
    const int chunk = (n + INIT_THREADS - 1) / INIT_THREADS;
    const int o0 = min(n, tid * chunk), o1 = min(n, o0 + chunk);
    int c = (int)(u[0] * (double)n);
    if (c >= n) c = n - 1;
    if (tid == 0) { M[0] = c; ismed[c] = 1; }
    for (int o = tid; o < n; o += INIT_THREADS) w[o] = D[(int64_t)o * ld + c];
    __syncthreads();
    for (int i = 1; i < k; ++i) {
        A part = 0;
        for (int o = o0; o < o1; ++o) part += (A)w[o];
        const A before = init_block_sum_prefix<A>(part, sh, &s_total);
        const A W = s_total;
        if (tid == 0) s_pick = INT_MAX;
        __syncthreads();
        if (W > 0) {
            const double r = u[i] * (double)W;
            if ((double)(before + part) > r && !((double)before > r)) {   // the crossing lies in this chunk
                A run = before;
                for (int o = o0; o < o1; ++o) {
                    run += (A)w[o];
                    if ((double)run > r) { atomicMin(&s_pick, o); break; }
                }
            }
        }
        __syncthreads();
        if (s_pick == INT_MAX) {                 // W = 0 (or r rounded up to W): smallest non-medoid
            for (int o = tid; o < n; o += INIT_THREADS)
                if (!ismed[o]) { atomicMin(&s_pick, o); break; }
            __syncthreads();
        }
        const int pick = s_pick;
        if (tid == 0) { M[i] = pick; ismed[pick] = 1; }
        for (int o = tid; o < n; o += INIT_THREADS) {
            const T d = D[(int64_t)o * ld + pick];
            if (d < w[o]) w[o] = d;
        }
        __syncthreads();
    }
}

// seq: k rows of (s + k) indices (-1 = padding); dnear: n scratch; S: s scratch.
template <typename T, typename A>
__global__ void __launch_bounds__(INIT_THREADS)
k_init_lab(const T* __restrict__ D, int64_t ld, int n, int k, int s, const int* __restrict__ seq,
           int* __restrict__ M, T* __restrict__ dnear, int* __restrict__ ismed, int* __restrict__ S) {
    __shared__ int s_m;
    __shared__ A sg[32];
    __shared__ int sc[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = 0; i < k; ++i) {
        if (tid == 0) {                          // the step's sample: first s non-medoids of the row
            const int* row = seq + (int64_t)i * (s + k);
            int m = 0;
            for (int j = 0; j < s + k && m < s; ++j) {
                const int c = row[j];
                if (c >= 0 && !ismed[c]) S[m++] = c;
            }
            s_m = m;
        }
        __syncthreads();
        const int m = s_m;
        A bg = amax<A>();
        int bc = INT_MAX;
        for (int a = tid; a < m; a += INIT_THREADS) {
            const int c = S[a];
            A g = 0;
            for (int b = 0; b < m; ++b) {        // sample order: the oracle's summation order
                const int o = S[b];
                const A d = (A)D[(int64_t)o * ld + c];
                if (i == 0) g += d;
                else {
                    const A delta = d - (A)dnear[o];
                    if (delta < 0) g += delta;
                }
            }
            if (g < bg || (g == bg && c < bc)) { bg = g; bc = c; }
        }
        // block lexicographic min of (g, c)
#pragma unroll
        for (int x = 16; x >= 1; x >>= 1) {
            const A og = __shfl_xor_sync(FULL, bg, x);
            const int oc = __shfl_xor_sync(FULL, bc, x);
            if (og < bg || (og == bg && oc < bc)) { bg = og; bc = oc; }
        }
        if (lane == 0) { sg[warp] = bg; sc[warp] = bc; }
        __syncthreads();
        if (warp == 0) {
            bg = sg[lane]; bc = sc[lane];
#pragma unroll
            for (int x = 16; x >= 1; x >>= 1) {
                const A og = __shfl_xor_sync(FULL, bg, x);
                const int oc = __shfl_xor_sync(FULL, bc, x);
                if (og < bg || (og == bg && oc < bc)) { bg = og; bc = oc; }
            }
            if (lane == 0) { sc[0] = bc; M[i] = bc; ismed[bc] = 1; }
        }
        __syncthreads();
        const int pick = sc[0];
        for (int o = tid; o < n; o += INIT_THREADS) {
            const T d = D[(int64_t)o * ld + pick];
            if (i == 0 || d < dnear[o]) dnear[o] = d;
        }
        __syncthreads();
    }
}

// FastCLARA (NEXT-3): the sub-matrix of a sample, sub[a][b] = d(x_S[a], x_S[b])
// = D[S[a]][S[b]] (reading R0 orientation), row stride lds.
template <typename T>
__global__ void k_gather_submatrix(const T* __restrict__ D, int64_t ld, const int* __restrict__ S, int s,
                                   T* __restrict__ sub, int64_t lds) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x, a = blockIdx.y;
    if (b >= s) return;
    sub[(int64_t)a * lds + b] = D[(int64_t)S[a] * ld + S[b]];
}

}  // namespace km
