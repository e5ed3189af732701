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
// (LAB) per step -- small next to one SWAP pass.  Default: ONE cooperative
// kernel over all SMs looping over the steps, grid syncs between a step's
// phases (*_coop); the single-block versions are kept for comparison.
#pragma once
#include "km_kernels.cuh"

namespace km {

constexpr int INIT_THREADS = 1024;

// Exclusive prefix over the threads of the block, in thread order (warp
// shuffle scans + a scan of the warp totals: a fixed tree, deterministic;
// exact for integer sums).  sh: >= 32 entries.
template <typename A>
__device__ __forceinline__ A init_block_sum_prefix(A v, A* sh, A* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
    A x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const A y = __shfl_up_sync(FULL, x, d);
        if (lane >= d) x += y;
    }
    __syncthreads();                             // sh may still be read by a previous call
    if (lane == 31) sh[warp] = x;
    __syncthreads();
    if (warp == 0) {
        A t = lane < nw ? sh[lane] : (A)0;
        const A t0 = t;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const A y = __shfl_up_sync(FULL, t, d);
            if (lane >= d) t += y;
        }
        if (lane < nw) sh[lane] = t - t0;       // exclusive warp offsets
        if (lane == 31) *total = t;
    }
    __syncthreads();
    return sh[warp] + (x - v);
}

// w: n entries of scratch (D's type), ismed: n flags (zero on entry).
template <typename T, typename A>
__global__ void __launch_bounds__(INIT_THREADS)
k_init_weighted(const T* __restrict__ D, int64_t ld, int n, int k, const double* __restrict__ u,
                int* __restrict__ M, T* __restrict__ w, int* __restrict__ ismed) {
    __shared__ A sh[32];
    __shared__ A sh2[INIT_THREADS];
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
        // the next thread's prefix (W for the last one): consecutive chunks
        // share their boundary value exactly, so one chunk holds the crossing
        sh2[tid] = before;
        if (tid == 0) s_pick = INT_MAX;
        __syncthreads();
        const A after = tid + 1 < INIT_THREADS ? sh2[tid + 1] : W;
        if (W > 0) {
            const double r = u[i] * (double)W;
            if ((double)after > r && !((double)before > r)) {   // the crossing lies in this chunk
                A run = before;
                int last = -1, got = -1;
                for (int o = o0; o < o1; ++o) {
                    const A wo = (A)w[o];
                    run += wo;
                    if (wo > 0) last = o;
                    if ((double)run > r) { got = o; break; }
                }
                // (float: the running sum may round just short of r at the end
                // of the chunk; the chunk's last positive weight is the pick)
                if (got < 0) got = last;
                if (got >= 0) atomicMin(&s_pick, got);
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

// Distance-weighted seeding over the whole GPU (cooperative; default): block
// b owns the contiguous objects [b*ch, (b+1)*ch).  Per step: block sums of
// w (coalesced) -> grid sync -> every block computes the same prefix of the
// block sums (fixed order), so exactly one block holds the crossing of
// u_i W (consecutive blocks share their boundary value exactly); it walks
// its chunk in order (warp scans of 32-object batches) -> grid sync -> every
// block folds the picked column into its w.  Exact on integer weights.
constexpr int INITW_THREADS = 512;
template <typename T, typename A>
__global__ void __launch_bounds__(INITW_THREADS)
k_init_weighted_coop(const T* __restrict__ D, int64_t ld, int n, int k, const double* __restrict__ u,
                     int* __restrict__ M, T* __restrict__ w, int* __restrict__ ismed, A* __restrict__ bsum,
                     int* __restrict__ picks) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ A sred[INITW_THREADS / 32];
    __shared__ A s_before, s_after, s_W;
    __shared__ int s_none;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nb = gridDim.x, b = blockIdx.x;
    const int ch = (n + nb - 1) / nb;
    const int o0 = min(n, b * ch), o1 = min(n, o0 + ch);
    int c = (int)(u[0] * (double)n);
    if (c >= n) c = n - 1;
    if (b == 0 && tid == 0) { M[0] = c; ismed[c] = 1; }
    for (int o = o0 + tid; o < o1; o += INITW_THREADS) w[o] = D[(int64_t)o * ld + c];
    __syncthreads();
    for (int i = 1; i < k; ++i) {
        // block sum of the chunk (fixed tree)
        A part = 0;
        for (int o = o0 + tid; o < o1; o += INITW_THREADS) part += (A)w[o];
#pragma unroll
        for (int x = 16; x >= 1; x >>= 1) part += __shfl_xor_sync(FULL, part, x);
        if (lane == 0) sred[warp] = part;
        __syncthreads();
        if (tid == 0) {
            A t = 0;
            for (int q = 0; q < INITW_THREADS / 32; ++q) t += sred[q];
            bsum[b] = t;
        }
        grid.sync();
        // prefix of the block sums, identical in every block: lane l adds the
        // blocks [l*g, (l+1)*g) serially, then an exclusive warp scan
        if (warp == 0) {
            const int g = (nb + 31) / 32;
            const int q0 = min(nb, lane * g), q1 = min(nb, q0 + g);
            A gs = 0;
            for (int q = q0; q < q1; ++q) gs += __ldcg(&bsum[q]);
            A x = gs;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const A y = __shfl_up_sync(FULL, x, d);
                if (lane >= d) x += y;
            }
            const A excl = x - gs;
            const A W = __shfl_sync(FULL, x, 31);
            // prefix before block q = excl of its lane + serial sum of the lane's blocks before q
            auto before_of = [&](int q) -> A {       // (warp-uniform q)
                if (q >= nb) return W;
                const int lq = q / g;
                A v = __shfl_sync(FULL, excl, lq);
                A run = 0;
                for (int r2 = lq * g; r2 < q; ++r2) run += __ldcg(&bsum[r2]);
                return v + run;
            };
            const A bef = before_of(b), aft = before_of(b + 1);
            if (lane == 0) { s_before = bef; s_after = aft; s_W = W; }
        }
        __syncthreads();
        const A W = s_W, bef = s_before, aft = s_after;
        const double r = u[i] * (double)W;
        // does any block cross?  [0, W) is partitioned by the shared boundaries
        const bool none = !(W > 0) || !((double)W > r);
        if (!none && (double)aft > r && !((double)bef > r)) {
            // this block: walk the chunk in index order, 32 objects per warp-0 step
            if (warp == 0) {
                A run = bef;
                int got = -1, last = -1;
                for (int base = o0; base < o1 && got < 0; base += 32) {
                    const int o = base + lane;
                    const A wo = o < o1 ? (A)w[o] : (A)0;
                    A x = wo;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const A y = __shfl_up_sync(FULL, x, d);
                        if (lane >= d) x += y;
                    }
                    const unsigned hit = __ballot_sync(FULL, o < o1 && (double)(run + x) > r);
                    const unsigned pos = __ballot_sync(FULL, o < o1 && wo > 0);
                    if (pos) last = base + 31 - __clz((int)pos);
                    if (hit) got = base + __ffs(hit) - 1;
                    run += __shfl_sync(FULL, x, 31);
                }
                // (float: the running sum may round just short of r at the end
                // of the chunk; the chunk's last positive weight is the pick)
                if (got < 0) got = last;
                if (lane == 0 && got >= 0) atomicMin(&picks[i], got);
            }
        }
        if (none) {                              // W = 0 (or r rounded up to W): smallest non-medoid
            if (tid == 0) s_none = INT_MAX;
            __syncthreads();
            for (int o = o0 + tid; o < o1; o += INITW_THREADS)
                if (!ismed[o]) { atomicMin(&s_none, o); break; }
            __syncthreads();
            if (tid == 0 && s_none != INT_MAX) atomicMin(&picks[i], s_none);
        }
        grid.sync();
        const int pick = __ldcg(&picks[i]);
        if (b == 0 && tid == 0) { M[i] = pick; ismed[pick] = 1; }
        for (int o = o0 + tid; o < o1; o += INITW_THREADS) {
            const T d = D[(int64_t)o * ld + pick];
            if (d < w[o]) w[o] = d;
        }
        __syncthreads();
    }
}

// seq: k rows of (s + k) indices (-1 = padding); dnear: n scratch; S: s
// scratch; sub: s x s scratch.  Per step, all phases run across the block:
// the sample (first s non-medoids of the row, in row order) by a block scan,
// its s x s sub-matrix gathered with all threads' loads in flight, then one
// thread per candidate sums its column of the gathered matrix in sample
// order (the oracle's summation order, so the choice is exact on float too).
template <typename T, typename A>
__global__ void __launch_bounds__(INIT_THREADS)
k_init_lab(const T* __restrict__ D, int64_t ld, int n, int k, int s, const int* __restrict__ seq,
           int* __restrict__ M, T* __restrict__ dnear, int* __restrict__ ismed, int* __restrict__ S,
           T* __restrict__ sub) {
    __shared__ int s_base;
    __shared__ int s_total;
    __shared__ int sh_scan[32];
    __shared__ A sg[32];
    __shared__ int sc[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int L = s + k;
    for (int i = 0; i < k; ++i) {
        // (1) the step's sample: first s non-medoids of row i, in row order
        const int* row = seq + (int64_t)i * L;
        if (tid == 0) s_base = 0;
        __syncthreads();
        for (int j0 = 0; j0 < L; j0 += INIT_THREADS) {
            const int base = s_base;
            if (base >= s) break;                // (uniform: s_base is shared)
            const int j = j0 + tid;
            const int c = j < L ? row[j] : -1;
            const int f = (c >= 0 && !ismed[c]) ? 1 : 0;
            const int pos = base + init_block_sum_prefix<int>(f, sh_scan, &s_total);
            if (f && pos < s) S[pos] = c;
            __syncthreads();
            if (tid == 0) s_base = base + s_total;
            __syncthreads();
        }
        const int m = min(s_base, s);
        __syncthreads();
        // (2) sub[b][a] = d(x_S[b], x_S[a]) = D[S[b]][S[a]]
        for (int64_t e = tid; e < (int64_t)m * m; e += INIT_THREADS) {
            const int b = (int)(e / m), a = (int)(e - (int64_t)b * m);
            sub[e] = D[(int64_t)S[b] * ld + S[a]];
        }
        __syncthreads();
        // (3) candidate a: gain over the sample, in sample order
        A bg = amax<A>();
        int bc = INT_MAX;
        for (int a = tid; a < m; a += INIT_THREADS) {
            const int c = S[a];
            A g = 0;
            for (int b = 0; b < m; ++b) {        // sample order: the oracle's summation order
                const A d = (A)sub[(int64_t)b * m + a];
                if (i == 0) g += d;
                else {
                    const A delta = d - (A)dnear[S[b]];
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
        // (4) d_nearest with the new medoid's column
        for (int o = tid; o < n; o += INIT_THREADS) {
            const T d = D[(int64_t)o * ld + pick];
            if (i == 0 || d < dnear[o]) dnear[o] = d;
        }
        __syncthreads();
    }
}

// LAB over the whole GPU (cooperative; default).  Per step i:
//   block 0: the sample (first s non-medoids of row i, block scan)  | grid sync
//   all blocks: gather the s x s sub-matrix; fold the previous step's
//     medoid column into d_nearest (own object chunk)                | grid sync
//   all blocks: one thread per candidate sums its column of the sub-matrix
//     in sample order (the oracle's order: exact on float), block min | grid sync
//   block 0: the lexicographic min over the blocks -> M[i], ismed    | grid sync
template <typename T, typename A>
__global__ void __launch_bounds__(INIT_THREADS)
k_init_lab_coop(const T* __restrict__ D, int64_t ld, int n, int k, int s, const int* __restrict__ seq,
                int* __restrict__ M, T* __restrict__ dnear, int* __restrict__ ismed, int* __restrict__ S,
                T* __restrict__ sub, int* __restrict__ ctl, Rec<A>* __restrict__ bmin) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ int s_base, s_total;
    __shared__ int sh_scan[32];
    __shared__ A sg[32];
    __shared__ int sc[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nb = gridDim.x, b = blockIdx.x;
    const int gt = b * INIT_THREADS + tid, nth = nb * INIT_THREADS;
    const int ch = (n + nb - 1) / nb;
    const int o0 = min(n, b * ch), o1 = min(n, o0 + ch);
    const int L = s + k;
    int prev = -1;                               // medoid of the previous step
    for (int i = 0; i < k; ++i) {
        if (b == 0) {
            const int* row = seq + (int64_t)i * L;
            if (tid == 0) s_base = 0;
            __syncthreads();
            for (int j0 = 0; j0 < L; j0 += INIT_THREADS) {
                const int base = s_base;
                if (base >= s) break;
                const int j = j0 + tid;
                const int c = j < L ? row[j] : -1;
                const int f = (c >= 0 && !ismed[c]) ? 1 : 0;
                const int pos = base + init_block_sum_prefix<int>(f, sh_scan, &s_total);
                if (f && pos < s) S[pos] = c;
                __syncthreads();
                if (tid == 0) s_base = base + s_total;
                __syncthreads();
            }
            if (tid == 0) ctl[0] = min(s_base, s);
        }
        grid.sync();
        const int m = __ldcg(&ctl[0]);
        for (int64_t e = gt; e < (int64_t)m * m; e += nth) {
            const int bb = (int)(e / m), a = (int)(e - (int64_t)bb * m);
            sub[e] = D[(int64_t)__ldcg(&S[bb]) * ld + __ldcg(&S[a])];
        }
        if (prev >= 0)
            for (int o = o0 + tid; o < o1; o += INIT_THREADS) {
                const T d = D[(int64_t)o * ld + prev];
                if (i == 1 || d < dnear[o]) dnear[o] = d;
            }
        grid.sync();
        A bg = amax<A>();
        int bc = INT_MAX;
        for (int a = gt; a < m; a += nth) {
            const int c = __ldcg(&S[a]);
            A g = 0;
            for (int bb = 0; bb < m; ++bb) {     // sample order: the oracle's summation order
                const A d = (A)__ldcg(&sub[(int64_t)bb * m + a]);
                if (i == 0) g += d;
                else {
                    const A delta = d - (A)__ldcg(&dnear[__ldcg(&S[bb])]);
                    if (delta < 0) g += delta;
                }
            }
            if (g < bg || (g == bg && c < bc)) { bg = g; bc = c; }
        }
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
            if (lane == 0) { Rec<A> r; r.v = bg; r.slot = 0; r.c = bc; bmin[b] = r; }
        }
        grid.sync();
        if (b == 0 && warp == 0) {
            Rec<A> best = rec_none<A>();
            for (int q = lane; q < nb; q += 32) {
                Rec<A> r; r.v = __ldcg(&bmin[q].v); r.slot = 0; r.c = __ldcg(&bmin[q].c);
                if (r.v < best.v || (r.v == best.v && r.c < best.c)) best = r;
            }
#pragma unroll
            for (int x = 16; x >= 1; x >>= 1) {
                const A og = __shfl_xor_sync(FULL, best.v, x);
                const int oc = __shfl_xor_sync(FULL, best.c, x);
                if (og < best.v || (og == best.v && oc < best.c)) { best.v = og; best.c = oc; }
            }
            if (lane == 0) { M[i] = best.c; ismed[best.c] = 1; ctl[1] = best.c; }
        }
        grid.sync();
        prev = __ldcg(&ctl[1]);
    }
    // the last medoid's column
    for (int o = o0 + tid; o < o1; o += INIT_THREADS) {
        const T d = D[(int64_t)o * ld + prev];
        if (k == 1 || d < dnear[o]) dnear[o] = d;
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
