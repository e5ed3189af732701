// km_kernels.cuh -- sm_100a kernels of the FastPAM SWAP / BUILD hot path.
//
// Kernel map:
//   a1/a5  k_gather_medoid_cols, k_gather_decided_col, k_assign_full, k_assign_incremental
//   a2     k_fp1_post phases 3-7 (km_post.cuh), k_part_meta
//   a3     k_swap_stream_seg2 (the HBM stream; Alg.3, Eq. eqn:better-change3)
//   a4     k_swap_combine  (per-candidate argmin over slots) + k_select
//   a7     k_build_tma / k_build_combine / k_build_select (Alg.1; incremental: km_build_delta.cuh)
//   a8     k_td_from_dn
#pragma once
#include "km_common.cuh"
#include <cooperative_groups.h>
#include <type_traits>

namespace km {

constexpr unsigned FULL = 0xffffffffu;
constexpr int SORT_CHUNK_MIN = 256;   // objects per block of the stable counting sort (at least)

// ---------------------------------------------------------------------------
// small helpers
// ---------------------------------------------------------------------------
template <typename T> struct Vec4;
template <> struct Vec4<float> { using type = float4; };
template <> struct Vec4<uint32_t> { using type = uint4; };

template <typename A>
__device__ __forceinline__ Rec<A> shfl_rec(const Rec<A>& r, int src_xor) {
    Rec<A> o;
    o.v = __shfl_xor_sync(FULL, r.v, src_xor);
    o.slot = __shfl_xor_sync(FULL, r.slot, src_xor);
    o.c = __shfl_xor_sync(FULL, r.c, src_xor);
    return o;
}

template <typename A>
__device__ __forceinline__ Rec<A> warp_min_rec(Rec<A> r) {
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        Rec<A> o = shfl_rec(r, s);
        if (rec_less(o, r)) r = o;
    }
    return r;
}

// Block-wide lexicographic min; result valid in thread 0.
template <typename A>
__device__ Rec<A> block_min_rec(Rec<A> r) {
    __shared__ Rec<A> sm[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    r = warp_min_rec(r);
    if (lane == 0) sm[warp] = r;
    __syncthreads();
    const int nw = (blockDim.x + 31) >> 5;
    if (warp == 0) {
        r = lane < nw ? sm[lane] : rec_none<A>();
        r = warp_min_rec(r);
    }
    __syncthreads();
    return r;
}

// Grid-wide lexicographic min with the last-block-done pattern: every block
// writes its partial; the last block to finish reduces them in block order
// (deterministic) and writes *out.  *counter must be 0 on entry; it is reset.
// Returns true in the last block (the minimum is then in thread 0's *res).
template <typename A>
__device__ bool grid_min_rec_last(Rec<A> r, Rec<A>* partials, unsigned* counter, Rec<A>* out, Rec<A>* res) {
    __shared__ bool am_last;
    r = block_min_rec(r);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = r;
        __threadfence();
        unsigned prev = atomicAdd(counter, 1u);
        am_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!am_last) return false;
    __threadfence();
    Rec<A> m = rec_none<A>();
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
        Rec<A> q;
        q.v = __ldcg(&partials[b].v);
        q.slot = __ldcg(&partials[b].slot);
        q.c = __ldcg(&partials[b].c);
        if (rec_less(q, m)) m = q;
    }
    m = block_min_rec(m);
    if (threadIdx.x == 0) {
        *out = m;
        *counter = 0;
        *res = m;
    }
    return true;
}
template <typename A>
__device__ void grid_min_rec(Rec<A> r, Rec<A>* partials, unsigned* counter, Rec<A>* out) {
    Rec<A> m;
    grid_min_rec_last(r, partials, counter, out, &m);
}

// ---------------------------------------------------------------------------
// a1/a5: medoid columns and the nearest/second cache
// ---------------------------------------------------------------------------

// Input validation (include/kmedoids.h conventions: d(x_o, x_o) = 0, d >= 0,
// no NaN).  *bad counts the violations:
//   k_validate_diag: the diagonal entries of the slab, D[o][o - col_begin]
//     for o in [col_begin, col_end) (a NaN also fails "== 0");
//   k_validate_cols: the k*n gathered medoid columns (float path: d < 0 or
//     NaN; the uint32 path has no invalid values).
template <typename T>
__global__ void k_validate_diag(const T* __restrict__ D, int64_t ld, int64_t col_begin, int64_t col_end,
                                int* __restrict__ bad) {
    const int64_t o = col_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int b = 0;
    if (o < col_end) b = !(D[o * ld + (o - col_begin)] == (T)0);
    b = __syncthreads_count(b);
    if (threadIdx.x == 0 && b) atomicAdd(bad, b);
}

template <typename T>
__global__ void k_validate_cols(const T* __restrict__ MC, int64_t cnt, int* __restrict__ bad) {
    int b = 0;
    if constexpr (std::is_same<T, float>::value) {
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
            b |= !(MC[i] >= 0.f);
    }
    b = __syncthreads_or(b);
    if (threadIdx.x == 0 && b) atomicAdd(bad, 1);
}

// Exact symmetry of the n x n matrix (kmedoids_set_symmetric): tile (bi, bj)
// with bi <= bj is compared with the transpose of tile (bj, bi) through
// shared memory (both read coalesced: one pass over D); *bad counts the
// mismatching pairs (bitwise comparison).
template <typename T>
__global__ void k_check_symmetric(const T* __restrict__ D, int64_t ld, int n, int* __restrict__ bad) {
    __shared__ T ta[32][33], tb[32][33];
    const int bi = blockIdx.y, bj = blockIdx.x;
    if (bj < bi) return;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;     // 32 x 8 threads
    for (int r = ty; r < 32; r += 8) {
        const int i = bi * 32 + r, j = bj * 32 + tx;
        ta[r][tx] = (i < n && j < n) ? D[(int64_t)i * ld + j] : (T)0;
        const int i2 = bj * 32 + r, j2 = bi * 32 + tx;
        tb[r][tx] = (i2 < n && j2 < n) ? D[(int64_t)i2 * ld + j2] : (T)0;
    }
    __syncthreads();
    int cnt = 0;
    for (int r = ty; r < 32; r += 8) {
        uint32_t a, b;                                  // bitwise (4-byte elements)
        const T va = ta[r][tx], vb = tb[tx][r];
        memcpy(&a, &va, 4); memcpy(&b, &vb, 4);
        cnt += a != b;
    }
    cnt = __syncthreads_count(cnt);
    if (threadIdx.x == 0 && cnt) atomicAdd(bad, cnt);
}

// MC[j][o] = d(x_o, m_j) for every slot j whose medoid lies in the local
// column range (single GPU: all of them).  grid = (ceil(n/256), k).
template <typename T>
__global__ void k_gather_medoid_cols(const T* __restrict__ D, int64_t ld, int n, int64_t col_begin,
                                     int64_t col_end, const int* __restrict__ M, T* __restrict__ MC) {
    const int j = blockIdx.y;
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t c = M[j];
    if (o >= n || c < col_begin || c >= col_end) return;
    MC[(int64_t)j * n + o] = D[(int64_t)o * ld + (c - col_begin)];
}

// Column of the decided swap/BUILD candidate: MC[slot][o] = d(x_o, x_c*),
// written only when the decision applies and c* is local.  For a sharded
// handle `colbuf` (n elements) also receives the column (pack for broadcast).
template <typename T, typename A>
__global__ void k_gather_decided_col(const T* __restrict__ D, int64_t ld, int n, int64_t col_begin,
                                     int64_t col_end, const Decision<A>* __restrict__ dec,
                                     T* __restrict__ MC, T* __restrict__ colbuf) {
    if (!dec->apply) return;
    const int64_t c = dec->c;
    if (c < col_begin || c >= col_end) return;
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= n) return;
    T v = D[(int64_t)o * ld + (c - col_begin)];
    if (MC) MC[(int64_t)dec->slot * n + o] = v;
    if (colbuf) colbuf[o] = v;
}

// Sharded: column c (global index, local to this rank) -> colbuf[o] = d(x_o, x_c).
template <typename T>
__global__ void k_gather_col(const T* __restrict__ D, int64_t ld, int n, int64_t col_begin, int c,
                             T* __restrict__ colbuf) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o < n) colbuf[o] = D[(int64_t)o * ld + (c - col_begin)];
}

// Columns cols[0..cnt) of the slab into out[j][o] (grid.y = cnt): the
// FastPAM2 sharded pack in one launch.
template <typename T>
__global__ void k_gather_cols(const T* __restrict__ D, int64_t ld, int n, int64_t col_begin,
                              const int* __restrict__ cols, T* __restrict__ out) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    const int c = cols[blockIdx.y];
    if (o < n) out[(int64_t)blockIdx.y * n + o] = D[(int64_t)o * ld + (c - col_begin)];
}

// Sharded, device-decided iteration (no host round trip): the status of the
// run, mirrored into pinned host memory by the decide kernel.
template <typename A>
struct alignas(16) ShardStatus {
    A td;            // TD after the iteration
    int32_t conv;    // sticky: 1 once an iteration found no improving swap
    int32_t iters;   // iterations counted (the converging one included; later ones not)
    int32_t swaps;
    int32_t apply;   // this iteration applied a swap
    int32_t calls;   // decide calls so far (iterations enqueued, counted or not)
    int32_t pad[3];
};
constexpr int SHARD_MIRRORS = 4;   // ring of pinned status copies, one per decide call

// Reading R1/R5 on the gathered records, as k_select, but sticky: after the
// converging iteration every further one is a no-op (apply = 0, nothing
// counted), so a caller may enqueue iterations ahead of reading the status.
// Applied swaps are appended to trace[] (dTD, slot, c).
template <typename A>
__global__ void k_shard_decide(const Rec<A>* __restrict__ recs, int nrec, A* __restrict__ td, int* __restrict__ M,
                               int* __restrict__ point_slot, Decision<A>* __restrict__ dec,
                               int* __restrict__ rescan_count, ShardStatus<A>* __restrict__ status,
                               ShardStatus<A>* __restrict__ mirror, Rec<A>* __restrict__ trace, int trace_cap) {
    *rescan_count = 0;
    dec->apply = 0;
    if (!status->conv) {
        Rec<A> b = rec_none<A>();
        for (int r = 0; r < nrec; ++r)
            if (rec_less(recs[r], b)) b = recs[r];
        bool improving;
        if (b.slot == INT_MAX) improving = false;
        else if (std::is_same<A, double>::value) improving = (double)b.v < -1e-12 * fabs((double)*td);
        else improving = b.v < 0;
        dec->iters += 1;
        status->iters += 1;
        dec->dtd = b.v;
        dec->slot = b.slot;
        dec->c = b.c;
        if (improving) {
            dec->apply = 1;
            const int old = M[b.slot];
            dec->old_m = old;
            M[b.slot] = b.c;
            point_slot[old] = -1;
            point_slot[b.c] = b.slot;
            *td += b.v;
            dec->swaps += 1;
            if (status->swaps < trace_cap) trace[status->swaps] = b;
            status->swaps += 1;
        } else {
            status->conv = 1;
        }
    }
    status->apply = dec->apply;
    status->td = *td;
    status->calls += 1;
    // pinned host ring: the host reads the copy of a given call once that
    // call's iteration is known complete, so every rank reads the same status
    mirror[(status->calls - 1) % SHARD_MIRRORS] = *status;
}

// The decided column into the exchange buffer: the owner rank copies column
// c* of its slab, every other rank writes zeros, so a SUM all-reduce of the
// buffers delivers the column everywhere (x + 0 = x exactly) without the host
// knowing the owner.
template <typename T, typename A>
__global__ void k_shard_pack_decided(const T* __restrict__ D, int64_t ld, int n, int64_t col_begin, int64_t col_end,
                                     const Decision<A>* __restrict__ dec, T* __restrict__ colbuf) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= n) return;
    const int64_t c = dec->c;
    const bool mine = dec->apply && c >= col_begin && c < col_end;
    colbuf[o] = mine ? D[(int64_t)o * ld + (c - col_begin)] : (T)0;
}

// Sharded: copy the broadcast column into MC[slot].
template <typename T, typename A>
__global__ void k_column_to_mc(const T* __restrict__ colbuf, int n, const Decision<A>* __restrict__ dec,
                               T* __restrict__ MC) {
    if (!dec->apply) return;
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o < n) MC[(int64_t)dec->slot * n + o] = colbuf[o];
}

// nearest = lexicographic argmin over slots of (d(x_o, m_j), j); second = the
// same over j != nearest (reading R2).  One thread per object; MC reads are
// coalesced across threads.  Needs k >= 2.
template <typename T>
__global__ void k_assign_full(const T* __restrict__ MC, int n, int k, int* __restrict__ near,
                              int* __restrict__ sec, T* __restrict__ dn, T* __restrict__ ds) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= n) return;
    T a = MC[o], b = MC[(int64_t)n + o];
    T d1, d2;
    int j1, j2;
    if (b < a) { d1 = b; j1 = 1; d2 = a; j2 = 0; } else { d1 = a; j1 = 0; d2 = b; j2 = 1; }
    for (int j = 2; j < k; ++j) {
        T d = MC[(int64_t)j * n + o];
        if (d < d1) { d2 = d1; j2 = j1; d1 = d; j1 = j; }
        else if (d < d2) { d2 = d; j2 = j; }
    }
    near[o] = j1; sec[o] = j2; dn[o] = d1; ds[o] = d2;
}

// Incremental update after slot i = dec->slot received a new medoid whose
// column is MC[i]: every object not served by slot i only compares the new
// medoid against its current (nearest, second) pair; objects whose nearest or
// second WAS slot i (about 2n/k of them) are appended to `rescan` and handled
// by k_assign_rescan (one warp per object).  Together equal to k_assign_full
// on the new medoid set (tested).  *rescan_count is reset by k_select.
template <typename T, typename A>
__global__ void k_assign_incremental(const T* __restrict__ MC, int n, int k,
                                     const Decision<A>* __restrict__ dec, int* __restrict__ near,
                                     int* __restrict__ sec, T* __restrict__ dn, T* __restrict__ ds,
                                     int* __restrict__ rescan, int* __restrict__ rescan_count) {
    if (!dec->apply) return;
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= n) return;
    const int i = dec->slot;
    const int j1 = near[o], j2 = sec[o];
    if (j1 == i || j2 == i) {
        rescan[atomicAdd(rescan_count, 1)] = o;
        return;
    }
    const T x = MC[(int64_t)i * n + o];
    const T d1 = dn[o], d2 = ds[o];
    if (x < d1 || (x == d1 && i < j1)) {
        near[o] = i; dn[o] = x; sec[o] = j1; ds[o] = d1;
    } else if (x < d2 || (x == d2 && i < j2)) {
        sec[o] = i; ds[o] = x;
    }
}

// (d, j) lexicographic top-2 of the k medoid columns for one object, one
// warp per listed object: lanes scan slots j = lane, lane+32, ... and the
// per-lane top-2 lists are merged with shuffles (result independent of the
// merge order, so deterministic).
template <typename T>
__device__ __forceinline__ bool lex_lt(T a, int ja, T b, int jb) { return a < b || (a == b && ja < jb); }

template <typename T, typename A>
__global__ void k_assign_rescan(const T* __restrict__ MC, int n, int k, const Decision<A>* __restrict__ dec,
                                const int* __restrict__ rescan, const int* __restrict__ rescan_count,
                                int* __restrict__ near, int* __restrict__ sec, T* __restrict__ dn,
                                T* __restrict__ ds) {
    if (!dec->apply) return;
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const int cnt = *rescan_count;
    for (int e = gw; e < cnt; e += nw) {
        const int o = rescan[e];
        T d1 = dmax<T>(), d2 = dmax<T>();
        int j1 = INT_MAX, j2 = INT_MAX;
        for (int j = lane; j < k; j += 32) {
            const T d = MC[(int64_t)j * n + o];
            if (lex_lt(d, j, d1, j1)) { d2 = d1; j2 = j1; d1 = d; j1 = j; }
            else if (lex_lt(d, j, d2, j2)) { d2 = d; j2 = j; }
        }
#pragma unroll
        for (int x = 16; x >= 1; x >>= 1) {
            const T e1 = __shfl_xor_sync(FULL, d1, x), e2 = __shfl_xor_sync(FULL, d2, x);
            const int f1 = __shfl_xor_sync(FULL, j1, x), f2 = __shfl_xor_sync(FULL, j2, x);
            // merge (d1,j1) <= (d2,j2) with (e1,f1) <= (e2,f2)
            if (lex_lt(e1, f1, d1, j1)) {
                if (lex_lt(d1, j1, e2, f2)) { d2 = d1; j2 = j1; } else { d2 = e2; j2 = f2; }
                d1 = e1; j1 = f1;
            } else if (lex_lt(e1, f1, d2, j2)) {
                d2 = e1; j2 = f1;
            }
        }
        if (lane == 0) { near[o] = j1; sec[o] = j2; dn[o] = d1; ds[o] = d2; }
    }
}

// TD = sum_o d_n(o) (Eq. eqn:td), fixed reduction order.
template <typename T, typename A>
__global__ void k_td_from_dn(const T* __restrict__ dn, int n, A* __restrict__ partials,
                             unsigned* __restrict__ counter, A* __restrict__ td) {
    __shared__ A sm[32];
    __shared__ bool am_last;
    A s = 0;
    for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < n; o += gridDim.x * blockDim.x) s += (A)dn[o];
#pragma unroll
    for (int x = 16; x >= 1; x >>= 1) s += __shfl_xor_sync(FULL, s, x);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        A t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sm[w];
        partials[blockIdx.x] = t;
        __threadfence();
        am_last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (am_last && threadIdx.x == 0) {
        __threadfence();
        A t = 0;
        for (int b = 0; b < (int)gridDim.x; ++b) t += __ldcg(&partials[b]);
        *td = t;
        *counter = 0;
    }
}

// ---------------------------------------------------------------------------
// a2: the slot sort, removal losses and part metadata run as phases of the
// cooperative k_fp1_post (km_post.cuh); k_part_meta is also used alone.
// ---------------------------------------------------------------------------
// Slot of the first / last row of every stream part (the post kernel's
// phase 7 computes the same).
template <typename T>
__global__ void k_part_meta(const RowInfo<T>* __restrict__ ri, int n, int P, int* __restrict__ head_slot,
                            int* __restrict__ tail_slot) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= P) return;
    const int64_t p0 = part_lo(q, n, P), p1 = part_lo(q + 1, n, P);
    head_slot[q] = ri[p0].slot;
    tail_slot[q] = ri[p1 - 1].slot;
}

namespace ptx {
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(bar)) : "memory");
}
// try_wait with a suspend-time hint: the warp sleeps until the phase
// completes (or the hint expires) instead of spinning through issue slots.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "KM_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n\t"
        "@!P bra KM_WAIT_%=;\n}" ::"r"(sa(bar)),
        "r"(parity), "r"(0x989680u)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// 8- / 4-byte stores with an L2 eviction-priority hint
__device__ __forceinline__ void st_hint(double* p, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" :: "l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint(long long* p, long long v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.b64 [%0], %1, %2;" :: "l"(p), "l"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint(int* p, int v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" :: "l"(p), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            sa(dst)),
        "l"(src), "r"(bytes), "r"(sa(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
                 "l"(src), "r"(bytes), "r"(sa(bar))
                 : "memory");
}
}  // namespace ptx

// ---------------------------------------------------------------------------
// a3: the SWAP-delta stream (Alg.3, Eq. eqn:better-change3).
//
// A CTA owns NC*128 consecutive candidate columns (lane l of consumer warp w
// owns 4 of them); blockIdx.y selects a part of the slot-sorted row order.
// Per candidate column c and row o (d = D[o][c]):
//     d < d_n(o):          plus_c += d - d_n(o);  acc_c[nearest(o)] += d_n - d_s
//     d_n(o) <= d < d_s(o): acc_c[nearest(o)] += d - d_s(o)
// Because rows arrive grouped by nearest(o), acc_c[i] is a running segment
// sum held in registers; at the end of each slot's segment R_i + acc_c[i] is
// final and enters a running lexicographic min, or is emitted as the part's
// head / tail partial sum (segments cut by part boundaries, completed by
// k_swap_combine).  No k-vector is ever materialised (FastPAM2 mode stores
// the complete per-slot sums instead).
//
// Delivery: a producer warp moves each row chunk of the column tile with one
// cp.async.bulk (TMA bulk copy, SASS UBLKCP) into an S-stage shared-memory
// ring guarded by mbarriers, and never lets a stage straddle two slots (a
// stage holds up to RB rows of ONE segment), so the consumers close a
// segment only between stages (one warp-uniform check).
// ---------------------------------------------------------------------------
// A threshold no value compares below (uint32: 0; float: -inf, false even for NaN).
template <typename T> __device__ __forceinline__ T never_lt();
template <> __device__ __forceinline__ uint32_t never_lt<uint32_t>() { return 0u; }
template <> __device__ __forceinline__ float never_lt<float>() { return -INFINITY; }

template <typename T> struct CmpLt;
template <> struct CmpLt<float> {
    // 1 if any a_u < b_u (u = 0..3)
    __device__ __forceinline__ static unsigned any4(float a0, float b0, float a1, float b1, float a2, float b2,
                                                    float a3, float b3) {
        unsigned r;
        asm("{\n\t.reg .pred p;\n\t"
            "setp.lt.f32 p, %1, %2;\n\t"
            "setp.lt.or.f32 p, %3, %4, p;\n\t"
            "setp.lt.or.f32 p, %5, %6, p;\n\t"
            "setp.lt.or.f32 p, %7, %8, p;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(r)
            : "f"(a0), "f"(b0), "f"(a1), "f"(b1), "f"(a2), "f"(b2), "f"(a3), "f"(b3));
        return r;
    }
};
template <> struct CmpLt<uint32_t> {
    __device__ __forceinline__ static unsigned any4(uint32_t a0, uint32_t b0, uint32_t a1, uint32_t b1, uint32_t a2,
                                                    uint32_t b2, uint32_t a3, uint32_t b3) {
        unsigned r;
        asm("{\n\t.reg .pred p;\n\t"
            "setp.lt.u32 p, %1, %2;\n\t"
            "setp.lt.or.u32 p, %3, %4, p;\n\t"
            "setp.lt.or.u32 p, %5, %6, p;\n\t"
            "setp.lt.or.u32 p, %7, %8, p;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(r)
            : "r"(a0), "r"(b0), "r"(a1), "r"(b1), "r"(a2), "r"(b2), "r"(a3), "r"(b3));
        return r;
    }
};

template <typename T, int NC, int RB, int S>
struct SegCfg {
    static constexpr int COLS = NC * 128;
    static constexpr int ROWB = COLS * (int)sizeof(T);
    static constexpr int DATAB = S * RB * ROWB;
    static constexpr int RIB = S * RB * 16;
    static constexpr int NBB = S * 4;                   // rows in each stage
    static constexpr int BARB = 2 * S * 8;
    static constexpr int RDB = S * RB * 16;             // float path: (double dn, double ds) per row
    static constexpr int SMEM = DATAB + RIB + RDB + 16 * ((NBB + 15) / 16) + BARB;
    static constexpr int THREADS = (NC + 1) * 32;
};


// ---------------------------------------------------------------------------
// a3 consumer (k_swap_stream_seg2).  Per-stage instruction count kept low
// (ncu source page of the round-1 predecessor: ~85 instructions per
// warp-stage outside the hit path, ~60 per hit column):
//   * columns no lane owns (beyond the slab) are filled once with the
//     largest value, so no per-stage threshold masking is needed;
//   * stage index / phase by counters (no modulo);
//   * one warp vote per column (VOTE.ANY) instead of mask building + REDUX;
//   * the hit terms in the form q = [d < d_s](d - d_s), t = [d < d_n](d - d_n):
//     acc += sum q - sum t, plus += sum t (Alg.3: for d < d_n the
//     row adds d_n - d_s = q - t to acc and t to plus; for d_n <= d < d_s it
//     adds q), which needs 8 fp64 selects per column instead of 16.
// Per row the terms are exact (differences of two f32 / u32 values are
// exact in fp64 / int64); only the summation grouping differs from the
// oracle's object order (reading R9).
// ---------------------------------------------------------------------------
template <typename T, typename A, int NC, int RB, int S, int MINB = 2>
__global__ void __launch_bounds__((NC + 1) * 32, MINB)
k_swap_stream_seg2(const T* __restrict__ D, int64_t ld, int w, int wpad, int n, int P,
                   const RowInfo<T>* __restrict__ ri, const A* __restrict__ R,
                   A* __restrict__ out_plus, A* __restrict__ out_head, A* __restrict__ out_tail,
                   A* __restrict__ out_imin, int* __restrict__ out_islot, A* __restrict__ out_acc,
                   const double2* __restrict__ rowd, bool acc_keep, const int* __restrict__ skip_if) {
    using C = SegCfg<T, NC, RB, S>;
    using V = typename Vec4<T>::type;
    static_assert(RB == 4, "four rows per stage");
    // a queued FastPAM1 iteration after convergence (Decision::done): no-op
    if (skip_if && __ldcg(skip_if)) return;
    extern __shared__ __align__(128) unsigned char smem[];
    T* sdata = reinterpret_cast<T*>(smem);
    RowInfo<T>* sri = reinterpret_cast<RowInfo<T>*>(smem + C::DATAB);
    double2* srd = reinterpret_cast<double2*>(smem + C::DATAB + C::RIB);
    int* snb = reinterpret_cast<int*>(smem + C::DATAB + C::RIB + C::RDB);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::DATAB + C::RIB + C::RDB + 16 * ((C::NBB + 15) / 16));
    uint64_t* empty = full + S;

    const int q = blockIdx.y;
    const int64_t p0 = part_lo(q, n, P), p1 = part_lo(q + 1, n, P);
    const int ctacol = blockIdx.x * C::COLS;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // consumer warps owning at least one column of the slab (all NC but in
    // the last, ragged column tile); the others leave at once, so a narrow
    // last tile streams at the pace of its active warps (C3: 288 of 896)
    const int nact = min(NC, (w - ctacol + 127) / 128);

    if (threadIdx.x == 0) {
        for (int st = 0; st < S; ++st) {
            ptx::mbar_init(&full[st], 1);
            ptx::mbar_init(&empty[st], nact);
        }
        ptx::fence_mbar_init();
    }
    // columns beyond the slab are never written by the bulk copies: give them
    // a value no threshold exceeds (each lane fills its own columns)
    if (warp < nact && ctacol + warp * 128 + lane * 4 >= wpad) {
        V big;
        const T b = dmax<T>();
        memcpy(&big.x, &b, sizeof(T)); memcpy(&big.y, &b, sizeof(T));
        memcpy(&big.z, &b, sizeof(T)); memcpy(&big.w, &b, sizeof(T));
        for (int r = 0; r < S * RB; ++r)
            *reinterpret_cast<V*>(sdata + (size_t)r * C::COLS + warp * 128 + lane * 4) = big;
    }
    __syncthreads();

    if (warp == NC) {
        // ---------------- producer warp ----------------
        const uint32_t cbytes = (uint32_t)min(C::COLS, wpad - ctacol) * (uint32_t)sizeof(T);
        const uint64_t pol = ptx::policy_evict_first();
        const uint64_t keep = ptx::policy_evict_last();   // row metadata: re-read by every column tile
        int64_t pr = p0;
        int s = 0, ph = 0, st = 0;
        // row metadata in a 64-row register window: lane l holds (o, slot)
        // of rows wb + l (current half) and wb + 32 + l (next half, loaded
        // 32 rows ahead), so forming a stage never waits on a global load
        // (round 1 reloaded the vacated rows every stage: one dependent L2
        // round trip in the producer's loop)
        int64_t wb = p0;
        int o_c = 0, s_c = -1, o_n = 0, s_n = -1;
        if (wb + lane < p1) { const RowInfo<T> r = ri[wb + lane]; o_c = r.o; s_c = r.slot; }
        if (wb + 32 + lane < p1) { const RowInfo<T> r = ri[wb + 32 + lane]; o_n = r.o; s_n = r.slot; }
        while (true) {
            if (st >= S) ptx::mbar_wait(&empty[s], ph ^ 1);
            if (pr >= p1) {
                if (lane == 0) {
                    snb[s] = 0;
                    ptx::mbar_arrive(&full[s]);
                }
                break;
            }
            // rows pr .. pr + RB - 1 (window positions li .. li + RB - 1 < 64)
            const int li = (int)(pr - wb);
            const int src = (li + lane) & 31;
            const int oc = __shfl_sync(FULL, o_c, src), sc = __shfl_sync(FULL, s_c, src);
            const int on = __shfl_sync(FULL, o_n, src), sn = __shfl_sync(FULL, s_n, src);
            const int o_l = li + lane < 32 ? oc : on, sl_l = li + lane < 32 ? sc : sn;
            const int slot0 = __shfl_sync(FULL, sl_l, 0);
            const unsigned same = __ballot_sync(FULL, lane < RB && sl_l == slot0 && pr + lane < p1);
            const int nb = __ffs(~same) - 1;
            if (lane == 0) {
                snb[s] = nb;
                ptx::mbar_expect_tx(&full[s], (uint32_t)nb * (cbytes + (rowd ? 32u : 16u)));
            }
            __syncwarp();
            KM_ASSERT(lane >= nb || (o_l >= 0 && o_l < n));
            if (lane < nb)
                ptx::bulk_g2s(sdata + (size_t)(s * RB + lane) * C::COLS, D + (int64_t)o_l * ld + ctacol, cbytes,
                              &full[s], pol);
            if (lane == 0) ptx::bulk_g2s(sri + s * RB, ri + pr, (uint32_t)nb * 16u, &full[s], keep);
            if (lane == 1 && rowd) ptx::bulk_g2s(srd + s * RB, rowd + pr, (uint32_t)nb * 16u, &full[s], keep);
            pr += nb;
            if (pr - wb >= 32) {                 // advance the window by 32 rows, prefetch the next half
                wb += 32;
                o_c = o_n; s_c = s_n;
                s_n = -1;
                if (wb + 32 + lane < p1) { const RowInfo<T> r = ri[wb + 32 + lane]; o_n = r.o; s_n = r.slot; }
            }
            ++st;
            if (++s == S) { s = 0; ph ^= 1; }
        }
        return;
    }

    // ---------------- consumer warps ----------------
    if (warp >= nact) return;
    const int cb = ctacol + warp * 128 + lane * 4;
    const bool active = cb < w;
    const int64_t obase = (int64_t)q * w + cb;
    const int jmax = active ? min(4, w - cb) : 0;
    // the part outputs (read by the combine right after the stream) are
    // stored with L2 evict_last, the streamed D rows are loaded evict_first
    const uint64_t keep = ptx::policy_evict_last();
    A plus[4], seg[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) { plus[j] = 0; seg[j] = 0; }
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (j < jmax) {
            ptx::st_hint(&out_imin[obase + j], amax<A>(), keep);
            ptx::st_hint(&out_islot[obase + j], -1, keep);
            ptx::st_hint(&out_head[obase + j], (A)0, keep);
        }
    int cur = ri[p0].slot;
    bool first = true;
    const T* srow0 = sdata + (warp * 128 + lane * 4);
    int s = 0, ph = 0;

    for (;;) {
        ptx::mbar_wait(&full[s], ph);
        const int nb = snb[s];
        if (nb == 0) break;
        const RowInfo<T>* srii = sri + s * RB;
        const int slot = srii[0].slot;
        if (slot != cur) {                       // segment boundary (warp-uniform, rare)
            if (first) {
#pragma unroll
                for (int j = 0; j < 4; ++j) if (j < jmax) ptx::st_hint(&out_head[obase + j], seg[j], keep);
                first = false;
            } else {
                const A rv = R[cur];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (j >= jmax) continue;
                    if (out_acc) {
                        if (acc_keep) ptx::st_hint(&out_acc[(int64_t)cur * w + cb + j], seg[j], keep);
                        else out_acc[(int64_t)cur * w + cb + j] = seg[j];
                    }
                    const A val = rv + seg[j];
                    if (val < out_imin[obase + j]) {
                        ptx::st_hint(&out_imin[obase + j], val, keep);
                        ptx::st_hint(&out_islot[obase + j], cur, keep);
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) seg[j] = 0;
            cur = slot;
        }
        T x[RB][4], dn[RB], ds[RB];
        const T* srow = srow0 + (size_t)(s * RB) * C::COLS;
#pragma unroll
        for (int u = 0; u < RB; ++u) {
            const V v = *reinterpret_cast<const V*>(srow + (size_t)u * C::COLS);
            memcpy(&x[u][0], &v.x, sizeof(T)); memcpy(&x[u][1], &v.y, sizeof(T));
            memcpy(&x[u][2], &v.z, sizeof(T)); memcpy(&x[u][3], &v.w, sizeof(T));
            dn[u] = srii[u].dn;
            ds[u] = srii[u].ds;
        }
        if (nb < RB) {                           // short stage at a segment end (rare)
#pragma unroll
            for (int u = 1; u < RB; ++u)
                if (u >= nb) { dn[u] = never_lt<T>(); ds[u] = never_lt<T>(); }
        }
        bool hit[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            hit[j] = __any_sync(FULL, CmpLt<T>::any4(x[0][j], ds[0], x[1][j], ds[1], x[2][j], ds[2], x[3][j], ds[3]));
        const int cs = s;
        if (++s == S) { s = 0; ph ^= 1; }
        if (!(hit[0] || hit[1] || hit[2] || hit[3])) {
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&empty[cs]);
            continue;
        }
        A dnA[RB], dsA[RB];
        if constexpr (Acc<T>::is_float) {       // widened thresholds staged by the producer
            const double2* sr = srd + cs * RB;
#pragma unroll
            for (int u = 0; u < RB; ++u) { const double2 qq = sr[u]; dnA[u] = qq.x; dsA[u] = qq.y; }
            if (nb < RB) {                              // rows beyond a short stage never compare below
#pragma unroll
                for (int u = 1; u < RB; ++u)
                    if (u >= nb) { dnA[u] = -INFINITY; dsA[u] = -INFINITY; }
            }
        } else {
#pragma unroll
            for (int u = 0; u < RB; ++u) { dnA[u] = (A)dn[u]; dsA[u] = (A)ds[u]; }
        }
        __syncwarp();                            // stage values are in registers: release it
        if (lane == 0) ptx::mbar_arrive(&empty[cs]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (hit[j]) {
                A tq[RB], tt[RB];
#pragma unroll
                for (int u = 0; u < RB; ++u) {
                    const A xa = (A)x[u][j];
                    // compared on the widened values (exact): the f32 dn / ds
                    // are dead after the vote (round 2: no spills, C4 stream
                    // -19 us, C3 -9 us against f32 compares here)
                    tq[u] = (xa < dsA[u]) ? xa - dsA[u] : (A)0;
                    tt[u] = (xa < dnA[u]) ? xa - dnA[u] : (A)0;
                }
                const A sq = (tq[0] + tq[1]) + (tq[2] + tq[3]);
                const A sp = (tt[0] + tt[1]) + (tt[2] + tt[3]);
                plus[j] += sp;
                seg[j] += sq - sp;
            }
        }
    }
    if (!active) return;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (j >= jmax) continue;
        if (first) { ptx::st_hint(&out_head[obase + j], seg[j], keep); ptx::st_hint(&out_tail[obase + j], (A)0, keep); }
        else ptx::st_hint(&out_tail[obase + j], seg[j], keep);
        ptx::st_hint(&out_plus[obase + j], plus[j], keep);
    }
}

// a4: complete the segments cut by part boundaries, take the lexicographic
// min over slots of (R_i + acc_i, i) (Alg.3, smaller slot on ties), add
// dTD^{+x_c}, mask medoids, and reduce (dTD, i, c) over the grid.
template <typename A, int QU = 8>
__global__ void k_swap_combine(int w, int64_t col_begin, int P, const A* __restrict__ in_plus,
                               const A* __restrict__ in_head, const A* __restrict__ in_tail,
                               const A* __restrict__ in_imin, const int* __restrict__ in_islot,
                               const int* __restrict__ head_slot, const int* __restrict__ tail_slot,
                               const A* __restrict__ R, const int* __restrict__ empty_slot,
                               const int* __restrict__ point_slot, A* __restrict__ cand_v,
                               int* __restrict__ cand_slot, Rec<A>* partials, unsigned* counter,
                               Rec<A>* out, A* __restrict__ acc_out = nullptr, A* __restrict__ plus_out = nullptr,
                               int k = 0, bool stage = false) {
    // R and the part head/tail slots staged in shared memory (when they fit):
    // the fold's R[s] lookups and slot compares then wait ~30 cycles, not an
    // L1/L2 round trip each (ncu: stalls on the DADD after every R load)
    extern __shared__ __align__(16) unsigned char comb_smem[];
    if (stage) {
        A* sR = reinterpret_cast<A*>(comb_smem);
        int* shs = reinterpret_cast<int*>(comb_smem + (size_t)k * sizeof(A));
        for (int i = threadIdx.x; i < k; i += blockDim.x) sR[i] = R[i];
        for (int i = threadIdx.x; i < P; i += blockDim.x) { shs[i] = head_slot[i]; shs[P + i] = tail_slot[i]; }
        __syncthreads();
        R = sR; head_slot = shs; tail_slot = shs + P;
    }
    const int cl = blockIdx.x * blockDim.x + threadIdx.x;
    Rec<A> best = rec_none<A>();
    if (cl < w) {
        A bv = amax<A>();
        int bs = INT_MAX;
        const int es = *empty_slot;
        if (es != INT_MAX) { bv = 0; bs = es; }
        auto fin = [&](int s, A sum) {
            KM_ASSERT(s >= 0 && s < k);
            if (acc_out) acc_out[(int64_t)s * w + cl] = sum;     // FastPAM2: complete acc_c[s]
            const A val = R[s] + sum;
            if (val < bv || (val == bv && s < bs)) { bv = val; bs = s; }
        };
        A plus = 0, carry = 0;
        int cs = -1;
        // QU parts loaded ahead (memory-level parallelism: one thread per
        // column gives only ~10 warps per SM at C4, so each keeps 5 QU loads
        // in flight); the part slots are read in the fold (shared memory)
        for (int q0 = 0; q0 < P; q0 += QU) {
            A pl[QU], hv[QU], tv[QU], iv[QU];
            int isl[QU];
#pragma unroll
            for (int u = 0; u < QU; ++u) {
                const int q = q0 + u;
                if (q < P) {
                    const int64_t idx = (int64_t)q * w + cl;
                    pl[u] = in_plus[idx]; hv[u] = in_head[idx]; tv[u] = in_tail[idx];
                    iv[u] = in_imin[idx]; isl[u] = in_islot[idx];
                }
            }
#pragma unroll
            for (int u = 0; u < QU; ++u) {
                if (q0 + u >= P) break;
                plus += pl[u];
                const int h = head_slot[q0 + u], t = tail_slot[q0 + u];
                if (h == cs) {
                    carry += hv[u];
                } else {
                    if (cs >= 0) fin(cs, carry);
                    cs = h;
                    carry = hv[u];
                }
                if (isl[u] >= 0 && (iv[u] < bv || (iv[u] == bv && isl[u] < bs))) { bv = iv[u]; bs = isl[u]; }
                if (t != h) {
                    fin(cs, carry);
                    cs = t;
                    carry = tv[u];
                }
            }
        }
        fin(cs, carry);
        if (plus_out) plus_out[cl] = plus;
        const A dtd = bv + plus;
        const int64_t c = col_begin + cl;
        const bool medoid = point_slot[c] >= 0;
        cand_v[cl] = dtd;
        cand_slot[cl] = medoid ? -1 : bs;
        if (!medoid) { best.v = dtd; best.slot = bs; best.c = (int)c; }
    }
    grid_min_rec(best, partials, counter, out);
}

// Acceptance (reading R5) and bookkeeping of the chosen swap (Alg.3):
// lexicographic min over the gathered per-rank records, then M[i*] <- c*,
// TD <- TD + dTD*.  Runs as one thread; identical on every rank.
template <typename A>
__global__ void k_select(const Rec<A>* __restrict__ recs, int nrec, A* __restrict__ td, int* __restrict__ M,
                         int* __restrict__ point_slot, Decision<A>* __restrict__ dec, int* __restrict__ rescan_count) {
    *rescan_count = 0;
    Rec<A> b = rec_none<A>();
    for (int r = 0; r < nrec; ++r)
        if (rec_less(recs[r], b)) b = recs[r];
    bool improving;
    if (b.slot == INT_MAX) improving = false;
    else if (std::is_same<A, double>::value) improving = (double)b.v < -1e-12 * fabs((double)*td);
    else improving = b.v < 0;
    dec->iters += 1;
    dec->apply = improving ? 1 : 0;
    dec->dtd = b.v;
    dec->slot = b.slot;
    dec->c = b.c;
    if (improving) {
        const int old = M[b.slot];
        dec->old_m = old;
        M[b.slot] = b.c;
        point_slot[old] = -1;
        point_slot[b.c] = b.slot;
        *td += b.v;
        dec->swaps += 1;
    }
}

// ---------------------------------------------------------------------------
// FasterPAM (Alg.4; readings F1-F5): eager acceptance inside a
// speculative candidate batch.  cand_v/cand_slot hold (min_i dTD(m_i, x_c),
// argmin) of every candidate of the batch window, evaluated on the current
// state (k_swap_combine).  The scan visits the window's positions lo..hi-1
// in ascending order (F1); the first improving candidate (F5 / R5) is the
// one Alg.4 swaps, because every earlier one was evaluated on exactly the
// state the sequential scan would see and found non-improving.  Later
// candidates of the batch are discarded (the host resumes behind the swap).
// One block; also resets the rescan counter and counts a pass (F3).
// ---------------------------------------------------------------------------
template <typename A>
__global__ void k_fp3_pick(const A* __restrict__ cand_v, const int* __restrict__ cand_slot, int lo, int hi,
                           int64_t win_begin, A* __restrict__ td, int* __restrict__ M, int* __restrict__ point_slot,
                           Decision<A>* __restrict__ dec, int* __restrict__ rescan_count, int new_pass) {
    __shared__ int first;
    if (threadIdx.x == 0) first = INT_MAX;
    __syncthreads();
    const A tdv = *td;
    for (int j = lo + (int)threadIdx.x; j < hi; j += blockDim.x) {
        if (cand_slot[j] < 0) continue;                       // medoid column (F1 skip)
        const A v = cand_v[j];
        bool imp;
        if (std::is_same<A, double>::value) imp = (double)v < -1e-12 * fabs((double)tdv);
        else imp = v < 0;
        if (imp) { atomicMin(&first, j); break; }             // this thread's first = its minimum
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    *rescan_count = 0;
    if (new_pass) dec->iters += 1;
    if (first == INT_MAX) { dec->apply = 0; return; }
    const int slot = cand_slot[first];
    const int c = (int)(win_begin + first);
    const A v = cand_v[first];
    const int old = M[slot];
    dec->apply = 1;
    dec->dtd = v;
    dec->slot = slot;
    dec->c = c;
    dec->old_m = old;
    M[slot] = c;
    point_slot[old] = -1;
    point_slot[c] = slot;
    *td = tdv + v;
    dec->swaps += 1;
}

// ---------------------------------------------------------------------------
// a6: FastPAM2 (reading R6)
// ---------------------------------------------------------------------------

// Per slot i: (v_i, c_i) = lexicographic min over local non-medoid candidates
// of (dTD(m_i, x_c), c) with dTD = R_i + acc_c[i] + dTD^{+x_c}
// (Eq. eqn:better-change3).  Slots with an empty segment have acc_c[i] = 0.
// One block per slot; reads row i of the k x w acc matrix (coalesced).
// SB slots per block (grid (ceil(k / SB), FP2_SPLIT)): the candidate's
// point_slot and plus are loaded once for SB rows of acc (at C5, k = 500,
// SB = 1 re-read them once per slot: 600 MB of L2 traffic beside the 400 MB
// of acc).  Per slot the same (v, c) lexicographic minimum.
template <typename A, int SB = 1>
__global__ void k_fp2_slot_best(int w, int k, int64_t col_begin, const A* __restrict__ acc,
                                const A* __restrict__ plus, const A* __restrict__ R,
                                const int* __restrict__ seg_start, const int* __restrict__ point_slot,
                                Rec<A>* __restrict__ part) {
    // block (ib, y) scans columns [y*w/SPLIT, (y+1)*w/SPLIT) of rows ib*SB .. ib*SB + SB - 1
    const int i0 = blockIdx.x * SB, y = blockIdx.y;
    bool empty[SB];
    A ri[SB];
    const A* arow[SB];
#pragma unroll
    for (int q = 0; q < SB; ++q) {
        const int i = min(i0 + q, k - 1);
        empty[q] = seg_start[i] == seg_start[i + 1];
        ri[q] = R[i];
        arow[q] = acc + (int64_t)i * w;
    }
    const int a = (int)((int64_t)y * w / gridDim.y), z = (int)((int64_t)(y + 1) * w / gridDim.y);
    Rec<A> b[SB];
#pragma unroll
    for (int q = 0; q < SB; ++q) b[q] = rec_none<A>();
    constexpr int U = SB >= 4 ? 2 : 4;        // columns loaded ahead per thread (memory-level parallelism)
    for (int c0l = a + threadIdx.x; c0l < z; c0l += U * blockDim.x) {
        A av[U][SB], pv[U];
        int ps[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int cl = c0l + u * blockDim.x;
            if (cl < z) {
                ps[u] = point_slot[col_begin + cl];
                pv[u] = plus[cl];
#pragma unroll
                for (int q = 0; q < SB; ++q) av[u][q] = empty[q] ? (A)0 : __ldcs(&arow[q][cl]);   // read once: streaming
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int cl = c0l + u * blockDim.x;
            if (cl >= z || ps[u] >= 0) continue;
#pragma unroll
            for (int q = 0; q < SB; ++q) {
                Rec<A> r; r.v = ri[q] + av[u][q] + pv[u]; r.slot = i0 + q; r.c = (int)(col_begin + cl);
                if (rec_less(r, b[q])) b[q] = r;        // same slot: (v, c) order
            }
        }
    }
#pragma unroll
    for (int q = 0; q < SB; ++q) {
        const Rec<A> m = block_min_rec(b[q]);
        if (threadIdx.x == 0 && i0 + q < k) part[(int64_t)(i0 + q) * gridDim.y + y] = m;
        __syncthreads();                          // block_min_rec's shared buffer is reused
    }
}

// Per slot: lexicographic min over the FP2_SPLIT partials (fixed order).
template <typename A>
__global__ void k_fp2_slot_reduce(int k, int split, const Rec<A>* __restrict__ part, Rec<A>* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= k) return;
    Rec<A> b = rec_none<A>();
    for (int y = 0; y < split; ++y) {
        const Rec<A> r = part[(int64_t)i * split + y];
        if (rec_less(r, b)) b = r;
    }
    out[i] = b;
}

// FastPAM2 steps 4-5 on the device (reading R6): the improving slots of the
// per-slot bests, ordered by (v_i, i) -- the rank of slot i is the number of
// improving slots before it in that order (k <= a few thousand: one block).
// Also the iteration's decision bookkeeping (the sequential kernel counts
// this iteration's swaps from 0, then adds the previous total back).
// Queued FastPAM2 iterations (kmedoids_swap_iters_variant): an iteration
// that finds no improving slot sets the sticky Decision::done (it is counted,
// P:1390-1392); a plan kernel behind it plans nothing and counts nothing, the
// stream behind it returns at once, and the sequential kernel restores the
// running swap total as after any pass.
template <typename A>
__device__ __forceinline__ void fp2_plan_done(Decision<A>* dec, int* m_out, int* swaps_prev) {
    *m_out = 0;
    dec->apply = 0;
    *swaps_prev = dec->swaps;
    dec->swaps = 0;
}

template <typename A>
__global__ void k_fp2_plan(const Rec<A>* __restrict__ best, int k, const A* __restrict__ td,
                           Decision<A>* __restrict__ dec, int* __restrict__ order, int* __restrict__ m_out,
                           int* __restrict__ swaps_prev, bool staged_ok, int sticky) {
    __shared__ int s_m, s_done;
    extern __shared__ __align__(16) unsigned char plan_smem[];   // k values and flags (when they fit)
    if (threadIdx.x == 0) { s_m = 0; s_done = sticky ? dec->done : 0; }
    __syncthreads();
    if (s_done) {                              // queued behind a converged pass: a no-op (fp2_plan_done)
        if (threadIdx.x == 0) fp2_plan_done(dec, m_out, swaps_prev);
        return;
    }
    const A tdv = *td;
    auto improving = [&](const Rec<A>& b) {
        if (b.slot == INT_MAX) return false;
        if (std::is_same<A, double>::value) return (double)b.v < -1e-12 * fabs((double)tdv);
        return b.v < 0;
    };
    // stage (v_i, improving_i) in shared memory: the O(k^2) ranking reads them k times
    A* sv = reinterpret_cast<A*>(plan_smem);
    unsigned char* simp = plan_smem + (size_t)k * sizeof(A);
    const bool staged = staged_ok;
    if (staged)
        for (int i = threadIdx.x; i < k; i += blockDim.x) {
            const Rec<A> b = best[i];
            sv[i] = b.v;
            simp[i] = improving(b) ? 1 : 0;
        }
    __syncthreads();
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
        const Rec<A> bi = best[i];
        if (!improving(bi)) continue;
        int rank = 0;
        if (staged) {
            for (int j = 0; j < k; ++j) {
                const A vj = sv[j];
                if (j != i && simp[j] && (vj < bi.v || (vj == bi.v && j < i))) ++rank;
            }
        } else {
            for (int j = 0; j < k; ++j) {
                const Rec<A> bj = best[j];
                if (j != i && improving(bj) && (bj.v < bi.v || (bj.v == bi.v && j < i))) ++rank;
            }
        }
        order[rank] = i;
        atomicAdd(&s_m, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        *m_out = s_m;
        dec->iters += 1;
        dec->apply = 0;
        *swaps_prev = dec->swaps;
        dec->swaps = 0;
        if (sticky && s_m == 0) dec->done = 1;
    }
}


// FastPAM2 steps 4-5 for k <= FP2_SORT_MAX in one block, with the per-slot
// reduction folded in: per slot, the lexicographic min over the column
// splits (fixed order, as k_fp2_slot_reduce) -> best[i]; the improving slots
// keyed by (v_i, i) and the non-improving ones by a sentinel, sorted by a
// bitonic network in shared memory (the keys are distinct: the same order as
// k_fp2_plan's ranks); order[0..m) = the first m keys.
constexpr int FP2_SORT_MAX = 2048;     // keys in 24 KB of shared memory
template <typename A>
__global__ void __launch_bounds__(1024)
k_fp2_plan_sort(const Rec<A>* __restrict__ part, int split, Rec<A>* __restrict__ best, int k, int npow2,
                const A* __restrict__ td, Decision<A>* __restrict__ dec, int* __restrict__ order,
                int* __restrict__ m_out, int* __restrict__ swaps_prev, int sticky) {
    __shared__ int s_m, s_done;
    extern __shared__ __align__(16) unsigned char sort_smem[];
    A* kv = reinterpret_cast<A*>(sort_smem);
    int* ki = reinterpret_cast<int*>(sort_smem + (size_t)npow2 * sizeof(A));
    if (threadIdx.x == 0) { s_m = 0; s_done = sticky ? dec->done : 0; }
    __syncthreads();
    if (s_done) {
        if (threadIdx.x == 0) fp2_plan_done(dec, m_out, swaps_prev);
        return;
    }
    const A tdv = *td;
    for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
        A v = amax<A>();
        int key = INT_MAX;
        if (i < k) {
            Rec<A> b = rec_none<A>();
            constexpr int U = 8;                 // partials loaded ahead (one round trip for FP2_SPLIT = 8)
            for (int y0 = 0; y0 < split; y0 += U) {
                Rec<A> r[U];
#pragma unroll
                for (int u = 0; u < U; ++u) r[u] = y0 + u < split ? part[(int64_t)i * split + y0 + u] : rec_none<A>();
#pragma unroll
                for (int u = 0; u < U; ++u) if (rec_less(r[u], b)) b = r[u];
            }
            best[i] = b;
            bool imp;
            if (b.slot == INT_MAX) imp = false;
            else if (std::is_same<A, double>::value) imp = (double)b.v < -1e-12 * fabs((double)tdv);
            else imp = b.v < 0;
            if (imp) { v = b.v; key = i; atomicAdd(&s_m, 1); }
        }
        kv[i] = v;
        ki[i] = key;
    }
    __syncthreads();
    for (int size = 2; size <= npow2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < (npow2 >> 1); t += blockDim.x) {
                const int a = 2 * t - (t & (stride - 1)), b = a + stride;
                const bool up = (a & size) == 0;
                const A va = kv[a], vb = kv[b];
                const int ia = ki[a], ib = ki[b];
                const bool gt = va > vb || (va == vb && ia > ib);
                if (gt == up) { kv[a] = vb; kv[b] = va; ki[a] = ib; ki[b] = ia; }
            }
            __syncthreads();
        }
    }
    const int m = s_m;
    for (int r = threadIdx.x; r < m; r += blockDim.x) order[r] = ki[r];
    if (threadIdx.x == 0) {
        *m_out = m;
        dec->iters += 1;
        dec->apply = 0;
        *swaps_prev = dec->swaps;
        dec->swaps = 0;
        if (sticky && m == 0) dec->done = 1;
    }
}

// The sequential phase of one FastPAM2 iteration as ONE cooperative kernel.
// order[0..m) are the improving slots sorted by (v_i, i) (host), best[i] =
// (v_i, i, c_i).  r = 0 applies best[order[0]] as is (it is FastPAM1's swap).
// Every later slot i (in order): skipped if c_i became a medoid, else
// dTD(m_i, x_c_i) is recomputed on the current cache in one pass over the
// objects,
//    sum_o [nearest(o)=i](d_s - d_n) + [d<d_n](d - d_n)
//        + [nearest(o)=i]([d<d_n](d_n - d_s) + [d_n<=d<d_s](d - d_s)),
// and the swap is applied iff it still improves (reading R5).  Applying =
// M[i] <- c, TD += dTD, MC[i] <- column c, incremental nearest/second update
// (+ warp rescans of the objects whose nearest/second was slot i).
//
// Speculative batches: the state changes only when a swap is applied (a few
// per iteration, while m is up to k), so the next FP2_B unskipped entries are
// re-evaluated TOGETHER on the current state in one pass over the objects
// (their columns land in cols[b][o]); the first improving entry of the batch
// is exactly the one the sequential loop applies next (every earlier entry
// was evaluated on the same state and rejected).  It is applied; entries
// after it were evaluated on a stale state and start the next batch.  Two
// grid syncs per batch (plus two per applied swap) instead of two per entry.
// Applied swaps are appended to trace[] (slot, c, dTD).
constexpr int FP2_B = 32;

// The next batch of the sequential phase, formed by one warp: plan entries q,
// q+1, ... in order, skipping those whose candidate became a medoid (and,
// owner-side rounds, colidx != null, those owned by another rank), until
// FP2_B are taken or q reaches m.  The 32 entries of a window are examined at
// once; q ends behind the last entry examined (entries skipped after the
// last one taken are consumed too: nothing changes the state within a batch).
template <typename A>
__device__ __forceinline__ void fp2_batch_window(const int* __restrict__ order, const Rec<A>* __restrict__ best,
                                                 const int* __restrict__ point_slot, const int* __restrict__ colidx,
                                                 int me, int maxcnt, int m, int lane, int& q, int& nb, int* s_r,
                                                 int* s_i, int* s_c, int* s_l) {
    while (q < m && nb < FP2_B) {
        const int qq = q + lane;
        bool ok = false;
        int i = 0, c = 0, l = 0;
        if (qq < m) {
            ok = true;
            if (colidx) {
                const int ci = colidx[qq];
                ok = ci / maxcnt == me;                  // another rank's candidate
                l = ci % maxcnt;
            }
            if (ok) {
                i = order[qq];
                c = best[i].c;
                ok = point_slot[c] < 0;                  // c became a medoid: skipped
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        const int nv = __popc(bal);
        const int take = min(nv, FP2_B - nb);
        const int rank = __popc(bal & ((1u << lane) - 1u));
        if (ok && rank < take) {
            s_r[nb + rank] = qq; s_i[nb + rank] = i; s_c[nb + rank] = c;
            if (s_l) s_l[nb + rank] = l;
        }
        q = take < nv ? q + (int)__fns(bal, 0, take) + 1 : q + 32;
        nb += take;
    }
    q = min(q, m);
}

// pinned host destinations of one FastPAM2 iteration's outcome (single-GPU
// device-plan path; null pointers elsewhere): written by block 0 at the end
// of k_fp2_sequential instead of four device-to-host copies after it
template <typename A>
struct F2HostOut {
    Decision<A>* dec;
    A* td;
    int* swaps;          // this iteration's swaps
    Rec<A>* trace;       // its first min(swaps, trace_cap) records
};

template <typename T, typename A>
__global__ void __launch_bounds__(256)
k_fp2_sequential(const T* __restrict__ D, int64_t ld, const T* __restrict__ colsrc, const int* __restrict__ colidx,
                 int n, int k, const int* __restrict__ order, const int* __restrict__ m_dev,
                 const Rec<A>* __restrict__ best, int* __restrict__ M, int* __restrict__ point_slot,
                 T* __restrict__ MC, int* __restrict__ near, int* __restrict__ sec, T* __restrict__ dn,
                 T* __restrict__ ds, T* __restrict__ cols, A* __restrict__ td, A* __restrict__ partials,
                 Decision<A>* __restrict__ dec, Rec<A>* __restrict__ trace, int trace_cap,
                 int* __restrict__ rescan, int* __restrict__ rescan_count, int sym, int* __restrict__ swaps_iter,
                 const int* __restrict__ swaps_prev, F2HostOut<A> hout) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ A sred[8][FP2_B];
    __shared__ int s_r[FP2_B], s_c[FP2_B], s_i[FP2_B];
    __shared__ int s_nb, s_next, s_pick;
    __shared__ A s_v;
    const int nth = gridDim.x * blockDim.x;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int gwarp = tid >> 5, nwarps = nth >> 5;
    const int m = *m_dev;
    int r = 0, round = 0;
    while (r < m) {
        // ---- batch (every block identically: the state is the same everywhere);
        // the barrier keeps thread 0 from overwriting the shared batch / pick
        // values before every thread of the block has read the last ones
        __syncthreads();
        if (wib == 0) {
            // warp 0 forms the batch, 32 plan entries per window (their loads
            // in parallel; round 1: thread 0 walked the entries one dependent
            // load chain at a time, ~1 us per entry)
            int nb = 0, q = r;
            if (r == 0) {                            // FastPAM1's swap, applied as is
                if (lane == 0) { s_r[0] = 0; s_i[0] = order[0]; s_c[0] = best[order[0]].c; }
                nb = 1; q = 1;
            } else {
                fp2_batch_window(order, best, point_slot, nullptr, 0, 1, m, lane, q, nb, s_r, s_i, s_c, nullptr);
            }
            if (lane == 0) { s_nb = nb; s_next = q; }
        }
        __syncthreads();
        const int nb = s_nb;
        if (nb == 0) break;                          // (uniform across blocks)
        const A tdv = __ldcg(td);
        if (tid == 0) *rescan_count = 0;             // the last rescan list was consumed before a grid sync
        // ---- phase 1: columns of the batch, partial re-evaluations
        A part[FP2_B];
#pragma unroll
        for (int b = 0; b < FP2_B; ++b) part[b] = 0;
        for (int o = tid; o < n; o += nth) {
            const T a = dn[o], bb = ds[o];
            const int no = near[o];
#pragma unroll
            for (int b = 0; b < FP2_B; ++b) {
                if (b >= nb) continue;               // (fully unrolled: part[] stays in registers)
                // column c of the batch: the gathered copy (sharded), row c when D is
                // declared symmetric (coalesced: 4n bytes instead of n sectors), else
                // the strided column
                const T x = colsrc ? colsrc[(int64_t)colidx[s_r[b]] * n + o]
                                   : sym ? D[(int64_t)s_c[b] * ld + o] : D[(int64_t)o * ld + s_c[b]];
                cols[(int64_t)b * n + o] = x;
                if (r > 0) {
                    A f = 0;
                    if (x < a) f += (A)x - (A)a;
                    if (no == s_i[b]) {
                        f += (A)bb - (A)a;
                        if (x < a) f += (A)a - (A)bb;
                        else if (x < bb) f += (A)x - (A)bb;
                    }
                    part[b] += f;
                }
            }
        }
        A* pbuf = partials + (size_t)(round & 1) * gridDim.x * FP2_B;   // double-buffered across batches
        if (r > 0) {
#pragma unroll
            for (int b = 0; b < FP2_B; ++b) {
                if (b >= nb) continue;
                A t = part[b];
#pragma unroll
                for (int x = 16; x >= 1; x >>= 1) t += __shfl_xor_sync(FULL, t, x);
                if (lane == 0) sred[wib][b] = t;
            }
            __syncthreads();
            if (threadIdx.x < FP2_B && threadIdx.x < nb) {
                A t = 0;
                for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sred[w][threadIdx.x];
                pbuf[(size_t)blockIdx.x * FP2_B + threadIdx.x] = t;
            }
        }
        grid.sync();
        // ---- phase 2: every block reduces the partials in the same order (warp
        // w: entries b = w, w+8, ...; strided loads + xor butterfly, identical
        // bits everywhere) and picks the first improving entry
        if (r == 0) {
            if (threadIdx.x == 0) { s_pick = 0; s_v = best[s_i[0]].v; }
        } else {
            for (int b = wib; b < nb; b += (int)(blockDim.x >> 5)) {
                A t = 0;
                for (int q = lane; q < (int)gridDim.x; q += 32) t += __ldcg(&pbuf[(size_t)q * FP2_B + b]);
#pragma unroll
                for (int x = 16; x >= 1; x >>= 1) t += __shfl_xor_sync(FULL, t, x);
                if (lane == 0) sred[0][b] = t;       // sred rows are free again
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                int pick = -1;
                for (int b = 0; b < nb && pick < 0; ++b) {
                    const A v = sred[0][b];
                    bool ok;
                    if (std::is_same<A, double>::value) ok = (double)v < -1e-12 * fabs((double)tdv);
                    else ok = v < 0;
                    if (ok) { pick = b; s_v = v; }
                }
                s_pick = pick;
            }
        }
        __syncthreads();
        const int pick = s_pick;
        if (pick < 0) {                              // no entry of the batch improves
            r = s_next;
            ++round;
            continue;
        }
        const int i = s_i[pick], c = s_c[pick];
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            const A v = s_v;
            const int old = M[i];
            M[i] = c;
            point_slot[old] = -1;
            point_slot[c] = i;
            *td = tdv + v;
            const int sw = dec->swaps;
            if (sw < trace_cap) { Rec<A> t; t.v = v; t.slot = i; t.c = c; trace[sw] = t; }
            dec->swaps = sw + 1;
            dec->apply = 1;
            dec->slot = i;
            dec->c = c;
            dec->dtd = v;
            dec->old_m = old;
        }
        // ---- phase 3: MC[i] <- column c, incremental nearest/second update;
        // objects whose nearest/second was slot i are listed for a rescan
        const T* colp = cols + (int64_t)pick * n;
        for (int o = tid; o < n; o += nth) {
            const T x = colp[o];
            MC[(int64_t)i * n + o] = x;
            const int j1 = near[o], j2 = sec[o];
            if (j1 == i || j2 == i) {
                rescan[atomicAdd(rescan_count, 1)] = o;
            } else {
                const T d1 = dn[o], d2 = ds[o];
                if (x < d1 || (x == d1 && i < j1)) { near[o] = i; dn[o] = x; sec[o] = j1; ds[o] = d1; }
                else if (x < d2 || (x == d2 && i < j2)) { sec[o] = i; ds[o] = x; }
            }
        }
        grid.sync();
        // ---- phase 4: (d, j) lexicographic top-2 of the listed objects, one warp
        // each (lanes over the slots; as k_assign_rescan)
        const int cnt = __ldcg(rescan_count);
        for (int e = gwarp; e < cnt; e += nwarps) {
            const int o = __ldcg(&rescan[e]);
            T d1 = dmax<T>(), d2 = dmax<T>();
            int j1 = INT_MAX, j2 = INT_MAX;
#pragma unroll 8
            for (int j = lane; j < k; j += 32) {
                const T d = __ldcg(&MC[(int64_t)j * n + o]);
                if (lex_lt(d, j, d1, j1)) { d2 = d1; j2 = j1; d1 = d; j1 = j; }
                else if (lex_lt(d, j, d2, j2)) { d2 = d; j2 = j; }
            }
#pragma unroll
            for (int x = 16; x >= 1; x >>= 1) {
                const T e1 = __shfl_xor_sync(FULL, d1, x), e2 = __shfl_xor_sync(FULL, d2, x);
                const int f1 = __shfl_xor_sync(FULL, j1, x), f2 = __shfl_xor_sync(FULL, j2, x);
                if (lex_lt(e1, f1, d1, j1)) {
                    if (lex_lt(d1, j1, e2, f2)) { d2 = d1; j2 = j1; } else { d2 = e2; j2 = f2; }
                    d1 = e1; j1 = f1;
                } else if (lex_lt(e1, f1, d2, j2)) {
                    d2 = e1; j2 = f1;
                }
            }
            if (lane == 0) { near[o] = j1; sec[o] = j2; dn[o] = d1; ds[o] = d2; }
        }
        grid.sync();
        r = s_r[pick] + 1;
        ++round;
    }
    // this iteration's swaps (counted from 0) and, device-plan path, the
    // running total restored (block 0 / thread 0 is dec's only writer)
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const int sw = dec->swaps;
        *swaps_iter = sw;
        if (swaps_prev) dec->swaps = sw + *swaps_prev;
        if (hout.dec) {
            *hout.dec = *dec;
            *hout.td = *td;
            *hout.swaps = sw;
        }
    }
    if (hout.trace && blockIdx.x == 0) {
        __syncthreads();                         // the trace records were written by thread 0
        const int cnt = min(*swaps_iter, trace_cap);
        for (int t = threadIdx.x; t < cnt; t += blockDim.x) hout.trace[t] = trace[t];
    }
}

// ---------------------------------------------------------------------------
// a7: BUILD (Alg.1)
// ---------------------------------------------------------------------------
// MODE 0 (first medoid):  acc_c = sum_o d(x_o, x_c)
// MODE 1 (later medoids): acc_c = sum_o min(d(x_o, x_c) - d_n(o), 0)
// (medoid rows have d_n = 0 and contribute 0 since D >= 0; the x_o = x_c row
// contributes -d_n(c): reading R3).
// The producer / ring of the SWAP stream with rows in natural order; per
// stage the consumers
// fold "d < d_n" over the 4 rows x 4 columns into a REDUX.OR mask and
// update only the columns with a hit (MODE 1), or sum every element with a
// 4-row tree (MODE 0).  3 CTAs x 8 warps per SM.
template <typename T, typename A, int NC, int RB, int S, int MINB, int MODE>
__global__ void __launch_bounds__((NC + 1) * 32, MINB)
k_build_tma(const T* __restrict__ D, int64_t ld, int w, int wpad, int n, int P, const T* __restrict__ dnear,
            A* __restrict__ out) {
    using C = SegCfg<T, NC, RB, S>;
    using V = typename Vec4<T>::type;
    extern __shared__ __align__(128) unsigned char smem[];
    T* sdata = reinterpret_cast<T*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::DATAB);
    uint64_t* empty = full + S;
    const int q = blockIdx.y;
    const int64_t p0 = part_lo(q, n, P), p1 = part_lo(q + 1, n, P);
    const int nstages = (int)((p1 - p0 + RB - 1) / RB);
    const int ctacol = blockIdx.x * C::COLS;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int st = 0; st < S; ++st) {
            ptx::mbar_init(&full[st], 1);
            ptx::mbar_init(&empty[st], NC);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    if (warp == NC) {
        const uint32_t cbytes = (uint32_t)min(C::COLS, wpad - ctacol) * (uint32_t)sizeof(T);
        const uint64_t pol = ptx::policy_evict_first();
        for (int st = 0; st < nstages; ++st) {
            const int s = st % S;
            if (st >= S) ptx::mbar_wait(&empty[s], ((st / S) & 1) ^ 1);
            const int64_t pr = p0 + (int64_t)st * RB;
            const int nb = (int)min((int64_t)RB, p1 - pr);
            if (lane == 0) ptx::mbar_expect_tx(&full[s], (uint32_t)nb * cbytes);
            __syncwarp();
            if (lane < nb)
                ptx::bulk_g2s(sdata + (size_t)(s * RB + lane) * C::COLS, D + (pr + lane) * ld + ctacol, cbytes,
                              &full[s], pol);
        }
        return;
    }
    const int cb = ctacol + warp * 128 + lane * 4;
    const bool active = cb < w;
    A acc[4] = {0, 0, 0, 0};
    for (int st = 0; st < nstages; ++st) {
        const int s = st % S;
        const int64_t pr = p0 + (int64_t)st * RB;
        const int nb = (int)min((int64_t)RB, p1 - pr);
        T dv[RB];
#pragma unroll
        for (int u = 0; u < RB; ++u)        // d_nearest of the stage's rows (uniform loads, L1)
            dv[u] = (MODE == 1 && u < nb) ? dnear[pr + u] : never_lt<T>();
        ptx::mbar_wait(&full[s], (st / S) & 1);
        T x[RB][4];
        const T* srow = sdata + (size_t)(s * RB) * C::COLS + (warp * 128 + lane * 4);
#pragma unroll
        for (int u = 0; u < RB; ++u) {
            const V v = *reinterpret_cast<const V*>(srow + (size_t)u * C::COLS);
            memcpy(&x[u][0], &v.x, sizeof(T)); memcpy(&x[u][1], &v.y, sizeof(T));
            memcpy(&x[u][2], &v.z, sizeof(T)); memcpy(&x[u][3], &v.w, sizeof(T));
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&empty[s]);
        if (MODE == 0) {
            if (!active) continue;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                A t[RB];
#pragma unroll
                for (int u = 0; u < RB; ++u) t[u] = (u < nb) ? (A)x[u][j] : (A)0;
                acc[j] += (t[0] + t[1]) + (t[2] + t[3]);
            }
        } else {
#pragma unroll
            for (int u = 0; u < RB; ++u) dv[u] = active ? dv[u] : never_lt<T>();
            static_assert(RB == 4, "mask folding assumes 4 rows per stage");
            unsigned m = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                m |= CmpLt<T>::any4(x[0][j], dv[0], x[1][j], dv[1], x[2][j], dv[2], x[3][j], dv[3]) << j;
            const unsigned wm = __reduce_or_sync(FULL, m);
            if (wm == 0) continue;
            A dA[RB];
#pragma unroll
            for (int u = 0; u < RB; ++u) dA[u] = (A)dv[u];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (wm & (1u << j)) {
                    A t[RB];
#pragma unroll
                    for (int u = 0; u < RB; ++u) t[u] = (x[u][j] < dv[u]) ? (A)x[u][j] - dA[u] : (A)0;
                    acc[j] += (t[0] + t[1]) + (t[2] + t[3]);
                }
            }
        }
    }
    if (!active) return;
    const int64_t base = (int64_t)q * w;
    const uint64_t keep = ptx::policy_evict_last();   // read by the gain combine right after
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (cb + j < w) ptx::st_hint(&out[base + cb + j], acc[j], keep);
}

// Per candidate: sum the parts in order; MODE 0 removes the x_o = x_c term
// (Alg.1 P:288 "x_o != x_c"); non-medoids enter a (value, c) min (slot = 0).
template <typename T, typename A, int MODE>
__global__ void k_build_combine(const T* __restrict__ D, int64_t ld, int w, int64_t col_begin, int P,
                                const A* __restrict__ in, const int* __restrict__ point_slot,
                                Rec<A>* partials, unsigned* counter, Rec<A>* out) {
    const int cl = blockIdx.x * blockDim.x + threadIdx.x;
    Rec<A> best = rec_none<A>();
    if (cl < w) {
        const int64_t c = col_begin + cl;
        A s = 0;
        for (int q = 0; q < P; ++q) s += in[(int64_t)q * w + cl];
        if (MODE == 0) s -= (A)D[c * ld + cl];
        if (point_slot[c] < 0) { best.v = s; best.slot = 0; best.c = (int)c; }
    }
    grid_min_rec(best, partials, counter, out);
}

// BUILD step bookkeeping: slot `step` <- c*, TD <- value (step
// 0) or TD + dTD* (later steps).
template <typename A>
__device__ __forceinline__ void build_take(const Rec<A>& b, int step, A* __restrict__ td, int* __restrict__ M,
                                           int* __restrict__ point_slot, Decision<A>* __restrict__ dec) {
    dec->apply = 1;
    dec->dtd = b.v;
    dec->slot = step;
    dec->c = b.c;
    dec->old_m = -1;
    M[step] = b.c;
    point_slot[b.c] = step;
    if (step == 0) *td = b.v; else *td += b.v;
}
template <typename A>
__global__ void k_build_select(const Rec<A>* __restrict__ recs, int nrec, int step, A* __restrict__ td,
                               int* __restrict__ M, int* __restrict__ point_slot, Decision<A>* __restrict__ dec) {
    Rec<A> b = rec_none<A>();
    for (int r = 0; r < nrec; ++r)
        if (rec_less(recs[r], b)) b = recs[r];
    build_take(b, step, td, M, point_slot, dec);
}

// d_nearest update (P:295-298 for step 0, P:313-316 later): medoids get 0.
template <typename T, typename A>
__global__ void k_build_dn(const T* __restrict__ MC, int n, const Decision<A>* __restrict__ dec,
                           const int* __restrict__ point_slot, T* __restrict__ dn) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= n) return;
    const int step = dec->slot;
    const T x = MC[(int64_t)step * n + o];
    if (point_slot[o] >= 0) dn[o] = 0;
    else if (step == 0 || x < dn[o]) dn[o] = x;
}

}  // namespace km
