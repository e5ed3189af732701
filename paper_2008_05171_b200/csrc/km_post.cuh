// km_post.cuh -- everything of a FastPAM1 iteration after the stream, in ONE
// cooperative kernel (SURVEY 8(a) rows a4 (accept), a5 (apply + cache
// update) and a2 (slot sort, removal loss) for the NEXT iteration).
//
// The launch list of the default bench (profiles/r1d_launches_summary.md)
// shows the non-stream part of a C4 step as ten small kernels (select,
// column gather, incremental update, rescan, histogram, two scans, scatter,
// removal loss, part metadata), each latency-bound, plus a launch gap each.
// Here they are phases of one kernel separated by grid syncs (~1.2 us each,
// measured; 4 of them when a swap is applied), with the same arithmetic and
// the same deterministic orders:
//   0 select    lexicographic min of the gathered records, acceptance R5
//               (every block; block 0 records M / point_slot / TD / dec after
//               the next sync that follows phase 0)     -- as k_select
//   1 apply     MC[i*] <- column c*; incremental nearest/second for the
//               block's chunk of objects and its histogram of the new
//               nearest slots; objects whose nearest/second was slot i* listed
//   2 rescan    warp per listed object, (d, slot) top-2, added to its chunk's
//               histogram                                -- as k_assign_rescan
//   3 histogram per block chunk (only without a swap / prep only)
//   4 scan      warp per slot over its chunk counts; slot totals
//   5 scan      every block: exclusive scan of the totals -> segment starts
//   6 scatter   stable (slot, o) order, warp-ranked        -- as k_slot_scatter
//   7 R, parts  removal loss per slot (fixed tree), empty slot, part heads/tails
#pragma once
#include "km_kernels.cuh"

namespace km {

constexpr int POST_THREADS = 256;
constexpr int POST_MAX_BLOCKS = 768;                  // chunk counts per slot scanned in registers
constexpr int POST_MAX_PER = POST_MAX_BLOCKS / 32;

template <typename T, typename A>
struct PostArgs {
    const T* D;
    int64_t ld;
    int n, k;
    int64_t c0, c1;          // local column range of the slab
    const Rec<A>* recs;      // per-rank best records (single GPU: 1)
    int nrec;
    A* td;
    int* M;
    int* point_slot;
    Decision<A>* dec;
    T* MC;
    int *near, *sec;
    T *dn, *ds;
    int* rescan;
    int* rescan_count;       // 0 on entry; reset to 0 on exit
    int* counts;             // [k][gridDim]
    int* offsets;            // [k][gridDim]
    int* slot_tot;           // [k]
    int* seg_start;          // [k+1]
    int* empty_slot;
    RowInfo<T>* ri;
    double2* rowd;           // float path: widened thresholds, sorted order (may be null)
    A* R;
    int P;
    int *head_slot, *tail_slot;
    int prep_only;             // 1: phases 3-7 only (slot sort, R, parts of the current cache)
    Decision<A>* h_dec;        // pinned host mirrors written at the end (or null)
    A* h_td;
    unsigned long long* tph;   // measurement aid (KM_STEP_PROF): globaltimer after each phase, or null
};

__device__ __forceinline__ void post_stamp(unsigned long long* tph, int i) {
    if (tph && blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        tph[i] = t;
    }
}

template <typename T>
__device__ __forceinline__ RowInfo<T> post_ld_ri(const RowInfo<T>* p) {
    const int4 v = __ldcg(reinterpret_cast<const int4*>(p));
    RowInfo<T> r;
    memcpy(&r, &v, sizeof(r));
    return r;
}

template <typename T, typename A>
__global__ void __launch_bounds__(POST_THREADS)
k_fp1_post(PostArgs<T, A> g) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ int post_smem[];           // k ints: histogram / scatter cursors
    __shared__ Decision<A> sdec;
    const int lane = threadIdx.x & 31;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    const int gwarp = tid >> 5, nwarps = nth >> 5;
    const int n = g.n, k = g.k, B = gridDim.x, b = blockIdx.x;
    post_stamp(g.tph, 0);

    Decision<A> d{};
    // block b owns the objects [ob0, ob1) in the apply and histogram phases
    const int ochunk = (n + B - 1) / B;
    const int ob0 = min(n, b * ochunk), ob1 = min(n, ob0 + ochunk);
    bool counted = false;
    if (!g.prep_only) {
        // ---- 0 select (every block decides identically; block 0 records)
        if (threadIdx.x == 0) {
            Rec<A> best = rec_none<A>();
            for (int r = 0; r < g.nrec; ++r) {
                const Rec<A> x = g.recs[r];
                if (rec_less(x, best)) best = x;
            }
            const A tdv = *g.td;
            bool improving;
            if (best.slot == INT_MAX) improving = false;
            else if (std::is_same<A, double>::value) improving = (double)best.v < -1e-12 * fabs((double)tdv);
            else improving = best.v < 0;
            Decision<A> d = *g.dec;
            d.iters += 1;
            d.apply = improving ? 1 : 0;
            d.dtd = best.v;
            d.slot = best.slot;
            d.c = best.c;
            if (improving) {
                d.old_m = g.M[best.slot];
                d.swaps += 1;
            }
            sdec = d;
        }
        __syncthreads();
        d = sdec;
        post_stamp(g.tph, 1);
        // (block 0 records the decision in M / point_slot / TD / dec after
        // the histogram's grid sync, when every block has read them; phases
        // 1-3 do not read them)

        // ---- 1 apply: column c*, incremental nearest/second, over the block's
        // chunk of objects; the chunk's histogram of the new nearest slots is
        // counted on the way (the rescanned objects are added in phase 2)
        if (d.apply) {
            const int i = d.slot;
            const bool local = d.c >= g.c0 && d.c < g.c1;
            int* hh = post_smem;
            for (int s = threadIdx.x; s < k; s += blockDim.x) hh[s] = 0;
            __syncthreads();
            for (int o = ob0 + threadIdx.x; o < ob1; o += blockDim.x) {
                if (local) g.MC[(int64_t)i * n + o] = g.D[(int64_t)o * g.ld + (d.c - g.c0)];
            }
            // (the column is read back below by the same thread: same o mapping)
            for (int o = ob0 + threadIdx.x; o < ob1; o += blockDim.x) {
                const int j1 = __ldcg(&g.near[o]), j2 = __ldcg(&g.sec[o]);
                if (j1 == i || j2 == i) {
                    g.rescan[atomicAdd(g.rescan_count, 1)] = o;
                    continue;
                }
                const T x = g.MC[(int64_t)i * n + o];
                const T d1 = __ldcg(&g.dn[o]), d2 = __ldcg(&g.ds[o]);
                if (x < d1 || (x == d1 && i < j1)) {
                    g.near[o] = i; g.dn[o] = x; g.sec[o] = j1; g.ds[o] = d1;
                    atomicAdd(&hh[i], 1);
                } else {
                    if (x < d2 || (x == d2 && i < j2)) { g.sec[o] = i; g.ds[o] = x; }
                    atomicAdd(&hh[j1], 1);
                }
            }
            __syncthreads();
            for (int s = threadIdx.x; s < k; s += blockDim.x) g.counts[(int64_t)s * B + b] = hh[s];
            grid.sync(); post_stamp(g.tph, 2);
            // ---- 2 rescan
            const int cnt = __ldcg(g.rescan_count);
            for (int e = gwarp; e < cnt; e += nwarps) {
                const int o = __ldcg(&g.rescan[e]);
                T d1 = dmax<T>(), d2 = dmax<T>();
                int j1 = INT_MAX, j2 = INT_MAX;
    #pragma unroll 8
                for (int j = lane; j < k; j += 32) {
                    const T dd = __ldcg(&g.MC[(int64_t)j * n + o]);
                    if (lex_lt(dd, j, d1, j1)) { d2 = d1; j2 = j1; d1 = dd; j1 = j; }
                    else if (lex_lt(dd, j, d2, j2)) { d2 = dd; j2 = j; }
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
                if (lane == 0) {
                    g.near[o] = j1; g.sec[o] = j2; g.dn[o] = d1; g.ds[o] = d2;
                    atomicAdd(&g.counts[(int64_t)j1 * B + o / ochunk], 1);   // the owner chunk's histogram
                }
            }
            grid.sync(); post_stamp(g.tph, 3);
            counted = true;
        }

    }
    // ---- 3 histogram of the block's chunk (when no swap was applied, or
    // prep only; otherwise counted in phases 1-2)
    const int e0 = ob0, e1 = ob1;
    if (!counted) {
        int* h = post_smem;
        for (int s = threadIdx.x; s < k; s += blockDim.x) h[s] = 0;
        __syncthreads();
        for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) atomicAdd(&h[__ldcg(&g.near[e])], 1);
        __syncthreads();
        for (int s = threadIdx.x; s < k; s += blockDim.x) g.counts[(int64_t)s * B + b] = h[s];
        grid.sync(); post_stamp(g.tph, 4);
    }
    if (!g.prep_only && b == 0 && threadIdx.x == 0) {
        *g.dec = d;
        if (d.apply) {
            g.M[d.slot] = d.c;
            g.point_slot[d.old_m] = -1;
            g.point_slot[d.c] = d.slot;
            *g.td = *g.td + d.dtd;
        }
    }

    // ---- 4 within-slot exclusive scan over the chunks, warp per slot: all
    // B counts of the slot loaded first (coalesced, one memory round trip),
    // then B/32 register-only warp scans
    for (int s = gwarp; s < k; s += nwarps) {
        const int* cs = g.counts + (int64_t)s * B;
        int cv[POST_MAX_PER];
#pragma unroll
        for (int i = 0; i < POST_MAX_PER; ++i) {
            const int bb = i * 32 + lane;
            cv[i] = bb < B ? __ldcg(&cs[bb]) : 0;
        }
        int run = 0;
        int* os = g.offsets + (int64_t)s * B;
#pragma unroll
        for (int i = 0; i < POST_MAX_PER; ++i) {
            if (i * 32 >= B) break;
            int incl = cv[i];
#pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
                const int y = __shfl_up_sync(FULL, incl, dd);
                if (lane >= dd) incl += y;
            }
            const int bb = i * 32 + lane;
            if (bb < B) os[bb] = run + incl - cv[i];
            run += __shfl_sync(FULL, incl, 31);
        }
        if (lane == 0) g.slot_tot[s] = run;
    }
    grid.sync(); post_stamp(g.tph, 5);

    // ---- 5 exclusive scan of the slot totals, by EVERY block into its shared
    // memory (no grid sync: the scatter below reads the block's own copy);
    // block 0 also writes seg_start[] for the removal loss and the stream
    {
        __shared__ int wsum[POST_THREADS / 32];
        int* segs = post_smem;                   // k ints: seg_start, then the scatter cursors
        const int per = (k + blockDim.x - 1) / blockDim.x;
        const int a = threadIdx.x * per, z = min(k, a + per);
        int sum = 0;
        for (int i = a; i < z; ++i) sum += __ldcg(&g.slot_tot[i]);
        int incl = sum;
#pragma unroll
        for (int dd = 1; dd < 32; dd <<= 1) {
            const int y = __shfl_up_sync(FULL, incl, dd);
            if (lane >= dd) incl += y;
        }
        if (lane == 31) wsum[threadIdx.x >> 5] = incl;
        __syncthreads();
        int base = 0;
        for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) base += wsum[w];
        int run = base + incl - sum;
        for (int i = a; i < z; ++i) {
            segs[i] = run;
            if (b == 0) g.seg_start[i] = run;
            run += __ldcg(&g.slot_tot[i]);
        }
        if (b == 0 && threadIdx.x == blockDim.x - 1) g.seg_start[k] = run;
        if (b == 0 && threadIdx.x == 0) *g.empty_slot = INT_MAX;
        __syncthreads();
    }
    post_stamp(g.tph, 6);

    // ---- 6 stable scatter into (slot, o) order: warp 0 of each block
    if (threadIdx.x < 32) {
        int* cur = post_smem;                    // seg_start of this block's copy + its chunk offsets
        for (int s = lane; s < k; s += 32) cur[s] += __ldcg(&g.offsets[(int64_t)s * B + b]);
        __syncwarp();
        const unsigned lt = (1u << lane) - 1u;
        for (int base = e0; base < e1; base += 32) {
            const int e = base + lane;
            const bool valid = e < e1;
            const int s = valid ? __ldcg(&g.near[e]) : -1 - lane;
            const unsigned peers = __match_any_sync(FULL, s);
            const int rank = __popc(peers & lt);
            const int leader = __ffs(peers) - 1;
            int bp = 0;
            if (valid && lane == leader) bp = cur[s];
            bp = __shfl_sync(FULL, bp, leader);
            __syncwarp();
            if (valid && lane == leader) cur[s] = bp + __popc(peers);
            __syncwarp();
            if (valid) {
                RowInfo<T> r;
                r.o = e; r.slot = s; r.dn = __ldcg(&g.dn[e]); r.ds = __ldcg(&g.ds[e]);
                const int pos = bp + rank;
                g.ri[pos] = r;
                if (g.rowd) g.rowd[pos] = make_double2((double)r.dn, (double)r.ds);
            }
        }
    }
    grid.sync(); post_stamp(g.tph, 7);

    // ---- 7 removal loss (warp per slot, fixed tree) and part metadata
    for (int s = gwarp; s < k; s += nwarps) {
        const int a = __ldcg(&g.seg_start[s]), z = __ldcg(&g.seg_start[s + 1]);
        A sum = 0;
        for (int p = a + lane; p < z; p += 32) {
            const RowInfo<T> r = post_ld_ri(&g.ri[p]);
            sum += (A)r.ds - (A)r.dn;
        }
#pragma unroll
        for (int x = 16; x >= 1; x >>= 1) sum += __shfl_xor_sync(FULL, sum, x);
        if (lane == 0) {
            g.R[s] = sum;
            if (a == z) atomicMin(g.empty_slot, s);
        }
    }
    for (int q = tid; q < g.P; q += nth) {
        const int64_t p0 = part_lo(q, n, g.P), p1 = part_lo(q + 1, n, g.P);
        g.head_slot[q] = post_ld_ri(&g.ri[p0]).slot;
        g.tail_slot[q] = post_ld_ri(&g.ri[p1 - 1]).slot;
    }
    if (b == 0 && threadIdx.x == 0) {
        *g.rescan_count = 0;
        // the decision and TD straight into pinned host memory (visible to the
        // host once the stream is synchronised): no copy nodes after the kernel
        if (g.h_dec) {
            *g.h_dec = d;
            *g.h_td = *g.td;
        }
    }
    post_stamp(g.tph, 8);
}

}  // namespace km
