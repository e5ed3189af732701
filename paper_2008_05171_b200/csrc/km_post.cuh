// km_post.cuh -- everything of a FastPAM1 iteration after the stream, in ONE
// cooperative kernel (SURVEY 8(a) rows a4 (accept), a5 (apply + cache
// update) and a2 (slot sort, removal loss) for the NEXT iteration).
//
// Block b owns the objects of one contiguous chunk [ob0, ob1).  Three phases
// separated by TWO grid syncs:
//   A  select   lexicographic min of the gathered records, acceptance R5
//               (every block decides identically)           -- Alg.3
//      apply    MC[i*] <- column c* for the chunk; incremental nearest /
//               second (O(1) per object); the chunk's objects
//               whose nearest or second was slot i* are rescanned by the
//               block's own warps (top-2 over the k medoid columns; the new
//               column of those objects was written by this block, so no
//               grid sync is needed); the result equals a from-scratch
//               assignment (reading R2)
//      count    per slot: the chunk's object count and its partial removal
//               loss sum (ds - dn) (int64: exact, float: fp64 in
//               object order within the chunk)
//   -- grid sync --
//   B  scan     warp per slot: exclusive scan of the chunk counts -> chunk
//               offsets, slot total; R_i = fixed-order tree over the chunk
//               partials; empty slot (block 0 records the decision: M,
//               point_slot, TD, dec)
//   -- grid sync --
//   C  scatter  every block scans the slot totals into its shared memory
//               (segment starts), places its chunk in stable (slot, o) order
//               (warp-ranked), and the part head / tail slots come from a
//               binary search of the segment starts (no pass over the rows).
// All orders are fixed: deterministic; exact on int64 (reading R9 for float).
// Round 1's version had four grid syncs (separate rescan, slot-scan and
// removal-loss phases) and a global rescan list.
#pragma once
#include "km_kernels.cuh"

namespace km {

constexpr int POST_THREADS = 256;
constexpr int POST_MAX_BLOCKS = 512;                  // chunk counts per slot scanned in registers (16 per lane)
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
    int* rescan;             // [n]: block b lists its rescans in [ob0, ob1)
    int* rescan_count;       // reset to 0 on exit (shared with the unfused kernels)
    int* counts;             // [k][gridDim]
    int* offsets;            // [k][gridDim]
    A* rpart;                // [k][gridDim] partial removal losses
    int* slot_tot;           // [k]
    int* seg_start;          // [k+1]
    int* empty_slot;
    RowInfo<T>* ri;
    double2* rowd;           // float path: widened thresholds, sorted order (may be null)
    A* R;
    int P;
    int *head_slot, *tail_slot;
    int prep_only;             // 1: phases count, B, C only (slot sort, R, parts of the current cache)
    int allow_reg;             // 0: always the chunk loops (KM_POST_REG=0, tests of chunks > POST_THREADS)
    int sym;                   // D declared exactly symmetric (single GPU): d(o, c*) read from row c*
    IterMirror<A>* h_ring;     // pinned host ring of iteration outcomes (or null)
    int ring;                  // its size
    int* seq;                  // device counter of FastPAM1 post launches (ring slot = seq % ring)
    unsigned long long* tph;   // measurement aid (KM_STEP_PROF): globaltimer after each phase, or null
    // phase 0 (fused combine, FastPAM1 single-handle path): the stream's part
    // outputs [P][w] are folded here instead of by k_swap_combine
    int fuse;                  // 1: run phase 0; recs/nrec are then ignored
    int w;                     // local columns
    int stage0;                // 1: R and the part slots staged in dynamic shared memory
    const A *pp_plus, *pp_head, *pp_tail, *pp_imin;
    const int* pp_islot;
    A* cand_v;                 // [w] dTD of the best swap per candidate (medoids: slot -1)
    int* cand_slot;
    Rec<A>* blk_recs;          // [gridDim] per-block best record
};

constexpr int POST_QU = 5;     // part outputs loaded ahead per lane in phase 0 (P <= 40: one batch per range)
constexpr int POST_RG = 4;     // phase-0 column groups per round (merged by warps 0..3 in parallel)

// Phase-0 range state of one lane (column) over a contiguous range of parts:
// the first segment piece (may continue the previous range), the open piece
// at the end (may continue into the next), the best completed segment / part
// interior minimum in between, and the partial dTD^{+x_c} sum.
template <typename A>
struct RangeState {
    A plus, hc, tc, bv;
    int hs, ts, bs, single;    // single: the whole range lies in one segment (hs == ts)
};

// dynamic shared memory of k_fp1_post: k ints (16-aligned) | k A | [k A | 2P ints]
// (phase-0 staging) | range states (16-aligned)
template <typename A>
__host__ __device__ inline size_t post_rs_offset(int k, int P, bool stage) {
    const size_t base = ((size_t)k * sizeof(int) + 15) / 16 * 16 + (size_t)k * sizeof(A);
    return (base + (stage ? (size_t)k * sizeof(A) + 2 * (size_t)P * sizeof(int) : 0) + 15) / 16 * 16;
}
template <typename A>
__host__ __device__ inline size_t post_rs_bytes() { return (size_t)POST_RG * (POST_THREADS / 32) * 32 * sizeof(RangeState<A>); }

__device__ __forceinline__ void post_stamp(unsigned long long* tph, int i) {
    if (tph && blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        tph[i] = t;
    }
}

// One iteration outcome into the pinned ring: the payload, a system-scope
// fence, then the sequence number (a host poller that sees seq == q reads a
// complete entry).
template <typename A>
__device__ __forceinline__ void ring_put(IterMirror<A>& m, const Decision<A>& d, A td, int q, int noop) {
    m.d = d;
    m.td = td;
    m.noop = noop;
    __threadfence_system();
    *reinterpret_cast<volatile int*>(&m.seq) = q;
}

template <typename T, typename A>
__global__ void __launch_bounds__(POST_THREADS, 3)
k_fp1_post(PostArgs<T, A> g) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    // dynamic shared memory: k ints (histogram, later segment starts /
    // scatter cursors) then k A's (partial removal losses), 16-byte aligned
    extern __shared__ __align__(16) unsigned char post_smem_raw[];
    int* hh = reinterpret_cast<int*>(post_smem_raw);
    A* pr = reinterpret_cast<A*>(post_smem_raw + (((size_t)g.k * sizeof(int) + 15) / 16) * 16);
    __shared__ Decision<A> sdec;
    __shared__ int s_nres;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    const int gwarp = tid >> 5, nwarps = nth >> 5;
    const int n = g.n, k = g.k, B = gridDim.x, b = blockIdx.x;
    post_stamp(g.tph, 0);

    Decision<A> d{};
    if (!g.prep_only) {
        // a previous pass converged (sticky): this queued iteration is a no-op
        // (the stream kernel returned at once); record the unchanged outcome.
        // Every block reads dec here, before block 0 may write it (after a
        // grid sync), so the exit is grid-uniform.
        if (__ldcg(&g.dec->done)) {
            if (b == 0 && threadIdx.x == 0) {
                Decision<A> dd = *g.dec;
                dd.apply = 0;
                const int q = *g.seq;
                if (g.h_ring) ring_put(g.h_ring[q % g.ring], dd, *g.td, q, 1);
                *g.seq = q + 1;
            }
            return;
        }
    }
    const int ochunk = (n + B - 1) / B;
    const int ob0 = min(n, b * ochunk), ob1 = min(n, ob0 + ochunk);
    for (int s = threadIdx.x; s < k; s += blockDim.x) { hh[s] = 0; pr[s] = 0; }
    if (threadIdx.x == 0) s_nres = 0;

    // chunks of at most POST_THREADS objects (n <= POST_THREADS * blocks:
    // every BASELINE config) keep one object per thread in registers; the
    // cache loads are issued before the decision is known
    const bool reg = g.allow_reg && ob1 - ob0 <= POST_THREADS;
    const int myo = ob0 + threadIdx.x;
    const bool have = reg && myo < ob1;
    int j1 = 0, j2 = 0;
    T d1 = 0, d2 = 0;
    if (have) { j1 = __ldcg(&g.near[myo]); j2 = __ldcg(&g.sec[myo]); d1 = __ldcg(&g.dn[myo]); d2 = __ldcg(&g.ds[myo]); }

    const bool fused = g.fuse && !g.prep_only;
    if (fused) {
        // ---- 0: combine (a4, Alg.3).  Column groups of 32 (lane =
        // column); the 8 warps of the block split the P parts into 8
        // contiguous ranges and fold them at once (more loads in flight than
        // one thread folding all P parts); warp 0 then merges the 8 range
        // states in part order.  Lexicographic minima are order-free; the
        // fp64 sums of a segment cut by parts and of dTD^{+x_c} are grouped
        // by range (reading R9; exact on int64).
        const int P = g.P, w = g.w;
        // range states [POST_RG][8 warps][32 lanes] after the staging area (dynamic)
        typedef RangeState<A> RSRow[POST_THREADS / 32][32];
        RSRow* rs = reinterpret_cast<RSRow*>(post_smem_raw + post_rs_offset<A>(k, P, g.stage0 != 0));
        const A* sR = g.R;
        const int *hsl = g.head_slot, *tsl = g.tail_slot;
        if (g.stage0) {
            A* r_s = pr + k;
            int* h_s = reinterpret_cast<int*>(r_s + k);
            for (int i = threadIdx.x; i < k; i += blockDim.x) r_s[i] = __ldcg(&g.R[i]);
            for (int i = threadIdx.x; i < P; i += blockDim.x) { h_s[i] = __ldcg(&g.head_slot[i]); h_s[P + i] = __ldcg(&g.tail_slot[i]); }
            __syncthreads();
            sR = r_s; hsl = h_s; tsl = h_s + P;
        }
        const int es = __ldcg(g.empty_slot);
        const int nw8 = POST_THREADS / 32;
        const int qa = warp * P / nw8, qb = (warp + 1) * P / nw8;
        const int ngrp = (w + 31) >> 5;
        Rec<A> best = rec_none<A>();
        // rounds of up to POST_RG column groups: every warp folds its part
        // range for each group of the round (no barrier in between, so the
        // warps' loads overlap), then warp r merges group r of the round
        for (int g0 = b; g0 < ngrp; g0 += POST_RG * B) {
            for (int r = 0; r < POST_RG; ++r) {
                const int grp = g0 + r * B;
                if (grp >= ngrp) break;
                const int cl = grp * 32 + lane;
                const bool valid = cl < w;
                RangeState<A> st;
                st.plus = 0; st.hc = 0; st.tc = 0; st.bv = amax<A>();
                st.hs = -1; st.ts = -1; st.bs = INT_MAX; st.single = 1;
                A carry = 0;
                int cs = -1;
                for (int q0 = qa; q0 < qb; q0 += POST_QU) {
                    A pl[POST_QU], hv[POST_QU], tv[POST_QU], iv[POST_QU];
                    int isl[POST_QU];
#pragma unroll
                    for (int u = 0; u < POST_QU; ++u) {
                        const int q = q0 + u;
                        if (valid && q < qb) {
                            const int64_t idx = (int64_t)q * w + cl;
                            pl[u] = __ldcg(&g.pp_plus[idx]); hv[u] = __ldcg(&g.pp_head[idx]);
                            tv[u] = __ldcg(&g.pp_tail[idx]); iv[u] = __ldcg(&g.pp_imin[idx]);
                            isl[u] = __ldcg(&g.pp_islot[idx]);
                        } else {
                            pl[u] = 0; hv[u] = 0; tv[u] = 0; iv[u] = 0; isl[u] = -1;
                        }
                    }
#pragma unroll
                    for (int u = 0; u < POST_QU; ++u) {
                        const int q = q0 + u;
                        if (q >= qb) break;
                        // a completed segment (s, sum): the range's first one may
                        // continue the previous range -> kept as the head piece
                        auto fin = [&](int s, A sum) {
                            if (st.single) { st.hs = s; st.hc = sum; st.single = 0; }
                            else {
                                const A val = sR[s] + sum;
                                if (val < st.bv || (val == st.bv && s < st.bs)) { st.bv = val; st.bs = s; }
                            }
                        };
                        st.plus += pl[u];
                        const int h = hsl[q], t = tsl[q];
                        if (h == cs) carry += hv[u];
                        else {
                            if (cs >= 0) fin(cs, carry);
                            cs = h;
                            carry = hv[u];
                        }
                        if (isl[u] >= 0 && (iv[u] < st.bv || (iv[u] == st.bv && isl[u] < st.bs))) { st.bv = iv[u]; st.bs = isl[u]; }
                        if (t != h) {
                            fin(cs, carry);
                            cs = t;
                            carry = tv[u];
                        }
                    }
                }
                st.ts = cs; st.tc = carry;
                if (st.single) { st.hs = cs; st.hc = carry; }
                rs[r][warp][lane] = st;
            }
            __syncthreads();
            {
                const int grp = g0 + warp * B;
                const int cl = grp * 32 + lane;
                if (warp < POST_RG && grp < ngrp && cl < w) {
                    A bv = amax<A>();
                    int bs = INT_MAX;
                    if (es != INT_MAX) { bv = 0; bs = es; }
                    auto fin = [&](int s, A sum) {
                        KM_ASSERT(s >= 0 && s < k);
                        const A val = sR[s] + sum;
                        if (val < bv || (val == bv && s < bs)) { bv = val; bs = s; }
                    };
                    A plus = 0, cr = 0;
                    int c_s = -1;
                    for (int r = 0; r < nw8; ++r) {
                        if (r * P / nw8 == (r + 1) * P / nw8) continue;      // empty range
                        const RangeState<A> x = rs[warp][r][lane];
                        plus += x.plus;
                        if (x.bs != INT_MAX && (x.bv < bv || (x.bv == bv && x.bs < bs))) { bv = x.bv; bs = x.bs; }
                        if (x.single) {
                            if (x.hs == c_s) cr += x.hc;
                            else { if (c_s >= 0) fin(c_s, cr); c_s = x.hs; cr = x.hc; }
                        } else {
                            if (x.hs == c_s) fin(c_s, cr + x.hc);
                            else { if (c_s >= 0) fin(c_s, cr); fin(x.hs, x.hc); }
                            c_s = x.ts; cr = x.tc;
                        }
                    }
                    fin(c_s, cr);
                    const A dtd = bv + plus;
                    const int64_t c = g.c0 + cl;
                    const bool medoid = __ldcg(&g.point_slot[c]) >= 0;
                    g.cand_v[cl] = dtd;
                    g.cand_slot[cl] = medoid ? -1 : bs;
                    if (!medoid) {
                        Rec<A> x; x.v = dtd; x.slot = bs; x.c = (int)c;
                        if (rec_less(x, best)) best = x;
                    }
                }
            }
            __syncthreads();                     // rs is rewritten by the next round
        }
        {
            __shared__ Rec<A> wbest[POST_THREADS / 32];
            best = warp_min_rec(best);
            if (lane == 0) wbest[warp] = best;
            __syncthreads();
            if (warp == 0) {
                best = lane < POST_THREADS / 32 ? wbest[lane] : rec_none<A>();
                best = warp_min_rec(best);
                if (lane == 0) g.blk_recs[b] = best;
            }
        }
        grid.sync();
        post_stamp(g.tph, 6);
    }
    if (b == 0 && threadIdx.x == 0) *g.empty_slot = INT_MAX;   // (read by the stream and the combine / phase 0)

    // ---- A: select
    if (!g.prep_only) {
        Rec<A> best = rec_none<A>();
        if (fused) {                            // every block: min over the block records (order-free)
            if (warp == 0) {
                // one 16-byte load per record, all of a lane's records in flight
                static_assert(sizeof(Rec<A>) == 16, "Rec is 16 bytes");
                const int4* br = reinterpret_cast<const int4*>(g.blk_recs);
                for (int i0 = 0; i0 * 32 < B; i0 += 8) {
                    int4 raw[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int r = (i0 + i) * 32 + lane;
                        raw[i] = r < B ? __ldcg(&br[r]) : make_int4(0, 0, INT_MAX, INT_MAX);
                    }
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        if ((i0 + i) * 32 + lane >= B) continue;
                        Rec<A> x;
                        memcpy(&x, &raw[i], sizeof(x));
                        if (rec_less(x, best)) best = x;
                    }
                }
                best = warp_min_rec(best);
            }
        }
        if (threadIdx.x == 0) {
            if (!fused)
                for (int r = 0; r < g.nrec; ++r) {
                    const Rec<A> x = g.recs[r];
                    if (rec_less(x, best)) best = x;
                }
            const A tdv = *g.td;
            bool improving;
            if (best.slot == INT_MAX) improving = false;
            else if (std::is_same<A, double>::value) improving = (double)best.v < -1e-12 * fabs((double)tdv);
            else improving = best.v < 0;
            Decision<A> dd = *g.dec;
            dd.iters += 1;
            dd.apply = improving ? 1 : 0;
            dd.dtd = best.v;
            dd.slot = best.slot;
            dd.c = best.c;
            if (improving) {
                dd.old_m = g.M[best.slot];
                dd.swaps += 1;
            } else {
                dd.done = 1;
            }
            sdec = dd;
        }
    }
    __syncthreads();
    if (!g.prep_only) d = sdec;
    post_stamp(g.tph, 1);

    // ---- A: apply (column c*, incremental nearest/second, in-block rescans)
    if (!g.prep_only && d.apply) {
        __shared__ int r_j1[POST_THREADS], r_j2[POST_THREADS];
        __shared__ T r_d1[POST_THREADS], r_d2[POST_THREADS];
        const int i = d.slot;
        const bool local = d.c >= g.c0 && d.c < g.c1;
        int myent = -1;
        if (reg) {
            if (have) {
                // column c* of D (n scattered sectors), or row c* when D is
                // symmetric (one coalesced 4n-byte read, the same values)
                const T x = !local ? g.MC[(int64_t)i * n + myo]
                                   : g.sym ? g.D[(int64_t)d.c * g.ld + myo] : g.D[(int64_t)myo * g.ld + (d.c - g.c0)];
                if (local) g.MC[(int64_t)i * n + myo] = x;
                if (j1 == i || j2 == i) {
                    myent = atomicAdd(&s_nres, 1);
                    KM_ASSERT(ob0 + myent < ob1);
                    g.rescan[ob0 + myent] = myo;
                } else if (x < d1 || (x == d1 && i < j1)) {
                    j2 = j1; d2 = d1; j1 = i; d1 = x;
                    g.near[myo] = j1; g.dn[myo] = d1; g.sec[myo] = j2; g.ds[myo] = d2;
                } else if (x < d2 || (x == d2 && i < j2)) {
                    j2 = i; d2 = x;
                    g.sec[myo] = j2; g.ds[myo] = d2;
                }
            }
        } else {
            for (int o = ob0 + threadIdx.x; o < ob1; o += blockDim.x)
                if (local) g.MC[(int64_t)i * n + o] = g.D[(int64_t)o * g.ld + (d.c - g.c0)];
            // (the column is read back below by the same thread: same o mapping)
            for (int o = ob0 + threadIdx.x; o < ob1; o += blockDim.x) {
                const int a1 = __ldcg(&g.near[o]), a2 = __ldcg(&g.sec[o]);
                if (a1 == i || a2 == i) {
                    g.rescan[ob0 + atomicAdd(&s_nres, 1)] = o;
                    continue;
                }
                const T x = g.MC[(int64_t)i * n + o];
                const T e1 = __ldcg(&g.dn[o]), e2 = __ldcg(&g.ds[o]);
                if (x < e1 || (x == e1 && i < a1)) {
                    g.near[o] = i; g.dn[o] = x; g.sec[o] = a1; g.ds[o] = e1;
                } else if (x < e2 || (x == e2 && i < a2)) {
                    g.sec[o] = i; g.ds[o] = x;
                }
            }
        }
        __syncthreads();
        const int nres = s_nres;
        for (int e = warp; e < nres; e += POST_THREADS / 32) {
            const int o = g.rescan[ob0 + e];
            KM_ASSERT(o >= ob0 && o < ob1);
            T q1 = dmax<T>(), q2 = dmax<T>();
            int k1 = INT_MAX, k2 = INT_MAX;
#pragma unroll 8
            for (int j = lane; j < k; j += 32) {
                const T dd = __ldcg(&g.MC[(int64_t)j * n + o]);
                if (lex_lt(dd, j, q1, k1)) { q2 = q1; k2 = k1; q1 = dd; k1 = j; }
                else if (lex_lt(dd, j, q2, k2)) { q2 = dd; k2 = j; }
            }
#pragma unroll
            for (int x = 16; x >= 1; x >>= 1) {
                const T e1 = __shfl_xor_sync(FULL, q1, x), e2 = __shfl_xor_sync(FULL, q2, x);
                const int f1 = __shfl_xor_sync(FULL, k1, x), f2 = __shfl_xor_sync(FULL, k2, x);
                if (lex_lt(e1, f1, q1, k1)) {
                    if (lex_lt(q1, k1, e2, f2)) { q2 = q1; k2 = k1; } else { q2 = e2; k2 = f2; }
                    q1 = e1; k1 = f1;
                } else if (lex_lt(e1, f1, q2, k2)) {
                    q2 = e1; k2 = f1;
                }
            }
            if (lane == 0) {
                KM_ASSERT(k1 >= 0 && k1 < k && k2 >= 0 && k2 < k && k1 != k2);
                g.near[o] = k1; g.sec[o] = k2; g.dn[o] = q1; g.ds[o] = q2;
                if (reg) { r_j1[e] = k1; r_j2[e] = k2; r_d1[e] = q1; r_d2[e] = q2; }
            }
        }
        __syncthreads();                        // the chunk's cache is final (block-visible)
        if (myent >= 0) { j1 = r_j1[myent]; j2 = r_j2[myent]; d1 = r_d1[myent]; d2 = r_d2[myent]; }
    }
    post_stamp(g.tph, 2);

    // ---- A: count -- per slot, the chunk's objects and partial removal loss
    {
        for (int base = ob0; base < ob1; base += POST_THREADS) {
            const int o = base + threadIdx.x;
            const bool v = o < ob1;
            int s = 0;
            A val = 0;
            if (v) {
                if (reg) { s = j1; val = (A)d2 - (A)d1; }
                else { s = __ldcg(&g.near[o]); val = (A)__ldcg(&g.ds[o]) - (A)__ldcg(&g.dn[o]); }
                KM_ASSERT(s >= 0 && s < k && val >= 0);
                atomicAdd(&hh[s], 1);
            }
            if constexpr (std::is_same<A, double>::value) {
                // float path, deterministic: per warp, the leader of each
                // slot's peers sums their values in lane order; the warps'
                // sums then enter pr[] in warp order (one warp at a time)
                const unsigned peers = __match_any_sync(FULL, v ? s : -1 - lane);
                const int leader = __ffs(peers) - 1;
                A acc = 0;
#pragma unroll
                for (int t = 0; t < 32; ++t) {
                    const A vt = __shfl_sync(FULL, val, t);
                    if ((peers >> t) & 1u) acc += vt;
                }
                const int nw = (min(POST_THREADS, ob1 - base) + 31) >> 5;
                for (int w = 0; w < nw; ++w) {
                    if (warp == w && v && lane == leader) pr[s] += acc;
                    __syncthreads();
                }
            } else {
                if (v) atomicAdd(reinterpret_cast<unsigned long long*>(&pr[s]), (unsigned long long)val);   // exact
            }
        }
        __syncthreads();
        for (int s = threadIdx.x; s < k; s += blockDim.x) {
            g.counts[(int64_t)s * B + b] = hh[s];
            g.rpart[(int64_t)s * B + b] = pr[s];
        }
    }
    grid.sync(); post_stamp(g.tph, 3);

    if (!g.prep_only && b == 0 && threadIdx.x == 0) {
        // every block has read dec / M / td (phase A): record the decision
        *g.dec = sdec;
        if (sdec.apply) {
            g.M[sdec.slot] = sdec.c;
            g.point_slot[sdec.old_m] = -1;
            g.point_slot[sdec.c] = sdec.slot;
            *g.td = *g.td + sdec.dtd;
        }
    }

    // ---- B: warp per slot -- chunk offsets (all B counts loaded first, then
    // register-only warp scans), slot total, removal loss (fixed tree)
    for (int s = gwarp; s < k; s += nwarps) {
        const int* cs = g.counts + (int64_t)s * B;
        const A* ps = g.rpart + (int64_t)s * B;
        int cv[POST_MAX_PER];
        A rsum = 0;
#pragma unroll
        for (int i = 0; i < POST_MAX_PER; ++i) {
            const int bb = i * 32 + lane;
            cv[i] = bb < B ? __ldcg(&cs[bb]) : 0;
            if (bb < B) rsum += __ldcg(&ps[bb]);
        }
#pragma unroll
        for (int x = 16; x >= 1; x >>= 1) rsum += __shfl_xor_sync(FULL, rsum, x);
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
        if (lane == 0) {
            g.slot_tot[s] = run;
            g.R[s] = rsum;
            if (run == 0) atomicMin(g.empty_slot, s);
        }
    }
    grid.sync(); post_stamp(g.tph, 4);

    // ---- C: segment starts (every block, its shared memory; block 0 also
    // writes seg_start[] for the FastPAM2 / window paths), stable scatter of
    // the chunk, part head / tail slots
    {
        __shared__ int wsum[POST_THREADS / 32];
        int* segs = hh;                          // k ints: segment starts, then the scatter cursors
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
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        int base = 0;
        for (int w = 0; w < warp; ++w) base += wsum[w];
        int run = base + incl - sum;
        for (int i = a; i < z; ++i) {
            segs[i] = run;
            if (b == 0) g.seg_start[i] = run;
            run += __ldcg(&g.slot_tot[i]);
        }
        if (b == 0 && threadIdx.x == blockDim.x - 1) g.seg_start[k] = run;
        __syncthreads();
        // part metadata: the slot of sorted position p is the last s with
        // segs[s] <= p (empty slots share their successor's start)
        for (int q = tid; q < g.P; q += nth) {
            const int64_t p0 = part_lo(q, n, g.P), p1 = part_lo(q + 1, n, g.P);
            for (int side = 0; side < 2; ++side) {
                const int64_t p = side == 0 ? p0 : p1 - 1;
                int lo = 0, hi = k - 1;              // segs[0] = 0 <= p
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (segs[mid] <= p) lo = mid; else hi = mid - 1;
                }
                KM_ASSERT(lo >= 0 && lo < k && segs[lo] <= p && (lo == k - 1 || segs[lo + 1] > p));
                if (side == 0) g.head_slot[q] = lo; else g.tail_slot[q] = lo;
            }
        }
        __syncthreads();                        // the part search reads segs; the cursors overwrite them
        // stable scatter into (slot, o) order: every warp ranks its 32 objects
        // among same-slot peers (match_any); the warps then take their slot
        // ranges from the cursors one after another (warp order = object order)
        int* cur = segs;
        for (int s = threadIdx.x; s < k; s += blockDim.x) cur[s] += __ldcg(&g.offsets[(int64_t)s * B + b]);
        __syncthreads();
        const unsigned lt = (1u << lane) - 1u;
        for (int base = ob0; base < ob1; base += POST_THREADS) {
            const int e = base + threadIdx.x;
            const bool valid = e < ob1;
            int s = -1 - lane;
            T en = 0, es = 0;
            if (valid) {
                if (reg) { s = j1; en = d1; es = d2; }
                else { s = __ldcg(&g.near[e]); en = __ldcg(&g.dn[e]); es = __ldcg(&g.ds[e]); }
            }
            const unsigned peers = __match_any_sync(FULL, s);
            const int rank = __popc(peers & lt);
            const int leader = __ffs(peers) - 1;
            int bp = 0;
            const int nw = (min(POST_THREADS, ob1 - base) + 31) >> 5;
            for (int w = 0; w < nw; ++w) {
                if (warp == w && valid && lane == leader) { bp = cur[s]; cur[s] = bp + __popc(peers); }
                __syncthreads();
            }
            bp = __shfl_sync(FULL, bp, leader);
            if (valid) {
                RowInfo<T> r;
                r.o = e; r.slot = s; r.dn = en; r.ds = es;
                const int pos = bp + rank;
                KM_ASSERT(pos >= 0 && pos < n && s >= 0 && s < k);
                g.ri[pos] = r;
                if (g.rowd) g.rowd[pos] = make_double2((double)en, (double)es);
            }
        }
    }
    if (b == 0 && threadIdx.x == 0) {
        *g.rescan_count = 0;
        if (!g.prep_only) {
            // the outcome straight into pinned host memory (visible to the host
            // once the launch's completion event is observed, or once it
            // reads seq == q: seq is written last, behind a system fence)
            const int q = *g.seq;
            if (g.h_ring) ring_put(g.h_ring[q % g.ring], sdec, *g.td, q, 0);
            *g.seq = q + 1;
        }
    }
    post_stamp(g.tph, 5);
}

}  // namespace km
