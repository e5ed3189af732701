// km_fasterpam.cuh -- FasterPAM's eager scan inside one candidate window
// (Alg.4; readings F1-F5 and "FasterPAM").
//
// The host streams a window of candidate columns once on the current state
// (k_swap_stream_seg2 in FastPAM2 mode + k_swap_combine): acc[i][j] (the
// complete per-slot sums of Eq. eqn:better-change3) and plus[j] (dTD^{+x_c})
// for every window column j.  ONE cooperative kernel then runs Alg.4's scan
// over the window:
//
//   pick     first window position j >= p whose candidate is improving:
//            min_i (R_i + acc[i][j]) + plus[j] < 0 (reading R5), slots tied
//            to the smaller index (F4); warps evaluate consecutive positions
//   apply    M[i*] <- c*, TD += dTD; MC[i*] <- column c*; nearest/second of
//            every object (incremental; warp rescans for objects whose
//            nearest/second was slot i*), equal to a from-scratch assignment
//   correct  the objects whose (nearest, d_n, d_s) changed (about 3n/k) are
//            listed in object order; for the window positions still ahead,
//            acc/plus are corrected by their old and new terms, R by the
//            change of (d_s - d_n):  the window's values become those of a
//            fresh evaluation on the new state (exact on the integer path;
//            fp64 re-association on the float path, reading R9)
//
// and repeats from j+1, so no swap discards the window (the speculative
// batch path re-streams after every swap).  Work per swap is O(n) for the
// cache plus O(m * L) dissimilarities for the correction (m changed objects,
// L positions ahead), instead of an O(n * window) re-stream.  Everything the
// scan needs between swaps (acc, plus, R, cache) stays in L2.
//
// Determinism: the changed list is compacted in object order; corrections
// are summed per (event group, touched slot, column) in a fixed order, so
// the float path is reproducible run to run.
#pragma once
#include "km_kernels.cuh"

namespace km {

constexpr int FP3_TMAX = 32;     // touched slots a correction step handles (else: re-stream)
constexpr int FP3_TV = 8;        // GLOBAL correction: touched slots per slice (4 columns per lane)
constexpr int FP3_EV = 16;      // D loads in flight per lane in the correction (events ahead; 32 measured slower)
constexpr int FP3_G = 32;        // event groups of the correction (columns x groups warps)
constexpr int FP3_THREADS = 256;
constexpr int FP3_WARPS = FP3_THREADS / 32;
constexpr int FP3_SMEM = FP3_WARPS * (FP3_TMAX * 32 + FP3_TMAX) * 8;   // per warp: [TMAX][32] acc + [TMAX] R

enum { FP3_DONE = 0, FP3_STALE = 1 };

template <typename T>
struct alignas(16) Fp3Chg {      // one object whose (nearest, d_n, d_s) changed
    int32_t o, near_old, near_new, pad;
    T dn_old, ds_old, dn_new, ds_new;
};

struct Fp3Ctl {
    int first[3];        // pick rounds (rotating, see k_fp3_window)
    int nres;            // rescan list length
    int m;               // changed objects
    int T;               // touched slots
    int status;          // FP3_DONE / FP3_STALE
    int p_end;           // window position the scan reached
    int swaps;           // swaps made in this window
    int pad[7];
    unsigned long long tphase[8];   // ns per phase (block 0's view), for tuning
};

__device__ __forceinline__ unsigned long long fp3_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

template <typename T, typename A>
struct Fp3Args {
    const T* D;
    int64_t ld;
    int n, k;
    int64_t c0;          // global index of slab column 0
    int a;               // window start (slab column)
    int ww;              // window width = row stride of acc
    int lo, hi;          // scan range (window-local positions)
    int L;               // correction horizon (positions ahead of a swap)
    A* acc;              // [k][ww]
    A* plus;             // [ww]
    A* R;                // [k]
    int* M;
    int* point_slot;
    T* MC;               // [k][n]
    T* MCt;              // [n][k]: the same distances object-major (coalesced rescans)
    int *near, *sec;
    T *dn, *ds;
    A* td;
    Decision<A>* dec;
    Rec<A>* trace;
    int trace_cap;
    // scratch
    A* cand_v;           // [ww]
    int* cand_s;         // [ww]
    int* flag;           // [n]
    int* old_near;       // [n]
    T *old_dn, *old_ds;  // [n]
    int* rescan;         // [n]
    int* blk_cnt;        // [gridDim]
    Fp3Chg<T>* chg;      // [chg_cap]
    int chg_cap;
    int* touched_flag;   // [k], zero between steps
    int* touched_map;    // [k] slot -> touched index
    int* touched;        // [k]
    A* part_acc;         // [FP3_G][FP3_TMAX][L]
    A* part_plus;        // [FP3_G][L]
    A* part_R;           // [FP3_G][FP3_TMAX]
    Fp3Ctl* ctl;
    int new_pass;        // count a pass in dec->iters (F3)
    // GLOBAL mode (incremental FastPAM1): best swap over all candidates per iteration
    int max_iters;
    Rec<A>* gpart;       // [gridDim] per-block best records
};

template <typename T>
__device__ __forceinline__ Fp3Chg<T> fp3_ld_chg(const Fp3Chg<T>* p) {
    static_assert(sizeof(Fp3Chg<T>) == 32, "Fp3Chg layout");
    const int4 a = __ldcg(reinterpret_cast<const int4*>(p));
    const int4 b = __ldcg(reinterpret_cast<const int4*>(p) + 1);
    Fp3Chg<T> e;
    memcpy(&e, &a, 16);
    memcpy(reinterpret_cast<char*>(&e) + 16, &b, 16);
    return e;
}

template <typename A>
__device__ __forceinline__ bool fp3_improving(A v, A tdv) {
    if (std::is_same<A, double>::value) return (double)v < -1e-12 * fabs((double)tdv);
    return v < 0;
}

// Alg.3 P:883-889 terms of one object for a candidate at dissimilarity x:
// tp -> dTD^{+x_c}, ta -> acc_c[nearest(o)].
template <typename T, typename A>
__device__ __forceinline__ void fp3_terms(T x, T dnv, T dsv, A& tp, A& ta) {
    const bool c1 = x < dnv, c2 = x < dsv;
    tp = c1 ? (A)x - (A)dnv : (A)0;
    ta = c1 ? (A)dnv - (A)dsv : (c2 ? (A)x - (A)dsv : (A)0);
}

// Block-wide exclusive prefix of one int per thread (blockDim = FP3_THREADS);
// returns the prefix, *total receives the block sum.
__device__ __forceinline__ int fp3_block_scan(int v, int* total) {
    __shared__ int wsum[FP3_WARPS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, d);
        if (lane >= d) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int base = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < FP3_WARPS; ++w) {
        const int s = wsum[w];
        if (w < warp) base += s;
        tot += s;
    }
    __syncthreads();
    *total = tot;
    return base + incl - v;
}

// MCt[o][j] = MC[j][o] (32x32 tiles through shared memory).
template <typename T>
__global__ void k_fp3_transpose_mc(const T* __restrict__ MC, int n, int k, T* __restrict__ MCt) {
    __shared__ T tile[32][33];
    const int o0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int j = j0 + r, o = o0 + threadIdx.x;
        if (j < k && o < n) tile[r][threadIdx.x] = MC[(int64_t)j * n + o];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int o = o0 + r, j = j0 + threadIdx.x;
        if (j < k && o < n) MCt[(int64_t)o * k + j] = tile[threadIdx.x][r];
    }
}

// GLOBAL = false: FasterPAM's eager scan of one window (Alg.4).
// GLOBAL = true: incremental FastPAM1 (Alg.3's best swap per iteration, key
// R1) over ALL candidates: the stored k-vectors acc[i][c] / plus[c] (a
// FastPAM2-mode stream pass) are corrected after every swap for every
// candidate, so an iteration reads the changed objects' rows instead of D.
template <typename T, typename A, bool GLOBAL>
__global__ void __launch_bounds__(FP3_THREADS)
k_fp3_window(Fp3Args<T, A> g) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char fp3_smem[];
    __shared__ int s_off;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    const int gwarp = tid >> 5, nwarps = nth >> 5;
    const int n = g.n, k = g.k;
    Fp3Ctl* ctl = g.ctl;
    int p = g.lo, vhi = g.hi;   // positions [p, vhi) hold values of the current state
    int rnd = 0;                // pick rounds so far (selects ctl->first[rnd % 3])
    int swaps = 0;
    int status = FP3_DONE;
    if (g.new_pass && blockIdx.x == 0 && threadIdx.x == 0) g.dec->iters += 1;
    unsigned long long tlast = fp3_now();

    int iters_done = 0;
    bool converged = false;
    while (GLOBAL ? (iters_done < g.max_iters) : (p < vhi)) {
        // ------------------------------------------------------------ pick
        if (blockIdx.x == 0 && threadIdx.x == 0) ctl->nres = 0;
        for (int b = tid; b < (int)gridDim.x; b += nth) g.blk_cnt[b] = 0;
        int found = INT_MAX;
        const A tdv = __ldcg(g.td);
        int gslot = 0;
        A gv = 0;
        // R_i staged in shared memory for the pick (the correction's buffer is idle here)
        A* sR = reinterpret_cast<A*>(fp3_smem);
        const bool r_smem = (size_t)k * sizeof(A) <= (size_t)FP3_SMEM;
        if (r_smem) {
            for (int i = threadIdx.x; i < k; i += blockDim.x) sR[i] = __ldcg(&g.R[i]);
            __syncthreads();
        }
        if constexpr (GLOBAL) {
            // lexicographic min of (dTD, slot, c) over every non-medoid candidate (R1);
            // one thread per candidate, slots in ascending order (strict <): the
            // acc[i][j .. j+31] reads of a warp are contiguous
            __shared__ Rec<A> sbest[FP3_WARPS];
            Rec<A> best = rec_none<A>();
            for (int j = tid; j < g.hi; j += nth) {
                const int64_t cc = g.c0 + g.a + j;
                if (__ldcg(&g.point_slot[cc]) >= 0) continue;
                A bv = amax<A>();
                int bs = INT_MAX;
                const A* aj = g.acc + j;
#pragma unroll 8
                for (int i = 0; i < k; ++i) {
                    const A v = (r_smem ? sR[i] : __ldcg(&g.R[i])) + __ldcg(aj + (int64_t)i * g.ww);
                    if (v < bv) { bv = v; bs = i; }
                }
                Rec<A> r; r.v = bv + __ldcg(&g.plus[j]); r.slot = bs; r.c = (int)cc;
                if (rec_less(r, best)) best = r;
            }
            best = warp_min_rec(best);
            if (lane == 0) sbest[warp] = best;
            __syncthreads();
            if (threadIdx.x == 0) {
                Rec<A> b = rec_none<A>();
                for (int w2 = 0; w2 < FP3_WARPS; ++w2) if (rec_less(sbest[w2], b)) b = sbest[w2];
                g.gpart[blockIdx.x] = b;
            }
            if (blockIdx.x == 0 && threadIdx.x == 0) g.dec->iters += 1;   // a pass
            grid.sync();
            Rec<A> b = rec_none<A>();
            for (int q2 = threadIdx.x; q2 < (int)gridDim.x; q2 += blockDim.x) {
                Rec<A> r;
                r.v = __ldcg(&g.gpart[q2].v); r.slot = __ldcg(&g.gpart[q2].slot); r.c = __ldcg(&g.gpart[q2].c);
                if (rec_less(r, b)) b = r;
            }
            b = block_min_rec(b);
            __shared__ Rec<A> sfin;
            if (threadIdx.x == 0) sfin = b;
            __syncthreads();
            b = sfin;
            ++iters_done;
            if (b.slot == INT_MAX || !fp3_improving(b.v, tdv)) { converged = true; break; }
            found = (int)(b.c - g.c0 - g.a);
            gslot = b.slot;
            gv = b.v;
        } else
        for (int base = p; base < vhi; base += nwarps) {
            const int slot_now = rnd % 3;
            // first[(rnd+1)%3] was last read before the previous round's sync
            if (blockIdx.x == 0 && threadIdx.x == 0) ctl->first[(rnd + 1) % 3] = INT_MAX;
            const int j = base + gwarp;
            if (j < vhi && __ldcg(&g.point_slot[g.c0 + g.a + j]) < 0) {
                A bv = amax<A>();
                int bs = INT_MAX;
#pragma unroll 8
                for (int i = lane; i < k; i += 32) {
                    const A v = (r_smem ? sR[i] : __ldcg(&g.R[i])) + __ldcg(&g.acc[(int64_t)i * g.ww + j]);
                    if (v < bv) { bv = v; bs = i; }
                }
#pragma unroll
                for (int x = 16; x >= 1; x >>= 1) {
                    const A ov = __shfl_xor_sync(FULL, bv, x);
                    const int os = __shfl_xor_sync(FULL, bs, x);
                    if (ov < bv || (ov == bv && os < bs)) { bv = ov; bs = os; }
                }
                const A v = bv + __ldcg(&g.plus[j]);
                if (lane == 0) {
                    g.cand_v[j] = v;
                    g.cand_s[j] = bs;
                    if (fp3_improving(v, tdv)) atomicMin(&ctl->first[slot_now], j);
                }
            }
            grid.sync();
            if (blockIdx.x == 0 && threadIdx.x == 0) { const unsigned long long tn = fp3_now(); ctl->tphase[0] += tn - tlast; tlast = tn; }
            found = __ldcg(&ctl->first[slot_now]);
            ++rnd;
            if (found != INT_MAX) break;
        }
        if (found == INT_MAX) { p = vhi; break; }

        // ------------------------------------------------------------ apply
        const int j = found;
        const int slot = GLOBAL ? gslot : __ldcg(&g.cand_s[j]);
        const A v = GLOBAL ? gv : __ldcg(&g.cand_v[j]);
        const int64_t c = g.c0 + g.a + j;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            const int old = g.M[slot];
            g.M[slot] = (int)c;
            g.point_slot[old] = -1;
            g.point_slot[c] = slot;
            *g.td = tdv + v;
            if (swaps < g.trace_cap) { Rec<A> t; t.v = v; t.slot = slot; t.c = (int)c; g.trace[swaps] = t; }
            g.dec->swaps += 1;
            g.dec->apply = 1;
            g.dec->slot = slot;
            g.dec->c = (int)c;
            g.dec->dtd = v;
            g.dec->old_m = old;
        }
        ++swaps;
        // block b of the compaction owns objects [b*chunk, (b+1)*chunk)
        const int chunk = (n + (int)gridDim.x - 1) / (int)gridDim.x;
        auto mark_changed = [&](int o, int jold, int jnew) {
            atomicAdd(&g.blk_cnt[o / chunk], 1);
            g.touched_flag[jold] = 1;
            g.touched_flag[jnew] = 1;
        };
        for (int o = tid; o < n; o += nth) {
            const T x = g.D[(int64_t)o * g.ld + (c - g.c0)];
            g.MC[(int64_t)slot * n + o] = x;
            g.MCt[(int64_t)o * k + slot] = x;
            const int j1 = __ldcg(&g.near[o]), j2 = __ldcg(&g.sec[o]);
            const T d1 = __ldcg(&g.dn[o]), d2 = __ldcg(&g.ds[o]);
            g.old_near[o] = j1; g.old_dn[o] = d1; g.old_ds[o] = d2;
            if (j1 == slot || j2 == slot) {
                g.rescan[atomicAdd(&ctl->nres, 1)] = o;
                g.flag[o] = 0;
            } else if (x < d1 || (x == d1 && slot < j1)) {
                g.near[o] = slot; g.dn[o] = x; g.sec[o] = j1; g.ds[o] = d1;
                g.flag[o] = 1;
                mark_changed(o, j1, slot);
            } else if (x < d2 || (x == d2 && slot < j2)) {
                g.sec[o] = slot; g.ds[o] = x;
                g.flag[o] = (x != d2) ? 1 : 0;
                if (x != d2) mark_changed(o, j1, j1);
            } else {
                g.flag[o] = 0;
            }
        }
        grid.sync();
        if (blockIdx.x == 0 && threadIdx.x == 0) { const unsigned long long tn = fp3_now(); ctl->tphase[1] += tn - tlast; tlast = tn; }
        // rescans: (d, slot) lexicographic top-2 over the k medoid columns
        {
            const int nres = __ldcg(&ctl->nres);
            for (int e = gwarp; e < nres; e += nwarps) {
                const int o = __ldcg(&g.rescan[e]);
                T d1 = dmax<T>(), d2 = dmax<T>();
                int j1 = INT_MAX, j2 = INT_MAX;
#pragma unroll 8
                for (int jj = lane; jj < k; jj += 32) {
                    const T d = __ldcg(&g.MCt[(int64_t)o * k + jj]);
                    if (lex_lt(d, jj, d1, j1)) { d2 = d1; j2 = j1; d1 = d; j1 = jj; }
                    else if (lex_lt(d, jj, d2, j2)) { d2 = d; j2 = jj; }
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
                    const int jo = __ldcg(&g.old_near[o]);
                    const bool ch = j1 != jo || d1 != __ldcg(&g.old_dn[o]) || d2 != __ldcg(&g.old_ds[o]);
                    g.flag[o] = ch ? 1 : 0;
                    if (ch) mark_changed(o, jo, j1);
                }
            }
        }
        grid.sync();
        if (blockIdx.x == 0 && threadIdx.x == 0) { const unsigned long long tn = fp3_now(); ctl->tphase[2] += tn - tlast; tlast = tn; }
        // ------------------------------------------------------------ changed list
        // (per-block counts and touched slots were gathered during apply/rescan)
        const int ob0 = min(n, (int)blockIdx.x * chunk), ob1 = min(n, ob0 + chunk);
        {
            int part = 0, tot = 0;
            for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
                const int cb = __ldcg(&g.blk_cnt[b]);
                if (b < (int)blockIdx.x) part += cb;
                tot += cb;
            }
            int off, m_all;
            fp3_block_scan(part, &off);                    // block sums
            fp3_block_scan(tot, &m_all);
            if (threadIdx.x == 0) s_off = off;
            __syncthreads();
            int run = s_off;
            if (m_all <= g.chg_cap) {
                for (int o0 = ob0; o0 < ob1; o0 += blockDim.x) {
                    const int o = o0 + threadIdx.x;
                    const int f = (o < ob1 && __ldcg(&g.flag[o])) ? 1 : 0;
                    int bt;
                    const int r = fp3_block_scan(f, &bt);
                    if (f) {
                        Fp3Chg<T> e;
                        e.o = o; e.near_old = __ldcg(&g.old_near[o]); e.near_new = __ldcg(&g.near[o]); e.pad = 0;
                        e.dn_old = __ldcg(&g.old_dn[o]); e.ds_old = __ldcg(&g.old_ds[o]);
                        e.dn_new = __ldcg(&g.dn[o]); e.ds_new = __ldcg(&g.ds[o]);
                        g.chg[run + r] = e;
                    }
                    run += bt;
                }
            }
            if (blockIdx.x == 0) {
                // touched slots in ascending order
                int tb = 0;
                for (int s0 = 0; s0 < k; s0 += blockDim.x) {
                    const int s = s0 + threadIdx.x;
                    const int f = (s < k && __ldcg(&g.touched_flag[s])) ? 1 : 0;
                    int bt;
                    const int r = fp3_block_scan(f, &bt);
                    if (f) {
                        g.touched[tb + r] = s;
                        g.touched_map[s] = tb + r;
                    }
                    tb += bt;
                }
                if (threadIdx.x == 0) { ctl->m = m_all; ctl->T = tb; }
            }
        }
        grid.sync();
        if (blockIdx.x == 0 && threadIdx.x == 0) { const unsigned long long tn = fp3_now(); ctl->tphase[4] += tn - tlast; tlast = tn; }
        const int m = __ldcg(&ctl->m), T_ = __ldcg(&ctl->T);
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            ctl->pad[0] += __ldcg(&ctl->nres); ctl->pad[1] += m; ctl->pad[2] += T_;
        }
        const int cl0 = GLOBAL ? 0 : j + 1;              // GLOBAL: every candidate is corrected
        const int cl1 = GLOBAL ? vhi : min(vhi, j + 1 + g.L);
        if (m > g.chg_cap) {
            // too many changes for the correction step: the rest of the
            // window is stale; the host re-streams from j + 1
            status = FP3_STALE;
            p = j + 1;
            // reset the touched flags for the next window
            for (int s = tid; s < k; s += nth) g.touched_flag[s] = 0;
            break;
        }
        // ------------------------------------------------------------ correct
        // touched slots are handled FP3_TMAX at a time (per-warp shared-memory
        // accumulators); plus / R deltas of the non-slot terms in the first slice
        // GLOBAL with few touched slots (the common case): 4 columns per lane in
        // slices of FP3_TV slots (a slice costs about a quarter of a narrow
        // one); otherwise 1 column per lane, slices of FP3_TMAX (uniform across
        // the grid: T_ is)
        // (FasterPAM's 4096-column windows stay narrow: measured 2x slower wide,
        // too few 128-column items to occupy the grid with <= FP3_G groups)
        const bool wide = GLOBAL && T_ <= 3 * FP3_TV;
        const int SL = wide ? FP3_TV : FP3_TMAX;             // touched slots per slice
        for (int tb = 0; tb < T_; tb += SL) {
        const int TS = min(SL, T_ - tb);
        __syncthreads();
        if (wide) {
            // GLOBAL (every candidate): warp item = (event group q, 128-column
            // tile u), 4 columns per lane read as one 16-byte load per event
            // (4x fewer loads and sequential batches than 32-column tiles);
            // accumulators [slot][4][32 lanes] in shared memory (conflict-free)
            A* sacc = reinterpret_cast<A*>(fp3_smem) + (size_t)warp * (FP3_TMAX * 32 + FP3_TMAX);
            A* srs = sacc + FP3_TV * 128;
            const int ncols = cl1 - cl0;
            // tiles start at the 16-byte boundary at or below column cl0 (the
            // window start is arbitrary in FasterPAM); columns outside
            // [cl0, cl1) are masked
            const int sh = (int)((g.a + cl0) & 3);
            const int ntl = max((ncols + sh + 127) / 128, 1);
            const int G = min(FP3_G, max(1, nwarps / ntl));
            const int items = G * ntl;
            for (int it = gwarp; it < items; it += nwarps) {
                const int q = it / ntl, u = it % ntl;
                const int col = u * 128 + lane * 4 - sh;    // offset of column 0 of this lane (may be < 0)
                const int jlo = max(0, -col), jhi = max(0, min(4, ncols - col));   // valid jj in [jlo, jhi)
                const bool anyv = jlo < jhi;
                const int64_t dcol = (int64_t)g.a + cl0 + (anyv ? col : 0);
                const bool vec = jlo == 0 && jhi == 4 && ((dcol | g.ld) & 3) == 0;
                for (int t = 0; t < TS * 4; ++t) sacc[t * 32 + lane] = 0;
                if (lane < FP3_TV) srs[lane] = 0;
                __syncwarp();
                A pl[4] = {0, 0, 0, 0};
                const int e0 = (int)((int64_t)q * m / G), e1 = (int)((int64_t)(q + 1) * m / G);
                for (int eb = e0; eb < e1; eb += 32) {
                    const int nb = min(32, e1 - eb);
                    int o_l = 0, to_l = 0, tn_l = 0;
                    T dno = 0, dso = 0, dnn = 0, dsn = 0;
                    if (lane < nb) {
                        const Fp3Chg<T> ch = fp3_ld_chg(&g.chg[eb + lane]);
                        o_l = ch.o;
                        to_l = __ldcg(&g.touched_map[ch.near_old]) - tb;
                        tn_l = __ldcg(&g.touched_map[ch.near_new]) - tb;
                        dno = ch.dn_old; dso = ch.ds_old; dnn = ch.dn_new; dsn = ch.ds_new;
                    }
                    constexpr int EV4 = 8;
                    for (int e8 = 0; e8 < nb; e8 += EV4) {
                        T x[EV4][4];
#pragma unroll
                        for (int v8 = 0; v8 < EV4; ++v8) {
                            const int oo = __shfl_sync(FULL, o_l, (e8 + v8) & 31);
                            const T* src = g.D + (int64_t)oo * g.ld + dcol;
                            if (vec) {
                                typename Vec4<T>::type w4 = *reinterpret_cast<const typename Vec4<T>::type*>(src);
                                memcpy(&x[v8][0], &w4.x, sizeof(T)); memcpy(&x[v8][1], &w4.y, sizeof(T));
                                memcpy(&x[v8][2], &w4.z, sizeof(T)); memcpy(&x[v8][3], &w4.w, sizeof(T));
                            } else {
#pragma unroll
                                for (int jj = 0; jj < 4; ++jj) x[v8][jj] = (jj >= jlo && jj < jhi) ? src[jj] : dmax<T>();
                            }
                        }
#pragma unroll
                        for (int v8 = 0; v8 < EV4; ++v8) {
                            const int src_l = (e8 + v8) & 31;
                            const T a_dso = __shfl_sync(FULL, dso, src_l), a_dsn = __shfl_sync(FULL, dsn, src_l);
                            const T mx = max(a_dso, a_dsn);
                            const bool hit = (x[v8][0] < mx) | (x[v8][1] < mx) | (x[v8][2] < mx) | (x[v8][3] < mx);
                            const bool any_hit = __any_sync(FULL, hit);
                            if (!any_hit && u != 0) continue;  // u == 0 items also carry the R deltas
                            const T a_dno = __shfl_sync(FULL, dno, src_l), a_dnn = __shfl_sync(FULL, dnn, src_l);
                            const int a_to = __shfl_sync(FULL, to_l, src_l), a_tn = __shfl_sync(FULL, tn_l, src_l);
                            if (e8 + v8 < nb) {
                                const bool io = (unsigned)a_to < (unsigned)TS, in_ = (unsigned)a_tn < (unsigned)TS;
                                if (any_hit) {
#pragma unroll
                                    for (int jj = 0; jj < 4; ++jj) {
                                        A tpo, tao, tpn, tan_;
                                        fp3_terms<T, A>(x[v8][jj], a_dno, a_dso, tpo, tao);
                                        fp3_terms<T, A>(x[v8][jj], a_dnn, a_dsn, tpn, tan_);
                                        if (tb == 0) pl[jj] += tpn - tpo;
                                        if (io) sacc[(a_to * 4 + jj) * 32 + lane] -= tao;
                                        if (in_) sacc[(a_tn * 4 + jj) * 32 + lane] += tan_;
                                    }
                                }
                                if (u == 0 && lane == 0) {
                                    if (io) srs[a_to] -= (A)a_dso - (A)a_dno;
                                    if (in_) srs[a_tn] += (A)a_dsn - (A)a_dnn;
                                }
                            }
                        }
                    }
                }
                __syncwarp();
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    if (jj < jlo || jj >= jhi) continue;
                    for (int t = 0; t < TS; ++t)
                        g.part_acc[((int64_t)q * FP3_TV + t) * g.L + col + jj] = sacc[(t * 4 + jj) * 32 + lane];
                    if (tb == 0) g.part_plus[(int64_t)q * g.L + col + jj] = pl[jj];
                }
                if (u == 0 && lane < TS) g.part_R[q * FP3_TMAX + lane] = srs[lane];
                __syncwarp();
            }
        } else
        // warp item = (event group q, 32-column tile u) of [cl0, cl1).  The
        // group's events are loaded 32 at a time (one per lane) and
        // broadcast by shuffles; D loads are issued 8 events ahead.
        {
            A* sacc = reinterpret_cast<A*>(fp3_smem) + (size_t)warp * (FP3_TMAX * 32 + FP3_TMAX);
            A* srs = sacc + FP3_TMAX * 32;
            const int ncols = cl1 - cl0;
            const int ntile = (ncols + 31) / 32;
            const int ntl = max(ntile, 1);              // u == 0 items also carry the R deltas
            const int G = min(FP3_G, max(1, nwarps / ntl));   // event groups: about one item per warp
            const int items = G * ntl;
            for (int it = gwarp; it < items; it += nwarps) {
                const int q = it / ntl, u = it % ntl;
                const int col = u * 32 + lane;          // offset in [0, L)
                const bool act = col < ncols;
                const int64_t dcol = (int64_t)g.a + (act ? cl0 + col : 0);
                for (int t = 0; t < TS; ++t) sacc[t * 32 + lane] = 0;
                if (lane < FP3_TMAX) srs[lane] = 0;
                __syncwarp();
                A pl = 0;
                const int e0 = (int)((int64_t)q * m / G), e1 = (int)((int64_t)(q + 1) * m / G);
                for (int eb = e0; eb < e1; eb += 32) {
                    const int nb = min(32, e1 - eb);
                    int o_l = 0, to_l = 0, tn_l = 0;
                    T dno = 0, dso = 0, dnn = 0, dsn = 0;
                    if (lane < nb) {
                        const Fp3Chg<T> ch = fp3_ld_chg(&g.chg[eb + lane]);
                        o_l = ch.o;
                        to_l = __ldcg(&g.touched_map[ch.near_old]) - tb;   // slice-local, may be outside
                        tn_l = __ldcg(&g.touched_map[ch.near_new]) - tb;
                        dno = ch.dn_old; dso = ch.ds_old; dnn = ch.dn_new; dsn = ch.ds_new;
                    }
                    for (int e8 = 0; e8 < nb; e8 += FP3_EV) {
                        T x[FP3_EV];
#pragma unroll
                        for (int v8 = 0; v8 < FP3_EV; ++v8) {
                            const int oo = __shfl_sync(FULL, o_l, (e8 + v8) & 31);
                            x[v8] = g.D[(int64_t)oo * g.ld + dcol];
                        }
#pragma unroll
                        for (int v8 = 0; v8 < FP3_EV; ++v8) {
                            const int src = (e8 + v8) & 31;
                            const T a_dso = __shfl_sync(FULL, dso, src), a_dsn = __shfl_sync(FULL, dsn, src);
                            // a term is non-zero only where d < d_s (old or new): most (o, c)
                            // pairs miss both, and the warp skips them together
                            const bool any_hit = __any_sync(FULL, act && (x[v8] < a_dso || x[v8] < a_dsn));
                            if (!any_hit && u != 0) continue;  // u == 0 items also carry the R deltas
                            const T a_dno = __shfl_sync(FULL, dno, src), a_dnn = __shfl_sync(FULL, dnn, src);
                            const int a_to = __shfl_sync(FULL, to_l, src), a_tn = __shfl_sync(FULL, tn_l, src);
                            if (e8 + v8 < nb) {
                                A tpo, tao, tpn, tan_;
                                fp3_terms<T, A>(x[v8], a_dno, a_dso, tpo, tao);
                                fp3_terms<T, A>(x[v8], a_dnn, a_dsn, tpn, tan_);
                                if (tb == 0) pl += tpn - tpo;
                                const bool io = (unsigned)a_to < (unsigned)TS, in_ = (unsigned)a_tn < (unsigned)TS;
                                if (io) sacc[a_to * 32 + lane] -= tao;
                                if (in_) sacc[a_tn * 32 + lane] += tan_;
                                if (u == 0 && lane == 0) {
                                    if (io) srs[a_to] -= (A)a_dso - (A)a_dno;
                                    if (in_) srs[a_tn] += (A)a_dsn - (A)a_dnn;
                                }
                            }
                        }
                    }
                }
                __syncwarp();
                if (act) {
                    for (int t = 0; t < TS; ++t)
                        g.part_acc[((int64_t)q * FP3_TMAX + t) * g.L + col] = sacc[t * 32 + lane];
                    if (tb == 0) g.part_plus[(int64_t)q * g.L + col] = pl;
                }
                if (u == 0 && lane < TS) g.part_R[q * FP3_TMAX + lane] = srs[lane];
                __syncwarp();
            }
        }
        grid.sync();
        if (blockIdx.x == 0 && threadIdx.x == 0) { const unsigned long long tn = fp3_now(); ctl->tphase[5] += tn - tlast; tlast = tn; }
        {
            const int ncols = cl1 - cl0;
            const int G = wide ? min(FP3_G, max(1, nwarps / max((ncols + (int)((g.a + cl0) & 3) + 127) / 128, 1)))
                               : min(FP3_G, max(1, nwarps / max((ncols + 31) / 32, 1)));
            const int TSTR = wide ? FP3_TV : FP3_TMAX;           // part_acc slot stride per group
            // acc[slot_t][col] += sum_q part_acc[q][t][col]  (fixed order)
            for (int it = tid; it < TS * ncols; it += nth) {
                const int t = it / ncols, col = it % ncols;
                A s = 0;
#pragma unroll 8
                for (int q = 0; q < G; ++q) s += __ldcg(&g.part_acc[((int64_t)q * TSTR + t) * g.L + col]);
                A* dst = &g.acc[(int64_t)__ldcg(&g.touched[tb + t]) * g.ww + cl0 + col];
                *dst = __ldcg(dst) + s;
            }
            for (int col = tid; tb == 0 && col < ncols; col += nth) {
                A s = 0;
#pragma unroll 8
                for (int q = 0; q < G; ++q) s += __ldcg(&g.part_plus[(int64_t)q * g.L + col]);
                g.plus[cl0 + col] = __ldcg(&g.plus[cl0 + col]) + s;
            }
            // R_s += sum over changed objects of the change of (d_s - d_n) in slot s
            for (int t = tid; t < TS; t += nth) {
                A rs = 0;
                for (int q = 0; q < G; ++q) rs += __ldcg(&g.part_R[q * FP3_TMAX + t]);
                const int sl = __ldcg(&g.touched[tb + t]);
                g.R[sl] = __ldcg(&g.R[sl]) + rs;
            }
            if (tb + SL >= T_)
                for (int s = tid; s < k; s += nth) g.touched_flag[s] = 0;
        }
        grid.sync();
        }   // slices of touched slots
        if (blockIdx.x == 0 && threadIdx.x == 0) { const unsigned long long tn = fp3_now(); ctl->tphase[6] += tn - tlast; tlast = tn; }
        if (!GLOBAL) { p = j + 1; vhi = cl1; }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctl->status = status;
        ctl->p_end = p;
        ctl->swaps = swaps;
        ctl->pad[3] = converged ? 1 : 0;
        ctl->pad[4] = iters_done;
    }
}

}  // namespace km
