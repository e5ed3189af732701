// km_fp2_owner.cuh -- the sequential phase of a column-sharded FastPAM2
// iteration (reading R6) with OWNER-SIDE re-evaluation.
//
// The gather form (kmedoids_fp2_shard_apply) all-gathers the column of every
// planned candidate (R x maxcnt x n elements per rank) and runs
// k_fp2_sequential redundantly on every rank.  Here the plan stays where the
// columns are: one sequential-phase *round* is
//
//   k_fp2_owned_eval   every rank re-evaluates, on the current (replicated)
//                      state, the unskipped plan entries from position r on
//                      whose candidate it owns, in plan order and in batches
//                      of FP2_B, and stops at its first improving one; it
//                      publishes (position, dTD, slot, c) and that column
//   all-gather         of the per-rank round buffers (caller; R x (32 + n T))
//   k_fp2_round_apply  every rank takes the smallest published position: it
//                      is exactly the entry the sequential loop applies next
//                      (every unskipped entry before it, on any rank, was
//                      evaluated on the same state and rejected); the swap is
//                      applied (M, TD, MC[i] <- column, incremental nearest /
//                      second, warp rescans) and the next round starts behind
//                      it.  No published position: the iteration is over.
//
// Round 0 applies plan entry 0 as is (it is FastPAM1's swap).  Rounds per
// iteration = applied swaps + 1, and each moves one column, instead of all m
// planned columns up front.
//
// The per-entry arithmetic and reduction tree are those of k_fp2_sequential
// (same grid, same per-thread object stride, same warp / block / grid
// sums), so a re-evaluated dTD has the same bits as on one GPU: the sharded
// trace equals the single-GPU trace (float path included).
#pragma once
#include "km_kernels.cuh"

namespace km {

// Header of a round buffer (16-byte aligned; the column follows at +32 bytes).
template <typename A>
struct alignas(16) Fp2RoundRec {
    int32_t pos;     // plan position of the published entry, INT_MAX = none
    int32_t pad;
    A v;             // its dTD on the round's state
    int32_t slot;
    int32_t c;
    int32_t pad2[2];
};
static_assert(sizeof(Fp2RoundRec<double>) == 32, "round header is 32 bytes");
static_assert(sizeof(Fp2RoundRec<long long>) == 32, "round header is 32 bytes");

template <typename T>
__host__ __device__ inline size_t fp2_round_stride(int64_t n) {
    return (32 + (size_t)n * sizeof(T) + 15) / 16 * 16;
}

// colsrc: this rank's planned candidate columns (kmedoids_fp2_shard_plan packs
// them: local column l at colsrc[l*n]); colidx[q] = owner * maxcnt + l for
// plan position q; r_dev: first plan position of the round.
template <typename T, typename A>
__global__ void __launch_bounds__(256)
k_fp2_owned_eval(const T* __restrict__ colsrc, const int* __restrict__ colidx, int me, int maxcnt, int n,
                 const int* __restrict__ order, const int* __restrict__ m_dev, const Rec<A>* __restrict__ best,
                 const int* __restrict__ point_slot, const int* __restrict__ near, const T* __restrict__ dn,
                 const T* __restrict__ ds, const A* __restrict__ td, A* __restrict__ partials,
                 const int* __restrict__ r_dev, int* __restrict__ rescan_count, unsigned char* __restrict__ out) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ A sred[8][FP2_B];
    __shared__ int s_r[FP2_B], s_c[FP2_B], s_i[FP2_B], s_l[FP2_B];
    __shared__ int s_nb, s_next, s_pick;
    __shared__ A s_v;
    const int nth = gridDim.x * blockDim.x;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    Fp2RoundRec<A>* hdr = reinterpret_cast<Fp2RoundRec<A>*>(out);
    T* ocol = reinterpret_cast<T*>(out + 32);
    const int m = *m_dev;
    const int r0 = *r_dev;
    if (tid == 0) *rescan_count = 0;             // consumed by the apply kernel that follows
    auto publish_none = [&]() {
        if (tid == 0) {
            Fp2RoundRec<A> h{};
            h.pos = INT_MAX; h.v = 0; h.slot = INT_MAX; h.c = INT_MAX;
            *hdr = h;
        }
    };
    auto publish = [&](int pos, A v, int i, int c, int l) {
        for (int o = tid; o < n; o += nth) ocol[o] = colsrc[(int64_t)l * n + o];
        if (tid == 0) {
            Fp2RoundRec<A> h{};
            h.pos = pos; h.v = v; h.slot = i; h.c = c;
            *hdr = h;
        }
    };
    if (r0 >= m) { publish_none(); return; }
    if (r0 == 0) {                               // FastPAM1's swap, applied as is (its owner publishes it)
        const int i = order[0];
        const Rec<A> b = best[i];
        const int ci = colidx[0];
        if (ci / maxcnt == me) publish(0, b.v, i, b.c, ci % maxcnt);
        else publish_none();
        return;
    }
    const A tdv = __ldcg(td);
    int q = r0, round = 0;
    while (true) {
        __syncthreads();
        if (wib == 0) {                          // warp 0 forms the batch (own entries only)
            int nb = 0;
            fp2_batch_window(order, best, point_slot, colidx, me, maxcnt, m, lane, q, nb, s_r, s_i, s_c, s_l);
            if (lane == 0) { s_nb = nb; s_next = q; }
        }
        __syncthreads();
        const int nb = s_nb;
        q = s_next;
        if (nb == 0) { publish_none(); return; }                // (uniform across blocks)
        // ---- the re-evaluations of the batch (k_fp2_sequential phase 1)
        A part[FP2_B];
#pragma unroll
        for (int b = 0; b < FP2_B; ++b) part[b] = 0;
        for (int o = tid; o < n; o += nth) {
            const T a = dn[o], bb = ds[o];
            const int no = near[o];
#pragma unroll
            for (int b = 0; b < FP2_B; ++b) {
                if (b >= nb) continue;
                const T x = colsrc[(int64_t)s_l[b] * n + o];
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
        A* pbuf = partials + (size_t)(round & 1) * gridDim.x * FP2_B;
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
        grid.sync();
        // ---- grid sums in k_fp2_sequential's order, first improving entry
        for (int b = wib; b < nb; b += (int)(blockDim.x >> 5)) {
            A t = 0;
            for (int qq = lane; qq < (int)gridDim.x; qq += 32) t += __ldcg(&pbuf[(size_t)qq * FP2_B + b]);
#pragma unroll
            for (int x = 16; x >= 1; x >>= 1) t += __shfl_xor_sync(FULL, t, x);
            if (lane == 0) sred[0][b] = t;
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
        __syncthreads();
        const int pick = s_pick;
        if (pick >= 0) { publish(s_r[pick], s_v, s_i[pick], s_c[pick], s_l[pick]); return; }
        ++round;
    }
}

// Every rank, after the all-gather of the R round buffers (stride bytes
// apart): apply the published entry with the smallest plan position (if any).
// state[0] = first plan position of the next round, state[1] = 1 while
// another round is needed.
template <typename T, typename A>
__global__ void __launch_bounds__(256)
k_fp2_round_apply(const unsigned char* __restrict__ recv, int nranks, size_t stride, int n, int k,
                  const int* __restrict__ m_dev, int* __restrict__ M, int* __restrict__ point_slot,
                  T* __restrict__ MC, int* __restrict__ near, int* __restrict__ sec, T* __restrict__ dn,
                  T* __restrict__ ds, A* __restrict__ td, Decision<A>* __restrict__ dec, Rec<A>* __restrict__ trace,
                  int trace_cap, int* __restrict__ rescan, int* __restrict__ rescan_count, int* __restrict__ state) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ int s_w;
    const int nth = gridDim.x * blockDim.x;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int gwarp = tid >> 5, nwarps = nth >> 5;
    if (threadIdx.x == 0) {
        int w = -1, bp = INT_MAX;
        for (int r = 0; r < nranks; ++r) {
            const int p = reinterpret_cast<const Fp2RoundRec<A>*>(recv + (size_t)r * stride)->pos;
            if (p < bp) { bp = p; w = r; }
        }
        s_w = w;
    }
    __syncthreads();
    const int w = s_w;
    if (w < 0) {                                 // nothing improves: the iteration is over
        if (tid == 0) { state[0] = *m_dev; state[1] = 0; }
        return;
    }
    const Fp2RoundRec<A> h = *reinterpret_cast<const Fp2RoundRec<A>*>(recv + (size_t)w * stride);
    const T* col = reinterpret_cast<const T*>(recv + (size_t)w * stride + 32);
    const int i = h.slot, c = h.c;
    KM_ASSERT(i >= 0 && i < k && c >= 0 && c < n);
    if (tid == 0) {
        const int old = M[i];
        M[i] = c;
        point_slot[old] = -1;
        point_slot[c] = i;
        *td = *td + h.v;
        const int sw = dec->swaps;
        if (sw < trace_cap) { Rec<A> t; t.v = h.v; t.slot = i; t.c = c; trace[sw] = t; }
        dec->swaps = sw + 1;
        dec->apply = 1;
        dec->slot = i;
        dec->c = c;
        dec->dtd = h.v;
        dec->old_m = old;
        state[0] = h.pos + 1;
        state[1] = h.pos + 1 < *m_dev ? 1 : 0;
    }
    // MC[i] <- column c, incremental nearest/second; objects whose nearest /
    // second was slot i listed for a rescan (k_fp2_sequential phase 3)
    for (int o = tid; o < n; o += nth) {
        const T x = col[o];
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
    // (d, j) lexicographic top-2 of the listed objects, one warp each (phase 4)
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
}

}  // namespace km
