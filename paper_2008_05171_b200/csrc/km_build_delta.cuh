// km_build_delta.cuh -- incremental PAM BUILD (Alg.1; readings R3/R4).
//
// BUILD's step gain(c) = sum_o min(d(x_o, x_c) - d_nearest(o), 0) (medoids
// contribute 0 because their d_nearest is 0; the x_o = x_c term included,
// R3).  Recomputing it from scratch costs a full pass over D per step
// (k passes: 2 TB at C4).  But after a step only the objects whose
// d_nearest decreased change their term, so every step after the first full
// gain pass updates the stored gains exactly:
//   gain(c) += sum_{o changed} [min(d(o,c) - dn_new(o), 0) - min(d(o,c) - dn_old(o), 0)]
// reading only the ROWS of the changed objects (contiguous, coalesced).  Step
// i changes about n/i objects, so BUILD reads ~(2 + ln k) n^2 elements instead
// of k n^2 (exact on int64; fp64 re-association on the float path, R9).
//
//   k_build_dn_delta  gather d(., c*) into MC, new d_nearest, per-chunk
//                     counts of the changed objects
//   k_chunk_scan      exclusive scan of the chunk counts (one block)
//   k_changed_scatter changed objects in object order (deterministic) with
//                     their old / new d_nearest
//   k_build_delta_tma the TMA-ring stream over the listed rows (as
//                     k_build_tma), per (part, column) sums of the deltas
//   k_build_gain_combine  gains += parts (or = parts for the full pass),
//                     lexicographic min of (gain, c) over non-medoids
#pragma once
#include "km_kernels.cuh"

namespace km {

constexpr int BD_CHUNK_THREADS = 256;

// grid: B blocks, block b owns objects [b*chunk, min(n, (b+1)*chunk))
template <typename T, typename A>
__global__ void __launch_bounds__(BD_CHUNK_THREADS)
k_build_dn_delta(const T* __restrict__ D, int64_t ld, int n, int64_t col_begin, const Decision<A>* __restrict__ dec,
                 T* __restrict__ MC, const int* __restrict__ point_slot, T* __restrict__ dn,
                 T* __restrict__ dn_old, int* __restrict__ flag, int chunk, int* __restrict__ cnt,
                 int from_mc /* sharded: the column is already in MC (broadcast) */) {
    const int step = dec->slot;
    const int64_t c = dec->c;
    const int o0 = min(n, (int)blockIdx.x * chunk), o1 = min(n, o0 + chunk);
    int count = 0;
    for (int ob = o0; ob < o1; ob += blockDim.x) {
        const int o = ob + threadIdx.x;
        int f = 0;
        if (o < o1) {
            T x;
            if (from_mc) x = MC[(int64_t)step * n + o];
            else { x = D[(int64_t)o * ld + (c - col_begin)]; MC[(int64_t)step * n + o] = x; }
            const T old = dn[o];
            const T nw = point_slot[o] >= 0 ? (T)0 : (x < old ? x : old);
            if (nw != old) { f = 1; dn_old[o] = old; dn[o] = nw; }
            flag[o] = f;
        }
        count += __syncthreads_count(f);
    }
    if (threadIdx.x == 0) cnt[blockIdx.x] = count;
}

// exclusive scan of cnt[0..B) in place into off, total into *m (B <= 4096)
__global__ void k_chunk_scan(const int* __restrict__ cnt, int B, int* __restrict__ off, int* __restrict__ m) {
    __shared__ int sh[1024];
    const int per = (B + 1023) / 1024;
    const int a = threadIdx.x * per, z = min(B, a + per);
    int s = 0;
    for (int i = a; i < z; ++i) s += cnt[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int d = 1; d < 1024; d <<= 1) {
        const int v = threadIdx.x >= d ? sh[threadIdx.x - d] : 0;
        __syncthreads();
        sh[threadIdx.x] += v;
        __syncthreads();
    }
    int run = sh[threadIdx.x] - s;
    for (int i = a; i < z; ++i) { off[i] = run; run += cnt[i]; }
    if (threadIdx.x == 1023) *m = sh[1023];
}

template <typename T>
__global__ void __launch_bounds__(BD_CHUNK_THREADS)
k_changed_scatter(int n, const int* __restrict__ flag, const T* __restrict__ dn_old, const T* __restrict__ dn,
                  int chunk, const int* __restrict__ off, int* __restrict__ lst_o, T* __restrict__ lst_old,
                  T* __restrict__ lst_new) {
    __shared__ int wsum[BD_CHUNK_THREADS / 32];
    const int o0 = min(n, (int)blockIdx.x * chunk), o1 = min(n, o0 + chunk);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int run = off[blockIdx.x];
    for (int ob = o0; ob < o1; ob += blockDim.x) {
        const int o = ob + threadIdx.x;
        const int f = (o < o1) ? flag[o] : 0;
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (lane == 0) wsum[warp] = __popc(bal);
        __syncthreads();
        int base = 0, tot = 0;
        for (int w2 = 0; w2 < BD_CHUNK_THREADS / 32; ++w2) { if (w2 < warp) base += wsum[w2]; tot += wsum[w2]; }
        if (f) {
            const int pos = run + base + __popc(bal & ((1u << lane) - 1u));
            lst_o[pos] = o; lst_old[pos] = dn_old[o]; lst_new[pos] = dn[o];
        }
        run += tot;
        __syncthreads();
    }
}

// Parts of the delta stream for m listed rows: at least BD_ROWS_MIN rows per
// part (late steps list a few hundred rows: the 1-2 us fixed cost of a CTA,
// ring set-up and drain, then dominates), at most P.  A deterministic function
// of m, so the stream and the combine agree without a host round trip.
constexpr int BD_ROWS_MIN = 64;
__host__ __device__ inline int bd_parts(int m, int P) {
    const int p = (m + BD_ROWS_MIN - 1) / BD_ROWS_MIN;
    return p < 1 ? 1 : (p > P ? P : p);
}

// k_build_dn_delta + k_chunk_scan + k_changed_scatter as ONE cooperative
// kernel (one grid sync instead of two kernel boundaries): block b owns the
// objects [b*chunk, (b+1)*chunk); phase A as k_build_dn_delta, then every
// block sums the counts of the blocks before it (its list offset; block 0
// also writes the total *m) and places its changed objects in object order
// (the same list, bit for bit, as the three kernels).
template <typename T, typename A>
__global__ void __launch_bounds__(BD_CHUNK_THREADS)
k_build_changed(const T* __restrict__ D, int64_t ld, int n, int64_t col_begin, const Decision<A>* __restrict__ dec,
                T* __restrict__ MC, const int* __restrict__ point_slot, T* __restrict__ dn, T* __restrict__ dn_old,
                int* __restrict__ flag, int chunk, int* __restrict__ cnt, int* __restrict__ lst_o,
                T* __restrict__ lst_old, T* __restrict__ lst_new, int* __restrict__ m_out) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ int wsum[BD_CHUNK_THREADS / 32];
    __shared__ int s_off;
    const int step = dec->slot;
    const int64_t c = dec->c;
    const int o0 = min(n, (int)blockIdx.x * chunk), o1 = min(n, o0 + chunk);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int count = 0;
    for (int ob = o0; ob < o1; ob += blockDim.x) {
        const int o = ob + threadIdx.x;
        int f = 0;
        if (o < o1) {
            const T x = D[(int64_t)o * ld + (c - col_begin)];
            MC[(int64_t)step * n + o] = x;
            const T old = dn[o];
            const T nw = point_slot[o] >= 0 ? (T)0 : (x < old ? x : old);
            if (nw != old) { f = 1; dn_old[o] = old; dn[o] = nw; }
            flag[o] = f;
        }
        count += __syncthreads_count(f);
    }
    if (threadIdx.x == 0) cnt[blockIdx.x] = count;
    grid.sync();
    {
        // offset = sum of the counts of blocks 0..b-1 (fixed order: exact int)
        int s = 0, t = 0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
            const int v = __ldcg(&cnt[b]);
            if (b < (int)blockIdx.x) s += v;
            t += v;
        }
#pragma unroll
        for (int x = 16; x >= 1; x >>= 1) {
            s += __shfl_xor_sync(0xffffffffu, s, x);
            t += __shfl_xor_sync(0xffffffffu, t, x);
        }
        if (lane == 0) wsum[warp] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            int a = 0;
            for (int w2 = 0; w2 < BD_CHUNK_THREADS / 32; ++w2) a += wsum[w2];
            s_off = a;
        }
        __syncthreads();
        if (lane == 0) wsum[warp] = t;
        __syncthreads();
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            int a = 0;
            for (int w2 = 0; w2 < BD_CHUNK_THREADS / 32; ++w2) a += wsum[w2];
            *m_out = a;
        }
        __syncthreads();
    }
    int run = s_off;
    for (int ob = o0; ob < o1; ob += blockDim.x) {
        const int o = ob + threadIdx.x;
        const int f = (o < o1) ? flag[o] : 0;
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (lane == 0) wsum[warp] = __popc(bal);
        __syncthreads();
        int base = 0, tot = 0;
        for (int w2 = 0; w2 < BD_CHUNK_THREADS / 32; ++w2) { if (w2 < warp) base += wsum[w2]; tot += wsum[w2]; }
        if (f) {
            const int pos = run + base + __popc(bal & ((1u << lane) - 1u));
            lst_o[pos] = o; lst_old[pos] = dn_old[o]; lst_new[pos] = dn[o];
        }
        run += tot;
        __syncthreads();
    }
}

// The delta stream: as k_build_tma (MODE 1) over the rows lst_o[0..*m), with
// two thresholds per row.  Part q of Pe = bd_parts(m, P) covers list entries
// [q*m/Pe, (q+1)*m/Pe); CTAs with q >= Pe leave at once.
template <typename T, typename A, int NC, int RB, int S, int MINB>
__global__ void __launch_bounds__((NC + 1) * 32, MINB)
k_build_delta_tma(const T* __restrict__ D, int64_t ld, int w, int wpad, int P, const int* __restrict__ m_dev,
                  const int* __restrict__ lst_o, const T* __restrict__ lst_old, const T* __restrict__ lst_new,
                  A* __restrict__ out) {
    using C = SegCfg<T, NC, RB, S>;
    using V = typename Vec4<T>::type;
    extern __shared__ __align__(128) unsigned char smem[];
    T* sdata = reinterpret_cast<T*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::DATAB);
    uint64_t* empty = full + S;
    const int m = *m_dev;
    const int q = blockIdx.y;
    const int Pe = bd_parts(m, P);
    if (q >= Pe) return;
    const int64_t p0 = part_lo_uniform(q, m, Pe), p1 = part_lo_uniform(q + 1, m, Pe);   // a few changed rows: no tilt
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
        // the list entries in a 64-row register window, the next 32 loaded
        // 32 rows ahead (no dependent global load in front of a stage's copies)
        int64_t wb = p0;
        int o_c = wb + lane < p1 ? lst_o[wb + lane] : 0;
        int o_n = wb + 32 + lane < p1 ? lst_o[wb + 32 + lane] : 0;
        for (int st = 0; st < nstages; ++st) {
            const int s = st % S;
            if (st >= S) ptx::mbar_wait(&empty[s], ((st / S) & 1) ^ 1);
            const int64_t pr = p0 + (int64_t)st * RB;
            const int nb = (int)min((int64_t)RB, p1 - pr);
            const int li = (int)(pr - wb);
            const int src = (li + lane) & 31;
            const int oc = __shfl_sync(FULL, o_c, src), on = __shfl_sync(FULL, o_n, src);
            const int o = li + lane < 32 ? oc : on;
            if (lane == 0) ptx::mbar_expect_tx(&full[s], (uint32_t)nb * cbytes);
            __syncwarp();
            if (lane < nb)
                ptx::bulk_g2s(sdata + (size_t)(s * RB + lane) * C::COLS, D + (int64_t)o * ld + ctacol, cbytes,
                              &full[s], pol);
            if (pr + RB - wb >= 32) {            // the next stage starts in the next half
                wb += 32;
                o_c = o_n;
                o_n = wb + 32 + lane < p1 ? lst_o[wb + 32 + lane] : 0;
            }
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
        T vo[RB], vn[RB];
#pragma unroll
        for (int u = 0; u < RB; ++u) {
            vo[u] = (u < nb && active) ? lst_old[pr + u] : never_lt<T>();
            vn[u] = (u < nb && active) ? lst_new[pr + u] : never_lt<T>();
        }
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
        static_assert(RB == 4, "four rows per stage");
        unsigned mk = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j)       // a term can change only where d < d_nearest_old
            mk |= CmpLt<T>::any4(x[0][j], vo[0], x[1][j], vo[1], x[2][j], vo[2], x[3][j], vo[3]) << j;
        if (__reduce_or_sync(0xffffffffu, mk) == 0) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            A t[RB];
#pragma unroll
            for (int u = 0; u < RB; ++u) {
                const A xa = (A)x[u][j];
                const A to = (x[u][j] < vo[u]) ? xa - (A)vo[u] : (A)0;
                const A tn = (x[u][j] < vn[u]) ? xa - (A)vn[u] : (A)0;
                t[u] = tn - to;
            }
            acc[j] += (t[0] + t[1]) + (t[2] + t[3]);
        }
    }
    if (!active) return;
    const int64_t base = (int64_t)q * w;
    const uint64_t keep = ptx::policy_evict_last();   // read by the gain combine right after
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (cb + j < w) ptx::st_hint(&out[base + cb + j], acc[j], keep);
}

// gain[c] (+)= sum of the parts (m_dev: the delta stream's bd_parts(*m_dev, P)
// parts, else P); lexicographic min of (gain, c) over non-medoids.  With
// sel_step >= 0 (single GPU) the last block also takes the BUILD step itself
// (k_build_select's bookkeeping: medoid sel_step <- c*, TD += gain), after
// every block has read point_slot.
template <typename A>
__global__ void k_build_gain_combine(int w, int64_t col_begin, int P, const A* __restrict__ in, int accumulate,
                                     A* __restrict__ gain, int* __restrict__ point_slot, Rec<A>* partials,
                                     unsigned* counter, Rec<A>* out, const int* __restrict__ m_dev = nullptr,
                                     int sel_step = -1, A* __restrict__ td = nullptr, int* __restrict__ M = nullptr,
                                     Decision<A>* __restrict__ dec = nullptr) {
    const int cl = blockIdx.x * blockDim.x + threadIdx.x;
    const int Pe = m_dev ? bd_parts(*m_dev, P) : P;
    Rec<A> best = rec_none<A>();
    if (cl < w) {
        A s = 0;
        for (int q = 0; q < Pe; ++q) s += in[(int64_t)q * w + cl];
        const A g = accumulate ? gain[cl] + s : s;
        gain[cl] = g;
        const int64_t c = col_begin + cl;
        if (point_slot[c] < 0) { best.v = g; best.slot = 0; best.c = (int)c; }
    }
    Rec<A> m;
    if (grid_min_rec_last(best, partials, counter, out, &m) && sel_step >= 0 && threadIdx.x == 0)
        build_take(m, sel_step, td, M, point_slot, dec);
}

}  // namespace km
