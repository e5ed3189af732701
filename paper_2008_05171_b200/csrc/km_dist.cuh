// km_dist.cuh -- dissimilarity-matrix materialisation (
// PAPER P:272-278 "a dissimilarity matrix D ... is computed in advance",
// computing it dominates FasterPAM's time on MNIST).
//
// Writes the column slab [c0, c1) of all n rows of D, row stride ld, i.e.
// directly in the layout a (possibly sharded) kmedoids handle borrows.
//
//   L2 (float32): d(x_i, x_j) = sqrt(max(0, |x_i|^2 + |x_j|^2 - 2 <x_i, x_j>)).
//     The inner products are a contraction and run on the 5th-generation
//     tensor cores: tcgen05.mma kind::tf32, M = 128 rows x N = 128 columns
//     per tile, accumulator in TMEM, operands in shared memory (K-major,
//     no-swizzle core matrices).  f32 accuracy from tf32 inputs by the
//     3-term split x = hi + lo (hi = tf32(x), lo = tf32(x - hi)):
//     <x,y> ~ hi.hi + hi.lo + lo.hi, fp32 accumulation (the dropped lo.lo
//     term is < 2^-22 |x||y|).  Norms are exact fp64 sums rounded to f32.
//     The points are centred first (x - mean; k_dist_mean), so the error
//     follows |x - mu|^2 + |y - mu|^2 instead of |x|^2 + |y|^2.
//     The diagonal is set to 0 exactly (d(x, x) = 0).
//   L1 (uint32): d(x_i, x_j) = sum_t |x_it - x_jt| on integer coordinates
//     (the C1/C5 "L1 of round(100 x)" dissimilarities), exact, CUDA cores
//     (an absolute-difference sum is not a contraction).
#pragma once
#include <cuda.h>
#include "km_kernels.cuh"

namespace km {

constexpr int DT_M = 128;       // rows per tile (TMEM lanes)
constexpr int DT_N = 128;       // columns per tile (TMEM columns, fp32)

__device__ __forceinline__ uint32_t dt_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ float dt_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// Shared-memory matrix descriptor, K-major, no swizzle (canonical layout
// ((8, m), (T, 2)) : ((1T, SBO), (1, LBO)) in 16-byte units): core matrices of
// 8 rows x 16 bytes; LBO = byte distance between the two K-adjacent core
// matrices of one instruction, SBO = byte distance between 8-row groups.
__device__ __forceinline__ uint64_t dt_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;          // descriptor version (sm_100)
    // base offset 0, LBO mode 0, layout type 0 = SWIZZLE_NONE (bits 61-63)
    return d;
}

// Instruction descriptor: D f32, A/B tf32, both K-major, M x N.
__host__ __device__ constexpr uint32_t dt_idesc(int M, int N) {
    return (1u << 4)                       // c_format = F32
         | (2u << 7)                       // a_format = TF32
         | (2u << 10)                      // b_format = TF32
         | ((uint32_t)(N >> 3) << 17)      // n_dim
         | ((uint32_t)(M >> 4) << 24);     // m_dim
}

__device__ __forceinline__ void dt_mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
        :: "r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

// Element (r, k) of a K-major no-swizzle tile with kc = Kpad/4 chunks of 4
// tf32 per 8-row group: core matrix (r/8, k/4), 8 rows x 4 floats each.
__device__ __forceinline__ int dt_off(int r, int k, int kc) {
    return (((r >> 3) * kc + (k >> 2)) << 5) + ((r & 7) << 2) + (k & 3);
}

// Centering (round 2): distances are translation invariant, while the
// error of the norm expansion |x|^2 + |y|^2 - 2<x,y> scales with |x|^2 +
// |y|^2.  The operands are therefore x - mu, mu = the per-dimension mean of
// all n points (fp64 sums in a fixed order, rounded to f32; any mu is exact
// in the mathematics, the rounding of x - mu costs 2^-24 |x - mu|).
// Two launches, fixed order: block b of DM_BLOCKS sums rows [b n / B,
// (b + 1) n / B) (thread (ty, tx): dimension tx, rows ty, ty + lanes, ...;
// coalesced), its lanes combined in ty order -> part[b][t]; then one thread
// per dimension adds the B partials in block order.  (Round 2's first form,
// one block per dimension with strided loads, took 40-90 us at C3 / C4.)
constexpr int DM_BLOCKS = 256;
__global__ void __launch_bounds__(256) k_dist_mean_part(const float* __restrict__ X, int n, int d,
                                                        double* __restrict__ part) {
    __shared__ double ws[256];
    const int lanes = (int)blockDim.x / d;
    const int tx = threadIdx.x % d, ty = threadIdx.x / d;
    const int64_t r0 = (int64_t)blockIdx.x * n / gridDim.x, r1 = (int64_t)(blockIdx.x + 1) * n / gridDim.x;
    double s = 0;
    if (ty < lanes) {
#pragma unroll 4
        for (int64_t i = r0 + ty; i < r1; i += lanes) s += (double)X[i * d + tx];
    }
    ws[threadIdx.x] = s;
    __syncthreads();
    if ((int)threadIdx.x < d) {
        double a = 0;
        for (int y = 0; y < lanes; ++y) a += ws[y * d + threadIdx.x];
        part[(int64_t)blockIdx.x * d + threadIdx.x] = a;
    }
}
__global__ void k_dist_mean_fin(const double* __restrict__ part, int nb, int n, int d, float* __restrict__ mu) {
    const int t = threadIdx.x;
    if (t >= d) return;
    double a = 0;
#pragma unroll 8
    for (int b = 0; b < nb; ++b) a += part[(int64_t)b * d + t];
    mu[t] = (float)(a / (double)n);
}

__device__ __forceinline__ float dt_centered(const float* X, const float* mu, int64_t j, int d, int k) {
    const float v = X[j * d + k];
    return mu ? v - mu[k] : v;
}

// fp64 squared norms of the (centred) points rounded to f32: nrm[i] = |x_i - mu|^2
__global__ void k_dist_norms(const float* __restrict__ X, const float* __restrict__ mu, int n, int d,
                             float* __restrict__ nrm) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0;
    for (int t = 0; t < d; ++t) { const double v = dt_centered(X, mu, i, d, t); s += v * v; }
    nrm[i] = (float)s;
}

// Operand pre-pass: rows [r0, r1) of X as 128-row tiles in exactly the
// shared-memory image the MMA reads -- [hi core matrices (128 x dpad)][lo
// core matrices][128 squared norms] -- so that one TMA bulk copy moves a
// whole tile.  Rows beyond r1 and columns beyond d are zero.
__host__ __device__ inline int64_t dt_tile_floats(int dpad) { return 2LL * DT_M * dpad + DT_M; }

__global__ void k_dist_pack(const float* __restrict__ X, const float* __restrict__ mu, const float* __restrict__ nrm,
                            int d, int dpad, int64_t r0, int64_t r1, float* __restrict__ out) {
    const int kc = dpad / 4;
    const int64_t tile = blockIdx.x;
    float* o = out + tile * dt_tile_floats(dpad);
    for (int idx = threadIdx.x; idx < DT_M * dpad; idx += blockDim.x) {
        const int r = idx / dpad, k = idx - r * dpad;
        const int64_t j = r0 + tile * DT_M + r;
        const float v = (j < r1 && k < d) ? dt_centered(X, mu, j, d, k) : 0.f;
        const float hi = dt_tf32(v);
        o[dt_off(r, k, kc)] = hi;
        o[DT_M * dpad + dt_off(r, k, kc)] = dt_tf32(v - hi);
    }
    for (int r = threadIdx.x; r < DT_M; r += blockDim.x) {
        const int64_t j = r0 + tile * DT_M + r;
        o[2 * DT_M * dpad + r] = j < r1 ? nrm[j] : 0.f;
    }
}

// Persistent CTAs (one per SM, 8 warps) over work items (128-row tile,
// range of 128-column tiles).  Per column tile: one thread issues
// 3 * dpad/8 tcgen05.mma (hi.hi, hi.lo, lo.hi) into a TMEM accumulator
// (128 lanes x 128 fp32 columns) and commits to an mbarrier; as soon as the
// MMAs are done the next B tile is fetched by a TMA bulk copy (it lands
// while the epilogue runs); the 8 warps read the accumulator (warp w: lanes
// 32(w%4).., columns 64(w/4)..), form the distances and stage the tile in
// shared memory; one thread writes it with 128 TMA bulk copies (a 512-byte
// row segment each) that overlap the next tile (two staging buffers when
// they fit).  Requires d <= 64 (dpad = roundup(d, 8)).
constexpr int DT_WARPS = 8;
constexpr int DT_THREADS = DT_WARPS * 32;
constexpr int DT_SROW = DT_N + 4;                   // staging row stride (floats): 528 B, 4-way bank spread

__host__ __device__ inline size_t dt_smem_bytes(int dpad, int nstage) {
    return (size_t)2 * dt_tile_floats(dpad) * sizeof(float) + (size_t)nstage * DT_M * DT_SROW * sizeof(float);
}

__device__ __forceinline__ void dt_bulk_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(dt_smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(dt_smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(dt_smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void dt_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile("{\n\t.reg .pred p;\n\t"
                     "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}\n"
                     : "=r"(done) : "r"(dt_smem_u32(bar)), "r"(phase) : "memory");
    }
}

__global__ void __launch_bounds__(DT_THREADS, 1)
k_dist_l2_tc(const float* __restrict__ PA, const float* __restrict__ PB, int n, int dpad, int nstage, int nsplit,
             float* __restrict__ D, int64_t ld, int64_t c0, int64_t c1) {
    extern __shared__ __align__(1024) unsigned char dsm[];
    const int64_t TF = dt_tile_floats(dpad);
    const uint32_t tbytes = (uint32_t)(TF * sizeof(float));
    float* sA = reinterpret_cast<float*>(dsm);
    float* sB = sA + TF;
    float* stage0 = sB + TF;                            // nstage x [128][DT_SROW]
    const float* sny = sB + 2 * DT_M * dpad;            // |x_j|^2 of the B tile
    __shared__ __align__(8) uint64_t bar_mma, bar_a, bar_b;
    __shared__ uint32_t tmem_base_s;
    __shared__ float sny_keep[DT_N];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int q = warp & 3, half = warp >> 2;           // TMEM lane quarter, column half

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(dt_smem_u32(&tmem_base_s)), "n"(DT_N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(dt_smem_u32(&bar_mma)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(dt_smem_u32(&bar_a)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(dt_smem_u32(&bar_b)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base_s;
    const uint32_t idesc = dt_idesc(DT_M, DT_N);
    const uint32_t lbo = 128, sbo = (uint32_t)(dpad / 4) * 128;
    const int64_t ntile_c = (c1 - c0 + DT_N - 1) / DT_N;
    const int64_t nm = (n + DT_M - 1) / DT_M;
    const int64_t items = nm * nsplit;
    uint32_t ph_mma = 0, ph_a = 0, ph_b = 0;
    int64_t tcount = 0;                                  // tiles done by this CTA (staging rotation)

    for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
        const int64_t mt = item / nsplit;
        const int m0 = (int)(mt * DT_M);
        const int sp = (int)(item % nsplit);
        const int64_t t0 = ntile_c * sp / nsplit, t1 = ntile_c * (sp + 1) / nsplit;
        if (t0 >= t1) continue;
        if (tid == 0) {                                  // A tile and the first B tile of the item
            dt_bulk_load(sA, PA + mt * TF, tbytes, &bar_a);
            dt_bulk_load(sB, PB + t0 * TF, tbytes, &bar_b);
        }
        dt_wait(&bar_a, ph_a); ph_a ^= 1;
        const int rowq = m0 + q * 32 + lane;             // this thread's row (TMEM lane q*32+lane)
        const float nx = sA[2 * DT_M * dpad + q * 32 + lane];
        for (int64_t tc = t0; tc < t1; ++tc, ++tcount) {
            const int64_t n0 = c0 + tc * DT_N;
            if (tid == 0) {
                dt_wait(&bar_b, ph_b);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t sa_hi = dt_smem_u32(sA), sa_lo = sa_hi + DT_M * dpad * 4;
                const uint32_t sb_hi = dt_smem_u32(sB), sb_lo = sb_hi + DT_N * dpad * 4;
                for (int s = 0; s < dpad / 8; ++s) {
                    const uint32_t ko = (uint32_t)s * 2 * 128;   // two 16-byte K chunks per instruction
                    dt_mma_tf32(tmem, dt_desc(sa_hi + ko, lbo, sbo), dt_desc(sb_hi + ko, lbo, sbo), idesc, s > 0);
                    dt_mma_tf32(tmem, dt_desc(sa_hi + ko, lbo, sbo), dt_desc(sb_lo + ko, lbo, sbo), idesc, 1);
                    dt_mma_tf32(tmem, dt_desc(sa_lo + ko, lbo, sbo), dt_desc(sb_hi + ko, lbo, sbo), idesc, 1);
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                             :: "r"(dt_smem_u32(&bar_mma)) : "memory");
            }
            ph_b ^= 1;
            dt_wait(&bar_mma, ph_mma); ph_mma ^= 1;      // accumulator ready, B consumed
            asm volatile("tcgen05.fence::after_thread_sync;");
            // the B norms are needed by the epilogue: copy them out before B is refilled
            if (tid < DT_N) sny_keep[tid] = sny[tid];
            __syncthreads();
            if (tid == 0 && tc + 1 < t1) dt_bulk_load(sB, PB + (tc + 1) * TF, tbytes, &bar_b);   // lands during the epilogue
            if (warp == 0) {
                // the staging buffer of this tile was last read by the bulk
                // stores of tile tcount - nstage (issued by the lanes of warp 0)
                if (nstage == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            __syncthreads();
            float* stg = stage0 + (size_t)(tcount % nstage) * DT_M * DT_SROW;
#pragma unroll 1
            for (int cc = 0; cc < 2; ++cc) {
                const int col0 = half * 64 + cc * 32;
                uint32_t v[32];
                const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)col0;
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
                    "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                      "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                      "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
                      "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
                      "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                float* srow = stg + (size_t)(q * 32 + lane) * DT_SROW + col0;
#pragma unroll
                for (int j = 0; j < 32; j += 4) {
                    float o4[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const float dot = __uint_as_float(v[j + u]);
                        const float d2 = fmaf(-2.f, dot, nx + sny_keep[col0 + j + u]);
                        o4[u] = (n0 + col0 + j + u == rowq) ? 0.f : sqrtf(fmaxf(d2, 0.f));
                    }
                    *reinterpret_cast<float4*>(srow + j) = make_float4(o4[0], o4[1], o4[2], o4[3]);
                }
            }
            // staging -> global: 128 row segments by bulk copies (async proxy)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncthreads();                             // also: TMEM free for the next MMA
            const int wcols = (int)((c1 - n0) < (int64_t)DT_N ? (c1 - n0) : (int64_t)DT_N);
            if ((wcols & 3) == 0) {
                if (warp == 0) {                         // 4 row copies per lane of warp 0
                    const uint32_t bytes = (uint32_t)wcols * 4;
                    for (int r = lane; r < DT_M && m0 + r < n; r += 32) {
                        float* g = D + (int64_t)(m0 + r) * ld + (n0 - c0);
                        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                                     :: "l"(g), "r"(dt_smem_u32(stg + (size_t)r * DT_SROW)), "r"(bytes) : "memory");
                    }
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
            } else {                                     // ragged last tile: plain stores
                for (int idx = tid; idx < DT_M * wcols; idx += DT_THREADS) {
                    const int r = idx / wcols, cidx = idx - r * wcols;
                    if (m0 + r < n) D[(int64_t)(m0 + r) * ld + (n0 - c0) + cidx] = stg[(size_t)r * DT_SROW + cidx];
                }
                __syncthreads();
            }
        }
    }
    if (warp == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "n"(DT_N));
}

// ---------------------------------------------------------------------------
// Warp-specialised L2 kernel (default).  9 warps per CTA, one CTA per SM,
// persistent over (128-row tile, column range) items:
//   warp 8, one lane: TMA bulk loads of the packed A / B operand tiles (B in a
//     2-stage ring), tcgen05.mma (3 * dpad/8 per tile) into one of TWO TMEM
//     accumulators (2 x 128 columns), tcgen05.commit to the epilogue's
//     "full" barrier and to the B stage's "empty" barrier;
//   warps 0-7: epilogue -- tcgen05.ld of 32 lanes x 64 columns each, release
//     the accumulator, d = sqrt(max(0, |x|^2 + |y|^2 - 2 dot)) (norms from
//     global memory, L1/L2 resident), 128B-swizzled staging, and four 2-D TMA
//     tensor stores (32 x 128 boxes) per tile issued by one lane; the
//     stores run while the next tile is computed.
// The MMA of tile t+1 overlaps the epilogue of tile t (TMEM double buffer);
// the B tile of t+2 is fetched as soon as the MMAs of t are done.  Edges
// (rows beyond n, columns beyond the slab) are clipped by the tensor store.
// ---------------------------------------------------------------------------
constexpr unsigned FULL_MASK_DW = 0xffffffffu;
constexpr int DW_EPI_WARPS = 16;
// TMEM accumulators (128 columns each; 4 = all 512 columns): the MMAs run up
// to DW_NACC - 1 tiles ahead of the epilogue
constexpr int DW_NACC = 4;                     // 4 per TMEM lane quarter
constexpr int DW_CPW = DT_N / (DW_EPI_WARPS / 4);    // accumulator columns per epilogue warp
constexpr int DW_THREADS = (DW_EPI_WARPS + 1) * 32;

__host__ __device__ inline int64_t dw_tile_floats(int dpad) { return 2LL * DT_M * dpad; }
// raw (uncentred) points of a 128-row / 128-column tile for the exact
// recomputation, rows padded to dpad + 4 floats (4-way bank spread of the
// per-lane 16-byte shared-memory loads)
__host__ __device__ inline int dw_raw_stride(int dpad) { return dpad + 4; }
__host__ __device__ inline int64_t dw_raw_floats(int dpad) { return (int64_t)DT_M * dw_raw_stride(dpad); }
__host__ __device__ inline size_t dw_smem_bytes(int dpad, int nstage) {
    // A + 2 B stages + nstage x 64 KB staging (4 boxes of 128 rows x 128 B), 1 KB alignment slack
    return (size_t)3 * dw_tile_floats(dpad) * sizeof(float) + (size_t)nstage * 4 * DT_M * 128 + 1024;
}

// hi / lo core matrices of rows [r0, r1), 128-row tiles (no norms appended)
__global__ void k_dist_pack2(const float* __restrict__ X, const float* __restrict__ mu, int d, int dpad, int64_t r0,
                             int64_t r1, float* __restrict__ out) {
    const int kc = dpad / 4;
    const int64_t tile = blockIdx.x;
    float* o = out + tile * dw_tile_floats(dpad);
    for (int idx = threadIdx.x; idx < DT_M * dpad; idx += blockDim.x) {
        const int r = idx / dpad, k = idx - r * dpad;
        const int64_t j = r0 + tile * DT_M + r;
        const float v = (j < r1 && k < d) ? dt_centered(X, mu, j, d, k) : 0.f;
        const float hi = dt_tf32(v);
        o[dt_off(r, k, kc)] = hi;
        o[DT_M * dpad + dt_off(r, k, kc)] = dt_tf32(v - hi);
    }
}

// raw points of rows [r0, r1) in 128-row tiles [tile][row][dpad + 4] (zero padded)
__global__ void k_dist_pack_raw(const float* __restrict__ X, int d, int dpad, int64_t r0, int64_t r1,
                                float* __restrict__ out) {
    const int rs = dw_raw_stride(dpad);
    const int64_t tile = blockIdx.x;
    float* o = out + tile * dw_raw_floats(dpad);
    for (int idx = threadIdx.x; idx < DT_M * rs; idx += blockDim.x) {
        const int r = idx / rs, k = idx - r * rs;
        const int64_t j = r0 + tile * DT_M + r;
        o[idx] = (j < r1 && k < d) ? X[j * d + k] : 0.f;
    }
}

__device__ __forceinline__ void dw_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(dt_smem_u32(bar)) : "memory");
}

__device__ __forceinline__ float dw_sqrt(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Exact value of a pair whose norm expansion cancels: d^2 = sum_t (x_t - y_t)^2
// over the raw points (f32 differences, two fp32 fused accumulators over the
// even / odd 4-blocks of t, then added: relative error <= (d + 2) 2^-24 on
// d^2), correctly rounded sqrt.  The points come from the padded raw tiles
// (L1 / L2 resident); all 16-byte loads of a pair are issued at once.
template <int DP>
__device__ __forceinline__ float dw_exact_t(const float* xr, const float* yc) {
    float4 a[DP / 4], c[DP / 4];
#pragma unroll
    for (int i = 0; i < DP / 4; ++i) {
        a[i] = __ldg(reinterpret_cast<const float4*>(xr) + i);
        c[i] = __ldg(reinterpret_cast<const float4*>(yc) + i);
    }
    float acc[2] = {0.f, 0.f};
#pragma unroll
    for (int i = 0; i < DP / 4; ++i) {
        const float e0 = a[i].x - c[i].x, e1 = a[i].y - c[i].y, e2 = a[i].z - c[i].z, e3 = a[i].w - c[i].w;
        float& r = acc[i & 1];
        r = fmaf(e0, e0, r); r = fmaf(e1, e1, r); r = fmaf(e2, e2, r); r = fmaf(e3, e3, r);
    }
    return __fsqrt_rn(acc[0] + acc[1]);
}
__device__ __forceinline__ float dw_exact(const float* xr, const float* yc, int dpad) {   // zero padding adds 0
    switch (dpad) {
        case 8: return dw_exact_t<8>(xr, yc);
        case 16: return dw_exact_t<16>(xr, yc);
        case 24: return dw_exact_t<24>(xr, yc);
        case 32: return dw_exact_t<32>(xr, yc);
        case 40: return dw_exact_t<40>(xr, yc);
        case 48: return dw_exact_t<48>(xr, yc);
        case 56: return dw_exact_t<56>(xr, yc);
        default: return dw_exact_t<64>(xr, yc);
    }
}

__global__ void __launch_bounds__(DW_THREADS, 1)
k_dist_l2_ws(const __grid_constant__ CUtensorMap tmap, const float* __restrict__ PA, const float* __restrict__ PB,
             const float* __restrict__ nrm, int n, int dpad, int nsplit, int nstage, int64_t c0, int64_t c1,
             const float* __restrict__ RA, const float* __restrict__ RB, float tau) {
    extern __shared__ __align__(1024) unsigned char dsm_raw[];
    // 1 KB alignment for the 128B-swizzled staging boxes
    unsigned char* dsm = dsm_raw + ((1024 - (dt_smem_u32(dsm_raw) & 1023)) & 1023);
    const int64_t TF = dw_tile_floats(dpad);
    const uint32_t tbytes = (uint32_t)(TF * sizeof(float));
    unsigned char* stage0 = dsm;                         // nstage x 4 boxes x 16 KB (1 KB aligned)
    float* sA = reinterpret_cast<float*>(dsm + (size_t)nstage * 4 * DT_M * 128);
    float* sB0 = sA + TF;                                // 2 stages
    // exact fix-up (tau > 0): raw point tiles RA (rows) / RB (slab columns)
    const bool fix = tau > 0.f;
    const int64_t RF = dw_raw_floats(dpad);
    const int rst = dw_raw_stride(dpad);
    __shared__ __align__(8) uint64_t bar_a, bar_bfull[2], bar_bempty[2], bar_tfull[DW_NACC], bar_tempty[DW_NACC];
    __shared__ uint32_t tmem_base_s;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    if (warp == DW_EPI_WARPS) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(dt_smem_u32(&tmem_base_s)), "n"(DW_NACC * DT_N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(dt_smem_u32(&bar_a)));
        for (int i = 0; i < 2; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(dt_smem_u32(&bar_bfull[i])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(dt_smem_u32(&bar_bempty[i])));
        }
        for (int i = 0; i < DW_NACC; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(dt_smem_u32(&bar_tfull[i])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(dt_smem_u32(&bar_tempty[i])), "r"(DW_EPI_WARPS));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base_s;
    const int64_t ntile_c = (c1 - c0 + DT_N - 1) / DT_N;
    const int64_t nm = (n + DT_M - 1) / DT_M;
    const int64_t items = nm * nsplit;

    if (warp == DW_EPI_WARPS) {
        // ====================== TMA + MMA (one lane) ======================
        if (lane == 0) {
            const uint32_t idesc = dt_idesc(DT_M, DT_N);
            const uint32_t lbo = 128, sbo = (uint32_t)(dpad / 4) * 128;
            uint32_t ph_a = 0, ph_bf[2] = {0, 0}, ph_be[2] = {0, 0}, ph_te[DW_NACC] = {};
            int64_t t = 0;                               // tiles issued by this CTA
            bool pending[2] = {false, false};            // B stage has an MMA commit not yet waited for
            for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
                const int64_t mt = item / nsplit;
                const int sp = (int)(item % nsplit);
                const int64_t t0 = ntile_c * sp / nsplit, t1 = ntile_c * (sp + 1) / nsplit;
                if (t0 >= t1) continue;
                // the A tile is rewritten: every MMA issued so far must be complete
                for (int s = 0; s < 2; ++s)
                    if (pending[s]) { dt_wait(&bar_bempty[s], ph_be[s]); ph_be[s] ^= 1; pending[s] = false; }
                dt_bulk_load(sA, PA + mt * TF, tbytes, &bar_a);
                // the first two B tiles of the item
                for (int64_t k = 0; k < 2 && t0 + k < t1; ++k) {
                    const int s = (int)((t + k) & 1);
                    dt_bulk_load(sB0 + s * TF, PB + (t0 + k) * TF, tbytes, &bar_bfull[s]);
                }
                dt_wait(&bar_a, ph_a); ph_a ^= 1;
                for (int64_t tc = t0; tc < t1; ++tc, ++t) {
                    const int s = (int)(t & 1);                      // B stage
                    const int sa = (int)(t % DW_NACC);               // TMEM accumulator
                    dt_wait(&bar_bfull[s], ph_bf[s]); ph_bf[s] ^= 1;
                    if (t >= DW_NACC) { dt_wait(&bar_tempty[sa], ph_te[sa]); ph_te[sa] ^= 1; }   // accumulator drained
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t sa_hi = dt_smem_u32(sA), sa_lo = sa_hi + DT_M * dpad * 4;
                    const uint32_t sb_hi = dt_smem_u32(sB0 + s * TF), sb_lo = sb_hi + DT_N * dpad * 4;
                    const uint32_t acc = tmem + (uint32_t)(sa * DT_N);
                    for (int kk = 0; kk < dpad / 8; ++kk) {
                        const uint32_t ko = (uint32_t)kk * 2 * 128;
                        dt_mma_tf32(acc, dt_desc(sa_hi + ko, lbo, sbo), dt_desc(sb_hi + ko, lbo, sbo), idesc, kk > 0);
                        dt_mma_tf32(acc, dt_desc(sa_hi + ko, lbo, sbo), dt_desc(sb_lo + ko, lbo, sbo), idesc, 1);
                        dt_mma_tf32(acc, dt_desc(sa_lo + ko, lbo, sbo), dt_desc(sb_hi + ko, lbo, sbo), idesc, 1);
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                                 :: "r"(dt_smem_u32(&bar_tfull[sa])) : "memory");
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                                 :: "r"(dt_smem_u32(&bar_bempty[s])) : "memory");
                    pending[s] = true;
                    // B stage s is refilled with tile tc + 2 once these MMAs are done
                    if (tc + 2 < t1) {
                        dt_wait(&bar_bempty[s], ph_be[s]); ph_be[s] ^= 1; pending[s] = false;
                        dt_bulk_load(sB0 + s * TF, PB + (tc + 2) * TF, tbytes, &bar_bfull[s]);
                    }
                }
            }
            for (int s = 0; s < 2; ++s)
                if (pending[s]) { dt_wait(&bar_bempty[s], ph_be[s]); ph_be[s] ^= 1; }
        }
    } else {
        // ====================== epilogue warps 0-15 ======================
        const int q = warp & 3, part = warp >> 2;       // TMEM lane quarter, column part
        uint32_t ph_tf[DW_NACC] = {};
        int64_t t = 0;
        for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
            const int64_t mt = item / nsplit;
            const int m0 = (int)(mt * DT_M);
            const int sp = (int)(item % nsplit);
            const int64_t t0 = ntile_c * sp / nsplit, t1 = ntile_c * (sp + 1) / nsplit;
            if (t0 >= t1) continue;
            const int row = m0 + q * 32 + lane;
            const float nx = row < n ? nrm[row] : 0.f;
            for (int64_t tc = t0; tc < t1; ++tc, ++t) {
                const int s = (int)(t % DW_NACC);                   // TMEM accumulator
                const int64_t n0 = c0 + tc * DT_N;
                const int64_t cb = n0 + part * DW_CPW;
                dt_wait(&bar_tfull[s], ph_tf[s]); ph_tf[s] ^= 1;
                asm volatile("tcgen05.fence::after_thread_sync;");
                uint32_t v[DW_CPW];
#pragma unroll
                for (int ch = 0; ch < DW_CPW / 32; ++ch) {
                    const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(s * DT_N + part * DW_CPW + ch * 32);
                    uint32_t* w = v + ch * 32;
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
                        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                        : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
                          "=r"(w[7]), "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]),
                          "=r"(w[14]), "=r"(w[15]), "=r"(w[16]), "=r"(w[17]), "=r"(w[18]), "=r"(w[19]), "=r"(w[20]),
                          "=r"(w[21]), "=r"(w[22]), "=r"(w[23]), "=r"(w[24]), "=r"(w[25]), "=r"(w[26]), "=r"(w[27]),
                          "=r"(w[28]), "=r"(w[29]), "=r"(w[30]), "=r"(w[31])
                        : "r"(taddr));
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) dw_arrive(&bar_tempty[s]);  // accumulator s may be overwritten
                // distances (norms of the columns: same addresses across the warp -> broadcast)
                // column norms: 16-byte loads with no per-element bounds in whole,
                // aligned parts (all but the slab's last part when c0 % 4 == 0)
                const bool whole = (cb + DW_CPW <= c1) && ((cb & 3) == 0);
                uint32_t fl = 0;                             // columns of this lane's row to recompute
#pragma unroll
                for (int j = 0; j < DW_CPW; j += 4) {
                    float4 ny4;
                    if (whole) ny4 = __ldg(reinterpret_cast<const float4*>(nrm + cb + j));
                    else {
                        ny4.x = cb + j < c1 ? nrm[cb + j] : 0.f;
                        ny4.y = cb + j + 1 < c1 ? nrm[cb + j + 1] : 0.f;
                        ny4.z = cb + j + 2 < c1 ? nrm[cb + j + 2] : 0.f;
                        ny4.w = cb + j + 3 < c1 ? nrm[cb + j + 3] : 0.f;
                    }
                    const float ny[4] = {ny4.x, ny4.y, ny4.z, ny4.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const float s2 = nx + ny[u];
                        const float d2 = fmaf(-2.f, __uint_as_float(v[j + u]), s2);
                        // cancellation: d^2 small against |x|^2 + |y|^2 -> recomputed below
                        if (d2 < tau * s2) fl |= 1u << (j + u);
                        v[j + u] = __float_as_uint(dw_sqrt(fmaxf(d2, 0.f)));
                    }
                }
                const int64_t dj = (int64_t)row - cb;       // this lane's diagonal column, if in its part
                // Each warp stages its own 32 rows x 32 columns (one 4 KB box, 128B
                // swizzle: 16-byte chunk c of row r at c ^ (r & 7)) and lane 0 issues
                // its tensor store: no CTA-wide barrier in the epilogue.  The box was
                // last read by this lane's store of tile t - nstage.
                static_assert(DW_CPW == 32, "one 32-column box per warp");
                unsigned char* box = stage0 + (size_t)(t % nstage) * DW_EPI_WARPS * 4096 + (size_t)warp * 4096;
                if (lane == 0) {
                    if (nstage == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                    else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                }
                __syncwarp();
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    *reinterpret_cast<uint4*>(box + lane * 128 + ((c ^ (lane & 7)) << 4)) =
                        make_uint4(v[c * 4], v[c * 4 + 1], v[c * 4 + 2], v[c * 4 + 3]);
                // d(x, x) = 0 exactly: one scalar overwrite in the staging box, only
                // in tiles that cross the diagonal (kept out of the per-element loop)
                if (dj >= 0 && dj < DW_CPW) {
                    const int jj = (int)dj;
                    *reinterpret_cast<float*>(box + lane * 128 + (((jj >> 2) ^ (lane & 7)) << 4) + (jj & 3) * 4) = 0.f;
                }
                if (fix) {
                    // Pairs whose d^2 is small against |x|^2 + |y|^2 (within-cluster
                    // pairs; the norm expansion cancels there) are recomputed from
                    // the raw points by the definition
                    // (P:272-278).  The warp's flagged (row, column) pairs are
                    // packed: entry g goes to lane g % 32 (its row lane by a binary
                    // search of the warp's prefix counts, its column by __fns), so
                    // a round serves up to 32 pairs whichever rows they are in.
                    if (row >= n) fl = 0;
                    if (cb + DW_CPW > c1) {
                        const int64_t nv = c1 - cb;          // valid columns of this part (< 32)
                        fl &= nv <= 0 ? 0u : ((1u << (int)nv) - 1u);
                    }
                    const int cnt = __popc(fl);
                    int incl = cnt;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(FULL_MASK_DW, incl, o);
                        if (lane >= o) incl += y;
                    }
                    const int excl = incl - cnt;
                    const int total = __shfl_sync(FULL_MASK_DW, incl, 31);
                    if (total > 0) {
                        __syncwarp();                        // the box rows written above are warp-visible
                        const float* rrow = RA + mt * RF + (size_t)(q * 32) * rst;
                        const float* rcol = RB + ((n0 - c0) / DT_N) * RF + (size_t)(part * DW_CPW) * rst;
                        for (int g0 = 0; g0 < total; g0 += 32) {
                            const int g = g0 + lane;
                            // source lane: the last lane whose exclusive prefix <= g
                            int src = 0;
#pragma unroll
                            for (int step = 16; step >= 1; step >>= 1) {
                                const int ex = __shfl_sync(FULL_MASK_DW, excl, src + step);
                                if (ex <= g) src += step;
                            }
                            const unsigned sfl = __shfl_sync(FULL_MASK_DW, fl, src);
                            const int sex = __shfl_sync(FULL_MASK_DW, excl, src);
                            if (g < total) {
                                const int jj = (int)__fns(sfl, 0, g - sex + 1);
                                const float val = dw_exact(rrow + (size_t)src * rst, rcol + (size_t)jj * rst, dpad);
                                *reinterpret_cast<float*>(box + src * 128 + (((jj >> 2) ^ (src & 7)) << 4) + (jj & 3) * 4) = val;
                            }
                        }
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    const int x = (int)(n0 - c0) + part * DW_CPW;
                    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                                 :: "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(x), "r"(m0 + q * 32),
                                    "r"(dt_smem_u32(box))
                                 : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
            }
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == DW_EPI_WARPS)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "n"(DW_NACC * DT_N));
}

// L1 on integer coordinates: 64 x 64 output tile per block, 256 threads
// (each 4 x 4 outputs), coordinates staged through shared memory.
__global__ void __launch_bounds__(256)
k_dist_l1_u32(const int32_t* __restrict__ Xq, int n, int d, uint32_t* __restrict__ D, int64_t ld, int64_t c0,
              int64_t c1, const int* __restrict__ exact_f32 = nullptr) {
    if (exact_f32 && *exact_f32) return;      // k_dist_l1_f32x / u16x2 produces this matrix
    constexpr int TB = 64, KB = 32;
    __shared__ int32_t sa[KB][TB + 1], sb[KB][TB + 1];
    const int i0 = blockIdx.y * TB;
    const int64_t j0 = c0 + (int64_t)blockIdx.x * TB;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    uint32_t acc[4][4] = {};
    for (int k0 = 0; k0 < d; k0 += KB) {
        for (int idx = threadIdx.x; idx < TB * KB; idx += 256) {
            const int r = idx / KB, k = idx % KB;
            sa[k][r] = (i0 + r < n && k0 + k < d) ? Xq[(int64_t)(i0 + r) * d + k0 + k] : 0;
            sb[k][r] = (j0 + r < c1 && k0 + k < d) ? Xq[(j0 + r) * d + k0 + k] : 0;
        }
        __syncthreads();
        const int kn = min(KB, d - k0);
        for (int k = 0; k < kn; ++k) {
            int32_t a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) { a[u] = sa[k][ty * 4 + u]; b[u] = sb[k][tx * 4 + u]; }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] += (uint32_t)abs(a[u] - b[v]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int i = i0 + ty * 4 + u;
        if (i >= n) continue;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int64_t j = j0 + tx * 4 + v;
            if (j < c1) D[(int64_t)i * ld + (j - c0)] = (j == i) ? 0u : acc[u][v];
        }
    }
}

// Per-dimension coordinate range of the L1 input (decides whether the fp32
// kernel below is exact): rng[2t] = min_t, rng[2t+1] = max_t (pre-set by
// k_dist_l1_range_init), then k_dist_l1_decide sets rng[2d] = 1 iff every
// sum_t (max_t - min_t) < 2^24 (computed in int64).
__global__ void k_dist_l1_range_init(int d, int* __restrict__ rng) {
    for (int t = threadIdx.x; t < d; t += blockDim.x) { rng[2 * t] = INT_MAX; rng[2 * t + 1] = INT_MIN; }
}
// rng[2d] = 2: every range < 2^16 (k_dist_l1_u16x2, exact in 32-bit integer
// arithmetic); 1: sum of ranges < 2^24 (k_dist_l1_f32x); 0: k_dist_l1_u32.
__global__ void k_dist_l1_decide(int d, int* __restrict__ rng, int allow_packed) {
    __shared__ long long tot, mx;
    if (threadIdx.x == 0) { tot = 0; mx = 0; }
    __syncthreads();
    constexpr long long LIM = 1ll << 24;
    for (int t = threadIdx.x; t < d; t += blockDim.x) {
        const long long lo = rng[2 * t], hi = rng[2 * t + 1];
        atomicAdd((unsigned long long*)&tot, (unsigned long long)(hi - lo));
        atomicMax((unsigned long long*)&mx, (unsigned long long)(hi - lo));
    }
    __syncthreads();
    if (threadIdx.x == 0) rng[2 * d] = (allow_packed && mx < 65536) ? 2 : tot < LIM ? 1 : 0;
}
__global__ void k_dist_l1_range(const int32_t* __restrict__ Xq, int n, int d, int* __restrict__ rng) {
    const int t = blockIdx.y;
    int lo = INT_MAX, hi = INT_MIN;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int v = Xq[i * d + t];
        lo = min(lo, v); hi = max(hi, v);
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if ((threadIdx.x & 31) == 0) { atomicMin(&rng[2 * t], lo); atomicMax(&rng[2 * t + 1], hi); }
}

// L1 in fp32 arithmetic, exact: with coordinates translated per dimension
// to y_t = x_t - min_t >= 0 (L1 is translation invariant) and
// S_i = sum_t y_it,
//     sum_t |y_it - y_jt| = S_i + S_j - 2 sum_t min(y_it, y_jt).
// The kernel accumulates 2 min(.,.) in fp32; when sum_t (max_t - min_t) <
// 2^24 (decided on the device by k_dist_l1_decide) every partial sum is an
// even integer below 2^25, which fp32 represents exactly, so the result
// equals the integer definition bit for bit.  Per element one FMNMX (ALU
// pipe) and one FFMA with an immediate operand (FMA pipe), i.e. both issue
// pipes in parallel, instead of three integer-ALU instructions.  128 x 128
// tile per block, 8 x 8 outputs per thread (rows ty*4 + {0..3} and
// 64 + ty*4 + {0..3}, likewise columns), operands transposed into shared
// memory as [dim][row] floats and read as float4.
constexpr int L1F_TB = 128, L1F_KB = 32, L1F_LD = L1F_TB + 4;

// S_i of the translated coordinates (only when the fp32 kernel is used).
__global__ void k_dist_l1_rowsum(const int32_t* __restrict__ Xq, int n, int d, const int* __restrict__ rng,
                                 int* __restrict__ rowsum) {
    if (!rng[2 * d]) return;                  // the integer kernel needs no row sums
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int sum = 0;
    for (int t = 0; t < d; ++t) sum += Xq[(int64_t)i * d + t] - __ldg(&rng[2 * t]);
    rowsum[i] = sum;
}

__global__ void __launch_bounds__(256, 2)
k_dist_l1_f32x(const int32_t* __restrict__ Xq, int n, int d, uint32_t* __restrict__ D, int64_t ld, int64_t c0,
               int64_t c1, bool vec, const int* __restrict__ rng, const int* __restrict__ rowsum) {
    if (rng[2 * d] != 1) return;              // another L1 kernel produces this matrix
    __shared__ __align__(16) float sa[L1F_KB][L1F_LD], sb[L1F_KB][L1F_LD];
    const int i0 = blockIdx.y * L1F_TB;
    const int64_t j0 = c0 + (int64_t)blockIdx.x * L1F_TB;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    float acc[8][8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 8; ++v) acc[u][v] = 0.f;
    for (int k0 = 0; k0 < d; k0 += L1F_KB) {
        // 128 rows x 32 dims per operand: consecutive threads take consecutive
        // dims of one row (coalesced), written transposed; padding is 0
#pragma unroll
        for (int it = 0; it < L1F_TB * L1F_KB / 256; ++it) {
            const int idx = it * 256 + threadIdx.x;
            const int r = idx / L1F_KB, k = idx % L1F_KB;
            const bool kin = k0 + k < d;
            const int lo = kin ? __ldg(&rng[2 * (k0 + k)]) : 0;
            sa[k][r] = (i0 + r < n && kin) ? (float)(Xq[(int64_t)(i0 + r) * d + k0 + k] - lo) : 0.f;
            sb[k][r] = (j0 + r < c1 && kin) ? (float)(Xq[(j0 + r) * d + k0 + k] - lo) : 0.f;
        }
        __syncthreads();
        const int kn = min(L1F_KB, d - k0);
#pragma unroll 4
        for (int k = 0; k < kn; ++k) {
            const float4 a0 = *reinterpret_cast<const float4*>(&sa[k][ty * 4]);
            const float4 a1 = *reinterpret_cast<const float4*>(&sa[k][64 + ty * 4]);
            const float4 b0 = *reinterpret_cast<const float4*>(&sb[k][tx * 4]);
            const float4 b1 = *reinterpret_cast<const float4*>(&sb[k][64 + tx * 4]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
                for (int v = 0; v < 8; ++v) acc[u][v] = fmaf(fminf(a[u], b[v]), 2.0f, acc[u][v]);
        }
        __syncthreads();
    }
    int sj[8];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int64_t j = j0 + h * 64 + tx * 4 + v;
            sj[h * 4 + v] = j < c1 ? __ldg(&rowsum[j]) : 0;
        }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int i = i0 + (u < 4 ? ty * 4 + u : 64 + ty * 4 + (u - 4));
        if (i >= n) continue;
        const int si = __ldg(&rowsum[i]);
        uint32_t* Drow = D + (int64_t)i * ld - c0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t j = j0 + h * 64 + tx * 4;
            uint32_t o[4];
#pragma unroll
            for (int v = 0; v < 4; ++v)
                o[v] = (j + v == i) ? 0u : (uint32_t)(si + sj[h * 4 + v] - (int)acc[u][h * 4 + v]);
            if (vec && j + 3 < c1) {
                *reinterpret_cast<uint4*>(Drow + j) = make_uint4(o[0], o[1], o[2], o[3]);
            } else {
#pragma unroll
                for (int v = 0; v < 4; ++v) if (j + v < c1) Drow[j + v] = o[v];
            }
        }
    }
}

// L1 in packed 16-bit integer arithmetic, exact: with translated coordinates
// y_t = x_t - min_t < 2^16 (every range below 2^16, decided on the device),
//     sum_t |y_it - y_jt| = S_i + S_j - 2 sum_t min(y_it, y_jt)   (mod 2^32).
// Two consecutive dimensions of a row are packed in one 32-bit word; ONE
// VIMNMX.U16x2 gives both minima of a (row, column) pair and ONE IDP.2A
// (dp2a with weights (1, 1)) adds them into a 32-bit accumulator: one
// instruction per element instead of two (k_dist_l1_f32x), no overflow
// (the accumulator is 32-bit), no flushes.
//
// The words are packed once (k_dist_l1_pack16) in the exact shared-memory
// image a tile uses -- [128-row tile][dim pair][row] -- so a block fetches its
// A and B operands with two bulk copies (no per-element loads, no
// registers: the first version spent most stall samples waiting on its
// element loads).  Tile and thread layout as k_dist_l1_f32x.
constexpr int L1P_KP = 32;                     // dim pairs per shared-memory chunk (d <= 64: one chunk)

// packed operand tiles of the rows [r0, r1): out[(tile * dp + p) * 128 + r]
__global__ void k_dist_l1_pack16(const int32_t* __restrict__ Xq, int d, int64_t r0, int64_t r1,
                                 const int* __restrict__ rng, uint32_t* __restrict__ out) {
    if (rng[2 * d] != 2) return;
    const int dp = (d + 1) >> 1;
    const int64_t tile = blockIdx.x;
    for (int idx = threadIdx.x; idx < dp * L1F_TB; idx += blockDim.x) {
        const int p = idx / L1F_TB, r = idx % L1F_TB;
        const int64_t row = r0 + tile * L1F_TB + r;
        const int t0 = 2 * p, t1 = t0 + 1;
        uint32_t w = 0u;
        if (row < r1) {
            const int32_t* xr = Xq + row * d;
            const uint32_t y0 = (uint32_t)(xr[t0] - __ldg(&rng[2 * t0]));
            const uint32_t y1 = t1 < d ? (uint32_t)(xr[t1] - __ldg(&rng[2 * t1])) : 0u;
            w = y0 | (y1 << 16);
        }
        out[(tile * dp + p) * L1F_TB + r] = w;
    }
}

__global__ void __launch_bounds__(256, 2)
k_dist_l1_u16x2(const uint32_t* __restrict__ PA, const uint32_t* __restrict__ PB, int n, int d,
                uint32_t* __restrict__ D, int64_t ld, int64_t c0, int64_t c1, bool vec, const int* __restrict__ rng,
                const int* __restrict__ rowsum) {
    if (rng[2 * d] != 2) return;              // another L1 kernel produces this matrix
    __shared__ __align__(128) uint32_t sa[L1P_KP][L1F_TB], sb[L1P_KP][L1F_TB];
    __shared__ __align__(8) uint64_t bar;
    const int i0 = blockIdx.y * L1F_TB;
    const int64_t j0 = c0 + (int64_t)blockIdx.x * L1F_TB;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int dp = (d + 1) >> 1;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(dt_smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t acc[8][8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 8; ++v) acc[u][v] = 0u;
    uint32_t ph = 0;
    for (int p0 = 0; p0 < dp; p0 += L1P_KP) {
        const int kn = min(L1P_KP, dp - p0);
        if (threadIdx.x == 0) {
            // one arrival announcing both copies' bytes, then the two copies
            const uint32_t bytes = (uint32_t)kn * L1F_TB * 4u;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                         :: "r"(dt_smem_u32(&bar)), "r"(2u * bytes) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         :: "r"(dt_smem_u32(&sa[0][0])), "l"(PA + ((int64_t)blockIdx.y * dp + p0) * L1F_TB),
                            "r"(bytes), "r"(dt_smem_u32(&bar)) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         :: "r"(dt_smem_u32(&sb[0][0])), "l"(PB + ((int64_t)blockIdx.x * dp + p0) * L1F_TB),
                            "r"(bytes), "r"(dt_smem_u32(&bar)) : "memory");
        }
        dt_wait(&bar, ph); ph ^= 1;
#pragma unroll 4
        for (int kp = 0; kp < kn; ++kp) {
            const uint4 a0 = *reinterpret_cast<const uint4*>(&sa[kp][ty * 4]);
            const uint4 a1 = *reinterpret_cast<const uint4*>(&sa[kp][64 + ty * 4]);
            const uint4 b0 = *reinterpret_cast<const uint4*>(&sb[kp][tx * 4]);
            const uint4 b1 = *reinterpret_cast<const uint4*>(&sb[kp][64 + tx * 4]);
            const uint32_t a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const uint32_t b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
                for (int v = 0; v < 8; ++v) acc[u][v] = __dp2a_lo(__vminu2(a[u], b[v]), 0x0101u, acc[u][v]);
        }
        __syncthreads();                          // the tiles are overwritten by the next chunk
    }
    uint32_t sj[8];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int64_t j = j0 + h * 64 + tx * 4 + v;
            sj[h * 4 + v] = j < c1 ? (uint32_t)__ldg(&rowsum[j]) : 0u;
        }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int i = i0 + (u < 4 ? ty * 4 + u : 64 + ty * 4 + (u - 4));
        if (i >= n) continue;
        const uint32_t si = (uint32_t)__ldg(&rowsum[i]);
        uint32_t* Drow = D + (int64_t)i * ld - c0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t j = j0 + h * 64 + tx * 4;
            uint32_t o[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) o[v] = (j + v == i) ? 0u : si + sj[h * 4 + v] - 2u * acc[u][h * 4 + v];
            if (vec && j + 3 < c1) {
                *reinterpret_cast<uint4*>(Drow + j) = make_uint4(o[0], o[1], o[2], o[3]);
            } else {
#pragma unroll
                for (int v = 0; v < 4; ++v) if (j + v < c1) Drow[j + v] = o[v];
            }
        }
    }
}

}  // namespace km
