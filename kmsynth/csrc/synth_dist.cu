// synth_dist.cu -- materialise a synthetic dissimilarity matrix on the GPU.
//
// INPUT GENERATOR (kmsynth), not part of the method: it turns the seeded
// point sets of kmsynth/__init__.py into the dense matrix D that both the
// CUDA path and the oracle consume.  It holds none of the FastPAM arithmetic.
//
// metric 0 (L1 on integer coordinates):  D[o][c] = sum_t |x_ot - x_ct|  (exact, uint32)
// metric 1 (Euclidean, fp64 coordinates): D[o][c] = f32(sqrt(sum_t (x_ot - x_ct)^2))
//   with every fp64 operation individually rounded in t order (no FMA), so the
//   result is bit-identical to kmsynth.dist_numpy.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {
constexpr int TILE = 32;
constexpr int KT = 16;   // coordinates staged per step

template <int METRIC, typename X>
__global__ void k_dist(const X* __restrict__ pts, int n, int d, int64_t c0, int64_t c1, int64_t ld, void* out) {
    __shared__ X so[TILE][KT + 1];
    __shared__ X sc[TILE][KT + 1];
    const int tx = threadIdx.x, ty = threadIdx.y;          // 32 x 8
    const int64_t obase = (int64_t)blockIdx.y * TILE, cbase = c0 + (int64_t)blockIdx.x * TILE;
    long long iacc[4] = {0, 0, 0, 0};
    double facc[4] = {0, 0, 0, 0};
    for (int t0 = 0; t0 < d; t0 += KT) {
        for (int r = ty; r < TILE; r += 8) {
            for (int t = tx; t < KT; t += 32) {
                int64_t o = obase + r, c = cbase + r;
                so[r][t] = (o < n && t0 + t < d) ? pts[o * d + t0 + t] : (X)0;
                sc[r][t] = (c < c1 && t0 + t < d) ? pts[c * d + t0 + t] : (X)0;
            }
        }
        __syncthreads();
        const int tend = min(KT, d - t0);
        for (int t = 0; t < tend; ++t) {
            const X xc = sc[tx][t];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const X xo = so[ty + 8 * q][t];
                if (METRIC == 0) {
                    long long df = (long long)xo - (long long)xc;
                    iacc[q] += df < 0 ? -df : df;
                } else {
                    double df = __dsub_rn((double)xo, (double)xc);
                    facc[q] = __dadd_rn(facc[q], __dmul_rn(df, df));
                }
            }
        }
        __syncthreads();
    }
    const int64_t c = cbase + tx;
    if (c >= c1) return;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int64_t o = obase + ty + 8 * q;
        if (o >= n) continue;
        if (METRIC == 0) ((uint32_t*)out)[o * ld + (c - c0)] = (uint32_t)iacc[q];
        else ((float*)out)[o * ld + (c - c0)] = __double2float_rn(__dsqrt_rn(facc[q]));
    }
}
}  // namespace

extern "C" int kmsynth_dist(const void* pts_dev, int metric, int n, int d, int64_t c0, int64_t c1, int64_t ld,
                            void* out_dev, void* stream) {
    dim3 blk(32, 8);
    dim3 grd((unsigned)((c1 - c0 + TILE - 1) / TILE), (unsigned)((n + TILE - 1) / TILE));
    cudaStream_t st = (cudaStream_t)stream;
    if (metric == 0) k_dist<0, int32_t><<<grd, blk, 0, st>>>((const int32_t*)pts_dev, n, d, c0, c1, ld, out_dev);
    else k_dist<1, double><<<grd, blk, 0, st>>>((const double*)pts_dev, n, d, c0, c1, ld, out_dev);
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Measurement helper (bench.py): the read-only HBM bandwidth of this GPU in the
// same job -- a grid-stride 128-bit load stream over `bytes` of a buffer,
// XOR-folded into one word so the loads cannot be removed.  Not part of the
// method; a denominator for the stream kernel's roofline besides the copy peak.
// ---------------------------------------------------------------------------
namespace {
__global__ void k_read_stream(const uint4* __restrict__ p, int64_t n16, unsigned* __restrict__ sink) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {
        uint4 a, b, c, e;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "l"(p + i));
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(p + i + stride));
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(c.x), "=r"(c.y), "=r"(c.z), "=r"(c.w) : "l"(p + i + 2 * stride));
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(e.x), "=r"(e.y), "=r"(e.z), "=r"(e.w) : "l"(p + i + 3 * stride));
        acc.x ^= a.x ^ b.x ^ c.x ^ e.x; acc.y ^= a.y ^ b.y ^ c.y ^ e.y;
        acc.z ^= a.z ^ b.z ^ c.z ^ e.z; acc.w ^= a.w ^ b.w ^ c.w ^ e.w;
    }
    for (; i < n16; i += stride) { const uint4 a = p[i]; acc.x ^= a.x; acc.y ^= a.y; acc.z ^= a.z; acc.w ^= a.w; }
    const unsigned v = acc.x ^ acc.y ^ acc.z ^ acc.w;
    if (v == 0x9e3779b9u) atomicXor(sink, v);   // practically never taken; keeps the loads alive
}
__global__ void k_write_stream(uint4* __restrict__ p, int64_t n16, unsigned v) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const uint4 w = make_uint4(v, v, v, v);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride)
        asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p + i), "r"(w.x), "r"(w.y),
                     "r"(w.z), "r"(w.w) : "memory");
}
// Read-only stream through TMA bulk copies into a shared-memory ring (what
// the SWAP stream's producer does, with no consumer work): CTA-strided 16 KB
// chunks, RING stages in flight per CTA.
constexpr int RB_CHUNK = 16384, RB_RING = 4;
__global__ void __launch_bounds__(32) k_read_bulk(const unsigned char* __restrict__ p, int64_t nchunks) {
    extern __shared__ __align__(128) unsigned char rsm[];
    __shared__ __align__(8) unsigned long long bar[RB_RING];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < RB_RING; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((unsigned)__cvta_generic_to_shared(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    unsigned ph[RB_RING] = {0, 0, 0, 0};
    int64_t issued = 0, done = 0;
    const int64_t first = blockIdx.x, step = gridDim.x;
    auto issue = [&](int64_t c, int s) {
        const unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(RB_CHUNK) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"((unsigned)__cvta_generic_to_shared(rsm + s * RB_CHUNK)), "l"(p + c * RB_CHUNK),
                        "r"(RB_CHUNK), "r"(b) : "memory");
    };
    for (int64_t c = first; c < nchunks && issued < RB_RING; c += step) issue(c, (int)(issued++ % RB_RING));
    for (int64_t c = first; c < nchunks; c += step) {
        const int s = (int)(done % RB_RING);
        const unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
        unsigned ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\t"
                         "selp.u32 %0, 1, 0, q;\n\t}" : "=r"(ok) : "r"(b), "r"(ph[s]) : "memory");
        ph[s] ^= 1;
        ++done;
        const int64_t nxt = first + (int64_t)(done + RB_RING - 1) * step;
        if (nxt < nchunks) issue(nxt, s);
    }
}
}  // namespace

// Read-only HBM bandwidth through TMA bulk copies (GB/s, best of reps).
extern "C" double kmsynth_read_peak_bulk(const void* buf, int64_t bytes, int reps, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int64_t nchunks = bytes / RB_CHUNK;
    if (nchunks < 1) return -1.0;
    const int smem = RB_CHUNK * RB_RING;
    if (cudaFuncSetAttribute(k_read_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return -1.0;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    double best = 0.0;
    for (int per_sm : {3, 4}) {
        k_read_bulk<<<nsm * per_sm, 32, smem, st>>>((const unsigned char*)buf, nchunks);     // warm-up
        if (cudaGetLastError() != cudaSuccess) continue;
        for (int r = 0; r < reps; ++r) {
            cudaEventRecord(a, st);
            k_read_bulk<<<nsm * per_sm, 32, smem, st>>>((const unsigned char*)buf, nchunks);
            cudaEventRecord(b, st);
            cudaEventSynchronize(b);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, a, b);
            if (!(ms > 0.f)) continue;
            const double gbs = (double)nchunks * RB_CHUNK / (ms * 1e-3) / 1e9;
            if (gbs > best) best = gbs;
        }
    }
    cudaEventDestroy(a); cudaEventDestroy(b);
    return best;
}

// Best of `reps` timed write-only passes over buf (its contents are
// overwritten); returns GB/s (written bytes / time).
extern "C" double kmsynth_write_peak(void* buf, int64_t bytes, int reps, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int64_t n16 = bytes / 16;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    k_write_stream<<<nsm * 8, 256, 0, st>>>((uint4*)buf, n16, 0u);     // warm-up
    double best = 0.0;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a, st);
        k_write_stream<<<nsm * 8, 256, 0, st>>>((uint4*)buf, n16, (unsigned)r);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        const double gbs = (double)n16 * 16 / (ms * 1e-3) / 1e9;
        if (gbs > best) best = gbs;
    }
    cudaEventDestroy(a); cudaEventDestroy(b);
    return best;
}

// Best of `reps` timed passes (CUDA events); returns GB/s (read bytes / time).
extern "C" double kmsynth_read_peak(const void* buf, int64_t bytes, int reps, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    unsigned* sink = nullptr;
    if (cudaMalloc(&sink, sizeof(unsigned)) != cudaSuccess) return -1.0;
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int64_t n16 = bytes / 16;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    // the best of several launch shapes (blocks per SM x threads), so the
    // denominator is not an artefact of one occupancy choice
    const int shapes[3][2] = {{8, 256}, {4, 512}, {16, 256}};
    k_read_stream<<<nsm * 8, 256, 0, st>>>((const uint4*)buf, n16, sink);     // warm-up
    double best = 0.0;
    for (const auto& sh : shapes)
        for (int r = 0; r < reps; ++r) {
            cudaEventRecord(a, st);
            k_read_stream<<<nsm * sh[0], sh[1], 0, st>>>((const uint4*)buf, n16, sink);
            if (cudaGetLastError() != cudaSuccess) break;     // shape not launchable: skip it
            cudaEventRecord(b, st);
            cudaEventSynchronize(b);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, a, b);
            if (!(ms > 0.f)) continue;
            const double gbs = (double)n16 * 16 / (ms * 1e-3) / 1e9;
            if (gbs > best) best = gbs;
        }
    cudaEventDestroy(a); cudaEventDestroy(b);
    cudaFree(sink);
    return best;
}
