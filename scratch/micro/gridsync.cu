// grid.sync() cost on B200 for several cooperative grid shapes
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__device__ unsigned int g_cnt;
__device__ volatile unsigned int g_gen;
__global__ void k_sync(int iters, int* out) {
    cg::grid_group grid = cg::this_grid();
    for (int i = 0; i < iters; ++i) grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = iters;
}
// simple sense-reversal barrier: one atomic per block
__device__ __forceinline__ void my_sync(unsigned nb, unsigned& gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned g0 = gen;
        if (atomicAdd(&g_cnt, 1) == nb - 1) { g_cnt = 0; __threadfence(); g_gen = g0 + 1; }
        else { while (g_gen == g0) { __nanosleep(20); } }
        gen = g0 + 1;
        __threadfence();
    }
    __syncthreads();
}
__global__ void k_mysync(int iters, int* out) {
    unsigned gen = g_gen;
    for (int i = 0; i < iters; ++i) my_sync(gridDim.x, gen);
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = iters;
}
int main() {
    int* out; cudaMalloc(&out, 4);
    int shapes[][2] = {{148, 256}, {296, 256}, {444, 256}, {148, 512}, {148, 1024}, {592, 256}};
    for (auto& s : shapes) {
        for (int variant = 0; variant < 2; ++variant) {
            int iters = 2000;
            void* args[] = {&iters, &out};
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            void* fn = variant ? (void*)k_mysync : (void*)k_sync;
            cudaLaunchCooperativeKernel(fn, s[0], s[1], args, 0, 0);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel(fn, s[0], s[1], args, 0, 0);
            cudaEventRecord(b);
            cudaError_t e = cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("%s blocks %d x %d: %.3f us per sync (%s)\n", variant ? "mysync" : "cg", s[0], s[1], ms * 1e3 / iters,
                   cudaGetErrorString(e));
        }
    }
}
