// Microbenchmark: cost of one grid-wide barrier on B200 (cooperative groups
// grid.sync() vs a hand-rolled sense-reversal barrier), for the persistent SITE
// loop's three barriers per round.  nvcc -gencode arch=compute_100a,code=sm_100a
// -o gridsync_bench gridsync_bench.cu && ./gridsync_bench
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, unsigned* sink) {
    cg::grid_group g = cg::this_grid();
    unsigned acc = 0;
    for (int i = 0; i < iters; ++i) { acc += threadIdx.x; g.sync(); }
    if (acc == 0xdeadbeef) *sink = acc;
}

// one arrival counter + a generation word; the last arriving CTA bumps the generation
__global__ void k_custom(int iters, unsigned* count, volatile unsigned* gen, unsigned* sink) {
    unsigned acc = 0;
    for (int i = 0; i < iters; ++i) {
        acc += threadIdx.x;
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned g0 = *gen;
            __threadfence();
            if (atomicAdd(count, 1u) == gridDim.x - 1) {
                *count = 0;
                __threadfence();
                atomicAdd((unsigned*)gen, 1u);
            } else {
                while (*gen == g0) {}
            }
            __threadfence();
        }
        __syncthreads();
    }
    if (acc == 0xdeadbeef) *sink = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned *sink, *cnt, *gen;
    cudaMalloc(&sink, 4); cudaMalloc(&cnt, 4); cudaMalloc(&gen, 4);
    cudaMemset(cnt, 0, 4); cudaMemset(gen, 0, 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 2000;
    for (int per = 1; per <= 4; per *= 2) {
        const int grid = sms * per;
        void* args[] = {(void*)&iters, (void*)&sink};
        cudaLaunchCooperativeKernel((void*)k_cg, grid, 256, args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_cg, grid, 256, args, 0, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        void* args2[] = {(void*)&iters, (void*)&cnt, (void*)&gen, (void*)&sink};
        cudaLaunchCooperativeKernel((void*)k_custom, grid, 256, args2, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_custom, grid, 256, args2, 0, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms2; cudaEventElapsedTime(&ms2, a, b);
        printf("grid %d CTAs x 256: cg grid.sync %.2f us, custom barrier %.2f us (err %s)\n", grid, ms * 1e3 / iters,
               ms2 * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
