// Microbenchmark: cost of one grid-wide barrier on this GPU (148 CTAs x 512
// threads): cooperative_groups grid.sync() vs a hand-rolled atomic barrier.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void cg_sync(int iters, double* sink)
{
    auto g = cg::this_grid();
    double acc = threadIdx.x;
    for (int i = 0; i < iters; i++) {
        acc += 1.0;
        g.sync();
    }
    if (acc < 0) sink[0] = acc;
}

__device__ unsigned int bar_count = 0;
__device__ volatile unsigned int bar_gen = 0;

__device__ __forceinline__ void my_sync()
{
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int gen = bar_gen;
        __threadfence();
        if (atomicAdd(&bar_count, 1) == gridDim.x - 1) {
            bar_count = 0;
            __threadfence();
            bar_gen = gen + 1;
        } else {
            while (bar_gen == gen) { }
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void my_sync_k(int iters, double* sink)
{
    double acc = threadIdx.x;
    for (int i = 0; i < iters; i++) {
        acc += 1.0;
        my_sync();
    }
    if (acc < 0) sink[0] = acc;
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* sink;
    cudaMalloc(&sink, 8);
    const int iters = 20000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int threads : {128, 512}) {
        int it = iters;
        void* args[] = {&it, &sink};
        cudaLaunchCooperativeKernel((void*)cg_sync, sms, threads, args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)cg_sync, sms, threads, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("cg grid.sync   %d CTAs x %d thr: %.3f us/sync (%s)\n", sms, threads,
               ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
        cudaLaunchCooperativeKernel((void*)my_sync_k, sms, threads, args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)my_sync_k, sms, threads, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("atomic barrier %d CTAs x %d thr: %.3f us/sync (%s)\n", sms, threads,
               ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
