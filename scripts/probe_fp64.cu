// Microbenchmark: FP64 FMA (DFMA) vs FP64 tensor MMA (DMMA.8x8x4) throughput
// per SM on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int C>
__global__ void k_dmma(int iters, double* out)
{
    double acc[C][2];
    for (int c = 0; c < C; c++) acc[c][0] = acc[c][1] = threadIdx.x;
    double a = 1.0000001, b = 0.9999999;
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int c = 0; c < C; c++) dmma(acc[c][0], acc[c][1], a, b);
    double s = 0;
    for (int c = 0; c < C; c++) s += acc[c][0] + acc[c][1];
    if (s == 1.2345) out[0] = s;
}
template <int C>
__global__ void k_dfma(int iters, double* out)
{
    double acc[C];
    for (int c = 0; c < C; c++) acc[c] = threadIdx.x + c;
    const double a = 1.0000001, b = 1e-9;
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int c = 0; c < C; c++) acc[c] = fma(acc[c], a, b);
    double s = 0;
    for (int c = 0; c < C; c++) s += acc[c];
    if (s == 1.2345) out[0] = s;
}
int main()
{
    double* out;
    cudaMalloc(&out, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4096;
    for (int warps : {4, 8, 16, 32}) {
        k_dmma<8><<<sms, 32 * warps>>>(iters, out);
        cudaEventRecord(a);
        k_dmma<8><<<sms, 32 * warps>>>(iters, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double fma = (double)sms * warps * iters * 8 * 256;
        printf("DMMA warps/SM=%2d: %.2f TFLOPS (%.1f FMA/clk/SM at 1.965 GHz)\n", warps,
               2 * fma / ms / 1e9, fma / sms / (ms * 1e-3 * 1.965e9));
        k_dfma<8><<<sms, 32 * warps>>>(iters, out);
        cudaEventRecord(a);
        k_dfma<8><<<sms, 32 * warps>>>(iters, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        fma = (double)sms * warps * 32 * iters * 8;
        printf("DFMA warps/SM=%2d: %.2f TFLOPS (%.1f FMA/clk/SM)\n", warps, 2 * fma / ms / 1e9,
               fma / sms / (ms * 1e-3 * 1.965e9));
    }
    return 0;
}
