// Microbenchmark: random 160-byte row gathers from an L2-resident table,
// (a) LDG.128, 10 lanes per row (3 rows per warp instruction), U rows in flight
// per lane; (b) TMA bulk copies (cp.async.bulk, one 160 B row per lane) into a
// per-warp shared-memory ring tracked by mbarriers.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void gather_ldg(const float4* __restrict__ tab, const int* __restrict__ idx, int64_t nrows_req,
                           float* out)
{
    const int lane = threadIdx.x & 31;
    const int slot = lane / 10, c4 = lane % 10;
    const bool on = slot < 3;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    float4 acc = make_float4(0, 0, 0, 0);
    constexpr int U = 16;
    for (int64_t base = gw * 3 * U; base < nrows_req; base += nw * 3 * U) {
        float4 x[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t q = base + u * 3 + slot;
            x[u] = (on && q < nrows_req) ? __ldg(tab + (int64_t)idx[q] * 10 + c4) : make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; u++) { acc.x += x[u].x; acc.y += x[u].y; acc.z += x[u].z; acc.w += x[u].w; }
    }
    if (acc.x + acc.y + acc.z + acc.w == 1.2345f) out[0] = acc.y;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int STAGES, int ROWS>
__global__ void gather_tma(const float* __restrict__ tab, const int* __restrict__ idx, int64_t nrows_req,
                           float* out)
{
    extern __shared__ __align__(128) unsigned char sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwc = blockDim.x >> 5;
    float* buf = reinterpret_cast<float*>(sm) + (int64_t)warp * STAGES * ROWS * 40;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)nwc * STAGES * ROWS * 160) + warp * STAGES;
    if (lane == 0)
        for (int s = 0; s < STAGES; s++)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + s)));
    __syncwarp();
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int64_t gw = (int64_t)blockIdx.x * nwc + warp;
    const int64_t nw = (int64_t)gridDim.x * nwc;
    const int64_t nchunks = (nrows_req + ROWS - 1) / ROWS;
    // my chunks: gw, gw + nw, ...
    int64_t issued = 0, consumed = 0;
    const int64_t mine = gw < nchunks ? (nchunks - 1 - gw) / nw + 1 : 0;
    float acc = 0.f;
    auto issue = [&](int64_t j) {
        const int s = (int)(j % STAGES);
        const int64_t chunk = gw + j * nw;
        float* dst = buf + (int64_t)s * ROWS * 40;
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bars + s)),
                         "r"(ROWS * 160) : "memory");
        __syncwarp();
        for (int r = lane; r < ROWS; r += 32) {
            const int64_t q = chunk * ROWS + r;
            const int row = q < nrows_req ? idx[q] : 0;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 160, [%2];" ::"r"(
                    smem_u32(dst + r * 40)),
                "l"(tab + (int64_t)row * 40), "r"(smem_u32(bars + s))
                : "memory");
        }
    };
    for (; issued < mine && issued < STAGES; issued++) issue(issued);
    for (; consumed < mine; consumed++) {
        const int s = (int)(consumed % STAGES);
        const unsigned par = (unsigned)((consumed / STAGES) & 1);
        unsigned done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(smem_u32(bars + s)), "r"(par) : "memory");
        const float* src = buf + (int64_t)s * ROWS * 40;
        for (int e = lane; e < ROWS * 40; e += 32) acc += src[e];
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (issued < mine) issue(issued++);
    }
    if (acc == 1.2345f) out[0] = acc;
}

int main()
{
    const int64_t ntab = 100000 * 25 / 10;  // 250k rows x 160 B = 40 MB
    const int64_t nreq = 16 * 1000 * 1000;  // 16M row gathers = 2.56 GB
    float4* tab;
    int* idx;
    float* out;
    cudaMalloc(&tab, ntab * 160);
    cudaMemset(tab, 0, ntab * 160);
    cudaMalloc(&idx, nreq * 4);
    cudaMalloc(&out, 8);
    int* h = (int*)malloc(nreq * 4);
    uint64_t st = 88172645463325252ull;
    for (int64_t i = 0; i < nreq; i++) {
        st ^= st << 13; st ^= st >> 7; st ^= st << 17;
        h[i] = (int)(st % ntab);
    }
    cudaMemcpy(idx, h, nreq * 4, cudaMemcpyHostToDevice);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    for (int occ : {1, 2, 3, 4}) {
        gather_ldg<<<sms * occ, 256>>>(tab, idx, nreq, out);
        cudaEventRecord(a);
        gather_ldg<<<sms * occ, 256>>>(tab, idx, nreq, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("LDG  %d CTA/SM: %.3f ms  %.2f TB/s (%s)\n", occ, ms, nreq * 160.0 / ms / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    }
    {
        constexpr int ST = 4, RW = 32;
        const int warps = 8;
        const size_t smem = (size_t)warps * ST * RW * 160 + warps * ST * 8;
        cudaFuncSetAttribute(gather_tma<ST, RW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        gather_tma<ST, RW><<<sms, 32 * warps, smem>>>((float*)tab, idx, nreq, out);
        cudaEventRecord(a);
        gather_tma<ST, RW><<<sms, 32 * warps, smem>>>((float*)tab, idx, nreq, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("TMA  %d warps x %d stages x %d rows: %.3f ms  %.2f TB/s (%s)\n", warps, ST, RW, ms,
               nreq * 160.0 / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    {
        constexpr int ST = 2, RW = 32;
        const int warps = 16;
        const size_t smem = (size_t)warps * ST * RW * 160 + warps * ST * 8;
        cudaFuncSetAttribute(gather_tma<ST, RW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        gather_tma<ST, RW><<<sms, 32 * warps, smem>>>((float*)tab, idx, nreq, out);
        cudaEventRecord(a);
        gather_tma<ST, RW><<<sms, 32 * warps, smem>>>((float*)tab, idx, nreq, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("TMA  %d warps x %d stages x %d rows: %.3f ms  %.2f TB/s (%s)\n", warps, ST, RW, ms,
               nreq * 160.0 / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
