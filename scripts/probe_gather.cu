// Microbenchmark: random 160-byte row gathers from an L2-resident table,
// (a) LDG.128, 10 lanes per row (3 rows per warp instruction), U rows in flight
// per lane; (b) TMA bulk copies (cp.async.bulk, one 160 B row per lane) into a
// per-warp shared-memory ring tracked by mbarriers.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
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

// (a2) 256-bit loads (LDG.E.ENL2.256, sm_100): 5 lanes per 160 B row, 6 rows
// per warp instruction
struct f8 { float4 lo, hi; };
__device__ __forceinline__ f8 ldg256(const float* p)
{
    f8 v;
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v.lo.x), "=f"(v.lo.y), "=f"(v.lo.z), "=f"(v.lo.w), "=f"(v.hi.x), "=f"(v.hi.y),
                   "=f"(v.hi.z), "=f"(v.hi.w)
                 : "l"(p));
    return v;
}

template <int U>
__global__ void gather_ldg256(const float* __restrict__ tab, const int* __restrict__ idx, int64_t nrows_req,
                              float* out)
{
    const int lane = threadIdx.x & 31;
    const int slot = lane / 5, c8 = lane % 5;
    const bool on = slot < 6;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    float4 acc = make_float4(0, 0, 0, 0);
    for (int64_t base = gw * 6 * U; base < nrows_req; base += nw * 6 * U) {
        f8 x[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t q = base + u * 6 + slot;
            if (on && q < nrows_req) x[u] = ldg256(tab + (int64_t)idx[q] * 40 + c8 * 8);
            else x[u].lo = x[u].hi = make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            acc.x += x[u].lo.x + x[u].hi.x; acc.y += x[u].lo.y + x[u].hi.y;
            acc.z += x[u].lo.z + x[u].hi.z; acc.w += x[u].lo.w + x[u].hi.w;
        }
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

// (c) TMA tile::gather4 (sm_100a): one instruction gathers 4 rows of a 2-D
// tensor map (box 40 x 1 f32 = one 160 B row) into 640 contiguous bytes of
// shared memory; lanes 0..ROWS/4-1 of the warp issue a chunk's gathers.
template <int STAGES, int ROWS>
__global__ void gather_tma4(const __grid_constant__ CUtensorMap tmap, const int* __restrict__ idx,
                            int64_t nrows_req, float* out)
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
    int64_t issued = 0, consumed = 0;
    const int64_t mine = gw < nchunks ? (nchunks - 1 - gw) / nw + 1 : 0;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    auto issue = [&](int64_t j) {
        const int s = (int)(j % STAGES);
        const int64_t chunk = gw + j * nw;
        float* dst = buf + (int64_t)s * ROWS * 40;
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bars + s)),
                         "r"(ROWS * 160) : "memory");
        __syncwarp();
        if (lane < ROWS / 4) {
            int r4[4];
            for (int u = 0; u < 4; u++) {
                const int64_t q = chunk * ROWS + 4 * lane + u;
                r4[u] = q < nrows_req ? idx[q] : 0;
            }
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst + 4 * lane * 40)),
                "l"(&tmap), "r"(0), "r"(r4[0]), "r"(r4[1]), "r"(r4[2]), "r"(r4[3]),
                "r"(smem_u32(bars + s))
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
        const float4* src = reinterpret_cast<const float4*>(buf + (int64_t)s * ROWS * 40);
        for (int e = lane; e < ROWS * 10; e += 32) {
            const float4 x = src[e];
            acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
        }
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (issued < mine) issue(issued++);
    }
    if (acc.x + acc.y + acc.z + acc.w == 1.2345f) out[0] = acc.x;
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                CUtensorMapFloatOOBfill);

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
    for (int occ : {1, 2, 3, 4}) {
        auto run = [&](auto kern, const char* nm) {
            kern<<<sms * occ, 256>>>((const float*)tab, idx, nreq, out);
            cudaEventRecord(a);
            kern<<<sms * occ, 256>>>((const float*)tab, idx, nreq, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("%s %d CTA/SM: %.3f ms  %.2f TB/s (%s)\n", nm, occ, ms, nreq * 160.0 / ms / 1e9,
                   cudaGetErrorString(cudaGetLastError()));
        };
        run(gather_ldg256<4>, "LDG256 U4 ");
        run(gather_ldg256<8>, "LDG256 U8 ");
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
    {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult qr;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
        CUtensorMap tmap;
        cuuint64_t dims[2] = {40, (cuuint64_t)ntab};
        cuuint64_t strides[1] = {160};
        cuuint32_t box[2] = {40, 1};
        cuuint32_t estr[2] = {1, 1};
        CUresult cr = ((EncodeTiled)fn)(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, tab, dims, strides, box,
                                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("tensor map encode: %d\n", (int)cr);
        auto run = [&](auto kern, int warps, int ctas_per_sm, size_t smem, const char* name, int st, int rw) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            kern<<<sms * ctas_per_sm, 32 * warps, smem>>>(tmap, idx, nreq, out);
            cudaEventRecord(a);
            kern<<<sms * ctas_per_sm, 32 * warps, smem>>>(tmap, idx, nreq, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("TMA gather4 %s %d CTA/SM x %d warps x %d stages x %d rows: %.3f ms  %.2f TB/s (%s)\n", name,
                   ctas_per_sm, warps, st, rw, ms, nreq * 160.0 / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
        };
        run(gather_tma4<4, 32>, 8, 1, (size_t)8 * 4 * 32 * 160 + 8 * 4 * 8, "", 4, 32);
        run(gather_tma4<2, 32>, 8, 2, (size_t)8 * 2 * 32 * 160 + 8 * 2 * 8, "", 2, 32);
        run(gather_tma4<2, 16>, 16, 2, (size_t)16 * 2 * 16 * 160 + 16 * 2 * 8, "", 2, 16);
        run(gather_tma4<4, 16>, 16, 1, (size_t)16 * 4 * 16 * 160 + 16 * 4 * 8, "", 4, 16);
        run(gather_tma4<2, 16>, 32, 1, (size_t)32 * 2 * 16 * 160 + 32 * 2 * 8, "", 2, 16);
        run(gather_tma4<8, 8>, 16, 1, (size_t)16 * 8 * 8 * 160 + 16 * 8 * 8, "", 8, 8);
    }
    return 0;
}
