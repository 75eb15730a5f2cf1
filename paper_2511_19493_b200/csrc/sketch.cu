// sketch.cu — K4/K5: the implicit low-rank sketch P X = (1/B) sum_b E_b E_b^T X
// without materialising P or the one-hot M, plus the skinny Gram / small
// matmul kernels of the QR and Rayleigh-Ritz steps.
//
// Reference: lowrank_proximity (proximity.py:367-420): Omega from
// Pcg32(seed, SEQ_FACTOR).normals((n, k)) (rng.py:102-115), then
// Y = M @ (Mt @ X) with M the 1/sqrt(B)-scaled CSR one-hot (proximity.py:88-97,
// scipy SpMM), np.linalg.qr, T = Q^T (M Mt Q), eigh.
//
// Per sketch pass (X -> Y):
//   leaf_sums   one warp per leaf walks that leaf's run of the bucketed
//               permutation (K2) and gathers the members' X rows (f32,
//               L2-resident) as float4 lanes, accumulating in f64 in a fixed
//               order -> S (f32, one row per leaf of every tree).
//   leaf_gather one warp per sample reads its B codes (coalesced row of the
//               (n, B) membership) and gathers the B leaf-sum rows, f64
//               accumulation, scale 1/B.
// Both are deterministic (no atomics), so the factors are bit-reproducible
// run to run, as the reference's are (tests/test_proximity.py:229-232).
#include "../csrc/host/pcg32.h"
#include "common.cuh"

namespace rfxc {

// --------------------------------------------------------------- normals
constexpr int NORMAL_PAIRS_PER_THREAD = 64;

__global__ void normals_kernel(uint64_t st0, uint64_t inc, int64_t count, double* __restrict__ out)
{
    const int64_t npairs = (count + 1) / 2;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t p0 = t * NORMAL_PAIRS_PER_THREAD;
    if (p0 >= npairs) return;
    const int64_t p1 = min(npairs, p0 + NORMAL_PAIRS_PER_THREAD);
    uint64_t s[2] = {st0, inc};
    rfx_pcg32_advance(s, (uint64_t)(2 * p0));
    const double two_pi = 2.0 * 3.141592653589793;
    for (int64_t q = p0; q < p1; q++) {
        const double u1 = ((double)rfx_pcg32_next(s) + 1.0) / 4294967296.0;
        const double u2 = (double)rfx_pcg32_next(s) / 4294967296.0;
        const double r = sqrt(-2.0 * log(u1));
        const double a = two_pi * u2;
        out[2 * q] = r * cos(a);
        if (2 * q + 1 < count) out[2 * q + 1] = r * sin(a);
    }
}

__global__ void pack_f32_kernel(const double* __restrict__ in, int64_t n, int k, int ld,
                                float* __restrict__ out)
{
    const int64_t total = n * ld;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / ld;
        const int c = (int)(e % ld);
        out[e] = c < k ? (float)in[i * k + c] : 0.0f;
    }
}

// -------------------------------------------------------------- leaf sums
// Lanes cover one 32-float4 (128-column) chunk of a row: lane = slot*k4c + c4,
// R = 32 / k4c rows per warp step.  Leaves are taken 32 at a time per warp
// (their run bounds fetched in one coalesced load); a leaf's member ids are
// fetched 32 at a time (coalesced) and then up to SK_U row loads per lane are
// issued back to back before any is consumed, so a small leaf costs about
// two memory round trips instead of one per member.
constexpr int SK_U = 8;

__device__ __forceinline__ void add4(double& a0, double& a1, double& a2, double& a3, float4 x)
{
    a0 += (double)x.x;
    a1 += (double)x.y;
    a2 += (double)x.z;
    a3 += (double)x.w;
}

__global__ void __launch_bounds__(256)
leaf_sums_kernel(const int32_t* __restrict__ perm, const int64_t* __restrict__ seg, int64_t g_lo,
                 int64_t g_hi, const float4* __restrict__ X4, int k4, float4* __restrict__ S4)
{
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int cc = 0; cc < k4; cc += 32) {
        const int k4c = min(32, k4 - cc);
        const int R = 32 / k4c;
        const int slot = lane / k4c, c4 = lane % k4c;
        const bool on = slot < R;
        for (int64_t g0 = g_lo + warp * 32; g0 < g_hi; g0 += nwarps * 32) {
            const int64_t gj = g0 + lane;
            int64_t sj = 0, ej = 0;
            if (gj < g_hi) {
                sj = seg[gj];
                ej = seg[gj + 1];
            }
            const int nleaf = (int)min64(32, g_hi - g0);
            for (int jj = 0; jj < nleaf; jj++) {
                const int64_t s = __shfl_sync(0xffffffffu, sj, jj);
                const int64_t e = __shfl_sync(0xffffffffu, ej, jj);
                double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
                for (int64_t base = s; base < e; base += 32) {
                    const int m = (int)min64(32, e - base);
                    const int32_t rid = lane < m ? __ldg(perm + base + lane) : 0;
                    for (int t0 = 0; t0 < m; t0 += R * SK_U) {
                        float4 x[SK_U];
#pragma unroll
                        for (int u = 0; u < SK_U; u++) {
                            const int t = t0 + u * R + slot;
                            const int r = __shfl_sync(0xffffffffu, rid, min(t, 31));
                            x[u] = (on && t < m) ? __ldg(X4 + (int64_t)r * k4 + cc + c4) : z4;
                        }
#pragma unroll
                        for (int u = 0; u < SK_U; u++) add4(a0, a1, a2, a3, x[u]);
                    }
                }
                for (int sl = 1; sl < R; sl++) {
                    const int src = min(31, lane + sl * k4c);
                    const double b0 = __shfl_sync(0xffffffffu, a0, src);
                    const double b1 = __shfl_sync(0xffffffffu, a1, src);
                    const double b2 = __shfl_sync(0xffffffffu, a2, src);
                    const double b3 = __shfl_sync(0xffffffffu, a3, src);
                    if (slot == 0) { a0 += b0; a1 += b1; a2 += b2; a3 += b3; }
                }
                if (slot == 0)
                    S4[(g0 + jj - g_lo) * k4 + cc + c4] =
                        make_float4((float)a0, (float)a1, (float)a2, (float)a3);
            }
        }
    }
}

// ------------------------------------------------------------ leaf gather
__global__ void __launch_bounds__(256)
leaf_gather_kernel(const int32_t* __restrict__ codes, int64_t n, int Bl,
                   const int64_t* __restrict__ leaf_base, const float4* __restrict__ S4, int k,
                   int k4, double scale, int accumulate, double* __restrict__ Y)
{
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int cc = 0; cc < k4; cc += 32) {
        const int k4c = min(32, k4 - cc);
        const int R = 32 / k4c;
        const int slot = lane / k4c, c4 = lane % k4c;
        const bool on = slot < R;
        const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int64_t i = warp; i < n; i += nwarps) {
            const int32_t* row = codes + i * Bl;
            double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
            // global leaf ids of this lane's tree in the chunk (next chunk prefetched)
            int32_t cnext = lane < Bl ? __ldg(row + lane) : 0;
            for (int b0 = 0; b0 < Bl; b0 += 32) {
                const int bl = b0 + lane;
                const int32_t code = cnext;
                if (b0 + 32 + lane < Bl) cnext = __ldg(row + b0 + 32 + lane);
                const int64_t gl = bl < Bl ? leaf_base[bl] + (int64_t)code : 0;
                const int nb = min(32, Bl - b0);
                for (int t0 = 0; t0 < nb; t0 += R * SK_U) {
                    float4 x[SK_U];
#pragma unroll
                    for (int u = 0; u < SK_U; u++) {
                        const int t = t0 + u * R + slot;
                        const int64_t g = __shfl_sync(0xffffffffu, gl, min(t, 31));
                        x[u] = (on && t < nb) ? __ldg(S4 + g * k4 + cc + c4) : z4;
                    }
#pragma unroll
                    for (int u = 0; u < SK_U; u++) add4(a0, a1, a2, a3, x[u]);
                }
            }
            for (int sl = 1; sl < R; sl++) {
                const int src = min(31, lane + sl * k4c);
                const double b0 = __shfl_sync(0xffffffffu, a0, src);
                const double b1 = __shfl_sync(0xffffffffu, a1, src);
                const double b2 = __shfl_sync(0xffffffffu, a2, src);
                const double b3 = __shfl_sync(0xffffffffu, a3, src);
                if (slot == 0) { a0 += b0; a1 += b1; a2 += b2; a3 += b3; }
            }
            if (slot == 0) {
                const double v[4] = {a0, a1, a2, a3};
                double* y = Y + i * k + 4 * (cc + c4);
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    if (4 * (cc + c4) + q < k) {
                        const double val = scale * v[q];
                        y[q] = accumulate ? y[q] + val : val;
                    }
                }
            }
        }
    }
}

// ------------------------------------------------------------------ Gram
constexpr int GRAM_ROWS = 32;
constexpr int GRAM_THREADS = 256;

int gram_parts(int64_t n)
{
    return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 128), (int64_t)sm_count() * 4));
}

__global__ void __launch_bounds__(GRAM_THREADS)
gram_partial_kernel(const double* __restrict__ A, int lda, const double* __restrict__ Bm, int ldb,
                    int64_t n, int ka, int kb, int64_t rows_per_part, double* __restrict__ parts)
{
    // 4x4 register tiles of C over (ka x kb); row groups split this part's rows
    // and are combined in a fixed order through shared memory.
    extern __shared__ double gsm[];  // tiles x 16
    const int64_t r0 = blockIdx.x * rows_per_part;
    const int64_t r1 = min64(n, r0 + rows_per_part);
    const int TA = (ka + 3) / 4, TB = (kb + 3) / 4, tiles = TA * TB;
    const int groups = max(1, GRAM_THREADS / tiles);
    const int tid = threadIdx.x;
    const int g = tid / tiles;
    for (int e = tid; e < tiles * 16; e += GRAM_THREADS) gsm[e] = 0.0;
    __syncthreads();
    for (int tile0 = 0; tile0 < tiles; tile0 += GRAM_THREADS) {
        const int tile = tiles > GRAM_THREADS ? tile0 + tid : tid % tiles;
        const bool active = tile < tiles && g < groups;
        double acc[16];
#pragma unroll
        for (int e = 0; e < 16; e++) acc[e] = 0.0;
        const int ta = tile / TB, tb = tile % TB;
        if (active) {
            bool va[4], vb[4];
#pragma unroll
            for (int x = 0; x < 4; x++) {
                va[x] = 4 * ta + x < ka;
                vb[x] = 4 * tb + x < kb;
            }
            const int gstep = tiles > GRAM_THREADS ? 1 : groups;
            const int gi = tiles > GRAM_THREADS ? 0 : g;
            for (int64_t i = r0 + gi; i < r1; i += gstep) {
                double qa[4], qb[4];
#pragma unroll
                for (int x = 0; x < 4; x++) {
                    qa[x] = va[x] ? __ldg(A + i * lda + 4 * ta + x) : 0.0;
                    qb[x] = vb[x] ? __ldg(Bm + i * ldb + 4 * tb + x) : 0.0;
                }
#pragma unroll
                for (int x = 0; x < 4; x++)
#pragma unroll
                    for (int y = 0; y < 4; y++) acc[4 * x + y] += qa[x] * qb[y];
            }
        }
        if (tiles > GRAM_THREADS) {
            if (active)
#pragma unroll
                for (int e = 0; e < 16; e++) gsm[tile * 16 + e] = acc[e];
        } else {
            for (int gg = 0; gg < groups; gg++) {  // fixed combine order
                if (g == gg && active)
#pragma unroll
                    for (int e = 0; e < 16; e++) gsm[tile * 16 + e] += acc[e];
                __syncthreads();
            }
        }
        if (tiles <= GRAM_THREADS) break;
    }
    __syncthreads();
    double* out = parts + (int64_t)blockIdx.x * ka * kb;
    for (int e = tid; e < ka * kb; e += GRAM_THREADS) {
        const int a = e / kb, b = e % kb;
        out[e] = gsm[((a >> 2) * TB + (b >> 2)) * 16 + 4 * (a & 3) + (b & 3)];
    }
}

// C[:, c0:c0+kb] (row stride ldc) = sum over parts, fixed order
__global__ void gram_final_kernel(const double* __restrict__ parts, int nparts, int ka, int kb,
                                  double* __restrict__ C, int ldc, int c0)
{
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    const int E = ka * kb;
    if (e >= E) return;
    double s = 0.0;
    for (int q = 0; q < nparts; q++) s += parts[(int64_t)q * E + e];
    C[(e / kb) * ldc + c0 + e % kb] = s;
}

// --------------------------------------------------------- small matmul
__global__ void __launch_bounds__(256)
matmul_small_kernel(const double* __restrict__ Y, int64_t n, int ka, const double* __restrict__ M,
                    int kb, double* __restrict__ Z, float* __restrict__ Z32, int ld32)
{
    extern __shared__ double ysm[];  // 16 rows x ka
    constexpr int RB = 16;
    const int64_t r0 = blockIdx.x * (int64_t)RB;
    const int m = (int)min64(RB, n - r0);
    for (int e = threadIdx.x; e < RB * ka; e += blockDim.x) {
        const int r = e / ka;
        ysm[e] = r < m ? Y[(r0 + r) * ka + e % ka] : 0.0;
    }
    __syncthreads();
    const int wcols = Z32 ? max(kb, ld32) : kb;
    for (int e = threadIdx.x; e < RB * wcols; e += blockDim.x) {
        const int r = e / wcols, c = e % wcols;
        if (r >= m) continue;
        double s = 0.0;
        if (c < kb)
            for (int a = 0; a < ka; a++) s += ysm[r * ka + a] * __ldg(M + (int64_t)a * kb + c);
        if (c < kb) Z[(r0 + r) * kb + c] = s;
        if (Z32 && c < ld32) Z32[(r0 + r) * ld32 + c] = c < kb ? (float)s : 0.0f;
    }
}

}  // namespace rfxc

using namespace rfxc;

extern "C" int rfxc_normals(int64_t seed, int64_t seq, int64_t count, double* d_out, void* stream)
{
    if (count < 0) return fail(RFXC_EDATA, "normals: negative count");
    if (count == 0) return RFXC_OK;
    uint64_t s[2];
    rfx_pcg32_make(seed, seq, s);
    const int64_t threads = ceil_div(ceil_div(count, 2), NORMAL_PAIRS_PER_THREAD);
    normals_kernel<<<(unsigned)ceil_div(threads, 128), 128, 0, as_stream(stream)>>>(s[0], s[1],
                                                                                   count, d_out);
    return check_launch("normals");
}

extern "C" int rfxc_pack_f32(const double* d_in, int64_t n, int32_t k, int32_t ld, float* d_out,
                             void* stream)
{
    if (n < 1 || k < 1 || ld < k) return fail(RFXC_EDATA, "pack_f32: bad shape");
    int grid = (int)std::min<int64_t>(ceil_div(n * ld, 256), (int64_t)sm_count() * 16);
    pack_f32_kernel<<<grid, 256, 0, as_stream(stream)>>>(d_in, n, k, ld, d_out);
    return check_launch("pack_f32");
}

extern "C" int rfxc_leaf_sums(const int32_t* d_perm, const int64_t* d_seg, int64_t g_lo,
                              int64_t g_hi, const float* d_X, int32_t k, int32_t ld, float* d_S,
                              void* stream)
{
    if (g_lo < 0 || g_hi < g_lo || k < 1 || ld < k || (ld & 3))
        return fail(RFXC_EDATA, "leaf_sums: bad shape (ld must be a multiple of 4 >= k)");
    if (g_hi == g_lo) return RFXC_OK;
    const int64_t warps = g_hi - g_lo;
    int grid = (int)std::min<int64_t>(ceil_div(warps, 8), (int64_t)sm_count() * 32);
    leaf_sums_kernel<<<grid, 256, 0, as_stream(stream)>>>(
        d_perm, d_seg, g_lo, g_hi, reinterpret_cast<const float4*>(d_X), ld / 4,
        reinterpret_cast<float4*>(d_S));
    return check_launch("leaf_sums");
}

extern "C" int rfxc_leaf_gather(const int32_t* d_codes_nb, int64_t n, int32_t Bl,
                                const int64_t* d_leaf_base, const float* d_S, int32_t k,
                                int32_t ld, double scale, int32_t accumulate, double* d_Y,
                                void* stream)
{
    if (n < 1 || Bl < 1 || k < 1 || ld < k || (ld & 3))
        return fail(RFXC_EDATA, "leaf_gather: bad shape");
    int grid = (int)std::min<int64_t>(ceil_div(n, 8), (int64_t)sm_count() * 32);
    leaf_gather_kernel<<<grid, 256, 0, as_stream(stream)>>>(
        d_codes_nb, n, Bl, d_leaf_base, reinterpret_cast<const float4*>(d_S), k, ld / 4, scale,
        accumulate, d_Y);
    return check_launch("leaf_gather");
}

extern "C" int rfxc_gram_parts(int64_t n) { return gram_parts(n); }

extern "C" int rfxc_gram(const double* d_A, const double* d_B, int64_t n, int32_t ka, int32_t kb,
                         double* d_partials, double* d_C, void* stream)
{
    // d_partials must hold rfxc_gram_parts(n) * ka * kb doubles
    if (n < 1 || ka < 1 || kb < 1 || ka > 64 * GRAM_THREADS)
        return fail(RFXC_EDATA, "gram: bad shape ka=%d kb=%d", ka, kb);
    cudaStream_t st = as_stream(stream);
    const int parts = gram_parts(n);
    const int64_t rpp = ceil_div(n, parts);
    // columns per launch: at most 768 4x4 tiles (96 KB of tile accumulators)
    const int TA = (ka + 3) / 4;
    const int kbc = std::max(4, std::min<int>((kb + 3) / 4 * 4, 4 * (768 / TA)));
    for (int c0 = 0; c0 < kb; c0 += kbc) {
        const int w = std::min(kbc, kb - c0);
        const size_t smem = (size_t)TA * ((w + 3) / 4) * 16 * 8;
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(gram_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
        gram_partial_kernel<<<parts, GRAM_THREADS, smem, st>>>(d_A, ka, d_B + c0, kb, n, ka, w, rpp,
                                                               d_partials);
        int rc = check_launch("gram_partial");
        if (rc) return rc;
        gram_final_kernel<<<(unsigned)ceil_div((int64_t)ka * w, 256), 256, 0, st>>>(
            d_partials, parts, ka, w, d_C, kb, c0);
        rc = check_launch("gram_final");
        if (rc) return rc;
    }
    return RFXC_OK;
}

extern "C" int rfxc_matmul_small(const double* d_Y, int64_t n, int32_t ka, const double* d_M,
                                 int32_t kb, double* d_Z, float* d_Z32, int32_t ld32, void* stream)
{
    if (n < 1 || ka < 1 || kb < 1) return fail(RFXC_EDATA, "matmul_small: bad shape");
    const size_t smem = (size_t)16 * ka * 8;
    matmul_small_kernel<<<(unsigned)ceil_div(n, 16), 256, smem, as_stream(stream)>>>(
        d_Y, n, ka, d_M, kb, d_Z, d_Z32, ld32);
    return check_launch("matmul_small");
}
