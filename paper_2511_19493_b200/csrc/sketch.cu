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
#include <cooperative_groups.h>

#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace rfxc {

// --------------------------------------------------------------- normals
#ifndef RFXC_NORMAL_PAIRS
#define RFXC_NORMAL_PAIRS 16
#endif
constexpr int NORMAL_PAIRS_PER_THREAD = RFXC_NORMAL_PAIRS;

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
        int64_t i;
        int c;
        if (total < (int64_t(1) << 32)) {  // 32-bit index math
            i = (int64_t)((uint32_t)e / (uint32_t)ld);
            c = (int)((uint32_t)e - (uint32_t)i * (uint32_t)ld);
        } else {
            i = e / ld;
            c = (int)(e % ld);
        }
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
                    const int32_t rid = lane < m ? (__ldg(perm + base + lane) & 0x7fffffff) : 0;
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
// C = A^T B for skinny row-major f64 A (n, ka), B (n, kb) on the FP64 tensor
// cores: every warp walks 4-row steps of its CTA's contiguous row range,
// loading A^T (8 x 4) and B (4 x 8) fragments straight from the rows and
// accumulating all (ka/8 x kb/8) output tiles in registers with DMMA.8x8x4;
// the CTA's warps are combined in a fixed order in shared memory and one warp
// per entry then adds the per-CTA partials in block order.  Deterministic.
constexpr int GRAM_THREADS = 256;

// partial-sum slots a Gram launch may write (the staged kernel uses up to one
// part per SM of >= 64 rows, the fallback up to two per SM of >= 256 rows)
int gram_parts(int64_t n)
{
    const int64_t staged = std::min<int64_t>(ceil_div(n, 64), (int64_t)sm_count());
    const int64_t fallback = std::min<int64_t>(ceil_div(n, 256), (int64_t)sm_count() * 2);
    return (int)std::max<int64_t>(1, std::max(staged, fallback));
}

// TAM x TBM accumulator tiles (compile-time indices); runtime TA <= TAM, TB <= TBM
template <int TAM, int TBM>
__global__ void __launch_bounds__(GRAM_THREADS, 2)
gram_partial_kernel(const double* __restrict__ A, int lda, const double* __restrict__ Bm, int ldb,
                    int64_t n, int ka, int kb, int64_t rows_per_part, double* __restrict__ parts)
{
    extern __shared__ double gsm[];  // TA*TB tiles x 64
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t r0 = blockIdx.x * rows_per_part;
    const int64_t r1 = min64(n, r0 + rows_per_part);
    const int TA = (ka + 7) / 8, TB = (kb + 7) / 8;
    double acc[TAM][TBM][2];
#pragma unroll
    for (int x = 0; x < TAM; x++)
#pragma unroll
        for (int y = 0; y < TBM; y++) acc[x][y][0] = acc[x][y][1] = 0.0;
    const int fr = lane & 3, fc = lane >> 2;  // fragment row (k) / column
    double af[TAM], bf[TBM], an[TAM], bn[TBM];
    auto load = [&](int64_t base, double* fa, double* fb) {
        const int64_t row = base + fr;
        const bool rv = row < r1;
#pragma unroll
        for (int x = 0; x < TAM; x++) {
            const int c = 8 * x + fc;
            fa[x] = (rv && x < TA && c < ka) ? __ldg(A + row * lda + c) : 0.0;
        }
#pragma unroll
        for (int y = 0; y < TBM; y++) {
            const int c = 8 * y + fc;
            fb[y] = (rv && y < TB && c < kb) ? __ldg(Bm + row * ldb + c) : 0.0;
        }
    };
    int64_t base = r0 + 4 * warp;
    load(base, af, bf);
    for (; base < r1; base += 4 * nw) {
        load(base + 4 * nw, an, bn);  // next step's fragments in flight
#pragma unroll
        for (int x = 0; x < TAM; x++)
#pragma unroll
            for (int y = 0; y < TBM; y++)
                if (x < TA && y < TB) dmma884(acc[x][y][0], acc[x][y][1], af[x], bf[y]);
#pragma unroll
        for (int x = 0; x < TAM; x++) af[x] = an[x];
#pragma unroll
        for (int y = 0; y < TBM; y++) bf[y] = bn[y];
    }
    // every warp parks its tiles, then one fixed-order sum over the warps
    const int tiles = TA * TB;
#pragma unroll
    for (int x = 0; x < TAM; x++)
#pragma unroll
        for (int y = 0; y < TBM; y++) {
            if (x < TA && y < TB) {
                double* d = gsm + ((int64_t)warp * tiles + x * TB + y) * 64 + fc * 8 + 2 * fr;
                d[0] = acc[x][y][0];
                d[1] = acc[x][y][1];
            }
        }
    __syncthreads();
    double* out = parts + (int64_t)blockIdx.x * ka * kb;
    for (int e = threadIdx.x; e < ka * kb; e += blockDim.x) {
        const int a = e / kb, b = e % kb;
        const int64_t off = ((a >> 3) * TB + (b >> 3)) * 64 + (a & 7) * 8 + (b & 7);
        double v = 0.0;
        for (int w = 0; w < nw; w++) v += gsm[(int64_t)w * tiles * 64 + off];
        out[e] = v;
    }
}

// C[:, c0:c0+kb] (row stride ldc) = sum over parts in block order, warp per entry
__global__ void gram_final_kernel(const double* __restrict__ parts, int nparts, int ka, int kb,
                                  double* __restrict__ C, int ldc, int c0, int a0)
{
    const int lane = threadIdx.x & 31;
    const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int E = ka * kb;
    if (e >= E) return;
    double s = 0.0;
    for (int q = lane; q < nparts; q += 32) s += parts[(int64_t)q * E + e];
    s = warp_sum(s);
    if (lane == 0) C[(a0 + e / kb) * ldc + c0 + e % kb] = s;
}

// Staged Gram (ka, kb <= 128): a CTA per SM streams its contiguous row range
// through shared memory in 32-row chunks (cp.async, zero-filled past the
// end, next chunk in flight while the current one is multiplied) and every
// warp owns whole 8x8 output tiles (upper tiles only when A == B), so no
// cross-warp reduction is needed; the CTA's tiles go to parts[blk] and
// gram_final adds the parts in block order.  Deterministic.
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// rows per staged chunk: 64 (measured best) when two stages fit the shared
// memory, else 32 (wide non-symmetric Grams)
constexpr int GS_CH_BIG = 64, GS_CH_SMALL = 32;
constexpr int GS_MAXST = 8;

// wait until at most n (< GS_MAXST) cp.async groups of this thread are pending
__device__ __forceinline__ void cp_async_wait_dyn(int n)
{
    switch (n) {
        case 0: cp_async_wait<0>(); break;
        case 1: cp_async_wait<1>(); break;
        case 2: cp_async_wait<2>(); break;
        case 3: cp_async_wait<3>(); break;
        case 4: cp_async_wait<4>(); break;
        case 5: cp_async_wait<5>(); break;
        case 6: cp_async_wait<6>(); break;
        default: cp_async_wait<7>(); break;
    }
}

__device__ __forceinline__ void cp_async8z(void* smem, const void* gmem, bool ok)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int n = ok ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}

__host__ __device__ inline int gs_ld(int cols) { return cols + ((4 - cols % 16) + 16) % 16; }

constexpr int GS_THREADS = 512;

template <int MT, int GS_CH>
__global__ void __launch_bounds__(GS_THREADS, 1)
gram_stage_kernel(const double* __restrict__ A, const double* __restrict__ Bm, int64_t n, int ka,
                  int kb, int sym, int64_t rpp, int nst, double* __restrict__ parts)
{
    extern __shared__ __align__(16) double gss[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int fr = lane & 3, fc = lane >> 2;
    const int TA = (ka + 7) / 8, TB = (kb + 7) / 8;
    const int lsa = gs_ld(8 * TA), lsb = sym ? lsa : gs_ld(8 * TB);
    const int per = GS_CH * (lsa + (sym ? 0 : lsb));
    const int64_t r0 = blockIdx.x * rpp, r1 = min64(n, r0 + rpp);
    const int NT = sym ? TA * (TA + 1) / 2 : TA * TB;
    int ta[MT], tb[MT];
#pragma unroll
    for (int m = 0; m < MT; m++) {
        int t = warp + (GS_THREADS / 32) * m, a = 0, b = -1;
        if (t < NT) {
            if (sym) {
                while (t >= TA - a) { t -= TA - a; a++; }
                b = a + t;
            } else {
                a = t / TB;
                b = t % TB;
            }
        }
        ta[m] = a;
        tb[m] = b;
    }
    double acc[MT][2];
#pragma unroll
    for (int m = 0; m < MT; m++) acc[m][0] = acc[m][1] = 0.0;
    // each thread copies a fixed column of every rstep-th row of a chunk
    const int GA = 8 * TA, GB = 8 * TB;
    const int ca = threadIdx.x % GA, ra0 = threadIdx.x / GA, rsa = (int)blockDim.x / GA;
    const int cb = threadIdx.x % GB, rb0 = threadIdx.x / GB, rsb = (int)blockDim.x / GB;
    // (threads beyond rsa * GA / rsb * GB copy nothing: with GA not dividing
    // the block, their rows would repeat other threads' rows — a write-write
    // race compute-sanitizer's racecheck reported)
    auto stage = [&](int64_t c, int buf) {
        double* sa = gss + buf * per;
        if (ra0 < GS_CH && ra0 < rsa)
            for (int row = ra0; row < GS_CH; row += rsa) {
                const int64_t g = c + row;
                const bool ok = g < r1 && ca < ka;
                cp_async8z(sa + row * lsa + ca, ok ? A + g * ka + ca : A, ok);
            }
        if (!sym && rb0 < GS_CH && rb0 < rsb) {
            double* sb = sa + GS_CH * lsa;
            for (int row = rb0; row < GS_CH; row += rsb) {
                const int64_t g = c + row;
                const bool ok = g < r1 && cb < kb;
                cp_async8z(sb + row * lsb + cb, ok ? Bm + g * kb + cb : Bm, ok);
            }
        }
        cp_async_commit();
    };
    // nst-deep pipeline: chunks it+1 .. it+nst-1 in flight while chunk it is used
    const int nch = (int)((r1 - r0 + GS_CH - 1) / GS_CH);
    for (int j = 0; j < nst - 1; j++) {
        if (j < nch) stage(r0 + (int64_t)j * GS_CH, j);
        else cp_async_commit();
    }
    int bl = nst - 1, bu = 0;  // buffer to load into / to use
    for (int it = 0; it < nch; it++) {
        // chunk it has landed (this thread's copies; the barrier makes every
        // thread's visible) and every warp is done with chunk it - 1, whose
        // buffer the next stage overwrites (compute-sanitizer racecheck)
        cp_async_wait_dyn(nst - 2);
        __syncthreads();
        const int nx = it + nst - 1;
        if (nx < nch) stage(r0 + (int64_t)nx * GS_CH, bl);
        else cp_async_commit();
        bl = bl + 1 == nst ? 0 : bl + 1;
        const double* sa = gss + bu * per;
        const double* sb = sym ? sa : sa + GS_CH * lsa;
        bu = bu + 1 == nst ? 0 : bu + 1;
#pragma unroll
        for (int ks = 0; ks < GS_CH / 4; ks++) {
            const double* ra = sa + (4 * ks + fr) * lsa + fc;
            const double* rb = sb + (4 * ks + fr) * lsb + fc;
#pragma unroll
            for (int m = 0; m < MT; m++)
                if (tb[m] >= 0) dmma884(acc[m][0], acc[m][1], ra[8 * ta[m]], rb[8 * tb[m]]);
        }
    }
    double* out = parts + (int64_t)blockIdx.x * ka * kb;
#pragma unroll
    for (int m = 0; m < MT; m++) {
        if (tb[m] < 0) continue;
        const int a = 8 * ta[m] + fc;
#pragma unroll
        for (int j = 0; j < 2; j++) {
            const int b = 8 * tb[m] + 2 * fr + j;
            if (a < ka && b < kb) {
                out[a * kb + b] = acc[m][j];
                if (sym && ta[m] != tb[m]) out[b * kb + a] = acc[m][j];
            }
        }
    }
}

template <int MT, int GS_CH>
static void gram_stage_go(const double* d_A, const double* d_B, int64_t n, int ka, int kb, int sym,
                          int parts, int64_t rpp, double* d_partials, cudaStream_t st)
{
    const int TA = (ka + 7) / 8, TB = (kb + 7) / 8;
    const size_t per = (size_t)GS_CH * (gs_ld(8 * TA) + (sym ? 0 : gs_ld(8 * TB))) * 8;
    const int nst = (int)std::max<size_t>(2, std::min<size_t>(GS_MAXST, (size_t)(200 * 1024) / per));
    const size_t smem = per * nst;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(gram_stage_kernel<MT, GS_CH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024);
        attr = true;
    }
    gram_stage_kernel<MT, GS_CH><<<parts, GS_THREADS, smem, st>>>(d_A, d_B, n, ka, kb, sym, rpp, nst,
                                                                   d_partials);
}

template <int MT>
static int launch_gram_stage(const double* d_A, const double* d_B, int64_t n, int ka, int kb,
                             double* d_partials, double* d_C, cudaStream_t st)
{
    const int sym = (d_A == d_B && ka == kb) ? 1 : 0;
    const int parts = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 64), sm_count()));
    const int64_t rpp = ceil_div(n, parts);
    const int TA = (ka + 7) / 8, TB = (kb + 7) / 8;
    const size_t per_big = (size_t)GS_CH_BIG * (gs_ld(8 * TA) + (sym ? 0 : gs_ld(8 * TB))) * 8;
    if (2 * per_big <= (size_t)200 * 1024)
        gram_stage_go<MT, GS_CH_BIG>(d_A, d_B, n, ka, kb, sym, parts, rpp, d_partials, st);
    else
        gram_stage_go<MT, GS_CH_SMALL>(d_A, d_B, n, ka, kb, sym, parts, rpp, d_partials, st);
    int rc = check_launch("gram_stage");
    if (rc) return rc;
    gram_final_kernel<<<(unsigned)ceil_div((int64_t)ka * kb * 32, 256), 256, 0, st>>>(
        d_partials, parts, ka, kb, d_C, kb, 0, 0);
    return check_launch("gram_final");
}

// --------------------------------------------------------- small matmul
// Z (n, kb) = Y (n, ka) M (ka, kb) on the FP64 tensor cores, optional zero-
// padded f32 copy (n, ld32).  M (zero-padded to 4-row x 8-column tiles) sits
// in shared memory; a warp computes 8-row blocks: A fragments straight from
// the rows of Y, all kb/8 output tiles in registers.
constexpr int MM_MAXTB = 16;  // kb <= 128

template <int TBM>
__global__ void __launch_bounds__(256)
matmul_small_kernel(const double* __restrict__ Y, int64_t n, int ka, const double* __restrict__ M,
                    int kb, double* __restrict__ Z, float* __restrict__ Z32, int ld32)
{
    extern __shared__ double msm[];  // [KS*4 x TBM*8] zero-padded M
    const int KS = (ka + 3) / 4;
    constexpr int mw = TBM * 8;
    for (int e = threadIdx.x; e < KS * 4 * mw; e += blockDim.x) {
        const int a = e / mw, c = e % mw;
        msm[e] = (a < ka && c < kb) ? M[a * kb + c] : 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int fr = lane & 3, fc = lane >> 2;
    const int64_t nblk = (n + 7) / 8;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t blk = gw; blk < nblk; blk += nwarps) {
        const int64_t arow = blk * 8 + fc;  // A fragment row (lane / 4)
        const bool av = arow < n;
        double acc[TBM][2];
#pragma unroll
        for (int t = 0; t < TBM; t++) acc[t][0] = acc[t][1] = 0.0;
        for (int k0 = 0; k0 < KS; k0 += 8) {  // 8 k-steps of A fragments in flight
            double a[8];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const int c = 4 * (k0 + u) + fr;
                a[u] = (av && k0 + u < KS && c < ka) ? __ldg(Y + arow * ka + c) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; u++) {
                if (k0 + u < KS) {
                    const double* mrow = msm + (4 * (k0 + u) + fr) * mw + fc;
#pragma unroll
                    for (int t = 0; t < TBM; t++) dmma884(acc[t][0], acc[t][1], a[u], mrow[8 * t]);
                }
            }
        }
        const int64_t orow = blk * 8 + fc;  // output row (lane / 4)
        if (orow < n) {
#pragma unroll
            for (int t = 0; t < TBM; t++) {
                const int c = 8 * t + 2 * fr;
                if (c < kb) Z[orow * kb + c] = acc[t][0];
                if (c + 1 < kb) Z[orow * kb + c + 1] = acc[t][1];
                if (Z32) {
                    if (c < ld32) Z32[orow * ld32 + c] = c < kb ? (float)acc[t][0] : 0.0f;
                    if (c + 1 < ld32) Z32[orow * ld32 + c + 1] = c + 1 < kb ? (float)acc[t][1] : 0.0f;
                }
            }
        }
    }
}

// ============================================================ fused pass
// One sketch pass Y = scale * sum_b E_b E_b^T X.  Trees are processed in
// batches of T <= 32 whose leaf sums fit next to X in L2 (rfxc_sketch_plan),
// so the leaf sums never round-trip HBM, where the two-kernel path writes all
// sum(L) x ld sums and gathers them back per (sample, tree).  Per batch two
// launches on one stream (phase A on an auxiliary stream when two leaf-sum
// buffers fit, overlapping the previous batch's phase B):
//
// Phase A (skp_phase_a; one item of positions of the bucketed perm per
// resident warp): three row slots of k4 float4 lanes walk 32-position
// sub-chunks in order, gathering X rows, summing each leaf segment in f32
// (<= 32 rows) and closing a leaf at every RFXC_PERM_FIRST flag; the slots'
// cut segments are joined in position order in an f64 carry.  Leaves cut by
// an item boundary leave one f64 piece per item; the last piece to arrive
// (acq_rel per-leaf counter) adds the pieces in item order and writes the
// sum, so results are bit-reproducible.
// Phase B (skp_phase_b; 24 samples per warp): lane t reads the sample's code
// in tree b0+t (one coalesced segment of the (n, B) membership), the T
// leaf-sum rows are gathered as float4 lanes and summed in f32, and the sum
// is added to Y in f64 (scaled by 1/B in the last batch).
constexpr int SKP_SAMPLES = 24;  // max samples per phase-B item (A.spw: one wave of resident warps)
constexpr int SKP_RMAX = 4;      // row slots per warp (lane groups of k4 lanes)
constexpr int SKP_MAX_T = 32;

struct SkpLayout {
    int64_t S, part, cnt, ctr, item_leaf, ypart, total;
};

__host__ __device__ inline int64_t align256(int64_t x) { return (x + 255) / 256 * 256; }

__host__ __device__ inline int64_t skp_items_per_batch(int64_t n, int T, int64_t item)
{
    return (T * n + item - 1) / item;
}

__host__ __device__ inline int skp_nbatch(int Bl, int T) { return (Bl + T - 1) / T; }

__host__ __device__ inline SkpLayout skp_layout(int64_t n, int Bl, int T, int ld, int k,
                                                int64_t s_rows, int nbuf, int64_t item)
{
    SkpLayout L;
    const int64_t ipb = skp_items_per_batch(n, T, item);
    const int nb = skp_nbatch(Bl, T);
    int64_t off = 0;
    L.S = off;         off += align256(nbuf * s_rows * ld * 4);
    L.part = off;      off += align256(2 * ipb * ld * 8);
    L.cnt = off;       off += align256(s_rows * 4);
    L.ctr = off;       off += align256(2 * (int64_t)(nb + 1) * 4);
    L.item_leaf = off; off += align256(nb * ipb * 4);
    L.ypart = off;     off += align256((int64_t)nb * n * ld * 4);  // per-batch f32 sums of phase B
    L.total = off;
    return L;
}

struct SkpArgs {
    const uint32_t* perm;
    const int64_t* seg;
    const int32_t* codes;      // (n, Bl)
    const int64_t* leaf_base;  // (Bl + 1)
    const int32_t* has_empty;
    const float* X;            // (n, ld)
    double* Y;                 // (n, k)
    float* P;                  // nbatch x n x ld: phase B's f32 batch sums (null: Y read-modify-write)
    float* S;                  // 2 x s_rows x ld
    double* part;              // ipb x 2 x k
    int32_t* cnt;              // s_rows
    unsigned* ctr;             // 2 x (nbatch + 1)
    const int32_t* item_leaf;  // nbatch x ipb
    int64_t n, s_rows, ipb, item;
    int spw;                   // phase-B samples per warp
    int Bl, k, ld, T, nbatch;
    int nbuf;                  // leaf-sum buffers (1: A(e), B(e) on one stream)
    double scale;
    unsigned long long* timing;  // unused
};

// item_leaf[e * ipb + it]: global leaf containing the first position of item
// it of batch e (last g with seg[g] <= P < seg[g + 1]).
__global__ void skp_item_leaf_kernel(const int64_t* __restrict__ seg,
                                     const int64_t* __restrict__ leaf_base, int64_t n, int Bl,
                                     int T, int64_t ipb, int64_t item, int32_t* __restrict__ item_leaf)
{
    const int nb = skp_nbatch(Bl, T);
    const int64_t total = nb * ipb;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int e = (int)(q / ipb);
        const int64_t it = q % ipb;
        const int b0 = e * T, b1 = min(Bl, b0 + T);
        const int64_t P = (int64_t)b0 * n + it * item;
        if (P >= (int64_t)b1 * n) {
            item_leaf[q] = -1;
            continue;
        }
        int64_t a = leaf_base[b0], z = leaf_base[b1];  // answer in [a, z)
        while (z - a > 1) {
            const int64_t m = (a + z) >> 1;
            if (seg[m] <= P) a = m;
            else z = m;
        }
        item_leaf[q] = (int32_t)a;
    }
}



// Emit one finished (or cut) leaf segment held by the slot-0 lanes (lane c4
// owns columns 4c4..4c4+3 in f64).  kind: 0 = whole leaf, 1 = first segment
// of the item cut at its start, 2 = last segment cut at its end, 3 = both
// (the item lies inside the leaf).  Cut segments leave an f64 piece per item;
// the last piece to arrive adds them in item order and writes the sum.
// leaf of bucketed position P: the last g in [lo, hi) with seg[g] <= P (an
// empty leaf shares its start with the next one, so it is never returned)
__device__ __forceinline__ int skp_leaf_at(const int64_t* __restrict__ seg, int lo, int hi, int64_t P)
{
    while (hi - lo > 1) {
        const int m = (lo + hi) >> 1;
        if (__ldg(seg + m) <= P) lo = m;
        else hi = m;
    }
    return lo;
}

__device__ __forceinline__ int atom_add_acq_rel_gpu(int32_t* p, int v)
{
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ void skp_emit(const SkpArgs& A, double a0, double a1, double a2,
                                         double a3, int64_t g, int kind, int64_t it, int64_t pos0,
                                         int64_t g0, float4* Sb, int lane, bool lead)
{
    const double acc[4] = {a0, a1, a2, a3};
    const int k4 = A.ld >> 2;
    if (kind == 0) {
        if (lead) Sb[(g - g0) * k4 + lane] = make_float4((float)acc[0], (float)acc[1],
                                                         (float)acc[2], (float)acc[3]);
        return;
    }
    const int slot = kind == 2 ? 1 : 0;
    double* pp = A.part + (it * 2 + slot) * A.ld + 4 * lane;
    if (lead) {
#pragma unroll
        for (int q = 0; q < 4; q++) __stcg(pp + q, acc[q]);
    }
    // the warp barrier orders the lanes' piece stores before lane 0's release;
    // the last arriver's acquire (and the barrier of the shuffle) orders the
    // piece loads after every other item's release
    __syncwarp();
    int last = 0;
    if (lane == 0) {
        const int64_t s = A.seg[g], e = A.seg[g + 1];
        const int npieces = (int)(((e - 1 - pos0) / A.item) - ((s - pos0) / A.item)) + 1;
        const int old = atom_add_acq_rel_gpu(A.cnt + (g - g0), 1);
        last = (old == npieces - 1);
        if (last) A.cnt[g - g0] = 0;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return;
    if (lead) {
        const int64_t s = A.seg[g], e = A.seg[g + 1];
        const int64_t i0 = (s - pos0) / A.item, i1 = (e - 1 - pos0) / A.item;
        double t[4] = {0.0, 0.0, 0.0, 0.0};
        for (int64_t j = i0; j <= i1; j++) {
            const double* src = A.part + (j * 2 + (j == i0 ? 1 : 0)) * A.ld + 4 * lane;
#pragma unroll
            for (int q = 0; q < 4; q++) t[q] += __ldcg(src + q);
        }
        Sb[(g - g0) * k4 + lane] = make_float4((float)t[0], (float)t[1], (float)t[2], (float)t[3]);
    }
}

__device__ __forceinline__ void f4add(float4& a, const float4 x)
{
    a.x += x.x;
    a.y += x.y;
    a.z += x.z;
    a.w += x.w;
}

// slot partials (lane = slot * k4 + c4) -> slot 0, fixed order
__device__ __forceinline__ void slot_combine(float4& a, int R, int k4, int slot, int lane)
{
    for (int sl = 1; sl < R; sl++) {
        const int src = min(31, lane + sl * k4);
        const float ox = __shfl_sync(0xffffffffu, a.x, src);
        const float oy = __shfl_sync(0xffffffffu, a.y, src);
        const float oz = __shfl_sync(0xffffffffu, a.z, src);
        const float ow = __shfl_sync(0xffffffffu, a.w, src);
        if (slot == 0) {
            a.x += ox;
            a.y += oy;
            a.z += oz;
            a.w += ow;
        }
    }
}

// Per-warp shared scratch: SKP_RMAX x 32 uint32 (phase A perm values /
// phase B leaf-sum row ids).
// slot stride 36 words: the slots' same-position entries fall in different
// bank groups (a stride of 32 made every slot read hit the same bank)
constexpr int SKP_SLOT = 36;
constexpr int SKP_SCRATCH = SKP_RMAX * SKP_SLOT + 2 * 32 * 4;  // + head/tail float4 per lane
constexpr int SKP_UA = 4;
#ifndef SKP_BRANCHLESS_A
#define SKP_BRANCHLESS_A 1
#endif
#ifndef SKP_JOIN_SHFL
#define SKP_JOIN_SHFL 1
#endif
#ifndef SKP_FUSE_FINAL
#define SKP_FUSE_FINAL 1
#endif
#ifndef SKP_BL_UNROLL
#define SKP_BL_UNROLL 2
#endif
constexpr int kSkpBlUnroll = SKP_BL_UNROLL;
#ifndef SKP_MINB_A
#define SKP_MINB_A 3
#endif   // phase A row loads in flight per lane
#ifndef SKP_UB_DEF
#define SKP_UB_DEF 4
#endif
#ifndef SKP_MINB_B
#define SKP_MINB_B 4
#endif
constexpr int SKP_UB = SKP_UB_DEF;  // phase B row loads in flight per lane

// Phase A item: positions [P0, P1) of batch e, in steps of R sub-chunks of
// 32 positions.  Slot s (lanes s*k4 .. s*k4+k4-1, lane c4 owning float4
// column c4) walks sub-chunk s of the step in position order with coalesced
// row loads (SKP_UA in flight), summing each leaf segment in f32 and writing
// the leaf sums of segments that start and end inside its sub-chunk.  The
// segments cut by sub-chunk boundaries (head / tail partials of every slot)
// are then joined in position order into one f64 carry held by every slot,
// which is emitted when its leaf ends (a piece when cut by the item edge).
// Leaf ids follow from the first-member flags, or, when the bucketing saw an
// empty leaf (device flag, uniform), from a search of the run starts.
template <int K4>
__device__ void skp_phase_a(const SkpArgs& A, int e, int64_t it, uint32_t* pbuf, int lane)
{
    const int b0 = e * A.T, b1 = min(A.Bl, b0 + A.T);
    const int64_t pos0 = (int64_t)b0 * A.n, pend = (int64_t)b1 * A.n;
    const int64_t P0 = pos0 + it * A.item, P1 = min64(P0 + A.item, pend);
    const int g0 = (int)A.leaf_base[b0];
    float4* Sb = reinterpret_cast<float4*>(A.S + (int64_t)(e % A.nbuf) * A.s_rows * A.ld);
    const int k4 = K4 ? K4 : (A.ld >> 2);  // compile-time for the common widths
    const int R = min(SKP_RMAX, 32 / k4);
    const int slot = lane / k4, c4 = lane - slot * k4;
    const bool on = slot < R;
    const int nsub = (int)((P1 - P0 + 31) >> 5);
    const float4* X4 = reinterpret_cast<const float4*>(A.X);
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);

    int tail_first = 1;
    if (lane == 0 && P1 < pend) tail_first = (__ldg(A.perm + P1) & RFXC_PERM_FIRST) != 0;
    const bool tail_open = !__shfl_sync(0xffffffffu, tail_first, 0);
    const int gi = A.item_leaf[(int64_t)e * A.ipb + it];
    const int gN = (int)A.leaf_base[b1];
    const bool he = *A.has_empty != 0;

    // carry: the open segment at the current position (f64, every lane holds
    // its column group), its leaf, whether it was cut at the item start and
    // whether it holds any row yet
    double cy[4] = {0.0, 0.0, 0.0, 0.0};
    int cleaf = gi;
    int ckind = 1;
    bool cvalid = false;
    int flags_before = 0;  // flagged positions in (P0, current sub-chunk start)

    uint32_t pv[SKP_RMAX];
    auto load_pv = [&](int s0) {
#pragma unroll
        for (int j = 0; j < SKP_RMAX; j++) {
            const int64_t q = P0 + 32 * (int64_t)(s0 + j) + lane;
            pv[j] = (j < R && s0 + j < nsub && q < P1) ? __ldcs(A.perm + q) : 0u;  // streamed once
        }
    };
    load_pv(0);
    for (int s0 = 0; s0 < nsub; s0 += R) {
        unsigned fl[SKP_RMAX];
        int mm[SKP_RMAX];
#pragma unroll
        for (int j = 0; j < SKP_RMAX; j++) {
            mm[j] = (int)max64(0, min64(32, P1 - (P0 + 32 * (int64_t)(s0 + j))));
            fl[j] = __ballot_sync(0xffffffffu, lane < mm[j] && (pv[j] & RFXC_PERM_FIRST));
            pbuf[j * SKP_SLOT + lane] = (pv[j] & ~RFXC_PERM_FIRST) * (uint32_t)k4;  // row offset in float4
        }
        if (s0 == 0 && (fl[0] & 1u)) { ckind = 0; }  // the item starts a leaf
        __syncwarp();
        if (s0 + R < nsub) load_pv(s0 + R);  // prefetch the next step's perm values
        // this slot's sub-chunk
        unsigned fs = 0;
        int m = 0;
        int before = flags_before;
#pragma unroll
        for (int j = 0; j < SKP_RMAX; j++) {
            const unsigned fj = (s0 == 0 && j == 0) ? (fl[j] & ~1u) : fl[j];  // P0 itself never counts
            if (j == slot) { fs = fl[j]; m = mm[j]; }
            if (j < slot) before += __popc(fj);
        }
        const bool first_sub = (s0 == 0 && slot == 0);
        // leaf of this slot's first position (first-member flags count leaves
        // unless some leaf is empty; then the run starts are searched)
        const int64_t q0 = P0 + 32 * (int64_t)(s0 + slot);
        int cur = he ? skp_leaf_at(A.seg, g0, gN, q0) : gi + before + ((fs & 1u) && !first_sub ? 1 : 0);
        bool inside = (fs & 1u) != 0;  // current segment started inside this sub-chunk
        float4 acc = z4;
        // this slot's head (segment before its first leaf start) and tail go
        // through shared memory to the join (one 16-byte access per lane)
        float4* hsm = reinterpret_cast<float4*>(pbuf + SKP_RMAX * SKP_SLOT);
        float4* tsm = hsm + 32;
        const uint32_t* pb = pbuf + (on ? slot : 0) * SKP_SLOT;  // idle lanes shadow slot 0
        const char* xb = reinterpret_cast<const char*>(X4 + c4);
        // leaf starts at p in (0, m)
        const unsigned fsx = (fs & ~1u) & (m >= 32 ? 0xffffffffu : ((1u << m) - 1u));
        auto flush = [&](int p) {
            if (inside) {
                if (on) Sb[(uint32_t)(cur - g0) * k4 + c4] = acc;
            } else {
                hsm[lane] = acc;
            }
            cur = he ? skp_leaf_at(A.seg, g0, gN, q0 + p) : cur + 1;
            inside = true;
        };  // the caller restarts acc with the row at p
        static_assert(SKP_UA == 4, "index loads are uint4");
        if (!he && P1 - (P0 + 32 * (int64_t)s0) >= 32 * R && SKP_BRANCHLESS_A) {
            // every slot has 32 positions and leaf ids follow the flags: no
            // branches.  Each leaf start p closes the running segment: the
            // first one of a slot that started outside a leaf closes the head
            // (-> shared memory), every other one the leaf at the running row
            // offset of S.  The masks are fixed per sub-chunk, so each row
            // costs three bit tests, the two predicated stores, the offset
            // step and the four (predicated) adds.
            const unsigned hm = inside ? 0u : (fsx & (0u - fsx));
            const unsigned smk = fsx & ~hm;
            uint32_t so = (uint32_t)(cur - g0) * k4 + c4;
#pragma unroll kSkpBlUnroll
            for (int p0 = 0; p0 < 32; p0 += 4) {
                const uint4 ix = *reinterpret_cast<const uint4*>(pb + p0);
                float4 x[4];
                x[0] = __ldg(reinterpret_cast<const float4*>(xb + ((size_t)ix.x << 4)));
                x[1] = __ldg(reinterpret_cast<const float4*>(xb + ((size_t)ix.y << 4)));
                x[2] = __ldg(reinterpret_cast<const float4*>(xb + ((size_t)ix.z << 4)));
                x[3] = __ldg(reinterpret_cast<const float4*>(xb + ((size_t)ix.w << 4)));
                const unsigned f = fsx >> p0, sf = smk >> p0, hf = hm >> p0;
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const bool fl = (f >> u) & 1u;
                    if ((sf >> u) & 1u) Sb[so] = acc;
                    if ((hf >> u) & 1u) hsm[lane] = acc;
                    so += fl ? (uint32_t)k4 : 0u;
                    acc.x = fl ? x[u].x : acc.x + x[u].x;
                    acc.y = fl ? x[u].y : acc.y + x[u].y;
                    acc.z = fl ? x[u].z : acc.z + x[u].z;
                    acc.w = fl ? x[u].w : acc.w + x[u].w;
                }
            }
            cur += __popc(fsx);
            inside = inside || fsx != 0u;
        } else if (P1 - (P0 + 32 * (int64_t)s0) >= 32 * R) {
            // every slot has 32 positions: no predicates (lanes past the last
            // slot re-read slot 0's rows and never store)
#pragma unroll 2
            for (int p0 = 0; p0 < 32; p0 += 4) {
                const uint4 ix = *reinterpret_cast<const uint4*>(pb + p0);
                const float4 x0 = __ldg(reinterpret_cast<const float4*>(xb + ((size_t)ix.x << 4)));
                const float4 x1 = __ldg(reinterpret_cast<const float4*>(xb + ((size_t)ix.y << 4)));
                const float4 x2 = __ldg(reinterpret_cast<const float4*>(xb + ((size_t)ix.z << 4)));
                const float4 x3 = __ldg(reinterpret_cast<const float4*>(xb + ((size_t)ix.w << 4)));
                const unsigned f4 = (fsx >> p0) & 0xFu;
                if (f4 == 0u) {
                    f4add(acc, x0);
                    f4add(acc, x1);
                    f4add(acc, x2);
                    f4add(acc, x3);
                } else {
                    if (f4 & 1u) { flush(p0); acc = x0; } else { f4add(acc, x0); }
                    if (f4 & 2u) { flush(p0 + 1); acc = x1; } else { f4add(acc, x1); }
                    if (f4 & 4u) { flush(p0 + 2); acc = x2; } else { f4add(acc, x2); }
                    if (f4 & 8u) { flush(p0 + 3); acc = x3; } else { f4add(acc, x3); }
                }
            }
        } else {
            for (int p0 = 0; p0 < 32; p0 += 4) {
                const uint4 ix = *reinterpret_cast<const uint4*>(pb + p0);
                const uint32_t ixs[4] = {ix.x, ix.y, ix.z, ix.w};
                float4 x[4];
#pragma unroll
                for (int u = 0; u < 4; u++)
                    x[u] = (on && p0 + u < m) ? __ldg(reinterpret_cast<const float4*>(xb + ((size_t)ixs[u] << 4))) : z4;
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    if ((fsx >> (p0 + u)) & 1u) {
                        flush(p0 + u);
                        acc = x[u];
                    } else {
                        f4add(acc, x[u]);
                    }
                }
            }
        }
        if (!SKP_JOIN_SHFL) tsm[lane] = acc;
        __syncwarp();
        // join the slots' cut segments in position order (uniform over the warp)
#pragma unroll
        for (int j = 0; j < SKP_RMAX; j++) {
            if (j >= R || s0 + j >= nsub) break;
            const int src = j * k4 + c4;
            float4 tj;
            if (SKP_JOIN_SHFL) {  // slot j's tail straight from its lanes' registers
                tj.x = __shfl_sync(0xffffffffu, acc.x, src);
                tj.y = __shfl_sync(0xffffffffu, acc.y, src);
                tj.z = __shfl_sync(0xffffffffu, acc.z, src);
                tj.w = __shfl_sync(0xffffffffu, acc.w, src);
            } else {
                tj = tsm[src];
            }
            const int curj = __shfl_sync(0xffffffffu, cur, j * k4);
            const unsigned fj = (s0 == 0 && j == 0) ? (fl[j] & ~1u) : fl[j];
            const bool starts = (fl[j] & 1u) != 0;
            if (fj == 0 && !starts) {  // the whole sub-chunk continues the carry
                cy[0] += (double)tj.x;
                cy[1] += (double)tj.y;
                cy[2] += (double)tj.z;
                cy[3] += (double)tj.w;
                cvalid = true;
                continue;
            }
            if (!starts) {  // head rows close the carried leaf
                const float4 hj = hsm[src];
                cy[0] += (double)hj.x;
                cy[1] += (double)hj.y;
                cy[2] += (double)hj.z;
                cy[3] += (double)hj.w;
                cvalid = true;
            }
            if (cvalid && (fj != 0)) skp_emit(A, cy[0], cy[1], cy[2], cy[3], cleaf, ckind, it, pos0, g0, Sb, lane, slot == 0);
            // the last segment of sub-chunk j becomes the carry
            cy[0] = (double)tj.x;
            cy[1] = (double)tj.y;
            cy[2] = (double)tj.z;
            cy[3] = (double)tj.w;
            cleaf = curj;
            if (fj != 0) ckind = 0;
            cvalid = true;
        }
#pragma unroll
        for (int j = 0; j < SKP_RMAX; j++) {
            if (j >= R || s0 + j >= nsub) break;
            flags_before += __popc((s0 == 0 && j == 0) ? (fl[j] & ~1u) : fl[j]);
        }
        __syncwarp();
    }
    const int kind = tail_open ? (ckind ? 3 : 2) : ckind;
    skp_emit(A, cy[0], cy[1], cy[2], cy[3], cleaf, kind, it, pos0, g0, Sb, lane, slot == 0);
}

// Phase B item: samples [i0, i0 + A.spw) against batch e's leaf sums.
// Slot s takes every R-th sample; its lanes gather the nT leaf-sum rows of
// that sample (coalesced, SKP_UB in flight), sum them in f32 and add the sum
// to Y in f64 (scaled by 1/B in the last batch).
template <int K4>
__device__ void skp_phase_b(const SkpArgs& A, int e, int64_t it, uint32_t* rbuf, int lane)
{
    const int b0 = e * A.T, b1 = min(A.Bl, b0 + A.T);
    const int nT = b1 - b0;
    const int64_t g0 = A.leaf_base[b0];
    const float4* Sb = reinterpret_cast<const float4*>(A.S + (int64_t)(e % A.nbuf) * A.s_rows * A.ld);
    const int k4 = K4 ? K4 : (A.ld >> 2);  // compile-time for the common widths
    const int R = min(SKP_RMAX, 32 / k4);
    const int slot = lane / k4, c4 = lane - slot * k4;
    const bool on = slot < R;
    const bool first = e == 0, last = e == A.nbatch - 1;
    const int64_t i0 = it * A.spw, i1 = min64(i0 + A.spw, A.n);
    const int32_t lb = lane < nT ? (int32_t)(A.leaf_base[b0 + lane] - g0) : 0;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    const int* rb = reinterpret_cast<const int*>(rbuf) + (on ? slot : 0) * SKP_SLOT;

    int32_t cn[SKP_RMAX];
    auto load_codes = [&](int64_t ib) {
#pragma unroll
        for (int j = 0; j < SKP_RMAX; j++) {
            const int64_t i = ib + j;
            cn[j] = (j < R && i < i1 && lane < nT) ? __ldcs(A.codes + i * A.Bl + b0 + lane) : 0;
        }
    };
    load_codes(i0);
    for (int64_t ib = i0; ib < i1; ib += R) {
#pragma unroll
        for (int j = 0; j < SKP_RMAX; j++) reinterpret_cast<int*>(rbuf)[j * SKP_SLOT + lane] = lb + cn[j];
        __syncwarp();
        if (ib + R < i1) load_codes(ib + R);
        const int64_t i = ib + slot;
        const bool act = on && i < i1;
        double yo[4] = {0.0, 0.0, 0.0, 0.0};
        double* y = A.Y + i * A.k + 4 * c4;
        // k = 4 * k4: the lane's 4 doubles are 32-byte aligned -> two 16-byte accesses
        const bool vec = K4 != 0 && A.k == 4 * k4;
        if (act && !first && !A.P) {
            if (vec) {
                const double2 lo = __ldcs(reinterpret_cast<const double2*>(y));
                const double2 hi = __ldcs(reinterpret_cast<const double2*>(y) + 1);
                yo[0] = lo.x; yo[1] = lo.y; yo[2] = hi.x; yo[3] = hi.y;
            } else {
#pragma unroll
                for (int q = 0; q < 4; q++)
                    if (4 * c4 + q < A.k) yo[q] = __ldcs(y + q);  // Y streams through L2
            }
        }
        float4 acc = z4;
        for (int t0 = 0; t0 < nT; t0 += SKP_UB) {
            float4 x[SKP_UB];
#pragma unroll
            for (int u = 0; u < SKP_UB; u++) {
                const int t = t0 + u;
                x[u] = (act && t < nT) ? __ldg(Sb + ((uint32_t)rb[t] * k4 + c4)) : z4;
            }
#pragma unroll
            for (int u = 0; u < SKP_UB; u++) f4add(acc, x[u]);
        }
        if (act && A.P && last && SKP_FUSE_FINAL) {
            // the last batch finishes the sample: the earlier batches'
            // partials and its own sum added in batch order in f64, times
            // 1/B — skp_final_kernel's additions in its order (same bits)
            const float4* P4 = reinterpret_cast<const float4*>(A.P);
            double v[4] = {0.0, 0.0, 0.0, 0.0};
            int e2 = 0;
            for (; e2 + 4 <= e; e2 += 4) {
                float4 x[4];
#pragma unroll
                for (int u = 0; u < 4; u++) x[u] = __ldcs(P4 + ((int64_t)(e2 + u) * A.n + i) * k4 + c4);
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    v[0] += (double)x[u].x;
                    v[1] += (double)x[u].y;
                    v[2] += (double)x[u].z;
                    v[3] += (double)x[u].w;
                }
            }
            for (; e2 < e; e2++) {
                const float4 x = __ldcs(P4 + ((int64_t)e2 * A.n + i) * k4 + c4);
                v[0] += (double)x.x;
                v[1] += (double)x.y;
                v[2] += (double)x.z;
                v[3] += (double)x.w;
            }
            v[0] += (double)acc.x;
            v[1] += (double)acc.y;
            v[2] += (double)acc.z;
            v[3] += (double)acc.w;
#pragma unroll
            for (int q = 0; q < 4; q++)
                if (4 * c4 + q < A.k) y[q] = v[q] * A.scale;
        } else if (act && A.P) {
            // the batch's f32 sum leaves once (16 B per lane); the f64 sum over
            // the batches (in batch order) is the last batch's (above), or
            // skp_final_kernel's when SKP_FUSE_FINAL is off
            __stcs(reinterpret_cast<float4*>(A.P + ((int64_t)e * A.n + i) * A.ld) + c4, acc);
        } else if (act) {
            const float a4[4] = {acc.x, acc.y, acc.z, acc.w};
            double v[4];
#pragma unroll
            for (int q = 0; q < 4; q++) {
                v[q] = yo[q] + (double)a4[q];
                if (last) v[q] *= A.scale;
            }
            if (vec) {
                __stcs(reinterpret_cast<double2*>(y), make_double2(v[0], v[1]));
                __stcs(reinterpret_cast<double2*>(y) + 1, make_double2(v[2], v[3]));
            } else {
#pragma unroll
                for (int q = 0; q < 4; q++)
                    if (4 * c4 + q < A.k) __stcs(y + q, v[q]);
            }
        }
        __syncwarp();
    }
}

// One phase of one tree batch per launch (A: leaf sums of batch e; B: gather
// of batch e into Y), one item per warp; launched back to back on one stream
// (A(0) B(0) A(1) B(1) ...), so one leaf-sum buffer suffices and each phase
// gets its own register budget (full occupancy for the gathers).
template <int PH, int K4>
__global__ void __launch_bounds__(256, PH == 0 ? SKP_MINB_A : SKP_MINB_B) sketch_phase_kernel(SkpArgs A, int e)
{
    extern __shared__ __align__(16) uint32_t skp_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* scratch = skp_smem + warp * SKP_SCRATCH;
    const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (PH == 0) {
        const int b0 = e * A.T, b1 = min(A.Bl, b0 + A.T);
        const int64_t nA = ((int64_t)(b1 - b0) * A.n + A.item - 1) / A.item;
        if (q < nA) skp_phase_a<K4>(A, e, q, scratch, lane);
    } else {
        const int64_t nB = (A.n + A.spw - 1) / A.spw;
        if (q < nB) skp_phase_b<K4>(A, e, q, scratch, lane);
    }
}

// Y[i, c] = scale * sum_e P[e, i, c] in batch order, f64 — the same
// additions, in the same order, as phase B's f64 read-modify-write of Y.
// Thread per (row, 4-column group): the nbatch float4 loads are independent.
__global__ void skp_final_kernel(const float* __restrict__ P, int nbatch, int64_t n, int ld, int k,
                                 double scale, double* __restrict__ Y)
{
    const int k4 = ld >> 2;
    const int64_t total = n * k4;
    const float4* P4 = reinterpret_cast<const float4*>(P);
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = q / k4;
        const int c4 = (int)(q - i * k4);
        double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
        int e = 0;
        for (; e + 4 <= nbatch; e += 4) {
            float4 x[4];
#pragma unroll
            for (int u = 0; u < 4; u++) x[u] = __ldcs(P4 + ((int64_t)(e + u) * n + i) * k4 + c4);
#pragma unroll
            for (int u = 0; u < 4; u++) {
                v0 += (double)x[u].x;
                v1 += (double)x[u].y;
                v2 += (double)x[u].z;
                v3 += (double)x[u].w;
            }
        }
        for (; e < nbatch; e++) {
            const float4 x = __ldcs(P4 + ((int64_t)e * n + i) * k4 + c4);
            v0 += (double)x.x;
            v1 += (double)x.y;
            v2 += (double)x.z;
            v3 += (double)x.w;
        }
        double* y = Y + i * k + 4 * c4;
        const double v[4] = {v0, v1, v2, v3};
#pragma unroll
        for (int u = 0; u < 4; u++)
            if (4 * c4 + u < k) y[u] = v[u] * scale;
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

extern "C" int rfxc_leaf_sums(const uint32_t* d_perm, const int64_t* d_seg, int64_t g_lo,
                              int64_t g_hi, const float* d_X, int32_t k, int32_t ld, float* d_S,
                              void* stream)
{
    if (g_lo < 0 || g_hi < g_lo || k < 1 || ld < k || (ld & 3))
        return fail(RFXC_EDATA, "leaf_sums: bad shape (ld must be a multiple of 4 >= k)");
    if (g_hi == g_lo) return RFXC_OK;
    const int64_t warps = g_hi - g_lo;
    int grid = (int)std::min<int64_t>(ceil_div(warps, 8), (int64_t)sm_count() * 32);
    leaf_sums_kernel<<<grid, 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const int32_t*>(d_perm), d_seg, g_lo, g_hi,
        reinterpret_cast<const float4*>(d_X), ld / 4,
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

template <int TAM, int TBM>
static int launch_gram(const double* d_A, const double* d_B, int64_t n, int ka_tot, int kb,
                       double* d_partials, double* d_C, cudaStream_t st)
{
    const int parts = gram_parts(n);
    const int64_t rpp = ceil_div(n, parts);
    for (int a0 = 0; a0 < ka_tot; a0 += 8 * TAM) {
        const int ka = std::min(8 * TAM, ka_tot - a0);
        const int TA = (ka + 7) / 8;
        for (int c0 = 0; c0 < kb; c0 += 8 * TBM) {
            const int w = std::min(8 * TBM, kb - c0);
            const size_t smem = (size_t)(GRAM_THREADS / 32) * TA * ((w + 7) / 8) * 64 * 8;
            auto kern = gram_partial_kernel<TAM, TBM>;
            if (smem > 48 * 1024)
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            kern<<<parts, GRAM_THREADS, smem, st>>>(d_A + a0, ka_tot, d_B + c0, kb, n, ka, w, rpp,
                                                    d_partials);
            int rc = check_launch("gram_partial");
            if (rc) return rc;
            gram_final_kernel<<<(unsigned)ceil_div((int64_t)ka * w * 32, 256), 256, 0, st>>>(
                d_partials, parts, ka, w, d_C, kb, c0, a0);
            rc = check_launch("gram_final");
            if (rc) return rc;
        }
    }
    return RFXC_OK;
}

extern "C" int rfxc_gram(const double* d_A, const double* d_B, int64_t n, int32_t ka, int32_t kb,
                         double* d_partials, double* d_C, void* stream)
{
    // d_partials must hold rfxc_gram_parts(n) * ka * kb doubles
    if (n < 1 || ka < 1 || kb < 1) return fail(RFXC_EDATA, "gram: bad shape ka=%d kb=%d", ka, kb);
    cudaStream_t st = as_stream(stream);
    const int TA = (ka + 7) / 8;
    if (ka <= 128 && kb <= 128) {
        const int TB = (kb + 7) / 8;
        const int NT = (d_A == d_B && ka == kb) ? TA * (TA + 1) / 2 : TA * TB;
        const int mt = (NT + GS_THREADS / 32 - 1) / (GS_THREADS / 32);
        if (mt <= 2) return launch_gram_stage<2>(d_A, d_B, n, ka, kb, d_partials, d_C, st);
        if (mt <= 4) return launch_gram_stage<4>(d_A, d_B, n, ka, kb, d_partials, d_C, st);
        if (mt <= 8) return launch_gram_stage<8>(d_A, d_B, n, ka, kb, d_partials, d_C, st);
        if (mt <= 16) return launch_gram_stage<16>(d_A, d_B, n, ka, kb, d_partials, d_C, st);
        return launch_gram_stage<32>(d_A, d_B, n, ka, kb, d_partials, d_C, st);
    }
    if (TA <= 2) return launch_gram<2, 16>(d_A, d_B, n, ka, kb, d_partials, d_C, st);
    if (TA <= 5) return launch_gram<5, 5>(d_A, d_B, n, ka, kb, d_partials, d_C, st);
    if (TA <= 8) return launch_gram<8, 4>(d_A, d_B, n, ka, kb, d_partials, d_C, st);
    return launch_gram<16, 2>(d_A, d_B, n, ka, kb, d_partials, d_C, st);
}

// wide outputs (kb > 128): plain FMA kernel, 16 rows of Y per CTA
__global__ void __launch_bounds__(256)
matmul_wide_kernel(const double* __restrict__ Y, int64_t n, int ka, const double* __restrict__ M,
                   int kb, double* __restrict__ Z, float* __restrict__ Z32, int ld32)
{
    extern __shared__ double ysm[];
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
        double acc = 0.0;
        if (c < kb)
            for (int a = 0; a < ka; a++) acc += ysm[r * ka + a] * __ldg(M + (int64_t)a * kb + c);
        if (c < kb) Z[(r0 + r) * kb + c] = acc;
        if (Z32 && c < ld32) Z32[(r0 + r) * ld32 + c] = c < kb ? (float)acc : 0.0f;
    }
}

template <int TBM>
static int launch_mm(const double* d_Y, int64_t n, int ka, const double* d_M, int kb, double* d_Z,
                     float* d_Z32, int ld32, cudaStream_t st)
{
    const int KS = (ka + 3) / 4;
    const size_t smem = (size_t)KS * 4 * TBM * 8 * 8;
    auto kern = matmul_small_kernel<TBM>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return fail(RFXC_ECUDA, "matmul attr: %s", cudaGetErrorString(e));
    }
    const int64_t warps = ceil_div(n, 8);
    const int grid = (int)std::min<int64_t>(ceil_div(warps, 8), (int64_t)sm_count() * 2);
    kern<<<grid, 256, smem, st>>>(d_Y, n, ka, d_M, kb, d_Z, d_Z32, ld32);
    return check_launch("matmul_small");
}

extern "C" int rfxc_matmul_small(const double* d_Y, int64_t n, int32_t ka, const double* d_M,
                                 int32_t kb, double* d_Z, float* d_Z32, int32_t ld32, void* stream)
{
    const int w = std::max<int>(kb, d_Z32 ? ld32 : 0);
    if (n < 1 || ka < 1 || kb < 1 || ka > 4096)
        return fail(RFXC_EDATA, "matmul_small: bad shape ka=%d kb=%d", ka, kb);
    cudaStream_t st = as_stream(stream);
    if (w > 8 * MM_MAXTB || ka > 512) {
        const size_t smem = (size_t)16 * ka * 8;
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(matmul_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
        matmul_wide_kernel<<<(unsigned)ceil_div(n, 16), 256, smem, st>>>(d_Y, n, ka, d_M, kb, d_Z,
                                                                         d_Z32, ld32);
        return check_launch("matmul_wide");
    }
    switch ((w + 7) / 8) {
        case 1: return launch_mm<1>(d_Y, n, ka, d_M, kb, d_Z, d_Z32, ld32, st);
        case 2: return launch_mm<2>(d_Y, n, ka, d_M, kb, d_Z, d_Z32, ld32, st);
        case 3: return launch_mm<3>(d_Y, n, ka, d_M, kb, d_Z, d_Z32, ld32, st);
        case 4: return launch_mm<4>(d_Y, n, ka, d_M, kb, d_Z, d_Z32, ld32, st);
        case 5: return launch_mm<5>(d_Y, n, ka, d_M, kb, d_Z, d_Z32, ld32, st);
        case 6: return launch_mm<6>(d_Y, n, ka, d_M, kb, d_Z, d_Z32, ld32, st);
        case 7: return launch_mm<7>(d_Y, n, ka, d_M, kb, d_Z, d_Z32, ld32, st);
        case 8: return launch_mm<8>(d_Y, n, ka, d_M, kb, d_Z, d_Z32, ld32, st);
        case 9: case 10: return launch_mm<10>(d_Y, n, ka, d_M, kb, d_Z, d_Z32, ld32, st);
        case 11: case 12: return launch_mm<12>(d_Y, n, ka, d_M, kb, d_Z, d_Z32, ld32, st);
        default: return launch_mm<16>(d_Y, n, ka, d_M, kb, d_Z, d_Z32, ld32, st);
    }
}

// Phase-A item (positions per warp): one item per resident phase-A warp of
// a batch, a multiple of 32, at least one 3-slot step
static int64_t skp_item_size(int64_t n, int T)
{
    const int64_t warps = (int64_t)sm_count() * SKP_MINB_A * 8;
    const int64_t item = (T * n + warps - 1) / warps;
    return std::max<int64_t>(96, (item + 31) / 32 * 32);
}

extern "C" int rfxc_sketch_plan(const int32_t* h_leaf_counts, int32_t Bl, int64_t n, int32_t k,
                                int64_t budget_bytes, int32_t* T_out, int64_t* s_rows_out,
                                int32_t* nbuf_out, int64_t* work_bytes_out)
{
    if (Bl < 1 || n < 1 || k < 1) return fail(RFXC_EDATA, "sketch_plan: bad shape");
    const int ld = (k + 3) / 4 * 4;
    // largest batch of trees whose leaf sums (nbuf buffers) fit the budget
    auto plan = [&](int nbuf, int64_t& rows_out) {
        int T = std::min(SKP_MAX_T, (int)Bl);
        for (; T >= 1; T--) {
            int64_t rows = 0;
            for (int b0 = 0; b0 < Bl; b0 += T) {
                int64_t s = 0;
                for (int b = b0; b < std::min<int>(Bl, b0 + T); b++) s += h_leaf_counts[b];
                rows = std::max(rows, s);
            }
            rows_out = std::max<int64_t>(rows, 1);
            if (nbuf * rows * ld * 4 <= budget_bytes || T == 1) break;
        }
        return T;
    };
    int64_t r1 = 1, r2 = 1;
    const int T1 = plan(1, r1), T2 = plan(2, r2);
    // two buffers (phase A of batch e+1 overlaps phase B of batch e) only when
    // that costs no batch size
    const int nbuf = (T2 == T1) ? 2 : 1;
    const int T = nbuf == 2 ? T2 : T1;
    const int64_t s_rows = nbuf == 2 ? r2 : r1;
    if (T_out) *T_out = T;
    if (s_rows_out) *s_rows_out = s_rows;
    if (nbuf_out) *nbuf_out = nbuf;
    if (work_bytes_out) *work_bytes_out = skp_layout(n, Bl, T, ld, k, s_rows, nbuf, skp_item_size(n, T)).total;
    return RFXC_OK;
}

extern "C" int rfxc_sketch_prepare(const int64_t* d_seg, const int64_t* d_leaf_base, int64_t n,
                                   int32_t Bl, int32_t k, int32_t T, int64_t s_rows, int32_t nbuf,
                                   void* d_work, void* stream)
{
    if (n < 1 || Bl < 1 || k < 1 || T < 1 || T > SKP_MAX_T || s_rows < 1)
        return fail(RFXC_EDATA, "sketch_prepare: bad shape");
    const int ld = (k + 3) / 4 * 4;
    if (nbuf < 1 || nbuf > 2) return fail(RFXC_EDATA, "sketch_prepare: nbuf must be 1 or 2");
    const int64_t item = skp_item_size(n, T);
    const SkpLayout L = skp_layout(n, Bl, T, ld, k, s_rows, nbuf, item);
    char* w = static_cast<char*>(d_work);
    cudaStream_t st = as_stream(stream);
    cudaError_t e = cudaMemsetAsync(w + L.cnt, 0, s_rows * 4, st);
    if (e != cudaSuccess) return fail(RFXC_ECUDA, "sketch_prepare: %s", cudaGetErrorString(e));
    const int64_t ipb = skp_items_per_batch(n, T, item);
    const int64_t total = skp_nbatch(Bl, T) * ipb;
    const int grid = (int)std::min<int64_t>(ceil_div(total, 256), (int64_t)sm_count() * 8);
    skp_item_leaf_kernel<<<grid, 256, 0, st>>>(d_seg, d_leaf_base, n, Bl, T, ipb, item,
                                               reinterpret_cast<int32_t*>(w + L.item_leaf));
    return check_launch("sketch_prepare");
}

template <int PH>
static void launch_phase(const SkpArgs& A, int e, cudaStream_t s)
{
    const size_t smem = (size_t)8 * SKP_SCRATCH * 4;
    int64_t items;
    if (PH == 0) {
        const int b0 = e * A.T, b1 = std::min(A.Bl, b0 + A.T);
        items = ((int64_t)(b1 - b0) * A.n + A.item - 1) / A.item;
    } else {
        items = (A.n + A.spw - 1) / A.spw;
    }
    if (A.ld == 40)  // k = r + 8 for the default rank 32
        sketch_phase_kernel<PH, 10><<<(unsigned)ceil_div(items, 8), 256, smem, s>>>(A, e);
    else
        sketch_phase_kernel<PH, 0><<<(unsigned)ceil_div(items, 8), 256, smem, s>>>(A, e);
}

// Phase A of batch e + 1 overlaps phase B of batch e: A runs on an auxiliary
// stream forked from `st` (two leaf-sum buffers; A(e) waits for B(e - 2)
// before overwriting its buffer), B stays on `st` in batch order (the Y
// accumulation order is fixed) and the last B joins everything back.
static void launch_final(const SkpArgs& A, cudaStream_t st)
{
    if (!A.P || SKP_FUSE_FINAL) return;  // fused: the last phase B wrote Y
    const int grid = (int)std::min<int64_t>(ceil_div(A.n * (A.ld / 4), 256), (int64_t)sm_count() * 16);
    skp_final_kernel<<<grid, 256, 0, st>>>(A.P, A.nbatch, A.n, A.ld, A.k, A.scale, A.Y);
}

static int launch_skp(SkpArgs& A, cudaStream_t st)
{
    if (A.nbuf < 2) {
        for (int e = 0; e < A.nbatch; e++) {
            launch_phase<0>(A, e, st);
            launch_phase<1>(A, e, st);
        }
        launch_final(A, st);
        return check_launch("sketch_pass");
    }
    static cudaStream_t aux[64] = {};
    static std::vector<cudaEvent_t> evs[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (!aux[dev]) cudaStreamCreateWithFlags(&aux[dev], cudaStreamNonBlocking);
    std::vector<cudaEvent_t>& ev = evs[dev];
    while ((int)ev.size() < 2 * A.nbatch + 1) {
        cudaEvent_t x;
        cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
        ev.push_back(x);
    }
    cudaStream_t sa = aux[dev];
    cudaEventRecord(ev[0], st);  // fork: X and the buffers are ready on st
    cudaStreamWaitEvent(sa, ev[0], 0);
    for (int e = 0; e < A.nbatch; e++) {
        if (e >= 2) cudaStreamWaitEvent(sa, ev[2 + 2 * (e - 2)], 0);  // B(e-2) released the buffer
        launch_phase<0>(A, e, sa);
        cudaEventRecord(ev[1 + 2 * e], sa);
        cudaStreamWaitEvent(st, ev[1 + 2 * e], 0);
        launch_phase<1>(A, e, st);
        cudaEventRecord(ev[2 + 2 * e], st);
    }
    launch_final(A, st);
    return check_launch("sketch_pass");
}

extern "C" int rfxc_sketch_pass(const uint32_t* d_perm, const int64_t* d_seg,
                                const int32_t* d_codes_nb, const int64_t* d_leaf_base,
                                const int32_t* d_has_empty, int64_t n, int32_t Bl,
                                const float* d_X, int32_t k, int32_t ld, double scale, int32_t T,
                                int64_t s_rows, int32_t nbuf, double* d_Y, void* d_work,
                                void* stream)
{
    if (n < 1 || Bl < 1 || k < 1 || ld != (k + 3) / 4 * 4 || T < 1 || T > SKP_MAX_T || s_rows < 1)
        return fail(RFXC_EDATA, "sketch_pass: bad shape (ld must be k rounded up to 4)");
    if (ld > 128) return fail(RFXC_EDATA, "sketch_pass: k=%d above 128", k);
    if (nbuf < 1 || nbuf > 2) return fail(RFXC_EDATA, "sketch_pass: nbuf must be 1 or 2");
    const int64_t item = skp_item_size(n, T);
    const SkpLayout L = skp_layout(n, Bl, T, ld, k, s_rows, nbuf, item);
    char* w = static_cast<char*>(d_work);
    cudaStream_t st = as_stream(stream);
    SkpArgs A;
    A.perm = d_perm;
    A.seg = d_seg;
    A.codes = d_codes_nb;
    A.leaf_base = d_leaf_base;
    A.has_empty = d_has_empty;
    A.X = d_X;
    A.Y = d_Y;
    // per-batch f32 partials + one ordered f64 sum (no per-batch f64 Y
    // read-modify-write); RFXC_SKETCH_YPART=0 restores the RMW
    {
        const char* yp = getenv("RFXC_SKETCH_YPART");
        A.P = (yp && yp[0] == '0') ? nullptr : reinterpret_cast<float*>(w + L.ypart);
    }
    A.S = reinterpret_cast<float*>(w + L.S);
    A.part = reinterpret_cast<double*>(w + L.part);
    A.cnt = reinterpret_cast<int32_t*>(w + L.cnt);
    A.ctr = reinterpret_cast<unsigned*>(w + L.ctr);
    A.item_leaf = reinterpret_cast<const int32_t*>(w + L.item_leaf);
    A.n = n;
    A.s_rows = s_rows;
    A.item = item;
    {   // phase B: all items in one wave of resident warps (4 CTAs x 8 warps per SM)
        const int64_t warps = (int64_t)sm_count() * SKP_MINB_B * 8;
        A.spw = (int)std::min<int64_t>(SKP_SAMPLES, std::max<int64_t>(1, (n + warps - 1) / warps));
    }
    A.ipb = skp_items_per_batch(n, T, item);
    A.Bl = Bl;
    A.k = k;
    A.ld = ld;
    A.T = T;
    A.nbatch = skp_nbatch(Bl, T);
    A.nbuf = nbuf;
    A.scale = scale;
    cudaError_t e = cudaMemsetAsync(A.ctr, 0, 2 * (size_t)(A.nbatch + 1) * 4, st);
    if (e != cudaSuccess) return fail(RFXC_ECUDA, "sketch_pass: %s", cudaGetErrorString(e));
    A.timing = nullptr;
    if (!getenv("RFXC_SKETCH_TIMING")) return launch_skp(A, st);
    // debug: time the pass (synchronous)
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    int rc = launch_skp(A, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    fprintf(stderr, "[sketch] pass %.3f ms, T=%d batches=%d\n", ms, A.T, A.nbatch);
    return rc;
}
