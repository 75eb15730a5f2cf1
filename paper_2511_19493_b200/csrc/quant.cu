// quant.cu — K6/K7: factor = Q Wr, QLORA quantisation, dequantisation, pmax.
//
// Reference: proximity.py:401-417 (factor_raw = Q @ (W_r * sqrt(lambda)),
// quantize, dequantize, pmax over the diagonal and 1024 sampled pairs) and
// quantize.py:83-140 (f32 / f16 casts, i8 per-column absmax/127 with
// round-half-even and clip to +-127, nf4 64-blocks of the column-major
// flatten against the 16-level codebook, low nibble first).
//
// Every division is a true IEEE f64 division and rint() is round-half-even,
// so for the same factor the device codes equal numpy's bit for bit.
#include <cuda_fp16.h>

#include "../csrc/host/pcg32.h"
#include "common.cuh"

namespace rfxc {

__constant__ double NF4_CB[16] = {
    -1.0, -0.6961928009986877, -0.5250730514526367, -0.39491748809814453,
    -0.28444138169288635, -0.18477343022823334, -0.09105003625154495, 0.0,
    0.07958029955625534, 0.16093020141124725, 0.24611230194568634, 0.33791524171829224,
    0.44070982933044434, 0.5626170039176941, 0.7229568362236023, 1.0};

int gram_parts(int64_t n);
}  // namespace rfxc
extern "C" int rfxc_matmul_small(const double* d_Y, int64_t n, int32_t ka, const double* d_M,
                                 int32_t kb, double* d_Z, float* d_Z32, int32_t ld32, void* stream);
namespace rfxc {

// F = Q @ Wr row by row; per-part column absmax.  Wr staged in shared memory
// (SW) or read through L1 when k x r is too large.
template <bool SW>
__global__ void __launch_bounds__(256)
factor_kernel(const double* __restrict__ Q, int64_t n, int k, const double* __restrict__ Wr, int r,
              int64_t rows_per_part, double* __restrict__ F, double* __restrict__ colmax_parts)
{
    extern __shared__ double wsm[];  // [k x r if SW] [blockDim partial maxima]
    double* cm = wsm + (SW ? k * r : 0);
    if (SW)
        for (int e = threadIdx.x; e < k * r; e += blockDim.x) wsm[e] = Wr[e];
    const double* W = SW ? wsm : Wr;
    __syncthreads();
    const int64_t r0 = blockIdx.x * rows_per_part, r1 = min(n, r0 + rows_per_part);
    // thread -> (row offset, column): columns fastest
    const int c = threadIdx.x % r;
    const int rstep = blockDim.x / r;
    const int roff = threadIdx.x / r;
    double m = 0.0;
    if (roff < rstep) {
        for (int64_t i = r0 + roff; i < r1; i += rstep) {
            double s = 0.0;
            for (int a = 0; a < k; a++) s += Q[i * k + a] * (SW ? W[a * r + c] : __ldg(W + a * r + c));
            F[i * r + c] = s;
            m = fmax(m, fabs(s));
        }
    }
    cm[threadIdx.x] = (roff < rstep) ? m : 0.0;
    __syncthreads();
    if (threadIdx.x < r) {
        double mm = 0.0;
        for (int q = 0; q < rstep; q++) mm = fmax(mm, cm[q * r + threadIdx.x]);
        colmax_parts[(int64_t)blockIdx.x * r + threadIdx.x] = mm;
    }
}

// per-part column absmax of F (n, r): thread (row offset, column), columns fastest
__global__ void __launch_bounds__(256)
colmax_kernel(const double* __restrict__ F, int64_t n, int r, int64_t rows_per_part,
              double* __restrict__ colmax_parts)
{
    __shared__ double cm[256];
    const int64_t r0 = blockIdx.x * rows_per_part, r1 = min(n, r0 + rows_per_part);
    const int c = threadIdx.x % r, rstep = blockDim.x / r, roff = threadIdx.x / r;
    double m = 0.0;
    if (roff < rstep)
        for (int64_t i = r0 + roff; i < r1; i += rstep) m = fmax(m, fabs(__ldg(F + i * r + c)));
    cm[threadIdx.x] = (roff < rstep) ? m : 0.0;
    __syncthreads();
    if (threadIdx.x < r) {
        double mm = 0.0;
        for (int q = 0; q < rstep; q++) mm = fmax(mm, cm[q * r + threadIdx.x]);
        colmax_parts[(int64_t)blockIdx.x * r + threadIdx.x] = mm;
    }
}

// a warp per column (max is order-free: the same value as a sequential scan)
__global__ void colmax_final_kernel(const double* __restrict__ parts, int nparts, int r,
                                     double* __restrict__ scales)
{
    const int c = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (c >= r) return;
    double m = 0.0;
    for (int q = lane; q < nparts; q += 32) m = fmax(m, __ldg(parts + (int64_t)q * r + c));
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) scales[c] = m / 127.0;  // quantize.py:95-96
}

__global__ void quant_i8_kernel(const double* __restrict__ F, int64_t total, int r,
                                const double* __restrict__ scales, int8_t* __restrict__ out)
{
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const double s = scales[total < (int64_t(1) << 32) ? (int)((uint32_t)e % (uint32_t)r) : (int)(e % r)];
        const double safe = s > 0.0 ? s : 1.0;
        double q = rint(F[e] / safe);
        q = fmin(127.0, fmax(-127.0, q));
        out[e] = (int8_t)q;
    }
}

__global__ void quant_cast_kernel(const double* __restrict__ F, int64_t total, int mode,
                                  void* __restrict__ out)
{
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        if (mode == RFXC_Q_F32) reinterpret_cast<float*>(out)[e] = (float)F[e];
        else reinterpret_cast<__half*>(out)[e] = __double2half(F[e]);
    }
}

// nf4: flat index f = c*n + i (column-major), block = f / 64.
__global__ void quant_nf4_kernel(const double* __restrict__ F, int64_t n, int r, int64_t nblocks,
                                 double* __restrict__ absmax, uint8_t* __restrict__ out)
{
    const int64_t blk = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (blk >= nblocks) return;
    const int64_t total = n * r;
    double m = 0.0;
    for (int q = 0; q < 64; q++) {
        const int64_t f = blk * 64 + q;
        if (f < total) m = fmax(m, fabs(F[(f % n) * r + f / n]));
    }
    absmax[blk] = m;
    const double safe = m > 0.0 ? m : 1.0;
    for (int q = 0; q < 64; q += 2) {
        uint8_t code[2];
        for (int h = 0; h < 2; h++) {
            const int64_t f = blk * 64 + q + h;
            const double x = f < total ? F[(f % n) * r + f / n] / safe : 0.0;
            int best = 0;
            double bd = fabs(x - NF4_CB[0]);
            for (int t = 1; t < 16; t++) {
                const double d = fabs(x - NF4_CB[t]);
                if (d < bd) { bd = d; best = t; }
            }
            code[h] = (uint8_t)best;
        }
        out[blk * 32 + q / 2] = (uint8_t)(code[0] | (code[1] << 4));
    }
}

__global__ void dequant_kernel(const void* __restrict__ data, const double* __restrict__ scales,
                               int64_t n, int r, int mode, double* __restrict__ dq)
{
    const int64_t total = n * r;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        double v;
        if (mode == RFXC_Q_I8) {
            v = (double)reinterpret_cast<const int8_t*>(data)[e] *
                scales[total < (int64_t(1) << 32) ? (int)((uint32_t)e % (uint32_t)r) : (int)(e % r)];
        } else if (mode == RFXC_Q_F32) {
            v = (double)reinterpret_cast<const float*>(data)[e];
        } else if (mode == RFXC_Q_F16) {
            v = (double)__half2float(reinterpret_cast<const __half*>(data)[e]);
        } else {
            const int64_t i = e / r, c = e % r;
            const int64_t f = c * n + i;
            const uint8_t byte = reinterpret_cast<const uint8_t*>(data)[f >> 1];
            const int code = (f & 1) ? (byte >> 4) : (byte & 0x0F);
            v = NF4_CB[code] * scales[f / 64];
        }
        dq[e] = v;
    }
}

// The 2048 bounded draws Pcg32(seed, SEQ_PMAX).bounded(n) of the pmax pairs
// (proximity.py:409-417) into pairs[], by the whole (256-thread) block.
__device__ void pmax_draws(uint64_t s0, uint64_t s1, uint32_t n, uint32_t* pairs)
{
    // the 2048 bounded draws of the sequential stream, generated in
    // parallel: thread t jumps ahead to raw draw PM_PER * t, keeps the
    // draws >= threshold (rfx_pcg32_bounded's acceptance test) and a block
    // scan of the accept counts gives every kept draw its place in the
    // bounded sequence; if the margin ever ran out, thread 0 redoes it
    // sequentially (exactly the same sequence either way)
    constexpr int PM_PER = 9;  // 256 * 9 = 2304 raw draws >= 2048 + margin
    const uint32_t b = n;
    const uint32_t thr = (uint32_t)((0x100000000ULL - b) % b);
    uint64_t st[2] = {s0, s1};
    rfx_pcg32_advance(st, (uint64_t)PM_PER * threadIdx.x);
    uint32_t raw[PM_PER];
    int cnt = 0;
#pragma unroll
    for (int u = 0; u < PM_PER; u++) {
        raw[u] = rfx_pcg32_next(st);
        cnt += raw[u] >= thr;
    }
    __shared__ int scan[256];
    scan[threadIdx.x] = cnt;
    __syncthreads();
    for (int o = 1; o < 256; o <<= 1) {  // inclusive Hillis-Steele scan
        const int v = threadIdx.x >= o ? scan[threadIdx.x - o] : 0;
        __syncthreads();
        scan[threadIdx.x] += v;
        __syncthreads();
    }
    int pos = scan[threadIdx.x] - cnt;
#pragma unroll
    for (int u = 0; u < PM_PER; u++)
        if (raw[u] >= thr) {
            if (pos < 2048) pairs[pos] = raw[u] % b;
            pos++;
        }
    const bool short_ = scan[255] < 2048;
    __syncthreads();
    if (short_ && threadIdx.x == 0) {
        uint64_t s[2] = {s0, s1};
        for (int t = 0; t < 2048; t++) pairs[t] = rfx_pcg32_bounded(s, b);
    }
    __syncthreads();
}

// pmax: block q < nparts -> max of diag over its rows; last block -> the
// 1024 sampled pairs (Pcg32(seed, SEQ_PMAX), i == j skipped, no redraw).
__global__ void __launch_bounds__(256)
pmax_kernel(const double* __restrict__ dq, int64_t n, int r, int64_t rows_per_part, int nparts,
            uint64_t s0, uint64_t s1, double* __restrict__ parts)
{
    __shared__ double red[32];
    __shared__ uint32_t pairs[2048];
    double m = -INFINITY;
    if ((int)blockIdx.x < nparts) {
        const int64_t r0 = blockIdx.x * rows_per_part, r1 = min(n, r0 + rows_per_part);
        for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
            double s = 0.0;
            if (r == 32) {  // all the row's loads in flight first, then the sum in column order
                double x[32];
#pragma unroll
                for (int c = 0; c < 32; c++) x[c] = __ldg(dq + i * 32 + c);
#pragma unroll
                for (int c = 0; c < 32; c++) s += x[c] * x[c];
            } else {
                for (int c = 0; c < r; c++) s += dq[i * r + c] * dq[i * r + c];
            }
            m = fmax(m, s);
        }
    } else {
        pmax_draws(s0, s1, (uint32_t)n, pairs);
        for (int t = threadIdx.x; t < 1024; t += blockDim.x) {
            const int64_t i = pairs[2 * t], j = pairs[2 * t + 1];
            if (i == j) continue;
            double s = 0.0;
            if (r == 32) {  // both rows' loads in flight first, then the sum in column order
                double a[32], b[32];
#pragma unroll
                for (int c = 0; c < 32; c++) {
                    a[c] = __ldg(dq + i * 32 + c);
                    b[c] = __ldg(dq + j * 32 + c);
                }
#pragma unroll
                for (int c = 0; c < 32; c++) s += a[c] * b[c];
            } else {
                for (int c = 0; c < r; c++) s += dq[i * r + c] * dq[j * r + c];
            }
            m = fmax(m, s);
        }
    }
    m = block_max(m, red);
    if (threadIdx.x == 0) parts[blockIdx.x] = m;
}

__global__ void __launch_bounds__(256) pmax_draws_kernel(uint64_t s0, uint64_t s1, uint32_t n,
                                                         uint32_t* __restrict__ out)
{
    __shared__ uint32_t pairs[2048];
    pmax_draws(s0, s1, n, pairs);
    __syncthreads();
    for (int t = threadIdx.x; t < 2048; t += blockDim.x) out[t] = pairs[t];
}

__global__ void max_final_kernel(const double* __restrict__ parts, int np, double* out)
{
    double m = -INFINITY;  // one warp; max is order-free
    for (int q = threadIdx.x; q < np; q += 32) m = fmax(m, __ldg(parts + q));
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) *out = m;
}

}  // namespace rfxc

using namespace rfxc;

extern "C" int rfxc_factor_quantize(const double* d_Q, int64_t n, int32_t k, const double* d_Wr,
                                    int32_t r, int32_t mode, double* d_factor,
                                    double* d_colmax_parts, double* d_scales, void* d_data,
                                    void* stream)
{
    if (n < 1 || k < 1 || r < 1 || r > 256) return fail(RFXC_EDATA, "factor_quantize: bad shape");
    cudaStream_t st = as_stream(stream);
    const int parts = gram_parts(n);
    const int64_t rpp = ceil_div(n, parts);
    const int threads = 256;
    if (k <= 128 && r <= 128) {
        // F = Q Wr on the FP64 tensor cores (the sketch's small matmul), then
        // the per-part column absmax
        int rc = rfxc_matmul_small(d_Q, n, k, d_Wr, r, d_factor, nullptr, 0, stream);
        if (rc) return rc;
        colmax_kernel<<<parts, threads, 0, st>>>(d_factor, n, r, rpp, d_colmax_parts);
        rc = check_launch("colmax");
        if (rc) return rc;
    } else {
        const bool sw = (size_t)k * r * 8 <= 160 * 1024;
        const size_t smem = ((sw ? (size_t)k * r : 0) + threads) * 8;
        if (sw) {
            if (smem > 48 * 1024)
                cudaFuncSetAttribute(factor_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem);
            factor_kernel<true><<<parts, threads, smem, st>>>(d_Q, n, k, d_Wr, r, rpp, d_factor,
                                                              d_colmax_parts);
        } else {
            factor_kernel<false><<<parts, threads, smem, st>>>(d_Q, n, k, d_Wr, r, rpp, d_factor,
                                                               d_colmax_parts);
        }
        int rc = check_launch("factor");
        if (rc) return rc;
    }
    const int64_t total = n * r;
    const int grid = (int)std::min<int64_t>(ceil_div(total, 256), (int64_t)sm_count() * 16);
    switch (mode) {
    case RFXC_Q_I8:
        colmax_final_kernel<<<(unsigned)ceil_div((int64_t)r * 32, 128), 128, 0, st>>>(d_colmax_parts, parts,
                                                                                   r, d_scales);
        quant_i8_kernel<<<grid, 256, 0, st>>>(d_factor, total, r, d_scales,
                                              reinterpret_cast<int8_t*>(d_data));
        break;
    case RFXC_Q_F32:
    case RFXC_Q_F16:
        quant_cast_kernel<<<grid, 256, 0, st>>>(d_factor, total, mode, d_data);
        break;
    case RFXC_Q_NF4: {
        const int64_t nb = ceil_div(total, 64);
        quant_nf4_kernel<<<(unsigned)ceil_div(nb, 128), 128, 0, st>>>(
            d_factor, n, r, nb, d_scales, reinterpret_cast<uint8_t*>(d_data));
        break;
    }
    default:
        return fail(RFXC_EDATA, "factor_quantize: unknown mode %d", mode);
    }
    return check_launch("quantize");
}

extern "C" int rfxc_dequantize(const void* d_data, const double* d_scales, int64_t n, int32_t r,
                               int32_t mode, double* d_dq, void* stream)
{
    if (n < 1 || r < 1 || mode < 0 || mode > RFXC_Q_NF4) return fail(RFXC_EDATA, "dequantize");
    const int grid = (int)std::min<int64_t>(ceil_div(n * r, 256), (int64_t)sm_count() * 16);
    dequant_kernel<<<grid, 256, 0, as_stream(stream)>>>(d_data, d_scales, n, r, mode, d_dq);
    return check_launch("dequantize");
}

extern "C" int rfxc_pmax_draws(int64_t seed, int64_t n, uint32_t* d_out, void* stream)
{
    if (n < 1 || n > UINT32_MAX) return fail(RFXC_EDATA, "pmax_draws: bad n");
    uint64_t s[2];
    rfx_pcg32_make(seed, RFX_SEQ_PMAX, s);
    pmax_draws_kernel<<<1, 256, 0, as_stream(stream)>>>(s[0], s[1], (uint32_t)n, d_out);
    return check_launch("pmax_draws");
}

extern "C" int rfxc_pmax(const double* d_dq, int64_t n, int32_t r, int64_t seed, double* d_parts,
                         double* d_out, void* stream)
{
    if (n < 1 || r < 1) return fail(RFXC_EDATA, "pmax: bad shape");
    if (n > UINT32_MAX) return fail(RFXC_EDATA, "pmax: n exceeds uint32");
    cudaStream_t st = as_stream(stream);
    const int parts = gram_parts(n);
    const int64_t rpp = ceil_div(n, parts);
    uint64_t s[2];
    rfx_pcg32_make(seed, RFX_SEQ_PMAX, s);
    pmax_kernel<<<parts + 1, 256, 0, st>>>(d_dq, n, r, rpp, parts, s[0], s[1], d_parts);
    int rc = check_launch("pmax");
    if (rc) return rc;
    max_final_kernel<<<1, 32, 0, st>>>(d_parts, parts + 1, d_out);
    return check_launch("pmax_final");
}
