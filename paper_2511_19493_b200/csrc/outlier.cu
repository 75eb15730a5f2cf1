// outlier.cu — SURVEY §8(f) rank 1: outlier_scores on the device.
//
// Reference: outlier_scores (proximity.py:432-485): score_i = mean over
// j != i of c(p_ij), c(p) = 1 / max(p, floor)^2 (floor = 1/B by default),
// for the FullTriangle (packed f64 upper triangle) and the low-rank factor
// (p_ij = clip(q_i . q_j, 0, 1), the diagonal term subtracted from the full
// row sum exactly as :475-479 does).  Per element the arithmetic is the
// reference's (an IEEE square, then an IEEE division); only the order of the
// row sums differs, and it is fixed, so scores are bit-reproducible.
//
// Packed triangle: a warp per row sums its contiguous segment (the row
// part); a CTA per block of OB_ROWS rows gives every column j its partial
// over those rows (thread per column, rows in order: coalesced, since the
// entries (i, j), (i, j + 1) are adjacent); one thread per j adds the row
// part and the block partials in block order.
//
// Low rank: a CTA per 128-row block I keeps Q_I in shared memory and streams
// 64-row column blocks Q_J through a cp.async double buffer; each of the 16
// warps owns one 8-row tile row and computes its 8 x 64 strip of Q_I Q_J^T
// on the FP64 tensor cores (DMMA.8x8x4), then applies c() and accumulates
// its rows' sums in registers (J blocks in order).  n^2 r work: ~20 ms at
// n = 100k, r = 32.
#include "common.cuh"

namespace rfxc {

constexpr int OB_ROWS = 256;

__device__ __forceinline__ double outlier_c(double p, double floor_)
{
    const double m = p > floor_ ? p : floor_;  // np.maximum(p, floor)
    return 1.0 / (m * m);
}

__global__ void outlier_rows_kernel(const double* __restrict__ packed, int64_t n, double floor_,
                                    double* __restrict__ rowsum)
{
    const int lane = threadIdx.x & 31;
    const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (i >= n) return;
    const int64_t start = i * (2 * n - i - 1) / 2, m = n - 1 - i;
    double s = 0.0;
    for (int64_t t = lane; t < m; t += 32) s += outlier_c(__ldcs(packed + start + t), floor_);
    s = warp_sum(s);
    if (lane == 0) rowsum[i] = s;
}

// colpart[blk][j] = sum over rows i of block blk with i < j of c(p_ij)
__global__ void outlier_cols_kernel(const double* __restrict__ packed, int64_t n, double floor_,
                                    double* __restrict__ colpart)
{
    const int64_t blk = blockIdx.y;
    const int64_t i0 = blk * OB_ROWS, i1 = min64(n, i0 + OB_ROWS);
    const int64_t j = i0 + 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= n) return;
    double s = 0.0;
    for (int64_t i = i0; i < i1 && i < j; i++)
        s += outlier_c(__ldcs(packed + i * (2 * n - i - 1) / 2 + (j - i - 1)), floor_);
    colpart[blk * n + j] = s;
}

__global__ void outlier_final_kernel(const double* __restrict__ rowsum,
                                     const double* __restrict__ colpart, int64_t n, int nblk,
                                     double* __restrict__ scores)
{
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= n) return;
    double s = rowsum[j];
    const int64_t last = min64(nblk, (j + OB_ROWS - 1) / OB_ROWS);  // blocks with rows < j
    for (int64_t b = 0; b < last; b++) s += colpart[b * n + j];
    scores[j] = s / (double)(n - 1);
}

// ------------------------------------------------------------- low rank
// Rows per CTA = 8 * WARPS, streamed column block OL_J: <16, 64> keeps 128
// rows of Q_I in shared memory; ranks whose (128 + 2 * 64) rows exceed it
// run <4, 32> (32 rows, 32-row column blocks).  Every lane sums the columns
// j = 2 fr + h (mod 8) in ascending order in both, so the scores are the same
// bits whichever variant runs.

__host__ __device__ inline int ol_ld(int rp) { return rp + ((4 - rp % 16) + 16) % 16; }

__device__ __forceinline__ void ol_cp8(void* smem, const void* gmem, bool ok)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(ok ? 8 : 0)
                 : "memory");
}

template <int WARPS, int OL_J>
__global__ void __launch_bounds__(WARPS * 32, 1)
outlier_lowrank_kernel(const double* __restrict__ Q, int64_t n, int r, double floor_,
                       double* __restrict__ scores)
{
    constexpr int OL_I = 8 * WARPS;
    extern __shared__ __align__(16) double osm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int fr = lane & 3, fc = lane >> 2;
    const int rp = (r + 3) / 4 * 4, lq = ol_ld(rp);
    double* qi = osm;                  // OL_I x lq
    double* qj = osm + OL_I * lq;      // 2 x OL_J x lq
    const int64_t i0 = blockIdx.x * (int64_t)OL_I;
    for (int e = threadIdx.x; e < OL_I * lq; e += blockDim.x) {
        const int row = e / lq, c = e % lq;
        const int64_t g = i0 + row;
        qi[e] = (g < n && c < r) ? Q[g * r + c] : 0.0;
    }
    auto stage = [&](int64_t j0, int buf) {
        double* dst = qj + buf * OL_J * lq;
        for (int e = threadIdx.x; e < OL_J * rp; e += blockDim.x) {
            const int row = e / rp, c = e % rp;
            const int64_t g = j0 + row;
            const bool ok = g < n && c < r;
            ol_cp8(dst + row * lq + c, ok ? Q + g * r + c : Q, ok);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    const int64_t nj = (n + OL_J - 1) / OL_J;
    stage(0, 0);
    const int64_t my_row = i0 + 8 * warp + fc;  // the row this lane accumulates
    double acc = 0.0, own = 0.0;
    const double* pa = qi + (8 * warp + fc) * lq + fr;
    for (int64_t jb = 0; jb < nj; jb++) {
        if (jb + 1 < nj) stage((jb + 1) * OL_J, (int)((jb + 1) & 1));
        else asm volatile("cp.async.commit_group;\n" ::: "memory");
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        __syncthreads();
        const double* qb = qj + (jb & 1) * OL_J * lq;
        double d[OL_J / 8][2];
#pragma unroll
        for (int t = 0; t < OL_J / 8; t++) d[t][0] = d[t][1] = 0.0;
        for (int ks = 0; ks < rp / 4; ks++) {
            const double a = pa[4 * ks];
#pragma unroll
            for (int t = 0; t < OL_J / 8; t++) dmma884(d[t][0], d[t][1], a, qb[(8 * t + fc) * lq + 4 * ks + fr]);
        }
#pragma unroll
        for (int t = 0; t < OL_J / 8; t++)
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int64_t j = jb * OL_J + 8 * t + 2 * fr + h;
                if (j < n) {
                    const double p = fmin(fmax(d[t][h], 0.0), 1.0);  // np.clip(., 0, 1)
                    const double c = outlier_c(p, floor_);
                    acc += c;
                    if (j == my_row) own = c;
                }
            }
        __syncthreads();
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    own += __shfl_xor_sync(0xffffffffu, own, 1);
    own += __shfl_xor_sync(0xffffffffu, own, 2);
    if (fr == 0 && my_row < n) scores[my_row] = (acc - own) / (double)(n - 1);
}

}  // namespace rfxc

using namespace rfxc;

extern "C" int64_t rfxc_outlier_work_bytes(int64_t n)
{
    const int64_t nblk = (n + OB_ROWS - 1) / OB_ROWS;
    return (nblk + 1) * n * 8;
}

extern "C" int rfxc_outlier_packed(const double* d_packed, int64_t n, double floor_,
                                   double* d_scores, void* d_work, void* stream)
{
    if (n < 2) return fail(RFXC_EDATA, "outlier scores need n >= 2");
    if (!(floor_ > 0.0)) return fail(RFXC_EDATA, "clamp_floor must be positive");
    cudaStream_t st = as_stream(stream);
    double* rowsum = static_cast<double*>(d_work);
    double* colpart = rowsum + n;
    const int nblk = (int)((n + OB_ROWS - 1) / OB_ROWS);
    outlier_rows_kernel<<<(unsigned)ceil_div(n * 32, 256), 256, 0, st>>>(d_packed, n, floor_, rowsum);
    int rc = check_launch("outlier_rows");
    if (rc) return rc;
    outlier_cols_kernel<<<dim3((unsigned)ceil_div(n, 256), nblk), 256, 0, st>>>(d_packed, n, floor_,
                                                                              colpart);
    rc = check_launch("outlier_cols");
    if (rc) return rc;
    outlier_final_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(rowsum, colpart, n, nblk,
                                                                     d_scores);
    return check_launch("outlier_final");
}

extern "C" int rfxc_outlier_lowrank(const double* d_dq, int64_t n, int32_t r, double floor_,
                                    double* d_scores, void* stream)
{
    if (n < 2) return fail(RFXC_EDATA, "outlier scores need n >= 2");
    if (r < 1 || r > 256) return fail(RFXC_EDATA, "outlier_lowrank: rank %d outside [1, 256]", r);
    if (!(floor_ > 0.0)) return fail(RFXC_EDATA, "clamp_floor must be positive");
    const int rp = (r + 3) / 4 * 4, lq = ol_ld(rp);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(outlier_lowrank_kernel<16, 64>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(outlier_lowrank_kernel<4, 32>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr = true;
    }
    const size_t big = (size_t)(128 + 2 * 64) * lq * 8, small = (size_t)(32 + 2 * 32) * lq * 8;
    if (big <= 227 * 1024)
        outlier_lowrank_kernel<16, 64><<<(unsigned)ceil_div(n, 128), 512, big,
                                         as_stream(stream)>>>(d_dq, n, r, floor_, d_scores);
    else if (small <= 227 * 1024)
        outlier_lowrank_kernel<4, 32><<<(unsigned)ceil_div(n, 32), 128, small,
                                       as_stream(stream)>>>(d_dq, n, r, floor_, d_scores);
    else
        return fail(RFXC_EDATA, "outlier_lowrank: rank %d too large", r);
    return check_launch("outlier_lowrank");
}
