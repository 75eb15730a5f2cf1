// pairs.cu — K3: exact same-leaf co-occurrence counts + TriBlock routing.
//
// Reference: accumulate_pair_counts (_kernels.py:483-510) orchestrated by
// _pair_counts (proximity.py:159-185), the /B of full_proximity
// (proximity.py:199-200), accumulate_pair_counts_block (_kernels.py:452-480)
// and the tier routing of triblock_proximity (proximity.py:301-327).
//
// Round-1 design: output-stationary 128x128 tiles of the upper triangle.
// Each CTA stages 32-tree slices of its row block's and column block's
// codes (read coalesced from the (n, B) membership) into shared memory and
// every thread accumulates an 8x8 register micro-tile of int32 counts with
// integer compares.  The count for (i, j) is sum_b [code_b(i) == code_b(j)],
// the same integer the reference accumulates one increment at a time, so the
// output is bit-exact by construction and independent of leaf sizes.  The
// epilogue fuses the layout: packed int32, packed f64 count/B (an IEEE
// division, bit-identical to counts / float(B)), or the TriBlock row block.
#include "common.cuh"

#include <cstdlib>

namespace rfxc {

constexpr int PT = 128;     // tile edge
constexpr int PK = 32;      // trees per smem slice
constexpr int PTHREADS = 256;

__device__ __forceinline__ int64_t row_start(int64_t i, int64_t n)
{
    return i * (2 * n - i - 1) / 2;  // packed index of (i, i+1)
}

template <int LAYOUT>
__global__ void __launch_bounds__(PTHREADS)
pair_tile_kernel(const int32_t* __restrict__ codes, int64_t n, int32_t B, int64_t row_lo,
                 int64_t row_hi, void* __restrict__ out, const int32_t* __restrict__ gate)
{
    if (gate && *gate != 0) return;  // the device chose the leaf walk
    const int64_t R = blockIdx.y, C = blockIdx.x;
    if (C < R) return;  // strictly below the diagonal band: j < i everywhere
    const int64_t i0 = row_lo + R * PT, j0 = row_lo + C * PT;
    if (i0 >= row_hi || j0 >= n) return;

    __shared__ __align__(16) int32_t As[PK][PT];
    __shared__ __align__(16) int32_t Bs[PK][PT];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    int acc[8][8];
#pragma unroll
    for (int a = 0; a < 8; a++)
#pragma unroll
        for (int c = 0; c < 8; c++) acc[a][c] = 0;

    for (int b0 = 0; b0 < B; b0 += PK) {
        const int kk = min(PK, B - b0);
        // coalesced along trees: lane -> tree, row loop across threads
        for (int e = tid; e < PT * PK; e += PTHREADS) {
            const int r = e / PK, k = e % PK;
            int32_t va = -1, vb = -2;  // distinct sentinels never compare equal
            if (k < kk) {
                const int64_t i = i0 + r, j = j0 + r;
                if (i < row_hi) va = __ldg(codes + i * B + b0 + k);
                if (j < n) vb = __ldg(codes + j * B + b0 + k);
            }
            As[k][r] = va;
            Bs[k][r] = vb;
        }
        __syncthreads();
#pragma unroll 4
        for (int k = 0; k < kk; k++) {
            const int4 a0 = *reinterpret_cast<const int4*>(&As[k][ty * 8]);
            const int4 a1 = *reinterpret_cast<const int4*>(&As[k][ty * 8 + 4]);
            const int4 c0 = *reinterpret_cast<const int4*>(&Bs[k][tx * 8]);
            const int4 c1 = *reinterpret_cast<const int4*>(&Bs[k][tx * 8 + 4]);
            const int ra[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const int rc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
            for (int a = 0; a < 8; a++)
#pragma unroll
                for (int c = 0; c < 8; c++) acc[a][c] += (ra[a] == rc[c]);
        }
        __syncthreads();
    }

    // epilogue: (i, j) with j > i only
#pragma unroll
    for (int a = 0; a < 8; a++) {
        const int64_t i = i0 + ty * 8 + a;
        if (i >= row_hi) continue;
        const int64_t rbase = row_start(i, n) - row_start(row_lo, n) - i - 1;
#pragma unroll
        for (int c = 0; c < 8; c++) {
            const int64_t j = j0 + tx * 8 + c;
            if (j <= i || j >= n) continue;
            if (LAYOUT == RFXC_UPPER_I32)
                reinterpret_cast<int32_t*>(out)[rbase + j] = acc[a][c];
            else if (LAYOUT == RFXC_UPPER_F64)
                reinterpret_cast<double*>(out)[rbase + j] = (double)acc[a][c] / (double)B;
            else
                reinterpret_cast<int32_t*>(out)[(i - row_lo) * n + j] = acc[a][c];
        }
    }
}

// ------------------------------------------------- leaf-segmented counts
// The reference's own formulation (accumulate_pair_counts, _kernels.py:
// 491-510): per tree, every same-leaf pair (i, j) of the bucketed samples
// adds one.  Here it is row-stationary so that the output is written once,
// coalesced: a CTA owns output row i (a window of its columns at a time) as
// packed 16-bit counters in shared memory; for every tree a warp reads the
// members that follow i in its leaf's run of the K2 bucket (one coalesced
// 32-entry read of perm from pos_nb[i, b] + 1 up to the next first-member
// flag), and bumps their counters with shared-memory atomics.  Work is
// n*B warp-steps + (same-leaf pairs)/32 instead of n^2*B/2 compares, so at
// the configs' leaf sizes (0.8 % of pairs share a leaf per tree at 50k) the
// kernel is bound by writing the triangle, not by the counting.  Integer
// sums: bit-exact and order-independent.
constexpr int SEG_THREADS = 512;
#ifndef RFXC_SEG_UNROLL
#define RFXC_SEG_UNROLL 16
#endif
constexpr int SEG_UNROLL = RFXC_SEG_UNROLL;
constexpr int SEG_QUOT_MAX = 4096;

// pos_tm[b * n + sample] = absolute index of the sample in perm (tree b);
// perm16 (nullable, n <= 65536): the sample ids as 16-bit values — half the
// bytes for the leaf walk, so the whole bucket stays L2-resident.
__global__ void perm_inverse_kernel(const uint32_t* __restrict__ perm, int64_t total, int64_t n,
                                    uint32_t* __restrict__ pos_tm, uint16_t* __restrict__ perm16)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += stride) {
        const int64_t b = e / n;
        const uint32_t s = __ldg(perm + e) & ~RFXC_PERM_FIRST;
        pos_tm[b * n + s] = (uint32_t)e;
        if (perm16) perm16[e] = (uint16_t)s;
    }
}

// sum over leaves of s (s - 1) / 2 from the run starts (integer, exact).
__global__ void same_leaf_pairs_kernel(const int64_t* __restrict__ seg, int64_t leaves,
                                       unsigned long long* __restrict__ out)
{
    unsigned long long acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < leaves; g += stride) {
        const unsigned long long s = (unsigned long long)(seg[g + 1] - seg[g]);
        acc += s * (s - (s > 0)) / 2;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

// Dynamic shared memory of pair_seg_kernel: counters (win/2 words, padded to
// 8 bytes) | quotient table (B + 1 doubles, f64 layout, B <= SEG_QUOT_MAX) |
// entry prefix over the trees (B + 1 int32) | run base per tree (B uint32).
__host__ __device__ __forceinline__ int64_t seg_cnt_words(int64_t win)
{
    return (((win + 1) / 2) + 1) & ~(int64_t)1;
}

template <int LAYOUT>
__host__ __device__ __forceinline__ bool seg_has_quot(int32_t B)
{
    return LAYOUT == RFXC_UPPER_F64 && B <= SEG_QUOT_MAX;
}

template <int LAYOUT>
__host__ __device__ __forceinline__ int64_t seg_smem_bytes(int64_t win, int32_t B)
{
    return seg_cnt_words(win) * 4 + (seg_has_quot<LAYOUT>(B) ? (int64_t)(B + 1) * 8 : 0) +
           (int64_t)(2 * B + 2) * 4;
}

template <int LAYOUT, typename IDX>
__global__ void __launch_bounds__(SEG_THREADS, 2)
pair_seg_kernel(const uint32_t* __restrict__ pos_nb, const IDX* __restrict__ perm,
                const int32_t* __restrict__ codes_nb, const int64_t* __restrict__ seg,
                const int64_t* __restrict__ leaf_base, int64_t n, int32_t B, int64_t row_lo,
                int64_t row_hi, int64_t win, void* __restrict__ out,
                const int32_t* __restrict__ gate)
{
    if (gate && *gate != 1) return;  // the device chose the compare tiles
    extern __shared__ __align__(16) uint32_t cnt[];
    constexpr int NW = SEG_THREADS / 32;
    __shared__ int32_t s_wsum[NW];
    const int64_t i = row_lo + blockIdx.x;
    if (i >= row_hi) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t rbase = row_start(i, n) - row_start(row_lo, n) - i - 1;
    const double dB = (double)B;
    double* quot = reinterpret_cast<double*>(cnt + seg_cnt_words(win));
    int32_t* s_end = reinterpret_cast<int32_t*>(quot + (seg_has_quot<LAYOUT>(B) ? B + 1 : 0));
    uint32_t* s_base = reinterpret_cast<uint32_t*>(s_end + B + 1);
    // f64 layout: the B + 1 possible quotients c / B (each one IEEE
    // division), so the epilogue is a table lookup
    if (seg_has_quot<LAYOUT>(B))
        for (int c = tid; c <= B; c += SEG_THREADS) quot[c] = (double)c / dB;

    // Tree b: the members of i's leaf that follow i in its run of perm
    // (samples > i, ascending) — m_b of them from perm index p_b + 1.  Thread
    // tid owns trees [tid*per, (tid+1)*per); a block scan turns the m_b into
    // the flat entry space [0, T) that the warps then split evenly.
    const int per = (B + SEG_THREADS - 1) / SEG_THREADS;
    const int bl = min(B, tid * per), bh = min(B, bl + per);
    int32_t mine = 0;
    for (int b = bl; b < bh; b++) {
        const uint32_t p = __ldg(pos_nb + i * B + b);
        const int64_t g = __ldg(leaf_base + b) + __ldg(codes_nb + i * B + b);
        const int32_t m = (int32_t)(__ldg(seg + g + 1) - (int64_t)p - 1);
        s_end[b + 1] = m;  // temporarily m_b
        s_base[b] = p + 1u;
        mine += m;
    }
    int32_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    int32_t before = incl - mine;
    for (int w = 0; w < warp; w++) before += s_wsum[w];
    for (int b = bl; b < bh; b++) {  // m_b -> inclusive prefix; base - exclusive prefix
        const int32_t m = s_end[b + 1];
        s_base[b] -= (uint32_t)before;  // mod 2^32: + flat entry = perm index
        before += m;
        s_end[b + 1] = before;
    }
    if (tid == 0) s_end[0] = 0;
    __syncthreads();
    const int32_t T = s_end[B];
    // warp w walks entries [e_lo, e_hi), one per lane per step
    const int32_t e_lo = (int32_t)((int64_t)T * warp / NW);
    const int32_t e_hi = (int32_t)((int64_t)T * (warp + 1) / NW);

    for (int64_t c0 = i + 1; c0 < n; c0 += win) {
        const int64_t c1 = min64(n, c0 + win);
        const int64_t words = (c1 - c0 + 1) >> 1;
        const uint32_t wc0 = (uint32_t)c0, wlen = (uint32_t)(c1 - c0);
        for (int64_t w = tid; w < words; w += SEG_THREADS) cnt[w] = 0u;
        __syncthreads();
        // t = tree of this lane's entry: upper-bound search once, then it only
        // moves forward
        int t = 0;
        {
            const int32_t e = e_lo + lane;
            int lo = 0, hi = B;  // largest t with s_end[t] <= e
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (s_end[mid] <= e) lo = mid;
                else hi = mid;
            }
            t = lo;
        }
        // the current tree's end and base stay in registers; reloaded only
        // when the lane's entry crosses into the next tree
        int32_t tend = s_end[t + 1];
        uint32_t tbase = s_base[t];
        // full groups of SEG_UNROLL lane steps (no bounds checks), then the tail
        int32_t e0 = e_lo + lane;
        const int32_t e_full = e_hi - 32 * (SEG_UNROLL - 1);  // e0 < e_full: the whole group fits
        for (; e0 < e_full; e0 += 32 * SEG_UNROLL) {
            uint32_t v[SEG_UNROLL];
#pragma unroll
            for (int u = 0; u < SEG_UNROLL; u++) {
                const int32_t e = e0 + u * 32;
                while (tend <= e) {
                    t++;
                    tend = s_end[t + 1];
                    tbase = s_base[t];
                }
                v[u] = (uint32_t)__ldg(perm + (uint32_t)(tbase + (uint32_t)e));
            }
#pragma unroll
            for (int u = 0; u < SEG_UNROLL; u++) {
                // column offset in the window: one unsigned compare covers both ends
                const uint32_t o = (v[u] & ~RFXC_PERM_FIRST) - wc0;
                if (o < wlen) atomicAdd(cnt + (o >> 1), 1u << ((o & 1u) << 4));
            }
        }
        for (; e0 < e_hi; e0 += 32) {
            while (tend <= e0) {
                t++;
                tend = s_end[t + 1];
                tbase = s_base[t];
            }
            const uint32_t v = (uint32_t)__ldg(perm + (uint32_t)(tbase + (uint32_t)e0));
            const uint32_t o = (v & ~RFXC_PERM_FIRST) - wc0;
            if (o < wlen) atomicAdd(cnt + (o >> 1), 1u << ((o & 1u) << 4));
        }
        __syncthreads();
        // the row leaves once, streamed past L2 (evict-first) so the perm runs
        // the other rows walk stay resident
        for (int64_t j = c0 + tid; j < c1; j += SEG_THREADS) {
            const int64_t o = j - c0;
            const int32_t c = (int32_t)((cnt[o >> 1] >> ((o & 1) << 4)) & 0xffffu);
            if (LAYOUT == RFXC_UPPER_I32)
                __stcs(reinterpret_cast<int32_t*>(out) + rbase + j, c);
            else if (LAYOUT == RFXC_UPPER_F64)
                __stcs(reinterpret_cast<double*>(out) + rbase + j,
                       seg_has_quot<LAYOUT>(B) ? quot[c] : (double)c / dB);
            else
                __stcs(reinterpret_cast<int32_t*>(out) + (i - row_lo) * n + j, c);
        }
        __syncthreads();
    }
}

// gate = 1 (leaf walk) when the same-leaf pairs are at most share x units:
// both K3 kernels are launched and the one not chosen exits at once, so the
// choice needs no host round trip
__global__ void pair_gate_kernel(const unsigned long long* __restrict__ pairs, double units,
                                 double share, int32_t* __restrict__ gate)
{
    if (threadIdx.x == 0) *gate = ((double)*pairs <= share * units) ? 1 : 0;
}

// ---------------------------------------------------------------- TriBlock
constexpr double ZERO_TIER = 1e-6;  // proximity.py:39

__global__ void triblock_count_kernel(const int32_t* __restrict__ counts, int64_t n, int32_t B,
                                      int64_t row_lo, int64_t row_hi, double tau,
                                      int64_t* __restrict__ row_counts)
{
    const int lane = threadIdx.x & 31;
    const int64_t rows = row_hi - row_lo;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const double dB = (double)B;
    for (int64_t r = warp; r < rows; r += nwarps) {
        const int64_t i = row_lo + r;
        const int32_t* row = counts + (row_start(i, n) - row_start(row_lo, n));
        const int64_t m = n - i - 1;
        int hot = 0, cold = 0;
        for (int64_t q = lane; q < m; q += 32) {
            const double v = (double)row[q] / dB;
            if (v > ZERO_TIER) {
                if (v >= tau) hot++;
                else cold++;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            hot += __shfl_xor_sync(0xffffffffu, hot, o);
            cold += __shfl_xor_sync(0xffffffffu, cold, o);
        }
        if (lane == 0) {
            row_counts[r] = hot;
            row_counts[rows + r] = cold;
        }
    }
}

__global__ void triblock_emit_kernel(const int32_t* __restrict__ counts, int64_t n, int32_t B,
                                     int64_t row_lo, int64_t row_hi, double tau,
                                     const int64_t* __restrict__ row_off, int32_t* hot_i,
                                     int32_t* hot_j, double* hot_v, int32_t* cold_i,
                                     int32_t* cold_j, double* cold_v)
{
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t rows = row_hi - row_lo;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const double dB = (double)B;
    for (int64_t r = warp; r < rows; r += nwarps) {
        const int64_t i = row_lo + r;
        const int32_t* row = counts + (row_start(i, n) - row_start(row_lo, n));
        const int64_t m = n - i - 1;
        int64_t ph = row_off[r], pc = row_off[rows + r];
        for (int64_t q0 = 0; q0 < m; q0 += 32) {
            const int64_t q = q0 + lane;
            double v = 0.0;
            if (q < m) v = (double)row[q] / dB;
            const bool keep = v > ZERO_TIER;
            const bool is_hot = keep && v >= tau, is_cold = keep && !(v >= tau);
            const unsigned mh = __ballot_sync(0xffffffffu, is_hot);
            const unsigned mc = __ballot_sync(0xffffffffu, is_cold);
            const int32_t j = (int32_t)(i + 1 + q);
            if (is_hot) {
                const int64_t at = ph + __popc(mh & lt);
                hot_i[at] = (int32_t)i;
                hot_j[at] = j;
                hot_v[at] = v;
            }
            if (is_cold) {
                const int64_t at = pc + __popc(mc & lt);
                cold_i[at] = (int32_t)i;
                cold_j[at] = j;
                cold_v[at] = v;
            }
            ph += __popc(mh);
            pc += __popc(mc);
        }
    }
}

// Single-CTA exclusive scan (int64), chunked with a running carry.
__global__ void __launch_bounds__(1024)
scan_i64_kernel(const int64_t* __restrict__ in, int64_t count, int64_t* __restrict__ out,
                int64_t* total)
{
    __shared__ int64_t wsum[32];
    __shared__ int64_t carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < count; base += 1024) {
        const int64_t idx = base + tid;
        const int64_t v = idx < count ? in[idx] : 0;
        int64_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        int64_t before = carry;
        for (int w = 0; w < warp; w++) before += wsum[w];
        if (idx < count) out[idx] = before + incl - v;
        __syncthreads();
        if (tid == 0) {
            int64_t s = 0;
            for (int w = 0; w < 32; w++) s += wsum[w];
            carry += s;
        }
        __syncthreads();
    }
    if (tid == 0 && total) *total = carry;
}

}  // namespace rfxc

using namespace rfxc;

extern "C" int rfxc_pair_counts(const int32_t* d_codes_nb, int64_t n, int32_t B, int64_t row_lo,
                                int64_t row_hi, int32_t layout, void* d_out, const int32_t* d_gate,
                                void* stream)
{
    if (n < 2 || B < 1 || row_lo < 0 || row_hi > n || row_lo >= row_hi)
        return fail(RFXC_EDATA, "pair_counts: bad shape n=%lld rows=[%lld,%lld)", (long long)n,
                    (long long)row_lo, (long long)row_hi);
    cudaStream_t st = as_stream(stream);
    const int64_t rb = ceil_div(row_hi - row_lo, PT), cb = ceil_div(n - row_lo, PT);
    if (rb > 65535) return fail(RFXC_EDATA, "pair_counts: too many row blocks; shard rows");
    dim3 grid((unsigned)cb, (unsigned)rb);
    switch (layout) {
    case RFXC_UPPER_I32:
        pair_tile_kernel<RFXC_UPPER_I32><<<grid, PTHREADS, 0, st>>>(d_codes_nb, n, B, row_lo,
                                                                    row_hi, d_out, d_gate);
        break;
    case RFXC_UPPER_F64:
        pair_tile_kernel<RFXC_UPPER_F64><<<grid, PTHREADS, 0, st>>>(d_codes_nb, n, B, row_lo,
                                                                    row_hi, d_out, d_gate);
        break;
    case RFXC_BLOCK_I32: {
        if (d_gate) return fail(RFXC_EDATA, "pair_counts: the gated launch takes packed layouts");
        cudaError_t e = cudaMemsetAsync(d_out, 0, (size_t)(row_hi - row_lo) * n * 4, st);
        if (e != cudaSuccess) return fail(RFXC_ECUDA, "memset: %s", cudaGetErrorString(e));
        pair_tile_kernel<RFXC_BLOCK_I32><<<grid, PTHREADS, 0, st>>>(d_codes_nb, n, B, row_lo,
                                                                    row_hi, d_out, d_gate);
        break;
    }
    default:
        return fail(RFXC_EDATA, "pair_counts: unknown layout %d", layout);
    }
    return check_launch("pair_counts");
}

extern "C" int rfxc_perm_positions(const uint32_t* d_perm, int64_t n, int32_t Bl,
                                   uint32_t* d_pos_tm, uint16_t* d_perm16, void* stream)
{
    if (d_perm16 && n > 65536) return fail(RFXC_EDATA, "perm_positions: 16-bit ids need n <= 65536");
    const int64_t total = n * (int64_t)Bl;
    if (n < 1 || Bl < 1 || total >= ((int64_t)1 << 32))
        return fail(RFXC_EDATA, "perm_positions: n*Bl = %lld outside [1, 2^32)", (long long)total);
    const int grid = (int)std::min<int64_t>(ceil_div(total, 256), (int64_t)sm_count() * 16);
    perm_inverse_kernel<<<grid, 256, 0, as_stream(stream)>>>(d_perm, total, n, d_pos_tm, d_perm16);
    return check_launch("perm_positions");
}

extern "C" int rfxc_same_leaf_pairs(const int64_t* d_seg, int64_t leaves, uint64_t* d_out,
                                    void* stream)
{
    cudaStream_t st = as_stream(stream);
    cudaError_t e = cudaMemsetAsync(d_out, 0, sizeof(uint64_t), st);
    if (e != cudaSuccess) return fail(RFXC_ECUDA, "memset: %s", cudaGetErrorString(e));
    if (leaves <= 0) return RFXC_OK;
    const int grid = (int)std::min<int64_t>(ceil_div(leaves, 256), (int64_t)sm_count() * 8);
    same_leaf_pairs_kernel<<<grid, 256, 0, st>>>(d_seg, leaves,
                                                 reinterpret_cast<unsigned long long*>(d_out));
    return check_launch("same_leaf_pairs");
}

extern "C" int rfxc_pair_kernel_gate(const uint64_t* d_pairs, int64_t n, int32_t B, double share,
                                     int32_t* d_gate, void* stream)
{
    const double units = (double)n * (double)(n - 1) / 2.0 * (double)B;
    pair_gate_kernel<<<1, 32, 0, as_stream(stream)>>>(
        reinterpret_cast<const unsigned long long*>(d_pairs), units, share, d_gate);
    return check_launch("pair_kernel_gate");
}

template <int LAYOUT, typename IDX>
static int launch_seg(const uint32_t* pos_nb, const IDX* perm, const int32_t* codes_nb,
                      const int64_t* seg, const int64_t* leaf_base, int64_t n, int32_t B,
                      int64_t row_lo, int64_t row_hi, int64_t cap, void* out, const int32_t* gate,
                      cudaStream_t st)
{
    // two CTAs per SM: the counters get what the per-tree tables leave of
    // ~100 KB (48k columns at B = 500)
    const int64_t budget = 100 * 1024;
    const int64_t fixed = seg_smem_bytes<LAYOUT>(0, B);
    if (fixed > budget - 4096)
        return fail(RFXC_EDATA, "pair_counts_leaf: B=%d too large for the shared tables", B);
    int64_t win = std::min<int64_t>(cap, 2 * ((budget - fixed) / 4 - 2));
    win = std::max<int64_t>(1, std::min<int64_t>(n - 1 - row_lo, win));
    const size_t smem = (size_t)seg_smem_bytes<LAYOUT>(win, B);
    cudaError_t e = cudaFuncSetAttribute(pair_seg_kernel<LAYOUT, IDX>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return fail(RFXC_ECUDA, "pair_seg smem: %s", cudaGetErrorString(e));
    pair_seg_kernel<LAYOUT, IDX><<<(unsigned)(row_hi - row_lo), SEG_THREADS, smem, st>>>(
        pos_nb, perm, codes_nb, seg, leaf_base, n, B, row_lo, row_hi, win, out, gate);
    return check_launch("pair_counts_leaf");
}

template <typename IDX>
static int pair_counts_leaf_t(const uint32_t* d_pos_nb, const IDX* d_perm, const int32_t* d_codes_nb,
                              const int64_t* d_seg, const int64_t* d_leaf_base, int64_t n,
                              int32_t B, int64_t row_lo, int64_t row_hi, int32_t layout,
                              void* d_out, const int32_t* gate, cudaStream_t st)
{
    int64_t win = INT64_MAX;  // launch_seg sizes the window to the shared memory
    if (const char* w = getenv("RFXC_PAIRS_WINDOW")) win = std::max<int64_t>(2, atoll(w));  // tests
    switch (layout) {
    case RFXC_UPPER_I32:
        return launch_seg<RFXC_UPPER_I32, IDX>(d_pos_nb, d_perm, d_codes_nb, d_seg, d_leaf_base,
                                               n, B, row_lo, row_hi, win, d_out, gate, st);
    case RFXC_UPPER_F64:
        return launch_seg<RFXC_UPPER_F64, IDX>(d_pos_nb, d_perm, d_codes_nb, d_seg, d_leaf_base,
                                               n, B, row_lo, row_hi, win, d_out, gate, st);
    case RFXC_BLOCK_I32: {
        if (gate) return fail(RFXC_EDATA, "pair_counts_leaf: the gated launch takes packed layouts");
        cudaError_t e = cudaMemsetAsync(d_out, 0, (size_t)(row_hi - row_lo) * n * 4, st);
        if (e != cudaSuccess) return fail(RFXC_ECUDA, "memset: %s", cudaGetErrorString(e));
        return launch_seg<RFXC_BLOCK_I32, IDX>(d_pos_nb, d_perm, d_codes_nb, d_seg, d_leaf_base,
                                               n, B, row_lo, row_hi, win, d_out, gate, st);
    }
    default:
        return fail(RFXC_EDATA, "pair_counts_leaf: unknown layout %d", layout);
    }
}

extern "C" int rfxc_pair_counts_leaf(const uint32_t* d_pos_nb, const void* d_perm, int32_t idx_bytes,
                                     const int32_t* d_codes_nb, const int64_t* d_seg,
                                     const int64_t* d_leaf_base, int64_t n, int32_t B,
                                     int64_t row_lo, int64_t row_hi, int32_t layout, void* d_out,
                                     const int32_t* d_gate, void* stream)
{
    if (n < 2 || B < 1 || row_lo < 0 || row_hi > n || row_lo >= row_hi)
        return fail(RFXC_EDATA, "pair_counts_leaf: bad shape n=%lld rows=[%lld,%lld)",
                    (long long)n, (long long)row_lo, (long long)row_hi);
    if (B > 4096) return fail(RFXC_EDATA, "pair_counts_leaf: B=%d > 4096 (shared per-tree tables)", B);
    if (row_hi - row_lo > 0x7fffffffLL) return fail(RFXC_EDATA, "pair_counts_leaf: rows");
    if (idx_bytes == 2 && n > 65536) return fail(RFXC_EDATA, "pair_counts_leaf: 16-bit ids need n <= 65536");
    cudaStream_t st = as_stream(stream);
    if (idx_bytes == 2)
        return pair_counts_leaf_t(d_pos_nb, static_cast<const uint16_t*>(d_perm), d_codes_nb, d_seg,
                                  d_leaf_base, n, B, row_lo, row_hi, layout, d_out, d_gate, st);
    if (idx_bytes != 4) return fail(RFXC_EDATA, "pair_counts_leaf: idx_bytes must be 2 or 4");
    return pair_counts_leaf_t(d_pos_nb, static_cast<const uint32_t*>(d_perm), d_codes_nb, d_seg,
                              d_leaf_base, n, B, row_lo, row_hi, layout, d_out, d_gate, st);
}

extern "C" int rfxc_triblock_count(const int32_t* d_counts_upper, int64_t n, int32_t B,
                                   int64_t row_lo, int64_t row_hi, double tau,
                                   int64_t* d_row_counts, void* stream)
{
    if (row_lo < 0 || row_hi > n || row_lo >= row_hi) return fail(RFXC_EDATA, "triblock: rows");
    int64_t rows = row_hi - row_lo;
    int grid = (int)std::min<int64_t>(ceil_div(rows * 32, 256), (int64_t)sm_count() * 16);
    triblock_count_kernel<<<grid, 256, 0, as_stream(stream)>>>(d_counts_upper, n, B, row_lo,
                                                               row_hi, tau, d_row_counts);
    return check_launch("triblock_count");
}

extern "C" int rfxc_triblock_emit(const int32_t* d_counts_upper, int64_t n, int32_t B,
                                  int64_t row_lo, int64_t row_hi, double tau,
                                  const int64_t* d_row_offsets, int32_t* d_hot_i, int32_t* d_hot_j,
                                  double* d_hot_v, int32_t* d_cold_i, int32_t* d_cold_j,
                                  double* d_cold_v, void* stream)
{
    if (row_lo < 0 || row_hi > n || row_lo >= row_hi) return fail(RFXC_EDATA, "triblock: rows");
    int64_t rows = row_hi - row_lo;
    int grid = (int)std::min<int64_t>(ceil_div(rows * 32, 256), (int64_t)sm_count() * 16);
    triblock_emit_kernel<<<grid, 256, 0, as_stream(stream)>>>(
        d_counts_upper, n, B, row_lo, row_hi, tau, d_row_offsets, d_hot_i, d_hot_j, d_hot_v,
        d_cold_i, d_cold_j, d_cold_v);
    return check_launch("triblock_emit");
}

extern "C" int rfxc_exclusive_scan_i64(const int64_t* d_in, int64_t count, int64_t* d_out,
                                       int64_t* d_total, void* stream)
{
    if (count < 0) return fail(RFXC_EDATA, "scan: negative count");
    scan_i64_kernel<<<1, 1024, 0, as_stream(stream)>>>(d_in, count, d_out, d_total);
    return check_launch("exclusive_scan_i64");
}
