// bucket.cu — K2: per-tree stable counting sort of samples by leaf.
//
// Reference: the counting sort inside accumulate_pair_counts[_block]
// (_kernels.py:458-468, :491-501), which the reference redoes for every
// tree (and for every (row block, tree) in TriBlock).  Here it runs once per
// tree and the result (perm + per-leaf run starts) is shared by the sketch
// (K4) and the pair kernels.
//
// One CTA per tree, W warps.  Warp w owns the contiguous sample range
// [w n/W, (w+1) n/W) and keeps its own 16-bit leaf histogram in shared
// memory (two counters per 32-bit word, incremented with word atomics), so
// the W ranges are counted and scattered in parallel:
//   (1) per-warp histograms, (2) per leaf: run start (block scan over the
//   leaf totals) and the exclusive prefix of the warp counts -> every
//   warp's private cursor, (3) stable scatter: each warp walks its range in
//   32-sample steps, __match_any_sync groups equal leaves, the group leader
//   advances its cursor and every lane writes at cursor + rank-in-group.
// Ranges are ordered and each warp walks its own range in ascending order,
// so members come out ascending inside every leaf (the reference's bucket
// order).  The first member of every leaf carries bit 31 (RFXC_PERM_FIRST)
// so the sketch can find leaf boundaries from perm alone; an empty leaf sets
// *has_empty.  Trees with too many leaves for shared memory fall back to a
// single-warp scatter over global counters.
#include "common.cuh"

namespace rfxc {

constexpr int BUCKET_SMEM_BUDGET = 220 * 1024;

// smem: hist (W x Lp/2 words, Lp = L rounded up to even) | start (L int32)
__global__ void __launch_bounds__(512)
bucket_kernel(const int32_t* __restrict__ codes_tm, int64_t n,
              const int64_t* __restrict__ leaf_base, int32_t Bl,
              uint32_t* __restrict__ perm, int64_t* __restrict__ seg,
              int32_t* __restrict__ has_empty)
{
    extern __shared__ uint32_t bsm[];
    __shared__ int32_t warp_sums[32];
    __shared__ int32_t carry;
    const int b = blockIdx.x;
    const int64_t g0 = leaf_base[b];
    const int32_t L = (int32_t)(leaf_base[b + 1] - g0);
    const int Lw = (L + 1) >> 1;  // 32-bit words per warp histogram
    const int W = blockDim.x >> 5;
    uint32_t* hist = bsm;                                    // W * Lw words
    int32_t* start = reinterpret_cast<int32_t*>(bsm + (int64_t)W * Lw);
    const int32_t* codes = codes_tm + (int64_t)b * n;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t lo = n * warp / W, hi = n * (warp + 1) / W;

    for (int e = tid; e < W * Lw; e += blockDim.x) hist[e] = 0u;
    __syncthreads();
    // (1) per-warp 16-bit histograms (ranges hold < 65536 samples)
    uint32_t* h = hist + (int64_t)warp * Lw;
    constexpr int U = 8;  // code loads in flight per lane
    for (int64_t base = lo; base < hi; base += 32 * U) {
        int c[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t i = base + u * 32 + lane;
            c[u] = i < hi ? __ldg(codes + i) : -1;
        }
#pragma unroll
        for (int u = 0; u < U; u++)
            if (c[u] >= 0) atomicAdd(h + (c[u] >> 1), (c[u] & 1) ? 0x10000u : 1u);
    }
    __syncthreads();

    // (2) leaf totals -> run starts (block scan)
    if (tid == 0) carry = 0;
    __syncthreads();
    int empty = 0, big = 0;
    for (int base = 0; base < L; base += blockDim.x) {
        const int l = base + tid;
        int tot = 0;
        if (l < L) {
            const int sh = (l & 1) * 16;
            for (int w = 0; w < W; w++) tot += (int)((hist[(int64_t)w * Lw + (l >> 1)] >> sh) & 0xffffu);
            empty |= (tot == 0);
            big |= (tot >= 65536);
        }
        int incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) warp_sums[warp] = incl;
        __syncthreads();
        int before = carry;
        for (int w = 0; w < warp; w++) before += warp_sums[w];
        if (l < L) {
            const int excl = before + incl - tot;
            start[l] = excl;
            seg[g0 + l] = (int64_t)b * n + excl;
        }
        __syncthreads();
        if (tid == 0) {
            int s = 0;
            for (int w = 0; w < W; w++) s += warp_sums[w];
            carry += s;
        }
        __syncthreads();
    }
    if (__syncthreads_or(empty) && tid == 0) atomicExch(has_empty, 1);
    if (b == Bl - 1 && tid == 0) seg[leaf_base[Bl]] = (int64_t)Bl * n;
    uint32_t* out = perm + (int64_t)b * n;
    const unsigned lt = (1u << lane) - 1u;

    if (__syncthreads_or(big)) {
        // a leaf with >= 65536 members: 16-bit prefixes could overflow, so
        // one warp scatters the whole tree with 32-bit cursors (rare)
        if (warp != 0) return;
        for (int64_t base = 0; base < n; base += 32) {
            const int64_t i = base + lane;
            const int c = i < n ? __ldg(codes + i) : -1;
            const unsigned peers = __match_any_sync(0xffffffffu, c);
            const int leader = __ffs(peers) - 1;
            int cur = 0;
            if (lane == leader && c >= 0) {
                cur = start[c];
                start[c] = cur + __popc(peers);
            }
            cur = __shfl_sync(0xffffffffu, cur, leader);
            if (c >= 0) {
                const int pos = cur + __popc(peers & lt);
                const bool first = (int64_t)pos == seg[g0 + c] - (int64_t)b * n;
                out[pos] = (uint32_t)i | (first ? RFXC_PERM_FIRST : 0u);
            }
            __syncwarp();
        }
        return;
    }

    // per leaf: warp counts -> exclusive prefix over the warps, in place
    // (two leaves share a word, so the halves are rewritten with atomics)
    for (int l = tid; l < L; l += blockDim.x) {
        const int sh = (l & 1) * 16;
        int pre = 0;
        for (int w = 0; w < W; w++) {
            uint32_t* word = hist + (int64_t)w * Lw + (l >> 1);
            const int c = (int)((*word >> sh) & 0xffffu);
            atomicAdd(word, (uint32_t)(pre - c) << sh);
            pre += c;
        }
    }
    __syncthreads();

    // (3) stable scatter of this warp's range (U steps of codes in flight)
    int cn[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
        const int64_t i = lo + u * 32 + lane;
        cn[u] = i < hi ? __ldg(codes + i) : -1;
    }
    for (int64_t base = lo; base < hi; base += 32) {
        const int64_t i = base + lane;
        const int c = cn[0];
#pragma unroll
        for (int u = 0; u + 1 < U; u++) cn[u] = cn[u + 1];
        {
            const int64_t ia = base + U * 32 + lane;
            cn[U - 1] = ia < hi ? __ldg(codes + ia) : -1;
        }
        const unsigned peers = __match_any_sync(0xffffffffu, c);
        const int leader = __ffs(peers) - 1;
        int rel = 0;
        if (lane == leader && c >= 0) {
            const int sh = (c & 1) * 16;
            uint32_t* word = h + (c >> 1);
            rel = (int)((*word >> sh) & 0xffffu);
            atomicAdd(word, (uint32_t)__popc(peers) << sh);
        }
        rel = __shfl_sync(0xffffffffu, rel, leader);
        if (c >= 0) {
            const int r = rel + __popc(peers & lt);
            out[start[c] + r] = (uint32_t)i | (r == 0 ? RFXC_PERM_FIRST : 0u);
        }
        __syncwarp();
    }
}

// Single-warp fallback for trees whose histograms do not fit shared memory:
// counters in global scratch (L ints per tree).
__global__ void __launch_bounds__(256)
bucket_global_kernel(const int32_t* __restrict__ codes_tm, int64_t n,
                     const int64_t* __restrict__ leaf_base, int32_t Bl,
                     uint32_t* __restrict__ perm, int64_t* __restrict__ seg,
                     int32_t* __restrict__ scratch, int32_t* __restrict__ has_empty)
{
    __shared__ int32_t warp_sums[8];
    __shared__ int32_t carry;
    const int b = blockIdx.x;
    const int64_t g0 = leaf_base[b];
    const int32_t L = (int32_t)(leaf_base[b + 1] - g0);
    int32_t* cnt = scratch + g0;
    const int32_t* codes = codes_tm + (int64_t)b * n;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    for (int l = tid; l < L; l += 256) cnt[l] = 0;
    __syncthreads();
    for (int64_t i = tid; i < n; i += 256) atomicAdd(&cnt[codes[i]], 1);
    __syncthreads();
    if (tid == 0) carry = 0;
    __syncthreads();
    int empty = 0;
    const int64_t tree_base = (int64_t)b * n;
    for (int base = 0; base < L; base += 256) {
        const int l = base + tid;
        const int v = l < L ? cnt[l] : 0;
        empty |= (l < L && v == 0);
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) warp_sums[warp] = incl;
        __syncthreads();
        int before = carry;
        for (int w = 0; w < warp; w++) before += warp_sums[w];
        if (l < L) {
            cnt[l] = before + incl - v;
            seg[g0 + l] = tree_base + before + incl - v;
        }
        __syncthreads();
        if (tid == 0) {
            int s = 0;
            for (int w = 0; w < 8; w++) s += warp_sums[w];
            carry += s;
        }
        __syncthreads();
    }
    if (__syncthreads_or(empty) && tid == 0) atomicExch(has_empty, 1);
    if (b == Bl - 1 && tid == 0) seg[leaf_base[Bl]] = (int64_t)Bl * n;
    if (warp != 0) return;
    uint32_t* out = perm + tree_base;
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t base = 0; base < n; base += 32) {
        const int64_t i = base + lane;
        const int c = i < n ? __ldg(codes + i) : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, c);
        const int leader = __ffs(peers) - 1;
        int st = 0;
        if (lane == leader && c >= 0) {
            st = cnt[c];
            cnt[c] = st + __popc(peers);
        }
        st = __shfl_sync(0xffffffffu, st, leader);
        if (c >= 0) {
            const int pos = st + __popc(peers & lt);
            const bool first = (int64_t)pos == seg[g0 + c] - tree_base;
            out[pos] = (uint32_t)i | (first ? RFXC_PERM_FIRST : 0u);
        }
        __syncwarp();
    }
}

}  // namespace rfxc

using namespace rfxc;

extern "C" int rfxc_bucket(const int32_t* d_codes_tm, int64_t n, int32_t Bl,
                           const int64_t* d_leaf_base, int32_t max_leaf_count,
                           uint32_t* d_perm, int64_t* d_seg, int32_t* d_scratch,
                           int32_t* d_has_empty, void* stream)
{
    if (n < 1 || Bl < 1 || max_leaf_count < 1) return fail(RFXC_EDATA, "bucket: bad shape");
    if (n >= (int64_t)RFXC_PERM_FIRST) return fail(RFXC_EDATA, "bucket: n exceeds 2^31");
    cudaStream_t st = as_stream(stream);
    cudaError_t e = cudaMemsetAsync(d_has_empty, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return fail(RFXC_ECUDA, "bucket memset: %s", cudaGetErrorString(e));
    const int64_t Lw = (max_leaf_count + 1) / 2;
    // most warps whose 16-bit histograms (+ run starts) fit shared memory;
    // every warp range must stay below 65536 samples
    int W = 16;
    while (W > 1 && (W * Lw + max_leaf_count) * 4 > BUCKET_SMEM_BUDGET) W >>= 1;
    const size_t smem = (size_t)(W * Lw + max_leaf_count) * 4;
    if (smem <= BUCKET_SMEM_BUDGET && ceil_div(n, W) < 65536) {
        if (smem > 48 * 1024) {
            e = cudaFuncSetAttribute(bucket_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem);
            if (e != cudaSuccess) return fail(RFXC_ECUDA, "bucket attr: %s", cudaGetErrorString(e));
        }
        bucket_kernel<<<Bl, 32 * W, smem, st>>>(d_codes_tm, n, d_leaf_base, Bl, d_perm, d_seg,
                                                d_has_empty);
    } else {
        if (!d_scratch) return fail(RFXC_EDATA, "bucket: scratch required for %d leaves",
                                    max_leaf_count);
        bucket_global_kernel<<<Bl, 256, 0, st>>>(d_codes_tm, n, d_leaf_base, Bl, d_perm, d_seg,
                                                 d_scratch, d_has_empty);
    }
    return check_launch("bucket");
}
