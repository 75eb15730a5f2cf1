// bucket.cu — K2: per-tree stable counting sort of samples by leaf.
//
// Reference: the counting sort inside accumulate_pair_counts[_block]
// (_kernels.py:458-468, :491-501), which the reference redoes for every
// tree (and for every (row block, tree) in TriBlock).  Here it runs once per
// tree and the result (perm + per-leaf run starts) is shared by the sketch
// (K4) and the pair kernels.
//
// One CTA per tree: (1) leaf histogram with shared-memory atomics (global
// scratch when the tree has too many leaves for shared memory), (2) block
// exclusive scan -> run starts, (3) stable scatter by a single warp walking
// the samples in order: __match_any_sync groups equal leaves inside each
// 32-sample step, the group leader advances the leaf cursor, and every lane
// writes at cursor + rank-within-group.  Ascending order inside every leaf
// is therefore guaranteed (the reference's bucket order).
#include "common.cuh"

namespace rfxc {

constexpr int BUCKET_THREADS = 256;
constexpr int BUCKET_SMEM_MAX = 48 * 1024;  // counters in smem up to 48K leaves

template <bool SMEM>
__global__ void __launch_bounds__(BUCKET_THREADS)
bucket_kernel(const int32_t* __restrict__ codes_tm, int64_t n,
              const int64_t* __restrict__ leaf_base, int32_t Bl,
              int32_t* __restrict__ perm, int64_t* __restrict__ seg,
              int32_t* __restrict__ scratch)
{
    extern __shared__ int32_t smem_cnt[];
    __shared__ int32_t warp_sums[BUCKET_THREADS / 32];
    __shared__ int32_t carry;
    const int b = blockIdx.x;
    const int64_t g0 = leaf_base[b];
    const int32_t L = (int32_t)(leaf_base[b + 1] - g0);
    int32_t* cnt = SMEM ? smem_cnt : scratch + g0;
    const int32_t* codes = codes_tm + (int64_t)b * n;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    for (int l = tid; l < L; l += BUCKET_THREADS) cnt[l] = 0;
    __syncthreads();
    for (int64_t i = tid; i < n; i += BUCKET_THREADS) atomicAdd(&cnt[codes[i]], 1);
    __syncthreads();

    // exclusive scan of the counters in chunks of BUCKET_THREADS
    if (tid == 0) carry = 0;
    __syncthreads();
    const int64_t tree_base = (int64_t)b * n;
    for (int base = 0; base < L; base += BUCKET_THREADS) {
        int l = base + tid;
        int v = l < L ? cnt[l] : 0;
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) warp_sums[warp] = incl;
        __syncthreads();
        int before = carry;
        for (int w = 0; w < warp; w++) before += warp_sums[w];
        int excl = before + incl - v;
        if (l < L) {
            cnt[l] = excl;
            seg[g0 + l] = tree_base + excl;
        }
        __syncthreads();
        if (tid == 0) {
            int s = 0;
            for (int w = 0; w < BUCKET_THREADS / 32; w++) s += warp_sums[w];
            carry += s;
        }
        __syncthreads();
    }
    if (b == Bl - 1 && tid == 0) seg[leaf_base[Bl]] = (int64_t)Bl * n;

    // stable scatter: one warp, samples in ascending order
    if (warp != 0) return;
    int32_t* out = perm + tree_base;
    const unsigned lt = (1u << lane) - 1u;
    constexpr int U = 4;
    for (int64_t base = 0; base < n; base += 32 * U) {
        int32_t c[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            int64_t i = base + u * 32 + lane;
            c[u] = i < n ? __ldg(codes + i) : -1;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            int64_t i = base + u * 32 + lane;
            unsigned peers = __match_any_sync(0xffffffffu, c[u]);
            int leader = __ffs(peers) - 1;
            int start = 0;
            if (lane == leader && c[u] >= 0) {
                start = cnt[c[u]];
                cnt[c[u]] = start + __popc(peers);
            }
            start = __shfl_sync(0xffffffffu, start, leader);
            if (i < n) out[start + __popc(peers & lt)] = (int32_t)i;
            __syncwarp();
        }
    }
}

}  // namespace rfxc

using namespace rfxc;

extern "C" int rfxc_bucket(const int32_t* d_codes_tm, int64_t n, int32_t Bl,
                           const int64_t* d_leaf_base, int32_t max_leaf_count,
                           int32_t* d_perm, int64_t* d_seg, int32_t* d_scratch, void* stream)
{
    if (n < 1 || Bl < 1 || max_leaf_count < 1) return fail(RFXC_EDATA, "bucket: bad shape");
    if (n > INT32_MAX) return fail(RFXC_EDATA, "bucket: n exceeds int32");
    cudaStream_t st = as_stream(stream);
    if (max_leaf_count <= BUCKET_SMEM_MAX) {
        size_t smem = (size_t)max_leaf_count * 4;
        if (smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(
                bucket_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return fail(RFXC_ECUDA, "bucket attr: %s", cudaGetErrorString(e));
        }
        bucket_kernel<true><<<Bl, BUCKET_THREADS, smem, st>>>(d_codes_tm, n, d_leaf_base, Bl,
                                                              d_perm, d_seg, d_scratch);
    } else {
        if (!d_scratch) return fail(RFXC_EDATA, "bucket: scratch required for %d leaves",
                                    max_leaf_count);
        bucket_kernel<false><<<Bl, BUCKET_THREADS, 0, st>>>(d_codes_tm, n, d_leaf_base, Bl,
                                                            d_perm, d_seg, d_scratch);
    }
    return check_launch("bucket");
}
