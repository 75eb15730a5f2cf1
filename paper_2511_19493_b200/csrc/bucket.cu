// bucket.cu — K2: per-tree stable counting sort of samples by leaf.
//
// Reference: the counting sort inside accumulate_pair_counts[_block]
// (_kernels.py:458-468, :491-501), which the reference redoes for every
// tree (and for every (row block, tree) in TriBlock).  Here it runs once per
// tree and the result (perm + per-leaf run starts) is shared by the sketch
// (K4) and the pair kernels.
//
// Stable LSD radix sort of (leaf, sample) pairs, 8-bit digits, one CTA per
// tree (details at radix_bucket_kernel).  Shared memory does not grow with
// the leaf count, so every tree size takes the same path.  The first member
// of every leaf carries bit 31 (RFXC_PERM_FIRST) so the sketch can find leaf
// boundaries from perm alone; an empty leaf sets *has_empty.
#include "common.cuh"

namespace rfxc {

// One read of the codes histograms every digit of every pass (digit totals
// do not depend on the order).  Each pass then streams the tree in tiles of
// W*32*U elements: the tile is ranked stably by digit in shared memory
// (equal-digit lanes of a 32-element step found by ANDing 8 bit-plane
// ballots, per-warp counts, a digit-major/warp-minor scan) and written out
// run by run at the per-digit cursors, so global writes are contiguous runs
// rather than single 8-byte scatters.  The last pass writes the permutation
// directly, tagging leaf starts and recording run starts (an empty leaf
// starts where the next one does).  Pass p>0 reads what pass p-1 wrote to
// the per-CTA scratch pair.
constexpr int RB_MAXPASS = 4;
#ifndef RFXC_RB_W
#define RFXC_RB_W 16
#endif
#ifndef RFXC_RB_MINB
#define RFXC_RB_MINB 2
#endif
constexpr int RB_W = RFXC_RB_W;  // warps per CTA
constexpr int RB_MINB = RFXC_RB_MINB;  // resident CTAs per SM
static_assert(RB_W >= 8, "the 256-digit scans need at least 256 threads");
#ifndef RFXC_RB_U
#define RFXC_RB_U 8
#endif
constexpr int RB_U = RFXC_RB_U;  // 32-element steps per warp per tile

template <int W, int U>
struct RbSmem {
    uint2 tile[W * 32 * U];
    int cnt[W][256];
    int hist[RB_MAXPASS][256];
    int tstart[256], tcount[256], cursor[256], dbegin[256], delta[256];
    uint32_t lastk[256];
    int wsum[W];
};

// exclusive scan of v over the 256 threads tid < 256 (8 warps); returns the
// exclusive prefix, all RB_T threads must call it
__device__ __forceinline__ int rb_scan256(int v, int* wsum)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (threadIdx.x < 256 && lane == 31) wsum[warp] = incl;
    __syncthreads();
    int before = 0;
    if (threadIdx.x < 256)
        for (int w = 0; w < warp; w++) before += wsum[w];
    __syncthreads();
    return before + incl - v;
}

template <int W, int U, int MINB>
__global__ void __launch_bounds__(W * 32, MINB)
radix_bucket_kernel(const int32_t* __restrict__ codes_tm, int64_t n,
                    const int64_t* __restrict__ leaf_base, int32_t tree_lo, int32_t Bl, int npass,
                    uint2* __restrict__ tmp, uint32_t* __restrict__ perm,
                    int64_t* __restrict__ seg, int32_t* __restrict__ has_empty)
{
    constexpr int RB_T = W * 32;
    constexpr int TILE = RB_T * U;
    extern __shared__ __align__(16) unsigned char rb_raw[];
    RbSmem<W, U>& S = *reinterpret_cast<RbSmem<W, U>*>(rb_raw);
    const int b = tree_lo + blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
    const int nn = (int)n;
    const int32_t* codes = codes_tm + (int64_t)b * n;
    uint2* const T0 = tmp + (int64_t)blockIdx.x * 2 * n;
    uint32_t* out = perm + (int64_t)b * n;
    const int64_t g0 = leaf_base[b];
    const int64_t L = leaf_base[b + 1] - g0;
    const int64_t row0 = (int64_t)b * n;
    const unsigned lt = (1u << lane) - 1u;

    for (int e = tid; e < RB_MAXPASS * 256; e += RB_T) (&S.hist[0][0])[e] = 0;
    __syncthreads();
    for (int i0 = tid; i0 < nn; i0 += RB_T * 4) {
        uint32_t key[4];
#pragma unroll
        for (int u = 0; u < 4; u++) key[u] = i0 + u * RB_T < nn ? (uint32_t)__ldg(codes + i0 + u * RB_T) : 0u;
#pragma unroll
        for (int u = 0; u < 4; u++)
            if (i0 + u * RB_T < nn)
                for (int p = 0; p < npass; p++) atomicAdd(&S.hist[p][(key[u] >> (8 * p)) & 255u], 1);
    }
    __syncthreads();

    int empty = 0;
    for (int pass = 0; pass < npass; pass++) {
        const int sh = 8 * pass;
        const bool last = pass == npass - 1;
        const uint2* src = pass == 0 ? nullptr : T0 + ((pass - 1) & 1) * n;
        uint2* dst = T0 + (pass & 1) * n;
        {
            const int v = tid < 256 ? S.hist[pass][tid] : 0;
            const int ex = rb_scan256(v, S.wsum);
            if (tid < 256) {
                S.cursor[tid] = ex;
                S.dbegin[tid] = ex;
                S.lastk[tid] = 0xffffffffu;
            }
        }
        for (int t0 = 0; t0 < nn; t0 += TILE) {
            for (int e = tid; e < W * 256; e += RB_T) (&S.cnt[0][0])[e] = 0;
            __syncthreads();
            // rank inside the warp's 32*U elements (stable: steps in order,
            // lanes in order inside a step)
            const int wb = t0 + warp * 32 * U;
            uint2 kv[U];
            int rk[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int i = wb + 32 * u + lane;
                kv[u] = make_uint2(0xffffffffu, 0u);
                if (i < nn) kv[u] = pass == 0 ? make_uint2((uint32_t)__ldcs(codes + i), (uint32_t)i) : __ldcs(src + i);
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                // lanes holding the same digit: AND of 8 bit-plane ballots
                const unsigned valid = __ballot_sync(0xffffffffu, wb + 32 * u + lane < nn);
                const unsigned d = (kv[u].x >> sh) & 255u;
                unsigned peers = valid;
#pragma unroll
                for (int bit = 0; bit < 8; bit++) {
                    const unsigned m = __ballot_sync(0xffffffffu, (d >> bit) & 1u);
                    peers &= ((d >> bit) & 1u) ? m : ~m;
                }
                const bool ok = (valid >> lane) & 1u;
                const int base = ok ? S.cnt[warp][d] : 0;
                const int r = __popc(peers & lt);
                __syncwarp();
                if (ok && (peers >> lane) == 1u) S.cnt[warp][d] = base + r + 1;  // last of its group
                __syncwarp();
                rk[u] = base + r;
            }
            __syncthreads();
            int tot = 0;
            if (tid < 256) {
                for (int w = 0; w < W; w++) {
                    const int c = S.cnt[w][tid];
                    S.cnt[w][tid] = tot;
                    tot += c;
                }
            }
            const int ts = rb_scan256(tot, S.wsum);
            if (tid < 256) {
                S.tstart[tid] = ts;
                S.tcount[tid] = tot;
                S.delta[tid] = S.cursor[tid] - ts;
                for (int w = 0; w < W; w++) S.cnt[w][tid] += ts;
            }
            __syncthreads();
#pragma unroll
            for (int u = 0; u < U; u++)
                if (wb + 32 * u + lane < nn) S.tile[S.cnt[warp][(kv[u].x >> sh) & 255u] + rk[u]] = kv[u];
            __syncthreads();
            const int tn = min(TILE, nn - t0);
            if (!last) {
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int j = tid + u * RB_T;
                    if (j < tn) {
                        const uint2 v = S.tile[j];
                        const int gpos = j + S.delta[(v.x >> sh) & 255u];
                        __stcg(reinterpret_cast<unsigned long long*>(dst + gpos),
                               (unsigned long long)v.x | ((unsigned long long)v.y << 32));
                    }
                }
            } else {
                for (int j = tid; j < tn; j += RB_T) {
                    const uint2 v = S.tile[j];
                    const int d = (int)((v.x >> sh) & 255u);
                    const int gpos = j + S.delta[d];
                    const bool first_tile = j == S.tstart[d];
                    const bool first_all = first_tile && gpos == S.dbegin[d];
                    const uint32_t prevk = first_tile ? S.lastk[d] : S.tile[j - 1].x;
                    const bool first = first_all || prevk != v.x;
                    out[gpos] = v.y | (first ? RFXC_PERM_FIRST : 0u);
                    if (first) {
                        const uint32_t glo = first_all ? ((uint32_t)d << sh) : prevk + 1u;
                        for (uint32_t c = glo; c <= v.x; c++) seg[g0 + c] = row0 + gpos;
                        empty |= v.x > glo;
                    }
                }
            }
            __syncthreads();
            if (tid < 256) {
                const int c = S.tcount[tid];
                if (c > 0) {
                    S.lastk[tid] = S.tile[S.tstart[tid] + c - 1].x;
                    S.cursor[tid] += c;
                }
            }
            __syncthreads();
        }
    }
    // empty leaves after the last member of every top digit
    if (tid < 256) {
        const int sh = 8 * (npass - 1);
        const int d = tid;
        const int c = S.hist[npass - 1][d];
        const int64_t klo = c > 0 ? (int64_t)S.lastk[d] + 1 : ((int64_t)d << sh);
        const int64_t khi = min(((int64_t)d + 1) << sh, L);
        for (int64_t k = klo; k < khi; k++) seg[g0 + k] = row0 + S.dbegin[d] + c;
        empty |= khi > klo;
    }
    if (__syncthreads_or(empty) && tid == 0) atomicExch(has_empty, 1);
    if (b == Bl - 1 && tid == 0) seg[leaf_base[Bl]] = (int64_t)Bl * n;
}

}  // namespace rfxc

using namespace rfxc;

extern "C" int64_t rfxc_bucket_scratch_bytes(int64_t n, int32_t Bl)
{
    const int64_t chunk = std::min<int64_t>(Bl, (int64_t)sm_count() * RB_MINB);
    return chunk * 2 * n * 8;
}

extern "C" int rfxc_bucket_trees(const int32_t* d_codes_tm, int64_t n, int32_t Bl,
                                 const int64_t* d_leaf_base, int32_t max_leaf_count,
                                 int32_t tree_lo, int32_t tree_hi, uint32_t* d_perm, int64_t* d_seg,
                                 void* d_scratch, int32_t* d_has_empty, void* stream)
{
    if (n < 1 || Bl < 1 || max_leaf_count < 1) return fail(RFXC_EDATA, "bucket: bad shape");
    if (tree_lo < 0 || tree_hi > Bl || tree_lo > tree_hi) return fail(RFXC_EDATA, "bucket: bad tree range");
    if (n >= (int64_t)RFXC_PERM_FIRST) return fail(RFXC_EDATA, "bucket: n exceeds 2^31");
    if (!d_scratch) return fail(RFXC_EDATA, "bucket: scratch required");
    cudaStream_t st = as_stream(stream);
    int bits = 0;
    while (bits < 31 && ((int64_t)1 << bits) < max_leaf_count) bits++;
    const int npass = std::max(1, (bits + 7) / 8);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(radix_bucket_kernel<RB_W, RB_U, RB_MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(RbSmem<RB_W, RB_U>));
        attr = true;
    }
    const int64_t chunk = std::min<int64_t>(Bl, (int64_t)sm_count() * RB_MINB);
    uint2* tmp = static_cast<uint2*>(d_scratch);
    for (int64_t t0 = tree_lo; t0 < tree_hi; t0 += chunk) {
        const int nb = (int)std::min<int64_t>(chunk, tree_hi - t0);
        radix_bucket_kernel<RB_W, RB_U, RB_MINB><<<nb, RB_W * 32, sizeof(RbSmem<RB_W, RB_U>), st>>>(
            d_codes_tm, n, d_leaf_base, (int)t0, Bl, npass, tmp, d_perm, d_seg, d_has_empty);
        const int rc = check_launch("bucket");
        if (rc) return rc;
    }
    return RFXC_OK;
}

extern "C" int rfxc_bucket(const int32_t* d_codes_tm, int64_t n, int32_t Bl,
                           const int64_t* d_leaf_base, int32_t max_leaf_count,
                           uint32_t* d_perm, int64_t* d_seg, void* d_scratch,
                           int32_t* d_has_empty, void* stream)
{
    if (n < 1 || Bl < 1 || max_leaf_count < 1) return fail(RFXC_EDATA, "bucket: bad shape");
    cudaError_t e = cudaMemsetAsync(d_has_empty, 0, sizeof(int32_t), as_stream(stream));
    if (e != cudaSuccess) return fail(RFXC_ECUDA, "bucket memset: %s", cudaGetErrorString(e));
    return rfxc_bucket_trees(d_codes_tm, n, Bl, d_leaf_base, max_leaf_count, 0, Bl, d_perm, d_seg,
                             d_scratch, d_has_empty, stream);
}
