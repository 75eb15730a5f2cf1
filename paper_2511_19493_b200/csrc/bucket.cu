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


// ------------------------------------------------------------ radix path
// Stable LSD radix sort of (leaf, sample) pairs per tree, 8-bit digits, one
// CTA per tree.  One read of the codes histograms every digit of every pass
// (digit totals do not depend on the order).  Each pass then streams the tree
// in tiles of RB_TILE elements: the tile is ranked stably by digit in shared
// memory (per-warp counts, __match_any_sync inside a 32-element step, a
// digit-major/warp-minor scan) and written out run by run at the per-digit
// cursors, so the global writes are contiguous runs rather than single 8-byte
// scatters.  The last pass writes the permutation directly, tagging leaf
// starts and recording run starts (empty leaves start where the next one does).
constexpr int RB_W = 16;
constexpr int RB_T = RB_W * 32;
constexpr int RB_U = 8;
constexpr int RB_TILE = RB_T * RB_U;
constexpr int RB_MAXPASS = 4;

struct RbSmem {
    uint2 tile[RB_TILE];
    int cnt[RB_W][256];
    int hist[RB_MAXPASS][256];
    int tstart[256], tcount[256], cursor[256], dbegin[256];
    uint32_t lastk[256];
    int wsum[RB_W];
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

__global__ void __launch_bounds__(RB_T, 2)
radix_bucket_kernel(const int32_t* __restrict__ codes_tm, int64_t n,
                    const int64_t* __restrict__ leaf_base, int32_t tree_lo, int32_t Bl, int npass,
                    uint2* __restrict__ tmp, uint32_t* __restrict__ perm,
                    int64_t* __restrict__ seg, int32_t* __restrict__ has_empty)
{
    extern __shared__ __align__(16) unsigned char rb_raw[];
    RbSmem& S = *reinterpret_cast<RbSmem*>(rb_raw);
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
        for (int t0 = 0; t0 < nn; t0 += RB_TILE) {
            for (int e = tid; e < RB_W * 256; e += RB_T) (&S.cnt[0][0])[e] = 0;
            __syncthreads();
            // rank inside the warp's 32*RB_U elements
            const int wb = t0 + warp * 32 * RB_U;
            uint2 kv[RB_U];
            int rk[RB_U];
#pragma unroll
            for (int u = 0; u < RB_U; u++) {
                const int i = wb + 32 * u + lane;
                kv[u] = make_uint2(0xffffffffu, 0u);
                if (i < nn) kv[u] = pass == 0 ? make_uint2((uint32_t)__ldcs(codes + i), (uint32_t)i) : __ldcs(src + i);
            }
#pragma unroll
            for (int u = 0; u < RB_U; u++) {
                const bool ok = wb + 32 * u + lane < nn;
                const int d = ok ? (int)((kv[u].x >> sh) & 255u) : -1;
                const unsigned peers = __match_any_sync(0xffffffffu, d);
                const int leader = __ffs(peers) - 1;
                int base = 0;
                if (lane == leader && ok) {
                    base = S.cnt[warp][d];
                    S.cnt[warp][d] = base + __popc(peers);
                }
                rk[u] = __shfl_sync(0xffffffffu, base, leader) + __popc(peers & lt);
                __syncwarp();
            }
            __syncthreads();
            int tot = 0;
            if (tid < 256) {
                for (int w = 0; w < RB_W; w++) {
                    const int c = S.cnt[w][tid];
                    S.cnt[w][tid] = tot;
                    tot += c;
                }
            }
            const int ts = rb_scan256(tot, S.wsum);
            if (tid < 256) {
                S.tstart[tid] = ts;
                S.tcount[tid] = tot;
                for (int w = 0; w < RB_W; w++) S.cnt[w][tid] += ts;
            }
            __syncthreads();
#pragma unroll
            for (int u = 0; u < RB_U; u++)
                if (wb + 32 * u + lane < nn) S.tile[S.cnt[warp][(kv[u].x >> sh) & 255u] + rk[u]] = kv[u];
            __syncthreads();
            const int tn = min(RB_TILE, nn - t0);
            for (int j = tid; j < tn; j += RB_T) {
                const uint2 v = S.tile[j];
                const int d = (int)((v.x >> sh) & 255u);
                const int gpos = S.cursor[d] + j - S.tstart[d];
                if (!last) {
                    __stcg(reinterpret_cast<unsigned long long*>(dst + gpos),
                           (unsigned long long)v.x | ((unsigned long long)v.y << 32));
                    continue;
                }
                const bool first_tile = j == S.tstart[d];
                const bool first_all = first_tile && S.cursor[d] == S.dbegin[d];
                const uint32_t prevk = first_tile ? S.lastk[d] : S.tile[j - 1].x;
                const bool first = first_all || prevk != v.x;
                out[gpos] = v.y | (first ? RFXC_PERM_FIRST : 0u);
                if (first) {
                    const uint32_t glo = first_all ? ((uint32_t)d << sh) : prevk + 1u;
                    for (uint32_t c = glo; c <= v.x; c++) seg[g0 + c] = row0 + gpos;
                    empty |= v.x > glo;
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
    const int64_t chunk = std::min<int64_t>(Bl, (int64_t)sm_count() * 2);
    return chunk * 2 * n * 8;
}

extern "C" int rfxc_bucket(const int32_t* d_codes_tm, int64_t n, int32_t Bl,
                           const int64_t* d_leaf_base, int32_t max_leaf_count,
                           uint32_t* d_perm, int64_t* d_seg, void* d_scratch,
                           int32_t* d_has_empty, void* stream)
{
    if (n < 1 || Bl < 1 || max_leaf_count < 1) return fail(RFXC_EDATA, "bucket: bad shape");
    if (n >= (int64_t)RFXC_PERM_FIRST) return fail(RFXC_EDATA, "bucket: n exceeds 2^31");
    if (!d_scratch) return fail(RFXC_EDATA, "bucket: scratch required");
    cudaStream_t st = as_stream(stream);
    cudaError_t e = cudaMemsetAsync(d_has_empty, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return fail(RFXC_ECUDA, "bucket memset: %s", cudaGetErrorString(e));
    int bits = 0;
    while (bits < 31 && ((int64_t)1 << bits) < max_leaf_count) bits++;
    const int npass = std::max(1, (bits + 7) / 8);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(radix_bucket_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(RbSmem));
        attr = true;
    }
    const int64_t chunk = std::min<int64_t>(Bl, (int64_t)sm_count() * 2);
    for (int64_t t0 = 0; t0 < Bl; t0 += chunk) {
        const int nb = (int)std::min<int64_t>(chunk, Bl - t0);
        radix_bucket_kernel<<<nb, RB_T, sizeof(RbSmem), st>>>(d_codes_tm, n, d_leaf_base, (int)t0, Bl, npass,
                                                 static_cast<uint2*>(d_scratch), d_perm, d_seg,
                                                 d_has_empty);
        const int rc = check_launch("bucket");
        if (rc) return rc;
    }
    return RFXC_OK;
}
