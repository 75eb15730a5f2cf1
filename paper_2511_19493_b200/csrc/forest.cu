// forest.cu — K0 (forest flattening) and K1 (forest traversal to leaf codes).
//
// Reference: descend / descend_all (_kernels.py:333-374) driven per tree by
// leaf_membership (proximity.py:100-116), leaf ordinals from
// Tree.leaf_codes (forest.py:95-99).
//
// Design (B200): a CTA owns a tile of T samples and walks them down a chunk
// of trees.  The tile's feature rows are staged once into shared memory with
// coalesced column loads (Dataset.values is column-major), so every
// per-level feature read is a shared-memory access; node records (8 B in the
// f32 layout) are read through the read-only L1 path, where the upper levels
// of the tree currently being walked by every warp of the SM stay resident.
// Each thread advances ILP independent root-to-leaf chains (one per tree) so
// dependent node loads overlap.  Codes are written tree-major, coalesced.
//
// Exactness of the f32 layout: thresholds are rounded toward -inf to f32.
// For any f32-representable x, x <= t (f64)  <=>  x <= RD_f32(t), so the
// comparison is bit-exact with the reference whenever every value is
// f32-exact (checked by rfxc_values_to_f32; otherwise the f64 layout runs).
#include "common.cuh"

#include <cstdlib>

namespace rfxc {

// ---------------------------------------------------------------- K0 pack
__global__ void values_to_f32_kernel(const double* __restrict__ in, int64_t count,
                                     float* __restrict__ out, int32_t* inexact)
{
    int bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        double x = in[i];
        float f = (float)x;
        out[i] = f;
        bad |= ((double)f != x);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(inexact, 1);
}

__host__ __device__ inline int feature_bits(int p)
{
    int fb = 1;
    while ((1 << fb) < p) fb++;
    return fb;
}

// One CTA per tree: block-wide exclusive scan of the terminal flags gives the
// dense leaf ordinal of every terminal (forest.py:95-99).
template <int LAYOUT>
__global__ void pack_kernel(const int8_t* __restrict__ status,
                            const int32_t* __restrict__ split_var,
                            const double* __restrict__ threshold,
                            const int64_t* __restrict__ cat_mask,
                            const int32_t* __restrict__ left,
                            const int32_t* __restrict__ leaf_code,
                            const int64_t* __restrict__ node_off,
                            const uint8_t* __restrict__ col_cat, int fb,
                            void* nodes_out, int32_t* leaf_counts)
{
    __shared__ int warp_tot[32];
    __shared__ int carry;
    const int b = blockIdx.x;
    const int64_t o = node_off[b], nc = node_off[b + 1] - o;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < nc; base += blockDim.x) {
        int64_t t = base + threadIdx.x;
        int is_leaf = (t < nc) ? (status[o + t] == 1) : 0;
        unsigned ball = __ballot_sync(0xffffffffu, is_leaf);
        int within = __popc(ball & ((1u << lane) - 1u));
        if (lane == 0) warp_tot[warp] = __popc(ball);
        __syncthreads();
        int before = carry;
        for (int w = 0; w < warp; w++) before += warp_tot[w];
        if (t < nc) {
            int64_t g = o + t;
            if (LAYOUT == RFXC_NODES_F32) {
                uint2 rec;
                if (is_leaf) {
                    rec.x = (uint32_t)(leaf_code ? leaf_code[g] : before + within);
                    rec.y = 0u;
                } else {
                    int f = split_var[g];
                    uint32_t cat = col_cat[f] == 1;
                    rec.x = cat ? (uint32_t)(cat_mask[g] & 0xffffffffLL)
                                : __float_as_uint(__double2float_rd(threshold[g]));
                    rec.y = ((uint32_t)left[g] << (fb + 1)) | (cat << fb) | (uint32_t)f;
                }
                reinterpret_cast<uint2*>(nodes_out)[g] = rec;
            } else {
                int4 rec;
                if (is_leaf) {
                    rec = make_int4(0, 0, -1, leaf_code ? leaf_code[g] : before + within);
                } else {
                    int f = split_var[g];
                    int cat = col_cat[f] == 1;
                    long long bits = cat ? (long long)cat_mask[g]
                                         : __double_as_longlong(threshold[g]);
                    rec = make_int4((int)(bits & 0xffffffffLL), (int)(bits >> 32),
                                    f | (cat << 30), left[g]);
                }
                reinterpret_cast<int4*>(nodes_out)[g] = rec;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int s = 0;
            for (int w = 0; w < nw; w++) s += warp_tot[w];
            carry += s;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) leaf_counts[b] = carry;
}

// ------------------------------------------------------------ K1 traverse
#ifndef RFXC_TRAV_G
#define RFXC_TRAV_G 8
#endif
#ifndef RFXC_TRAV_ILP
#define RFXC_TRAV_ILP 1
#endif
#ifndef RFXC_TRAV_T
#define RFXC_TRAV_T 128
#endif
constexpr int TRAV_T = RFXC_TRAV_T;     // samples per CTA (one X row each in shared memory)
constexpr int TRAV_G = RFXC_TRAV_G;     // tree groups per CTA: TRAV_T * TRAV_G threads share the tile
constexpr int TRAV_ILP = RFXC_TRAV_ILP; // independent tree chains per thread

// TOP > 0 (f32 node layout): the top TOP node records (node ids < TOP — the
// trainer numbers nodes breadth-first, so ids < 2^d - 1 cover the first d
// levels) of the TRAV_G * TRAV_ILP trees a CTA walks per round are staged in
// shared memory before the round, so every walk's first levels (where all
// samples of the tile meet) are shared-memory reads; deeper levels go
// through the read-only path.  Rounds are CTA-synchronous.
template <int LAYOUT, bool SMEM_X, int TOP, bool NUMERIC = false>
__global__ void __launch_bounds__(TRAV_T * TRAV_G, 2048 / (TRAV_T * TRAV_G))
traverse_kernel(const void* __restrict__ nodes_v, const int64_t* __restrict__ node_off,
                int fb, int p, int tree_lo, int tree_hi, int trees_per_chunk,
                const void* __restrict__ values_v, int64_t n, int64_t row_lo, int64_t row_hi,
                int32_t* __restrict__ codes_tm)
{
    using V = typename std::conditional<LAYOUT == RFXC_NODES_F64, double, float>::type;
    constexpr bool B2 = LAYOUT == RFXC_NODES_F32_B2;
    static_assert(TOP == 0 || LAYOUT == RFXC_NODES_F32, "tree tops: f32 layout only");
    constexpr int RT = TRAV_G * TRAV_ILP;  // trees per round
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V* xs = reinterpret_cast<V*>(smem_raw);
    const V* __restrict__ X = reinterpret_cast<const V*>(values_v);
    const int t = threadIdx.x % TRAV_T;   // sample within the tile
    const int grp = threadIdx.x / TRAV_T; // tree group
    const int64_t i0 = row_lo + (int64_t)blockIdx.x * TRAV_T;
    const int64_t i = i0 + t;
    const bool valid = i < row_hi;
    const int stride = p + 1;  // odd row stride spreads banks
    uint2* tops = reinterpret_cast<uint2*>(
        smem_raw + (SMEM_X ? ((size_t)TRAV_T * stride * sizeof(V) + 15) / 16 * 16 : 0));
    if (SMEM_X) {
        // coalesced: consecutive threads read consecutive samples of feature f
        for (int f = grp; f < p; f += TRAV_G) {
            V v = valid ? X[(int64_t)f * n + i] : V(0);
            xs[t * stride + f] = v;
        }
        __syncthreads();
    }
    const int b_begin = tree_lo + blockIdx.y * trees_per_chunk;
    const int b_end = min(tree_hi, b_begin + trees_per_chunk);
    if (TOP == 0 && !valid) return;
    const V* xrow = xs + t * stride;  // this sample's staged row
    // its 32-bit shared-window address, so a visit's x is one LEA + LDS
    const uint32_t xaddr = (uint32_t)__cvta_generic_to_shared(xrow);
    const uint32_t fmask = (1u << fb) - 1u;

    // round j: trees b_begin + j*RT + [0, RT); group g takes its ILP
    // consecutive trees of the round
    for (int b0 = b_begin; b0 < b_end; b0 += RT) {
        if (TOP > 0) {
            __syncthreads();  // the previous round's walks are done with the tops
            const uint2* nodes = reinterpret_cast<const uint2*>(nodes_v);
            for (int e = threadIdx.x; e < RT * TOP; e += TRAV_T * TRAV_G) {
                const int slot = e / TOP, id = e % TOP;
                const int tb = b0 + slot;
                if (tb < b_end) {
                    const int64_t o = node_off[tb];
                    if (o + id < node_off[tb + 1]) tops[e] = __ldg(nodes + o + id);
                }
            }
            __syncthreads();
            if (!valid) continue;
        }
        const int b = b0 + grp * TRAV_ILP;
        int64_t base[TRAV_ILP];
        const uint2* nptr[TRAV_ILP];  // f32 layout: the chain's tree, so a visit is one IMAD.WIDE
        uint32_t id[TRAV_ILP];
        uint2 xr[TRAV_ILP];  // B2: record of the chain's current block root
        int32_t code[TRAV_ILP];
        uint32_t actm = 0;  // bit c: chain c still walking
#pragma unroll
        for (int c = 0; c < TRAV_ILP; c++) {
            const bool live = (b + c) < b_end;
            if (live) actm |= 1u << c;
            base[c] = live ? node_off[b + c] : 0;
            // opaque to the optimiser, so a visit is one IMAD.WIDE off the
            // chain's tree instead of a 64-bit (base + id) rebuilt each time
            const uint2* np = reinterpret_cast<const uint2*>(nodes_v) + base[c];
            asm("mov.b64 %0, %1;" : "=l"(nptr[c]) : "l"(np));
            id[c] = 0;
            code[c] = 0;
            if (B2) xr[c] = live ? __ldg(np) : make_uint2(0u, 0u);
        }
        while (actm) {
#pragma unroll
            for (int c = 0; c < TRAV_ILP; c++) {
                if (!(actm & (1u << c))) continue;
                if (B2) {
                    // two levels per dependent load: decide at block root x,
                    // then one 256-bit load brings the chosen child's record
                    // and that child's children pair; decide at the child
                    const uint2 nd = xr[c];
                    if (nd.y == 0u) {
                        code[c] = (int32_t)nd.x;
                        actm &= ~(1u << c);
                        continue;
                    }
                    auto decide = [&](const uint32_t rx, const uint32_t ry) {
                        const uint32_t f = ry & fmask;
                        float v;
                        if (SMEM_X)
                            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(xaddr + 4u * f));
                        else
                            v = (float)X[(int64_t)f * n + i];
                        if (!NUMERIC && ((ry >> fb) & 1u)) {
                            const uint32_t lv = (uint32_t)(int)v;
                            return lv < 32u ? (bool)((rx >> lv) & 1u) : false;
                        }
                        return v <= __uint_as_float(rx);
                    };
                    const bool go = decide(nd.x, nd.y);
                    const bool rint = (nd.y >> (fb + 1)) & 1u;
                    const uint32_t g = (nd.y >> (fb + 2)) + ((!go && rint) ? 4u : 0u);
                    uint32_t a[8];
                    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                 : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]),
                                   "=r"(a[6]), "=r"(a[7])
                                 : "l"(nptr[c] + g));
                    const bool first = go || rint;  // group1 starts with R's copy
                    const uint32_t yx = first ? a[0] : a[2], yy = first ? a[1] : a[3];
                    if (yy == 0u) {
                        code[c] = (int32_t)yx;
                        actm &= ~(1u << c);
                        continue;
                    }
                    xr[c] = decide(yx, yy) ? make_uint2(a[4], a[5]) : make_uint2(a[6], a[7]);
                } else if (LAYOUT == RFXC_NODES_F32) {
                    const uint2 nd = (TOP > 0 && id[c] < (uint32_t)TOP)
                                         ? tops[(grp * TRAV_ILP + c) * TOP + id[c]]
                                         : __ldg(nptr[c] + id[c]);
                    if (nd.y == 0u) {
                        code[c] = (int32_t)nd.x;
                        actm &= ~(1u << c);
                        continue;
                    }
                    const uint32_t f = nd.y & fmask;
                    float v;
                    if (SMEM_X)
                        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(xaddr + 4u * f));
                    else
                        v = (float)X[(int64_t)f * n + i];
                    bool go;
                    if (!NUMERIC && ((nd.y >> fb) & 1u)) {
                        uint32_t lv = (uint32_t)(int)v;
                        go = lv < 32u ? ((nd.x >> lv) & 1u) : false;
                    } else {
                        go = v <= __uint_as_float(nd.x);
                    }
                    id[c] = (nd.y >> (fb + 1)) + (go ? 0u : 1u);
                } else {
                    int4 nd = __ldg(reinterpret_cast<const int4*>(nodes_v) + base[c] + id[c]);
                    if (nd.z < 0) {
                        code[c] = nd.w;
                        actm &= ~(1u << c);
                        continue;
                    }
                    const int f = nd.z & 0x3fffffff;
                    const double v = SMEM_X ? (double)xrow[f] : (double)X[(int64_t)f * n + i];
                    long long bits = ((long long)(unsigned)nd.y << 32) | (unsigned)nd.x;
                    bool go;
                    if (nd.z & (1 << 30)) {
                        long long lv = (long long)v;
                        go = (lv >= 0 && lv < 64) ? ((bits >> lv) & 1LL) : false;
                    } else {
                        go = v <= __longlong_as_double(bits);
                    }
                    id[c] = (uint32_t)nd.w + (go ? 0u : 1u);
                }
            }
        }
#pragma unroll
        for (int c = 0; c < TRAV_ILP; c++)
            if ((b + c) < b_end) codes_tm[(int64_t)(b + c - tree_lo) * n + i] = code[c];
    }
}

#ifndef TRP_TPB
#define TRP_TPB 4
#endif
// out[map(c) * ld_out + r] = in[r * ld_in + c] for r < rows, c < cols
// (map = identity when col_map is null): 32 x 32 tiles through shared memory
__global__ void transpose_i32_kernel(const int32_t* __restrict__ in, int64_t rows,
                                     int64_t cols, int64_t ld_in, int32_t* __restrict__ out,
                                     int64_t ld_out, const int32_t* __restrict__ col_map)
{
    __shared__ int32_t tile[TRP_TPB][32][33];
    const int64_t c0 = (int64_t)blockIdx.x * 32;
    // TRP_TPB 32 x 32 tiles stacked along the rows per block, so every output
    // row gets a 32 * TRP_TPB * 4-byte contiguous segment
#pragma unroll
    for (int q = 0; q < TRP_TPB; q++) {
        const int64_t r0 = ((int64_t)blockIdx.y * TRP_TPB + q) * 32;
        for (int k = threadIdx.y; k < 32; k += blockDim.y) {
            int64_t r = r0 + k, c = c0 + threadIdx.x;
            if (r < rows && c < cols) tile[q][k][threadIdx.x] = in[r * ld_in + c];
        }
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t c = c0 + k;
        if (c >= cols) continue;
        const int64_t oc = col_map ? (int64_t)__ldg(col_map + c) : c;
#pragma unroll
        for (int q = 0; q < TRP_TPB; q++) {
            const int64_t r = ((int64_t)blockIdx.y * TRP_TPB + q) * 32 + threadIdx.x;
            if (r < rows) out[oc * ld_out + r] = tile[q][threadIdx.x][k];
        }
    }
}

// Sample order for the traversal: samples grouped by their leaf in one tree
// (counts, exclusive scan, scatter).  The slot of a sample inside its leaf's
// group comes from an atomic and is not reproducible — only which samples
// share a traversal tile depends on it, never a leaf code.
__global__ void leaf_hist_kernel(const int32_t* __restrict__ codes, int64_t n, int32_t* __restrict__ cnt)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(cnt + __ldg(codes + i), 1);
}

__global__ void __launch_bounds__(1024) leaf_scan_kernel(int32_t* __restrict__ cnt, int nleaf)
{
    __shared__ int32_t wsum[32];
    __shared__ int32_t carry;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nleaf; base += 1024) {
        const int i = base + (int)threadIdx.x;
        const int v = i < nleaf ? cnt[i] : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        int before = carry;
        for (int w = 0; w < warp; w++) before += wsum[w];
        if (i < nleaf) cnt[i] = before + x - v;  // exclusive
        __syncthreads();
        if (threadIdx.x == 1023) carry = before + x;
        __syncthreads();
    }
}

__global__ void leaf_scatter_kernel(const int32_t* __restrict__ codes, int64_t n, int32_t* __restrict__ cur,
                                    int32_t* __restrict__ order)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        order[atomicAdd(cur + __ldg(codes + i), 1)] = (int32_t)i;
}

// Xp[f * n + j] = X[f * n + order[j]] (column-major (n, p) f32 values)
__global__ void permute_rows_f32_kernel(const float* __restrict__ X, int64_t n, int p,
                                        const int32_t* __restrict__ order, float* __restrict__ Xp)
{
    const int64_t total = n * p;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = q / n, j = q - f * n;
        Xp[q] = __ldg(X + f * n + __ldg(order + j));
    }
}

}  // namespace rfxc

using namespace rfxc;

extern "C" int rfxc_values_to_f32(const double* d_values, int64_t count, float* d_out,
                                  int32_t* d_inexact, void* stream)
{
    if (count < 0) return fail(RFXC_EDATA, "values_to_f32: negative count");
    if (count == 0) return RFXC_OK;
    int grid = (int)std::min<int64_t>(ceil_div(count, 256), (int64_t)sm_count() * 8);
    values_to_f32_kernel<<<grid, 256, 0, as_stream(stream)>>>(d_values, count, d_out, d_inexact);
    return check_launch("values_to_f32");
}

extern "C" int rfxc_forest_pack(const int8_t* d_status, const int32_t* d_split_var,
                                const double* d_threshold, const int64_t* d_cat_mask,
                                const int32_t* d_left, const int32_t* d_leaf_code,
                                const int64_t* d_node_off, int32_t B,
                                int64_t total_nodes, const uint8_t* d_col_cat, int32_t p,
                                int32_t layout, void* d_nodes, int32_t* d_leaf_counts,
                                void* stream)
{
    if (B < 1 || p < 1 || total_nodes < B) return fail(RFXC_EDATA, "forest_pack: bad shape");
    const int fb = feature_bits(p);
    if (layout == RFXC_NODES_F32) {
        pack_kernel<RFXC_NODES_F32><<<B, 256, 0, as_stream(stream)>>>(
            d_status, d_split_var, d_threshold, d_cat_mask, d_left, d_leaf_code, d_node_off, d_col_cat, fb,
            d_nodes, d_leaf_counts);
    } else if (layout == RFXC_NODES_F64) {
        pack_kernel<RFXC_NODES_F64><<<B, 256, 0, as_stream(stream)>>>(
            d_status, d_split_var, d_threshold, d_cat_mask, d_left, d_leaf_code, d_node_off, d_col_cat, fb,
            d_nodes, d_leaf_counts);
    } else {
        return fail(RFXC_EDATA, "forest_pack: unknown layout %d", layout);
    }
    return check_launch("forest_pack");
}

template <int LAYOUT, bool SMEM_X, int TOP, bool NUMERIC = false>
static int launch_traverse(const void* d_nodes, const int64_t* d_node_off, int p, int tree_lo,
                           int tree_hi, const void* d_values, int64_t n, int64_t row_lo,
                           int64_t row_hi, int32_t* d_codes_tm, size_t smem, cudaStream_t st)
{
    auto kern = traverse_kernel<LAYOUT, SMEM_X, TOP, NUMERIC>;
    if (TOP > 0) smem = (smem + 15) / 16 * 16 + (size_t)TRAV_G * TRAV_ILP * TOP * 8;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return fail(RFXC_ECUDA, "traverse attr: %s", cudaGetErrorString(e));
    }
    int occ = 1;
    const int threads = TRAV_T * TRAV_G;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
    occ = std::max(occ, 1);
    const int64_t tiles = ceil_div(row_hi - row_lo, TRAV_T);
    const int nt = tree_hi - tree_lo;
    // enough CTAs for ~6 waves; every chunk a multiple of the trees one CTA
    // walks per step (TRAV_G groups x TRAV_ILP chains)
    const int step = TRAV_G * TRAV_ILP;
    int64_t want = (int64_t)sm_count() * occ * 6;
    int chunks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(want, tiles),
                                                             ceil_div(nt, step)));
    int per = (int)ceil_div(nt, chunks);
    per = (int)ceil_div(per, step) * step;
    chunks = (int)ceil_div(nt, per);
    dim3 grid((unsigned)tiles, (unsigned)chunks);
    kern<<<grid, threads, smem, st>>>(d_nodes, d_node_off, feature_bits(p), p, tree_lo, tree_hi,
                                      per, d_values, n, row_lo, row_hi, d_codes_tm);
    return check_launch("leaf_codes");
}

// Tree-top staging (RFXC_TRAV_TOP = node records per tree in shared memory,
// 0 = off): see traverse_kernel.  Off by default — measured slower on B200
// (DESIGN.md §7): the tree tops are L1-resident already.
static int trav_top()
{
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("RFXC_TRAV_TOP");
        v = e ? atoi(e) : 0;
        v = v >= 255 ? 255 : v >= 127 ? 127 : v >= 63 ? 63 : 0;
    }
    return v;
}

extern "C" int rfxc_leaf_codes_rows(const void* d_nodes, const int64_t* d_node_off,
                                    int32_t layout, int32_t p, int32_t tree_lo, int32_t tree_hi,
                                    const void* d_values, int64_t n, int64_t row_lo,
                                    int64_t row_hi, int32_t* d_codes_tm, void* stream)
{
    if (n < 1 || p < 1 || tree_lo < 0 || tree_hi <= tree_lo)
        return fail(RFXC_EDATA, "leaf_codes: bad shape");
    if (row_lo < 0 || row_hi > n || row_lo >= row_hi) return fail(RFXC_EDATA, "leaf_codes: bad rows");
    cudaStream_t st = as_stream(stream);
    const size_t vsz = layout == RFXC_NODES_F64 ? 8 : 4;
    const size_t smem = (size_t)TRAV_T * (p + 1) * vsz;
    const bool use_smem = smem <= 112 * 1024;
#define RFXC_TRAV(L, S, TOP) \
    launch_traverse<L, S, TOP>(d_nodes, d_node_off, p, tree_lo, tree_hi, d_values, n, row_lo, \
                               row_hi, d_codes_tm, S ? smem : 0, st)
    if (layout == RFXC_NODES_F32_B2_NUMERIC)
        return use_smem ? launch_traverse<RFXC_NODES_F32_B2, true, 0, true>(
                              d_nodes, d_node_off, p, tree_lo, tree_hi, d_values, n, row_lo, row_hi,
                              d_codes_tm, smem, st)
                        : launch_traverse<RFXC_NODES_F32_B2, false, 0, true>(
                              d_nodes, d_node_off, p, tree_lo, tree_hi, d_values, n, row_lo, row_hi,
                              d_codes_tm, 0, st);
    if (layout == RFXC_NODES_F32_B2)
        return use_smem ? RFXC_TRAV(RFXC_NODES_F32_B2, true, 0) : RFXC_TRAV(RFXC_NODES_F32_B2, false, 0);
    if (layout == RFXC_NODES_F32_NUMERIC) {  // f32 records, no categorical split anywhere
        if (use_smem && trav_top() == 0)
            return launch_traverse<RFXC_NODES_F32, true, 0, true>(d_nodes, d_node_off, p, tree_lo,
                                                                 tree_hi, d_values, n, row_lo, row_hi,
                                                                 d_codes_tm, smem, st);
        layout = RFXC_NODES_F32;
    }
    if (layout == RFXC_NODES_F32 && use_smem) {
        switch (trav_top()) {
            case 255: return RFXC_TRAV(RFXC_NODES_F32, true, 255);
            case 127: return RFXC_TRAV(RFXC_NODES_F32, true, 127);
            case 63: return RFXC_TRAV(RFXC_NODES_F32, true, 63);
            default: return RFXC_TRAV(RFXC_NODES_F32, true, 0);
        }
    }
    if (layout == RFXC_NODES_F32) return RFXC_TRAV(RFXC_NODES_F32, false, 0);
    if (layout == RFXC_NODES_F64)
        return use_smem ? RFXC_TRAV(RFXC_NODES_F64, true, 0) : RFXC_TRAV(RFXC_NODES_F64, false, 0);
#undef RFXC_TRAV
    return fail(RFXC_EDATA, "leaf_codes: unknown layout %d", layout);
}

extern "C" int rfxc_leaf_codes(const void* d_nodes, const int64_t* d_node_off, int32_t layout,
                               int32_t p, int32_t tree_lo, int32_t tree_hi,
                               const void* d_values, int64_t n, int32_t* d_codes_tm,
                               void* stream)
{
    return rfxc_leaf_codes_rows(d_nodes, d_node_off, layout, p, tree_lo, tree_hi, d_values, n, 0,
                                n, d_codes_tm, stream);
}

// rows [row_lo, row_hi) of a column-major (n, p) host matrix into the same
// rows of its device copy (one strided DMA): lets a sample block's traversal
// start before the rest of the values have crossed PCIe
extern "C" int rfxc_h2d_rows(void* d_dst, const void* h_src, int64_t n, int64_t p, int32_t elem,
                             int64_t row_lo, int64_t row_hi, void* stream)
{
    if (row_lo < 0 || row_hi > n || row_lo > row_hi || elem < 1)
        return fail(RFXC_EDATA, "h2d_rows: bad range");
    if (row_hi == row_lo) return RFXC_OK;
    const size_t pitch = (size_t)n * elem;
    const cudaError_t e = cudaMemcpy2DAsync(
        static_cast<char*>(d_dst) + row_lo * elem, pitch,
        static_cast<const char*>(h_src) + row_lo * elem, pitch, (size_t)(row_hi - row_lo) * elem,
        (size_t)p, cudaMemcpyHostToDevice, as_stream(stream));
    if (e != cudaSuccess) return fail(RFXC_ECUDA, "h2d_rows: %s", cudaGetErrorString(e));
    return RFXC_OK;
}

extern "C" int rfxc_transpose_i32_ex(const int32_t* d_in, int64_t rows, int64_t cols, int64_t ld_in,
                                     int32_t* d_out, int64_t ld_out, const int32_t* d_col_map,
                                     void* stream)
{
    if (rows < 0 || cols < 0 || ld_in < cols || ld_out < rows)
        return fail(RFXC_EDATA, "transpose: bad shape");
    if (rows == 0 || cols == 0) return RFXC_OK;
    dim3 grid((unsigned)ceil_div(cols, 32), (unsigned)ceil_div(rows, 32 * TRP_TPB));
    transpose_i32_kernel<<<grid, dim3(32, 8), 0, as_stream(stream)>>>(d_in, rows, cols, ld_in, d_out, ld_out,
                                                                       d_col_map);
    return check_launch("transpose_i32");
}

extern "C" int rfxc_transpose_i32(const int32_t* d_in, int64_t rows, int64_t cols,
                                  int32_t* d_out, void* stream)
{
    return rfxc_transpose_i32_ex(d_in, rows, cols, cols, d_out, rows, nullptr, stream);
}

extern "C" int rfxc_leaf_order(const int32_t* d_codes, int64_t n, int32_t nleaf, int32_t* d_order,
                               int32_t* d_scratch, void* stream)
{
    if (n < 1 || nleaf < 1) return fail(RFXC_EDATA, "leaf_order: bad shape");
    cudaStream_t st = as_stream(stream);
    cudaError_t e = cudaMemsetAsync(d_scratch, 0, (size_t)nleaf * 4, st);
    if (e != cudaSuccess) return fail(RFXC_ECUDA, "leaf_order: %s", cudaGetErrorString(e));
    const int grid = (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)sm_count() * 8);
    leaf_hist_kernel<<<grid, 256, 0, st>>>(d_codes, n, d_scratch);
    leaf_scan_kernel<<<1, 1024, 0, st>>>(d_scratch, nleaf);
    leaf_scatter_kernel<<<grid, 256, 0, st>>>(d_codes, n, d_scratch, d_order);
    return check_launch("leaf_order");
}

extern "C" int rfxc_permute_rows_f32(const float* d_X, int64_t n, int32_t p, const int32_t* d_order,
                                     float* d_Xp, void* stream)
{
    if (n < 1 || p < 1) return fail(RFXC_EDATA, "permute_rows: bad shape");
    const int grid = (int)std::min<int64_t>(ceil_div(n * p, 256), (int64_t)sm_count() * 16);
    permute_rows_f32_kernel<<<grid, 256, 0, as_stream(stream)>>>(d_X, n, p, d_order, d_Xp);
    return check_launch("permute_rows_f32");
}

// ------------------------------------------------------------- OOB votes
// the out-of-bag votes the trainer accumulates
// (oob_votes_tree, _kernels.py:377-385, called per tree in forest.py:287-290)
// recomputed from the K1 leaf codes: votes[i, class(leaf_b(i))] += 1 for every
// tree b with inbag[b, i] == 0.  A thread per sample walks the trees in order
// (coalesced codes / inbag rows); counts up to OOB_LOCAL classes stay in
// registers, more use integer atomics (order-free, exact).
constexpr int OOB_LOCAL = 16;

__global__ void oob_votes_kernel(const int32_t* __restrict__ codes_tm, int64_t n, int Bl,
                                 const int64_t* __restrict__ leaf_base,
                                 const int32_t* __restrict__ leaf_class,
                                 const int32_t* __restrict__ inbag, int C,
                                 long long* __restrict__ votes)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    long long loc[OOB_LOCAL];
#pragma unroll
    for (int c = 0; c < OOB_LOCAL; c++) loc[c] = 0;
    for (int b = 0; b < Bl; b++) {
        if (__ldg(inbag + (int64_t)b * n + i) != 0) continue;
        const int cls = __ldg(leaf_class + __ldg(leaf_base + b) + __ldg(codes_tm + (int64_t)b * n + i));
        if (C <= OOB_LOCAL) {
#pragma unroll
            for (int c = 0; c < OOB_LOCAL; c++) loc[c] += (c == cls);
        } else {
            atomicAdd(reinterpret_cast<unsigned long long*>(votes + i * C + cls), 1ull);
        }
    }
    if (C <= OOB_LOCAL)
        for (int c = 0; c < C; c++) votes[i * C + c] = loc[c];
}

extern "C" int rfxc_oob_votes(const int32_t* d_codes_tm, int64_t n, int32_t Bl,
                              const int64_t* d_leaf_base, const int32_t* d_leaf_class,
                              const int32_t* d_inbag, int32_t C, int64_t* d_votes, void* stream)
{
    if (n < 1 || Bl < 1 || C < 1) return fail(RFXC_EDATA, "oob_votes: bad shape");
    cudaStream_t st = as_stream(stream);
    if (C > OOB_LOCAL) {
        const cudaError_t e = cudaMemsetAsync(d_votes, 0, (size_t)n * C * 8, st);
        if (e != cudaSuccess) return fail(RFXC_ECUDA, "oob_votes memset: %s", cudaGetErrorString(e));
    }
    oob_votes_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(
        d_codes_tm, n, Bl, d_leaf_base, d_leaf_class, d_inbag, C,
        reinterpret_cast<long long*>(d_votes));
    return check_launch("oob_votes");
}
