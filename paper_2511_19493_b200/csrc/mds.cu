// mds.cu — K8/K9: factor-space MDS power iteration in one persistent kernel.
//
// Reference: gram_matvec + _hadamard_square_matvec (mds.py:140-181) and
// mds_lowrank (mds.py:184-268): for each of k eigenpairs, start from
// Pcg32(seed + c, SEQ_POWER).normals(n), orthogonalise against the found
// vectors, iterate w = G v - sum_f lambda_f (v_f.v) v_f, project out the
// found vectors, lambda = v.w, v <- w/|w| with the sign aligned to the
// previous iterate, stop when max|v_new - v| < tol or at the iteration cap;
// relative residual |G v - lambda v| / |lambda|; stop at lambda <= 0.
// Coordinates sqrt(lambda) * v, largest-|component| positive
// (mds.py:83-86, :257-261).
//
// G v = -1/2 H D2 H v with D2 u = pmax^2 (sum u) 1 - 2 pmax P u + (P o P) u on
// the UNclamped P = Q Q^T (mds.py:177-179).  With q' = [q | 1] the single
// reduction S' = sum_i u_i q'_i q'_i^T holds S = Q^T diag(u) Q (so that
// (P o P)u_i = q_i^T S q_i — the Khatri-Rao identity of mds.py:147-152
// without the n x r^2 expansion), t = Q^T u (P u_i = q_i . t) and sum(u);
// mean(z) follows in closed form from the constants C' = sum q'q'^T.  S' is
// linear in u, so it is accumulated for the raw v and corrected by
// -mean(v) C' afterwards, which lets the convergence reduction of an update
// ride along with the next matvec's reduction.
//
// B200 mapping: one CTA per SM (cooperative); CTA c owns a contiguous row
// slice and keeps its factor slice in shared memory as int8 codes (code *
// scale is bit-identical to the dequantised factor; other modes read the
// f64 factor from L2).  Both O(n r^2) products run on the FP64 tensor cores
// (DMMA.8x8x4): the S' reduction with one warp per 8x8 tile of the upper
// triangle (A^T B with A = diag(v) Q', B = Q', k-steps of 4 rows), and the
// row pass Z = Q S, PPu_i = sum_c Z_ic q_ic, with warps on 8-row blocks.
// Per iteration: three grid barriers (S' partials -> distributed totals ->
// projections), every reduction in a fixed order, so results are
// bit-reproducible and every stopping decision is identical in every CTA.
#include <cooperative_groups.h>

#include <cstdlib>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace rfxc {

constexpr int XA = 16;         // extra reduction-A slots: sum v, dmax, d_f (f < 8), sum v c, sum v d
constexpr int XS_SUM = 0, XS_DMAX = 1, XS_D = 2, XS_CI = 10, XS_DI = 11;
constexpr int BS = 24;         // reduction-B slots
constexpr int MAXRT = 24;      // r <= 192
constexpr int SMS_MAXRP = 96;  // S kept in shared memory up to RP = 96
constexpr int SMEM_BUDGET = 222 * 1024;  // + ~3 KB of static shared memory
#ifndef RFXC_MDS_I8F_THREADS
#define RFXC_MDS_I8F_THREADS 256
#endif
constexpr int MDS_I8F_THREADS = RFXC_MDS_I8F_THREADS;  // int8-resident fast path (r <= 32)

enum { QS_F64 = 0, QS_I8 = 1, QS_GLOBAL = 2 };

struct MdsArgs {
    const double* dq;       // (n, r) f64 dequantised factor (global)
    const int8_t* codes;    // (n, r) int8 codes (QS_I8) or null
    const double* scales;   // (r) per-column scales (QS_I8)
    int64_t n;
    int r;
    int r8;                 // row stride of the int8 slice (RP: columns >= r are zero)
    double pmax;
    const double* pmax_dev;  // when set, pmax is read from device memory (rfxc_pmax's output)
    int k;
    int max_it;
    double tol;
    int mode;               // 0: MDS, 1: one gram_matvec of V[0] into w
    int qs;                 // QS_* storage of the factor slice
    int64_t rpb;            // rows per CTA
    int TP;                 // 8-column tiles of q' (r + 1 columns)
    int NT;                 // upper-triangle tiles TP (TP + 1) / 2
    int PE;                 // reduction-A entries per CTA: NT * 64 + XA
    double* V;              // k x n: start vectors in, found vectors out
    double* w;              // n
    double* sparts;         // grid x PE
    double* tot;            // PE
    double* cst;            // NT * 64: C' = sum q' q'^T
    double* sc;             // RP x (RP + 4): mean-corrected S of the last reduction (zero padded)
    double* tc;             // RP + 4: mean-corrected t; tc[RP] = su
    double* ci;             // n: q_i^T C q_i (C = Q^T Q)
    double* di;             // n: q_i . c (c = Q^T 1)
    int RPs;                // RP of the instantiated kernel (sc stride RPs + 4)
    double* bparts;         // 2 x grid x BS
    double* coords;         // n x k
    double* info;           // k x 4
    int32_t* k_used;
    unsigned long long* timing;  // debug (RFXC_MDS_TIMING): per-phase ns of CTA 0
};

__device__ __forceinline__ unsigned long long gtime()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define MDS_T(slot)                                                                 \
    do {                                                                            \
        if (A.timing && blockIdx.x == 0 && threadIdx.x == 0) {                      \
            const unsigned long long now_ = gtime();                                \
            A.timing[slot] += now_ - t_last;                                        \
            t_last = now_;                                                          \
        }                                                                           \
    } while (0)

struct Sm {
    const double* q64;  // rows x ldq f64 factor (QS_F64)
    int ldq;
    const int8_t* q8;   // rows x r codes (QS_I8)
    const double* sc;   // r scales
    double* us;         // rows: v of this slice
    double* S;          // RP x RP mean-corrected S (zero padded)
    double* ts;         // PE: this matvec's reduction-A totals (staged)
    double* t;          // RP
    double* red;        // 16 x 32
    double* bc;         // BS broadcast slots
    double* kc;         // 2 constants
    int* tab;           // NT x 2 tile coordinates
    double* buf;        // QS_I8 (RT <= 4): warps x NV x 32 cross-warp partials
};

__host__ __device__ __forceinline__ int rp_of(int r) { return 8 * ((r + 7) / 8); }
// f64 slice row stride: >= RP (the zero-padded width) and = 4 (mod 16)
// doubles, so the 4 rows of a DMMA fragment land on different bank groups
__host__ __device__ __forceinline__ int ldq_of(int rp) { return rp + ((4 - rp % 16) + 16) % 16; }
__host__ __device__ __forceinline__ int64_t pad16(int64_t x) { return (x + 31) / 32 * 32; }  // rows: 8 k-steps of 4

// q'(row, c) of the local slice (c == r is the constant-one column)
template <int QS>
__device__ __forceinline__ double qp(const MdsArgs& A, const Sm& s, int64_t r0, int64_t i, int c)
{
    if (c < A.r) {
        if (QS == QS_F64) return s.q64[i * s.ldq + c];
        if (QS == QS_I8) return (double)s.q8[i * A.r8 + c] * s.sc[c];
        return __ldg(A.dq + (r0 + i) * A.r + c);
    }
    return c == A.r ? 1.0 : 0.0;
}

// raw factor value of slice row i, column c < r (no column checks)
template <int QS>
__device__ __forceinline__ double qraw(const MdsArgs& A, const Sm& s, int64_t r0, int64_t i, int c)
{
    if (QS == QS_F64) return s.q64[i * s.ldq + c];
    if (QS == QS_I8) return (double)s.q8[i * A.r8 + c] * s.sc[c];
    return __ldg(A.dq + (r0 + i) * A.r + c);
}

// Reduction A partial of this CTA: S'(x) tiles (one warp per 8x8 tile of the
// upper triangle, DMMA over 4-row k-steps, four independent accumulator
// chains summed in order), written to sparts[blk].
template <int QS>
__device__ void spass(const MdsArgs& A, const Sm& s, int64_t r0, int64_t rows, const double* x)
{
    (void)r0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int fr = lane & 3, fc = lane >> 2;
    const int r = A.r;
    double* out = A.sparts + (int64_t)blockIdx.x * A.PE;
    if constexpr (QS == QS_F64) {
        // zero-padded slice (rows to 16, columns to ldq): the factor tiles
        // (both tile columns inside the zero-padded factor) run on DMMA with no
        // checks; t = sum x_i q_i and sum x_i (the constant-one column) are a
        // plain reduction written over the (a, r) entries afterwards
        const int ldq = s.ldq;
        const int RTq = (r + 7) / 8;
        const int64_t rows16 = pad16(rows);
        const int nw = (int)(blockDim.x >> 5);
        for (int t = warp; t < A.NT; t += nw) {
            const int ta = s.tab[2 * t], tb = s.tab[2 * t + 1];
            if (tb >= RTq) continue;
            const double* pa = s.q64 + fr * ldq + 8 * ta + fc;
            const double* pb = s.q64 + fr * ldq + 8 * tb + fc;
            const double* px = x + fr;
            // eight independent accumulator chains over the 4-row k-steps
            double d[8][2];
#pragma unroll
            for (int u = 0; u < 8; u++) d[u][0] = d[u][1] = 0.0;
            for (int base = 0; base < rows16; base += 32) {
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const int off = base + 4 * u;
                    dmma884(d[u][0], d[u][1], px[off] * pa[off * ldq], pb[off * ldq]);
                }
            }
#pragma unroll
            for (int j = 0; j < 2; j++)
                out[t * 64 + fc * 8 + 2 * fr + j] = ((d[0][j] + d[1][j]) + (d[2][j] + d[3][j])) +
                                                    ((d[4][j] + d[5][j]) + (d[6][j] + d[7][j]));
        }
        __syncthreads();
        // t_a (a < r) and su (a = r): one warp per column, lanes over rows
        for (int a = warp; a <= r; a += nw) {
            double acc = 0.0;
            if (a < r)
                for (int i = lane; i < rows; i += 32) acc += x[i] * s.q64[i * ldq + a];
            else
                for (int i = lane; i < rows; i += 32) acc += x[i];
            acc = warp_sum(acc);
            if (lane == 0) {
                const int ta = a >> 3, tb = r >> 3;
                const int t = ta * A.TP - ta * (ta - 1) / 2 + (tb - ta);
                out[t * 64 + (a & 7) * 8 + (r & 7)] = acc;
            }
        }
        return;
    }
    for (int t = warp; t < A.NT; t += (int)(blockDim.x >> 5)) {
        const int ca = 8 * s.tab[2 * t] + fc, cb = 8 * s.tab[2 * t + 1] + fc;
        // q' column: a factor column, the constant-one column r, or zero padding
        const bool fa = ca < r, fb = cb < r;
        const double oa = ca == r ? 1.0 : 0.0, ob = cb == r ? 1.0 : 0.0;
        const int ka = fa ? ca : 0, kb = fb ? cb : 0;
        double d[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
        for (int64_t base = 0; base < rows; base += 16) {
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int64_t i = base + 4 * u + fr;
                const bool ok = i < rows;
                const int64_t ii = ok ? i : 0;
                const double xi = ok ? x[ii] : 0.0;
                const double qa = fa ? qraw<QS>(A, s, r0, ii, ka) : oa;
                const double qb = fb ? qraw<QS>(A, s, r0, ii, kb) : ob;
                dmma884(d[u][0], d[u][1], xi * qa, ok ? qb : 0.0);
            }
        }
        out[t * 64 + fc * 8 + 2 * fr] = (d[0][0] + d[1][0]) + (d[2][0] + d[3][0]);
        out[t * 64 + fc * 8 + 2 * fr + 1] = (d[0][1] + d[1][1]) + (d[2][1] + d[3][1]);
    }
}

// S'(x) partial of this CTA for a smem-resident f64 slice with r <= 8 * RT
// (RT <= 4): four warps split the 4-row k-steps and each accumulates the
// whole upper triangle (one B fragment per column tile per k-step, the A
// fragment is x times it, RT(RT+1)/2 DMMA chains) plus t = sum x q and
// sum x; the four warp partials are added in warp order 3, 2, 1, 0 through
// shared memory `buf` (>= 32 * (RT(RT+1) + RT + 1) doubles).  Warps >= SP_W
// run `extra()` while the first SP_W warps multiply.
constexpr int SP_W = 4;
template <int RT, typename Extra>
__device__ void spass4(const MdsArgs& A, const Sm& s, int64_t rows, const double* x, double* buf,
                       Extra&& extra)
{
    constexpr int NP = RT * (RT + 1) / 2;
    constexpr int NV = 2 * NP + RT + 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int fr = lane & 3, fc = lane >> 2;
    const int r = A.r, ldq = s.ldq;
    double* out = A.sparts + (int64_t)blockIdx.x * A.PE;
    double v[NV];
#pragma unroll
    for (int j = 0; j < NV; j++) v[j] = 0.0;
    if (warp < SP_W) {
        const int nks = (int)(pad16(rows) >> 2);
        const int k0 = warp * nks / SP_W, k1 = (warp + 1) * nks / SP_W;
        const double* pq = s.q64 + fc;
#pragma unroll 2
        for (int ks = k0; ks < k1; ks++) {
            const int i = 4 * ks + fr;
            const double xq = x[i];
            double b[RT], a[RT];
#pragma unroll
            for (int t = 0; t < RT; t++) {
                b[t] = pq[i * ldq + 8 * t];
                a[t] = xq * b[t];
                v[2 * NP + t] += a[t];
            }
            v[2 * NP + RT] += xq;
            int pi = 0;
#pragma unroll
            for (int ta = 0; ta < RT; ta++)
#pragma unroll
                for (int tb = ta; tb < RT; tb++, pi++) dmma884(v[2 * pi], v[2 * pi + 1], a[ta], b[tb]);
        }
        // t and sum x over the 4 row phases of the fragment
#pragma unroll
        for (int j = 2 * NP; j < NV; j++) {
            v[j] += __shfl_xor_sync(0xffffffffu, v[j], 1);
            v[j] += __shfl_xor_sync(0xffffffffu, v[j], 2);
        }
    } else {
        extra();  // the other warps do the caller's row sums meanwhile
    }
    for (int w = SP_W - 1; w >= 1; w--) {
        if (warp == w) {
#pragma unroll
            for (int j = 0; j < NV; j++) buf[j * 32 + lane] = v[j];
        }
        __syncthreads();
        if (warp == w - 1) {
#pragma unroll
            for (int j = 0; j < NV; j++) v[j] += buf[j * 32 + lane];
        }
        __syncthreads();
    }
    if (warp == 0) {
        const int RTq = (r + 7) / 8;
        int pi = 0;
#pragma unroll
        for (int ta = 0; ta < RT; ta++)
#pragma unroll
            for (int tb = ta; tb < RT; tb++, pi++) {
                if (tb >= RTq) continue;
                const int t = ta * A.TP - ta * (ta - 1) / 2 + (tb - ta);
                out[t * 64 + fc * 8 + 2 * fr] = v[2 * pi];
                out[t * 64 + fc * 8 + 2 * fr + 1] = v[2 * pi + 1];
            }
        if (fr == 0) {
            const int tbr = r >> 3;
#pragma unroll
            for (int t = 0; t < RT; t++) {
                const int a = 8 * t + fc;
                if (a < r) {
                    const int ta = a >> 3;
                    out[(ta * A.TP - ta * (ta - 1) / 2 + (tbr - ta)) * 64 + (a & 7) * 8 + (r & 7)] = v[2 * NP + t];
                }
            }
            if (fc == 0)
                out[(tbr * A.TP - tbr * (tbr - 1) / 2) * 64 + (r & 7) * 8 + (r & 7)] = v[2 * NP + RT];
        }
    }
}

// S'(x) partial of this CTA for the int8-resident slice (codes c, per-column
// scales s; q = c * s), r <= 8 * RT, RT <= 4, every warp of the CTA on the
// FP64 tensor cores: warp w takes a contiguous share of the 4-row k-steps
// and accumulates the whole upper triangle of S_c = sum_i x_i c_i c_i^T
// (integer codes are exact in f64: A = x * c, B = c), t_c = sum x c and
// sum x; the warps' partials meet in shared memory `buf` (warps x NV x 32
// doubles) and are added in warp order; the CTA partial is written in the
// q-space (S_ab = s_a s_b S_c,ab, t_a = s_a t_c,a) the reductions use.
template <int RT, typename Extra>
__device__ void spass_i8(const MdsArgs& A, const Sm& s, int64_t rows, const double* x, double* buf,
                         Extra&& extra)
{
    constexpr int NP = RT * (RT + 1) / 2;
    constexpr int NV = 2 * NP + RT + 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = (int)(blockDim.x >> 5);
    const int fr = lane & 3, fc = lane >> 2;
    const int r = A.r;
    double* out = A.sparts + (int64_t)blockIdx.x * A.PE;
    double v[NV];
#pragma unroll
    for (int j = 0; j < NV; j++) v[j] = 0.0;
    {
        const int nks = (int)(pad16(rows) >> 2);
        const int k0 = warp * nks / nw, k1 = (warp + 1) * nks / nw;
        // lane's columns 8t + fc of the zero-padded slice (codes beyond r are 0)
        // column 8 t + fc of row i sits at byte fc * RT + t (permuted slice)
        const int8_t* pq = s.q8 + fc * RT;
        const int ldc = A.r8;
#pragma unroll 2
        for (int ks = k0; ks < k1; ks++) {
            const int i = 4 * ks + fr;
            const double xq = x[i];
            double b[RT], a[RT];
            if constexpr (RT == 4) {
                const int wd = *reinterpret_cast<const int*>(pq + i * ldc);
#pragma unroll
                for (int t = 0; t < 4; t++) b[t] = (double)(int8_t)(wd >> (8 * t));
            } else {
#pragma unroll
                for (int t = 0; t < RT; t++) b[t] = (double)pq[i * ldc + t];
            }
#pragma unroll
            for (int t = 0; t < RT; t++) {
                a[t] = xq * b[t];
                v[2 * NP + t] += a[t];
            }
            v[2 * NP + RT] += xq;
            int pi = 0;
#pragma unroll
            for (int ta = 0; ta < RT; ta++)
#pragma unroll
                for (int tb = ta; tb < RT; tb++, pi++) dmma884(v[2 * pi], v[2 * pi + 1], a[ta], b[tb]);
        }
#pragma unroll
        for (int j = 2 * NP; j < NV; j++) {
            v[j] += __shfl_xor_sync(0xffffffffu, v[j], 1);
            v[j] += __shfl_xor_sync(0xffffffffu, v[j], 2);
        }
    }
#pragma unroll
    for (int j = 0; j < NV; j++) buf[(warp * NV + j) * 32 + lane] = v[j];
    extra((int)threadIdx.x, (int)blockDim.x);  // the caller's row sums meanwhile
    __syncthreads();
    // value (j, lane) of the CTA partial: the warps' values in warp order
    const int RTq = (r + 7) / 8, tbr = r >> 3;
    for (int e = threadIdx.x; e < NV * 32; e += (int)blockDim.x) {
        const int j = e >> 5, ln = e & 31, efr = ln & 3, efc = ln >> 2;
        double acc = 0.0;
        for (int w = 0; w < nw; w++) acc += buf[(w * NV + j) * 32 + ln];
        if (j < 2 * NP) {
            // tile pi = j / 2, fragment element (efc, 2 efr + j % 2)
            int pi = j >> 1, ta = 0;
            while (pi >= RT - ta) { pi -= RT - ta; ta++; }
            const int tb = ta + pi;
            if (tb >= RTq) continue;
            const int a = 8 * ta + efc, bcol = 8 * tb + 2 * efr + (j & 1);
            // (a, r) and (r, r) are the t / sum slots written below; every
            // other entry beyond the factor is zero padding
            if ((bcol == r && a <= r)) continue;
            const int t = ta * A.TP - ta * (ta - 1) / 2 + (tb - ta);
            out[t * 64 + efc * 8 + 2 * efr + (j & 1)] =
                (a < r && bcol < r) ? (s.sc[a] * s.sc[bcol]) * acc : 0.0;
        } else if (j < 2 * NP + RT) {
            if (efr != 0) continue;  // the four row phases were already added
            const int a = 8 * (j - 2 * NP) + efc;
            if (a < r) {
                const int ta = a >> 3;
                out[(ta * A.TP - ta * (ta - 1) / 2 + (tbr - ta)) * 64 + (a & 7) * 8 + (r & 7)] =
                    s.sc[a] * acc;
            }
        } else if (ln == 0) {
            out[(tbr * A.TP - tbr * (tbr - 1) / 2) * 64 + (r & 7) * 8 + (r & 7)] = acc;
        }
    }
}

// fixed-order block reduction of m <= 16 per-thread values into out[0..m)
// (warp trees, then the warp partials in warp order); red >= 16 * warps
__device__ void block_sums(double* v, int m, double* red, double* out)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
#pragma unroll
    for (int j = 0; j < 16; j++)
        if (j < m) {
            const double x = warp_sum(v[j]);
            if (lane == 0) red[warp * 16 + j] = x;
        }
    __syncthreads();
    if ((int)threadIdx.x < m) {
        double t = 0.0;
        for (int w = 0; w < nw; w++) t += red[w * 16 + threadIdx.x];
        out[threadIdx.x] = t;
    }
    __syncthreads();
}

// Distributed final reduction of the grid's reduction-A partials into tot:
// one warp per entry, lanes over blocks in order; the dmax slot takes a max.
__device__ void final_a(const MdsArgs& A, int entries, const int* tab)
{
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * (int)(blockDim.x >> 5) + (threadIdx.x >> 5), nw = gridDim.x * (int)(blockDim.x >> 5);
    const int dm = A.NT * 64 + XS_DMAX;
    const int r = A.r, SL = A.RPs + 4;
    if (gw >= entries) return;
    for (int e = gw; e < entries; e += nw) {
        // the entry and mean(v) (the sum slot, in its own entry's order) from
        // one pass over the CTA partials; C' of the entry fetched alongside
        const double ce = (lane == 0 && e < A.NT * 64) ? A.cst[e] : 0.0;
        double v = 0.0, sv = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) {
            const double x = A.sparts[(int64_t)b * A.PE + e];
            sv += A.sparts[(int64_t)b * A.PE + A.NT * 64 + XS_SUM];
            v = (e == dm) ? fmax(v, x) : v + x;
        }
        v = (e == dm) ? warp_max(v) : warp_sum(v);
        const double mean = warp_sum(sv) / (double)A.n;
        if (lane != 0) continue;
        A.tot[e] = v;
        if (e >= A.NT * 64 || !A.sc) continue;
        // S'(v) entry -> mean-corrected S, t or su
        const int t = e >> 6, ta = tab[2 * t], tb = tab[2 * t + 1];
        const int a = 8 * ta + ((e >> 3) & 7), b = 8 * tb + (e & 7);
        const double c = v - mean * ce;
        if (a < r && b < r) {
            A.sc[a * SL + b] = c;
            if (ta != tb) A.sc[b * SL + a] = c;
        } else if (a < r && b == r) {
            A.tc[a] = c;
        } else if (a == r && b == r) {
            A.tc[A.RPs] = c;
        }
    }
}

// redundant per-CTA sum of m reduction-B partials (buffer `par`) -> s.bc
__device__ void final_b(const MdsArgs& A, const Sm& s, int par, int m)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double* p = A.bparts + (int64_t)par * gridDim.x * BS;
    for (int j = warp; j < m; j += (int)(blockDim.x >> 5)) {
        double v = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) v += p[(int64_t)b * BS + j];
        v = warp_sum(v);
        if (lane == 0) s.bc[j] = v;
    }
    __syncthreads();
}

// S'(x) entry (a, b) of the tiled upper triangle in `src`
__device__ __forceinline__ double tile_entry(const double* src, const int* tab, int TP, int a, int b)
{
    if (a > b) { const int q = a; a = b; b = q; }
    const int ta = a >> 3, tb = b >> 3;
    const int t = ta * TP - ta * (ta - 1) / 2 + (tb - ta);
    (void)tab;
    return src[t * 64 + (a & 7) * 8 + (b & 7)];
}

// One deflated Gram matvec of the slice's v (s.us) given the reduced totals:
// builds S and t in shared memory, then the DMMA row pass writes w for the
// slice and returns (in thread-local accumulators of the row-owner lanes)
// the projections needed afterwards.  mode: 0 -> e_f = V_f.w, v.w, w.w;
// 1 -> residual sum (w - lam v)^2.
template <int QS, int RT>
__device__ void rowpass(const MdsArgs& A, const Sm& s, int64_t r0, int64_t rows, int nf,
                        const double* lam_s, int comp, int rmode, double lam, double* bacc)
{
    constexpr bool SMS = RT * 8 <= SMS_MAXRP;
    const int r = A.r, RP = 8 * RT, TP = A.TP;
    const int64_t n = A.n;
    // totals staged in shared memory (one coalesced pass), then the mean-
    // corrected S, t and the closed-form mean of z
    const double* T = A.tot;
    const double mean = rmode == 3 ? 0.0 : T[A.NT * 64 + XS_SUM] / (double)n;
    double ct = 0.0, sgm = 0.0, su = 0.0;
    if (rmode == 3) {
        // s.S / s.t hold C and c: the row pass gives c_i and d_i
    } else if (SMS) {
        // S, t and su were corrected by final_a; the two scalar sums follow
        // from the per-row constants: sum_ab S_ab C_ab = sum_i v_i c_i - mean |C|^2
        for (int e = threadIdx.x; e < RP * (RP + 4); e += (int)blockDim.x) s.S[e] = A.sc[e];
        for (int a = threadIdx.x; a < RP; a += (int)blockDim.x) s.t[a] = A.tc[a];
        su = A.tc[RP];
        sgm = T[A.NT * 64 + XS_CI] - mean * s.kc[0];
        ct = T[A.NT * 64 + XS_DI] - mean * s.kc[1];
        __syncthreads();
    } else {
        for (int e = threadIdx.x; e < r * r; e += (int)blockDim.x) {
            const int a = e / r, b = e % r;
            const double g = tile_entry(A.cst, s.tab, TP, a, b);
            sgm += (tile_entry(T, s.tab, TP, a, b) - mean * g) * g;
        }
        for (int a = threadIdx.x; a < RP; a += (int)blockDim.x) {
            double v = 0.0;
            if (a < r) {
                const double c = tile_entry(A.cst, s.tab, TP, a, r);
                v = tile_entry(T, s.tab, TP, a, r) - mean * c;
                ct += c * v;
            }
            s.t[a] = v;
        }
        __syncthreads();
        su = tile_entry(T, s.tab, TP, r, r) - mean * tile_entry(A.cst, s.tab, TP, r, r);
        ct = block_sum(ct, s.red);
        sgm = block_sum(sgm, s.red);
    }
    const double pm = A.pmax_dev ? __ldg(A.pmax_dev) : A.pmax;
    const double mz = (pm * pm) * su - 2.0 * pm * ct / (double)n + sgm / (double)n;
    double dfl[8];
    for (int f = 0; f < nf; f++) dfl[f] = lam_s[f] * T[A.NT * 64 + XS_D + f];
    if (A.timing && blockIdx.x == 0 && threadIdx.x == 0) A.timing[11] = gtime();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int fr = lane & 3, fc = lane >> 2;
    const int KS = (r + 3) / 4;
    // int8 fast path: the lane's fragments of S~ = D S D (D = diag(scales), so
    // the A operands are the exact integer codes) and of t~ = D t stay in
    // registers for the whole row loop
    constexpr bool I8F = QS == QS_I8 && SMS && RT <= 4;
    constexpr int NPF = RT * (RT + 1) / 2;
    double sf[I8F ? 2 * NPF : 1], tf[I8F ? 2 * RT : 1];
    if constexpr (I8F) {
        int pi = 0;
#pragma unroll
        for (int ta = 0; ta < RT; ta++)
#pragma unroll
            for (int tb = ta; tb < RT; tb++, pi++)
#pragma unroll
                for (int ks = 0; ks < 2; ks++) {
                    const int kr = 8 * ta + 4 * ks + fr, col = 8 * tb + fc;
                    const double sk = kr < r ? s.sc[kr] : 0.0, sc2 = col < r ? s.sc[col] : 0.0;
                    // off-diagonal tile pairs count twice (symmetric S): the
                    // exact factor 2 rides in the fragment
                    const double wgt = ta == tb ? 1.0 : 2.0;
                    sf[2 * pi + ks] = wgt * ((sk * s.S[kr * (RP + 4) + col]) * sc2);
                }
#pragma unroll
        for (int j = 0; j < 2 * RT; j++) {
            const int col = 4 * j + fr;
            tf[j] = col < r ? s.sc[col] * s.t[col] : 0.0;
        }
    }
    for (int64_t row0 = 8 * (int64_t)warp; row0 < rows; row0 += 8 * (int)(blockDim.x >> 5)) {
        const int64_t ia = row0 + fc;  // fragment / output row of this lane
        const bool va = ia < rows;
        double acc[RT][2];
#pragma unroll
        for (int tn = 0; tn < RT; tn++) acc[tn][0] = acc[tn][1] = 0.0;
        double ppu = 0.0, pu = 0.0;
        if constexpr (I8F) {
            // the lane's 4 RT codes of the row: A-fragment columns 4 j + fr and the
            // epilogue columns 8 tb + 2 fr + h (zero-padded slice: rows to 16,
            // columns to RP), converted exactly to f64
            // permuted slice: column c at byte (c % 8) * RT + c / 8.  A fragment j
            // = column 4 j + fr, epilogue j = column 8 (j / 2) + 2 fr + j % 2
            const int8_t* row = s.q8 + ia * A.r8;
            double af[2 * RT], ep[2 * RT];
            if constexpr (RT == 4) {
                const int* w = reinterpret_cast<const int*>(row);
                const int wa0 = w[fr], wa1 = w[4 + fr], we0 = w[2 * fr], we1 = w[2 * fr + 1];
#pragma unroll
                for (int j = 0; j < 2 * RT; j++) {
                    af[j] = (double)(int8_t)(((j & 1) ? wa1 : wa0) >> (8 * (j >> 1)));
                    ep[j] = (double)(int8_t)(((j & 1) ? we1 : we0) >> (8 * (j >> 1)));
                }
            } else {
#pragma unroll
                for (int j = 0; j < 2 * RT; j++) {
                    af[j] = (double)row[(4 * (j & 1) + fr) * RT + (j >> 1)];
                    ep[j] = (double)row[(2 * fr + (j & 1)) * RT + (j >> 1)];
                }
            }
            // z_tb = sum over ta <= tb of the row's codes (tile ta) times S~(ta, tb):
            // one accumulator per column tile, the tile pairs and k-steps
            // accumulated on the tensor core (pairs ordered ks-major so the
            // chains interleave across tiles)
            double z[RT][2];
#pragma unroll
            for (int tb = 0; tb < RT; tb++) z[tb][0] = z[tb][1] = 0.0;
#pragma unroll
            for (int ta = 0; ta < RT; ta++)
#pragma unroll
                for (int ks = 0; ks < 2; ks++) {
#pragma unroll
                    for (int tb = ta; tb < RT; tb++) {
                        const int pi = ta * RT - ta * (ta - 1) / 2 + (tb - ta);
                        dmma884(z[tb][0], z[tb][1], af[2 * ta + ks], sf[2 * pi + ks]);
                    }
                }
#pragma unroll
            for (int tb = 0; tb < RT; tb++)
                ppu += z[tb][0] * ep[2 * tb] + z[tb][1] * ep[2 * tb + 1];
#pragma unroll
            for (int j = 0; j < 2 * RT; j++) pu += af[j] * tf[j];
        } else if constexpr (QS == QS_F64 && SMS) {
            // q^T S q over the upper-triangle tile pairs of the symmetric S:
            // Z = Q_(ta) S_(ta,tb) (2 k-steps), then ppu += w Z . Q_(tb)
            const double* pq = s.q64 + ia * s.ldq;
            constexpr int NP = RT * (RT + 1) / 2;
            double z[NP][2];
            // all tile pairs' DMMAs first (independent accumulators), then the epilogue
#pragma unroll
            for (int ks = 0; ks < 2; ks++) {
                int pi = 0;
#pragma unroll
                for (int ta = 0; ta < RT; ta++) {
                    const int kr = 8 * ta + 4 * ks + fr;
                    const double a = pq[kr];
#pragma unroll
                    for (int tb = ta; tb < RT; tb++, pi++) {
                        if (ks == 0) z[pi][0] = z[pi][1] = 0.0;
                        dmma884(z[pi][0], z[pi][1], a, s.S[kr * (RP + 4) + 8 * tb + fc]);
                    }
                }
            }
            {
                int pi = 0;
#pragma unroll
                for (int ta = 0; ta < RT; ta++)
#pragma unroll
                    for (int tb = ta; tb < RT; tb++, pi++) {
                        const double wgt = ta == tb ? 1.0 : 2.0;
                        ppu += wgt * (z[pi][0] * pq[8 * tb + 2 * fr] + z[pi][1] * pq[8 * tb + 2 * fr + 1]);
                    }
            }
#pragma unroll
            for (int j = 0; j < 2 * RT; j++) pu += pq[4 * j + fr] * s.t[4 * j + fr];
        } else {
            for (int ks = 0; ks < KS; ks++) {
                const int c = 4 * ks + fr;
                const double a = (va && c < r) ? qp<QS>(A, s, r0, ia, c) : 0.0;
                const int kr = 4 * ks + fr;
#pragma unroll
                for (int tn = 0; tn < RT; tn++) {
                    double b;
                    if (SMS) {
                        b = s.S[kr * (RP + 4) + 8 * tn + fc];
                    } else {
                        const int cb = 8 * tn + fc;
                        b = (kr < r && cb < r) ? tile_entry(T, s.tab, TP, kr, cb) -
                                                     mean * tile_entry(A.cst, s.tab, TP, kr, cb)
                                               : 0.0;
                    }
                    dmma884(acc[tn][0], acc[tn][1], a, b);
                }
            }
            if (va) {
#pragma unroll
                for (int tn = 0; tn < RT; tn++) {
                    const int c = 8 * tn + 2 * fr;
                    if (c < r) ppu += acc[tn][0] * qp<QS>(A, s, r0, ia, c);
                    if (c + 1 < r) ppu += acc[tn][1] * qp<QS>(A, s, r0, ia, c + 1);
                }
                for (int c = fr; c < r; c += 4) pu += qp<QS>(A, s, r0, ia, c) * s.t[c];
            }
        }
        ppu += __shfl_xor_sync(0xffffffffu, ppu, 1);
        ppu += __shfl_xor_sync(0xffffffffu, ppu, 2);
        pu += __shfl_xor_sync(0xffffffffu, pu, 1);
        pu += __shfl_xor_sync(0xffffffffu, pu, 2);
        if (rmode == 3) {
            if (va && fr == 0) {
                A.ci[r0 + ia] = ppu;
                A.di[r0 + ia] = pu;
            }
            continue;
        }
        if (va && fr == 0) {
            const int64_t g = r0 + ia;
            const double zi = (pm * pm) * su - 2.0 * pm * pu + ppu;
            double yi = -0.5 * (zi - mz);
            for (int f = 0; f < nf; f++) yi -= dfl[f] * A.V[(int64_t)f * n + g];
            A.w[g] = yi;
            if (rmode == 0) {
                for (int f = 0; f < nf; f++) bacc[f] += A.V[(int64_t)f * n + g] * yi;
                bacc[nf] += s.us[ia] * yi;
                bacc[nf + 1] += yi * yi;
            } else if (rmode == 1) {
                const double e = yi - lam * s.us[ia];
                bacc[0] += e * e;
            }
        }
    }
    (void)comp;
    if (A.timing && blockIdx.x == 0 && threadIdx.x == 0) A.timing[12] += gtime() - A.timing[11];
    __syncthreads();
}

// grid-wide sum of m per-thread values (one barrier, redundant final)
__device__ void grid_sum(const MdsArgs& A, const Sm& s, cg::grid_group& grid, int& par, double* v,
                         int m)
{
    double* p = A.bparts + (int64_t)par * gridDim.x * BS;
    block_sums(v, m, s.red, s.bc);
    if (threadIdx.x < m) p[(int64_t)blockIdx.x * BS + threadIdx.x] = s.bc[threadIdx.x];
    grid.sync();
    final_b(A, s, par, m);
    for (int j = 0; j < m; j++) v[j] = s.bc[j];
    __syncthreads();
    par ^= 1;
}

template <int QS, int RT, int NTH>
__global__ void __launch_bounds__(NTH, 1) mds_kernel(MdsArgs A)
{
    extern __shared__ __align__(16) unsigned char msm[];
    __shared__ double red[16 * 32];
    __shared__ double bc[BS];
    __shared__ double kc[2];  // sum_ab C_ab^2, sum_a c_a^2
    __shared__ double lam_s[8];
    __shared__ int tab[2 * 300];
    cg::grid_group grid = cg::this_grid();
    constexpr bool SMS = RT * 8 <= SMS_MAXRP;
    const int r = A.r, RP = 8 * RT;
    const int64_t n = A.n;
    const int64_t r0 = min64(n, blockIdx.x * A.rpb);
    const int64_t rows = min64(n, r0 + A.rpb) - r0;

    // shared memory: [S RPxRP if SMS] [t RP] [us rpb] [scales r] [codes pad16(rpb) x RP]
    // [I8F: cross-warp partials warps x NV x 32]
    constexpr bool I8F = QS == QS_I8 && SMS && RT <= 4;
    Sm s;
    s.S = reinterpret_cast<double*>(msm);
    s.t = s.S + (SMS ? RP * (RP + 4) : 0);
    s.ts = s.t + RP;
    s.us = s.ts;
    double* scs = s.us + pad16(A.rpb);
    s.sc = scs;
    s.q8 = reinterpret_cast<const int8_t*>(scs + r);
    s.ldq = ldq_of(RP);
    s.q64 = scs + r;
    s.red = red;
    s.bc = bc;
    s.kc = kc;
    s.tab = tab;
    s.buf = scs + r + (pad16(A.rpb) * RP + 7) / 8;
    if (threadIdx.x == 0) {
        int t = 0;
        for (int a = 0; a < A.TP; a++)
            for (int b = a; b < A.TP; b++) {
                tab[2 * t] = a;
                tab[2 * t + 1] = b;
                t++;
            }
    }
    if (QS == QS_I8) {
        int8_t* q8 = reinterpret_cast<int8_t*>(scs + r);
        for (int e = threadIdx.x; e < r; e += (int)blockDim.x) scs[e] = A.scales[e];
        // zero-padded to pad16(rpb) rows x RP columns (A.r8 = RP); the fast
        // path (RT <= 4) stores column c of a row at byte (c % 8) * RT + c / 8,
        // so a DMMA fragment's RT codes (columns fc, fc + 8, ...) are one load
        for (int64_t e = threadIdx.x; e < pad16(A.rpb) * RP; e += (int)blockDim.x) {
            const int64_t i = e / RP;
            const int c = (int)(e % RP);
            const int at = I8F ? (c % 8) * RT + c / 8 : c;
            q8[i * RP + at] = (i < rows && c < r) ? A.codes[(r0 + i) * r + c] : (int8_t)0;
        }
    } else if (QS == QS_F64) {  // zero-padded to pad16(rpb) rows x ldq columns
        double* q64 = scs + r;
        const int64_t tot = pad16(A.rpb) * s.ldq;
        for (int64_t e = threadIdx.x; e < tot; e += (int)blockDim.x) {
            const int64_t i = e / s.ldq;
            const int c = (int)(e % s.ldq);
            q64[e] = (i < rows && c < r) ? A.dq[(r0 + i) * r + c] : 0.0;
        }
    }
    for (int64_t i = threadIdx.x; i < pad16(A.rpb); i += (int)blockDim.x) s.us[i] = 0.0;
    __syncthreads();
    int par = 0;
    const int EA = A.NT * 64 + XA;

    constexpr bool SP4 = QS == QS_F64 && SMS && RT >= 2 && RT <= 4;
    // S' reduction of s.us; `extra(t0, stride)` (row sums over rows t0, t0 +
    // stride, ...) runs on the warps the reduction leaves idle
    auto sreduce = [&](auto&& extra) {
        if constexpr (I8F) {
            spass_i8<RT>(A, s, rows, s.us, s.buf, extra);
        } else if constexpr (SP4) {
            spass4<RT>(A, s, rows, s.us, s.S, [&]() {
                extra((int)threadIdx.x - 32 * SP_W, (int)blockDim.x - 32 * SP_W);
            });
        } else {
            spass<QS>(A, s, r0, rows, s.us);
            extra((int)threadIdx.x, (int)blockDim.x);
        }
    };
    // constants C' = sum q' q'^T (u = 1)
    for (int64_t i = threadIdx.x; i < rows; i += (int)blockDim.x) s.us[i] = 1.0;
    __syncthreads();
    sreduce([](int, int) {});
    grid.sync();
    {
        const int lane = threadIdx.x & 31;
        const int gw = blockIdx.x * (int)(blockDim.x >> 5) + (threadIdx.x >> 5), nw = gridDim.x * (int)(blockDim.x >> 5);
        for (int e = gw; e < A.NT * 64; e += nw) {
            double v = 0.0;
            for (int b = lane; b < (int)gridDim.x; b += 32) v += A.sparts[(int64_t)b * A.PE + e];
            v = warp_sum(v);
            if (lane == 0) A.cst[e] = v;
        }
        // zero padding of the corrected S / t written by final_a
        if (SMS) {
            const int nsc = RP * (RP + 4);
            for (int e = blockIdx.x * (int)blockDim.x + threadIdx.x; e < nsc + RP + 4;
                 e += gridDim.x * (int)blockDim.x) {
                if (e < nsc) A.sc[e] = 0.0;
                else A.tc[e - nsc] = 0.0;
            }
        }
    }
    grid.sync();
    if (SMS) {
        // per-row constants c_i = q_i^T C q_i, d_i = q_i . c and |C|^2, |c|^2,
        // with C = Q^T Q and c = Q^T 1 staged in s.S / s.t
        const int SL = RP + 4;
        double f2 = 0.0, n2 = 0.0;
        for (int e = threadIdx.x; e < RP * SL; e += (int)blockDim.x) {
            const int a = e / SL, b = e % SL;
            double v = 0.0;
            if (a < r && b < r) {
                v = tile_entry(A.cst, s.tab, A.TP, a, b);
                f2 += v * v;
            }
            s.S[e] = v;
        }
        for (int a = threadIdx.x; a < RP; a += (int)blockDim.x) {
            const double v = a < r ? tile_entry(A.cst, s.tab, A.TP, a, r) : 0.0;
            n2 += v * v;
            s.t[a] = v;
        }
        f2 = block_sum(f2, s.red);
        n2 = block_sum(n2, s.red);
        if (threadIdx.x == 0) {
            kc[0] = f2;
            kc[1] = n2;
        }
        __syncthreads();
        double dummy[BS];
        rowpass<QS, RT>(A, s, r0, rows, 0, lam_s, 0, 3, 0.0, dummy);
    }

    // reduction A of the slice's v (s.us) with nf deflation dots and the
    // previous update's max change; leaves the totals in A.tot
    unsigned long long t_last = gtime();
    auto reduce_a = [&](int nf, double dmax_local) {
        MDS_T(0);
        double x[XS_DI + 1];
#pragma unroll
        for (int j = 0; j <= XS_DI; j++) x[j] = 0.0;
        sreduce([&](int t0, int stride) {
            for (int64_t i = t0; i < rows; i += stride) {
                const double vi = s.us[i];
                x[XS_SUM] += vi;
#pragma unroll
                for (int f = 0; f < 8; f++)
                    if (f < nf) x[XS_D + f] += A.V[(int64_t)f * n + r0 + i] * vi;
                if (SMS) {
                    x[XS_CI] += A.ci[r0 + i] * vi;
                    x[XS_DI] += A.di[r0 + i] * vi;
                }
            }
        });
        MDS_T(1);
        double* out = A.sparts + (int64_t)blockIdx.x * A.PE + A.NT * 64;
        block_sums(x, XS_DI + 1, s.red, s.bc);
        const double dm = block_max(dmax_local, s.red);
        if (threadIdx.x <= XS_DI) out[threadIdx.x] = threadIdx.x == XS_DMAX ? dm : s.bc[threadIdx.x];
        MDS_T(2);
        grid.sync();
        MDS_T(3);
        final_a(A, EA, s.tab);
        MDS_T(4);
        grid.sync();
        MDS_T(5);
    };

    if (A.mode == 1) {  // a single gram_matvec of V[0]
        for (int64_t i = threadIdx.x; i < rows; i += (int)blockDim.x) s.us[i] = A.V[r0 + i];
        __syncthreads();
        reduce_a(0, 0.0);
        double bacc[BS] = {};
        rowpass<QS, RT>(A, s, r0, rows, 0, lam_s, 0, 2, 0.0, bacc);
        return;
    }

    int kused = 0;
    for (int comp = 0; comp < A.k; comp++) {
        double* v = A.V + (int64_t)comp * n;
        for (int f = 0; f < comp; f++) {  // start vector: sequential Gram-Schmidt
            const double* vf = A.V + (int64_t)f * n;
            double dd[1] = {0.0};
            for (int64_t i = r0 + threadIdx.x; i < r0 + rows; i += (int)blockDim.x) dd[0] += vf[i] * v[i];
            grid_sum(A, s, grid, par, dd, 1);
            for (int64_t i = r0 + threadIdx.x; i < r0 + rows; i += (int)blockDim.x) v[i] -= dd[0] * vf[i];
            __syncthreads();
        }
        double nn[1] = {0.0};
        for (int64_t i = r0 + threadIdx.x; i < r0 + rows; i += (int)blockDim.x) nn[0] += v[i] * v[i];
        grid_sum(A, s, grid, par, nn, 1);
        const double nv = sqrt(nn[0]);
        if (nv == 0.0) break;
        for (int64_t i = threadIdx.x; i < rows; i += (int)blockDim.x) {
            const double x = v[r0 + i] / nv;
            v[r0 + i] = x;
            s.us[i] = x;
        }
        __syncthreads();

        double lam = 0.0, dmax_local = 0.0;
        bool conv = false, stop = false;
        int it = 0;
        double rel = INFINITY;
        while (true) {
            reduce_a(comp, dmax_local);
            const bool check = it >= 1;
            const double dmax = A.tot[A.NT * 64 + XS_DMAX];
            const bool done = (check && dmax < A.tol) || it >= A.max_it;
            if (check && dmax < A.tol) conv = true;
            // the matvec of this v: an iteration step, or (done) the residual
            double bacc[BS];
            for (int j = 0; j < BS; j++) bacc[j] = 0.0;
            rowpass<QS, RT>(A, s, r0, rows, comp, lam_s, comp, done ? 1 : 0, lam, bacc);
            MDS_T(6);
            const int m = done ? 1 : comp + 2;
            {
                double* p = A.bparts + (int64_t)par * gridDim.x * BS;
                block_sums(bacc, m, s.red, s.bc);
                if (threadIdx.x < m) p[(int64_t)blockIdx.x * BS + threadIdx.x] = s.bc[threadIdx.x];
                MDS_T(7);
                grid.sync();
                MDS_T(8);
                final_b(A, s, par, m);
                par ^= 1;
                MDS_T(9);
            }
            if (done) {
                rel = (lam != 0.0) ? sqrt(s.bc[0]) / fabs(lam) : INFINITY;
                break;
            }
            // e_f = v_f.w (bc[f]), v.w (bc[comp]), w.w (bc[comp+1]); g_f = v_f.v (tot d_f)
            it++;
            lam = s.bc[comp];
            double nw2 = s.bc[comp + 1];
            double ef[8];
            for (int f = 0; f < comp; f++) {
                ef[f] = s.bc[f];
                lam -= ef[f] * A.tot[A.NT * 64 + XS_D + f];
                nw2 -= ef[f] * ef[f];
            }
            const double nw = sqrt(fmax(nw2, 0.0));
            __syncthreads();
            if (nw == 0.0) {
                lam = 0.0;
                conv = true;
                stop = true;
                break;
            }
            const double sg = (lam / nw < 0.0) ? -1.0 : 1.0;  // sign of v_new . v
            dmax_local = 0.0;
            for (int64_t i = threadIdx.x; i < rows; i += (int)blockDim.x) {
                const int64_t g = r0 + i;
                double wi = A.w[g];
                for (int f = 0; f < comp; f++) wi -= ef[f] * A.V[(int64_t)f * n + g];
                double vn = wi / nw;
                if (sg < 0) vn = -vn;
                dmax_local = fmax(dmax_local, fabs(vn - s.us[i]));
                s.us[i] = vn;
                v[g] = vn;
            }
            __syncthreads();
            MDS_T(10);
        }
        if (stop || lam <= 0.0) break;
        if (threadIdx.x == 0) lam_s[comp] = lam;
        __syncthreads();
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            A.info[comp * 4 + 0] = lam;
            A.info[comp * 4 + 1] = (double)it;
            A.info[comp * 4 + 2] = rel;
            A.info[comp * 4 + 3] = conv ? 1.0 : 0.0;
        }
        kused = comp + 1;
    }
    // coordinates: sqrt(lambda) * v with the largest-|component| positive
    for (int c = 0; c < kused; c++) {
        const double* v = A.V + (int64_t)c * n;
        double bv = -1.0;
        int64_t bi = INT64_MAX;
        for (int64_t i = r0 + threadIdx.x; i < r0 + rows; i += (int)blockDim.x) {
            const double a = fabs(v[i]);
            if (a > bv) { bv = a; bi = i; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
        }
        __shared__ double wv[32];
        __shared__ int64_t wi[32];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if (lane == 0) { wv[warp] = bv; wi[warp] = bi; }
        __syncthreads();
        double* p = A.bparts + (int64_t)par * gridDim.x * BS;
        if (threadIdx.x == 0) {
            double vv = wv[0];
            int64_t ii = wi[0];
            for (int w = 1; w < (int)(blockDim.x >> 5); w++)
                if (wv[w] > vv || (wv[w] == vv && wi[w] < ii)) { vv = wv[w]; ii = wi[w]; }
            p[(int64_t)blockIdx.x * BS] = vv;
            p[(int64_t)blockIdx.x * BS + 1] = __longlong_as_double((long long)ii);
        }
        grid.sync();
        if (threadIdx.x == 0) {
            double vv = -1.0;
            int64_t ii = INT64_MAX;
            for (int b = 0; b < (int)gridDim.x; b++) {
                const double pv = p[(int64_t)b * BS];
                const int64_t pi = (int64_t)__double_as_longlong(p[(int64_t)b * BS + 1]);
                if (pv > vv || (pv == vv && pi < ii)) { vv = pv; ii = pi; }
            }
            bc[0] = v[ii] < 0.0 ? -1.0 : 1.0;
        }
        par ^= 1;
        __syncthreads();
        const double sl = sqrt(lam_s[c]) * bc[0];
        for (int64_t i = r0 + threadIdx.x; i < r0 + rows; i += (int)blockDim.x) A.coords[i * A.k + c] = sl * v[i];
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *A.k_used = kused;
}

// ------------------------------------------------------------------- host
struct Layout {
    int64_t V, w, sparts, tot, cst, bparts, sc, tc, ci, di, bytes;
};

static int grid_size() { return sm_count(); }

static void shape(MdsArgs& A)
{
    A.TP = (A.r + 1 + 7) / 8;
    A.NT = A.TP * (A.TP + 1) / 2;
    A.PE = A.NT * 64 + XA;
}

static int rt_inst(int r)
{
    const int rt = (r + 7) / 8;
    if (rt <= 1) return 1;
    if (rt <= 2) return 2;
    if (rt <= 4) return 4;
    if (rt <= 8) return 8;
    if (rt <= 12) return 12;
    if (rt <= 16) return 16;
    return 24;
}

static Layout mds_layout(int64_t n, int r, int k)
{
    MdsArgs A{};
    A.r = r;
    shape(A);
    const int G = grid_size();
    Layout L;
    int64_t o = 0;
    auto take = [&](int64_t count) {
        const int64_t at = o;
        o += ((count * 8 + 255) / 256) * 256;
        return at;
    };
    L.V = take((int64_t)k * n);
    L.w = take(n);
    L.sparts = take((int64_t)G * A.PE);
    L.tot = take(A.PE);
    L.cst = take((int64_t)A.NT * 64);
    L.bparts = take(2LL * G * BS);
    const int RP = 8 * rt_inst(r);
    L.sc = take((int64_t)RP * (RP + 4));
    L.tc = take(RP + 4);
    L.ci = take(n);
    L.di = take(n);
    L.bytes = o;
    return L;
}


static size_t plan_smem(MdsArgs& A)
{
    const int r = A.r, RP = 8 * rt_inst(r);
    const bool sms = RP <= SMS_MAXRP;
    A.rpb = (A.n + grid_size() - 1) / grid_size();
    const size_t fixed =
        ((sms ? (size_t)RP * (RP + 4) : 0) + RP + (size_t)pad16(A.rpb) + r) * 8;
    const size_t f64 = (size_t)pad16(A.rpb) * ldq_of(RP) * 8;
    const size_t i8 = ((size_t)pad16(A.rpb) * RP + 7) / 8 * 8;
    A.r8 = RP;
    // int8-resident slice with the all-warp DMMA reduction and the
    // register-resident row pass (r <= 32): preferred whenever the codes exist
    const bool fast = A.codes && sms && RP <= 32 && !getenv("RFXC_MDS_F64");
    const int RTf = RP / 8, NV = RTf * (RTf + 1) + RTf + 1;
    const size_t fbuf = (size_t)(MDS_I8F_THREADS / 32) * NV * 32 * 8;
    if (fast && fixed + i8 + fbuf <= SMEM_BUDGET) {
        A.qs = QS_I8;
        return fixed + i8 + fbuf;
    }
    if (fixed + f64 <= SMEM_BUDGET) {
        A.qs = QS_F64;
        return fixed + f64;
    }
    if (A.codes && fixed + i8 + (RP <= 32 ? fbuf : 0) <= SMEM_BUDGET) {  // (r <= 32: fast path)
        A.qs = QS_I8;
        return fixed + i8 + (RP <= 32 ? fbuf : 0);
    }
    A.qs = QS_GLOBAL;
    return fixed;
}

template <int QS, int RT>
static int launch_q(MdsArgs& A, size_t smem, cudaStream_t st)
{
    // 16 warps while the row-pass accumulators fit 128 registers, else 8; the
    // int8 fast path keeps S fragments in registers: 8 warps
    constexpr int NTH = (QS == QS_I8 && RT <= 4) ? MDS_I8F_THREADS : (RT <= 8 ? 512 : 256);
    auto kern = mds_kernel<QS, RT, NTH>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)std::max<size_t>(smem, 1));
    if (e != cudaSuccess) return fail(RFXC_ECUDA, "mds attr: %s", cudaGetErrorString(e));
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NTH, smem);
    if (occ < 1) return fail(RFXC_ERUNTIME, "mds: kernel does not fit an SM (r=%d)", A.r);
    void* args[] = {&A};
    e = cudaLaunchCooperativeKernel((const void*)kern, dim3(grid_size()), dim3(NTH), args, smem, st);
    if (e != cudaSuccess) return fail(RFXC_ECUDA, "mds launch: %s", cudaGetErrorString(e));
    return check_launch("mds");
}

template <int RT>
static int launch_rt(MdsArgs& A, size_t smem, cudaStream_t st)
{
    if (A.qs == QS_F64) return launch_q<QS_F64, RT>(A, smem, st);
    if (A.qs == QS_I8) return launch_q<QS_I8, RT>(A, smem, st);
    return launch_q<QS_GLOBAL, RT>(A, smem, st);
}

static int launch_mds(MdsArgs& A, cudaStream_t st)
{
    if (A.r > 8 * MAXRT) return fail(RFXC_EDATA, "mds: rank %d above %d", A.r, 8 * MAXRT);
    const size_t smem = plan_smem(A);
    if (smem > SMEM_BUDGET)
        return fail(RFXC_EDATA, "mds: n=%lld r=%d too large for one GPU", (long long)A.n, A.r);
    switch (rt_inst(A.r)) {
        case 1: return launch_rt<1>(A, smem, st);
        case 2: return launch_rt<2>(A, smem, st);
        case 4: return launch_rt<4>(A, smem, st);
        case 8: return launch_rt<8>(A, smem, st);
        case 12: return launch_rt<12>(A, smem, st);
        case 16: return launch_rt<16>(A, smem, st);
        default: return launch_rt<24>(A, smem, st);
    }
}

static void bind(MdsArgs& A, const Layout& L, void* d_work)
{
    char* base = static_cast<char*>(d_work);
    A.V = reinterpret_cast<double*>(base + L.V);
    A.w = reinterpret_cast<double*>(base + L.w);
    A.sparts = reinterpret_cast<double*>(base + L.sparts);
    A.tot = reinterpret_cast<double*>(base + L.tot);
    A.cst = reinterpret_cast<double*>(base + L.cst);
    A.bparts = reinterpret_cast<double*>(base + L.bparts);
    A.sc = reinterpret_cast<double*>(base + L.sc);
    A.tc = reinterpret_cast<double*>(base + L.tc);
    A.ci = reinterpret_cast<double*>(base + L.ci);
    A.di = reinterpret_cast<double*>(base + L.di);
    A.RPs = 8 * rt_inst(A.r);
}

}  // namespace rfxc

using namespace rfxc;

extern "C" int64_t rfxc_mds_work_bytes(int64_t n, int32_t r, int32_t k)
{
    return mds_layout(n, r, std::max(k, 1)).bytes;
}

extern "C" int rfxc_mds_power(const double* d_dq, const int8_t* d_codes, const double* d_scales,
                              int64_t n, int32_t r, double pmax, const double* d_pmax, int32_t k,
                              int32_t max_iterations, double tol, int64_t seed, double* d_coords,
                              double* d_info, int32_t* d_k_used, void* d_work, void* stream)
{
    if (n < 1 || r < 1 || k < 1 || k > 8 || max_iterations < 1)
        return fail(RFXC_EDATA, "mds_power: bad arguments");
    cudaStream_t st = as_stream(stream);
    MdsArgs A{};
    A.dq = d_dq;
    A.codes = d_codes;
    A.scales = d_scales;
    A.n = n;
    A.r = r;
    A.pmax = pmax;
    A.pmax_dev = d_pmax;
    A.k = k;
    A.max_it = max_iterations;
    A.tol = tol;
    A.mode = 0;
    shape(A);
    bind(A, mds_layout(n, r, k), d_work);
    A.coords = d_coords;
    A.info = d_info;
    A.k_used = d_k_used;
    // start vectors Pcg32(seed + c, SEQ_POWER).normals(n)  (mds.py:210-211)
    for (int c = 0; c < k; c++) {
        const int rc = rfxc_normals(seed + c, 5, n, A.V + (int64_t)c * n, stream);
        if (rc) return rc;
    }
    cudaMemsetAsync(d_info, 0, (size_t)k * 4 * 8, st);
    cudaMemsetAsync(d_coords, 0, (size_t)n * k * 8, st);
    A.timing = nullptr;
    if (!getenv("RFXC_MDS_TIMING")) return launch_mds(A, st);
    cudaMalloc(&A.timing, 16 * 8);
    cudaMemsetAsync(A.timing, 0, 16 * 8, st);
    int rc = launch_mds(A, st);
    unsigned long long h[16];
    cudaMemcpy(h, A.timing, sizeof h, cudaMemcpyDeviceToHost);
    cudaFree(A.timing);
    const char* names[11] = {"other", "spass", "extras", "syncA1", "finalA", "syncA2", "rowpass",
                             "bparts", "syncB", "finalB", "update"};
    for (int i = 0; i < 11; i++) fprintf(stderr, "[mds] %-8s %9.3f ms\n", names[i], h[i] * 1e-6);
    fprintf(stderr, "[mds] rowpass main loop (CTA 0, thread 0) %9.3f ms\n", h[12] * 1e-6);
    return rc;
}

extern "C" int rfxc_gram_matvec(const double* d_dq, int64_t n, int32_t r, double pmax,
                                const double* d_v, double* d_w, void* d_work, void* stream)
{
    if (n < 1 || r < 1) return fail(RFXC_EDATA, "gram_matvec: bad arguments");
    cudaStream_t st = as_stream(stream);
    MdsArgs A{};
    A.dq = d_dq;
    A.n = n;
    A.r = r;
    A.pmax = pmax;
    A.k = 1;
    A.max_it = 1;
    A.tol = 1.0;
    A.mode = 1;
    shape(A);
    bind(A, mds_layout(n, r, 1), d_work);
    A.w = d_w;
    const cudaError_t e = cudaMemcpyAsync(A.V, d_v, (size_t)n * 8, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return fail(RFXC_ECUDA, "gram_matvec copy: %s", cudaGetErrorString(e));
    return launch_mds(A, st);
}
