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
// the UNclamped P = Q Q^T (mds.py:177-179).  With Q' = [Q | 1] the single
// reduction S' = Q'^T diag(u) Q' holds S = Q^T diag(u) Q (so that
// (P o P)u_i = q_i^T S q_i — the Khatri-Rao identity of mds.py:147-152
// without the n x r^2 expansion), t = Q^T u (P u_i = q_i . t) and sum(u).
// mean(z) follows in closed form from the constants Q^T 1 and Q^T Q, so a
// Gram matvec costs one S' pass + one row pass and two grid barriers.
//
// Layout: one CTA per SM (cooperative launch); CTA c owns a contiguous row
// slice and keeps that slice of the factor resident in shared memory for the
// whole run (f64 rows, or int8 codes x per-column scales for large n, odd
// row stride so lane-per-row reads are conflict-free; global memory is the
// fallback).  The kernel is templated on that storage so the inner loops are
// branch-free.  Every reduction has a fixed order (register tiles -> fixed
// smem combine -> fixed block order), so results are bit-reproducible and
// every stopping decision is identical in every CTA.  The work is FP64-FMA
// bound: per matvec and row, ~r(r+1)/2 FMAs in each of the two passes.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace rfxc {

constexpr int MT = 512;             // threads per CTA
constexpr int MW = MT / 32;         // warps per CTA
constexpr int SLOTS = 24;           // small-reduction slots per CTA
constexpr int SMEM_BUDGET = 220 * 1024;
constexpr int RMAX_REG = 32;        // rows held in registers for r <= 32

enum { QS_F64 = 0, QS_I8 = 1, QS_GLOBAL = 2 };

struct MdsArgs {
    const double* dq;       // (n, r) f64 dequantised factor (global)
    const int8_t* codes;    // (n, r) int8 codes (QS_I8) or null
    const double* scales;   // (r) per-column scales (QS_I8)
    int64_t n;
    int r;
    double pmax;
    int k;
    int max_it;
    double tol;
    int mode;               // 0: MDS, 1: one gram_matvec of V[0] into w
    int qs;                 // QS_* storage of the factor slice
    int64_t rpb;            // rows per CTA
    double* V;              // k x n: start vectors in, found vectors out
    double* w;              // n
    double* parts;          // 2 x grid x SLOTS (small reductions, double-buffered)
    double* sparts;         // grid x (E + 8) (S' partials + deflation dots)
    double* tot;            // E + 8: totals of the current matvec
    double* cst;            // E: constants Q'^T Q' (G = Q^T Q, c = Q^T 1, n)
    double* coords;         // n x k
    double* info;           // k x 4
    int32_t* k_used;
};

struct Ctx {
    cg::grid_group grid;
    int64_t r0, r1;
    int parity;
    double* red;     // >= 32
    double* bcast;   // SLOTS
};

__host__ __device__ __forceinline__ int ntile(int r) { return (r + 1 + 3) / 4; }
__host__ __device__ __forceinline__ int nentry(int r)
{
    const int t = ntile(r);
    return 16 * t * (t + 1) / 2;
}
__host__ __device__ __forceinline__ int tile_index(int ta, int tb, int T)
{
    return ta * T - ta * (ta - 1) / 2 + (tb - ta);  // ta <= tb
}

// ---------------------------------------------------------------- reductions
// Sum m (<= SLOTS) per-thread values over the grid; every thread gets totals.
__device__ void grid_sum(Ctx& C, const MdsArgs& A, double* v, int m)
{
    double* parts = A.parts + (int64_t)C.parity * gridDim.x * SLOTS;
    C.parity ^= 1;
    for (int j = 0; j < m; j++) {
        const double s = block_sum(v[j], C.red);
        if (threadIdx.x == 0) parts[blockIdx.x * SLOTS + j] = s;
    }
    C.grid.sync();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j = warp; j < m; j += MW) {  // one warp per slot, fixed order
        double s = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) s += parts[b * SLOTS + j];
        s = warp_sum(s);
        if (lane == 0) C.bcast[j] = s;
    }
    __syncthreads();
    for (int j = 0; j < m; j++) v[j] = C.bcast[j];
    __syncthreads();
}

// max of `mx` and sum of `sm` in one barrier
__device__ void grid_max_sum(Ctx& C, const MdsArgs& A, double& mx, double& sm)
{
    double* parts = A.parts + (int64_t)C.parity * gridDim.x * SLOTS;
    C.parity ^= 1;
    const double bm = block_max(mx, C.red);
    const double bs = block_sum(sm, C.red);
    if (threadIdx.x == 0) {
        parts[blockIdx.x * SLOTS] = bm;
        parts[blockIdx.x * SLOTS + 1] = bs;
    }
    C.grid.sync();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp < 2) {
        double s = warp == 0 ? -INFINITY : 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) {
            const double x = parts[b * SLOTS + warp];
            s = warp == 0 ? fmax(s, x) : s + x;
        }
        s = warp == 0 ? warp_max(s) : warp_sum(s);
        if (lane == 0) C.bcast[warp] = s;
    }
    __syncthreads();
    mx = C.bcast[0];
    sm = C.bcast[1];
    __syncthreads();
}

// (max |x|, first index) over the grid
__device__ int64_t grid_argmax_abs(Ctx& C, const MdsArgs& A, const double* x)
{
    double bv = -1.0;
    int64_t bi = INT64_MAX;
    for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += blockDim.x) {
        const double a = fabs(x[i]);
        if (a > bv) { bv = a; bi = i; }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    __shared__ double wv[MW];
    __shared__ int64_t wi[MW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) { wv[warp] = bv; wi[warp] = bi; }
    __syncthreads();
    double* parts = A.parts + (int64_t)C.parity * gridDim.x * SLOTS;
    C.parity ^= 1;
    if (threadIdx.x == 0) {
        double v = wv[0];
        int64_t ii = wi[0];
        for (int w = 1; w < MW; w++)
            if (wv[w] > v || (wv[w] == v && wi[w] < ii)) { v = wv[w]; ii = wi[w]; }
        parts[blockIdx.x * SLOTS] = v;
        parts[blockIdx.x * SLOTS + 1] = __longlong_as_double((long long)ii);
    }
    C.grid.sync();
    if (threadIdx.x == 0) {
        double v = -1.0;
        int64_t ii = INT64_MAX;
        for (int b = 0; b < (int)gridDim.x; b++) {
            const double pv = parts[b * SLOTS];
            const int64_t pi = (int64_t)__double_as_longlong(parts[b * SLOTS + 1]);
            if (pv > v || (pv == v && pi < ii)) { v = pv; ii = pi; }
        }
        C.bcast[0] = __longlong_as_double((long long)ii);
    }
    __syncthreads();
    const int64_t out = (int64_t)__double_as_longlong(C.bcast[0]);
    __syncthreads();
    return out;
}

// ------------------------------------------------------------- factor rows
// Factor slice accessor; QSM fixed at compile time (no per-element branch).
template <int QSM>
struct Rows {
    int r;
    int ld;              // row stride (odd for the shared-memory layouts)
    const double* f64;   // smem slice (QS_F64) or global dq (QS_GLOBAL)
    const int8_t* i8;    // smem codes (QS_I8)
    const double* sc;    // smem scales (QS_I8)
    int64_t base;        // first global row of the slice (QS_GLOBAL)

    __device__ __forceinline__ double q(int64_t row, int col) const  // col < r
    {
        if (QSM == QS_I8) return (double)i8[row * ld + col] * sc[col];
        if (QSM == QS_F64) return f64[row * ld + col];
        return __ldg(f64 + (base + row) * r + col);
    }
};

// S' partial of this CTA: sum over slice rows of u_i q'_i q'_i^T (q' = [q | 1])
// as 4x4 register tiles of the upper triangle; row groups split the slice
// and are combined in a fixed order.  Writes nentry(r) values to `out`.
template <int QSM>
__device__ __forceinline__ void tile_rows(const Rows<QSM>& Q, int ta, int tb, int r,
                                          const double* us, int64_t i0, int64_t rows,
                                          int64_t step, double* acc)
{
    bool va[4], vb[4];
#pragma unroll
    for (int x = 0; x < 4; x++) {
        va[x] = 4 * ta + x < r;
        vb[x] = 4 * tb + x < r;
    }
    for (int64_t i = i0; i < rows; i += step) {
        const double u = us[i];
        double qa[4], qb[4];
#pragma unroll
        for (int x = 0; x < 4; x++) {
            const int ca = 4 * ta + x, cb = 4 * tb + x;
            qa[x] = u * (va[x] ? Q.q(i, ca) : (ca == r ? 1.0 : 0.0));
            qb[x] = vb[x] ? Q.q(i, cb) : (cb == r ? 1.0 : 0.0);
        }
#pragma unroll
        for (int x = 0; x < 4; x++)
#pragma unroll
            for (int y = 0; y < 4; y++) acc[4 * x + y] += qa[x] * qb[y];
    }
}

template <int QSM>
__device__ void spass(const Rows<QSM>& Q, const double* us, int64_t rows, double* out,
                      double* scratch)
{
    const int r = Q.r, T = ntile(r);
    const int tiles = T * (T + 1) / 2;
    const int tid = threadIdx.x;
    double acc[16];
    if (tiles > MT) {  // large r: every thread owns whole tiles, all rows
        for (int tile = tid; tile < tiles; tile += MT) {
            int ta = 0, rem = tile;
            while (rem >= T - ta) { rem -= T - ta; ta++; }
#pragma unroll
            for (int e = 0; e < 16; e++) acc[e] = 0.0;
            tile_rows(Q, ta, ta + rem, r, us, 0, rows, 1, acc);
#pragma unroll
            for (int e = 0; e < 16; e++) out[tile * 16 + e] = acc[e];
        }
        __syncthreads();
        return;
    }
    const int groups = MT / tiles;
    const int g = tid / tiles, tile = tid % tiles;
#pragma unroll
    for (int e = 0; e < 16; e++) acc[e] = 0.0;
    int ta = 0, rem = tile;
    while (rem >= T - ta) { rem -= T - ta; ta++; }
    for (int tt = tid; tt < tiles * 16; tt += MT) scratch[tt] = 0.0;
    if (g < groups) tile_rows(Q, ta, ta + rem, r, us, g, rows, groups, acc);
    __syncthreads();
    for (int gg = 0; gg < groups; gg++) {  // fixed combine order
        if (g == gg) {
#pragma unroll
            for (int e = 0; e < 16; e++) scratch[tile * 16 + e] += acc[e];
        }
        __syncthreads();
    }
    for (int e = tid; e < tiles * 16; e += MT) out[e] = scratch[e];
    __syncthreads();
}

// S'[a][b] from the tiled upper triangle (any a, b)
__device__ __forceinline__ double sprime(const double* tot, int a, int b, int T)
{
    if (a > b) { const int s = a; a = b; b = s; }
    const int ta = a >> 2, tb = b >> 2, x = a & 3, y = b & 3;
    return tot[16 * tile_index(ta, tb, T) + 4 * x + y];
}

// Row pass, lane per row with the row in registers (r <= R): returns
// pu = q.t and ppu = q^T S q for slice row i.  S is symmetric (R x R,
// zero-padded, broadcast from shared memory), t = S'[:, r].
template <int QSM, int R>
__device__ __forceinline__ void row_terms_reg(const Rows<QSM>& Q, int64_t i, bool valid,
                                              const double* Sp, const double* tv, double& pu,
                                              double& ppu)
{
    double q[R];
#pragma unroll
    for (int b = 0; b < R; b++) q[b] = (valid && b < Q.r) ? Q.q(i, b) : 0.0;
    pu = 0.0;
    ppu = 0.0;
#pragma unroll
    for (int a = 0; a < R; a++) {
        double acc = 0.0;
#pragma unroll
        for (int b = a + 1; b < R; b++) acc += Sp[a * R + b] * q[b];
        ppu += q[a] * (Sp[a * R + a] * q[a] + 2.0 * acc);
        pu += q[a] * tv[a];
    }
}

// y = G x - sum_{f<nf} lam_f (v_f . x) v_f   (deflated_matvec, mds.py:203-207)
// sx: sum of x over all rows.  Two grid barriers.
template <int QSM>
__device__ void matvec(Ctx& C, const MdsArgs& A, const Rows<QSM>& Q, const double* x, double sx,
                       double* y, int nf, const double* lam, double* Sp, double* tv, double* us,
                       double* scratch)
{
    const int r = A.r, T = ntile(r), E = nentry(r);
    const int64_t n = A.n, rows = C.r1 - C.r0;
    const double mean = sx / (double)n;
    for (int64_t i = threadIdx.x; i < rows; i += MT) us[i] = x[C.r0 + i] - mean;
    double dl[8];
    for (int f = 0; f < nf; f++) dl[f] = 0.0;
    for (int64_t i = threadIdx.x; i < rows; i += MT)
        for (int f = 0; f < nf; f++) dl[f] += A.V[(int64_t)f * n + C.r0 + i] * x[C.r0 + i];
    __syncthreads();
    double* out = A.sparts + (int64_t)blockIdx.x * (E + 8);
    spass(Q, us, rows, out, scratch);
    for (int f = 0; f < nf; f++) {
        const double s = block_sum(dl[f], C.red);
        if (threadIdx.x == 0) out[E + f] = s;
    }
    C.grid.sync();
    {  // distributed final reduce: one warp per entry, lanes over blocks
        const int lane = threadIdx.x & 31;
        const int gw = blockIdx.x * MW + (threadIdx.x >> 5), nw = gridDim.x * MW;
        for (int e = gw; e < E + nf; e += nw) {
            double s = 0.0;
            for (int b = lane; b < (int)gridDim.x; b += 32)
                s += A.sparts[(int64_t)b * (E + 8) + e];
            s = warp_sum(s);
            if (lane == 0) A.tot[e] = s;
        }
    }
    C.grid.sync();
    // r <= 32: padded symmetric S (RP x RP) and t in shared memory; larger r
    // reads S' straight from the (L2-resident) totals
    const bool small = r <= RMAX_REG;
    const int RP = r <= 16 ? 16 : RMAX_REG;
    if (small) {
        for (int e = threadIdx.x; e < RP * RP; e += MT) {
            const int a = e / RP, b = e % RP;
            Sp[e] = (a < r && b < r) ? sprime(A.tot, a, b, T) : 0.0;
        }
        for (int a = threadIdx.x; a < RP; a += MT) tv[a] = a < r ? sprime(A.tot, a, r, T) : 0.0;
    }
    __syncthreads();
    const double su = sprime(A.tot, r, r, T);
    const double pm = A.pmax;
    double ct, sgm;  // c.t and <S, G> -> closed-form mean of z
    {
        double a = 0.0, b = 0.0;
        for (int e = threadIdx.x; e < r * r; e += MT)
            b += sprime(A.tot, e / r, e % r, T) * sprime(A.cst, e / r, e % r, T);
        for (int aa = threadIdx.x; aa < r; aa += MT)
            a += sprime(A.cst, aa, r, T) * sprime(A.tot, aa, r, T);
        ct = block_sum(a, C.red);
        sgm = block_sum(b, C.red);
    }
    const double mz = (pm * pm) * su - 2.0 * pm * ct / (double)n + sgm / (double)n;
    const double* d = A.tot + E;
    for (int64_t i0 = 0; i0 < rows; i0 += MT) {
        const int64_t i = i0 + threadIdx.x;
        const bool valid = i < rows;
        double pu, ppu;
        if (r <= 16) {
            row_terms_reg<QSM, 16>(Q, i, valid, Sp, tv, pu, ppu);
        } else if (r <= RMAX_REG) {
            row_terms_reg<QSM, RMAX_REG>(Q, i, valid, Sp, tv, pu, ppu);
        } else {  // generic: S' from the totals (L1/L2), row from the slice
            pu = 0.0;
            ppu = 0.0;
            if (valid) {
                for (int a = 0; a < r; a++) {
                    const double qa = Q.q(i, a);
                    double acc = 0.0;
                    for (int b = a + 1; b < r; b++) acc += sprime(A.tot, a, b, T) * Q.q(i, b);
                    ppu += qa * (sprime(A.tot, a, a, T) * qa + 2.0 * acc);
                    pu += qa * sprime(A.tot, a, r, T);
                }
            }
        }
        if (valid) {
            const double zi = (pm * pm) * su - 2.0 * pm * pu + ppu;
            double yi = -0.5 * (zi - mz);
            for (int f = 0; f < nf; f++) yi -= lam[f] * d[f] * A.V[(int64_t)f * n + C.r0 + i];
            y[C.r0 + i] = yi;
        }
    }
    __syncthreads();
}

template <int QSM>
__global__ void __launch_bounds__(MT, 1) mds_kernel(MdsArgs A)
{
    extern __shared__ __align__(16) unsigned char msm[];
    __shared__ double red[32];
    __shared__ double bcast[SLOTS];
    __shared__ double lam_s[8];
    const int r = A.r, T = ntile(r), E = nentry(r);
    const int RP = r <= 16 ? 16 : (r <= RMAX_REG ? RMAX_REG : 0);
    const int SCR = T * (T + 1) / 2 <= MT ? 16 * T * (T + 1) / 2 : 0;
    Ctx C{cg::this_grid(), 0, 0, 0, red, bcast};
    const int64_t n = A.n;
    C.r0 = min64(n, blockIdx.x * A.rpb);
    C.r1 = min64(n, C.r0 + A.rpb);
    const int64_t rows = C.r1 - C.r0;

    // shared memory: [S RPxRP] [t RP] [tile scratch] [u rpb] [factor slice]
    double* Sp = reinterpret_cast<double*>(msm);
    double* tv = Sp + RP * RP;
    double* scratch = tv + RP;
    double* us = scratch + SCR;
    unsigned char* qbase = reinterpret_cast<unsigned char*>(us + A.rpb);
    Rows<QSM> Q{r, r | 1, nullptr, nullptr, nullptr, C.r0};
    if (QSM == QS_F64) {
        double* qs = reinterpret_cast<double*>(qbase);
        for (int64_t e = threadIdx.x; e < rows * r; e += MT)
            qs[(e / r) * Q.ld + e % r] = A.dq[C.r0 * r + e];
        Q.f64 = qs;
    } else if (QSM == QS_I8) {
        double* sc = reinterpret_cast<double*>(qbase);
        int8_t* qs = reinterpret_cast<int8_t*>(sc + r);
        for (int e = threadIdx.x; e < r; e += MT) sc[e] = A.scales[e];
        for (int64_t e = threadIdx.x; e < rows * r; e += MT)
            qs[(e / r) * Q.ld + e % r] = A.codes[C.r0 * r + e];
        Q.i8 = qs;
        Q.sc = sc;
    } else {
        Q.f64 = A.dq;
    }
    __syncthreads();

    {  // constants Q'^T Q' (G = Q^T Q, c = Q^T 1) with u = 1
        for (int64_t i = threadIdx.x; i < rows; i += MT) us[i] = 1.0;
        __syncthreads();
        double* out = A.sparts + (int64_t)blockIdx.x * (E + 8);
        spass(Q, us, rows, out, scratch);
        C.grid.sync();
        const int lane = threadIdx.x & 31;
        const int gw = blockIdx.x * MW + (threadIdx.x >> 5), nw = gridDim.x * MW;
        for (int e = gw; e < E; e += nw) {
            double s = 0.0;
            for (int b = lane; b < (int)gridDim.x; b += 32)
                s += A.sparts[(int64_t)b * (E + 8) + e];
            s = warp_sum(s);
            if (lane == 0) A.cst[e] = s;
        }
        C.grid.sync();
    }

    if (A.mode == 1) {
        double s[1] = {0.0};
        for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += MT) s[0] += A.V[i];
        grid_sum(C, A, s, 1);
        matvec(C, A, Q, A.V, s[0], A.w, 0, lam_s, Sp, tv, us, scratch);
        return;
    }

    int kused = 0;
    for (int comp = 0; comp < A.k; comp++) {
        double* v = A.V + (int64_t)comp * n;
        for (int f = 0; f < comp; f++) {  // start vector: sequential Gram-Schmidt
            const double* vf = A.V + (int64_t)f * n;
            double dd[1] = {0.0};
            for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += MT) dd[0] += vf[i] * v[i];
            grid_sum(C, A, dd, 1);
            for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += MT) v[i] -= dd[0] * vf[i];
            __syncthreads();
        }
        double nn[1] = {0.0};
        for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += MT) nn[0] += v[i] * v[i];
        grid_sum(C, A, nn, 1);
        const double nv = sqrt(nn[0]);
        if (nv == 0.0) break;
        double sv[1] = {0.0};
        for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += MT) {
            v[i] /= nv;
            sv[0] += v[i];
        }
        grid_sum(C, A, sv, 1);
        double sumv = sv[0];

        double lam = 0.0;
        bool conv = false;
        int it = 0;
        for (it = 1; it <= A.max_it; it++) {
            matvec(C, A, Q, v, sumv, A.w, comp, lam_s, Sp, tv, us, scratch);
            // all projections in one reduction: e_f = v_f.w, g_f = v_f.v, v.w, w.w
            double dots[2 * 8 + 2];
            const int m = 2 * comp + 2;
            for (int j = 0; j < m; j++) dots[j] = 0.0;
            for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += MT) {
                const double wi = A.w[i], vi = v[i];
                for (int f = 0; f < comp; f++) {
                    const double vf = A.V[(int64_t)f * n + i];
                    dots[2 * f] += vf * wi;
                    dots[2 * f + 1] += vf * vi;
                }
                dots[2 * comp] += vi * wi;
                dots[2 * comp + 1] += wi * wi;
            }
            grid_sum(C, A, dots, m);
            // w' = w - sum_f e_f v_f (orthonormal v_f): v.w' and |w'|^2 in closed form
            lam = dots[2 * comp];
            double nw2 = dots[2 * comp + 1];
            for (int f = 0; f < comp; f++) {
                lam -= dots[2 * f] * dots[2 * f + 1];
                nw2 -= dots[2 * f] * dots[2 * f];
            }
            const double nw = sqrt(fmax(nw2, 0.0));
            if (nw == 0.0) {
                lam = 0.0;
                conv = true;
                break;
            }
            const double sg = (lam / nw < 0.0) ? -1.0 : 1.0;  // sign of v_new . v
            double dmax = 0.0, snew = 0.0;
            for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += MT) {
                double wi = A.w[i];
                for (int f = 0; f < comp; f++) wi -= dots[2 * f] * A.V[(int64_t)f * n + i];
                double vn = wi / nw;
                if (sg < 0) vn = -vn;
                dmax = fmax(dmax, fabs(vn - v[i]));
                v[i] = vn;
                snew += vn;
            }
            grid_max_sum(C, A, dmax, snew);
            sumv = snew;
            if (dmax < A.tol) {
                conv = true;
                break;
            }
        }
        if (it > A.max_it) it = A.max_it;
        // residual |deflated_matvec(v) - lam v| / |lam|  (mds.py:241-242)
        matvec(C, A, Q, v, sumv, A.w, comp, lam_s, Sp, tv, us, scratch);
        double rr[1] = {0.0};
        for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += MT) {
            const double e = A.w[i] - lam * v[i];
            rr[0] += e * e;
        }
        grid_sum(C, A, rr, 1);
        const double rel = (lam != 0.0) ? sqrt(rr[0]) / fabs(lam) : INFINITY;
        if (lam <= 0.0) break;
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
    for (int c = 0; c < kused; c++) {
        const double* v = A.V + (int64_t)c * n;
        const int64_t idx = grid_argmax_abs(C, A, v);
        const double sgn = v[idx] < 0.0 ? -1.0 : 1.0;
        const double sl = sqrt(lam_s[c]);
        for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += MT)
            A.coords[i * A.k + c] = sl * (sgn < 0 ? -v[i] : v[i]);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *A.k_used = kused;
}

// ------------------------------------------------------------------- host
struct Layout {
    int64_t V, w, parts, sparts, tot, cst, bytes;
};

static int grid_size() { return sm_count(); }

static Layout mds_layout(int64_t n, int r, int k)
{
    const int G = grid_size();
    const int64_t E = nentry(r);
    Layout L;
    int64_t o = 0;
    auto take = [&](int64_t count) {
        const int64_t at = o;
        o += ((count * 8 + 255) / 256) * 256;
        return at;
    };
    L.V = take((int64_t)k * n);
    L.w = take(n);
    L.parts = take(2LL * G * SLOTS);
    L.sparts = take((int64_t)G * (E + 8));
    L.tot = take(E + 8);
    L.cst = take(E + 8);
    L.bytes = o;
    return L;
}

// choose the factor storage; returns the dynamic shared memory size
static size_t plan_smem(MdsArgs& A)
{
    const int r = A.r;
    const int64_t T = ntile(r);
    const int RP = r <= 16 ? 16 : (r <= RMAX_REG ? RMAX_REG : 0);
    const int64_t SCR = T * (T + 1) / 2 <= MT ? 16 * T * (T + 1) / 2 : 0;
    const int ld = r | 1;
    A.rpb = (A.n + grid_size() - 1) / grid_size();
    const size_t fixed = ((size_t)RP * RP + RP + SCR + (size_t)A.rpb) * 8;
    const size_t f64_rows = (size_t)A.rpb * ld * 8;
    const size_t i8_rows = (size_t)r * 8 + (size_t)A.rpb * ld;
    if (fixed + f64_rows <= SMEM_BUDGET) {
        A.qs = QS_F64;
        return fixed + f64_rows;
    }
    if (A.codes && fixed + i8_rows <= SMEM_BUDGET) {
        A.qs = QS_I8;
        return fixed + i8_rows;
    }
    A.qs = QS_GLOBAL;
    return fixed;
}

template <int QSM>
static int launch_q(MdsArgs& A, size_t smem, cudaStream_t st)
{
    auto kern = mds_kernel<QSM>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)std::max<size_t>(smem, 1));
    if (e != cudaSuccess) return fail(RFXC_ECUDA, "mds attr: %s", cudaGetErrorString(e));
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, MT, smem);
    if (occ < 1) return fail(RFXC_ERUNTIME, "mds: kernel does not fit an SM (r=%d)", A.r);
    void* args[] = {&A};
    e = cudaLaunchCooperativeKernel((const void*)kern, dim3(grid_size()), dim3(MT), args, smem,
                                    st);
    if (e != cudaSuccess) return fail(RFXC_ECUDA, "mds launch: %s", cudaGetErrorString(e));
    return check_launch("mds");
}

static int launch_mds(MdsArgs& A, cudaStream_t st)
{
    const size_t smem = plan_smem(A);
    if (smem > SMEM_BUDGET)
        return fail(RFXC_EDATA, "mds: n=%lld r=%d too large for one GPU", (long long)A.n, A.r);
    if (A.qs == QS_F64) return launch_q<QS_F64>(A, smem, st);
    if (A.qs == QS_I8) return launch_q<QS_I8>(A, smem, st);
    return launch_q<QS_GLOBAL>(A, smem, st);
}

static void bind(MdsArgs& A, const Layout& L, void* d_work)
{
    char* base = static_cast<char*>(d_work);
    A.V = reinterpret_cast<double*>(base + L.V);
    A.w = reinterpret_cast<double*>(base + L.w);
    A.parts = reinterpret_cast<double*>(base + L.parts);
    A.sparts = reinterpret_cast<double*>(base + L.sparts);
    A.tot = reinterpret_cast<double*>(base + L.tot);
    A.cst = reinterpret_cast<double*>(base + L.cst);
}

}  // namespace rfxc

using namespace rfxc;

extern "C" int64_t rfxc_mds_work_bytes(int64_t n, int32_t r, int32_t k)
{
    return mds_layout(n, r, std::max(k, 1)).bytes;
}

extern "C" int rfxc_mds_power(const double* d_dq, const int8_t* d_codes, const double* d_scales,
                              int64_t n, int32_t r, double pmax, int32_t k,
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
    A.k = k;
    A.max_it = max_iterations;
    A.tol = tol;
    A.mode = 0;
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
    return launch_mds(A, st);
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
    bind(A, mds_layout(n, r, 1), d_work);
    A.w = d_w;
    const cudaError_t e = cudaMemcpyAsync(A.V, d_v, (size_t)n * 8, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return fail(RFXC_ECUDA, "gram_matvec copy: %s", cudaGetErrorString(e));
    return launch_mds(A, st);
}
