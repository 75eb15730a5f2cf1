// mds.cu — K8/K9: factor-space MDS power iteration in one persistent kernel.
//
// Reference: gram_matvec + _hadamard_square_matvec (mds.py:140-181) and
// mds_lowrank (mds.py:184-268): for each of k eigenpairs, start from
// Pcg32(seed + c, SEQ_POWER).normals(n), orthogonalise against the found
// vectors, iterate w = G v - sum_f lambda_f (v_f.v) v_f, project out the
// found vectors (sequential Gram-Schmidt), lambda = v.w, v <- w/|w| with the
// sign aligned to the previous iterate, stop when max|v_new - v| < tol or at
// the iteration cap; relative residual |G v - lambda v| / |lambda|; stop at
// lambda <= 0.  Coordinates sqrt(lambda) * v with the largest-|component|
// positive (mds.py:83-86, :257-261).
//
// G v = -1/2 H D2 H v with D2 u = pmax^2 (sum u) 1 - 2 pmax P u + (P o P) u and
// the UNclamped P = Q Q^T (mds.py:177-179).  (P o P) u is evaluated as
// q_i^T S q_i with S = Q^T diag(u) Q (r x r) — the Khatri-Rao identity of
// mds.py:147-152 without the n x r^2 expansion.
//
// One cooperative launch (one CTA per SM) runs the whole loop; every
// reduction is block-deterministic (fixed shuffle trees) and the grid-level
// combine runs in fixed block order, so results are bit-reproducible and the
// stopping decisions are identical in every CTA.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace rfxc {

constexpr int MDS_THREADS = 512;
constexpr int MDS_WARPS = MDS_THREADS / 32;
constexpr int MDS_CH = 32;          // rows staged per chunk in the S pass
constexpr int MDS_MAXE = 8;         // S-pass entries per thread per sweep
constexpr int MDS_SMEM_S_MAX = 96;  // r above this keeps S in global memory
constexpr int SLOT = 8;             // small-reduction slots per CTA

struct MdsArgs {
    const double* dq;
    int64_t n;
    int r;
    double pmax;
    int k;
    int max_it;
    double tol;
    int mode;  // 0: full MDS, 1: one gram_matvec of V[0] into w
    double* V;       // k x n: start vectors in, found vectors out
    double* w;       // n
    double* z;       // n
    double* parts;   // 2 x gridDim x SLOT (small reductions, double-buffered)
    double* sparts;  // gridDim x P2 (S-pass partials)
    double* tot;     // P2 totals
    double* Sg;      // r x r (global S when r > MDS_SMEM_S_MAX)
    double* coords;  // n x k
    double* info;    // k x 4
    int32_t* k_used;
};

struct Ctx {
    cg::grid_group grid;
    int64_t r0, r1;
    int parity;
    double* red;      // smem scratch 32
    double* bcast;    // smem SLOT
};

__device__ void grid_sum(Ctx& C, const MdsArgs& A, double* v, int m)
{
    double* parts = A.parts + (int64_t)C.parity * gridDim.x * SLOT;
    C.parity ^= 1;
    for (int j = 0; j < m; j++) {
        double s = block_sum(v[j], C.red);
        if (threadIdx.x == 0) parts[blockIdx.x * SLOT + j] = s;
        __syncthreads();
    }
    C.grid.sync();
    if (threadIdx.x < 32) {
        for (int j = 0; j < m; j++) {
            double s = 0.0;
            for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) s += parts[b * SLOT + j];
            s = warp_sum(s);
            if (threadIdx.x == 0) C.bcast[j] = s;
        }
    }
    __syncthreads();
    for (int j = 0; j < m; j++) v[j] = C.bcast[j];
    __syncthreads();
}

__device__ double grid_max(Ctx& C, const MdsArgs& A, double v)
{
    double* parts = A.parts + (int64_t)C.parity * gridDim.x * SLOT;
    C.parity ^= 1;
    double s = block_max(v, C.red);
    if (threadIdx.x == 0) parts[blockIdx.x * SLOT] = s;
    C.grid.sync();
    if (threadIdx.x < 32) {
        double m = -INFINITY;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) m = fmax(m, parts[b * SLOT]);
        m = warp_max(m);
        if (threadIdx.x == 0) C.bcast[0] = m;
    }
    __syncthreads();
    double out = C.bcast[0];
    __syncthreads();
    return out;
}

// (max |x|, first index) over the grid
__device__ int64_t grid_argmax_abs(Ctx& C, const MdsArgs& A, const double* x)
{
    double bv = -1.0;
    int64_t bi = INT64_MAX;
    for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += blockDim.x) {
        double a = fabs(x[i]);
        if (a > bv) { bv = a; bi = i; }
    }
    // warp then block
    for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    __shared__ double wv[MDS_WARPS];
    __shared__ int64_t wi[MDS_WARPS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) { wv[warp] = bv; wi[warp] = bi; }
    __syncthreads();
    double* parts = A.parts + (int64_t)C.parity * gridDim.x * SLOT;
    C.parity ^= 1;
    if (threadIdx.x == 0) {
        double v = wv[0];
        int64_t ii = wi[0];
        for (int w = 1; w < MDS_WARPS; w++)
            if (wv[w] > v || (wv[w] == v && wi[w] < ii)) { v = wv[w]; ii = wi[w]; }
        parts[blockIdx.x * SLOT] = v;
        parts[blockIdx.x * SLOT + 1] = __longlong_as_double((long long)ii);
    }
    C.grid.sync();
    if (threadIdx.x == 0) {
        double v = -1.0;
        int64_t ii = INT64_MAX;
        for (int b = 0; b < (int)gridDim.x; b++) {
            double pv = parts[b * SLOT];
            int64_t pi = (int64_t)__double_as_longlong(parts[b * SLOT + 1]);
            if (pv > v || (pv == v && pi < ii)) { v = pv; ii = pi; }
        }
        C.bcast[0] = __longlong_as_double((long long)ii);
    }
    __syncthreads();
    int64_t out = (int64_t)__double_as_longlong(C.bcast[0]);
    __syncthreads();
    return out;
}

__device__ __forceinline__ void tri_decode(int e, int r, int& a, int& b)
{
    // row-major upper triangle incl. diagonal: row a has r - a entries
    double R = 2.0 * r + 1.0;
    int aa = (int)((R - sqrt(R * R - 8.0 * e)) * 0.5);
    aa = max(0, min(r - 1, aa));
    while (aa > 0 && aa * r - aa * (aa - 1) / 2 > e) aa--;
    while (aa + 1 < r && (aa + 1) * r - (aa + 1) * aa / 2 <= e) aa++;
    a = aa;
    b = a + (e - (a * r - a * (a - 1) / 2));
}

// y = G x - sum_{f<nf} lam_f (v_f . x) v_f   (deflated_matvec, mds.py:203-207)
__device__ void matvec(Ctx& C, const MdsArgs& A, const double* x, double* y, int nf,
                       const double* lam, double* Ssm, double* stage)
{
    const int r = A.r;
    const int64_t n = A.n;
    const int ntri = r * (r + 1) / 2;
    const int P2 = ntri + r + 1 + nf;
    // mean of x
    double s1[1] = {0.0};
    for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += blockDim.x) s1[0] += x[i];
    grid_sum(C, A, s1, 1);
    const double mean = s1[0] / (double)n;

    // S pass: entries [0,ntri) S upper, [ntri, ntri+r) t, ntri+r: su, then d_f
    double* qs = stage;                  // MDS_CH x r
    double* us = stage + MDS_CH * r;     // MDS_CH
    double* xs = us + MDS_CH;            // MDS_CH
    double* out = A.sparts + (int64_t)blockIdx.x * P2;
    for (int ebase = 0; ebase < P2; ebase += MDS_THREADS * MDS_MAXE) {
        double acc[MDS_MAXE];
        int ea[MDS_MAXE], eb[MDS_MAXE];
#pragma unroll
        for (int q = 0; q < MDS_MAXE; q++) {
            acc[q] = 0.0;
            const int e = ebase + threadIdx.x + q * MDS_THREADS;
            ea[q] = -1;
            eb[q] = -1;
            if (e < ntri) tri_decode(e, r, ea[q], eb[q]);
            else if (e < ntri + r) { ea[q] = e - ntri; eb[q] = -2; }
            else if (e == ntri + r) { ea[q] = -3; }
            else if (e < P2) { ea[q] = -4; eb[q] = e - ntri - r - 1; }
        }
        for (int64_t base = C.r0; base < C.r1; base += MDS_CH) {
            const int m = (int)min64(MDS_CH, C.r1 - base);
            for (int t = threadIdx.x; t < m * r; t += blockDim.x)
                qs[t] = A.dq[base * r + t];
            for (int t = threadIdx.x; t < m; t += blockDim.x) {
                xs[t] = x[base + t];
                us[t] = x[base + t] - mean;
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < MDS_MAXE; q++) {
                const int a = ea[q], b = eb[q];
                if (a == -1 && b == -1) continue;
                double s = acc[q];
                if (a >= 0 && b >= 0) {
                    for (int t = 0; t < m; t++) s += us[t] * qs[t * r + a] * qs[t * r + b];
                } else if (a >= 0) {
                    for (int t = 0; t < m; t++) s += us[t] * qs[t * r + a];
                } else if (a == -3) {
                    for (int t = 0; t < m; t++) s += us[t];
                } else {
                    const double* vf = A.V + (int64_t)b * n + base;
                    for (int t = 0; t < m; t++) s += vf[t] * xs[t];
                }
                acc[q] = s;
            }
            __syncthreads();
        }
#pragma unroll
        for (int q = 0; q < MDS_MAXE; q++) {
            const int e = ebase + threadIdx.x + q * MDS_THREADS;
            if (e < P2) out[e] = acc[q];
        }
    }
    C.grid.sync();
    // distributed final reduce of the S-pass partials (fixed block order)
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < P2; e += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int b = 0; b < (int)gridDim.x; b++) s += A.sparts[(int64_t)b * P2 + e];
        A.tot[e] = s;
    }
    C.grid.sync();
    // expand S (symmetric) into smem or global
    double* S = (r <= MDS_SMEM_S_MAX) ? Ssm : A.Sg;
    if (r <= MDS_SMEM_S_MAX) {
        for (int e = threadIdx.x; e < ntri; e += blockDim.x) {
            int a, b;
            tri_decode(e, r, a, b);
            const double v = A.tot[e];
            S[a * r + b] = v;
            S[b * r + a] = v;
        }
        __syncthreads();
    } else {
        for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ntri; e += gridDim.x * blockDim.x) {
            int a, b;
            tri_decode(e, r, a, b);
            const double v = A.tot[e];
            S[a * r + b] = v;
            S[b * r + a] = v;
        }
        C.grid.sync();
    }
    const double* t = A.tot + ntri;
    const double su = A.tot[ntri + r];
    const double pm = A.pmax;
    // z_i = pmax^2 su - 2 pmax (q_i.t) + q_i^T S q_i   (mds.py:179)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* qrow = stage + MDS_CH * r + 2 * MDS_CH + warp * r;
    double zloc = 0.0;
    for (int64_t i = C.r0 + warp; i < C.r1; i += MDS_WARPS) {
        for (int a = lane; a < r; a += 32) qrow[a] = A.dq[i * r + a];
        __syncwarp();
        double pu = 0.0, ppu = 0.0;
        for (int a = lane; a < r; a += 32) {
            double sa = 0.0;
            for (int b = 0; b < r; b++) sa += S[b * r + a] * qrow[b];
            ppu += qrow[a] * sa;
            pu += qrow[a] * t[a];
        }
        pu = warp_sum(pu);
        ppu = warp_sum(ppu);
        const double zi = (pm * pm) * su - 2.0 * pm * pu + ppu;
        if (lane == 0) A.z[i] = zi;
        zloc += (lane == 0) ? zi : 0.0;
        __syncwarp();
    }
    __syncthreads();
    double s2[1] = {zloc};
    grid_sum(C, A, s2, 1);
    const double mz = s2[0] / (double)n;
    // y = -1/2 (z - mean z) - sum_f lam_f d_f v_f
    const double* d = A.tot + ntri + r + 1;
    for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += blockDim.x) {
        double yi = -0.5 * (A.z[i] - mz);
        for (int f = 0; f < nf; f++) yi -= lam[f] * d[f] * A.V[(int64_t)f * n + i];
        y[i] = yi;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(MDS_THREADS, 1) mds_kernel(MdsArgs A)
{
    extern __shared__ double msm[];
    __shared__ double red[32];
    __shared__ double bcast[SLOT];
    __shared__ double lam_s[8];
    const int r = A.r;
    double* Ssm = msm;                                       // r*r if small
    double* stage = msm + (r <= MDS_SMEM_S_MAX ? r * r : 0); // staging
    Ctx C{cg::this_grid(), 0, 0, 0, red, bcast};
    const int64_t n = A.n;
    const int64_t rpb = (n + gridDim.x - 1) / gridDim.x;
    C.r0 = min64(n, blockIdx.x * rpb);
    C.r1 = min64(n, C.r0 + rpb);

    if (A.mode == 1) {
        matvec(C, A, A.V, A.w, 0, lam_s, Ssm, stage);
        return;
    }
    int kused = 0;
    for (int comp = 0; comp < A.k; comp++) {
        double* v = A.V + (int64_t)comp * n;
        for (int f = 0; f < comp; f++) {
            const double* vf = A.V + (int64_t)f * n;
            double d[1] = {0.0};
            for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += blockDim.x) d[0] += vf[i] * v[i];
            grid_sum(C, A, d, 1);
            for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += blockDim.x) v[i] -= d[0] * vf[i];
            __syncthreads();
        }
        double nn[1] = {0.0};
        for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += blockDim.x) nn[0] += v[i] * v[i];
        grid_sum(C, A, nn, 1);
        const double nv = sqrt(nn[0]);
        if (nv == 0.0) break;
        for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += blockDim.x) v[i] /= nv;
        __syncthreads();

        double lam = 0.0;
        bool conv = false;
        int it = 0;
        for (it = 1; it <= A.max_it; it++) {
            matvec(C, A, v, A.w, comp, lam_s, Ssm, stage);
            for (int f = 0; f < comp; f++) {
                const double* vf = A.V + (int64_t)f * n;
                double d[1] = {0.0};
                for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += blockDim.x)
                    d[0] += vf[i] * A.w[i];
                grid_sum(C, A, d, 1);
                for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += blockDim.x)
                    A.w[i] -= d[0] * vf[i];
                __syncthreads();
            }
            double lw[2] = {0.0, 0.0};
            for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += blockDim.x) {
                lw[0] += v[i] * A.w[i];
                lw[1] += A.w[i] * A.w[i];
            }
            grid_sum(C, A, lw, 2);
            lam = lw[0];
            const double nw = sqrt(lw[1]);
            if (nw == 0.0) {
                lam = 0.0;
                conv = true;
                break;
            }
            const double sg = (lam / nw < 0.0) ? -1.0 : 1.0;  // sign of v_new . v
            double dmax = 0.0;
            for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += blockDim.x) {
                double vn = A.w[i] / nw;
                if (sg < 0) vn = -vn;
                dmax = fmax(dmax, fabs(vn - v[i]));
                v[i] = vn;
            }
            const double delta = grid_max(C, A, dmax);
            if (delta < A.tol) {
                conv = true;
                break;
            }
        }
        if (it > A.max_it) it = A.max_it;
        // residual |deflated_matvec(v) - lam v| / |lam|  (mds.py:241-242)
        matvec(C, A, v, A.w, comp, lam_s, Ssm, stage);
        double rr[1] = {0.0};
        for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += blockDim.x) {
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
    // coordinates: sqrt(lambda) * sign-fixed v  (mds.py:83-86, :257-261)
    for (int c = 0; c < kused; c++) {
        const double* v = A.V + (int64_t)c * n;
        const int64_t idx = grid_argmax_abs(C, A, v);
        const double sg = v[idx] < 0.0 ? -1.0 : 1.0;
        const double sl = sqrt(lam_s[c]);
        for (int64_t i = C.r0 + threadIdx.x; i < C.r1; i += blockDim.x)
            A.coords[i * A.k + c] = sl * (sg < 0 ? -v[i] : v[i]);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *A.k_used = kused;
}

struct Layout {
    int64_t V, w, z, parts, sparts, tot, Sg, bytes;
};

static int mds_grid()
{
    static int g = 0;
    if (!g) {
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mds_kernel, MDS_THREADS,
                                                      64 * 1024);
        g = sm_count() * std::max(1, std::min(occ, 1));
    }
    return g;
}

static Layout mds_layout(int64_t n, int r, int k)
{
    const int G = mds_grid();
    const int64_t P2 = (int64_t)r * (r + 1) / 2 + r + 1 + k;
    Layout L;
    int64_t o = 0;
    auto take = [&](int64_t count) { int64_t at = o; o += ((count * 8 + 255) / 256) * 256; return at; };
    L.V = take((int64_t)k * n);
    L.w = take(n);
    L.z = take(n);
    L.parts = take(2LL * G * SLOT);
    L.sparts = take((int64_t)G * P2);
    L.tot = take(P2);
    L.Sg = take((int64_t)r * r);
    L.bytes = o;
    return L;
}

static size_t mds_smem(int r)
{
    size_t s = (r <= MDS_SMEM_S_MAX ? (size_t)r * r : 0);
    s += (size_t)MDS_CH * r + MDS_CH * 2 + (size_t)MDS_WARPS * r;
    return s * 8;
}

static int launch_mds(MdsArgs& A, cudaStream_t st)
{
    const size_t smem = mds_smem(A.r);
    cudaError_t e = cudaFuncSetAttribute(mds_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)std::max<size_t>(smem, 1));
    if (e != cudaSuccess) return fail(RFXC_ECUDA, "mds attr: %s", cudaGetErrorString(e));
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mds_kernel, MDS_THREADS, smem);
    if (occ < 1) return fail(RFXC_ERUNTIME, "mds: kernel does not fit an SM (r=%d)", A.r);
    void* args[] = {&A};
    e = cudaLaunchCooperativeKernel((const void*)mds_kernel, dim3(mds_grid()), dim3(MDS_THREADS),
                                    args, smem, st);
    if (e != cudaSuccess) return fail(RFXC_ECUDA, "mds launch: %s", cudaGetErrorString(e));
    return check_launch("mds");
}

}  // namespace rfxc

using namespace rfxc;

extern "C" int64_t rfxc_mds_work_bytes(int64_t n, int32_t r, int32_t k)
{
    return mds_layout(n, r, std::max(k, 1)).bytes;
}

extern "C" int rfxc_mds_power(const double* d_dq, int64_t n, int32_t r, double pmax, int32_t k,
                              int32_t max_iterations, double tol, int64_t seed, double* d_coords,
                              double* d_info, int32_t* d_k_used, void* d_work, void* stream)
{
    if (n < 1 || r < 1 || k < 1 || k > 8 || max_iterations < 1)
        return fail(RFXC_EDATA, "mds_power: bad arguments");
    cudaStream_t st = as_stream(stream);
    Layout L = mds_layout(n, r, k);
    char* base = static_cast<char*>(d_work);
    MdsArgs A;
    A.dq = d_dq;
    A.n = n;
    A.r = r;
    A.pmax = pmax;
    A.k = k;
    A.max_it = max_iterations;
    A.tol = tol;
    A.mode = 0;
    A.V = reinterpret_cast<double*>(base + L.V);
    A.w = reinterpret_cast<double*>(base + L.w);
    A.z = reinterpret_cast<double*>(base + L.z);
    A.parts = reinterpret_cast<double*>(base + L.parts);
    A.sparts = reinterpret_cast<double*>(base + L.sparts);
    A.tot = reinterpret_cast<double*>(base + L.tot);
    A.Sg = reinterpret_cast<double*>(base + L.Sg);
    A.coords = d_coords;
    A.info = d_info;
    A.k_used = d_k_used;
    // start vectors Pcg32(seed + c, SEQ_POWER).normals(n)  (mds.py:210-211)
    for (int c = 0; c < k; c++) {
        int rc = rfxc_normals(seed + c, 5, n, A.V + (int64_t)c * n, stream);
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
    Layout L = mds_layout(n, r, 1);
    char* base = static_cast<char*>(d_work);
    MdsArgs A{};
    A.dq = d_dq;
    A.n = n;
    A.r = r;
    A.pmax = pmax;
    A.k = 1;
    A.max_it = 1;
    A.tol = 1.0;
    A.mode = 1;
    A.V = reinterpret_cast<double*>(base + L.V);
    A.w = d_w;
    A.z = reinterpret_cast<double*>(base + L.z);
    A.parts = reinterpret_cast<double*>(base + L.parts);
    A.sparts = reinterpret_cast<double*>(base + L.sparts);
    A.tot = reinterpret_cast<double*>(base + L.tot);
    A.Sg = reinterpret_cast<double*>(base + L.Sg);
    cudaError_t e = cudaMemcpyAsync(A.V, d_v, (size_t)n * 8, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return fail(RFXC_ECUDA, "gram_matvec copy: %s", cudaGetErrorString(e));
    return launch_mds(A, st);
}
