// linalg.cu — K5: the k x k dense steps of the randomised factorisation,
// on the device so the sketch / QR / Rayleigh-Ritz chain never waits on the
// host (k = r + 8 <= 110).
//
// Reference: np.linalg.qr (proximity.py:395, :397) and np.linalg.eigh of
// T = Q^T (P Q) (proximity.py:398-403).  The basis is shifted CholeskyQR3:
// for the n x k sketch Y, R1 = chol(Y^T Y + s I) with s = 11 (nk + k(k+1))
// u tr(Y^T Y), Q1 = Y R1^-1, then two plain CholeskyQR steps on Q1 (each a
// Gram, rfxc_chol_inv and a small matmul), orthonormal to O(u) for any
// cond(Y) < 1/u.  The eigen-map (rfxc_orth_map, Gram-eigen with directions
// below 1e-13 l_max dropped) is kept for callers that want a rank-revealing
// basis.  The k x k entry points run one CTA with the matrix in shared memory:
// cyclic Jacobi with the round-robin (circle) ordering, k/2 disjoint
// rotations per round; an entry is left alone once |a_pq| <= 1e-18
// sqrt(|a_pp a_qq|) and the sweeps stop after one without a rotation;
// eigenvalues sorted descending (ties keep index order).  Deterministic.
#include "common.cuh"

namespace rfxc {

constexpr int LA_MAXK = 110;
constexpr int LA_THREADS = 512;

// Symmetric eigendecomposition of the k x k matrix in A (row-major, shared
// memory, symmetrised on entry) -> w (descending) and V (row-major, column j
// = eigenvector j), both in shared memory.  scratch: >= 4 * (k/2 + 1) doubles
// + k ints.
__device__ void jacobi_eig(double* A, double* V, double* w, int k, double* rot, int* order)
{
    const int tid = threadIdx.x, nt = blockDim.x;
    const int kp = (k + 1) & ~1;  // even player count (index k is a dummy when k is odd)
    for (int e = tid; e < k * k; e += nt) {
        const int i = e / k, j = e % k;
        if (i < j) {
            const double s = 0.5 * (A[i * k + j] + A[j * k + i]);
            A[i * k + j] = s;
            A[j * k + i] = s;
        }
        V[e] = (i == j) ? 1.0 : 0.0;
    }
    __syncthreads();
    double* cs = rot;
    double* sn = rot + kp / 2;
    int* pp = reinterpret_cast<int*>(rot + kp);
    int* qq = pp + kp / 2;
    __shared__ int rotated;
    for (int sweep = 0; sweep < 60; sweep++) {
        if (tid == 0) rotated = 0;
        __syncthreads();
        for (int rnd = 0; rnd < kp - 1; rnd++) {
            for (int i = tid; i < kp / 2; i += nt) {
                int p, q;
                if (i == 0) {
                    p = kp - 1;
                    q = rnd;
                } else {
                    p = (rnd + i) % (kp - 1);
                    q = (rnd - i + (kp - 1)) % (kp - 1);
                }
                if (p > q) { const int t = p; p = q; q = t; }
                double c = 1.0, s = 0.0;
                if (q < k) {
                    const double apq = A[p * k + q];
                    const double app = A[p * k + p], aqq = A[q * k + q];
                    // skip entries already negligible next to their diagonal
                    if (apq != 0.0 && fabs(apq) > 1e-18 * sqrt(fabs(app) * fabs(aqq))) {
                        const double tau = (aqq - app) / (2.0 * apq);
                        const double t = (tau >= 0.0 ? 1.0 : -1.0) /
                                         (fabs(tau) + sqrt(1.0 + tau * tau));
                        c = 1.0 / sqrt(1.0 + t * t);
                        s = t * c;
                        rotated = 1;
                    }
                }
                cs[i] = c;
                sn[i] = s;
                pp[i] = p;
                qq[i] = q < k ? q : -1;
            }
            __syncthreads();
            // rows p, q <- J^T rows
            for (int e = tid; e < (kp / 2) * k; e += nt) {
                const int i = e / k, j = e % k;
                const int p = pp[i], q = qq[i];
                if (q < 0 || sn[i] == 0.0) continue;
                const double ap = A[p * k + j], aq = A[q * k + j];
                A[p * k + j] = cs[i] * ap - sn[i] * aq;
                A[q * k + j] = sn[i] * ap + cs[i] * aq;
            }
            __syncthreads();
            // columns p, q <- A J, V J
            for (int e = tid; e < (kp / 2) * k; e += nt) {
                const int i = e / k, j = e % k;
                const int p = pp[i], q = qq[i];
                if (q < 0 || sn[i] == 0.0) continue;
                const double c = cs[i], s = sn[i];
                const double ap = A[j * k + p], aq = A[j * k + q];
                A[j * k + p] = c * ap - s * aq;
                A[j * k + q] = s * ap + c * aq;
                const double vp = V[j * k + p], vq = V[j * k + q];
                V[j * k + p] = c * vp - s * vq;
                V[j * k + q] = s * vp + c * vq;
            }
            __syncthreads();
        }
        if (!rotated) break;
    }
    // descending order (stable: ties keep index order)
    if (tid == 0) {
        for (int i = 0; i < k; i++) order[i] = i;
        for (int i = 1; i < k; i++) {
            const int x = order[i];
            const double vx = A[x * k + x];
            int j = i - 1;
            while (j >= 0 && A[order[j] * k + order[j]] < vx) {
                order[j + 1] = order[j];
                j--;
            }
            order[j + 1] = x;
        }
    }
    __syncthreads();
    for (int i = tid; i < k; i += nt) w[i] = A[order[i] * k + order[i]];
    // permute V's columns in place through A (no longer needed)
    for (int e = tid; e < k * k; e += nt) A[e] = V[(e / k) * k + order[e % k]];
    __syncthreads();
    for (int e = tid; e < k * k; e += nt) V[e] = A[e];
    __syncthreads();
}

struct LaSmem {
    double* A;
    double* V;
    double* w;
    double* rot;
    int* order;
};

__device__ LaSmem la_smem(int k)
{
    extern __shared__ double la_raw[];
    LaSmem S;
    const int kp = (k + 1) & ~1;
    S.A = la_raw;
    S.V = S.A + k * k;
    S.w = S.V + k * k;
    S.rot = S.w + k;
    S.order = reinterpret_cast<int*>(S.rot + 2 * kp);
    return S;
}

// mode 0: orthonormalising map M (k x k) from the Gram G
// mode 1: Rayleigh-Ritz factor map Wr (k x r) = W_r sqrt(clip(l_r, 0)) from T
__global__ void __launch_bounds__(LA_THREADS) eig_map_kernel(const double* __restrict__ Gin, int k,
                                                             int r, int mode,
                                                             double* __restrict__ out)
{
    LaSmem S = la_smem(k);
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) S.A[e] = Gin[e];
    __syncthreads();
    jacobi_eig(S.A, S.V, S.w, k, S.rot, S.order);
    if (mode == 0) {
        const double top = fmax(S.w[0], 0.0);
        int kept = 0;
        for (int c = 0; c < k; c++) kept += S.w[c] > top * 1e-13;
        for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
            const int i = e / k, c = e % k;
            double v = 0.0;
            if (kept == 0) {
                if (c == 0) v = S.V[i * k] / sqrt(fmax(S.w[0], 1e-300));
            } else if (S.w[c] > top * 1e-13) {
                v = S.V[i * k + c] / sqrt(S.w[c]);
            }
            out[e] = v;
        }
    } else {
        for (int e = threadIdx.x; e < k * r; e += blockDim.x) {
            const int i = e / r, c = e % r;
            out[e] = c < k ? S.V[i * k + c] * sqrt(fmax(S.w[c], 0.0)) : 0.0;
        }
    }
}

#ifndef RFXC_CHOL_THREADS
#define RFXC_CHOL_THREADS 512
#endif
// Rinv (k x k, upper) with G + shift_rel tr(G) I = R^T R (Cholesky of the
// symmetrised matrix); a non-positive pivot gives a zero row/column.  One CTA,
// one barrier per step: step j updates the trailing upper triangle with the
// unscaled row j (a_ab -= a_ja a_jb / a_jj, every thread reads the pivot
// itself), rows are scaled at the end; the inverse is column-oriented back
// substitution (step m finalises row m of R^-1 and updates every row above).
constexpr int CHOL_THREADS = RFXC_CHOL_THREADS;

__global__ void __launch_bounds__(CHOL_THREADS) chol_inv_kernel(const double* __restrict__ Gin,
                                                                int k, double shift_rel,
                                                                double* __restrict__ Rinv)
{
    extern __shared__ double cs[];
    double* R = cs;          // k x k
    double* X = cs + k * k;  // k x k
    double* dg = X + k * k;  // k pivots
    __shared__ double red[32];
    const int tid = threadIdx.x, nt = blockDim.x;
    double tr = 0.0;
    for (int e = tid; e < k * k; e += nt) {
        const int i = e / k, j = e % k;
        const double v = 0.5 * (Gin[i * k + j] + Gin[j * k + i]);
        R[e] = v;
        X[e] = (i == j) ? 1.0 : 0.0;
        if (i == j) tr += v;
    }
    tr = block_sum(tr, red);
    if (shift_rel > 0.0)
        for (int i = tid; i < k; i += nt) R[i * k + i] += shift_rel * tr;
    __syncthreads();
    // step j: trailing upper triangle a_ab -= a_ja a_jb / a_jj (unscaled row
    // j); rows over warps, columns over lanes (no index division)
    const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    for (int j = 0; j < k - 1; j++) {
        const double d = R[j * k + j];
        if (d > 0.0) {
            const double inv = 1.0 / d;
            for (int a = j + 1 + warp; a < k; a += nw) {
                const double rja = R[j * k + a];
                for (int b = a + lane; b < k; b += 32) R[a * k + b] -= rja * R[j * k + b] * inv;
            }
        }
        __syncthreads();
    }
    for (int i = tid; i < k; i += nt) dg[i] = R[i * k + i];
    __syncthreads();
    for (int e = tid; e < k * k; e += nt) {
        const int a = e / k, b = e % k;
        const double d = dg[a];
        R[e] = (b >= a && d > 0.0) ? R[e] / sqrt(d) : 0.0;
    }
    __syncthreads();
    // X = R^-1, bottom-up: row m is final after dividing by r_mm; rows above
    // subtract r_im * X[m][m:] (columns >= m only: X is upper triangular)
    for (int m = k - 1; m >= 0; m--) {
        const double rmm = R[m * k + m];
        const int w = k - m;
        for (int c = tid; c < w; c += nt) {
            const double v = X[m * k + m + c];
            X[m * k + m + c] = rmm > 0.0 ? v / rmm : 0.0;
        }
        __syncthreads();
        for (int i = warp; i < m; i += nw) {
            const double rim = R[i * k + m];
            for (int c = m + lane; c < k; c += 32) X[i * k + c] -= rim * X[m * k + c];
        }
        __syncthreads();
    }
    for (int e = tid; e < k * k; e += nt) Rinv[e] = X[e];
}

static size_t eig_smem(int k)
{
    const int kp = (k + 1) & ~1;
    return (size_t)(2 * k * k + k + 2 * kp) * 8 + (size_t)k * 4 + 16;
}

}  // namespace rfxc

using namespace rfxc;

static int launch_eig_map(const double* d_G, int k, int r, int mode, double* d_out, void* stream)
{
    if (k < 1 || k > LA_MAXK || r < 0 || r > k) return fail(RFXC_EDATA, "eig: bad k=%d r=%d", k, r);
    const size_t smem = eig_smem(k);
    cudaError_t e = cudaFuncSetAttribute(eig_map_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return fail(RFXC_ECUDA, "eig attr: %s", cudaGetErrorString(e));
    eig_map_kernel<<<1, LA_THREADS, smem, as_stream(stream)>>>(d_G, k, r, mode, d_out);
    return check_launch("eig_map");
}

extern "C" int rfxc_orth_map(const double* d_G, int32_t k, double* d_M, void* stream)
{
    return launch_eig_map(d_G, k, k, 0, d_M, stream);
}

extern "C" int rfxc_ritz_factor_map(const double* d_T, int32_t k, int32_t r, double* d_Wr,
                                    void* stream)
{
    return launch_eig_map(d_T, k, r, 1, d_Wr, stream);
}

extern "C" int rfxc_chol_inv(const double* d_G, int32_t k, double shift_rel, double* d_Rinv,
                             void* stream)
{
    if (k < 1 || k > LA_MAXK) return fail(RFXC_EDATA, "chol_inv: bad k=%d", k);  // k*k <= 16 * 1024
    const size_t smem = ((size_t)2 * k * k + k) * 8;
    cudaError_t e = cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return fail(RFXC_ECUDA, "chol attr: %s", cudaGetErrorString(e));
    chol_inv_kernel<<<1, CHOL_THREADS, smem, as_stream(stream)>>>(d_G, k, shift_rel, d_Rinv);
    return check_launch("chol_inv");
}

__global__ void __launch_bounds__(LA_THREADS) sym_eig_kernel(const double* __restrict__ Ain, int k,
                                                             double* __restrict__ w,
                                                             double* __restrict__ V)
{
    LaSmem S = la_smem(k);
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) S.A[e] = Ain[e];
    __syncthreads();
    jacobi_eig(S.A, S.V, S.w, k, S.rot, S.order);
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) V[e] = S.V[e];
    for (int e = threadIdx.x; e < k; e += blockDim.x) w[e] = S.w[e];
}

extern "C" int rfxc_sym_eig(const double* d_A, int32_t k, double* d_w, double* d_V, void* stream)
{
    if (k < 1 || k > LA_MAXK) return fail(RFXC_EDATA, "sym_eig: bad k=%d", k);
    const size_t smem = eig_smem(k);
    cudaError_t e = cudaFuncSetAttribute(sym_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return fail(RFXC_ECUDA, "sym_eig attr: %s", cudaGetErrorString(e));
    sym_eig_kernel<<<1, LA_THREADS, smem, as_stream(stream)>>>(d_A, k, d_w, d_V);
    return check_launch("sym_eig");
}
