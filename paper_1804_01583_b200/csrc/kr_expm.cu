// kr_expm.cu — batched small-matrix exponentials and the basis-matrix projection (Eq. 2,
// PAPER.md:651-655; projected form of Alg. 4):
//     x_{d,j} = e^{H_d t_j} e_1,   c[j][r][d] = ||v_d|| * sum_l P_d[r][l] x_{d,j}[l],   t_j = j*step.
// One CTA per (time step j, direction d): scaling and squaring with the degree-13 diagonal Pade
// approximant (Higham 2005 coefficients, theta_13 = 5.3719; the paper defers to "squaring and scaling
// and Pade"), matrices held in shared memory (k <= 64), 16x16 threads with 4x4
// register micro-tiles per matmul, LU with partial pivoting for the Pade solve. j = 0 is exactly e_1
// (e^0 = I). Also records h(t_j) = e_k^T e^{H t_j} e_1 for the Lemma 1 diagnostic
// and integrates it (trapezoid on the t_j grid).
#include <math.h>

#include <algorithm>

#include "kr_internal.h"

namespace {

constexpr int ET = 256;

// C = A * B (n x n, leading dimension ld); caller synchronises before and after. 16 x 16 threads with MT x MT
// register micro-tiles (rows ty + 16 a, columns tx + 16 b) covering 16 MT >= n: the smallest tile that covers n, so
// no thread multiplies padding (n = 40: 48 x 48 instead of 64 x 64, 44 % fewer FMAs). Every C entry is summed over l
// in order whatever MT is (bitwise the same result).
template <int MT>
__device__ __forceinline__ void mm_t(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C,
                                     int n, int ld) {
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[MT][MT];
#pragma unroll
    for (int a = 0; a < MT; ++a)
#pragma unroll
        for (int b = 0; b < MT; ++b) acc[a][b] = 0.0;
    for (int l = 0; l < n; ++l) {
        double av[MT], bv[MT];
#pragma unroll
        for (int a = 0; a < MT; ++a) {
            const int i = ty + 16 * a;
            av[a] = i < n ? A[i * ld + l] : 0.0;
        }
#pragma unroll
        for (int b = 0; b < MT; ++b) {
            const int j = tx + 16 * b;
            bv[b] = j < n ? B[l * ld + j] : 0.0;
        }
#pragma unroll
        for (int a = 0; a < MT; ++a)
#pragma unroll
            for (int b = 0; b < MT; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
    }
#pragma unroll
    for (int a = 0; a < MT; ++a)
#pragma unroll
        for (int b = 0; b < MT; ++b) {
            const int i = ty + 16 * a, j = tx + 16 * b;
            if (i < n && j < n) C[i * ld + j] = acc[a][b];
        }
}
__device__ __forceinline__ void mm(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C,
                                   int n, int ld) {
    if (n <= 16)
        mm_t<1>(A, B, C, n, ld);
    else if (n <= 32)
        mm_t<2>(A, B, C, n, ld);
    else if (n <= 48)
        mm_t<3>(A, B, C, n, ld);
    else
        mm_t<4>(A, B, C, n, ld);
}

struct ExpmArgs {
    const double* H;     // [ndl][k+1][k]
    const double* P;     // [ndl][n_out][k]
    const double* beta0; // [ndl]
    const int32_t* keff; // [ndl]
    int k, n_out, ndl_stride;
    int64_t n_steps;
    double step;
    double* coeff;       // [(n_steps+1)][n_out][ndl_stride]
    double* hlast;       // [ndl][n_steps+1]
    // single-direction use by the large-k route's small checkpoints (doubling, powers and march kernels)
    int dsel = -1;               // >= 0: one CTA, for this local direction
    int nfix = 0;                // > 0: dimension (instead of keff)
    const double* Hsrc = nullptr;  // non-NULL: H from here, row stride hstride
    int hstride = 0;
};

// e^{H t} of the leading n x n block of H (row stride k) by scaling and squaring with the degree-13 diagonal
// Pade approximant (Higham 2005): six n x (n+1) buffers of shared memory in sm; returns the buffer holding the
// result (row stride n + 1). All threads of the CTA must call it.
__device__ double* pade13(const double* Hd, int k, int n, double t, double* sm, double* fac, int& piv_s, int& sq_s) {
    const int ld = n + 1;
    const int msz = n * ld;
    double* B0 = sm;
    double* B1 = B0 + msz;
    double* B2 = B1 + msz;
    double* B3 = B2 + msz;
    double* B4 = B3 + msz;
    double* B5 = B4 + msz;
    for (int e = threadIdx.x; e < n * n; e += ET) {
        const int r = e / n, c = e - r * n;
        B0[r * ld + c] = Hd[r * k + c] * t;
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // 1-norm (max column sum) -> number of squarings
        double cmax = 0.0;
        for (int c = threadIdx.x; c < n; c += 32) {
            double s = 0.0;
            for (int r = 0; r < n; ++r) s += fabs(B0[r * ld + c]);
            cmax = fmax(cmax, s);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cmax = fmax(cmax, __shfl_down_sync(0xffffffffu, cmax, o));
        if (threadIdx.x == 0) {
            const double theta13 = 5.371920351148152;
            int s = 0;
            if (cmax > theta13) s = (int)ceil(log2(cmax / theta13));
            while (ldexp(cmax, -s) > theta13) ++s;
            sq_s = s < 0 ? 0 : s;
        }
    }
    __syncthreads();
    const int s = sq_s;
    if (s > 0)
        for (int e = threadIdx.x; e < n * n; e += ET) {
            const int r = e / n, c = e - r * n;
            B0[r * ld + c] = ldexp(B0[r * ld + c], -s);
        }
    __syncthreads();
    const double b0 = 64764752532480000.0, b1 = 32382376266240000.0, b2 = 7771770303897600.0,
                 b3 = 1187353796428800.0, b4 = 129060195264000.0, b5 = 10559470521600.0, b6 = 670442572800.0,
                 b7 = 33522128640.0, b8 = 1323241920.0, b9 = 40840800.0, b10 = 960960.0, b11 = 16380.0,
                 b12 = 182.0, b13 = 1.0;
    mm(B0, B0, B1, n, ld);  // A2
    __syncthreads();
    mm(B1, B1, B2, n, ld);  // A4
    __syncthreads();
    mm(B2, B1, B3, n, ld);  // A6
    __syncthreads();
    for (int e = threadIdx.x; e < n * n; e += ET) {
        const int o = (e / n) * ld + e % n;
        B4[o] = b13 * B3[o] + b11 * B2[o] + b9 * B1[o];
    }
    __syncthreads();
    mm(B3, B4, B5, n, ld);  // A6 (b13 A6 + b11 A4 + b9 A2)
    __syncthreads();
    for (int e = threadIdx.x; e < n * n; e += ET) {
        const int r = e / n, c = e - r * n, o = r * ld + c;
        B5[o] = B5[o] + b7 * B3[o] + b5 * B2[o] + b3 * B1[o] + (r == c ? b1 : 0.0);
    }
    __syncthreads();
    mm(B0, B5, B4, n, ld);  // U = A * (...)
    __syncthreads();
    for (int e = threadIdx.x; e < n * n; e += ET) {
        const int o = (e / n) * ld + e % n;
        B5[o] = b12 * B3[o] + b10 * B2[o] + b8 * B1[o];
    }
    __syncthreads();
    mm(B3, B5, B0, n, ld);  // A6 (b12 A6 + b10 A4 + b8 A2)  (A no longer needed)
    __syncthreads();
    for (int e = threadIdx.x; e < n * n; e += ET) {
        const int r = e / n, c = e - r * n, o = r * ld + c;
        const double V = B0[o] + b6 * B3[o] + b4 * B2[o] + b2 * B1[o] + (r == c ? b0 : 0.0);
        const double U = B4[o];
        B1[o] = V + U;  // P
        B2[o] = V - U;  // Q
    }
    __syncthreads();
    // solve Q F = P: LU with partial pivoting (lowest index wins ties), F overwrites P
    double* Q = B2;
    double* F = B1;
    for (int c = 0; c < n; ++c) {
        if (threadIdx.x < 32) {
            double best = -1.0;
            int bi = c;
            for (int i = c + threadIdx.x; i < n; i += 32) {
                const double v = fabs(Q[i * ld + c]);
                if (v > best) {
                    best = v;
                    bi = i;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_down_sync(0xffffffffu, best, o);
                const int oi = __shfl_down_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) {
                    best = ob;
                    bi = oi;
                }
            }
            if (threadIdx.x == 0) piv_s = bi;
        }
        __syncthreads();
        const int p = piv_s;
        if (p != c)
            for (int col = threadIdx.x; col < n; col += ET) {
                double t0 = Q[c * ld + col];
                Q[c * ld + col] = Q[p * ld + col];
                Q[p * ld + col] = t0;
                t0 = F[c * ld + col];
                F[c * ld + col] = F[p * ld + col];
                F[p * ld + col] = t0;
            }
        __syncthreads();
        for (int i = c + 1 + threadIdx.x; i < n; i += ET) fac[i] = Q[i * ld + c] / Q[c * ld + c];
        __syncthreads();
        const int rows = n - c - 1;
        for (int e = threadIdx.x; e < rows * n; e += ET) {
            const int i = c + 1 + e / n, col = e % n;
            const double f = fac[i];
            F[i * ld + col] -= f * F[c * ld + col];
            if (col > c) Q[i * ld + col] -= f * Q[c * ld + col];
        }
        __syncthreads();
    }
    for (int i = n - 1; i >= 0; --i) {
        for (int col = threadIdx.x; col < n; col += ET) {
            double t0 = F[i * ld + col];
            for (int l = i + 1; l < n; ++l) t0 -= Q[i * ld + l] * F[l * ld + col];
            F[i * ld + col] = t0 / Q[i * ld + i];
        }
        __syncthreads();
    }
    // square s times
    double* X = F;
    double* Y = B3;
    for (int r = 0; r < s; ++r) {
        mm(X, X, Y, n, ld);
        __syncthreads();
        double* t0 = X;
        X = Y;
        Y = t0;
    }
    return X;
}

__global__ void __launch_bounds__(ET) expm_project_kernel(ExpmArgs a) {
    const int64_t j = blockIdx.x;
    const int d = blockIdx.y;
    const int n = a.keff[d];
    const int k = a.k;
    extern __shared__ double sm[];
    __shared__ double xs[64];
    __shared__ double fac[64];
    __shared__ int piv_s;
    __shared__ int sq_s;
    if (n <= 0) {
        for (int r = threadIdx.x; r < a.n_out; r += ET) a.coeff[(j * a.n_out + r) * a.ndl_stride + d] = 0.0;
        return;
    }
    const int ld = n + 1;
    if (j == 0) {
        for (int i = threadIdx.x; i < n; i += ET) xs[i] = i == 0 ? 1.0 : 0.0;  // e^{H 0} e_1 = e_1 exactly
    } else {
        const double* X = pade13(a.H + (int64_t)d * (k + 1) * k, k, n, (double)j * a.step, sm, fac, piv_s, sq_s);
        for (int i = threadIdx.x; i < n; i += ET) xs[i] = X[i * ld + 0];
    }
    __syncthreads();
    const double* Pd = a.P + (int64_t)d * a.n_out * k;
    const double bz = a.beta0[d];
    for (int r = threadIdx.x; r < a.n_out; r += ET) {
        double s = 0.0;
        for (int l = 0; l < n; ++l) s = fma(Pd[(int64_t)r * k + l], xs[l], s);
        a.coeff[(j * a.n_out + r) * a.ndl_stride + d] = bz * s;
    }
    if (threadIdx.x == 0) a.hlast[(int64_t)d * (a.n_steps + 1) + j] = xs[n - 1];
}

// The uniform time grid by doubling (one CTA per direction): E = e^{H delta} by the same Pade-13 scaling and
// squaring, then x_0 = e_1 and x_{2^q + j} = E^{2^q} x_j for j < 2^q (one small matrix-matrix product per
// level), E^{2^{q+1}} = (E^{2^q})^2 — log2(N) levels instead of N independent Pade-13 exponentials
// (C2: 42021 of them). x_j kept column-wise in global memory X [n][ldx] (L2-resident); then the projection
// c[j][r][d] = ||v_d|| (P x_j)_r and h(t_j) = x_j[n-1] for Lemma 1.
__global__ void __launch_bounds__(ET) expm_doubling_kernel(ExpmArgs a, double* xt, int ldx) {
    const int d = a.dsel >= 0 ? a.dsel : blockIdx.x;
    const int n = a.nfix > 0 ? a.nfix : a.keff[d];
    const int k = a.k;
    const int64_t np1 = a.n_steps + 1;
    extern __shared__ double sm[];
    __shared__ double fac[64];
    __shared__ int piv_s;
    __shared__ int sq_s;
    if (n <= 0) {
        for (int64_t e = threadIdx.x; e < np1 * a.n_out; e += ET)
            a.coeff[((e / a.n_out) * a.n_out + e % a.n_out) * a.ndl_stride + d] = 0.0;
        return;
    }
    const int ld = n + 1;
    double* X = xt + (a.dsel >= 0 ? 0 : (int64_t)d * 64 * ldx);  // [n][ldx]
    for (int l = threadIdx.x; l < n; l += ET) X[(int64_t)l * ldx] = l == 0 ? 1.0 : 0.0;  // x_0 = e_1 exactly
    const double* Hd = a.Hsrc ? a.Hsrc : a.H + (int64_t)d * (k + 1) * k;
    double* E = np1 > 1 ? pade13(Hd, a.Hsrc ? a.hstride : k, n, a.step, sm, fac, piv_s, sq_s) : sm;
    // powers in two buffers (Pw, Tw), the remaining four (contiguous, 4 n (n+1) doubles) stage column tiles of the
    // trajectory, so every product below reads shared memory only (a dot over n global-memory loads per output
    // was latency-bound: ~0.6 ms per C2 run)
    const int msz = n * ld;
    const int ei = (int)((E - sm) / msz);
    double* Pw = sm + (size_t)(ei == 1 ? 1 : 0) * msz;
    double* Tw = sm + (size_t)(ei == 1 ? 0 : 1) * msz;
    double* XT = sm + (size_t)2 * msz;
    const int TC = min(128, 4 * (n + 1));  // columns per tile: n x TC doubles fit the four buffers
    if (ei > 1) {
        for (int e = threadIdx.x; e < n * n; e += ET) {
            const int o = (e / n) * ld + e % n;
            Pw[o] = E[o];
        }
    }
    __syncthreads();
    for (int64_t w0 = 1; w0 < np1; w0 <<= 1) {
        const int64_t w = min(w0, np1 - w0);
        for (int64_t c0 = 0; c0 < w; c0 += TC) {  // X[:, w0 + c] = Pw X[:, c], c in [c0, c0 + tc)
            const int tc = (int)min((int64_t)TC, w - c0);
            for (int e = threadIdx.x; e < n * tc; e += ET) {
                const int l = e / tc, cc = e - l * tc;
                XT[l * TC + cc] = X[(int64_t)l * ldx + c0 + cc];
            }
            __syncthreads();
            // n x tc product, 4 x 8 register micro-tile per thread (16 x 16 threads cover 64 x 128); each output is
            // still one fma chain over l in order
            {
                const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
                double acc[4][8];
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 8; ++v) acc[u][v] = 0.0;
                for (int l = 0; l < n; ++l) {
                    double av[4], bv[8];
#pragma unroll
                    for (int u = 0; u < 4; ++u) av[u] = ty + 16 * u < n ? Pw[(ty + 16 * u) * ld + l] : 0.0;
#pragma unroll
                    for (int v = 0; v < 8; ++v) bv[v] = tx + 16 * v < tc ? XT[l * TC + tx + 16 * v] : 0.0;
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int v = 0; v < 8; ++v) acc[u][v] = fma(av[u], bv[v], acc[u][v]);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 8; ++v) {
                        const int i = ty + 16 * u, cc = tx + 16 * v;
                        if (i < n && cc < tc) X[(int64_t)i * ldx + w0 + c0 + cc] = acc[u][v];
                    }
            }
            __syncthreads();
        }
        if (2 * w0 < np1) {
            mm(Pw, Pw, Tw, n, ld);
            __syncthreads();
            double* t0 = Pw;
            Pw = Tw;
            Tw = t0;
        }
    }
    const double* Pd = a.P + (int64_t)d * a.n_out * k;
    const double bz = a.beta0[d];
    for (int64_t c0 = 0; c0 < np1; c0 += TC) {
        const int tc = (int)min((int64_t)TC, np1 - c0);
        for (int e = threadIdx.x; e < n * tc; e += ET) {
            const int l = e / tc, cc = e - l * tc;
            XT[l * TC + cc] = X[(int64_t)l * ldx + c0 + cc];
        }
        __syncthreads();
        for (int e = threadIdx.x; e < ((a.n_out + 3) / 4) * tc; e += ET) {  // 4 output rows per thread
            const int r0 = 4 * (e / tc), cc = e % tc;
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            for (int l = 0; l < n; ++l) {
                const double x = XT[l * TC + cc];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (r0 + q < a.n_out) acc[q] = fma(Pd[(int64_t)(r0 + q) * k + l], x, acc[q]);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (r0 + q < a.n_out) a.coeff[((c0 + cc) * a.n_out + r0 + q) * a.ndl_stride + d] = bz * acc[q];
        }
        for (int cc = threadIdx.x; cc < tc; cc += ET) a.hlast[(int64_t)d * np1 + c0 + cc] = XT[(n - 1) * TC + cc];
        __syncthreads();
    }
}

// The time grid over many CTAs (default): expm_powers_kernel (one CTA per direction) forms E = e^{H delta}
// by the Pade-13 scaling and squaring above and its powers E^{2^q}, q < Q (2^{Q-1} <= n_steps < 2^Q), into
// pw [ndl][Q][64][65]; expm_march_kernel (CTA s of direction d owns the columns [s B, s B + B)) starts from
// x_{sB} = prod_{bits q of sB} E^{2^q} e_1 (e_1 exactly for s = 0) and marches x_{j+1} = E x_j, with the
// projection c[j][., d] = ||v_d|| P x_j in the same matrix-vector product ([E; P] x_j, one pass). The one-CTA
// doubling above serialised ~0.3 ms per direction on one SM (C3); here it is the Pade-13 of one CTA plus a
// few microseconds.
constexpr int PW_LD = 65;
constexpr size_t PW_MAT = (size_t)64 * PW_LD;

__global__ void __launch_bounds__(ET) expm_powers_kernel(ExpmArgs a, double* pw, int Q) {
    const int d = a.dsel >= 0 ? a.dsel : blockIdx.x;
    const int n = a.nfix > 0 ? a.nfix : a.keff[d];
    if (n <= 0 || a.n_steps < 1) return;
    const int k = a.k;
    extern __shared__ double sm[];
    __shared__ double fac[64];
    __shared__ int piv_s;
    __shared__ int sq_s;
    const int ld = n + 1;
    const int msz = n * ld;
    const double* Hd = a.Hsrc ? a.Hsrc : a.H + (int64_t)d * (k + 1) * k;
    double* E = pade13(Hd, a.Hsrc ? a.hstride : k, n, a.step, sm, fac, piv_s, sq_s);
    const int ei = (int)((E - sm) / msz);
    double* X = E;
    double* Y = sm + (size_t)(ei == 0 ? 1 : 0) * msz;
    double* out = pw + (size_t)d * Q * PW_MAT;
    for (int q = 0; q < Q; ++q) {
        for (int e = threadIdx.x; e < n * n; e += ET) {
            const int r = e / n, c = e - r * n;
            out[(size_t)q * PW_MAT + r * PW_LD + c] = X[r * ld + c];
        }
        if (q + 1 < Q) {
            mm(X, X, Y, n, ld);
            __syncthreads();
            double* t0 = X;
            X = Y;
            Y = t0;
        }
    }
}

// y = M x for the rows [0, R) of M (row stride PW_LD, n columns); two threads per row split the columns, added
// in a fixed order. x, part in shared memory; all threads call it.
__device__ __forceinline__ void mv_rows(const double* M, int R, int n, const double* x, double* part, double* y) {
    const int i = threadIdx.x & 127, h = threadIdx.x >> 7;
    const int half = (n + 1) >> 1;
    const int l0 = h ? half : 0, l1 = h ? n : half;
    if (i < R) {
        double s = 0.0;
        for (int l = l0; l < l1; ++l) s = fma(M[i * PW_LD + l], x[l], s);
        part[h * 128 + i] = s;
    }
    __syncthreads();
    if (threadIdx.x < R) y[threadIdx.x] = part[threadIdx.x] + part[128 + threadIdx.x];
    __syncthreads();
}

__global__ void __launch_bounds__(ET) expm_march_kernel(ExpmArgs a, const double* pw, int Q, int B) {
    const int d = a.dsel >= 0 ? a.dsel : blockIdx.y;
    const int n = a.nfix > 0 ? a.nfix : a.keff[d];
    const int k = a.k;
    const int64_t np1 = a.n_steps + 1;
    const int64_t c0 = (int64_t)blockIdx.x * B, c1 = min(c0 + B, np1);
    if (c0 >= np1) return;
    if (n <= 0) {
        for (int64_t e = threadIdx.x; e < (c1 - c0) * a.n_out; e += ET)
            a.coeff[((c0 + e / a.n_out) * a.n_out + e % a.n_out) * a.ndl_stride + d] = 0.0;
        return;
    }
    extern __shared__ double sm[];
    double* M = sm;                                   // [n + n_out][PW_LD]: E, then the rows of P
    double* xv = M + (size_t)(64 + KR_MAX_OUT) * PW_LD;  // x_j
    double* yv = xv + 128;                            // [E; P] x_j
    double* part = yv + 128;                          // [2][128]
    const double* pwd = pw + (size_t)d * Q * PW_MAT;
    const double* Pd = a.P + (int64_t)d * a.n_out * k;
    const int R = n + a.n_out;
    for (int e = threadIdx.x; e < R * n; e += ET) {
        const int r = e / n, c = e - r * n;
        M[r * PW_LD + c] = r < n ? pwd[r * PW_LD + c] : Pd[(int64_t)(r - n) * k + c];
    }
    if (threadIdx.x < n) xv[threadIdx.x] = threadIdx.x == 0 ? 1.0 : 0.0;  // x_0 = e_1 exactly
    __syncthreads();
    for (int q = 0; q < Q; ++q)  // x_{c0} = prod over the set bits of c0 of E^{2^q}, applied to e_1
        if ((c0 >> q) & 1) {
            mv_rows(pwd + (size_t)q * PW_MAT, n, n, xv, part, yv);
            if (threadIdx.x < n) xv[threadIdx.x] = yv[threadIdx.x];
            __syncthreads();
        }
    const double bz = a.beta0[d];
    for (int64_t j = c0; j < c1; ++j) {
        mv_rows(M, R, n, xv, part, yv);  // yv[0..n) = E x_j = x_{j+1}, yv[n + r] = (P x_j)_r
        if (threadIdx.x < a.n_out) a.coeff[(j * a.n_out + threadIdx.x) * a.ndl_stride + d] = bz * yv[n + threadIdx.x];
        if (threadIdx.x == 0) a.hlast[(int64_t)d * np1 + j] = xv[n - 1];
        __syncthreads();
        if (threadIdx.x < n) xv[threadIdx.x] = yv[threadIdx.x];
        __syncthreads();
    }
}

// Lemma 1: beta0 h_{k+1,k} e^{max(mu,0) T} int_0^T |x_k(t)| dt, trapezoid on the t_j grid. One CTA per
// direction: each thread sums a contiguous run of trapezoids, the runs are combined in thread order (fixed order,
// bit-reproducible; a serial per-thread loop over 2000 dependent loads was ~0.25 ms).
__global__ void __launch_bounds__(256) lemma_kernel(const double* hlast, const double* beta0, const double* hnext,
                                                    const int32_t* keff, int64_t n_steps, double step, double mu,
                                                    double* lemma) {
    const int d = blockIdx.x;
    __shared__ double red[256];
    if (keff[d] <= 0) {
        if (threadIdx.x == 0) lemma[d] = 0.0;
        return;
    }
    const double* h = hlast + (int64_t)d * (n_steps + 1);
    const int64_t per = (n_steps + 255) / 256;
    const int64_t j0 = threadIdx.x * per, j1 = min(j0 + per, n_steps);
    double s = 0.0;
    for (int64_t j = j0; j < j1; ++j) s += 0.5 * step * (fabs(h[j]) + fabs(h[j + 1]));
    red[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double integral = 0.0;
        for (int t = 0; t < 256; ++t) integral += red[t];
        const double T = (double)n_steps * step;
        // an exact breakdown (h_{k+1,k} = 0) gives 0 even when e^{mu T} overflows (no 0 * inf = NaN)
        const double base = beta0[d] * hnext[d] * integral;
        lemma[d] = base == 0.0 ? 0.0 : base * exp(fmax(mu, 0.0) * T);
    }
}

}  // namespace

void kr_expm_prepare(kr_handle* h) {
    // the attribute is a per-kernel, process-wide maximum: always the largest (k = 64) size, so that handles of
    // different k (and the large route's small checkpoints) never lower it under each other
    const size_t smem = (size_t)6 * 64 * 65 * sizeof(double);
    KR_CUDA(cudaFuncSetAttribute(expm_project_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    KR_CUDA(cudaFuncSetAttribute(expm_doubling_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    h->expm_doubling = getenv("KR_EXPM_PADE") == nullptr;  // KR_EXPM_PADE=1: one Pade-13 per (step, direction)
    h->expm_onecta = getenv("KR_EXPM_ONECTA") != nullptr;  // KR_EXPM_ONECTA=1: the one-CTA doubling kernel
    if (h->expm_doubling && !h->expm_onecta) {
        int Q = 1;
        while (((int64_t)1 << Q) <= h->n_steps) ++Q;
        h->pw_q = Q;
        const size_t ndl = std::max<size_t>(1, h->my_dirs.size());
        KR_CUDA(kr_dev_malloc(reinterpret_cast<void**>(&h->d_pw), ndl * Q * PW_MAT * sizeof(double)));
        h->extra_allocs.push_back(h->d_pw);
        KR_CUDA(cudaFuncSetAttribute(expm_powers_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const size_t msm = ((size_t)(64 + KR_MAX_OUT) * PW_LD + 512) * sizeof(double);
        KR_CUDA(cudaFuncSetAttribute(expm_march_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msm));
    } else if (h->expm_doubling) {
        int ldx = 1;
        while (ldx < h->n_steps + 1) ldx <<= 1;
        h->xt_ld = ldx;
        KR_CUDA(kr_dev_malloc(reinterpret_cast<void**>(&h->d_xt),
                              (size_t)std::max<size_t>(1, h->my_dirs.size()) * 64 * ldx * sizeof(double)));
        h->extra_allocs.push_back(h->d_xt);
    }
}

// One direction at dimension kc <= 64 through the doubling kernel (the large-k route's small checkpoints):
// Hdense [kc][kc] on the device, trajectory scratch xt [64][ldx]; writes the coefficients of local
// direction dl and hlast. One launch.
void kr_expm_small_eval(kr_handle* h, int dl, int kc, const double* Hdense, int hstride, double* xt, int ldx) {
    const size_t smem = (size_t)6 * 64 * 65 * sizeof(double);
    KR_CUDA(cudaFuncSetAttribute(expm_doubling_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int ndl = (int)h->my_dirs.size();
    ExpmArgs a;
    a.H = nullptr;
    a.P = h->d_P;
    a.beta0 = h->d_beta0;
    a.keff = h->d_keff;
    a.k = h->k;
    a.n_out = h->n_out;
    a.ndl_stride = (h->part == KR_PART_DIRS && h->world > 1) ? (int)((h->n_dir + h->world - 1) / h->world) : ndl;
    a.n_steps = h->n_steps;
    a.step = h->step;
    a.coeff = h->d_coeff_loc;
    a.hlast = h->d_hlast;
    a.dsel = dl;
    a.nfix = kc;
    a.Hsrc = Hdense;
    a.hstride = hstride;
    if (h->d_pw && !h->expm_onecta) {
        // E = e^{H delta} and its powers in one CTA, then the time grid over many CTAs (as kr_expm_enqueue): the
        // one-CTA doubling took ~0.3 ms per checkpoint on one SM (81% of the paper-heat m = 100 adaptive run)
        expm_powers_kernel<<<1, ET, (size_t)6 * kc * (kc + 1) * sizeof(double), h->stream>>>(a, h->d_pw, h->pw_q);
        KR_CUDA(cudaGetLastError());
        h->launches++;
        const int64_t np1 = h->n_steps + 1;
        const int64_t B = std::max<int64_t>(8, (np1 + 443) / 444);
        const unsigned nseg = (unsigned)((np1 + B - 1) / B);
        const size_t msm = ((size_t)(64 + KR_MAX_OUT) * PW_LD + 512) * sizeof(double);
        expm_march_kernel<<<dim3(nseg, 1), ET, msm, h->stream>>>(a, h->d_pw, h->pw_q, (int)B);
    } else {
        expm_doubling_kernel<<<1, ET, (size_t)6 * kc * (kc + 1) * sizeof(double), h->stream>>>(a, xt, ldx);
    }
    KR_CUDA(cudaGetLastError());
    h->launches++;
}

void kr_expm_enqueue(kr_handle* h) {
    const int ndl = (int)h->my_dirs.size();
    if (ndl == 0) return;
    const int k = h->k;
    const size_t smem = (size_t)6 * k * (k + 1) * sizeof(double);
    ExpmArgs a;
    a.H = h->d_H;
    a.P = h->d_P;
    a.beta0 = h->d_beta0;
    a.keff = h->d_keff;
    a.k = k;
    a.n_out = h->n_out;
    a.ndl_stride = (h->part == KR_PART_DIRS && h->world > 1) ? (int)((h->n_dir + h->world - 1) / h->world) : ndl;
    a.n_steps = h->n_steps;
    a.step = h->step;
    a.coeff = h->d_coeff_loc;
    a.hlast = h->d_hlast;
    if (h->expm_doubling && !h->expm_onecta) {
        expm_powers_kernel<<<ndl, ET, smem, h->stream>>>(a, h->d_pw, h->pw_q);
        KR_CUDA(cudaGetLastError());
        h->launches++;
        // columns per CTA: about three CTAs per SM over all directions, at least 8 columns each
        const int64_t np1 = h->n_steps + 1;
        int64_t B = std::max<int64_t>(8, (np1 * ndl + 443) / 444);
        if (const char* e = getenv("KR_EXPM_B")) B = std::max(1, atoi(e));
        const unsigned nseg = (unsigned)((np1 + B - 1) / B);
        const size_t msm = ((size_t)(64 + KR_MAX_OUT) * PW_LD + 512) * sizeof(double);
        expm_march_kernel<<<dim3(nseg, ndl), ET, msm, h->stream>>>(a, h->d_pw, h->pw_q, (int)B);
    } else if (h->expm_doubling)
        expm_doubling_kernel<<<ndl, ET, smem, h->stream>>>(a, h->d_xt, h->xt_ld);
    else
        expm_project_kernel<<<dim3((unsigned)(h->n_steps + 1), ndl), ET, smem, h->stream>>>(a);
    KR_CUDA(cudaGetLastError());
    h->launches++;
    lemma_kernel<<<ndl, 256, 0, h->stream>>>(h->d_hlast, h->d_beta0, h->d_hnext, h->d_keff, h->n_steps, h->step,
                                             h->mu, h->d_lemma);
    KR_CUDA(cudaGetLastError());
    h->launches++;
}
