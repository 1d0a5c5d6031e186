// kr_arnoldi.cu — stored-basis Arnoldi with the whole GPU: the batched CSR SpMM of C2 (21 directions,
// SURVEY §8(a) a2-C / a3-A) and the lifted, nonsymmetric heat-with-heater system at 10^6 states (§8(f) NEXT-4,
// PAPER.md:1133-1147) — any stored-basis Arnoldi whose basis does not fit one CTA, or that has enough
// directions x rows to fill the GPU.
//
// Alg. 1 orthogonalises w = A v_{j-1} against every previous basis vector. MGS's j
// dependent dot/axpy pairs per step would be j grid-wide round trips; here the projection is classical
// Gram-Schmidt applied twice (CGS2: h = V^T w, w -= V h, repeated once), which is as accurate as MGS
// (orthogonality to O(eps)); the oracle keeps the paper's MGS — the difference is rounding.
//
// Every CTA owns one chunk of rows of one direction (grid = chunks x directions, sized to ~4 CTAs per SM).
// One Krylov step j >= 1 is four kernels, each ONE streaming pass over the basis rows of its chunk:
//   K1 apply_dots:   w = A v_{j-1} (CSR row or 7-point stencil cell per thread; long CSR rows by the whole
//                    CTA) fused with the first projection pass part1[b][l] = sum_{i in b} V[l][i] w[i];
//                    CTA 0 of each direction also finalises P[., j-1] = C v_{j-1} (Alg. 4's projection).
//   K2 update_dots:  h1 = sum_b part1[b] (chunk order); w' = w - V h1 fused with the second pass
//                    part2[b][l] = sum_{i in b} V[l][i] w'[i]  (the rows were just read: L1 / L2 hits).
//   K3 update_norm:  h2 = sum_b part2[b]; w'' = w' - V h2; H[., j-1] = h1 + h2; partials of ||w''||^2.
//   K4 normalize:    h_{j,j-1} = ||w''|| (chunk order), the breakdown test, v_j = w'' / h_{j,j-1},
//                    partials of C v_j.
// Every CTA recomputes the scalars it needs from the per-chunk partials in the same fixed order (no
// separate reduce kernels unless j x chunks is large), so results are bit-reproducible and no kernel
// reads a value another CTA of the same kernel writes.
#include <float.h>

#include <algorithm>

#include "kr_internal.h"

namespace {

constexpr int CT = 256;           // threads per CTA
constexpr int QB = 8;             // vectors per batched block reduction
constexpr int MAXCHUNK = 2048;    // rows per CTA (the chunk's w lives in shared memory)
constexpr int RED_INLINE = 4096;  // j x chunks above which a separate reduce kernel sums the partials

struct CgsArgs {
    double* V;  // [ndl][k+1][N]
    double* W;  // [ndl][N]
    int64_t N;
    int k, j;
    int64_t chunk;
    int nchunk;
    double* part;  // [ndl][nchunk][pstride]: D1 = 0 (k+1), D2 = k+1 (k+1), NRM = 2(k+1), PJ = 2(k+1)+1 (n_out)
    int pstride;
    double* hv;     // [ndl][2][k+1] reduced h per pass (separate-reduce mode)
    double* hmax2;  // [ndl][2] running max |H| entry, double-buffered by step parity
    int red_sep;
    double* H;  // [ndl][k+1][k]
    double* P;  // [ndl][n_out][k]
    const double* O;  // [n_out][N]
    int n_out;
    double* beta0;
    double* hnext;
    int32_t* keff;
    int32_t* done;
    int32_t* status;
    // operator: CSR (A' = [[A, b], [0, 0]] when lifted) ...
    const int64_t* rp;
    const int32_t* ci;
    const double* val;
    const double* b;
    int64_t n;
    const int64_t* longr;
    int n_long;
    int prew;  // CSR: w = A v_{j-1} already in W (the block SpMM, kr_csr_spmm), all rows including long ones
    // ... or the 7-point stencil with per-face corrections and the lifted affine column bl
    int64_t mx, my, mz;
    double cx, cy, cz;
    FaceCor fc;
    const double* bl;
};

__device__ __forceinline__ int64_t poff(const CgsArgs& a, int d, int b) {
    return ((int64_t)d * a.nchunk + b) * a.pstride;
}

// fixed-order reduction of QB per-thread sums at once: warp shuffles, then warps 0..7 in order; out[q], q < nq
__device__ __forceinline__ void block_reduce_q(double (&s)[QB], double* red, double* out, int nq) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < QB; ++q) {
        double v = s[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (lane == 0) red[wid * QB + q] = v;
    }
    __syncthreads();
    if ((int)threadIdx.x < nq) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < CT / 32; ++w) t += red[w * QB + threadIdx.x];
        out[threadIdx.x] = t;
    }
    __syncthreads();
}

__device__ __forceinline__ double block_reduce_1(double v, double* red) {  // valid on thread 0
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < CT / 32; ++w) t += red[w];
    __syncthreads();
    return t;
}

// out[q] = sum over the chunk rows of M[m0 + q][i] * xs[i - i0], q < nq; thread t owns rows i0 + t + CT m
__device__ __forceinline__ void chunk_dots(const double* __restrict__ M, int64_t ld, int m0, int nq,
                                           const double* xs, int64_t i0, int64_t i1, double* red, double* out) {
    double s[QB];
#pragma unroll
    for (int q = 0; q < QB; ++q) s[q] = 0.0;
    const double* Mb = M + (int64_t)m0 * ld;
    if (nq == QB) {
        for (int64_t i = i0 + threadIdx.x; i < i1; i += CT) {
            const double xi = xs[i - i0];
            double v[QB];
#pragma unroll
            for (int q = 0; q < QB; ++q) v[q] = Mb[(int64_t)q * ld + i];
#pragma unroll
            for (int q = 0; q < QB; ++q) s[q] = fma(v[q], xi, s[q]);
        }
    } else {
        for (int64_t i = i0 + threadIdx.x; i < i1; i += CT) {
            const double xi = xs[i - i0];
#pragma unroll
            for (int q = 0; q < QB; ++q)
                if (q < nq) s[q] = fma(Mb[(int64_t)q * ld + i], xi, s[q]);
        }
    }
    block_reduce_q(s, red, out, nq);
}

// w[i] -= sum_{l<j} V[l][i] hs[l] (accumulated in l order) for the thread's rows; ws = the new w; returns the
// thread's sum of new w^2 (used by the second pass)
__device__ __forceinline__ double chunk_update(const double* __restrict__ V, int64_t N, int j, const double* hs,
                                              double* w, double* ws, int64_t i0, int64_t i1) {
    double s2 = 0.0;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += 2 * CT) {
        const bool two = i + CT < i1;
        double a0 = 0.0, a1 = 0.0;
        const double* Vi = V + i;
        int l = 0;
        for (; l + 4 <= j; l += 4) {
            double v0[4], v1[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                v0[u] = Vi[(int64_t)(l + u) * N];
                v1[u] = two ? Vi[(int64_t)(l + u) * N + CT] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                a0 = fma(v0[u], hs[l + u], a0);
                a1 = fma(v1[u], hs[l + u], a1);
            }
        }
        for (; l < j; ++l) {
            a0 = fma(Vi[(int64_t)l * N], hs[l], a0);
            if (two) a1 = fma(Vi[(int64_t)l * N + CT], hs[l], a1);
        }
        const double y0 = w[i] - a0;
        w[i] = y0;
        ws[i - i0] = y0;
        s2 = fma(y0, y0, s2);
        if (two) {
            const double y1 = w[i + CT] - a1;
            w[i + CT] = y1;
            ws[i + CT - i0] = y1;
            s2 = fma(y1, y1, s2);
        }
    }
    return s2;
}

// sum over the chunks of a per-chunk partial (stride doubles apart), by one warp: lane t sums chunks t, t + 32, ...
// in order, a shuffle tree adds the lanes, lane 0's value is broadcast (the same association on every lane and in
// every CTA that computes it: bit-identical). All 32 lanes must call it.
__device__ __forceinline__ double chunk_sum_warp(const double* p, int nchunk, int64_t stride) {
    const int lane = threadIdx.x & 31;
    double s = 0.0;
    for (int c = lane; c < nchunk; c += 32) s += p[(int64_t)c * stride];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    return __shfl_sync(0xffffffffu, s, 0);
}

// hs[l] = h of pass `pass` for l < j: from the reduce kernel, or summed here over the chunks in order
__device__ __forceinline__ void load_h(const CgsArgs& a, int d, int pass, double* hs) {
    const int j = a.j;
    if (a.red_sep) {
        const double* hv = a.hv + ((int64_t)d * 2 + pass) * (a.k + 1);
        for (int l = threadIdx.x; l < j; l += CT) hs[l] = hv[l];
    } else {
        const int off = pass == 0 ? 0 : a.k + 1;
        for (int l = threadIdx.x; l < j; l += CT) {
            const double* p = a.part + poff(a, d, 0) + off + l;
            double s = 0.0;
#pragma unroll 8
            for (int b = 0; b < a.nchunk; ++b) s += p[(int64_t)b * a.pstride];
            hs[l] = s;
        }
    }
    __syncthreads();
}

// sum_e val[e] x[ci[e]] in entry order; entries fetched 4 at a time so the gathers of a row are in flight together
__device__ __forceinline__ double csr_row(const CgsArgs& a, const double* __restrict__ x, int64_t r) {
    double s = 0.0;
    const int64_t e1 = a.rp[r + 1];
    for (int64_t e = a.rp[r]; e < e1; e += 4) {
        double v[4], xv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const bool in = e + u < e1;
            v[u] = in ? a.val[e + u] : 0.0;
            xv[u] = in ? __ldg(&x[a.ci[e + u]]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (e + u < e1) s = fma(v[u], xv[u], s);
    }
    if (a.b) s = fma(a.b[r], x[a.n], s);
    return s;
}

__device__ __forceinline__ double stencil_row(const CgsArgs& a, const double* __restrict__ u, int64_t c) {
    const int64_t mx = a.mx, my = a.my, mz = a.mz;
    const int64_t z = c / (mx * my), rem = c - z * mx * my;
    const int64_t yy = rem / mx, x = rem - yy * mx;
    const double diag = 2.0 * (a.cx + a.cy + a.cz);
    const double sx = (x > 0 ? u[c - 1] : 0.0) + (x < mx - 1 ? u[c + 1] : 0.0);
    const double sy = (yy > 0 ? u[c - mx] : 0.0) + (yy < my - 1 ? u[c + mx] : 0.0);
    const double sz = (z > 0 ? u[c - mx * my] : 0.0) + (z < mz - 1 ? u[c + mx * my] : 0.0);
    const double dg = diag - (x == 0 ? a.fc.e[0] : 0.0) - (x == mx - 1 ? a.fc.e[1] : 0.0) -
                      (yy == 0 ? a.fc.e[2] : 0.0) - (yy == my - 1 ? a.fc.e[3] : 0.0) -
                      (z == 0 ? a.fc.e[4] : 0.0) - (z == mz - 1 ? a.fc.e[5] : 0.0);
    double v = a.cx * sx + a.cy * sy + a.cz * sz - dg * u[c];
    if (a.bl) v = fma(a.bl[c], u[a.n], v);  // lifted affine term: y = A u + b u_n
    return v;
}

struct Smem {  // dynamic shared memory layout: ws[chunk] | red[CT/32 * QB] | hs[k+1]
    double* ws;
    double* red;
    double* hs;
};
__device__ __forceinline__ Smem smem_layout(const CgsArgs& a) {
    extern __shared__ double sm[];
    Smem s;
    s.ws = sm;
    s.red = sm + a.chunk;
    s.hs = s.red + (CT / 32) * QB;
    return s;
}

// K1: w = A v_{j-1} for the chunk rows, then part1[b][l] = sum_i V[l][i] w[i], l < j; CTA 0 finalises P[., j-1]
template <int STENCIL>
__global__ void __launch_bounds__(CT) cgs_apply_dots_kernel(CgsArgs a) {
    const int d = blockIdx.y;
    if (a.done[d]) return;
    const Smem S = smem_layout(a);
    const int b = blockIdx.x, j = a.j;
    const int64_t N = a.N, i0 = (int64_t)b * a.chunk, i1 = min(i0 + a.chunk, N);
    if (b == 0)  // P[., j-1] = C v_{j-1}: a warp per output row over the chunk partials
        for (int r = threadIdx.x >> 5; r < a.n_out; r += CT / 32) {
            const double s = chunk_sum_warp(a.part + poff(a, d, 0) + 2 * (a.k + 1) + 1 + r, a.nchunk, a.pstride);
            if ((threadIdx.x & 31) == 0) a.P[((int64_t)d * a.n_out + r) * a.k + (j - 1)] = s;
        }
    const double* Vd = a.V + (int64_t)d * (a.k + 1) * N;
    const double* x = Vd + (int64_t)(j - 1) * N;
    double* w = a.W + (int64_t)d * N;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += CT) {
        double y = 0.0;
        if (!STENCIL && a.prew) {
            y = w[i];
        } else if (i < a.n) {  // the lifted row n of A' is zero
            if (STENCIL) {
                y = stencil_row(a, x, i);
            } else {
                if (a.rp[i + 1] - a.rp[i] > KR_LONG_ROW) continue;  // below, by the whole CTA
                y = csr_row(a, x, i);
            }
        }
        w[i] = y;
        S.ws[i - i0] = y;
    }
    if (!STENCIL && !a.prew)
        for (int q = 0; q < a.n_long; ++q) {  // long rows (e.g. the b^T row of a transposed lift)
            const int64_t r = a.longr[q];
            if (r < i0 || r >= i1) continue;
            double s = 0.0;  // thread t sums entries t, t + CT, ... in order, 8 gathers in flight
            const int64_t e1 = a.rp[r + 1];
            for (int64_t e = a.rp[r] + threadIdx.x; e < e1; e += 8 * CT) {
                double v[8], xv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const bool in = e + u * CT < e1;
                    v[u] = in ? a.val[e + u * CT] : 0.0;
                    xv[u] = in ? __ldg(&x[a.ci[e + u * CT]]) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (e + u * CT < e1) s = fma(v[u], xv[u], s);
            }
            double t = block_reduce_1(s, S.red);
            if (threadIdx.x == 0) {
                if (a.b) t = fma(a.b[r], x[a.n], t);
                w[r] = t;
                S.ws[r - i0] = t;
            }
        }
    __syncthreads();
    double* out = a.part + poff(a, d, b);
    for (int lb = 0; lb < j; lb += QB) chunk_dots(Vd, N, lb, min(QB, j - lb), S.ws, i0, i1, S.red, out + lb);
}

// K2: w' = w - V h1 and part2[b][l] = sum_i V[l][i] w'[i]; CTA 0 writes H[., j-1] = h1
__global__ void __launch_bounds__(CT) cgs_update_dots_kernel(CgsArgs a) {
    const int d = blockIdx.y;
    if (a.done[d]) return;
    const Smem S = smem_layout(a);
    const int b = blockIdx.x, j = a.j;
    const int64_t N = a.N, i0 = (int64_t)b * a.chunk, i1 = min(i0 + a.chunk, N);
    load_h(a, d, 0, S.hs);
    double* H = a.H + (int64_t)d * (a.k + 1) * a.k;
    if (b == 0)
        for (int l = threadIdx.x; l < j; l += CT) H[(int64_t)l * a.k + (j - 1)] = S.hs[l];
    const double* Vd = a.V + (int64_t)d * (a.k + 1) * N;
    (void)chunk_update(Vd, N, j, S.hs, a.W + (int64_t)d * N, S.ws, i0, i1);
    double* out = a.part + poff(a, d, b) + (a.k + 1);
    for (int lb = 0; lb < j; lb += QB) chunk_dots(Vd, N, lb, min(QB, j - lb), S.ws, i0, i1, S.red, out + lb);
}

// K3: w'' = w' - V h2; H[., j-1] += h2; partials of ||w''||^2
__global__ void __launch_bounds__(CT) cgs_update_norm_kernel(CgsArgs a) {
    const int d = blockIdx.y;
    if (a.done[d]) return;
    const Smem S = smem_layout(a);
    const int b = blockIdx.x, j = a.j;
    const int64_t N = a.N, i0 = (int64_t)b * a.chunk, i1 = min(i0 + a.chunk, N);
    load_h(a, d, 1, S.hs);
    double* H = a.H + (int64_t)d * (a.k + 1) * a.k;
    if (b == 0)
        for (int l = threadIdx.x; l < j; l += CT) {
            double& hl = H[(int64_t)l * a.k + (j - 1)];
            hl = hl + S.hs[l];
        }
    const double* Vd = a.V + (int64_t)d * (a.k + 1) * N;
    const double s2 = chunk_update(Vd, N, j, S.hs, a.W + (int64_t)d * N, S.ws, i0, i1);
    const double t = block_reduce_1(s2, S.red);
    if (threadIdx.x == 0) a.part[poff(a, d, b) + 2 * (a.k + 1)] = t;
}

// ||v_0||^2 partials of the start vector (j == 0)
__global__ void __launch_bounds__(CT) cgs_norm_kernel(CgsArgs a) {
    const int d = blockIdx.y;
    if (a.done[d]) return;
    __shared__ double red[CT / 32];
    const int b = blockIdx.x;
    const double* w = a.V + (int64_t)d * (a.k + 1) * a.N;
    const int64_t i0 = (int64_t)b * a.chunk, i1 = min(i0 + a.chunk, a.N);
    double s2 = 0.0;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += CT) s2 = fma(w[i], w[i], s2);
    const double t = block_reduce_1(s2, red);
    if (threadIdx.x == 0) a.part[poff(a, d, b) + 2 * (a.k + 1)] = t;
}

// K4: h_{j,j-1} = ||w|| (chunk order, every CTA), breakdown test / k_eff (CTA 0 writes the state), v_j = w / ||w||,
// partials of C v_j. j == 0 normalises the start vector in place (beta0).
__global__ void __launch_bounds__(CT) cgs_normalize_kernel(CgsArgs a) {
    const int d = blockIdx.y;
    if (a.done[d]) return;  // stopped (breakdown / k reached) at an earlier step: no new vector
    const Smem S = smem_layout(a);
    __shared__ double s_inv;
    __shared__ int s_go;
    const int b = blockIdx.x, j = a.j, k = a.k;
    const bool lead = b == 0;
    double s2 = 0.0;
    if (threadIdx.x < 32) s2 = chunk_sum_warp(a.part + poff(a, d, 0) + 2 * (k + 1), a.nchunk, a.pstride);
    if (threadIdx.x == 0) {
        const double nb = sqrt(s2);
        int go = 1;
        if (j == 0) {
            if (lead) {
                a.beta0[d] = nb;
                a.keff[d] = 1;
                a.hmax2[2 * d] = 0.0;
            }
            if (!(nb > 0.0) || !isfinite(nb)) {
                go = 0;
                if (lead) {
                    a.done[d] = 1;
                    a.keff[d] = 0;
                    a.status[d] = nb == 0.0 ? KR_EZERO : KR_ENONFINITE;
                }
            }
        } else {
            const double* H = a.H + (int64_t)d * (k + 1) * k;
            double hm = a.hmax2[2 * d + ((j - 1) & 1)];
            for (int l = 0; l < j; ++l) hm = fmax(hm, fabs(H[(int64_t)l * k + (j - 1)]));
            if (lead) a.H[(int64_t)d * (k + 1) * k + (int64_t)j * k + (j - 1)] = nb;
            if (!isfinite(nb)) {
                go = 0;
                if (lead) {
                    a.done[d] = 1;
                    a.status[d] = KR_ENONFINITE;
                }
            } else if (nb == 0.0 || nb <= 16.0 * DBL_EPSILON * hm || j == k) {  // breakdown / last column
                go = 0;
                if (lead) {
                    a.done[d] = 1;
                    a.keff[d] = j;
                    a.hnext[d] = nb;
                }
            } else if (lead) {
                a.hmax2[2 * d + (j & 1)] = fmax(hm, nb);
                a.keff[d] = j + 1;
            }
        }
        s_go = go;
        s_inv = go ? 1.0 / nb : 0.0;
    }
    __syncthreads();
    if (!s_go) return;
    const double inv = s_inv;
    const int64_t N = a.N, i0 = (int64_t)b * a.chunk, i1 = min(i0 + a.chunk, N);
    double* Vd = a.V + (int64_t)d * (k + 1) * N;
    const double* w = j == 0 ? Vd : a.W + (int64_t)d * N;
    double* vj = Vd + (int64_t)j * N;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += CT) {
        const double v = w[i] * inv;
        vj[i] = v;
        S.ws[i - i0] = v;
    }
    double* out = a.part + poff(a, d, b) + 2 * (k + 1) + 1;
    for (int rb = 0; rb < a.n_out; rb += QB) chunk_dots(a.O, N, rb, min(QB, a.n_out - rb), S.ws, i0, i1, S.red, out + rb);
}

// separate-reduce mode: hv[d][pass][l] = sum_b part[d][b][pass (k+1) + l] — a warp per l: lane t sums the chunks
// t, t + 32, ... in order, then a shuffle tree (fixed order: bit-reproducible). One thread per l summing ~600 chunks
// in sequence was latency-bound (84 us per call on the heater, 13% of its Arnoldi time).
__global__ void __launch_bounds__(256) cgs_reduce_kernel(CgsArgs a, int pass) {
    const int d = blockIdx.y;
    if (a.done[d]) return;
    const int lane = threadIdx.x & 31;
    const int l = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (l >= a.j) return;
    const double* p = a.part + poff(a, d, 0) + pass * (a.k + 1) + l;
    double s = 0.0;
    for (int b = lane; b < a.nchunk; b += 32) s += p[(int64_t)b * a.pstride];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) a.hv[((int64_t)d * 2 + pass) * (a.k + 1) + l] = s;
}

struct Geo {
    int64_t chunk;
    int nchunk;
};
Geo geometry(int64_t N, int ndl) {
    // ~4 CTAs per SM over all directions, at most MAXCHUNK rows per CTA, chunks a multiple of 32 rows
    const int64_t want = std::max<int64_t>(1, (148 * 4 + ndl - 1) / std::max(1, ndl));
    int64_t chunk = (N + want - 1) / want;
    chunk = std::min<int64_t>(MAXCHUNK, std::max<int64_t>(256, (chunk + 31) / 32 * 32));
    Geo g;
    g.chunk = chunk;
    g.nchunk = (int)((N + chunk - 1) / chunk);
    return g;
}

// at most (2048 + 64 + KR_K_MAX_ARNOLDI + 1) doubles = 33 KB: below the 48 KB default, no attribute needed
size_t smem_bytes(int64_t chunk, int k) { return (size_t)(chunk + (CT / 32) * QB + k + 1) * sizeof(double); }

}  // namespace

size_t kr_cgs_scratch_doubles(const kr_handle* h, int ndl) {
    const Geo g = geometry(h->N, ndl);
    const size_t pstride = 2 * (size_t)(h->k + 1) + 1 + KR_MAX_OUT;
    return (size_t)ndl * g.nchunk * pstride + (size_t)ndl * 2 * (h->k + 1) + 2 * (size_t)ndl;
}

// One Krylov step of the large-N stored-basis path with the semantics of the one-CTA MGS kernel: j == 0
// normalises the start vectors (beta0); j >= 1 applies the operator to v_{j-1} and orthogonalises, writing
// H[., j-1], h_{j,j-1}, the breakdown flag / k_eff and v_j. P[., j-1] is finalised by step j's first kernel, so
// after step j the columns P[., 0..j-1] are final (all that a Krylov dimension of j uses).
void kr_cgs_step(kr_handle* h, int j, int ndl, double* scratch) {
    const Geo g = geometry(h->N, ndl);
    CgsArgs a{};
    a.V = h->d_V;
    a.W = h->d_W;
    a.N = h->N;
    a.k = h->k;
    a.j = j;
    a.chunk = g.chunk;
    a.nchunk = g.nchunk;
    a.pstride = 2 * (h->k + 1) + 1 + KR_MAX_OUT;
    a.part = scratch;
    a.hv = scratch + (size_t)ndl * a.nchunk * a.pstride;
    a.hmax2 = a.hv + (size_t)ndl * 2 * (h->k + 1);
    a.red_sep = (int64_t)j * a.nchunk > RED_INLINE ? 1 : 0;
    a.H = h->d_H;
    a.P = h->d_P;
    a.O = h->d_O;
    a.n_out = h->n_out;
    a.beta0 = h->d_beta0;
    a.hnext = h->d_hnext;
    a.keff = h->d_keff;
    a.done = h->d_done;
    a.status = h->d_status;
    a.rp = h->d_rp;
    a.ci = h->d_ci;
    a.val = h->d_val;
    a.b = h->d_b;
    a.n = h->n;
    a.longr = h->d_long;
    a.n_long = (int)h->n_long;
    a.mx = h->mx;
    a.my = h->my;
    a.mz = h->mz;
    a.cx = h->cx;
    a.cy = h->cy;
    a.cz = h->cz;
    a.fc = kr_face_cor(h);
    a.bl = h->d_bl;
    cudaStream_t st = h->stream;
    const dim3 grid(a.nchunk, ndl);
    const size_t sm = smem_bytes(a.chunk, h->k);
    auto chk = [&]() {
        KR_CUDA(cudaGetLastError());
        h->launches++;
    };
    if (j == 0) {
        cgs_norm_kernel<<<grid, CT, 0, st>>>(a);
        chk();
    } else {
        if (h->op == KR_OP_CSR) {
            // A streamed once for all directions (block SpMM into W), then the first projection pass
            // (below 8 directions the operator stays fused into the first pass: C2T, 3 simulations, 2.35 vs 3.4 ms)
            a.prew = (ndl >= 8 && !getenv("KR_SPMM_PER_DIR")) ? 1 : 0;
            if (a.prew) kr_csr_spmm(h, h->d_V + (int64_t)(j - 1) * h->N, (int64_t)(h->k + 1) * h->N, h->d_W, h->N, ndl);
            cgs_apply_dots_kernel<0><<<grid, CT, sm, st>>>(a);
        } else {
            cgs_apply_dots_kernel<1><<<grid, CT, sm, st>>>(a);
        }
        chk();
        const dim3 rg((j + 7) / 8, ndl);  // a warp per h entry
        if (a.red_sep) {
            cgs_reduce_kernel<<<rg, 256, 0, st>>>(a, 0);
            chk();
        }
        cgs_update_dots_kernel<<<grid, CT, sm, st>>>(a);
        chk();
        if (a.red_sep) {
            cgs_reduce_kernel<<<rg, 256, 0, st>>>(a, 1);
            chk();
        }
        cgs_update_norm_kernel<<<grid, CT, sm, st>>>(a);
        chk();
    }
    cgs_normalize_kernel<<<grid, CT, sm, st>>>(a);
    chk();
}
