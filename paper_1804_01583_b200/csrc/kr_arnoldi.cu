// kr_arnoldi.cu — Arnoldi orthogonalisation for large operator dimension (the lifted,
// nonsymmetric heat-with-heater system at 10^6 states; any stored-basis Arnoldi whose
// N exceeds what one CTA holds).
//
// Alg. 1 orthogonalises w = A v_j against every previous basis vector. The one-CTA MGS
// kernel of kr_generic.cu keeps w on chip; beyond ~27k states the basis has to be streamed by the whole
// GPU, and MGS's j dependent dot/axpy pairs per step become j grid-wide round trips. Here the projection
// is classical Gram-Schmidt applied twice (CGS2: h = V^T w, w -= V h, repeated once), so each half-step is
// ONE streaming pass over the j basis vectors:
//   * dots:   part[b][l] = sum_{i in chunk b} V[l][i] w[i]   (grid = row chunks x blocks of 16 vectors)
//   * reduce: h[l] = sum_b part[b][l] in chunk order; H[l][j] accumulates h1 + h2
//   * update: w[i] -= sum_l V[l][i] h[l] (thread per row, coalesced over i), with sum w^2 partials on the
//     second pass; then h_{j+1,j} = ||w||, the breakdown test, v_{j+1} = w / h_{j+1,j} and
//     P[., j+1] = C v_{j+1} (Alg. 4's projection) in one more pass.
// Fixed chunking and fixed-order reductions: bit-reproducible. CGS2 is as accurate as MGS (orthogonality
// to O(eps)); the oracle keeps the paper's MGS — the difference is rounding.
#include <float.h>

#include <algorithm>

#include "kr_internal.h"

namespace {

constexpr int CT = 256;
constexpr int LB = 16;  // basis vectors per dots CTA

struct CgsArgs {
    double* V;         // [ndl][k+1][N]
    double* W;         // [ndl][N]
    int64_t N;
    int k, j;          // basis vectors v_0 .. v_{j-1} exist; w = A v_{j-1} (j >= 1), or v_0 itself (j == 0)
    int64_t chunk;     // rows per chunk
    int nchunk;
    double* part;      // [ndl][nchunk][k + 1 + KR_MAX_OUT]
    int pstride;
    double* hv;        // [ndl][k + 1] current projection coefficients
    double* H;         // [ndl][k+1][k]
    double* P;         // [ndl][n_out][k]
    const double* O;   // [n_out][N]
    int n_out;
    double* beta0;
    double* hnext;
    double* hmax;
    double* inv;       // [ndl] 1 / ||w||
    int32_t* keff;
    int32_t* done;
    int32_t* status;
};

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < CT / 32; ++w) r += red[w];
    __syncthreads();
    return r;  // valid on thread 0
}

// part[d][b][l] = sum_{i in chunk b} V[d][l][i] * w[d][i], l in [l0, l0 + LB) and l < j
__global__ void __launch_bounds__(CT) cgs_dots_kernel(CgsArgs a) {
    const int d = blockIdx.z;
    if (a.done[d]) return;
    const int b = blockIdx.x, l0 = blockIdx.y * LB;
    __shared__ double red[CT / 32];
    const double* V = a.V + (int64_t)d * (a.k + 1) * a.N;
    const double* w = a.W + (int64_t)d * a.N;
    const int64_t i0 = (int64_t)b * a.chunk, i1 = min(i0 + a.chunk, a.N);
    double s[LB];
#pragma unroll
    for (int q = 0; q < LB; ++q) s[q] = 0.0;
    const int nq = min(LB, a.j - l0);
    if (nq == LB) {  // full block: all LB basis loads of a row issued together
        for (int64_t i = i0 + threadIdx.x; i < i1; i += CT) {
            const double wi = w[i];
            double v[LB];
#pragma unroll
            for (int q = 0; q < LB; ++q) v[q] = __ldcs(&V[(int64_t)(l0 + q) * a.N + i]);
#pragma unroll
            for (int q = 0; q < LB; ++q) s[q] = fma(v[q], wi, s[q]);
        }
    } else {
        for (int64_t i = i0 + threadIdx.x; i < i1; i += CT) {
            const double wi = w[i];
#pragma unroll
            for (int q = 0; q < LB; ++q)
                if (q < nq) s[q] = fma(V[(int64_t)(l0 + q) * a.N + i], wi, s[q]);
        }
    }
    double* out = a.part + ((int64_t)d * a.nchunk + b) * a.pstride;
#pragma unroll
    for (int q = 0; q < LB; ++q) {
        if (l0 + q >= a.j) break;
        const double t = block_sum(s[q], red);
        if (threadIdx.x == 0) out[l0 + q] = t;
    }
}

// h[l] = sum_b part[b][l] (chunk order); H[l][j-1] (+)= h[l]; pass 0 stores, pass 1 accumulates
__global__ void cgs_reduce_kernel(CgsArgs a, int pass) {
    const int d = blockIdx.x;
    if (a.done[d]) return;
    double* H = a.H + (int64_t)d * (a.k + 1) * a.k;
    for (int l = threadIdx.x; l < a.j; l += blockDim.x) {
        double s = 0.0;
        for (int b = 0; b < a.nchunk; ++b) s += a.part[((int64_t)d * a.nchunk + b) * a.pstride + l];
        a.hv[(int64_t)d * (a.k + 1) + l] = s;
        double& hl = H[(int64_t)l * a.k + (a.j - 1)];
        hl = pass == 0 ? s : hl + s;
    }
}

// w[i] -= sum_l V[l][i] h[l]; with_norm: per-chunk partials of sum w^2 into part[b][k+1]
__global__ void __launch_bounds__(CT) cgs_update_kernel(CgsArgs a, int with_norm) {
    const int d = blockIdx.y;
    if (a.done[d]) return;
    const int b = blockIdx.x;
    __shared__ double red[CT / 32];
    __shared__ double hs[1024];
    const double* V = a.V + (int64_t)d * (a.k + 1) * a.N;
    double* w = a.W + (int64_t)d * a.N;
    const double* hv = a.hv + (int64_t)d * (a.k + 1);
    const int64_t i0 = (int64_t)b * a.chunk, i1 = min(i0 + a.chunk, a.N);
    double s2 = 0.0;
    for (int lb = 0; lb < a.j; lb += 1024) {  // h staged through shared memory in blocks of 1024
        const int ln = min(1024, a.j - lb);
        __syncthreads();
        for (int l = threadIdx.x; l < ln; l += CT) hs[l] = hv[lb + l];
        __syncthreads();
        // 4 rows per thread at a time, l unrolled: 16 independent basis loads in flight per thread
        for (int64_t ib = i0 + threadIdx.x; ib < i1; ib += 4 * CT) {
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            const double* Vb = V + (int64_t)lb * a.N + ib;
            int l = 0;
            for (; l + 4 <= ln; l += 4) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const double hl = hs[l + u];
                    const double* Vr = Vb + (int64_t)(l + u) * a.N;
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (ib + q * CT < i1) acc[q] = fma(__ldcs(Vr + q * CT), hl, acc[q]);
                }
            }
            for (; l < ln; ++l) {
                const double hl = hs[l];
                const double* Vr = Vb + (int64_t)l * a.N;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (ib + q * CT < i1) acc[q] = fma(Vr[q * CT], hl, acc[q]);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (ib + q * CT < i1) w[ib + q * CT] -= acc[q];
        }
    }
    if (with_norm) {
        __syncthreads();
        for (int64_t i = i0 + threadIdx.x; i < i1; i += CT) s2 = fma(w[i], w[i], s2);
        const double t = block_sum(s2, red);
        if (threadIdx.x == 0) a.part[((int64_t)d * a.nchunk + b) * a.pstride + a.k + 1] = t;
    }
}

// ||v_0|| partials for the start vector (j == 0): part[b][k+1]
__global__ void __launch_bounds__(CT) cgs_norm_kernel(CgsArgs a) {
    const int d = blockIdx.y;
    if (a.done[d]) return;
    const int b = blockIdx.x;
    __shared__ double red[CT / 32];
    const double* w = a.j == 0 ? a.V + (int64_t)d * (a.k + 1) * a.N : a.W + (int64_t)d * a.N;
    const int64_t i0 = (int64_t)b * a.chunk, i1 = min(i0 + a.chunk, a.N);
    double s2 = 0.0;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += CT) s2 = fma(w[i], w[i], s2);
    const double t = block_sum(s2, red);
    if (threadIdx.x == 0) a.part[((int64_t)d * a.nchunk + b) * a.pstride + a.k + 1] = t;
}

// h_{j,j-1} = ||w||, breakdown test, k_eff; 1/||w|| for the normalisation (one thread per direction)
__global__ void cgs_finalize_kernel(CgsArgs a) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= gridDim.x * blockDim.x || a.done[d]) return;
    double s = 0.0;
    for (int b = 0; b < a.nchunk; ++b) s += a.part[((int64_t)d * a.nchunk + b) * a.pstride + a.k + 1];
    const double nb = sqrt(s);
    const int j = a.j, k = a.k;
    double* H = a.H + (int64_t)d * (k + 1) * k;
    if (j == 0) {
        a.beta0[d] = nb;
        a.keff[d] = 1;
        a.hmax[d] = 0.0;
        if (!(nb > 0.0) || !isfinite(nb)) {
            a.done[d] = 1;
            a.keff[d] = 0;
            a.status[d] = nb == 0.0 ? KR_EZERO : KR_ENONFINITE;
            return;
        }
        a.inv[d] = 1.0 / nb;
        return;
    }
    double hm = a.hmax[d];
    for (int l = 0; l < j; ++l) hm = fmax(hm, fabs(H[(int64_t)l * k + (j - 1)]));
    H[(int64_t)j * k + (j - 1)] = nb;
    if (!isfinite(nb)) {
        a.done[d] = 1;
        a.status[d] = KR_ENONFINITE;
        return;
    }
    if (nb == 0.0 || nb <= 16.0 * DBL_EPSILON * hm || j == k) {  // breakdown or the extra column
        a.done[d] = 1;
        a.keff[d] = j;
        a.hnext[d] = nb;
        return;
    }
    a.hmax[d] = fmax(hm, nb);
    a.keff[d] = j + 1;
    a.inv[d] = 1.0 / nb;
}

// v_j = w / ||w|| and the per-chunk partials of C v_j (part[b][k+2+r])
__global__ void __launch_bounds__(CT) cgs_normalize_kernel(CgsArgs a) {
    const int d = blockIdx.y;
    if (a.done[d]) return;  // stopped (breakdown / k reached) at this or an earlier step: no new vector
    const int b = blockIdx.x;
    __shared__ double red[CT / 32];
    const double* w = a.j == 0 ? a.V + (int64_t)d * (a.k + 1) * a.N : a.W + (int64_t)d * a.N;
    double* vj = a.V + ((int64_t)d * (a.k + 1) + a.j) * a.N;
    const double inv = a.inv[d];
    const int64_t i0 = (int64_t)b * a.chunk, i1 = min(i0 + a.chunk, a.N);
    for (int64_t i = i0 + threadIdx.x; i < i1; i += CT) vj[i] = w[i] * inv;
    __syncthreads();
    for (int r = 0; r < a.n_out; ++r) {
        const double* Or = a.O + (int64_t)r * a.N;
        double t = 0.0;
        for (int64_t i = i0 + threadIdx.x; i < i1; i += CT) t = fma(Or[i], vj[i], t);
        const double s = block_sum(t, red);
        if (threadIdx.x == 0) a.part[((int64_t)d * a.nchunk + b) * a.pstride + a.k + 2 + r] = s;
    }
}

__global__ void cgs_project_kernel(CgsArgs a) {
    const int d = blockIdx.x;
    if (a.done[d]) return;
    for (int r = threadIdx.x; r < a.n_out; r += blockDim.x) {
        double s = 0.0;
        for (int b = 0; b < a.nchunk; ++b) s += a.part[((int64_t)d * a.nchunk + b) * a.pstride + a.k + 2 + r];
        a.P[((int64_t)d * a.n_out + r) * a.k + a.j] = s;
    }
}

}  // namespace

size_t kr_cgs_scratch_doubles(const kr_handle* h, int ndl) {
    const int64_t chunk = std::max<int64_t>(2048, (h->N + 148 * 4 - 1) / (148 * 4));
    const int64_t nchunk = (h->N + chunk - 1) / chunk;
    return (size_t)ndl * nchunk * (h->k + 2 + KR_MAX_OUT) + (size_t)ndl * (h->k + 1) + ndl;
}

// One Arnoldi step of the large-N path with the semantics of the one-CTA MGS kernel: j == 0 normalises the
// start vector (beta0, P[., 0]); j >= 1 orthogonalises w = A v_{j-1}, writes H[., j-1], h_{j,j-1}, the
// breakdown flag, v_j and P[., j]. `scratch` holds kr_cgs_scratch_doubles(h, ndl) doubles.
void kr_cgs_step(kr_handle* h, int j, int ndl, double* scratch) {
    CgsArgs a{};
    a.V = h->d_V;
    a.W = h->d_W;
    a.N = h->N;
    a.k = h->k;
    a.j = j;
    a.chunk = std::max<int64_t>(2048, (h->N + 148 * 4 - 1) / (148 * 4));
    a.nchunk = (int)((h->N + a.chunk - 1) / a.chunk);
    a.pstride = h->k + 2 + KR_MAX_OUT;
    a.part = scratch;
    a.hv = scratch + (size_t)ndl * a.nchunk * a.pstride;
    a.inv = a.hv + (size_t)ndl * (h->k + 1);
    a.H = h->d_H;
    a.P = h->d_P;
    a.O = h->d_O;
    a.n_out = h->n_out;
    a.beta0 = h->d_beta0;
    a.hnext = h->d_hnext;
    a.hmax = h->d_hmax;
    a.keff = h->d_keff;
    a.done = h->d_done;
    a.status = h->d_status;
    cudaStream_t st = h->stream;
    const dim3 rows(a.nchunk, ndl);
    auto chk = [&]() {
        KR_CUDA(cudaGetLastError());
        h->launches++;
    };
    if (j == 0) {
        cgs_norm_kernel<<<rows, CT, 0, st>>>(a);
        chk();
    } else {
        for (int pass = 0; pass < 2; ++pass) {  // CGS2
            cgs_dots_kernel<<<dim3(a.nchunk, (j + LB - 1) / LB, ndl), CT, 0, st>>>(a);
            chk();
            cgs_reduce_kernel<<<ndl, 256, 0, st>>>(a, pass);
            chk();
            cgs_update_kernel<<<rows, CT, 0, st>>>(a, pass == 1 ? 1 : 0);
            chk();
        }
    }
    cgs_finalize_kernel<<<1, ndl, 0, st>>>(a);
    chk();
    cgs_normalize_kernel<<<rows, CT, 0, st>>>(a);
    chk();
    cgs_project_kernel<<<ndl, 64, 0, st>>>(a);
    chk();
}
