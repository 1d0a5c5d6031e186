// kr_generic.cu — direction-batched Krylov iteration with a stored basis V (Arnoldi, Alg. 1,
// PAPER.md:617-635; or Lanczos, Alg. 3) for the CSR operator (optionally lifted,
// PAPER.md:157-165) and for small stencil problems; plus the vector fill kernels.
//
// Per Krylov step j, two launches for ALL directions of this rank:
//  1. the operator: W[d] = A V[d][j-1] — one CSR SpMM that streams A once for every direction
//     (thread per (row, direction)), or the matrix-free stencil;
//  2. orthogonalisation, one CTA (1024 threads) per direction: the new vector is held in registers
//     (EPT elements per thread), each previous basis vector is read ONCE per MGS iteration (dot, fixed
//     order block reduction, axpy from the same registers), then ||w||, breakdown, V[d][j] = w/||w||
//     and P[d][:, j] = C V[d][j] (Alg. 4's projection).
#include <float.h>

#include "kr_internal.h"

// ------------------------------------------------------------------------------------------------
// fills
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ double box_value(const DVec& v, int64_t x, int64_t y, int64_t z) {
    if (v.kind == KR_VEC_ALL) return v.value;
    if (v.kind == KR_VEC_BOX)
        return (x >= v.lo[0] && x < v.hi[0] && y >= v.lo[1] && y < v.hi[1] && z >= v.lo[2] && z < v.hi[2]) ? v.value
                                                                                                           : 0.0;
    return 0.0;
}

__global__ void fill_grid_kernel(double* dst, int64_t mx, int64_t my, int64_t pitch, int64_t nplanes, int64_t zbase,
                                 int64_t mz, DVec v) {
    const int64_t total = nplanes * my * pitch;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = e / (my * pitch), rem = e - b * my * pitch;
        const int64_t y = rem / pitch, x = rem - y * pitch;
        const int64_t gz = zbase + b;
        double val = 0.0;
        if (x < mx && gz >= 0 && gz < mz)
            val = v.kind == KR_VEC_RAND ? kr_rand_entry(v.seed, x + mx * (y + my * gz), v.value) : box_value(v, x, y, gz);
        dst[e] = val;
    }
}

__global__ void scatter_grid_kernel(double* dst, int64_t mx, int64_t my, int64_t pitch, int64_t nplanes, int64_t zbase,
                                    DVec v) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < v.nnz; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t idx = v.idx[e];
        const int64_t z = idx / (mx * my), rem = idx - z * mx * my;
        const int64_t y = rem / mx, x = rem - y * mx;
        const int64_t b = z - zbase;
        if (b >= 0 && b < nplanes) dst[(b * my + y) * pitch + x] = v.val[e];  // host merged duplicates
    }
}

void kr_fill_grid(cudaStream_t s, double* dst, int64_t mx, int64_t my, int64_t pitch, int64_t nplanes, int64_t zbase,
                  int64_t mz, const DVec& v, int64_t* launches) {
    const int64_t total = nplanes * my * pitch;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    fill_grid_kernel<<<blocks, 256, 0, s>>>(dst, mx, my, pitch, nplanes, zbase, mz, v);
    KR_CUDA(cudaGetLastError());
    (*launches)++;
    if (v.kind == KR_VEC_SPARSE && v.nnz > 0) {
        int b2 = (int)std::min<int64_t>((v.nnz + 255) / 256, 148 * 8);
        scatter_grid_kernel<<<b2, 256, 0, s>>>(dst, mx, my, pitch, nplanes, zbase, v);
        KR_CUDA(cudaGetLastError());
        (*launches)++;
    }
}

__global__ void fill_dense_kernel(double* dst, int64_t N, int64_t n, int64_t mx, int64_t my, int stencil, DVec v,
                                  int lift1) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < N; c += (int64_t)gridDim.x * blockDim.x) {
        double val = 0.0;
        if (c < n) {
            if (v.kind == KR_VEC_RAND) {
                val = kr_rand_entry(v.seed, c, v.value);
            } else if (stencil) {
                const int64_t z = c / (mx * my), rem = c - z * mx * my;
                const int64_t y = rem / mx, x = rem - y * mx;
                val = box_value(v, x, y, z);
            } else {
                if (v.kind == KR_VEC_ALL) val = v.value;
                if (v.kind == KR_VEC_BOX) val = (c >= v.lo[0] && c < v.hi[0]) ? v.value : 0.0;
            }
        } else {
            val = lift1 ? 1.0 : 0.0;
        }
        dst[c] = val;
    }
}

// All local start vectors at once (one launch instead of a fill + scatter per direction): V[dl][0][c] =
// v_dl[c] (box / all-grid by membership, sparse by binary search in the sorted, merged index list), the lifted
// coordinate lift1[dl].
__global__ void fill_dirs_kernel(double* V, int64_t vstride, int64_t N, int64_t n, int64_t mx, int64_t my, int stencil,
                                 const DVec* dirs, const int32_t* lift1) {
    const int dl = blockIdx.y;
    const DVec v = dirs[dl];
    double* dst = V + (int64_t)dl * vstride;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < N; c += (int64_t)gridDim.x * blockDim.x) {
        double val = 0.0;
        if (c >= n) {
            val = lift1[dl] ? 1.0 : 0.0;
        } else if (v.kind == KR_VEC_SPARSE) {
            int64_t lo = 0, hi = v.nnz;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (v.idx[mid] < c) lo = mid + 1; else hi = mid;
            }
            if (lo < v.nnz && v.idx[lo] == c) val = v.val[lo];
        } else if (v.kind == KR_VEC_RAND) {
            val = kr_rand_entry(v.seed, c, v.value);
        } else if (stencil) {
            const int64_t z = c / (mx * my), rem = c - z * mx * my;
            const int64_t y = rem / mx, x = rem - y * mx;
            val = box_value(v, x, y, z);
        } else {
            if (v.kind == KR_VEC_ALL) val = v.value;
            if (v.kind == KR_VEC_BOX) val = (c >= v.lo[0] && c < v.hi[0]) ? v.value : 0.0;
        }
        dst[c] = val;
    }
}

__global__ void scatter_dense_kernel(double* dst, DVec v) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < v.nnz; e += (int64_t)gridDim.x * blockDim.x)
        dst[v.idx[e]] = v.val[e];
}

void kr_fill_dense(cudaStream_t s, double* dst, int64_t N, int64_t n, int64_t mx, int64_t my, bool stencil,
                   const DVec& v, int lift1, double, int, int64_t* launches) {
    int blocks = (int)std::min<int64_t>((N + 255) / 256, 148 * 16);
    fill_dense_kernel<<<blocks, 256, 0, s>>>(dst, N, n, mx, my, stencil ? 1 : 0, v, lift1);
    KR_CUDA(cudaGetLastError());
    (*launches)++;
    if (v.kind == KR_VEC_SPARSE && v.nnz > 0) {
        int b2 = (int)std::min<int64_t>((v.nnz + 255) / 256, 148 * 8);
        scatter_dense_kernel<<<b2, 256, 0, s>>>(dst, v);
        KR_CUDA(cudaGetLastError());
        (*launches)++;
    }
}

// ------------------------------------------------------------------------------------------------
// operators, batched over directions: Y[d] = A X[d]  (X, Y with a per-direction stride)
// ------------------------------------------------------------------------------------------------
__global__ void spmm_csr_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                const double* __restrict__ val, const double* __restrict__ b, int64_t n, int64_t N,
                                const double* __restrict__ X, int64_t xstride, double* __restrict__ Y,
                                int64_t ystride, int ndl, const int32_t* __restrict__ done) {
    const int d = blockIdx.y;
    if (done[d]) return;
    const double* x = X + (int64_t)d * xstride;
    double* y = Y + (int64_t)d * ystride;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < N; r += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        if (r < n) {
            const int64_t e1 = rp[r + 1];
            if (e1 - rp[r] > KR_LONG_ROW) continue;  // long rows (e.g. the b^T row of a transposed lift): CTA each
            for (int64_t e = rp[r]; e < e1; ++e) s = fma(val[e], __ldg(&x[ci[e]]), s);
            if (b) s = fma(b[r], x[n], s);
        }
        y[r] = s;
    }
}

// Block SpMM (Alg. 1 line 3, for every direction at once): Y[d] = A' X[d] with each CSR
// row streamed ONCE per Krylov step for all local directions. A group of G lanes per row (G = the directions rounded
// up to a power of two, at most 32: 32 rows per warp for one direction, one row per warp for 17-32), lane = direction
// (a further pass per G directions): the group loads the row's entries G at a time (coalesced) and broadcasts them by
// shuffles; each lane gathers x_d[col] from its own direction's vector. Entries are summed in row order as in
// spmm_csr_kernel, so the results are those of one thread per (row, direction), bit for bit. The lifted row n of A'
// is zero; rows longer than KR_LONG_ROW are left to spmm_long_rows_kernel.
__global__ void __launch_bounds__(256) spmm_block_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                         const double* __restrict__ val, const double* __restrict__ b,
                                                         int64_t n, int64_t N, const double* __restrict__ X,
                                                         int64_t xstride, double* __restrict__ Y, int64_t ystride,
                                                         int ndl, const int32_t* __restrict__ done, int G) {
    const int lane = threadIdx.x & 31;
    const int rpw = 32 / G, g = lane % G, base = lane - g;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * rpw; r0 < N; r0 += nwarps * rpw) {
        const int64_t r = r0 + lane / G;
        const int64_t e0 = r < n ? rp[r] : 0, e1 = r < n ? rp[r + 1] : 0;
        const bool shortrow = e1 - e0 <= KR_LONG_ROW;
        const int len = (r < N && shortrow) ? (int)(e1 - e0) : 0;
        const int maxlen = __reduce_max_sync(0xffffffffu, len);
        for (int d0 = 0; d0 < ndl; d0 += G) {
            const int d = d0 + g;
            const bool act = r < N && shortrow && d < ndl && !done[d];
            const double* x = X + (int64_t)(act ? d : 0) * xstride;
            double s = 0.0;
            for (int eb = 0; eb < maxlen; eb += G) {
                double v = 0.0;
                int c = 0;
                if (eb + g < len) {
                    v = val[e0 + eb + g];
                    c = ci[e0 + eb + g];
                }
                const int tn = min(G, maxlen - eb);  // warp-uniform: no broadcasts past the longest row's end
                for (int t = 0; t < tn; ++t) {
                    const double vt = __shfl_sync(0xffffffffu, v, base + t);
                    const int ct = __shfl_sync(0xffffffffu, c, base + t);
                    if (act && eb + t < len) s = fma(vt, __ldg(&x[ct]), s);
                }
            }
            if (act) {
                if (r < n && b) s = fma(b[r], x[n], s);
                Y[(int64_t)d * ystride + r] = s;
            }
        }
    }
}

// rows with more than KR_LONG_ROW entries: one CTA per (long row, direction), fixed-order block reduction
__global__ void spmm_long_rows_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                      const double* __restrict__ val, const double* __restrict__ b, int64_t n,
                                      const int64_t* __restrict__ rows, const double* __restrict__ X, int64_t xstride,
                                      double* __restrict__ Y, int64_t ystride, const int32_t* __restrict__ done) {
    const int d = blockIdx.y;
    if (done[d]) return;
    const int64_t r = rows[blockIdx.x];
    const double* x = X + (int64_t)d * xstride;
    __shared__ double red[32];
    double s = 0.0;
    for (int64_t e = rp[r] + threadIdx.x; e < rp[r + 1]; e += blockDim.x) s = fma(val[e], __ldg(&x[ci[e]]), s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        if (b) t = fma(b[r], x[n], t);
        Y[(int64_t)d * ystride + r] = t;
    }
}

// Y[d] = A' X[d] for every local direction, one launch (+ the long rows): the block SpMM above from 8 directions
// (C2: 21); below, or with KR_SPMM_PER_DIR=1, one thread per (row, direction) — A re-read per direction from L2,
// which for a few directions is cheaper than the shuffles (the transpose dynamics of C2, 3 simulations: 2.35 vs
// 3.34 ms per bench step; C2 with 21 directions: 3.74-3.85 vs 3.86-3.95 ms)
void kr_csr_spmm(kr_handle* h, const double* X, int64_t xstride, double* Y, int64_t ystride, int ndl) {
    const int64_t N = h->N;
    if (ndl < 8 || getenv("KR_SPMM_PER_DIR")) {
        const int bx = (int)std::min<int64_t>((N + 255) / 256, 148 * 8);
        spmm_csr_kernel<<<dim3(bx, ndl), 256, 0, h->stream>>>(h->d_rp, h->d_ci, h->d_val, h->d_b, h->n, N, X, xstride, Y,
                                                              ystride, ndl, h->d_done);
    } else {
        int G = 1;
        while (G < ndl && G < 32) G <<= 1;  // lanes per row: the directions, up to a warp
        const int64_t rows_per_block = 8 * (32 / G);
        const int blocks = (int)std::min<int64_t>((N + rows_per_block - 1) / rows_per_block, 148 * 16);
        spmm_block_kernel<<<blocks, 256, 0, h->stream>>>(h->d_rp, h->d_ci, h->d_val, h->d_b, h->n, N, X, xstride, Y,
                                                         ystride, ndl, h->d_done, G);
    }
    KR_CUDA(cudaGetLastError());
    h->launches++;
    if (h->n_long) {
        spmm_long_rows_kernel<<<dim3((unsigned)h->n_long, ndl), 256, 0, h->stream>>>(
            h->d_rp, h->d_ci, h->d_val, h->d_b, h->n, h->d_long, X, xstride, Y, ystride, h->d_done);
        KR_CUDA(cudaGetLastError());
        h->launches++;
    }
}


__global__ void stencil_apply_kernel(int64_t mx, int64_t my, int64_t mz, double cx, double cy, double cz,
                                     const double* __restrict__ X, int64_t xstride, double* __restrict__ Y,
                                     int64_t ystride, const int32_t* __restrict__ done, FaceCor fc,
                                     const double* __restrict__ bl) {
    const int d = blockIdx.y;
    if (done[d]) return;
    const double* u = X + (int64_t)d * xstride;
    double* y = Y + (int64_t)d * ystride;
    const int64_t n = mx * my * mz;
    const double diag = 2.0 * (cx + cy + cz);
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t z = c / (mx * my), rem = c - z * mx * my;
        const int64_t yy = rem / mx, x = rem - yy * mx;
        const double sx = (x > 0 ? u[c - 1] : 0.0) + (x < mx - 1 ? u[c + 1] : 0.0);
        const double sy = (yy > 0 ? u[c - mx] : 0.0) + (yy < my - 1 ? u[c + mx] : 0.0);
        const double sz = (z > 0 ? u[c - mx * my] : 0.0) + (z < mz - 1 ? u[c + mx * my] : 0.0);
        const double dg = diag - (x == 0 ? fc.e[0] : 0.0) - (x == mx - 1 ? fc.e[1] : 0.0) -
                          (yy == 0 ? fc.e[2] : 0.0) - (yy == my - 1 ? fc.e[3] : 0.0) -
                          (z == 0 ? fc.e[4] : 0.0) - (z == mz - 1 ? fc.e[5] : 0.0);
        double v = cx * sx + cy * sy + cz * sz - dg * u[c];
        if (bl) v = fma(bl[c], u[n], v);  // lifted affine term: y = A u + b u_n
        y[c] = v;
    }
    if (bl && blockIdx.x == 0 && threadIdx.x == 0) y[n] = 0.0;  // the lifted row of A' is zero
}

// ------------------------------------------------------------------------------------------------
// orthogonalisation (one CTA of 1024 threads per direction)
// ------------------------------------------------------------------------------------------------
constexpr int OT = 1024;

__device__ __forceinline__ double block_sum_1024(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) red[wid] = v;
    __syncthreads();
    if (wid == 0) {
        v = red[lane];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (lane == 0) red[32] = v;
    }
    __syncthreads();
    const double r = red[32];
    __syncthreads();
    return r;
}

struct OrthoArgs {
    double* V;        // [ndl][k+1][N]
    const double* W;  // [ndl][N]  (A v_{j-1}); for j == 0 unused
    int64_t N;
    int k, j;         // producing basis vector index j (0 = init: normalise the start vector)
    int lanczos;
    double* H;        // [ndl][k+1][k]
    double* P;        // [ndl][n_out][k]
    const double* O;  // [n_out][N]
    int n_out;
    double* beta0;
    double* hnext;
    double* hmax;
    int32_t* keff;
    int32_t* done;
    int32_t* status;
};

// SW: keep w in shared memory (large N; registers would spill at 1024 threads x 64 registers).
template <int EPT, bool SW>
__global__ void __launch_bounds__(OT) ortho_kernel(OrthoArgs a) {
    const int d = blockIdx.x;
    if (a.done[d]) return;
    __shared__ double red[33];
    extern __shared__ double wsm[];
    const int64_t N = a.N;
    const int k = a.k, j = a.j;
    double* V = a.V + (int64_t)d * (k + 1) * N;
    double* H = a.H + (int64_t)d * (k + 1) * k;
    double wr[SW ? 1 : EPT];
#define WV(e) (SW ? wsm[threadIdx.x + (e) * OT] : wr[SW ? 0 : (e)])
    const double* src = (j == 0) ? V : a.W + (int64_t)d * N;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
        const int64_t c = threadIdx.x + (int64_t)e * OT;
        WV(e) = c < N ? src[c] : 0.0;
    }
    double hm = (j == 0) ? 0.0 : a.hmax[d];
    if (j > 0) {
        int l0 = 0;
        if (a.lanczos) {
            // Alg. 3: w -= H_{j-1,j} V_{j-2} with H_{j-1,j} = H_{j,j-1} (known), then one dot for alpha
            if (j >= 2) {
                const double bprev = H[(int64_t)(j - 1) * k + (j - 2)];
                const double* Vl = V + (int64_t)(j - 2) * N;
#pragma unroll
                for (int e = 0; e < EPT; ++e) {
                    const int64_t c = threadIdx.x + (int64_t)e * OT;
                    if (c < N) WV(e) = WV(e) - bprev * Vl[c];
                }
                if (threadIdx.x == 0) H[(int64_t)(j - 2) * k + (j - 1)] = bprev;
            }
            l0 = j - 1;
        }
        for (int l = l0; l <= j - 1; ++l) {  // MGS, the printed inner loop read as 1..i-1
            const double* Vl = V + (int64_t)l * N;
            double vl[EPT];
            double s = 0.0;
#pragma unroll
            for (int e = 0; e < EPT; ++e) {
                const int64_t c = threadIdx.x + (int64_t)e * OT;
                vl[e] = c < N ? Vl[c] : 0.0;
                s = fma(vl[e], WV(e), s);
            }
            const double h = block_sum_1024(s, red);
#pragma unroll
            for (int e = 0; e < EPT; ++e) WV(e) = WV(e) - h * vl[e];
            if (threadIdx.x == 0) H[(int64_t)l * k + (j - 1)] = h;
            hm = fmax(hm, fabs(h));
        }
    }
    double s = 0.0;
#pragma unroll
    for (int e = 0; e < EPT; ++e) s = fma(WV(e), WV(e), s);
    const double nb = sqrt(block_sum_1024(s, red));
    if (j == 0) {
        if (threadIdx.x == 0) {
            a.beta0[d] = nb;
            a.keff[d] = 1;
            a.hmax[d] = 0.0;
            if (!(nb > 0.0) || !isfinite(nb)) {
                a.done[d] = 1;
                a.keff[d] = 0;
                a.status[d] = nb == 0.0 ? KR_EZERO : KR_ENONFINITE;
            }
        }
        if (!(nb > 0.0) || !isfinite(nb)) return;
    } else {
        if (threadIdx.x == 0) H[(int64_t)j * k + (j - 1)] = nb;
        if (!isfinite(nb)) {
            if (threadIdx.x == 0) {
                a.done[d] = 1;
                a.status[d] = KR_ENONFINITE;
            }
            return;
        }
        if (nb == 0.0 || nb <= 16.0 * DBL_EPSILON * hm || j == k) {  // breakdown or extra column
            if (threadIdx.x == 0) {
                a.done[d] = 1;
                a.keff[d] = j;
                a.hnext[d] = nb;
            }
            return;
        }
        hm = fmax(hm, nb);
        if (threadIdx.x == 0) {
            a.hmax[d] = hm;
            a.keff[d] = j + 1;
        }
    }
    double* Vj = V + (int64_t)j * N;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
        const int64_t c = threadIdx.x + (int64_t)e * OT;
        WV(e) = WV(e) / nb;
        if (c < N) Vj[c] = WV(e);
    }
    // P_{., j} = C V_{*, j}
    for (int r = 0; r < a.n_out; ++r) {
        const double* Or = a.O + (int64_t)r * N;
        double t = 0.0;
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
            const int64_t c = threadIdx.x + (int64_t)e * OT;
            if (c < N) t = fma(Or[c], WV(e), t);
        }
        const double pr = block_sum_1024(t, red);
        if (threadIdx.x == 0) a.P[((int64_t)d * a.n_out + r) * k + j] = pr;
    }
#undef WV
}

static void launch_ortho(kr_handle* h, int j, int ndl) {
    if (h->use_cgs) {  // N > KR_ORTHO_ONE_CTA_MAX: stream the basis with the whole GPU (CGS2, kr_arnoldi.cu)
        kr_cgs_step(h, j, ndl, h->d_cgs);
        return;
    }
    OrthoArgs a;
    a.V = h->d_V;
    a.W = h->d_W;
    a.N = h->N;
    a.k = h->k;
    a.j = j;
    a.lanczos = h->method == KR_LANCZOS ? 1 : 0;
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
    const int64_t ept = (h->N + OT - 1) / OT;
    const size_t sm = (size_t)ept * OT * sizeof(double);
    if (ept <= 1)
        ortho_kernel<1, false><<<ndl, OT, 0, h->stream>>>(a);
    else if (ept <= 2)
        ortho_kernel<2, false><<<ndl, OT, 0, h->stream>>>(a);
    else if (ept <= 4)
        ortho_kernel<4, false><<<ndl, OT, 0, h->stream>>>(a);
    else if (ept <= 8)
        ortho_kernel<8, false><<<ndl, OT, 0, h->stream>>>(a);
    else if (ept <= 12)
        ortho_kernel<12, true><<<ndl, OT, 12 * OT * 8, h->stream>>>(a);
    else if (ept <= 16)
        ortho_kernel<16, true><<<ndl, OT, 16 * OT * 8, h->stream>>>(a);
    else if (ept <= 20)
        ortho_kernel<20, true><<<ndl, OT, 20 * OT * 8, h->stream>>>(a);
    else if (ept <= 24)
        ortho_kernel<24, true><<<ndl, OT, 24 * OT * 8, h->stream>>>(a);
    else if (ept <= 27)
        ortho_kernel<27, true><<<ndl, OT, 27 * OT * 8, h->stream>>>(a);
    else
        KR_THROW(KR_EDIM, "stored-basis Krylov path supports operator dimension <= 27648");
    (void)sm;
    KR_CUDA(cudaGetLastError());
    h->launches++;
}

__global__ void ge_reset(int32_t* done, int32_t* status, int ndl) {
    for (int d = threadIdx.x; d < ndl; d += blockDim.x) {
        done[d] = 0;
        status[d] = 0;
    }
}

void kr_ge_prepare() {
    KR_CUDA(cudaFuncSetAttribute(ortho_kernel<12, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * OT * 8));
    KR_CUDA(cudaFuncSetAttribute(ortho_kernel<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * OT * 8));
    KR_CUDA(cudaFuncSetAttribute(ortho_kernel<20, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 20 * OT * 8));
    KR_CUDA(cudaFuncSetAttribute(ortho_kernel<24, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 24 * OT * 8));
    KR_CUDA(cudaFuncSetAttribute(ortho_kernel<27, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 27 * OT * 8));
}

// Start of the stored-basis runs of all local directions: reset, v_0 = the start vectors, normalise (j = 0).
void kr_ge_enqueue_init(kr_handle* h) {
    const int ndl = (int)h->my_dirs.size();
    const int64_t N = h->N;
    const int k = h->k;
    ge_reset<<<1, 256, 0, h->stream>>>(h->d_done, h->d_status, ndl);
    KR_CUDA(cudaGetLastError());
    h->launches++;
    if (h->d_gdirs && ndl > 0) {
        const int blocks = (int)std::min<int64_t>((N + 255) / 256, 148 * 4);
        fill_dirs_kernel<<<dim3(blocks, ndl), 256, 0, h->stream>>>(h->d_V, (int64_t)(k + 1) * N, N, h->n, h->mx, h->my,
                                                                     h->op == KR_OP_STENCIL7 ? 1 : 0, h->d_gdirs,
                                                                     h->d_glift);
        KR_CUDA(cudaGetLastError());
        h->launches++;
    } else {
        for (int dl = 0; dl < ndl; ++dl) {
            const int d = h->my_dirs[dl];
            kr_fill_dense(h->stream, h->d_V + (int64_t)dl * (k + 1) * N, N, h->n, h->mx, h->my,
                          h->op == KR_OP_STENCIL7, h->dirs_h[d], h->dir_lift1[d], 1.0, 0, &h->launches);
        }
    }
    launch_ortho(h, 0, ndl);
}

// Krylov step j (1-based) of every local direction: w = A v_{j-1} for all directions at once (one SpMM /
// stencil launch), then the orthogonalisation producing v_j (stopped directions exit at once).
void kr_ge_enqueue_step(kr_handle* h, int j) {
    const int ndl = (int)h->my_dirs.size();
    const int64_t N = h->N;
    const int k = h->k;
    const int64_t vstride = (int64_t)(k + 1) * N;
    const int bx = (int)std::min<int64_t>((N + 255) / 256, 148 * 8);
    const FaceCor fc = kr_face_cor(h);
    const double* X = h->d_V + (int64_t)(j - 1) * N;
    const int evp = (h->timing && j < (int)h->ev_pair_of_step.size()) ? h->ev_pair_of_step[(size_t)j] : -1;
    const bool evj = evp >= 0;
    if (evj) KR_CUDA(kr_event_record(h->ev[2 * evp], h->stream));
    if (evj && (size_t)evp < h->ev_rec.size()) h->ev_rec[(size_t)evp] = 1;
    if (h->use_cgs) {  // operator fused into the first CGS2 pass (kr_arnoldi.cu): the events bracket the whole step
        kr_cgs_step(h, j, ndl, h->d_cgs);
        if (evj) KR_CUDA(kr_event_record(h->ev[2 * evp + 1], h->stream));
        return;
    }
    if (h->op == KR_OP_CSR) {
        kr_csr_spmm(h, X, vstride, h->d_W, N, ndl);
    } else {
        stencil_apply_kernel<<<dim3(bx, ndl), 256, 0, h->stream>>>(h->mx, h->my, h->mz, h->cx, h->cy, h->cz, X, vstride,
                                                                   h->d_W, N, h->d_done, fc, h->d_bl);
        KR_CUDA(cudaGetLastError());
        h->launches++;
    }
    if (evj) KR_CUDA(kr_event_record(h->ev[2 * evp + 1], h->stream));
    launch_ortho(h, j, ndl);
}

void kr_ge_enqueue_direction_set(kr_handle* h) {
    kr_ge_enqueue_init(h);
    for (int j = 1; j <= h->k; ++j) kr_ge_enqueue_step(h, j);
}
