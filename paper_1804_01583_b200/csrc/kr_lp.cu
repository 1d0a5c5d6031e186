// kr_lp.cu — the general per-step LP of the verification problem, batched over time
// steps: one CTA per step j solves
//     find z:  z_lo <= z <= z_hi,  I_z z <= iota,  U_y (B_j z + c_f,j) <= upsilon
// (initial set "I_x x0 <= iota_x" and unsafe set "U_x x <= upsilon_x" of §2.1, in the
// initial / output space coordinates of §3; the LP of Fig. 2(c), for
// a polytope instead of a box). B_j are the generator columns of the basis matrix (krylov_project), c_f,j
// the fixed-term column (z_f = 1). The system is unsafe at the first feasible step
// and the solver's assignment is the counter-example.
//
// B200 design: the paper solves one LP per step sequentially with a warm-started external solver; here
// every step's LP is independent (only the basis matrix changes), so all N+1 LPs run at
// once, one CTA each, as a dense Phase-I simplex in shared memory:
//   * variables s = z - z_lo in [0, z_hi - z_lo] (box rows explicit), rows normalised to max |a| = 1;
//   * a slack per row, an artificial where the right-hand side is negative; Phase I minimises the sum of
//     artificials — feasible iff its optimum is <= 1e-9;
//   * Bland's rule (smallest entering index, ratio-test ties to the smallest basic index): no cycling,
//     deterministic; pivot tolerance 1e-11;
//   * the witness is the final basic solution z = z_lo + s.
#include <math.h>

#include "kr_internal.h"

namespace {

constexpr int LT = 256;

struct LpArgs {
    const double* coeff;  // [(N+1)][o][nd] final basis-matrix layout
    int o, nd, ng, has_fixed;
    const double* zlo;    // [nd] (fixed direction: 1)
    const double* zhi;
    int m_init;
    const double* IA;     // [m_init][ng]
    const double* Ib;
    int m_uns;
    const double* UA;     // [m_uns][o]
    const double* Ub;
    int32_t* feas;        // [(N+1)]: 1 feasible, 0 infeasible, -1 iteration cap
    double* zw;           // [(N+1)][ng] witness per step
    int max_iter;
};

__global__ void __launch_bounds__(LT) lp_step_kernel(const LpArgs a) {
    const int64_t j = blockIdx.x;
    const int ng = a.ng, R = a.m_init + a.m_uns + ng;
    const int NC = ng + 2 * R + 1;  // [s | slack | artificial | rhs]
    const int RHS = NC - 1;
    extern __shared__ double sm[];
    double* T = sm;                // [R][NC]
    double* W = T + (size_t)R * NC;  // Phase-I objective row [NC]
    int* basis = reinterpret_cast<int*>(W + NC);
    __shared__ int s_enter, s_leave, s_done;
    __shared__ double s_red[LT];
    __shared__ int s_redi[LT];
    const double* Bj = a.coeff + j * (int64_t)a.o * a.nd;
    const int tid = threadIdx.x;

    // rows in the variables s = z - z_lo
    for (int r = tid; r < R; r += LT) {
        double* row = T + (size_t)r * NC;
        for (int c = 0; c < NC; ++c) row[c] = 0.0;
        double b;
        if (r < a.m_init) {
            b = a.Ib[r];
            for (int d = 0; d < ng; ++d) {
                const double v = a.IA[(int64_t)r * ng + d];
                row[d] = v;
                b -= v * a.zlo[d];
            }
        } else if (r < a.m_init + a.m_uns) {
            const int u = r - a.m_init;
            b = a.Ub[u];
            for (int q = 0; q < a.o; ++q) {  // - U (B_j z_lo + c_f)
                const double uq = a.UA[(int64_t)u * a.o + q];
                double y = a.has_fixed ? Bj[(int64_t)q * a.nd + ng] : 0.0;
                for (int d = 0; d < ng; ++d) y += Bj[(int64_t)q * a.nd + d] * a.zlo[d];
                b -= uq * y;
            }
            for (int d = 0; d < ng; ++d) {
                double v = 0.0;
                for (int q = 0; q < a.o; ++q) v += a.UA[(int64_t)u * a.o + q] * Bj[(int64_t)q * a.nd + d];
                row[d] = v;
            }
        } else {
            const int d = r - a.m_init - a.m_uns;
            row[d] = 1.0;
            b = a.zhi[d] - a.zlo[d];
        }
        double mx = 0.0;
        for (int d = 0; d < ng; ++d) mx = fmax(mx, fabs(row[d]));
        const double sc = mx > 0.0 ? 1.0 / mx : 1.0;
        for (int d = 0; d < ng; ++d) row[d] *= sc;
        b *= sc;
        row[ng + r] = 1.0;  // slack
        if (b < 0.0) {      // negate; the artificial is basic
            for (int d = 0; d < ng; ++d) row[d] = -row[d];
            row[ng + r] = -1.0;
            row[ng + R + r] = 1.0;
            row[RHS] = -b;
            basis[r] = ng + R + r;
        } else {
            row[RHS] = b;
            basis[r] = ng + r;
        }
    }
    __syncthreads();
    for (int c = tid; c < NC; c += LT) {
        double w = 0.0;
        if (c < ng + R || c == RHS)
            for (int r = 0; r < R; ++r)
                if (basis[r] >= ng + R) w += T[(size_t)r * NC + c];
        W[c] = w;
    }
    if (tid == 0) s_done = 0;
    __syncthreads();
    const double piv_tol = 1e-11;
    int it = 0;
    for (; it < a.max_iter; ++it) {
        // entering: smallest non-artificial column with a positive reduced cost (Bland)
        int best = NC;
        for (int c = tid; c < ng + R; c += LT)
            if (W[c] > piv_tol && c < best) best = c;
        s_redi[tid] = best;
        __syncthreads();
        for (int st = LT / 2; st > 0; st >>= 1) {
            if (tid < st) s_redi[tid] = min(s_redi[tid], s_redi[tid + st]);
            __syncthreads();
        }
        if (tid == 0) s_enter = s_redi[0];
        __syncthreads();
        const int e = s_enter;
        if (e >= NC) break;  // optimal
        // ratio test: min rhs / T[r][e] over T[r][e] > tol, ties to the smallest basic index
        double bv = INFINITY;
        int bi = 1 << 30;
        for (int r = tid; r < R; r += LT) {
            const double t = T[(size_t)r * NC + e];
            if (t > piv_tol) {
                const double th = T[(size_t)r * NC + RHS] / t;
                const int key = basis[r] * 1024 + r;
                if (th < bv || (th == bv && key < bi)) {
                    bv = th;
                    bi = key;
                }
            }
        }
        s_red[tid] = bv;
        s_redi[tid] = bi;
        __syncthreads();
        for (int st = LT / 2; st > 0; st >>= 1) {
            if (tid < st) {
                const double v2 = s_red[tid + st];
                const int i2 = s_redi[tid + st];
                if (v2 < s_red[tid] || (v2 == s_red[tid] && i2 < s_redi[tid])) {
                    s_red[tid] = v2;
                    s_redi[tid] = i2;
                }
            }
            __syncthreads();
        }
        if (tid == 0) s_leave = s_redi[0] == (1 << 30) ? -1 : (s_redi[0] & 1023);
        __syncthreads();
        const int l = s_leave;
        if (l < 0) break;  // unbounded direction cannot occur in Phase I (W is bounded below by 0)
        // pivot on (l, e)
        const double pv = T[(size_t)l * NC + e];
        for (int c = tid; c < NC; c += LT) T[(size_t)l * NC + c] /= pv;
        __syncthreads();
        for (int idx = tid; idx < (R + 1) * NC; idx += LT) {
            const int r = idx / NC, c = idx - r * NC;
            if (r == l) continue;
            double* row = r < R ? T + (size_t)r * NC : W;
            const double f = r < R ? T[(size_t)r * NC + e] : W[e];
            if (f != 0.0 && c != e) row[c] -= f * T[(size_t)l * NC + c];
        }
        __syncthreads();
        for (int r = tid; r <= R; r += LT) {  // the pivot column is exactly e_l afterwards
            if (r == l) continue;
            if (r < R)
                T[(size_t)r * NC + e] = 0.0;
            else
                W[e] = 0.0;
        }
        if (tid == 0) basis[l] = e;
        __syncthreads();
    }
    if (tid == 0) {
        double rmax = 0.0;
        for (int r = 0; r < R; ++r) rmax = fmax(rmax, fabs(T[(size_t)r * NC + RHS]));
        const bool capped = it >= a.max_iter;
        const bool ok = W[RHS] <= 1e-9 * (1.0 + rmax);
        a.feas[j] = capped ? -1 : (ok ? 1 : 0);
    }
    for (int d = tid; d < ng; d += LT) {
        double s = 0.0;
        for (int r = 0; r < R; ++r)
            if (basis[r] == d) s = T[(size_t)r * NC + RHS];
        a.zw[j * ng + d] = a.zlo[d] + s;
    }
}

// first feasible step, its witness (fixed coordinate 1) and outputs y = B_j z + c_f
__global__ void lp_first_kernel(const LpArgs a, int64_t np1, double* out /* [2 + nd + o] */) {
    __shared__ int64_t red[LT];
    int64_t best = np1;
    for (int64_t j = threadIdx.x; j < np1; j += LT)
        if (a.feas[j] == 1 && j < best) best = j;
    red[threadIdx.x] = best;
    __syncthreads();
    for (int st = LT / 2; st > 0; st >>= 1) {
        if (threadIdx.x < st) red[threadIdx.x] = min(red[threadIdx.x], red[threadIdx.x + st]);
        __syncthreads();
    }
    const int64_t j = red[0];
    if (threadIdx.x == 0) {
        out[0] = j < np1 ? 1.0 : 0.0;
        out[1] = (double)(j < np1 ? j : -1);
    }
    if (j >= np1) return;
    for (int d = threadIdx.x; d < a.nd; d += LT) out[2 + d] = d < a.ng ? a.zw[j * a.ng + d] : 1.0;
    const double* Bj = a.coeff + j * (int64_t)a.o * a.nd;
    for (int q = threadIdx.x; q < a.o; q += LT) {
        double y = 0.0;
        for (int d = 0; d < a.nd; ++d) y += Bj[(int64_t)q * a.nd + d] * (d < a.ng ? a.zw[j * a.ng + d] : 1.0);
        out[2 + a.nd + q] = y;
    }
}

}  // namespace

// Host side of krylov_check_lp (argument checks done by the caller). Returns the number of iterations cap
// hits. feas_h: host [(N+1)] or NULL; out_h: host [2 + nd + o].
void kr_lp_run(kr_handle* h, int m_init, const double* IA, const double* Ib, int m_uns, const double* UA,
               const double* Ub, int32_t* feas_h, double* out_h) {
    const int ng = h->n_gen_cf, nd = h->cf_ndir, o = h->cf_nout;
    const int64_t np1 = h->n_steps + 1;
    const int R = m_init + m_uns + ng;
    const int NC = ng + 2 * R + 1;
    const size_t smem = ((size_t)R * NC + NC) * sizeof(double) + (size_t)R * sizeof(int) + 16;
    if (smem > 200 * 1024) KR_THROW(KR_EINVAL, "LP too large for one CTA (reduce constraints / generators)");
    // device copies of the constraint blocks (small)
    const size_t nbytes = ((size_t)m_init * ng + m_init + (size_t)m_uns * o + m_uns) * sizeof(double);
    double* dbuf = nullptr;
    int32_t* dfeas = nullptr;
    double* dzw = nullptr;
    double* dout = nullptr;
    KR_CUDA(kr_dev_malloc(reinterpret_cast<void**>(&dbuf), nbytes + 64));
    KR_CUDA(kr_dev_malloc(reinterpret_cast<void**>(&dfeas), np1 * sizeof(int32_t)));
    KR_CUDA(kr_dev_malloc(reinterpret_cast<void**>(&dzw), (size_t)np1 * (ng > 0 ? ng : 1) * sizeof(double)));
    KR_CUDA(kr_dev_malloc(reinterpret_cast<void**>(&dout), (size_t)(2 + nd + o) * sizeof(double)));
    struct Free {  // back to the block cache once the stream no longer uses them
        void* p[4];
        cudaStream_t s;
        ~Free() {
            cudaStreamSynchronize(s);
            for (void* q : p)
                if (q) kr_dev_free(q);
        }
    } fr{{dbuf, dfeas, dzw, dout}, h->stream};
    double* dIA = dbuf;
    double* dIb = dIA + (size_t)m_init * ng;
    double* dUA = dIb + m_init;
    double* dUb = dUA + (size_t)m_uns * o;
    cudaStream_t st = h->stream;
    if (m_init) {
        KR_CUDA(cudaMemcpyAsync(dIA, IA, (size_t)m_init * ng * 8, cudaMemcpyHostToDevice, st));
        KR_CUDA(cudaMemcpyAsync(dIb, Ib, (size_t)m_init * 8, cudaMemcpyHostToDevice, st));
    }
    if (m_uns) {
        KR_CUDA(cudaMemcpyAsync(dUA, UA, (size_t)m_uns * o * 8, cudaMemcpyHostToDevice, st));
        KR_CUDA(cudaMemcpyAsync(dUb, Ub, (size_t)m_uns * 8, cudaMemcpyHostToDevice, st));
    }
    h->h2d_bytes += (int64_t)nbytes;
    LpArgs a{};
    a.coeff = h->d_cf;
    a.o = o;
    a.nd = nd;
    a.ng = ng;
    a.has_fixed = nd > ng ? 1 : 0;
    a.zlo = h->d_zlo;
    a.zhi = h->d_zhi;
    a.m_init = m_init;
    a.IA = dIA;
    a.Ib = dIb;
    a.m_uns = m_uns;
    a.UA = dUA;
    a.Ub = dUb;
    a.feas = dfeas;
    a.zw = dzw;
    a.max_iter = 50 * (R + ng) + 100;
    KR_CUDA(cudaFuncSetAttribute(lp_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    lp_step_kernel<<<(unsigned)np1, LT, smem, st>>>(a);
    KR_CUDA(cudaGetLastError());
    h->launches++;
    lp_first_kernel<<<1, LT, 0, st>>>(a, np1, dout);
    KR_CUDA(cudaGetLastError());
    h->launches++;
    KR_CUDA(cudaMemcpyAsync(out_h, dout, (size_t)(2 + nd + o) * 8, cudaMemcpyDeviceToHost, st));
    if (feas_h) KR_CUDA(cudaMemcpyAsync(feas_h, dfeas, np1 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    h->d2h_bytes += (int64_t)(2 + nd + o) * 8 + (feas_h ? np1 * 4 : 0);
    KR_CUDA(cudaStreamSynchronize(st));
}
