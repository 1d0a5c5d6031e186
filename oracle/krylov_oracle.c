/*
 * krylov_oracle.c — TEST INFRASTRUCTURE ONLY. Plain, slow, single-threaded fp64 CPU oracle for the
 * Krylov projected-reachability hot path of arXiv 1804.01583. Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl reference legs may load it.
 * It shares no code, header or constant with the CUDA path (paper_1804_01583_b200/), and the CUDA path
 * never calls it.
 *
 * Every function cites the passage it follows. PAPER.md line numbers are written P:<line>.
 * Compile with -O2 -ffp-contract=off (no FMA contraction: each line below is what gets rounded).
 *
 * Parity pins: see tests/test_oracle_pins.py. Nothing here is "parity unpinned" except the
 * fixed-k supplementary heat outputs at sizes where k is far from convergence.
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------------------------------
 * Sums. Pairwise (recursive halving) summation, SURVEY §8(c) C-alg step 3.1: a sequential sum over
 * 10^9 terms has an n*eps worst-case bound; halving keeps it at log2(n)*eps.
 * ------------------------------------------------------------------------------------------- */
double oracle_sum(const double* a, int64_t n) {
    if (n <= 8) {
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s += a[i];
        return s;
    }
    int64_t h = n / 2;
    return oracle_sum(a, h) + oracle_sum(a + h, n - h);
}

double oracle_dot(const double* a, const double* b, int64_t n) {
    if (n <= 8) {
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
        return s;
    }
    int64_t h = n / 2;
    return oracle_dot(a, b, h) + oracle_dot(a + h, b + h, n - h);
}

/* ---------------------------------------------------------------------------------------------
 * Operators. The operator A of x' = Ax + b. Two forms:
 *  - 7-point Dirichlet heat stencil, A = alpha * L_h with h_a = 1/(m_a+1) per axis
 *    (BASELINE.json configs): (Au)_c = alpha * sum_a (u_{c-a} - 2u_c + u_{c+a}) / h_a^2,
 *    neighbours outside the grid are 0. Linear index x + mx*(y + my*z).
 *  - CSR sparse A. If b != NULL the affine term is lifted into A:
 *    A' = [[A, b], [0, 0]] of size n+1, so y_r = sum_c a_rc x_c + b_r x_n and y_n = 0.
 * ------------------------------------------------------------------------------------------- */
typedef struct {
    int32_t op; /* 0 = stencil, 1 = CSR */
    int64_t mx, my, mz;
    double alpha;
    int64_t n;
    const int64_t* row_ptr;
    const int32_t* col_idx;
    const double* val;
    const double* b; /* NULL = no affine term; CSR or stencil: lifted x' = [[A, b], [0, 0]] x */
    /* stencil boundary per face (x-, x+, y-, y+, z-, z+): 0 Dirichlet (zero ghost, BASELINE configs),
       1 insulated (the missing neighbour is dropped), 2 insulated + exchange: diagonal -= gamma[f]
       (units of A). The paper's heat benchmark (SURVEY A1/A2 reconstruction): all faces
       insulated except x = 1 with exchange 0.5, A = 0.01 (L - (0.5/h) e_{x=m-1}). */
    int32_t bc[6];
    double gamma[6];
} oracle_op;

int64_t oracle_op_dim(const oracle_op* A) {
    if (A->op == 0) return A->mx * A->my * A->mz + (A->b ? 1 : 0);
    return A->n + (A->b ? 1 : 0);
}

void oracle_stencil_apply(int64_t mx, int64_t my, int64_t mz, double alpha, const double* u, double* y) {
    const double ihx2 = (double)(mx + 1) * (double)(mx + 1); /* 1/h_x^2, exact integer */
    const double ihy2 = (double)(my + 1) * (double)(my + 1);
    const double ihz2 = (double)(mz + 1) * (double)(mz + 1);
    for (int64_t z = 0; z < mz; ++z)
        for (int64_t yy = 0; yy < my; ++yy)
            for (int64_t x = 0; x < mx; ++x) {
                int64_t c = x + mx * (yy + my * z);
                double uc = u[c];
                double xm = x > 0 ? u[c - 1] : 0.0;
                double xp = x < mx - 1 ? u[c + 1] : 0.0;
                double ym = yy > 0 ? u[c - mx] : 0.0;
                double yp = yy < my - 1 ? u[c + mx] : 0.0;
                double zm = z > 0 ? u[c - mx * my] : 0.0;
                double zp = z < mz - 1 ? u[c + mx * my] : 0.0;
                double lx = (xm - 2.0 * uc + xp) * ihx2;
                double ly = (ym - 2.0 * uc + yp) * ihy2;
                double lz = (zm - 2.0 * uc + zp) * ihz2;
                y[c] = alpha * (lx + ly + lz);
            }
}

/* General boundaries: (Au)_c = alpha sum_axes sum_{s=+-} t_s / h_a^2 - sum_{faces f at c} gamma_f u_c with
 * t_s = u_{c+s} - u_c if the neighbour exists, -u_c on a Dirichlet face, 0 on an insulated face. */
void oracle_stencil_apply_bc(int64_t mx, int64_t my, int64_t mz, double alpha, const int32_t* bc, const double* gamma,
                             const double* u, double* y) {
    const int64_t m[3] = {mx, my, mz};
    const int64_t st[3] = {1, mx, mx * my};
    double ih2[3];
    for (int a = 0; a < 3; ++a) ih2[a] = (double)(m[a] + 1) * (double)(m[a] + 1);
    for (int64_t z = 0; z < mz; ++z)
        for (int64_t yy = 0; yy < my; ++yy)
            for (int64_t x = 0; x < mx; ++x) {
                const int64_t c = x + mx * (yy + my * z);
                const int64_t pos[3] = {x, yy, z};
                const double uc = u[c];
                double acc = 0.0, diag = 0.0;
                for (int a = 0; a < 3; ++a) {
                    double t = 0.0;
                    for (int sgn = 0; sgn < 2; ++sgn) {
                        const int face = 2 * a + sgn;
                        const int has = sgn == 0 ? pos[a] > 0 : pos[a] < m[a] - 1;
                        if (has)
                            t += u[c + (sgn == 0 ? -st[a] : st[a])] - uc;
                        else if (bc[face] == 0)
                            t += -uc;
                        else if (bc[face] == 2)
                            diag += gamma[face];
                    }
                    acc += t * ih2[a];
                }
                y[c] = alpha * acc - diag * uc;
            }
}

void oracle_csr_apply(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, const double* val,
                      const double* b, const double* x, double* y) {
    for (int64_t r = 0; r < n; ++r) {
        double s = 0.0;
        for (int64_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) s += val[e] * x[col_idx[e]];
        if (b) s += b[r] * x[n];
        y[r] = s;
    }
    if (b) y[n] = 0.0;
}

void oracle_op_apply(const oracle_op* A, const double* x, double* y) {
    int dirichlet = 1;
    for (int f = 0; f < 6; ++f) dirichlet &= A->bc[f] == 0;
    if (A->op == 0) {
        if (dirichlet)
            oracle_stencil_apply(A->mx, A->my, A->mz, A->alpha, x, y);
        else
            oracle_stencil_apply_bc(A->mx, A->my, A->mz, A->alpha, A->bc, A->gamma, x, y);
        if (A->b) { /* lifted affine term: y += b x_n, y_n = 0 */
            const int64_t n = A->mx * A->my * A->mz;
            for (int64_t c = 0; c < n; ++c) y[c] += A->b[c] * x[n];
            y[n] = 0.0;
        }
    } else
        oracle_csr_apply(A->n, A->row_ptr, A->col_idx, A->val, A->b, x, y);
}

/* ---------------------------------------------------------------------------------------------
 * Output rows of C (o x n): P_{r,i} = C_r . V_{*,i} (Alg. 4 lines "P_{*,1} = C V_{*,1}",
 * "P_{*,i} = C V_{*,i}"). Rows are given compactly: kind 0 sparse (idx, val),
 * kind 1 index box [lo,hi) times value (stencil: 3D; CSR: axis 0 only), kind 2 all-ones times value.
 * Entries beyond the unlifted length (the lifted coordinate) are 0.
 * ------------------------------------------------------------------------------------------- */
typedef struct {
    int32_t kind;
    int64_t nnz;
    const int64_t* idx;
    const double* val;
    int64_t lo[3], hi[3];
    double value;
} oracle_row;

double oracle_row_dot(const oracle_op* A, const oracle_row* r, const double* v) {
    if (r->kind == 0) {
        double* t = (double*)malloc(sizeof(double) * (size_t)(r->nnz > 0 ? r->nnz : 1));
        for (int64_t e = 0; e < r->nnz; ++e) t[e] = r->val[e] * v[r->idx[e]];
        double s = oracle_sum(t, r->nnz);
        free(t);
        return s;
    }
    int64_t nbase = A->op == 0 ? A->mx * A->my * A->mz : A->n;
    if (r->kind == 2) return r->value * oracle_sum(v, nbase);
    /* box */
    if (A->op != 0) {
        int64_t lo = r->lo[0] < 0 ? 0 : r->lo[0], hi = r->hi[0] > nbase ? nbase : r->hi[0];
        if (hi <= lo) return 0.0;
        return r->value * oracle_sum(v + lo, hi - lo);
    }
    int64_t x0 = r->lo[0], y0 = r->lo[1], z0 = r->lo[2], x1 = r->hi[0], y1 = r->hi[1], z1 = r->hi[2];
    if (x0 < 0) x0 = 0;
    if (y0 < 0) y0 = 0;
    if (z0 < 0) z0 = 0;
    if (x1 > A->mx) x1 = A->mx;
    if (y1 > A->my) y1 = A->my;
    if (z1 > A->mz) z1 = A->mz;
    if (x1 <= x0 || y1 <= y0 || z1 <= z0) return 0.0;
    int64_t cnt = (x1 - x0) * (y1 - y0) * (z1 - z0), e = 0;
    double* t = (double*)malloc(sizeof(double) * (size_t)cnt);
    for (int64_t z = z0; z < z1; ++z)
        for (int64_t yy = y0; yy < y1; ++yy)
            for (int64_t x = x0; x < x1; ++x) t[e++] = v[x + A->mx * (yy + A->my * z)];
    double s = r->value * oracle_sum(t, cnt);
    free(t);
    return s;
}

/* Breakdown rule ("If the norm ... is ever zero, the loop can terminate early"; SURVEY
 * §8(c) A10): stop when h_{i,i-1} == 0 or h_{i,i-1} <= 16 eps max|H entries computed so far|. */
static int breakdown(double h, double hmax) { return h == 0.0 || h <= 16.0 * DBL_EPSILON * hmax; }

/* ---------------------------------------------------------------------------------------------
 * Lanczos, literally Algorithm 3 with the projection of Algorithm 4:
 * only V_{i-2}, V_{i-1}, V_i are live ("free-memory(V_{*,i-2})"; Eq. 6) and
 * P_{*,i} = C V_{*,i} is recorded instead of V. Fixed k (the error control of Alg. 4 is NEXT-1).
 *
 * In: v (dim N = oracle_op_dim, NOT normalized; normalized here as V_{*,1} = v/||v||, Alg. line 1).
 * Out: alpha[0..k_eff-1] = H_{i,i}; beta[0..k_eff-1] = H_{i+1,i} (beta[k_eff-1] = h_{k+1,k}, the
 *      residual coupling used by Lemma 1); P[r*k + i] = P_{r,i+1}; *beta0 = ||v||; *k_eff.
 * Returns 0, or 7 if ||v|| = 0 (zero start vector).
 * ------------------------------------------------------------------------------------------- */
int oracle_lanczos(const oracle_op* A, const double* v, int32_t k, int32_t n_out, const oracle_row* rows,
                   double* alpha, double* beta, double* P, double* beta0, int32_t* k_eff) {
    int64_t N = oracle_op_dim(A);
    double nv = sqrt(oracle_dot(v, v, N));
    *beta0 = nv;
    if (nv == 0.0) return 7;
    double* Vm2 = (double*)calloc((size_t)N, sizeof(double)); /* V_{*,i-2} */
    double* Vm1 = (double*)malloc(sizeof(double) * (size_t)N); /* V_{*,i-1} */
    double* Vi = (double*)malloc(sizeof(double) * (size_t)N);  /* V_{*,i}   */
    for (int64_t c = 0; c < N; ++c) Vm1[c] = v[c] / nv;          /* V_{*,1} <- v */
    for (int32_t r = 0; r < n_out; ++r) P[(int64_t)r * k + 0] = oracle_row_dot(A, &rows[r], Vm1);
    double hmax = 0.0;
    *k_eff = k;
    for (int32_t i = 2; i <= k + 1; ++i) {
        oracle_op_apply(A, Vm1, Vi); /* V_{*,i} <- A V_{*,i-1} */
        if (i > 2) {
            double h = beta[i - 3]; /* H_{i-2,i-1} <- H_{i-1,i-2} */
            for (int64_t c = 0; c < N; ++c) Vi[c] = Vi[c] - h * Vm2[c];
        }
        double a = oracle_dot(Vm1, Vi, N); /* H_{i-1,i-1} <- V_{*,i-1}^T V_{*,i} */
        alpha[i - 2] = a;
        for (int64_t c = 0; c < N; ++c) Vi[c] = Vi[c] - a * Vm1[c];
        if (fabs(a) > hmax) hmax = fabs(a);
        double nb = sqrt(oracle_dot(Vi, Vi, N)); /* H_{i,i-1} <- ||V_{*,i}|| */
        beta[i - 2] = nb;
        if (breakdown(nb, hmax)) { /* exact: the approximation is exact at k_eff = i-1 */
            *k_eff = i - 1;
            break;
        }
        if (nb > hmax) hmax = nb;
        if (i == k + 1) break; /* the extra column V_{*,k+1} is discarded */
        for (int64_t c = 0; c < N; ++c) Vi[c] = Vi[c] / nb; /* V_{*,i} <- V_{*,i} / H_{i,i-1} */
        for (int32_t r = 0; r < n_out; ++r) P[(int64_t)r * k + (i - 1)] = oracle_row_dot(A, &rows[r], Vi);
        double* t = Vm2; /* rotate: free-memory(V_{*,i-2}) */
        Vm2 = Vm1;
        Vm1 = Vi;
        Vi = t;
    }
    free(Vm2);
    free(Vm1);
    free(Vi);
    return 0;
}

/* ---------------------------------------------------------------------------------------------
 * Arnoldi, literally Algorithm 1 with modified Gram-Schmidt. The printed inner loop
 * "for j from 1 to i" is read as j = 1..i-1 (j = i would project V_{*,i} against
 * itself). P_{*,i} = C V_{*,i} as in Alg. 4.
 * Out: H[(row)*k + col] for rows 0..k (the (k+1) x k Hessenberg, row k holds h_{k+1,k}),
 *      P[r*k + i], *beta0, *k_eff. Returns 0 or 7 (zero start vector).
 * ------------------------------------------------------------------------------------------- */
int oracle_arnoldi(const oracle_op* A, const double* v, int32_t k, int32_t n_out, const oracle_row* rows,
                   double* H, double* P, double* beta0, int32_t* k_eff) {
    int64_t N = oracle_op_dim(A);
    double nv = sqrt(oracle_dot(v, v, N));
    *beta0 = nv;
    if (nv == 0.0) return 7;
    memset(H, 0, sizeof(double) * (size_t)(k + 1) * (size_t)k);
    double* V = (double*)malloc(sizeof(double) * (size_t)N * (size_t)(k + 1));
    for (int64_t c = 0; c < N; ++c) V[c] = v[c] / nv; /* V_{*,1} <- v */
    for (int32_t r = 0; r < n_out; ++r) P[(int64_t)r * k + 0] = oracle_row_dot(A, &rows[r], V);
    double hmax = 0.0;
    *k_eff = k;
    for (int32_t i = 2; i <= k + 1; ++i) {
        double* Vi = V + (int64_t)(i - 1) * N;
        const double* Vprev = V + (int64_t)(i - 2) * N;
        oracle_op_apply(A, Vprev, Vi); /* V_{*,i} <- A V_{*,i-1} */
        for (int32_t j = 1; j <= i - 1; ++j) {
            const double* Vj = V + (int64_t)(j - 1) * N;
            double h = oracle_dot(Vj, Vi, N); /* H_{j,i-1} <- V_{*,j}^T V_{*,i} */
            H[(int64_t)(j - 1) * k + (i - 2)] = h;
            for (int64_t c = 0; c < N; ++c) Vi[c] = Vi[c] - h * Vj[c];
            if (fabs(h) > hmax) hmax = fabs(h);
        }
        double nb = sqrt(oracle_dot(Vi, Vi, N)); /* H_{i,i-1} <- ||V_{*,i}|| */
        H[(int64_t)(i - 1) * k + (i - 2)] = nb;
        if (breakdown(nb, hmax)) {
            *k_eff = i - 1;
            break;
        }
        if (nb > hmax) hmax = nb;
        if (i == k + 1) break;
        for (int64_t c = 0; c < N; ++c) Vi[c] = Vi[c] / nb; /* V_{*,i} <- V_{*,i} / H_{i,i-1} */
        for (int32_t r = 0; r < n_out; ++r) P[(int64_t)r * k + (i - 1)] = oracle_row_dot(A, &rows[r], Vi);
    }
    free(V);
    return 0;
}

/* ---------------------------------------------------------------------------------------------
 * Small dense matrix exponential by scaling and squaring with a diagonal Pade approximant — the
 * "squaring and scaling and Pade approximation (methods 2 and 3 [Moler-Van Loan])" that P:508-510
 * names; the version of Golub & Van Loan (Alg. 11.3.1): q = 8, scale by 2^-s so ||M/2^s||_inf <= 1/2,
 * N_q = sum c_j X^j, D_q = sum (-1)^j c_j X^j with c_j = c_{j-1} (q-j+1) / ((2q-j+1) j),
 * F = D_q^{-1} N_q (Gaussian elimination, partial pivoting), then F <- F^2 s times.
 * Deliberately a different Pade than the GPU's (SURVEY §8(c) C-alg step 4).
 * M, F: n x n row-major. Returns 0.
 * ------------------------------------------------------------------------------------------- */
static void matmul(int n, const double* X, const double* Y, double* Z) {
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = 0.0;
            for (int l = 0; l < n; ++l) s += X[i * n + l] * Y[l * n + j];
            Z[i * n + j] = s;
        }
}

int oracle_expm(int32_t n, const double* M, double* F) {
    if (n <= 0) return 0;
    size_t nn = (size_t)n * (size_t)n;
    double* A = (double*)malloc(sizeof(double) * nn);
    double* X = (double*)malloc(sizeof(double) * nn);
    double* T = (double*)malloc(sizeof(double) * nn);
    double* Nq = (double*)malloc(sizeof(double) * nn);
    double* Dq = (double*)malloc(sizeof(double) * nn);
    double nrm = 0.0;
    for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int j = 0; j < n; ++j) s += fabs(M[i * n + j]);
        if (s > nrm) nrm = s;
    }
    int s = 0;
    while (ldexp(nrm, -s) > 0.5) ++s;
    for (size_t e = 0; e < nn; ++e) A[e] = ldexp(M[e], -s);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double d = i == j ? 1.0 : 0.0;
            X[i * n + j] = d;
            Nq[i * n + j] = d;
            Dq[i * n + j] = d;
        }
    const int q = 8;
    double c = 1.0;
    for (int j = 1; j <= q; ++j) {
        c = c * (double)(q - j + 1) / ((double)(2 * q - j + 1) * (double)j);
        matmul(n, A, X, T);
        memcpy(X, T, sizeof(double) * nn);
        double sg = (j % 2 == 0) ? 1.0 : -1.0;
        for (size_t e = 0; e < nn; ++e) {
            Nq[e] = Nq[e] + c * X[e];
            Dq[e] = Dq[e] + sg * c * X[e];
        }
    }
    /* Solve Dq F = Nq by Gaussian elimination with partial pivoting. */
    for (int col = 0; col < n; ++col) {
        int piv = col;
        for (int i = col + 1; i < n; ++i)
            if (fabs(Dq[i * n + col]) > fabs(Dq[piv * n + col])) piv = i;
        if (piv != col)
            for (int j = 0; j < n; ++j) {
                double t = Dq[col * n + j];
                Dq[col * n + j] = Dq[piv * n + j];
                Dq[piv * n + j] = t;
                t = Nq[col * n + j];
                Nq[col * n + j] = Nq[piv * n + j];
                Nq[piv * n + j] = t;
            }
        for (int i = col + 1; i < n; ++i) {
            double f = Dq[i * n + col] / Dq[col * n + col];
            for (int j = col; j < n; ++j) Dq[i * n + j] = Dq[i * n + j] - f * Dq[col * n + j];
            for (int j = 0; j < n; ++j) Nq[i * n + j] = Nq[i * n + j] - f * Nq[col * n + j];
        }
    }
    for (int i = n - 1; i >= 0; --i)
        for (int j = 0; j < n; ++j) {
            double t = Nq[i * n + j];
            for (int l = i + 1; l < n; ++l) t = t - Dq[i * n + l] * F[l * n + j];
            F[i * n + j] = t / Dq[i * n + i];
        }
    for (int r = 0; r < s; ++r) {
        matmul(n, F, F, T);
        memcpy(F, T, sizeof(double) * nn);
    }
    free(A);
    free(X);
    free(T);
    free(Nq);
    free(Dq);
    return 0;
}

/* e^{H t_j} e_1 for t_j = (double)j * step, j = 0..n_steps (never accumulate t).
 * Eq. 2: e^{At}v ~= ||v|| V_k e^{H_k t} e_1, with one (V_k, H_k) reused for every t
 * (P:646-650). H: k x k row-major. X: (n_steps+1) x k. */
int oracle_expm_e1_times(int32_t k, const double* H, double step, int64_t n_steps, double* X) {
    size_t kk = (size_t)k * (size_t)k;
    double* M = (double*)malloc(sizeof(double) * kk);
    double* F = (double*)malloc(sizeof(double) * kk);
    for (int64_t j = 0; j <= n_steps; ++j) {
        double t = (double)j * step;
        for (size_t e = 0; e < kk; ++e) M[e] = H[e] * t;
        oracle_expm(k, M, F);
        for (int i = 0; i < k; ++i) X[j * k + i] = F[i * k + 0];
    }
    free(M);
    free(F);
    return 0;
}
