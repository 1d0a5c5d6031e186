// kr_tridc.cu — the large-k route's exponentials for the symmetric Lanczos tridiagonal H_k (Alg. 3/4)
// through its eigendecomposition, as the oracle computes them (oracle.eig_e1_times: x_j = Q e^{Lambda t_j} Q^T e_1),
// with the eigen-solve itself on the device: a bottom-up divide and conquer (Cuppen rank-one tearing of the
// tridiagonal at every off-diagonal, LAPACK-style deflation, secular roots by two-pole rational interpolation with
// a bisection safeguard, Gu-Eisenstat recomputed z so the eigenvectors stay orthogonal) that never forms Q: each
// node carries only the rows of its eigenvector matrix the path needs —
//   e_1^T Q      (Q^T e_1: the start vector in the eigenbasis),
//   e_k^T Q      (Lemma 1's e_k^T e^{H t} e_1),
//   P Q          (the projected basis of Alg. 4, Eq. 6: the outputs c_j = beta0 P x_j),
// so a merge is O(n^2) and the whole solve O(k^2) instead of the O(k^3) squarings of the Taylor route. Then
//   e_k^T x_j = sum_l (e_k^T Q)_l (e_1^T Q)_l e^{lambda_l t_j},  c_j = beta0 sum_l (P Q)_{:,l} (e_1^T Q)_l e^{lambda_l t_j}
// for every time point (t_0: x_0 = e_1 exactly, as the oracle). One cooperative kernel per checkpoint: the levels
// with nodes of up to 32 entries on a CTA per 32-block (merge a lane per entry, deflation by warp segments, roots /
// z / rows 8 lanes per entry; CTA barriers only), the larger levels in four grid-synced phases (merge + deflation a
// CTA per node; roots, z, rows a warp per entry with the node's scalars staged in shared memory), then the time
// grid a warp per t_j.
// Every sum has a fixed order (lane-strided partials, xor-butterfly), so runs are bitwise reproducible.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>

#include "kr_internal.h"

namespace cg = cooperative_groups;

namespace {

constexpr int NT = 256;  // threads per CTA
constexpr int NW = NT / 32;
constexpr int LOCAL = 32;  // node sizes handled by a CTA per 32-block
constexpr int LG = NT / LOCAL;  // lanes per entry in the 32-block levels
constexpr int RMAX = 8;    // carried rows accumulated per pass in the rows update
constexpr double EPSM = 0x1.0p-53;  // unit roundoff (LAPACK dlamch('E'))
constexpr uint8_t F_SMALL = 1, F_MARK = 2;
constexpr int LOC_D = 14 + RMAX, LOC_I = 7;  // doubles / ints per entry of a warp's 32-block in shared memory

struct DC {
    const LzScalars* sc;
    int kc;
    const double* P;  // [n_out][kstride]
    int kstride, n_out;
    int R, ld;  // carried rows (2 + n_out), leading dimension of the row arrays
    int lch;    // time-grid chunk of eigen-entries staged in shared memory
    size_t smem_bytes;  // dynamic shared memory of the launch
    double* lam;   // [ld] eigenvalues per node, ascending within the node
    double* W;     // [R][ld] carried rows: 0 = first row, 1 = last row, 2.. = P rows
    double* Wp;    // [R][ld] merged children rows (sorted, rotated) of the level being built
    // per-level scalars of the large nodes, at the node's offset lo
    double* dK;    // non-deflated poles
    double* zK;    // their z
    int* colK;     // their column in Wp
    double* dorg;  // root origin pole
    double* tau;   // root offset from its origin
    double* lamR;  // roots (dorg + tau)
    double* zh;    // Gu-Eisenstat z
    double* dval;  // deflated eigenvalues (ascending)
    int* dcol;     // their column in Wp
    int* rotP;     // deflation rotations
    int* rotN;
    double* rotC;
    double* rotS;
    int* ninfo;    // [3 ld] per node: K, deflated, rotations
    double* nrho;  // [ld] per node rho
    // time grid
    double step;
    int64_t n_steps;
    const double* beta0;
    double* coeff;
    int ndl_stride, dl;
    double* hlast;
    unsigned long long* prof;  // KR_TRIDC_PROF: %globaltimer at every grid barrier (CTA 0), else NULL
};

__device__ __forceinline__ void wstamp(const DC& g, int& k, int gw) {  // CTA 0's phases of the 32-block levels
    if (g.prof && gw == 0 && (threadIdx.x & 31) == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g.prof[100 + k] = t;
    }
    ++k;
}
__device__ __forceinline__ void wend(const DC& g, int k) {  // the latest CTA to finish the work before barrier k
    if (g.prof && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        atomicMax(g.prof + 150 + k, t);
    }
}
__device__ __forceinline__ void stamp(const DC& g, int& k) {
    if (g.prof && blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g.prof[k] = t;
    }
    ++k;
}

// One node's scalar arrays (pointers offset to the node): in global memory for the large nodes, in the CTA's
// shared memory for the nodes of a 32-block.
struct NodeArrays {
    double *dK, *zK, *dorg, *tau, *lamR, *zh, *dval, *rotC, *rotS;
    int *colK, *dcol, *rotP, *rotN;
    int* info;
    double* rho;
};
__device__ __forceinline__ NodeArrays node_global(const DC& g, int q, int lo) {
    return NodeArrays{g.dK + lo,   g.zK + lo,   g.dorg + lo, g.tau + lo,  g.lamR + lo, g.zh + lo,
                      g.dval + lo, g.rotC + lo, g.rotS + lo, g.colK + lo, g.dcol + lo, g.rotP + lo,
                      g.rotN + lo, g.ninfo + 3 * q, g.nrho + q};
}

// ---- teams that merge one node: the CTA (large nodes) or a segment of w lanes of warp 0 (the nodes of a 32-block:
// every lane of the warp calls in, each segment for its own node) ---------------------------------------------
struct CtaTeam {
    double* rd;  // NW doubles
    int* ri;     // NW + 1 ints
    __device__ int rank() const { return threadIdx.x; }
    __device__ int size() const { return NT; }
    __device__ int span(int n) const { return n; }  // trip bound of loops containing team scans
    __device__ void sync() const { __syncthreads(); }
    __device__ double max(double x) const {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
        __syncthreads();
        if ((threadIdx.x & 31) == 0) rd[threadIdx.x >> 5] = x;
        __syncthreads();
        double m = rd[0];
        for (int w = 1; w < NW; ++w) m = fmax(m, rd[w]);
        return m;
    }
    __device__ bool any(bool x) const { return __syncthreads_or(x) != 0; }
    // exclusive prefix of x in rank order, total in *tot
    __device__ int scan(int x, int* tot) const {
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        int v = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        __syncthreads();
        if (lane == 31) ri[w] = v;
        __syncthreads();
        int base = 0, all = 0;
        for (int q = 0; q < NW; ++q) {
            if (q < w) base += ri[q];
            all += ri[q];
        }
        *tot = all;
        return base + v - x;
    }
};
struct SegTeam {
    int w;  // segment width: a power of two <= 32
    __device__ int rank() const { return (threadIdx.x & 31) & (w - 1); }
    __device__ int size() const { return w; }
    __device__ int span(int) const { return w; }  // one chunk for every segment: the same shuffles in all of them
    __device__ void sync() const { __syncwarp(); }
    __device__ double max(double x) const {
        for (int o = w / 2; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
        return x;
    }
    __device__ bool any(bool x) const { return __any_sync(0xffffffffu, x); }  // warp-wide: one path for all segments
    __device__ int scan(int x, int* tot) const {
        int v = x;
        for (int o = 1; o < w; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, v, o, w);
            if (rank() >= o) v += y;
        }
        *tot = __shfl_sync(0xffffffffu, v, w - 1, w);
        return v - x;
    }
};

// 1/x without the IEEE division's slow-path branch (which serialises every division of a loop): the MUFU
// approximation refined by two Newton steps (relative error ~2^-52, not correctly rounded; deterministic)
__device__ __forceinline__ double frcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

// number of a[0..n) below v / not above v (a ascending)
__device__ __forceinline__ int count_lt(const double* a, int n, double v) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}
__device__ __forceinline__ int count_le(const double* a, int n, double v) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] <= v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// ---- group reductions over G lanes (G = 1: a thread, G = 32: a warp; every lane gets the same value) --------
template <int G>
__device__ __forceinline__ double gsum(double x) {
    if (G > 1) {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    }
    return x;
}
// N sums reduced together: the N shuffles of a level are independent and issue back to back
template <int G, int N>
__device__ __forceinline__ void gsumN(double (&v)[N]) {
    if (G > 1) {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
            double t[N];
#pragma unroll
            for (int q = 0; q < N; ++q) t[q] = __shfl_xor_sync(0xffffffffu, v[q], o);
#pragma unroll
            for (int q = 0; q < N; ++q) v[q] += t[q];
        }
    }
}
template <int G>
__device__ __forceinline__ double gprod(double x) {
    if (G > 1) {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) x *= __shfl_xor_sync(0xffffffffu, x, o);
    }
    return x;
}
template <int G>
__device__ __forceinline__ int gisum(int x) {
    if (G > 1) {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    }
    return x;
}

// ---- node geometry at level size s ---------------------------------------------------------------------------
struct Node {
    int lo, m, hi;
    __device__ bool merges() const { return m < hi; }
};
__device__ __forceinline__ Node node_of(int q, int s, int kc) {
    Node n;
    n.lo = q * s;
    n.hi = min(n.lo + s, kc);
    n.m = n.lo + s / 2;
    return n;
}

__device__ unsigned long long* g_prof_iters;  // KR_TRIDC_PROF: secular iterations (sum, roots, max), deflation scans

// ---- merge step 1: the children's sorted lists merged, z, the rows permuted ---------------------------------
// Children eigenvalues lamIn[0..n1), lamIn[n1..n) (each ascending) and rows in g.W at columns colLo + i. The
// tearing at the split (first index m of the right child) subtracts |b| from both adjacent diagonal entries (done
// at the leaves), so H = diag(H1', H2') + rho u u^T, u = e_{m-1} + sign(b) e_m, rho = |b|, b = beta[m] (1-based
// Lanczos arrays); in the children's eigenbases z = [last row of child 1; sign(b) first row of child 2]. Scaled
// as LAPACK: z / sqrt(2), rho * 2. Entry i goes to sorted position r: sD[r], sZ[r], Wp column colLo + r.
__device__ __forceinline__ void merge_entry(const DC& g, const double* lamIn, int n, int n1, double sg, int colLo,
                                            int i, double* sD, double* sZ) {
    const int ld = g.ld, R = g.R;
    const double v = lamIn[i];
    int r;
    double z;
    if (i < n1) {
        r = i + count_lt(lamIn + n1, n - n1, v);
        z = g.W[ld + colLo + i];
    } else {
        r = (i - n1) + count_le(lamIn, n1, v);
        z = sg * g.W[colLo + i];
    }
    sD[r] = v;
    sZ[r] = z * 0.70710678118654752440;
    g.Wp[colLo + r] = i < n1 ? g.W[colLo + i] : 0.0;
    g.Wp[ld + colLo + r] = i < n1 ? 0.0 : g.W[ld + colLo + i];
    for (int rr = 2; rr < R; ++rr) g.Wp[(size_t)rr * ld + colLo + r] = g.W[(size_t)rr * ld + colLo + i];
}

// ---- merge step 2: deflation in LAPACK dlaed2's order, rotations on the rows ---------------------------------
// sD, sZ: the node's sorted poles and z (n entries). Small rho |z_i| <= tol deflates i; between consecutive
// survivors p < q with rotation (c, s) zeroing z_p, |(d_q - d_p) c s| <= tol deflates p with the rotated pole
// (chains: q's pole and z change and q is tested against the next survivor). The survivors go to na.dK / zK /
// colK, the deflated to na.dval / dcol in ascending order, the rotations (in order) are applied to Wp.
template <class TM>
__device__ void deflate(const DC& g, const TM& tm, int n, double rho, int colLo, double* sA, double* sD,
                        double* sZ, int* sI, uint8_t* sF, const NodeArrays& na) {
    const int ld = g.ld, R = g.R;
    double mx = 0.0;
    for (int i = tm.rank(); i < n; i += tm.size()) mx = fmax(mx, fmax(fabs(sD[i]), fabs(sZ[i])));
    mx = tm.max(mx);
    const double tol = 8.0 * EPSM * mx;
    // flags: small z; MARK: the rotation test against the next survivor passes on the unmodified values (only
    // then, or after a modification, does the sequential scan do any arithmetic)
    bool mark_any = false;
    for (int i = tm.rank(); i < n; i += tm.size()) {
        uint8_t f = rho * fabs(sZ[i]) <= tol ? F_SMALL : 0;
        if (!f) {
            int j = i + 1;
            while (j < n && rho * fabs(sZ[j]) <= tol) ++j;
            if (j < n) {  // |(d_j - d_i) c s| <= tol with c s = -z_j z_i / (z_i^2 + z_j^2)
                const double zs = sZ[i], zc = sZ[j];
                if (fabs((sD[j] - sD[i]) * zc * zs) <= tol * fma(zc, zc, zs * zs)) {
                    f |= F_MARK;
                    mark_any = true;
                }
            }
        }
        sF[i] = f;
    }
    const bool any = tm.any(mark_any);  // synchronises: sF complete
    if (!any) {
        // no rotation anywhere: keep the survivors, deflate the small ones, both already in sorted order
        int kept = 0, defl = 0;
        for (int c0 = 0; c0 < tm.span(n); c0 += tm.size()) {
            const int i = c0 + tm.rank();
            const bool keep = i < n && !(sF[i] & F_SMALL);
            const bool dfl = i < n && (sF[i] & F_SMALL);
            int tk, td;
            const int pk = tm.scan(keep ? 1 : 0, &tk);
            const int pd = tm.scan(dfl ? 1 : 0, &td);
            if (keep) {
                na.dK[kept + pk] = sD[i];
                na.zK[kept + pk] = sZ[i];
                na.colK[kept + pk] = colLo + i;
            } else if (dfl) {
                na.dval[defl + pd] = sD[i];
                na.dcol[defl + pd] = colLo + i;
            }
            kept += tk;
            defl += td;
        }
        if (tm.rank() == 0) {
            na.info[0] = kept;
            na.info[1] = defl;
            na.info[2] = 0;
            *na.rho = rho;
        }
        tm.sync();
        return;
    }
    // the sequential scan (one thread, shared memory); deflated values insertion-sorted into sA / sI
    if (tm.rank() == 0) {
        int K = 0, nd = 0, nr = 0, pj = -1;
        bool pmod = false;
        auto keep = [&](int p) {
            na.dK[K] = sD[p];
            na.zK[K] = sZ[p];
            na.colK[K] = colLo + p;
            ++K;
        };
        auto defl = [&](double v, int p) {
            int j = nd;
            while (j > 0 && sA[j - 1] > v) {
                sA[j] = sA[j - 1];
                sI[j] = sI[j - 1];
                --j;
            }
            sA[j] = v;
            sI[j] = colLo + p;
            ++nd;
        };
        for (int nj = 0; nj < n; ++nj) {
            if (sF[nj] & F_SMALL) {
                defl(sD[nj], nj);
                continue;
            }
            if (pj < 0) {
                pj = nj;
                pmod = false;
                continue;
            }
            if (!pmod && !(sF[pj] & F_MARK)) {
                keep(pj);
                pj = nj;
                pmod = false;
                continue;
            }
            const double zs = sZ[pj], zc = sZ[nj];
            if (fabs((sD[nj] - sD[pj]) * zc * zs) <= tol * fma(zc, zc, zs * zs)) {
                const double t = sqrt(fma(zc, zc, zs * zs));  // z <= 1: no overflow
                const double c = zc / t, sn = -zs / t;
                sZ[nj] = t;
                sZ[pj] = 0.0;
                na.rotP[nr] = colLo + pj;
                na.rotN[nr] = colLo + nj;
                na.rotC[nr] = c;
                na.rotS[nr] = sn;
                ++nr;
                const double dp = sD[pj] * c * c + sD[nj] * sn * sn;
                sD[nj] = sD[pj] * sn * sn + sD[nj] * c * c;
                sD[pj] = dp;
                defl(dp, pj);
                pj = nj;
                pmod = true;
            } else {
                keep(pj);
                pj = nj;
                pmod = false;
            }
        }
        if (pj >= 0) keep(pj);
        na.info[0] = K;
        na.info[1] = nd;
        na.info[2] = nr;
        *na.rho = rho;
        if (g_prof_iters) {  // KR_TRIDC_PROF: nodes through the sequential scan, rotations
            atomicAdd(g_prof_iters + 7, 1ull);
            atomicAdd(g_prof_iters + 8, (unsigned long long)nr);
        }
    }
    tm.sync();
    const int ndf = na.info[1], nr = na.info[2];
    for (int i = tm.rank(); i < ndf; i += tm.size()) {
        na.dval[i] = sA[i];
        na.dcol[i] = sI[i];
    }
    // rotations, in order, on the carried rows (DROT: x' = c x + s y, y' = c y - s x)
    for (int rr = tm.rank(); rr < R; rr += tm.size()) {
        double* w = g.Wp + (size_t)rr * ld;
        for (int r = 0; r < nr; ++r) {
            const int a = na.rotP[r], bb = na.rotN[r];
            const double c = na.rotC[r], sn = na.rotS[r];
            const double x = w[a], y = w[bb];
            w[a] = c * x + sn * y;
            w[bb] = c * y - sn * x;
        }
    }
    tm.sync();
}


// ---- secular root j of f(lam) = 1 + rho sum_i z_i^2 / (d_i - lam), d ascending, rho > 0 -------------------------
// Root j < K-1 lies in (d_j, d_{j+1}), the last in (d_{K-1}, d_{K-1} + rho |z|^2]. It is represented as
// origin + tau with the origin the nearer pole, so d_i - lam = (d_i - d_origin) - tau is accurate. Iteration:
// the two sums on either side of the root each matched (value and derivative) by c + s / (pole - tau) at the two
// nearest poles, the quadratic's near root taken (Li's "middle way", as dlaed4), a bisection step whenever it
// leaves the bracket; stop when |f| is below its rounding bound.
template <int G>
__device__ void secular_root(const double* d, const double* z, int K, double rho, int j, int lane, bool active,
                             double* dorg_o, double* tau_o) {
    // every group of the warp runs the same loop (warp-wide shuffles and exit vote): inactive groups and K = 1
    // (root d_0 + rho z_0^2, exact) start frozen
    const long long c_start = clock64();
    const bool solve = active && K > 1;
    const bool interior = solve && j < K - 1;
    // interior root: the first pass is at the midpoint of (d_j, d_{j+1}) with the origin at d_j; its sign picks
    // the half and the origin (the nearer pole) and its sums feed the first rational step. Last root: origin
    // d_{K-1}, bracket (0, rho].
    int org = 0, p1 = 0;
    double lo = 0.0, hi = 0.0, tau = 0.0, gap = 0.0;
    if (interior) {
        org = j;
        p1 = j;
        gap = d[j + 1] - d[j];
        hi = gap;
        tau = 0.5 * gap;
    } else if (solve) {
        org = K - 1;
        p1 = K - 2;
        hi = rho;
        tau = 0.5 * rho;
    }
    const int p2 = p1 + 1;
    double dorg = solve ? d[org] : 0.0;
    double dl1 = solve ? d[p1] - dorg : 0.0, dl2 = solve ? d[p2] - dorg : 0.0;
    const int Ks = solve ? K : 0;
    int it = 0;
    bool fin = !solve;
    for (; it < 200; ++it) {
        double s1 = 0.0, s2 = 0.0, q1 = 0.0, q2 = 0.0, ea = 0.0;
#pragma unroll 4
        for (int i = lane; i < Ks; i += G) {
            const double r = frcp((d[i] - dorg) - tau);
            const double t = rho * z[i] * z[i] * r;
            const double tq = t * r;
            const bool left = i <= p1;
            ea += fabs(t);
            s1 += left ? t : 0.0;
            q1 += left ? tq : 0.0;
            s2 += left ? 0.0 : t;
            q2 += left ? 0.0 : tq;
        }
        double v5[5] = {s1, s2, q1, q2, ea};
        gsumN<G, 5>(v5);
        s1 = v5[0];
        s2 = v5[1];
        q1 = v5[2];
        q2 = v5[3];
        ea = v5[4];
        const double f = 1.0 + s1 + s2;
        // converged groups freeze; the loop ends when every group of the warp has (one warp-uniform exit, so the
        // shuffles always see the whole warp)
        if (!fin && fabs(f) <= 8.0 * EPSM * (1.0 + ea)) fin = true;
        if (!fin) {
            if (f > 0.0) hi = tau; else lo = tau;
            if (it == 0 && interior && f <= 0.0) {  // root in the upper half: origin d_{j+1} (shift by the gap)
                tau -= gap;
                lo -= gap;
                hi = 0.0;
                dl1 -= gap;
                dl2 = 0.0;
                dorg = d[j + 1];
            }
            // the matched pole terms b / (pole - tau) with b = q (pole - tau)^2: a = s - q (pole - tau), no division
            const double D1 = dl1 - tau, D2 = dl2 - tau;
            const double a1 = s1 - q1 * D1, a2 = s2 - q2 * D2;
            const double b1 = q1 * D1 * D1, b2 = q2 * D2 * D2;
            const double c = 1.0 + a1 + a2;
            const double B = c * (D1 + D2) + b1 + b2;
            const double C = D1 * D2 * f;
            double eta;
            if (c == 0.0) {
                eta = C * frcp(B);
            } else {
                const double disc = fmax(B * B - 4.0 * c * C, 0.0);
                eta = 2.0 * C * frcp(B + copysign(sqrt(disc), B));
            }
            double tn = tau + eta;
            const bool bis = !(tn > lo && tn < hi) || !isfinite(tn);
            if (bis) tn = 0.5 * (lo + hi);
            // a rational step below 1e-10 of the offset: the next one (quadratic convergence) is below rounding
            if (tn == tau || (!bis && fabs(eta) <= 1e-10 * fabs(tn))) fin = true;
            tau = tn;
        }
        if (__all_sync(0xffffffffu, fin)) break;
    }
    if (active && K == 1) {
        *dorg_o = d[0];
        *tau_o = rho * z[0] * z[0];
    } else {
        *dorg_o = dorg;
        *tau_o = tau;
    }
    if (g_prof_iters && lane == 0 && solve) {
        atomicAdd(g_prof_iters, (unsigned long long)it);
        atomicAdd(g_prof_iters + 1, 1ull);
        atomicMax(g_prof_iters + 2, (unsigned long long)it);
        atomicAdd(g_prof_iters + 3, (unsigned long long)(clock64() - c_start));
        if (G == 32) {
            atomicAdd(g_prof_iters + 4, (unsigned long long)(clock64() - c_start));
            atomicAdd(g_prof_iters + 5, 1ull);
            atomicAdd(g_prof_iters + 6, (unsigned long long)K);
        }
    }
}

// ---- Gu-Eisenstat z_x^2 = prod_j (lam_j - d_x) / (rho prod_{j != x} (d_j - d_x)), lam_j - d_x = (dorg_j - d_x) + tau_j
template <int G>
__device__ __forceinline__ double gu_eisenstat_z(const double* d, const double* dorg, const double* tau, int K,
                                                 double rho, double zsign, int x, int lane, bool active = true) {
    const int Ke = active ? K : 0;
    const double dx = active ? d[x] : 0.0;
    double p = 1.0;
#pragma unroll 4
    for (int j = lane; j < Ke; j += G) {
        const double lj = (dorg[j] - dx) + tau[j];
        p *= lj * frcp(j == x ? rho : d[j] - dx);
    }
    p = gprod<G>(p);
    return copysign(sqrt(fmax(p, 0.0)), zsign);
}

// ---- rows of eigenvector j: W[:, dst] = sum_i Wp[:, colK_i] u_i / |u|, u_i = zh_i / (d_i - lam_j) -------------
// STAGED: the K source columns are in shared memory as src[r * sld + i]; else read from Wp through colK.
template <int G, bool STAGED>
__device__ __forceinline__ void eigvec_rows(const DC& g, const double* d, const double* zh, const int* colK,
                                            const double* src, int sld, int Kn, double dorg, double tj, int dst,
                                            int lane, bool active = true) {
    const int K = active ? Kn : 0;  // inactive groups run the same reductions and write nothing
    double nrm = 0.0;
    for (int r0 = 0; r0 < g.R; r0 += RMAX) {
        double acc[RMAX];
#pragma unroll
        for (int r = 0; r < RMAX; ++r) acc[r] = 0.0;
#pragma unroll 4
        for (int i = lane; i < K; i += G) {
            const double u = zh[i] * frcp((d[i] - dorg) - tj);
            if (r0 == 0) nrm = fma(u, u, nrm);
            if (STAGED) {
#pragma unroll
                for (int r = 0; r < RMAX; ++r)
                    if (r0 + r < g.R) acc[r] = fma(src[(r0 + r) * sld + i], u, acc[r]);
            } else {
                const int col = colK[i];
#pragma unroll
                for (int r = 0; r < RMAX; ++r)
                    if (r0 + r < g.R) acc[r] = fma(__ldcg(&g.Wp[(size_t)(r0 + r) * g.ld + col]), u, acc[r]);
            }
        }
        double v[RMAX + 1];
#pragma unroll
        for (int r = 0; r < RMAX; ++r) v[r] = acc[r];
        v[RMAX] = nrm;
        gsumN<G, RMAX + 1>(v);
        if (r0 == 0) nrm = v[RMAX];
        const double inv = 1.0 / sqrt(nrm);
#pragma unroll
        for (int r = 0; r < RMAX; ++r)
            if (active && r0 + r < g.R && lane == 0) g.W[(size_t)(r0 + r) * g.ld + dst] = v[r] * inv;
    }
}

// ---- the kernel ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) tridc_kernel(const DC g) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double4 smem4[];
    double* smem = reinterpret_cast<double*>(smem4);
    __shared__ double red_d[NW];
    __shared__ int red_i[NW + 1];
    const int kc = g.kc, ld = g.ld;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int gw = (int)((blockIdx.x * (int64_t)NT + threadIdx.x) >> 5), nwarps = (int)(gridDim.x * NW);
    int ps = 0;
    stamp(g, ps);

    // leaves: d_i = a_i - |b_{i-1}| - |b_i| (the tearing at every off-diagonal), rows [1, 1, P[:, i]]
    for (int i = blockIdx.x * NT + threadIdx.x; i < kc; i += gridDim.x * NT) {
        double a = g.sc->alpha[i + 1];
        if (i > 0) a -= fabs(g.sc->beta[i]);
        if (i < kc - 1) a -= fabs(g.sc->beta[i + 1]);
        g.lam[i] = a;
        g.W[i] = 1.0;
        g.W[ld + i] = 1.0;
        for (int r = 0; r < g.n_out; ++r) g.W[(size_t)(2 + r) * ld + i] = g.P[(size_t)r * g.kstride + i];
    }
    __syncthreads();
    wend(g, ps);
    grid.sync();
    stamp(g, ps);

    // ---- levels s = 2 .. 32: a CTA per 32-block, everything but the rows in shared memory: merge a lane of warp 0
    // per entry, deflation a segment of s lanes of warp 0 per node, roots / z / rows a group of LG lanes per entry
    {
        constexpr int L = LOCAL;
        double* wsm = smem;
        double *sLam = wsm, *sA = wsm + L, *sD = wsm + 2 * L, *sZ = wsm + 3 * L;
        double *nK = wsm + 4 * L, *nZ = wsm + 5 * L, *nOrg = wsm + 6 * L, *nTau = wsm + 7 * L, *nLamR = wsm + 8 * L,
               *nZh = wsm + 9 * L, *nDv = wsm + 10 * L, *nRc = wsm + 11 * L, *nRs = wsm + 12 * L, *nRho = wsm + 13 * L,
               *sRows = wsm + 14 * L;  // [RMAX][L]
        int* wis = reinterpret_cast<int*>(smem + (size_t)LOC_D * L);
        int *sI = wis, *nCol = wis + L, *nDc = wis + 2 * L, *nRp = wis + 3 * L, *nRn = wis + 4 * L,
            *nInfo = wis + 5 * L;  // 3 ints per node (<= 16 nodes)
        uint8_t* sF = reinterpret_cast<uint8_t*>(wis + LOC_I * L);
        const int e = threadIdx.x / LG, gl = threadIdx.x % LG;  // entry of the group, lane in the group
        const int nblk = (kc + L - 1) / L;
        for (int blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
            const int b0 = blk * L;
            if (threadIdx.x < L && b0 + threadIdx.x < kc) sLam[threadIdx.x] = g.lam[b0 + threadIdx.x];
            __syncthreads();
            int wps = 0;
            if (gw == 0) wstamp(g, wps, 0);
            for (int s = 2; s <= L && s < 2 * kc; s <<= 1) {
                // the node of entry p of the block: offset loc, index in the block nib
                auto node_at = [&](int p, int& loc, Node& nd) {
                    loc = p & ~(s - 1);
                    nd = node_of((b0 + loc) / s, s, kc);
                };
                auto arrays = [&](int loc) {
                    const int nib = loc / s;
                    return NodeArrays{nK + loc,  nZ + loc,  nOrg + loc, nTau + loc, nLamR + loc, nZh + loc, nDv + loc,
                                      nRc + loc, nRs + loc, nCol + loc, nDc + loc,  nRp + loc,   nRn + loc,
                                      nInfo + 3 * nib, nRho + nib};
                };
                if (wib == 0) {
                    int loc;
                    Node nd;
                    node_at(lane, loc, nd);
                    const bool mg = b0 + lane < kc && nd.merges();
                    if (mg) {
                        const double b = g.sc->beta[nd.m];
                        merge_entry(g, sLam + loc, nd.hi - nd.lo, nd.m - nd.lo, b >= 0.0 ? 1.0 : -1.0, b0 + loc,
                                    lane - loc, sD + loc, sZ + loc);
                    }
                    __syncwarp();
                    // every lane calls in (segment of its node; n = 0 where the node does not merge)
                    const bool nm = b0 + loc < kc && nd.merges();
                    deflate(g, SegTeam{s}, nm ? nd.hi - nd.lo : 0, nm ? 2.0 * fabs(g.sc->beta[nd.m]) : 0.0, b0 + loc,
                            sA + loc, sD + loc, sZ + loc, sI + loc, sF + loc, arrays(loc));
                }
                __syncthreads();
                if (gw == 0) wstamp(g, wps, 0);
                int loc;
                Node nd;
                node_at(e, loc, nd);
                const bool mg = b0 + e < kc && nd.merges();
                const NodeArrays na = arrays(loc);
                const int i = e - loc;
                const int K = mg ? na.info[0] : 0, ndf = mg ? na.info[1] : 0;
                {
                    double dorg, t;
                    secular_root<LG>(na.dK, na.zK, K, mg ? *na.rho : 1.0, i, gl, mg && i < K, &dorg, &t);
                    if (mg && i < K && gl == 0) {
                        na.dorg[i] = dorg;
                        na.tau[i] = t;
                        na.lamR[i] = dorg + t;
                    }
                }
                __syncthreads();
                if (gw == 0) wstamp(g, wps, 0);
                {
                    const double zx = gu_eisenstat_z<LG>(na.dK, na.dorg, na.tau, K, mg ? *na.rho : 1.0,
                                                         mg && i < K ? na.zK[i] : 1.0, i, gl, mg && i < K);
                    if (mg && i < K && gl == 0) na.zh[i] = zx;
                    if (mg && i >= K && i < K + ndf) {  // deflated column: its place among the roots
                        const int dq = i - K;
                        const double v = na.dval[dq];
                        const int pos = dq + count_le(na.lamR, K, v);
                        if (gl == 0) sLam[loc + pos] = v;
                        const int col = na.dcol[dq];
                        for (int rr = gl; rr < g.R; rr += LG)
                            g.W[(size_t)rr * ld + b0 + loc + pos] = g.Wp[(size_t)rr * ld + col];
                    }
                    if (g.R <= RMAX && mg && i < K)  // the node's source columns into shared memory, [r][loc + i]
                        for (int rr = gl; rr < g.R; rr += LG) sRows[rr * L + loc + i] = g.Wp[(size_t)rr * ld + na.colK[i]];
                }
                __syncthreads();
                if (gw == 0) wstamp(g, wps, 0);
                {
                    const bool act = mg && i < K;
                    int pos = 0;
                    if (act) {
                        pos = i + count_lt(na.dval, ndf, na.lamR[i]);
                        if (gl == 0) sLam[loc + pos] = na.lamR[i];
                    }
                    const double dorg = act ? na.dorg[i] : 0.0, tj = act ? na.tau[i] : 0.0;
                    if (g.R <= RMAX)
                        eigvec_rows<LG, true>(g, na.dK, na.zh, nullptr, sRows + loc, L, K, dorg, tj, b0 + loc + pos, gl,
                                              act);
                    else
                        eigvec_rows<LG, false>(g, na.dK, na.zh, na.colK, nullptr, 0, K, dorg, tj, b0 + loc + pos, gl,
                                               act);
                }
                __syncthreads();
                if (gw == 0) wstamp(g, wps, 0);
            }
            if (threadIdx.x < L && b0 + threadIdx.x < kc) g.lam[b0 + threadIdx.x] = sLam[threadIdx.x];
            __syncthreads();
        }
    }
    __syncthreads();
    wend(g, ps);
    grid.sync();
    stamp(g, ps);

    // ---- levels s = 64 .. : merge + deflation a CTA per node (shared memory), then roots, z and rows by units of
    // NW entries of one node (a warp per entry) with the node's scalars staged in the CTA's shared memory;
    // a grid barrier between the four phases
    CtaTeam team{red_d, red_i};
    for (int s = 2 * LOCAL; s < 2 * kc; s <<= 1) {
        const int nq = (kc + s - 1) / s;
        const int sz = min(s, kc);  // the largest node of the level
        for (int q = blockIdx.x; q < nq; q += gridDim.x) {
            const Node nd = node_of(q, s, kc);
            if (!nd.merges()) continue;
            double* sA = smem;
            double* sD = sA + sz;
            double* sZ = sD + sz;
            int* sI = reinterpret_cast<int*>(sZ + sz);
            uint8_t* sF = reinterpret_cast<uint8_t*>(sI + sz);
            const int n = nd.hi - nd.lo, n1 = nd.m - nd.lo;
            const double b = g.sc->beta[nd.m];
            for (int i = threadIdx.x; i < n; i += NT) sA[i] = g.lam[nd.lo + i];
            __syncthreads();
            for (int i = threadIdx.x; i < n; i += NT) merge_entry(g, sA, n, n1, b >= 0.0 ? 1.0 : -1.0, nd.lo, i, sD, sZ);
            __syncthreads();
            deflate(g, team, n, 2.0 * fabs(b), nd.lo, sA, sD, sZ, sI, sF, node_global(g, q, nd.lo));
        }
        __syncthreads();
    wend(g, ps);
    grid.sync();
    stamp(g, ps);
        const int nunits = (kc + NW - 1) / NW;
        // roots
        for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
            const int p0 = u * NW, q = p0 / s;
            const Node nd = node_of(q, s, kc);
            if (!nd.merges()) continue;
            const int K = g.ninfo[3 * q], c0 = p0 - nd.lo;
            if (c0 >= K) continue;
            double* sd = smem;
            double* szz = smem + K;
            for (int i = threadIdx.x; i < K; i += NT) {
                sd[i] = g.dK[nd.lo + i];
                szz[i] = g.zK[nd.lo + i];
            }
            __syncthreads();
            const int j = c0 + wib;
            if (j < K) {
                double dorg, t;
                secular_root<32>(sd, szz, K, g.nrho[q], j, lane, true, &dorg, &t);
                if (lane == 0) {
                    g.dorg[nd.lo + j] = dorg;
                    g.tau[nd.lo + j] = t;
                    g.lamR[nd.lo + j] = dorg + t;
                }
            }
            __syncthreads();
        }
        __syncthreads();
    wend(g, ps);
    grid.sync();
    stamp(g, ps);
        // z (entries < K) and the deflated columns' places (K <= entry < K + deflated)
        for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
            const int p0 = u * NW, q = p0 / s;
            const Node nd = node_of(q, s, kc);
            if (!nd.merges()) continue;
            const int K = g.ninfo[3 * q], ndf = g.ninfo[3 * q + 1], c0 = p0 - nd.lo;
            if (c0 >= K + ndf) continue;
            double* sd = smem;
            double* so = smem + K;
            double* st = smem + 2 * K;
            double* sl = smem + 3 * K;
            for (int i = threadIdx.x; i < K; i += NT) {
                sd[i] = g.dK[nd.lo + i];
                so[i] = g.dorg[nd.lo + i];
                st[i] = g.tau[nd.lo + i];
                sl[i] = g.lamR[nd.lo + i];
            }
            __syncthreads();
            const int x = c0 + wib;
            if (x < K) {
                const double zx = gu_eisenstat_z<32>(sd, so, st, K, g.nrho[q], g.zK[nd.lo + x], x, lane);
                if (lane == 0) g.zh[nd.lo + x] = zx;
            } else if (x < K + ndf) {
                const int dq = x - K;
                const double v = g.dval[nd.lo + dq];
                int c = 0;
                for (int j = lane; j < K; j += 32) c += sl[j] <= v ? 1 : 0;
                const int pos = dq + gisum<32>(c);
                const int col = g.dcol[nd.lo + dq];
                if (lane == 0) g.lam[nd.lo + pos] = v;
                for (int rr = lane; rr < g.R; rr += 32)
                    g.W[(size_t)rr * ld + nd.lo + pos] = g.Wp[(size_t)rr * ld + col];
            }
            __syncthreads();
        }
        __syncthreads();
    wend(g, ps);
    grid.sync();
    stamp(g, ps);
        // eigenvectors: the carried rows
        for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
            const int p0 = u * NW, q = p0 / s;
            const Node nd = node_of(q, s, kc);
            if (!nd.merges()) continue;
            const int K = g.ninfo[3 * q], ndf = g.ninfo[3 * q + 1], c0 = p0 - nd.lo;
            if (c0 >= K) continue;
            double* sd = smem;
            double* szh = smem + K;
            double* sdv = smem + 2 * K;
            double* srow = smem + 2 * K + ndf;  // [R][K] when it fits
            const bool staged = (size_t)(2 * K + ndf + (size_t)g.R * K) * 8 + (size_t)K * 4 <= g.smem_bytes;
            int* scol = reinterpret_cast<int*>(staged ? srow + (size_t)g.R * K : srow);
            for (int i = threadIdx.x; i < K; i += NT) {
                sd[i] = g.dK[nd.lo + i];
                szh[i] = g.zh[nd.lo + i];
                scol[i] = g.colK[nd.lo + i];
            }
            for (int i = threadIdx.x; i < ndf; i += NT) sdv[i] = g.dval[nd.lo + i];
            if (staged)
                for (int e = threadIdx.x; e < g.R * K; e += NT) {
                    const int r = e / K, i = e - r * K;
                    srow[e] = g.Wp[(size_t)r * ld + g.colK[nd.lo + i]];
                }
            __syncthreads();
            const int j = c0 + wib;
            if (j < K) {
                const double lj = g.lamR[nd.lo + j];
                int c = 0;
                for (int i = lane; i < ndf; i += 32) c += sdv[i] < lj ? 1 : 0;
                const int pos = j + gisum<32>(c);
                if (lane == 0) g.lam[nd.lo + pos] = lj;
                if (staged)
                    eigvec_rows<32, true>(g, sd, szh, nullptr, srow, K, K, g.dorg[nd.lo + j], g.tau[nd.lo + j],
                                          nd.lo + pos, lane);
                else
                    eigvec_rows<32, false>(g, sd, szh, scol, nullptr, 0, K, g.dorg[nd.lo + j], g.tau[nd.lo + j],
                                           nd.lo + pos, lane);
            }
            __syncthreads();
        }
        __syncthreads();
    wend(g, ps);
    grid.sync();
    stamp(g, ps);
    }

    // ---- time grid: e_k^T x_j and c_j = beta0 P x_j, x_j = sum_l (Q^T e_1)_l e^{lambda_l t_j} Q[:, l]; a CTA per
    // NW time points, the eigen-data staged in chunks of lch entries (lambda, then w_r = W_0 W_r for r = 1..R-1)
    const double b0 = *g.beta0;
    const int no = g.n_out, R = g.R, lch = g.lch;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        g.hlast[0] = kc == 1 ? 1.0 : 0.0;  // x_0 = e_1 exactly
        for (int r = 0; r < no; ++r) g.coeff[(size_t)r * g.ndl_stride + g.dl] = b0 * g.P[(size_t)r * g.kstride];
    }
    double* sl = smem;
    double* sw = smem + lch;  // [R-1][lch]
    for (int64_t j0 = 1 + (int64_t)blockIdx.x * NW; j0 <= g.n_steps; j0 += (int64_t)gridDim.x * NW) {
        const int64_t j = j0 + wib;
        const double t = (double)j * g.step;
        for (int r0 = 0; r0 < R - 1; r0 += RMAX) {  // r = 0: the last row (h_j); r >= 1: P rows
            double acc[RMAX];
#pragma unroll
            for (int r = 0; r < RMAX; ++r) acc[r] = 0.0;
            for (int l0 = 0; l0 < kc; l0 += lch) {
                const int nl = min(lch, kc - l0);
                __syncthreads();
                for (int l = threadIdx.x; l < nl; l += NT) {
                    sl[l] = g.lam[l0 + l];
                    const double w0 = g.W[l0 + l];
                    for (int r = 0; r < R - 1; ++r) sw[(size_t)r * lch + l] = w0 * g.W[(size_t)(r + 1) * ld + l0 + l];
                }
                __syncthreads();
                if (j <= g.n_steps) {
#pragma unroll 2
                    for (int l = lane; l < nl; l += 32) {
                        const double e = exp(sl[l] * t);
#pragma unroll
                        for (int r = 0; r < RMAX; ++r)
                            if (r0 + r < R - 1) acc[r] = fma(sw[(size_t)(r0 + r) * lch + l], e, acc[r]);
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < RMAX; ++r) {
                if (r0 + r < R - 1) {
                    const double a = gsum<32>(acc[r]);
                    if (lane == 0 && j <= g.n_steps) {
                        if (r0 + r == 0)
                            g.hlast[j] = a;
                        else
                            g.coeff[((size_t)j * no + r0 + r - 1) * g.ndl_stride + g.dl] = b0 * a;
                    }
                }
            }
        }
    }
    __syncthreads();
    wend(g, ps);
    grid.sync();
    stamp(g, ps);
}

}  // namespace

// Largest dimension the divide-and-conquer route takes (the top merge stages 3 doubles + an int + a byte per
// entry in one CTA's shared memory); larger kc fall back to the Taylor route.
int kr_tridc_max_k() { return 6144; }

// Workspace for dimension kc (grown on demand, x1.5, capped at k).
static void tridc_alloc(kr_handle* h, int kc) {
    const int R = 2 + h->n_out;
    if (h->d_tdc && kc <= h->tdc_cap) return;
    int cap = std::max(kc, std::min(h->k, std::max(128, h->tdc_cap + h->tdc_cap / 2)));
    if (h->d_tdc) {
        KR_CUDA(cudaStreamSynchronize(h->stream));
        kr_dev_free(h->d_tdc);
        h->extra_allocs.erase(std::remove(h->extra_allocs.begin(), h->extra_allocs.end(), (void*)h->d_tdc),
                              h->extra_allocs.end());
        h->d_tdc = nullptr;
    }
    const size_t ld = (size_t)cap;
    const size_t doubles = ld * (2 * R + 11);  // W, Wp; lam dK zK dorg tau lamR zh dval rotC rotS nrho
    const size_t ints = ld * 7;                // colK dcol rotP rotN; ninfo (3 per node)
    KR_CUDA(kr_dev_malloc(reinterpret_cast<void**>(&h->d_tdc), doubles * 8 + ints * 4));
    h->extra_allocs.push_back(h->d_tdc);
    h->tdc_cap = cap;
}

// x_j = e^{H t_j} e_1 of the leading kc x kc block of direction dl's Lanczos tridiagonal: writes the projected
// coefficients c_j = beta0 P x_j into the local coefficient array and e_kc^T x_j into hl (Lemma 1's integrand).
void kr_tridc_eval(kr_handle* h, int dl, int kc, double* hl, int ndl_stride) {
    tridc_alloc(h, kc);
    const int R = 2 + h->n_out;
    const size_t ld = (size_t)h->tdc_cap;
    DC g{};
    g.sc = h->d_sc + dl;
    g.kc = kc;
    g.P = h->d_P + (size_t)dl * h->n_out * h->k;
    g.kstride = h->k;
    g.n_out = h->n_out;
    g.R = R;
    g.ld = (int)ld;
    double* p = reinterpret_cast<double*>(h->d_tdc);
    for (double** a : {&g.W, &g.Wp}) {
        *a = p;
        p += R * ld;
    }
    for (double** a : {&g.lam, &g.dK, &g.zK, &g.dorg, &g.tau, &g.lamR, &g.zh, &g.dval, &g.rotC, &g.rotS, &g.nrho}) {
        *a = p;
        p += ld;
    }
    int* ip = reinterpret_cast<int*>(p);
    for (int** a : {&g.colK, &g.dcol, &g.rotP, &g.rotN}) {
        *a = ip;
        ip += ld;
    }
    g.ninfo = ip;  // 3 ld
    g.step = h->step;
    g.n_steps = h->n_steps;
    g.beta0 = h->d_beta0 + dl;
    g.coeff = h->d_coeff_loc;
    g.ndl_stride = ndl_stride;
    g.dl = dl;
    g.hlast = hl;
    // shared memory: the top merge (3 doubles + int + byte per entry), the staged node scalars of the roots / z /
    // rows phases (4 doubles per entry), the warps' 32-blocks, the time-grid chunks
    g.lch = R > 16 ? 64 : 256;
    const size_t sm_top = kc > LOCAL ? (size_t)kc * 32 : 0;
    const size_t sm_loc = (size_t)LOCAL * (LOC_D * 8 + LOC_I * 4 + 1);
    const size_t sm_grid = (size_t)g.lch * R * 8;
    const size_t sm_rows = std::min<size_t>((size_t)kc * (8 * R + 28), 200 * 1024);  // staged rows of phase D
    const size_t smem = (std::max(std::max(std::max(sm_top, sm_loc), sm_grid), sm_rows) + 15) / 16 * 16;
    g.smem_bytes = smem;
    // the attribute belongs to the current device's context: set it on every call (handles on several GPUs)
    if (smem > 48 * 1024)
        KR_CUDA(cudaFuncSetAttribute(tridc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, sms = 148, per_sm = 0;
    KR_CUDA(cudaGetDevice(&dev));
    KR_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    KR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tridc_kernel, NT, smem));
    if (per_sm < 1) KR_THROW(KR_ECUDA, "tridc_kernel does not fit on an SM");
    const int64_t want = std::max<int64_t>((kc + NW - 1) / NW, (h->n_steps + NW - 1) / NW);
    int nb = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * std::min(per_sm, 2)));
    // beside a running multi-step launch: only the SM slots it leaves free (both kernels take half an SM each;
    // with more than 100 KB of shared memory two of these CTAs may not share an SM: wait for the steps instead)
    if (h->tdc_grid_cap > 0 && smem > 100 * 1024) {
        KR_CUDA(cudaStreamSynchronize(h->stream2));  // the main stream (swapped) holding the multi-step launch
    } else if (h->tdc_grid_cap > 0) {
        if (per_sm < 2) KR_THROW(KR_ECUDA, "eigen-solve beside the multi-step kernel needs two CTAs per SM");
        nb = std::min(nb, h->tdc_grid_cap);
    }
    static unsigned long long* prof = nullptr;  // KR_TRIDC_PROF diagnostics only (first device used)
    const bool want_prof = getenv("KR_TRIDC_PROF") != nullptr;
    if (want_prof && !prof) {
        KR_CUDA(cudaMalloc(&prof, 256 * 8));
        unsigned long long* pi = prof + 200;
        KR_CUDA(cudaMemcpyToSymbol(g_prof_iters, &pi, sizeof(pi)));
    }
    if (want_prof) KR_CUDA(cudaMemsetAsync(prof + 150, 0, 60 * 8, h->stream));
    g.prof = want_prof ? prof : nullptr;
    void* args[] = {(void*)&g};
    KR_CUDA(cudaLaunchCooperativeKernel((const void*)tridc_kernel, dim3(nb), dim3(NT), args, smem, h->stream));
    h->launches++;
    if (want_prof) {  // diagnostic: microseconds between the grid barriers
        unsigned long long t[256];
        KR_CUDA(cudaStreamSynchronize(h->stream));
        KR_CUDA(cudaMemcpy(t, prof, sizeof(t), cudaMemcpyDeviceToHost));
        int n = 3;
        for (int s = 2 * LOCAL; s < 2 * kc; s <<= 1) n += 4;
        fprintf(stderr, "tridc kc=%d nb=%d smem=%zu:", kc, nb, smem);
        for (int i = 1; i <= n; ++i) fprintf(stderr, " %.1f", (t[i] - t[i - 1]) * 1e-3);
        fprintf(stderr, " | work:");
        for (int i = 1; i <= n; ++i) fprintf(stderr, " %.1f", ((long long)t[150 + i] - (long long)t[i - 1]) * 1e-3);
        fprintf(stderr, " | warp 0 local:");
        for (int i = 101; i < 126; ++i) fprintf(stderr, " %.1f", (t[i] - t[i - 1]) * 1e-3);
        fprintf(stderr, " | secular iterations %llu over %llu roots, max %llu; cycles/root %.0f; warp roots %llu: cycles %.0f, K %.0f; sequential deflation scans %llu, rotations %llu\n", t[200], t[201], t[202], (double)t[203] / t[201], t[205], (double)t[204] / (t[205] ? t[205] : 1), (double)t[206] / (t[205] ? t[205] : 1), t[207], t[208]);
    }
}
