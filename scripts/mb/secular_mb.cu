// microbenchmark of the secular root solver (scripts only)
#include <cstdio>
#include <vector>
#include <cmath>
#include <algorithm>
constexpr double EPSM = 0x1.0p-53;
__device__ int g_it[4096];
__device__ long long g_cyc[4096];
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

template <int G>
__device__ void secular_root(const double* d, const double* z, int K, double rho, int j, int lane, double* dorg_o,
                             double* tau_o) {
    const long long c_start = clock64();
    if (K == 1) {
        *dorg_o = d[0];
        *tau_o = rho * z[0] * z[0];
        return;
    }
    int org, p1;
    double lo, hi;
    if (j < K - 1) {
        const double mid = 0.5 * (d[j + 1] - d[j]);
        double s = 0.0;
        for (int i0 = 0; i0 < K; i0 += G) {  // uniform trip count: the shuffles below see a converged warp
            const int i = i0 + lane;
            if (i < K) s += z[i] * z[i] * frcp((d[i] - d[j]) - mid);
        }
        const double fm = 1.0 + rho * gsum<G>(s);
        if (fm > 0.0) {
            org = j;
            lo = 0.0;
            hi = mid;
        } else {
            org = j + 1;
            lo = -mid;
            hi = 0.0;
        }
        p1 = j;
    } else {
        org = K - 1;
        lo = 0.0;
        hi = rho;
        p1 = K - 2;
    }
    const int p2 = p1 + 1;
    const double dorg = d[org];
    const double dl1 = d[p1] - dorg, dl2 = d[p2] - dorg;
    double tau = 0.5 * (lo + hi);
    int it = 0;
    for (; it < 200; ++it) {
        double s1 = 0.0, s2 = 0.0, q1 = 0.0, q2 = 0.0, ea = 0.0;
#pragma unroll 4
        for (int i0 = 0; i0 < K; i0 += G) {
            const int i = i0 + lane;
            if (i < K) {
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
        }
        double v5[5] = {s1, s2, q1, q2, ea};
        gsumN<G, 5>(v5);
        s1 = v5[0];
        s2 = v5[1];
        q1 = v5[2];
        q2 = v5[3];
        ea = v5[4];
        const double f = 1.0 + s1 + s2;
        // every lane holds the same sums: the exits below are warp-uniform (told to the compiler by the votes)
        if (G > 1 ? __all_sync(0xffffffffu, fabs(f) <= 8.0 * EPSM * (1.0 + ea)) : fabs(f) <= 8.0 * EPSM * (1.0 + ea)) break;
        if (f > 0.0) hi = tau; else lo = tau;
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
        if (!(tn > lo && tn < hi) || !isfinite(tn)) tn = 0.5 * (lo + hi);
        if (G > 1 ? __all_sync(0xffffffffu, tn == tau) : tn == tau) break;
        tau = tn;
    }
    *dorg_o = dorg;
    *tau_o = tau;
    if (lane == 0) { g_it[j] = it; g_cyc[j] = clock64() - c_start; }
}


__global__ void kern(const double* d, const double* z, int K, double rho) {
    extern __shared__ double sm[];
    double* sd = sm; double* sz = sm + K;
    for (int i = threadIdx.x; i < K; i += blockDim.x) { sd[i] = d[i]; sz[i] = z[i]; }
    __syncthreads();
    const int w = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x & 31;
    if (w < K) { double a, b; secular_root<32>(sd, sz, K, rho, w, lane, &a, &b); }
}
int main(int argc, char** argv) {
    int K = argc > 1 ? atoi(argv[1]) : 512;
    std::vector<double> d(K), z(K);
    srand(1);
    double s = 0; for (int i = 0; i < K; ++i) { d[i] = -1e5 * (double)i / K + 1e-3 * (rand() % 100); z[i] = 0.1 + (rand() % 1000) / 1000.0; s += z[i]*z[i]; }
    std::sort(d.begin(), d.end());
    for (auto& x : z) x /= sqrt(s);
    double *dd, *dz; cudaMalloc(&dd, K*8); cudaMalloc(&dz, K*8);
    cudaMemcpy(dd, d.data(), K*8, cudaMemcpyHostToDevice); cudaMemcpy(dz, z.data(), K*8, cudaMemcpyHostToDevice);
    for (int bs : {32, 256}) {
      int nb = (K + bs/32 - 1) / (bs/32);
      kern<<<nb, bs, 2*K*8>>>(dd, dz, K, 2e4);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a); kern<<<nb, bs, 2*K*8>>>(dd, dz, K, 2e4); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      std::vector<int> it(K); std::vector<long long> cy(K);
      cudaMemcpyFromSymbol(it.data(), g_it, K*4); cudaMemcpyFromSymbol(cy.data(), g_cyc, K*8);
      double si=0, sc=0; int mi=0; long long mc=0;
      for (int j=0;j<K;++j){si+=it[j]; sc+=cy[j]; mi=std::max(mi,it[j]); mc=std::max(mc,cy[j]);}
      printf("K=%d warps/CTA=%d: kernel %.1f us, iters avg %.2f max %d, cycles/root avg %.0f max %lld, cycles/iter %.0f\n", K, bs/32, ms*1e3, si/K, mi, sc/K, mc, sc/si);
    }
    return 0;
}
