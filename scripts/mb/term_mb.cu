// term-loop microbenchmark (scripts only): sum_i w_i / (d_i - tau) and its derivative over K terms, 32 lanes,
// several reciprocal flavours and unroll depths; cycles per term per warp
#include <cstdio>
__device__ __forceinline__ double frcp_mufu(double x) {
    double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0); r = fma(r, e, r); e = fma(-x, r, 1.0); return fma(r, e, r);
}
__device__ __forceinline__ double frcp_bits(double x) {
    const double ax = fabs(x);
    double r = __longlong_as_double(0x7FDE6238DA3C2118LL - __double_as_longlong(ax));
#pragma unroll
    for (int k = 0; k < 5; ++k) { const double e = fma(-ax, r, 1.0); r = fma(r, e, r); }
    return copysign(r, x);
}
__device__ __forceinline__ double frcp_f32(double x) {
    double r = (double)__frcp_rn((float)x);
    double e = fma(-x, r, 1.0); r = fma(r, e, r); e = fma(-x, r, 1.0); return fma(r, e, r);
}
template <int V, int U>
__global__ void kern(const double* d, const double* w, int K, double tau, double* out, long long* cyc) {
    extern __shared__ double sm[];
    double* sd = sm; double* sw = sm + K;
    for (int i = threadIdx.x; i < K; i += blockDim.x) { sd[i] = d[i]; sw[i] = w[i]; }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    long long t0 = clock64();
    double s[U], q[U];
    for (int u = 0; u < U; ++u) s[u] = q[u] = 0.0;
    for (int rep = 0; rep < 10; ++rep) {
        const double tr = tau + rep * 1e-9;
        for (int i0 = lane; i0 < K; i0 += 32 * U) {
            double dv[U], wv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {  // branch-free: out-of-range terms read entry 0 with weight 0
                const int i = i0 + 32 * u;
                const bool ok = i < K;
                dv[u] = sd[ok ? i : 0];
                wv[u] = ok ? sw[ok ? i : 0] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const double den = dv[u] - tr;
                const double r = V == 0 ? frcp_mufu(den) : (V == 1 ? frcp_bits(den) : (V == 2 ? frcp_f32(den) : 1.0 / den));
                const double t = wv[u] * r;
                s[u] += t; q[u] = fma(t, r, q[u]);
            }
        }
    }
    long long t1 = clock64();
    double a = 0; for (int u = 0; u < U; ++u) a += s[u] + q[u];
    out[blockIdx.x * blockDim.x + threadIdx.x] = a;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <int V, int U> void run(const char* name, double* dd, double* dw, int K, int warps, double* o, long long* c) {
    kern<V, U><<<148, 32 * warps, 2 * K * 8>>>(dd, dw, K, 0.5, o, c);
    kern<V, U><<<148, 32 * warps, 2 * K * 8>>>(dd, dw, K, 0.5, o, c);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-6s U=%d warps/SM=%2d K=%d: %.1f cycles per term per lane\n", name, U, warps, K, h / 10.0 / ((K + 31) / 32));
}
int main() {
    const int K = 544;
    double hd[K], hw[K];
    for (int i = 0; i < K; ++i) { hd[i] = -1.0 * i - 0.25; hw[i] = 1e-3 * (1 + i % 7); }
    double *dd, *dw, *o; long long* c;
    cudaMalloc(&dd, K * 8); cudaMalloc(&dw, K * 8); cudaMalloc(&o, 148 * 1024 * 8); cudaMalloc(&c, 8);
    cudaMemcpy(dd, hd, K * 8, cudaMemcpyHostToDevice); cudaMemcpy(dw, hw, K * 8, cudaMemcpyHostToDevice);
    for (int warps : {1, 8}) {
        run<0, 1>("mufu", dd, dw, K, warps, o, c); run<0, 2>("mufu", dd, dw, K, warps, o, c); run<0, 4>("mufu", dd, dw, K, warps, o, c); run<0, 8>("mufu", dd, dw, K, warps, o, c);
        run<1, 1>("bits", dd, dw, K, warps, o, c); run<1, 4>("bits", dd, dw, K, warps, o, c);
        run<2, 1>("f32", dd, dw, K, warps, o, c); run<2, 4>("f32", dd, dw, K, warps, o, c);
        run<3, 1>("div", dd, dw, K, warps, o, c); run<3, 4>("div", dd, dw, K, warps, o, c);
    }
    return 0;
}
