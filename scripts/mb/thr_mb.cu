// fp64 throughput microbenchmark (scripts only): independent DFMA chains per thread
#include <cstdio>
template <int C>
__global__ void k(double* out, long long* cyc, int n) {
    double x[C];
    for (int c = 0; c < C; ++c) x[c] = 1.0 + threadIdx.x * 1e-9 + c * 1e-7;
    const double y = 0.999999;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int c = 0; c < C; ++c) x[c] = fma(x[c], y, 1e-9);
    }
    long long t1 = clock64();
    double a = 0; for (int c = 0; c < C; ++c) a += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = a;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <int C> void run(int warps, double* o, long long* c) {
    const int n = 2000;
    k<C><<<148, 32 * warps>>>(o, c, n); k<C><<<148, 32 * warps>>>(o, c, n); cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("chains=%d warps/SM=%2d: %.2f cycles per DFMA per warp -> %.1f DFMA lanes/clk/SM\n", C, warps, h / (double)n / C, 32.0 * warps * C * n / h);
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 148 * 1024 * 8); cudaMalloc(&c, 8);
    for (int w : {1, 4, 8, 16, 32}) { run<1>(w, o, c); run<8>(w, o, c); }
    return 0;
}
