// dependent-latency microbenchmark (scripts only): cycles per dependent DFMA / DADD / MUFU.RCP64H / SHFL / FFMA
#include <cstdio>
__global__ void k(double* out, long long* cyc, double x0, int n) {
    double x = x0 + threadIdx.x * 1e-9, y = 1.0000001;
    float fx = (float)x0, fy = 1.0000001f;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, y, 1e-12);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) x = x + y;
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; }
    long long t3 = clock64();
    for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1);
    long long t4 = clock64();
    for (int i = 0; i < n; ++i) fx = fmaf(fx, fy, 1e-7f);
    long long t5 = clock64();
    for (int i = 0; i < n; ++i) x = x / (y + x * 1e-30);
    long long t6 = clock64();
    for (int i = 0; i < n; ++i) x = sqrt(x + 1.0);
    long long t7 = clock64();
    out[threadIdx.x] = x + fx;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; cyc[6] = t7 - t6; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64);
    const int n = 1000;
    for (int rep = 0; rep < 2; ++rep) {
        k<<<1, 32>>>(o, c, 1.5, n);
        long long h[7]; cudaMemcpy(h, c, 56, cudaMemcpyDeviceToHost);
        printf("cycles per dependent op: DFMA %.1f DADD %.1f RCP64H %.1f SHFL %.1f FFMA %.1f DDIV %.1f DSQRT %.1f\n", h[0] / (double)n, h[1] / (double)n,
               h[2] / (double)n, h[3] / (double)n, h[4] / (double)n, h[5] / (double)n, h[6] / (double)n);
    }
    return 0;
}
