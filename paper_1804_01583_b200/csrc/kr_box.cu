// kr_box.cu — per-step safety check over a box initial set.
// The LP of Fig. 2(c) with initial constraints z_lo <= z <= z_hi and ONE output
// half-space per row has the closed-form optimum  max/min_z sum_d c_d z_d = sum_d max/min(c_d z_lo_d,
// c_d z_hi_d)  — interval arithmetic on the basis-matrix entries. The first violating step (first-hit,
// PAPER.md:411-414, 918) and a witness z* are extracted on the device.
#include "kr_internal.h"

namespace {

struct DevCex {
    int32_t found;
    int64_t step;
    int32_t row;
    double y;
};

__global__ void box_bounds_kernel(const double* coeff, int64_t np1, int n_out, int n_dir, const double* zlo,
                                  const double* zhi, const int32_t* sense, const double* thr, double* lo, double* hi,
                                  int32_t* viol) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= np1 * n_out) return;
    const int r = (int)(e % n_out);
    const double* c = coeff + e * n_dir;
    double a = 0.0, b = 0.0;
    for (int d = 0; d < n_dir; ++d) {
        const double p = c[d] * zlo[d], q = c[d] * zhi[d];
        a += fmin(p, q);
        b += fmax(p, q);
    }
    lo[e] = a;
    hi[e] = b;
    const double th = thr[r];
    int v = 0;
    switch (sense[r]) {
        case KR_GE: v = b >= th; break;
        case KR_LE: v = a <= th; break;
        case KR_EQ: v = (a <= th) && (th <= b); break;
        default: v = 0;
    }
    viol[e] = v;
}

__global__ void first_violation_kernel(const double* coeff, const double* lo, const double* hi, const int32_t* viol,
                                       int64_t total, int n_out, int n_dir, const double* zlo, const double* zhi,
                                       const int32_t* sense, const double* thr, DevCex* cex, double* zw) {
    __shared__ int64_t best[256];
    int64_t b = total;
    for (int64_t e = threadIdx.x; e < total; e += blockDim.x)
        if (viol[e] && e < b) b = e;
    best[threadIdx.x] = b;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o && best[threadIdx.x + o] < best[threadIdx.x]) best[threadIdx.x] = best[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    const int64_t e = best[0];
    if (e >= total) {
        cex->found = 0;
        cex->step = -1;
        cex->row = -1;
        cex->y = 0.0;
        for (int d = 0; d < n_dir; ++d) zw[d] = 0.0;
        return;
    }
    const int r = (int)(e % n_out);
    const double* c = coeff + e * n_dir;
    const int s = sense[r];
    double lam = 0.0;
    if (s == KR_EQ) lam = (hi[e] == lo[e]) ? 0.0 : (thr[r] - lo[e]) / (hi[e] - lo[e]);
    double y = 0.0;
    for (int d = 0; d < n_dir; ++d) {
        const bool pos = c[d] >= 0.0;
        double z;
        if (s == KR_GE)
            z = pos ? zhi[d] : zlo[d];
        else if (s == KR_LE)
            z = pos ? zlo[d] : zhi[d];
        else
            z = pos ? zlo[d] + lam * (zhi[d] - zlo[d]) : zhi[d] - lam * (zhi[d] - zlo[d]);
        zw[d] = z;
        y += c[d] * z;
    }
    cex->found = 1;
    cex->step = e / n_out;
    cex->row = r;
    cex->y = y;
}

}  // namespace

size_t kr_box_cex_bytes() { return sizeof(DevCex); }

void kr_box_enqueue(kr_handle* h, const int32_t* d_sense, const double* d_thr) {
    const int64_t np1 = h->n_steps + 1;
    const int64_t total = np1 * h->cf_nout;
    double* lo = h->d_box;
    double* hi = h->d_box + total;
    int32_t* viol = reinterpret_cast<int32_t*>(h->d_box + 2 * total);
    box_bounds_kernel<<<(unsigned)((total + 255) / 256), 256, 0, h->stream>>>(
        h->d_cf, np1, h->cf_nout, h->cf_ndir, h->d_zlo, h->d_zhi, d_sense, d_thr, lo, hi, viol);
    KR_CUDA(cudaGetLastError());
    h->launches++;
    DevCex* cex = reinterpret_cast<DevCex*>(h->d_cex);
    double* zw = reinterpret_cast<double*>(reinterpret_cast<char*>(h->d_cex) + 64);
    first_violation_kernel<<<1, 256, 0, h->stream>>>(h->d_cf, lo, hi, viol, total, h->cf_nout, h->cf_ndir, h->d_zlo,
                                                     h->d_zhi, d_sense, d_thr, cex, zw);
    KR_CUDA(cudaGetLastError());
    h->launches++;
}

namespace {
// y_r = sum_d c[step][r][d] z_d (the basis matrix applied to one initial-space point)
__global__ void eval_outputs_kernel(const double* cf, int64_t step, int o, int nd, const double* z, double* y) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= o) return;
    const double* c = cf + (step * o + r) * (int64_t)nd;
    double s = 0.0;
    for (int d = 0; d < nd; ++d) s = fma(c[d], z[d], s);
    y[r] = s;
}
}  // namespace

void kr_eval_outputs(kr_handle* h, int64_t step, const double* z_h, double* y_h) {
    double* dz = nullptr;
    KR_CUDA(kr_dev_malloc(reinterpret_cast<void**>(&dz), ((size_t)h->cf_ndir + h->cf_nout) * sizeof(double)));
    double* dy = dz + h->cf_ndir;
    cudaError_t e = cudaMemcpyAsync(dz, z_h, (size_t)h->cf_ndir * 8, cudaMemcpyHostToDevice, h->stream);
    if (e == cudaSuccess) {
        eval_outputs_kernel<<<(h->cf_nout + 127) / 128, 128, 0, h->stream>>>(h->d_cf, step, h->cf_nout, h->cf_ndir, dz, dy);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(y_h, dy, (size_t)h->cf_nout * 8, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    kr_dev_free(dz);
    if (e != cudaSuccess) KR_THROW(KR_ECUDA, std::string("kr_eval_outputs: ") + cudaGetErrorString(e));
    h->launches++;
    h->h2d_bytes += (int64_t)h->cf_ndir * 8;
    h->d2h_bytes += (int64_t)h->cf_nout * 8;
}

