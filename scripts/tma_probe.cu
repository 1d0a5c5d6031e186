// Standalone probe of 3D TMA tile loads of fp64 planes (box wider than the tensor, negative start
// coordinates, OOB zero fill) — the access pattern of lz_step_kernel. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tma_probe scripts/tma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int BX, int BY>
__global__ void probe(const __grid_constant__ CUtensorMap tm, int x, int y, int z, double* out, int variant) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(BX * BY * 8)
                     : "memory");
        if (variant == 0)
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                "%4}], [%5];" ::"r"(smem_u32(smem)),
                "l"(reinterpret_cast<uint64_t>(&tm)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(&bar))
                : "memory");
        else
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                "%4}], [%5];" ::"r"(smem_u32(smem)),
                "l"(reinterpret_cast<uint64_t>(&tm)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(&bar))
                : "memory");
    }
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            smem_u32(&bar)),
        "r"(0)
        : "memory");
    const double* s = reinterpret_cast<const double*>(smem);
    for (int i = threadIdx.x; i < BX * BY; i += blockDim.x) out[i] = s[i];
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int BX, int BY>
int run(int mx, int my, int mz, int pitch, int x, int y, int z, int variant, int dtype = 0, int promo = 1) {
    double* g;
    size_t n = (size_t)pitch * my * mz;
    cudaMalloc(&g, n * 8);
    double* h = (double*)malloc(n * 8);
    for (size_t i = 0; i < n; ++i) h[i] = (double)i;
    cudaMemcpy(g, h, n * 8, cudaMemcpyHostToDevice);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[3] = {(cuuint64_t)mx, (cuuint64_t)my, (cuuint64_t)mz};
    cuuint64_t strides[2] = {(cuuint64_t)pitch * 8, (cuuint64_t)pitch * my * 8};
    cuuint32_t box[3] = {BX, BY, 1}, es[3] = {1, 1, 1};
    CUtensorMapDataType dt = dtype == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : dtype == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_INT64;
    CUtensorMapL2promotion pr = promo ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE;
    CUresult r = ((EncFn)fp)(&tm, dt, 3, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    double* out;
    cudaMalloc(&out, BX * BY * 8);
    cudaMemset(out, 0xff, BX * BY * 8);
    probe<BX, BY><<<1, 128, BX * BY * 8 + 128>>>(tm, x, y, z, out, variant);
    cudaError_t e = cudaDeviceSynchronize();
    double* ho = (double*)malloc(BX * BY * 8);
    cudaMemcpy(ho, out, BX * BY * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int j = 0; j < BY; ++j)
        for (int i = 0; i < BX; ++i) {
            int gx = x + i, gy = y + j;
            double want = (gx >= 0 && gx < mx && gy >= 0 && gy < my && z >= 0 && z < mz)
                              ? (double)((size_t)z * pitch * my + (size_t)gy * pitch + gx)
                              : 0.0;
            if (ho[j * BX + i] != want) ++bad;
        }
    printf("BX=%d BY=%d m=(%d,%d,%d) pitch=%d at (%d,%d,%d) variant=%d dtype=%d promo=%d: encode=%d launch=%s mismatches=%d\n", BX, BY,
           mx, my, mz, pitch, x, y, z, variant, dtype, promo, (int)r, cudaGetErrorString(e), bad);
    cudaFree(g);
    cudaFree(out);
    free(h);
    free(ho);
    return e != cudaSuccess;
}

int main(int argc, char** argv) {
    int variant = argc > 1 ? atoi(argv[1]) : 0;
    int which = argc > 2 ? atoi(argv[2]) : 0;
    int dtype = argc > 3 ? atoi(argv[3]) : 0;
    int promo = argc > 4 ? atoi(argv[4]) : 1;
    if (which == 10) return run<68, 11>(100, 100, 20, 100, -1, 5, 3, variant, dtype, promo);
    if (which == 11) return run<68, 11>(100, 100, 20, 100, 40, 5, 3, variant, dtype, promo);
    if (which == 12) return run<68, 11>(100, 100, 20, 100, 10, -1, 3, variant, dtype, promo);
    if (which == 13) return run<64, 8>(100, 100, 20, 100, 40, 5, 3, variant, dtype, promo);
    if (which == 14) return run<16, 8>(100, 100, 20, 100, 90, 5, 3, variant, dtype, promo);
    if (which == 15) return run<16, 8>(100, 100, 20, 100, 10, 5, 30, variant, dtype, promo);
    if (which == 0) return run<68, 11>(100, 100, 20, 100, -1, -1, 3, variant);
    if (which == 1) return run<68, 11>(40, 40, 43, 40, -1, -1, 0, variant);
    if (which == 2) return run<36, 11>(40, 40, 43, 40, 31, 7, 5, variant);
    if (which == 3) return run<66, 9>(1000, 50, 5, 1000, 64, 8, 2, variant);
    return 0;
}
