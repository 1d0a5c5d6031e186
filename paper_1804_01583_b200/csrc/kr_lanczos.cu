// kr_lanczos.cu — fused one-HBM-pass Lanczos step on the matrix-free 7-point Dirichlet heat stencil.
//
// Paper: Lanczos (Alg. 3) with the projection and 3-vector memory of Alg. 4
// (Eq. 6). The operator is A = alpha * L_h (BASELINE.json configs,
// SURVEY §8(c) A1).
//
// B200 design. Alg. 3 as printed makes ~5 passes over n-vectors per step
// (A v, axpy, dot, axpy, norm, scale: ~104 n bytes). Here one step is ONE pass that reads u_i and
// u_{i-1} and writes u_{i+1} (24 n bytes, the minimum the three-term recurrence must move):
//   * vectors are stored unnormalised, v_i = s_i u_i (s_i = 1/||u_i|| carried as a scalar);
//   * lookahead: with alpha_i known, w = s_i A u_i - alpha_i s_i u_i - beta_{i-1} s_{i-1} u_{i-1}
//     (Alg. 3 lines 3-9 in one expression), and in the same pass
//       beta_i^2 = sum w^2 and  alpha_{i+1} = v_{i+1}^T A v_{i+1} = w^T A w / beta_i^2,
//     where -w^T A w = sum_axes c_a sum_{edges} (w_b - w_a)^2 (+ c_a w^2 on ghost edges) is a sum of
//     non-negative terms (summation by parts, Dirichlet ghosts = 0) — no cancellation;
//   * the (x+1), (y+1), (z+1) neighbours of w are recomputed on a one-cell forward ring, so u_i is
//     read with a depth-2 halo in-plane (TMA box (TX+4) x (TY+3) from x0-2: TMA needs 16-byte aligned
//     starts in x) and u_{i-1} with depth 1;
//   * 2.5D z-march: each CTA owns a TX x TY column tile and a z-chunk; TMA (cp.async.bulk.tensor.3d)
//     streams haloed planes of u_i and u_{i-1} into an S-stage shared-memory ring guarded by
//     mbarriers (zero fill of out-of-bounds boxes gives the Dirichlet ghosts for free); the vertical
//     neighbours live in registers; w planes go through a 2-plane shared buffer;
//   * per-CTA partial sums (sum w^2, sum D, box-row projections C w) are reduced in a fixed order
//     (no floating-point atomics) so results are bit-reproducible.
#include <cuda.h>
#include <float.h>

#include "kr_internal.h"

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "KR_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra KR_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int x, int y, int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

struct StepArgs {
    double* out;  // buffer receiving u_{i+1} (buffer plane 0 = ghost below the slab)
    int64_t pitch, plane;
    int32_t mx, my, mz, nz, zoff, zchunk;
    double cx, cy, cz;  // alpha / h_a^2
    const LzScalars* sc;
    int32_t step;       // i (1-based); 0 = init pass
    int32_t has_prev;
    int32_t write_out;
    int32_t nqp;
    double* partials;   // [nblk][nqp]
    int32_t nbox;
    BoxRow box[KR_MAX_BOX];
};

template <int TX, int TY>
struct Geo {
    static constexpr int NT = 256;
    static constexpr int CW = TX + 4, CH = TY + 3;  // u_i box: x0-2 .. x0+TX+1, y0-1 .. y0+TY+1
    static constexpr int PW = TX + 2, PH = TY + 1;  // u_{i-1} box: x0 .. x0+TX+1, y0 .. y0+TY
    static constexpr int WW = TX + 1, WH = TY + 1;  // w plane on the tile + forward ring
    static constexpr int CBYTES = CW * CH * 8, PBYTES = PW * PH * 8;
    static constexpr int POFF = ((CBYTES + 127) / 128) * 128;  // TMA destinations are 128-byte aligned
    static constexpr int STAGE = ((POFF + PBYTES + 127) / 128) * 128;
    static constexpr int WBYTES = ((2 * WW * WH * 8 + 127) / 128) * 128;
    static constexpr int NTC = TX * TY;             // tile cells
    static constexpr int NCELL = NTC + TX + TY;     // + right column + top row (no corner)
    static constexpr int NSLOT = (NCELL + NT - 1) / NT;
    static constexpr int NTSLOT = (NTC + NT - 1) / NT;
};

template <int TX, int TY, int S>
constexpr size_t step_smem_bytes() {
    return (size_t)S * Geo<TX, TY>::STAGE + Geo<TX, TY>::WBYTES + 8 * S + 16;
}

template <int TX, int TY, int S, bool INIT>
__global__ void __launch_bounds__(256) lz_step_kernel(const __grid_constant__ CUtensorMap tmC,
                                                      const __grid_constant__ CUtensorMap tmP, const StepArgs a) {
    using G = Geo<TX, TY>;
    const LzScalars* sc = a.sc;
    if (sc->done) return;  // breakdown happened earlier: uniform early exit

    extern __shared__ __align__(128) unsigned char smem[];
    double* Wb0 = reinterpret_cast<double*>(smem + S * G::STAGE);
    double* Wb1 = Wb0 + G::WW * G::WH;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S * G::STAGE + G::WBYTES);

    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int zc0 = blockIdx.z * a.zchunk;
    const int zc1 = min(zc0 + a.zchunk, a.nz);
    const int pfirst = zc0 - 1, plast = zc1 + 1;
    const int npl = plast - pfirst + 1;
    const uint32_t txb = G::CBYTES + (a.has_prev ? G::PBYTES : 0);

    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int p) {
        const int s = (p - pfirst) % S;
        unsigned char* st = smem + s * G::STAGE;
        mbar_expect_tx(&bar[s], txb);
        tma_load_3d(st, &tmC, x0 - 2, y0 - 1, p + 1, &bar[s]);  // x start must be 16-byte aligned
        if (a.has_prev) tma_load_3d(st + G::POFF, &tmP, x0, y0, p + 1, &bar[s]);
    };
    if (tid == 0) {
        const int np = npl < S ? npl : S;
        for (int p = pfirst; p < pfirst + np; ++p) issue(p);
    }

    // step scalars: w = sa*A u_i - sb*u_i - sp*u_{i-1}
    double sa = 1.0, sb = 0.0, sp = 0.0;
    if (!INIT) {
        const int i = a.step;
        sa = sc->s[i];
        sb = sc->alpha[i] * sc->s[i];
        sp = (i > 1) ? sc->beta[i - 1] * sc->s[i - 1] : 0.0;
    }
    const double cx = a.cx, cy = a.cy, cz = a.cz;
    const double diag = 2.0 * (cx + cy + cz);

    int lx[G::NSLOT], ly[G::NSLOT];
    bool act[G::NSLOT], ing[G::NSLOT];
    uint32_t bm[G::NSLOT];
#pragma unroll
    for (int m = 0; m < G::NSLOT; ++m) {
        const int idx = tid + m * G::NT;
        int x, y;
        if (idx < G::NTC) {
            x = idx % TX;
            y = idx / TX;
        } else if (idx < G::NTC + TY) {
            x = TX;
            y = idx - G::NTC;
        } else {
            x = idx - G::NTC - TY;
            y = TY;
        }
        act[m] = idx < G::NCELL;
        lx[m] = x;
        ly[m] = y;
        const int gx = x0 + x, gy = y0 + y;
        ing[m] = act[m] && gx < a.mx && gy < a.my;
        uint32_t b = 0;
        for (int r = 0; r < a.nbox; ++r)
            if (gx >= a.box[r].lo[0] && gx < a.box[r].hi[0] && gy >= a.box[r].lo[1] && gy < a.box[r].hi[1])
                b |= 1u << r;
        bm[m] = b;
    }

    double up[G::NSLOT], uc[G::NSLOT], wp[G::NSLOT], wc[G::NSLOT];
    mbar_wait(&bar[0], 0);
    mbar_wait(&bar[1 % S], 0);
    {
        const double* C0 = reinterpret_cast<const double*>(smem + 0 * G::STAGE);
        const double* C1 = reinterpret_cast<const double*>(smem + (1 % S) * G::STAGE);
#pragma unroll
        for (int m = 0; m < G::NSLOT; ++m) {
            const int o = (ly[m] + 1) * G::CW + lx[m] + 2;
            up[m] = act[m] ? C0[o] : 0.0;
            uc[m] = act[m] ? C1[o] : 0.0;
            wp[m] = 0.0;
        }
    }

    double acc_ww = 0.0, acc_d = 0.0;
    double acc_b[KR_MAX_BOX];
#pragma unroll
    for (int r = 0; r < KR_MAX_BOX; ++r) acc_b[r] = 0.0;

    for (int q = zc0; q <= zc1; ++q) {
        const int pn = q + 1;
        {
            const int u = pn - pfirst;
            mbar_wait(&bar[u % S], (u / S) & 1);
        }
        const unsigned char* stq = smem + ((q - pfirst) % S) * G::STAGE;
        const double* Cq = reinterpret_cast<const double*>(stq);
        const double* Pq = reinterpret_cast<const double*>(stq + G::POFF);
        const double* Cn = reinterpret_cast<const double*>(smem + ((pn - pfirst) % S) * G::STAGE);
        const int gz = a.zoff + q;
        const bool zin = gz < a.mz;
        double* Wq = (q & 1) ? Wb1 : Wb0;
#pragma unroll
        for (int m = 0; m < G::NSLOT; ++m) {
            if (!act[m]) continue;
            const int x = lx[m], y = ly[m];
            const double un = Cn[(y + 1) * G::CW + x + 2];
            double w;
            if (INIT) {
                w = uc[m];
            } else {
                const double sx = Cq[(y + 1) * G::CW + x + 1] + Cq[(y + 1) * G::CW + x + 3];
                const double sy = Cq[y * G::CW + x + 2] + Cq[(y + 2) * G::CW + x + 2];
                const double sz = up[m] + un;
                const double Au = cx * sx + cy * sy + cz * sz - diag * uc[m];
                w = sa * Au - sb * uc[m];
                if (a.has_prev) w -= sp * Pq[y * G::PW + x];
            }
            if (!(ing[m] && zin)) w = 0.0;
            Wq[y * G::WW + x] = w;
            wc[m] = w;
            up[m] = uc[m];
            uc[m] = un;
        }
        if (q > zc0) {
            const double* Wp = (q & 1) ? Wb0 : Wb1;
            const int gzp = gz - 1;
            double* orow = a.out + (int64_t)q * a.plane;  // buffer plane of local plane q-1
#pragma unroll
            for (int m = 0; m < G::NTSLOT; ++m) {
                const int idx = tid + m * G::NT;
                if (idx >= G::NTC) continue;
                const int x = lx[m], y = ly[m];
                const double w0 = wp[m];
                const double dx = Wp[y * G::WW + x + 1] - w0;
                const double dy = Wp[(y + 1) * G::WW + x] - w0;
                const double dz = wc[m] - w0;
                double D = cx * dx * dx + cy * dy * dy + cz * dz * dz;
                if (x0 + x == 0) D += cx * w0 * w0;
                if (y0 + y == 0) D += cy * w0 * w0;
                if (gzp == 0) D += cz * w0 * w0;
                acc_ww += w0 * w0;
                acc_d += D;
                if (bm[m]) {
#pragma unroll
                    for (int r = 0; r < KR_MAX_BOX; ++r)
                        if (r < a.nbox && ((bm[m] >> r) & 1u) && gzp >= a.box[r].lo[2] && gzp < a.box[r].hi[2])
                            acc_b[r] += w0;
                }
                if (!INIT && a.write_out && ing[m]) orow[(int64_t)(y0 + y) * a.pitch + (x0 + x)] = w0;
            }
        }
#pragma unroll
        for (int m = 0; m < G::NSLOT; ++m) wp[m] = wc[m];
        __syncthreads();
        if (tid == 0) {
            if (q == zc0 && pfirst + S <= plast) issue(pfirst + S);
            if (q + S <= plast) issue(q + S);
        }
    }

    // fixed-order block reduction of (sum w^2, sum D, box rows)
    __shared__ double red[8][2 + KR_MAX_BOX];
    const int lane = tid & 31, wid = tid >> 5;
    auto wsum = [&](double v) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        return v;
    };
    double v0 = wsum(acc_ww), v1 = wsum(acc_d);
    if (lane == 0) {
        red[wid][0] = v0;
        red[wid][1] = v1;
    }
#pragma unroll
    for (int r = 0; r < KR_MAX_BOX; ++r) {
        if (r < a.nbox) {
            double v = wsum(acc_b[r]);
            if (lane == 0) red[wid][2 + r] = v;
        }
    }
    __syncthreads();
    if (tid < a.nqp) {
        double s = 0.0;
        for (int w = 0; w < 8; ++w) s += red[w][tid];
        const int64_t blk = blockIdx.x + (int64_t)gridDim.x * (blockIdx.y + (int64_t)gridDim.y * blockIdx.z);
        a.partials[blk * a.nqp + tid] = s;
    }
}

// Local reduction of the per-CTA partials of one slab, plus sparse output rows gathered from the
// freshly written vector. rankvec[0] = sum w^2, [1] = sum D, [2+r] = C_r w.
__global__ void __launch_bounds__(256) lz_local_reduce(const double* partials, int64_t nblk, int nqp,
                                                       const int32_t* box_slot, const double* box_val, int nbox,
                                                       int n_out,
                                                       const DVec* outs, SlabInfo si, int buf, int gather,
                                                       int64_t mx, int64_t my, int64_t pitch,
                                                       const LzScalars* sc, double* rankvec) {
    if (sc->done) return;
    __shared__ double red[256];
    __shared__ double res[2 + KR_MAX_OUT];
    const int tid = threadIdx.x;
    for (int r = tid; r < 2 + n_out; r += 256) res[r] = 0.0;
    __syncthreads();
    auto block_sum = [&](double v) -> double {
        red[tid] = v;
        __syncthreads();
        for (int o = 128; o > 0; o >>= 1) {
            if (tid < o) red[tid] += red[tid + o];
            __syncthreads();
        }
        double r = red[0];
        __syncthreads();
        return r;
    };
    for (int qi = 0; qi < nqp; ++qi) {
        double v = 0.0;
        for (int64_t b = tid; b < nblk; b += 256) v += partials[b * nqp + qi];
        double s = block_sum(v);
        if (tid == 0) {
            if (qi < 2)
                res[qi] = s;
            else
                res[2 + box_slot[qi - 2]] = s * box_val[qi - 2];
        }
    }
    if (gather) {
        const double* u = si.u[buf];
        const int64_t plane = my * pitch;
        for (int r = 0; r < n_out; ++r) {
            const DVec o = outs[r];
            if (o.kind != KR_VEC_SPARSE) continue;
            double v = 0.0;
            for (int64_t e = tid; e < o.nnz; e += 256) {
                const int64_t idx = o.idx[e];
                const int64_t z = idx / (mx * my), rem = idx - z * mx * my;
                const int64_t y = rem / mx, x = rem - y * mx;
                if (z >= si.z0 && z < si.z1) v += o.val[e] * u[(z - si.z0 + 1) * plane + y * pitch + x];
            }
            double s = block_sum(v);
            if (tid == 0) res[2 + r] = s;
        }
    }
    __syncthreads();
    for (int r = tid; r < 2 + n_out; r += 256) rankvec[r] = res[r];
}

// Scalar update after the (global) reduction: fixed-order sum over the R rank/slab vectors, then
// beta_i, alpha_{i+1}, s_{i+1}, H and P entries, breakdown test.
__global__ void lz_finalize(const double* rankvec, int R, int nq, int n_out, int step, int k, LzScalars* sc,
                            double* H, double* P, double* beta0_out, double* hnext_out, int32_t* keff_out) {
    if (threadIdx.x != 0 || sc->done) return;
    double S[2 + KR_MAX_OUT];
    for (int q = 0; q < nq; ++q) S[q] = 0.0;
    for (int r = 0; r < R; ++r)
        for (int q = 0; q < nq; ++q) S[q] += rankvec[(int64_t)r * nq + q];
    const double Sww = S[0], SD = S[1];
    if (step == 0) {
        const double b0 = sqrt(Sww);
        *beta0_out = b0;
        sc->beta0 = b0;
        if (!(b0 > 0.0) || !isfinite(b0)) {
            sc->status = (b0 == 0.0) ? KR_EZERO : KR_ENONFINITE;
            sc->done = 1;
            sc->k_eff = 0;
            *keff_out = 0;
            return;
        }
        sc->s[1] = 1.0 / b0;
        const double a1 = -SD / Sww;
        sc->alpha[1] = a1;
        sc->hmax = fabs(a1);
        H[0] = a1;
        for (int r = 0; r < n_out; ++r) P[(int64_t)r * k + 0] = sc->s[1] * S[2 + r];
        sc->k_eff = 1;
        *keff_out = 1;
        return;
    }
    const int i = step;
    const double b = sqrt(Sww);
    if (!isfinite(b)) {
        sc->status = KR_ENONFINITE;
        sc->done = 1;
        return;
    }
    sc->beta[i] = b;
    H[(int64_t)i * k + (i - 1)] = b;  // h_{i+1,i}: row i of the (k+1) x k Hessenberg
    if (b == 0.0 || b <= 16.0 * DBL_EPSILON * sc->hmax || i == k) {
        sc->done = 1;
        sc->k_eff = i;
        sc->h_next = b;
        *keff_out = i;
        *hnext_out = b;
        return;
    }
    H[(int64_t)(i - 1) * k + i] = b;
    sc->s[i + 1] = 1.0 / b;
    const double an = -SD / Sww;
    sc->alpha[i + 1] = an;
    H[(int64_t)i * k + i] = an;
    for (int r = 0; r < n_out; ++r) P[(int64_t)r * k + i] = sc->s[i + 1] * S[2 + r];
    sc->hmax = fmax(sc->hmax, fmax(b, fabs(an)));
    sc->k_eff = i + 1;
    *keff_out = i + 1;
}

__global__ void lz_reset(LzScalars* sc) {
    if (threadIdx.x == 0) {
        sc->done = 0;
        sc->k_eff = 0;
        sc->status = 0;
        sc->hmax = 0.0;
        sc->h_next = 0.0;
        sc->beta0 = 0.0;
    }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        KR_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) KR_THROW(KR_ECUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

void encode(CUtensorMap* tm, double* base, int64_t mx, int64_t my, int64_t nplanes, int64_t pitch, int bx, int by) {
    cuuint64_t dims[3] = {(cuuint64_t)mx, (cuuint64_t)my, (cuuint64_t)nplanes};
    cuuint64_t strides[2] = {(cuuint64_t)(pitch * 8), (cuuint64_t)(pitch * my * 8)};
    cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = get_encode()(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) KR_THROW(KR_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
}

constexpr int kS = 4;

}  // namespace

size_t kr_lz_step_smem(int TX, int TY) {
    if (TX == 64 && TY == 8) return step_smem_bytes<64, 8, kS>();
    if (TX == 32 && TY == 8) return step_smem_bytes<32, 8, kS>();
    if (TX == 64 && TY == 16) return step_smem_bytes<64, 16, kS>();
    return 0;
}

void kr_lz_encode_maps(kr_handle* h) {
    for (auto& sl : h->slabs)
        for (int b = 0; b < 3; ++b) {
            encode(&sl.tmC[b], sl.u[b], h->mx, h->my, sl.nz + 3, h->pitch, h->TX + 4, h->TY + 3);
            encode(&sl.tmP[b], sl.u[b], h->mx, h->my, sl.nz + 3, h->pitch, h->TX + 2, h->TY + 1);
        }
}

template <int TX, int TY, bool INIT>
static void set_smem_attr() {
    KR_CUDA(cudaFuncSetAttribute(lz_step_kernel<TX, TY, kS, INIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)step_smem_bytes<TX, TY, kS>()));
}

template <int TX, int TY>
static int occupancy_t() {
    set_smem_attr<TX, TY, false>();
    set_smem_attr<TX, TY, true>();
    int nb = 0;
    KR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, lz_step_kernel<TX, TY, kS, false>, 256,
                                                          step_smem_bytes<TX, TY, kS>()));
    return nb;
}

int kr_lz_occupancy(int TX, int TY) {
    if (TX == 64 && TY == 8) return occupancy_t<64, 8>();
    if (TX == 32 && TY == 8) return occupancy_t<32, 8>();
    if (TX == 64 && TY == 16) return occupancy_t<64, 16>();
    return 1;
}

void kr_lz_prepare(kr_handle* h) { (void)kr_lz_occupancy(h->TX, h->TY); }

template <int TX, int TY>
static void step_launch_t(kr_handle* h, Slab& sl, LzScalars* sc, int cur, int prev, int nxt, int step, bool init,
                          bool write) {
    StepArgs a{};
    a.out = sl.u[nxt];
    a.pitch = h->pitch;
    a.plane = h->pitch * h->my;
    a.mx = (int)h->mx;
    a.my = (int)h->my;
    a.mz = (int)h->mz;
    a.nz = (int)sl.nz;
    a.zoff = (int)sl.z0;
    a.zchunk = sl.zchunk;
    a.cx = h->cx;
    a.cy = h->cy;
    a.cz = h->cz;
    a.sc = sc;
    a.step = step;
    a.has_prev = (!init && step > 1) ? 1 : 0;
    a.write_out = write ? 1 : 0;
    a.nqp = h->nqp;
    a.partials = sl.partials;
    a.nbox = (int)h->boxes.size();
    for (int r = 0; r < a.nbox; ++r) a.box[r] = h->boxes[r];
    const size_t smem = step_smem_bytes<TX, TY, kS>();
    const CUtensorMap& tc = sl.tmC[cur];
    const CUtensorMap& tp = sl.tmP[prev < 0 ? cur : prev];
    if (init) {
        lz_step_kernel<TX, TY, kS, true><<<sl.grid, 256, smem, h->stream>>>(tc, tp, a);
    } else {
        lz_step_kernel<TX, TY, kS, false><<<sl.grid, 256, smem, h->stream>>>(tc, tp, a);
    }
    KR_CUDA(cudaGetLastError());
    h->launches++;
}

static void step_launch(kr_handle* h, Slab& sl, LzScalars* sc, int cur, int prev, int nxt, int step, bool init,
                        bool write) {
    if (h->TX == 64 && h->TY == 8)
        step_launch_t<64, 8>(h, sl, sc, cur, prev, nxt, step, init, write);
    else if (h->TX == 32 && h->TY == 8)
        step_launch_t<32, 8>(h, sl, sc, cur, prev, nxt, step, init, write);
    else if (h->TX == 64 && h->TY == 16)
        step_launch_t<64, 16>(h, sl, sc, cur, prev, nxt, step, init, write);
    else
        KR_THROW(KR_EINVAL, "unsupported tile");
}

static void halo_exchange_virtual(kr_handle* h, int buf) {
    const size_t pb = (size_t)h->pitch * h->my * sizeof(double);
    const int S = (int)h->slabs.size();
    for (int s = 0; s < S; ++s) {
        Slab& me = h->slabs[s];
        if (s > 0) {  // my first two owned planes -> lower neighbour's upper halo
            Slab& lo = h->slabs[s - 1];
            KR_CUDA(cudaMemcpyAsync(lo.u[buf] + (lo.nz + 1) * h->pitch * h->my, me.u[buf] + 1 * h->pitch * h->my,
                                    2 * pb, cudaMemcpyDeviceToDevice, h->stream));
        }
        if (s + 1 < S) {  // my last owned plane -> upper neighbour's lower halo
            Slab& hi = h->slabs[s + 1];
            KR_CUDA(cudaMemcpyAsync(hi.u[buf], me.u[buf] + me.nz * h->pitch * h->my, pb, cudaMemcpyDeviceToDevice,
                                    h->stream));
        }
    }
}

// Reduction + scalar update for one step (all slabs of this process, then across ranks).
static void reduce_and_finalize(kr_handle* h, int dl, int buf, int step, bool gather) {
    const int S = (int)h->slabs.size();
    int32_t* box_slot = h->d_box_slot;
    LzScalars* sc = h->d_sc + dl;
    const int R = S * h->world;
    double* rv_local = h->d_rankvec + (size_t)h->rank * S * h->nq;
    for (int s = 0; s < S; ++s) {
        Slab& sl = h->slabs[s];
        SlabInfo si;
        si.z0 = sl.z0;
        si.z1 = sl.z1;
        si.nz = sl.nz;
        for (int b = 0; b < 3; ++b) si.u[b] = sl.u[b];
        lz_local_reduce<<<1, 256, 0, h->stream>>>(sl.partials, sl.nblk, h->nqp, box_slot, h->d_box_val,
                                                  (int)h->boxes.size(),
                                                  h->n_out, h->d_outs, si, buf, gather ? 1 : 0, h->mx, h->my,
                                                  h->pitch, sc, rv_local + (size_t)s * h->nq);
        KR_CUDA(cudaGetLastError());
        h->launches++;
    }
    if (h->world > 1) kr_nccl_allgather(h->comm, rv_local, h->d_rankvec, (size_t)S * h->nq, h->stream);
    const int k = h->k;
    lz_finalize<<<1, 32, 0, h->stream>>>(h->d_rankvec, R, h->nq, h->n_out, step, k, sc,
                                         h->d_H + (size_t)dl * (k + 1) * k, h->d_P + (size_t)dl * h->n_out * k,
                                         h->d_beta0 + dl, h->d_hnext + dl, h->d_keff + dl);
    KR_CUDA(cudaGetLastError());
    h->launches++;
}

// Enqueue the complete Lanczos run for local direction dl on h->stream (capturable).
void kr_lz_enqueue_direction(kr_handle* h, int dl, bool capture_events) {
    const int d = h->my_dirs[dl];
    LzScalars* sc = h->d_sc + dl;
    lz_reset<<<1, 32, 0, h->stream>>>(sc);
    KR_CUDA(cudaGetLastError());
    h->launches++;
    // u_1 = v_d, materialised on every slab including halo planes (analytic: no exchange needed)
    for (auto& sl : h->slabs) {
        kr_fill_grid(h->stream, sl.u[0], h->mx, h->my, h->pitch, sl.nz + 3, sl.z0 - 1, h->mz, h->dirs_h[d],
                     &h->launches);
    }
    // init pass: beta0, alpha_1, P_{.,1}
    for (auto& sl : h->slabs) step_launch(h, sl, sc, 0, -1, 0, 0, true, false);
    reduce_and_finalize(h, dl, 0, 0, true);
    const int k = h->k;
    int evi = 0;
    for (int i = 1; i <= k; ++i) {
        const int cur = (i - 1) % 3, prev = (i >= 2) ? (i - 2) % 3 : -1, nxt = i % 3;
        const bool write = i < k;
        if (capture_events && dl == 0) KR_CUDA(cudaEventRecordWithFlags(h->ev[evi], h->stream, cudaEventRecordExternal));
        for (auto& sl : h->slabs) step_launch(h, sl, sc, cur, prev, nxt, i, false, write);
        if (capture_events && dl == 0) KR_CUDA(cudaEventRecordWithFlags(h->ev[evi + 1], h->stream, cudaEventRecordExternal));
        evi += 2;
        if (write) {
            if (h->slabs.size() > 1) halo_exchange_virtual(h, nxt);
            if (h->world > 1) kr_nccl_halo(h->comm, h, nxt, h->stream);
        }
        reduce_and_finalize(h, dl, nxt, i, write);
    }
}
