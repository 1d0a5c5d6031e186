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
//     where -w^T A w = sum_c d_c w_c^2 - 2 sum_axes c_a sum_{interior edges} w_a w_b (d_c the cell's diagonal of -A;
//     the product form, whose rounding is of the order of the oracle's own v^T (A v));
//   * the (x+1), (y+1), (z+1) neighbours of w are recomputed on a one-cell forward ring, so u_i is
//     read with a depth-2 halo in-plane (TMA box (TX+4) x (TY+3) from x0-2: TMA needs 16-byte aligned
//     starts in x) and u_{i-1} with depth 1;
//   * 2.5D z-march: each CTA owns a TX x TY column tile and a z-chunk; TMA (cp.async.bulk.tensor.3d)
//     streams haloed planes of u_i and u_{i-1} into an S-stage shared-memory ring guarded by
//     mbarriers (zero fill of out-of-bounds boxes gives the Dirichlet ghosts for free); the vertical
//     neighbours live in registers; w planes go through a 2-plane shared buffer;
//   * per-CTA partial sums (sum w^2, sum D, box-row projections C w) are reduced in a fixed order
//     (no floating-point atomics) so results are bit-reproducible.
#include <cooperative_groups.h>
#include <cuda.h>
#include <float.h>

#include <algorithm>
#include <type_traits>

#include "kr_internal.h"

namespace cg = cooperative_groups;

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
    // halo planes written straight into the neighbouring slabs' buffers (peer memory over NVLink, or the
    // sibling slab of a virtual-slab run): my owned planes 0, 1 -> lower neighbour planes lo_nz+1, +2;
    // my last owned plane -> upper neighbour plane 0. NULL = no such neighbour / message transport.
    double* rlo;
    double* rhi;
    int64_t rlo_plane0;  // offset (doubles) of the lower neighbour's plane lo_nz + 1
    int32_t rfence;      // 1: remote (other GPU) stores -> system-scope fence before the kernel ends
    int64_t pitch, plane;
    int32_t mx, my, mz, nz, zoff, zchunk;
    int32_t gx, gy, nitems;  // persistent work items: gx * gy tiles x ceil(nz / zchunk) chunks
    int32_t win;             // > 0: items ordered in windows of `win` tiles, z-chunk by z-chunk (lz_item_coords)
    int32_t zint;            // general faces: full interior tiles whose planes avoid both z faces take the Dirichlet march
    double cx, cy, cz;  // alpha / h_a^2
    // per-face boundary terms (x-, x+, y-, y+, z-, z+; kr_bc): ecor = diagonal correction of face cells
    // relative to the Dirichlet stencil ((bc != DIRICHLET) c_a - (bc == ROBIN) gamma); gq = coefficient of
    // w_c^2 in the edge form of -w^T A w for a face cell (DIRICHLET c_a, INSULATED 0, ROBIN gamma; the fill + init
    // kernel). Dirichlet: ecor = 0, gq = c. The step kernels' product form uses -ecor of face cells.
    double ecor[6], gq[6];
    const LzScalars* sc;
    int32_t step;       // i (1-based); 0 = init pass
    int32_t has_prev;
    int32_t write_out;
    int32_t nqp;
    double* partials;   // [nblk][nqp]
    int32_t nbox;
    uint32_t all_mask;  // box rows covering the whole grid: served by the plain sum of w
    BoxRow box[KR_MAX_BOX];
    // epilogue: the last CTA to finish reduces all partials in a fixed order (no float atomics)
    int32_t* counter;        // per-slab arrival counter (reset to 0 by the last CTA)
    double* rankvec;         // this slab's reduced vector [2 + n_out]
    const int32_t* box_slot; // output row of each box row
    const double* box_val;   // value of each box row
    const DVec* outs;        // sparse output rows are gathered from `gather_u`
    const double* gather_u;  // buffer holding the new vector (u_{i+1}, or u_1 for the init pass), or NULL
    int32_t n_out;
    int32_t fin;             // 1: this slab is the only contributor -> also do the scalar update
    int32_t k;
    double* H;
    double* P;
    double* beta0_out;
    double* hnext_out;
    int32_t* keff_out;
    LzScalars* scw;          // writable scalars (same as sc)
    DVec gen;                // init pass with an analytic generator (box / all): fill u_1 in the same pass
    // compact u_1 (Slab::CompactU1): TMA coordinates of the u_i ("C") / u_{i-1} ("P") maps are shifted by
    // these buffer-coordinate origins (0 for the full state buffers); work items start at tile (ix0, iy0)
    // and z-chunk iz0 (0 except for the init pass over the box region)
    int32_t shC[3], shP[3];
    int32_t ix0, iy0, iz0;
    // sparse output rows gathered from the compact u_1 (init pass) instead of gather_u
    const double* gc;
    int32_t gcx0, gcy0, gcp0, gcw, gch, gcd;
    int64_t gcpitch;
};

template <int NT>
__device__ void lz_epilogue(const StepArgs& a, const double* acc, double* red, int64_t plane_elems);

// tiles of >= 2048 cells run with 512 threads (one CTA per SM), smaller ones with 256 (two CTAs per SM)
template <int TX, int TY>
struct Geo {
    static constexpr int NT = (TX * TY >= 2048) ? 512 : 256;
    static constexpr int CW = TX + 4, CH = TY + 3;  // u_i box: x0-2 .. x0+TX+1, y0-1 .. y0+TY+1
    static constexpr int PW = TX + 2, PH = TY + 1;  // u_{i-1} box: x0 .. x0+TX+1, y0 .. y0+TY
    static constexpr int WW = TX + 1, WH = TY + 1;  // w plane on the tile + forward ring
    static constexpr int CBYTES = CW * CH * 8, PBYTES = PW * PH * 8;
    static constexpr int POFF = ((CBYTES + 127) / 128) * 128;  // TMA destinations are 128-byte aligned
    static constexpr int STAGE = ((POFF + PBYTES + 127) / 128) * 128;
    static constexpr int WBYTES = ((2 * WW * WH * 8 + 127) / 128) * 128;
    static constexpr int NTC = TX * TY;  // tile cells: NTC / NT per thread, always active
    static constexpr int TS = NTC / NT;
    static constexpr int NR = TX + TY;   // forward ring: right column + top row (no corner), tid < NR
    static_assert(NTC % NT == 0 && NR <= NT, "tile must map onto the CTA's threads");
};


// ================================================================================================
// Step kernel v2: 2 x 2 cells per thread.
// Lane l owns the x-pair (x0 + 2l, x0 + 2l + 1), warp w the row pair (y0 + 2w, y0 + 2w + 1). The centre values
// of a plane arrive as two 16-byte shared-memory loads; the in-pair x neighbours and the in-pair y neighbours are
// registers; only the outer x neighbours (x - 1, x + 2), the outer rows and u_{i-1} are loaded: 15 shared-memory
// instructions per 4 cells (v1, 4 cells strided in y per thread, every neighbour from shared memory: 36). The
// neighbour products of -w^T A w are kept per axis and combined with the edge coefficients once at the end of the
// kernel (acc2_wAw); with general faces the face cells' diagonal corrections go to one face accumulator.
// The forward ring (top row: warps 0-1, one cell per lane; right column: warp 2) is computed beside the tile.
// ================================================================================================
template <int TX, int TY, int R = 2>
struct Geo2 {
    static_assert(TX == 64, "v2 maps one x-pair per lane: TX = 64");
    static_assert(TY % R == 0 && TY / R >= 3, "the ring needs three warps");
    static constexpr int NT = 32 * TY / R;  // one warp per R rows
    static constexpr int CW = TX + 4, CH = TY + 3;  // u_i box: x0-2 .. x0+TX+1, y0-1 .. y0+TY+1
    static constexpr int PW = TX + 2, PH = TY + 1;  // u_{i-1} box: x0 .. x0+TX+1, y0 .. y0+TY
    static constexpr int WW = TX + 2, WH = TY + 1;  // w plane on the tile + forward ring, rows of 16-byte multiples
    static constexpr int CBYTES = CW * CH * 8, PBYTES = PW * PH * 8;
    static constexpr int POFF = ((CBYTES + 127) / 128) * 128;
    static constexpr int STAGE = ((POFF + PBYTES + 127) / 128) * 128;
    static constexpr int WBYTES = ((2 * WW * WH * 8 + 127) / 128) * 128;
};

template <int TX, int TY, int S>
constexpr size_t step2_smem_bytes() {
    return (size_t)S * Geo2<TX, TY>::STAGE + Geo2<TX, TY>::WBYTES + 8 * S + 16;
}

// The per-step values of the march (the rest of StepArgs is the same for every step of a run): the output buffer,
// the step's recurrence coefficients sa = s_i, sb = alpha_i s_i, sp = beta_{i-1} s_{i-1} (1, 0, 0 for the init pass)
struct StepDyn {
    double* out;
    double sa, sb, sp;
    int32_t has_prev, write_out;
};

struct Acc2 {
    double ww, sum;      // sum w^2, sum w
    double px, py, pz;   // sums of neighbour products w_c w_{c+e_a} over the interior edges per axis (coefficient c_a)
    double face;         // face cells: (d_c - diag) w_c^2, d_c the cell's diagonal of -A (Dirichlet: 0)
};

// -w^T A w = sum_c d_c w_c^2 - 2 sum_{interior edges} c_a w_a w_b = diag sum w^2 - 2 (cx px + cy py + cz pz) + face
__device__ __forceinline__ double acc2_wAw(const StepArgs& a, const Acc2& A) {
    return fma(2.0 * (a.cx + a.cy + a.cz), A.ww, fma(-2.0 * a.cx, A.px, fma(-2.0 * a.cy, A.py, fma(-2.0 * a.cz, A.pz, A.face))));
}

__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void st2(double* p, double a, double b) { *reinterpret_cast<double2*>(p) = make_double2(a, b); }

// R rows per thread: lane l owns the x-pair (x0 + 2l, +1) on the rows y0 + R w .. y0 + R w + R - 1 of warp w
// (cells c = 2 r + column). The in-pair x neighbours and the y neighbours inside the thread's rows are registers.
// BCM: 0 = Dirichlet everywhere; 1 = general faces, tile without x/y face cells (full, x0 > 0, y0 > 0): only the
// per-plane z-face terms; 2 = general faces, per-cell diagonal corrections (a tile at x0 = 0, y0 = 0 or ragged).
// -w^T A w is accumulated in the product form sum_c d_c w_c^2 - 2 sum_edges c_a w_a w_b (acc2_wAw): per cell the
// three forward-neighbour products (one FMA each, no differences), sum w^2, and for general faces the face cells'
// diagonal corrections; with Dirichlet faces no face code at all (edges to the zero ghosts drop out), so every
// full tile takes the unrolled march. The only per-plane branch is uniform: no z edge above the top plane.
// Box output rows are summed per warp (shuffle tree, fixed order) into wbox.
template <int TX, int TY, int R, int S, bool INIT, bool FULL, int BCM, bool HALO>
__device__ __forceinline__ void lz_march2(const CUtensorMap* tmC, const CUtensorMap* tmP, const StepArgs& a,
                                          const StepDyn& dyn, unsigned char* smem, double* Wb0, double* Wb1, uint64_t* bar, int x0, int y0,
                                          int zc0, int zc1, bool cta_box, Acc2& A, double (*wbox)[KR_MAX_BOX]) {
    using G = Geo2<TX, TY, R>;
    constexpr int CW = G::CW, PW = G::PW, WW = G::WW, NC = 2 * R;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int pfirst = zc0 - 1, plast = zc1 + 1;
    const bool has_prev = dyn.has_prev != 0;
    auto issue = [&](int p) {
        const int s = (p - pfirst) % S;
        unsigned char* st = smem + s * G::STAGE;
        const bool lp = has_prev && p > pfirst && p < plast;  // u_{i-1} is needed on planes zc0..zc1 only
        mbar_expect_tx(&bar[s], G::CBYTES + (lp ? G::PBYTES : 0));
        tma_load_3d(st, tmC, x0 - 2 - a.shC[0], y0 - 1 - a.shC[1], p + 1 - a.shC[2], &bar[s]);
        if (lp) tma_load_3d(st + G::POFF, tmP, x0 - a.shP[0], y0 - a.shP[1], p + 1 - a.shP[2], &bar[s]);
    };
    constexpr int ISSUER = G::NT - 32;  // lane 0 of the last warp (warps 0-2 carry the ring)
    if (tid == ISSUER) {
        const int np = min(plast - pfirst + 1, S);
        for (int p = pfirst; p < pfirst + np; ++p) issue(p);
    }
    const double sa = INIT ? 1.0 : dyn.sa, sb = INIT ? 0.0 : dyn.sb, sp = INIT ? 0.0 : dyn.sp;
    const double diag = 2.0 * (a.cx + a.cy + a.cz);
    const double scx = sa * a.cx, scy = sa * a.cy, scz = sa * a.cz;

    const int rx = 2 * lane, ry = R * wid;  // tile coordinates of the thread's first cell
    const int gx = x0 + rx, gy = y0 + ry;
    const int cb = (ry + 1) * CW + rx + 2, pb = ry * PW + rx, wb = ry * WW + rx;
    bool in[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) in[c] = FULL || (gx + (c & 1) < a.mx && gy + (c >> 1) < a.my);
    // face cells: low faces in any tile at x0 = 0 / y0 = 0; high faces only in ragged (not FULL) tiles
    double exy[NC];  // per-cell x/y diagonal corrections (BCM 2)
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        exy[c] = 0.0;
        if (BCM == 2) {
            const int cx_ = gx + (c & 1), cy_ = gy + (c >> 1);
            exy[c] = (cx_ == 0 ? a.ecor[0] : 0.0) + (cx_ == a.mx - 1 ? a.ecor[1] : 0.0) + (cy_ == 0 ? a.ecor[2] : 0.0) +
                     (cy_ == a.my - 1 ? a.ecor[3] : 0.0);
        }
    }
    uint32_t bm[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) bm[c] = 0u;
    if (cta_box)
        for (int c = 0; c < NC; ++c) {
            const int cx_ = gx + (c & 1), cy_ = gy + (c >> 1);
            for (int r = 0; r < a.nbox; ++r)
                if (!((a.all_mask >> r) & 1u) && cx_ >= a.box[r].lo[0] && cx_ < a.box[r].hi[0] && cy_ >= a.box[r].lo[1] &&
                    cy_ < a.box[r].hi[1])
                    bm[c] |= 1u << r;
        }
    // forward ring, one cell per lane on three warps (the barrier after each plane waits for the slowest warp,
    // so no warp takes more than one extra cell): the top row y0 + TY on warps 0 (x0 .. x0+31) and 1 (x0+32 ..
    // x0+63), the right column x0 + TX on warp 2 (lanes < TY)
    const bool ring = wid < 2 || (wid == 2 && lane < TY);
    int rcb = 0, rpb = 0, rwb = 0;
    bool rin = false;
    double rex = 0.0;
    if (ring) {
        const int rxx = wid < 2 ? 32 * wid + lane : TX, ryy = wid < 2 ? TY : lane;
        rcb = (ryy + 1) * CW + rxx + 2;
        rpb = ryy * PW + rxx;
        rwb = ryy * WW + rxx;
        const int grx = x0 + rxx, gry = y0 + ryy;
        rin = FULL || (grx < a.mx && gry < a.my);
        if (BCM)
            rex = (grx == 0 ? a.ecor[0] : 0.0) + (grx == a.mx - 1 ? a.ecor[1] : 0.0) + (gry == 0 ? a.ecor[2] : 0.0) +
                  (gry == a.my - 1 ? a.ecor[3] : 0.0);
    }
    double* optr = dyn.out + (int64_t)(zc0 + 1) * a.plane + (int64_t)gy * a.pitch + gx;

    // u of three consecutive planes (the thread's cells) in three register sets that take turns as u_{q-1}, u_q,
    // u_{q+1}; w of two consecutive planes in two sets (w_{q-1}, w_q): the interior loop is unrolled by six
    double U0[NC], U1[NC], U2[NC], WA[NC], WB[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) WA[c] = WB[c] = 0.0;
    double R0 = 0.0, R1 = 0.0, R2 = 0.0;
    mbar_wait(&bar[0], 0);
    mbar_wait(&bar[1 % S], 0);
    {
        const double* C0 = reinterpret_cast<const double*>(smem);
        const double* C1 = reinterpret_cast<const double*>(smem + (1 % S) * G::STAGE);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            double2 t = ld2(C0 + cb + r * CW);
            U0[2 * r] = t.x;
            U0[2 * r + 1] = t.y;
            t = ld2(C1 + cb + r * CW);
            U1[2 * r] = t.x;
            U1[2 * r + 1] = t.y;
        }
        if (ring) {
            R0 = C0[rcb];
            R1 = C1[rcb];
        }
    }
    int sq = 1 % S, sn = 2 % S;
    uint32_t ph = (2 / S) & 1;
    // one plane q: w_q on the tile (wc) and the ring (into the W buffer of q's parity), then the products of plane
    // q - 1 (wp = w_{q-1}; its x+2 / row+R neighbours from the W buffer written last iteration, its z+1 neighbour wc)
    constexpr bool UNROLL = FULL && BCM < 2;  // the first plane peeled, six planes per turn of the register rotation
    auto plane = [&](const double (&up)[2 * R], const double (&uc)[2 * R], double (&un)[2 * R], const double rp,
                     const double rc, double& rn, const double (&wp)[2 * R], double (&wc)[2 * R], const int q,
                     auto first) {
        constexpr bool FIRST = decltype(first)::value;  // q == zc0: w only, no products
        mbar_wait(&bar[sn], ph);
        const unsigned char* stq = smem + sq * G::STAGE;
        const double* Cq = reinterpret_cast<const double*>(stq);
        const double* Pq = reinterpret_cast<const double*>(stq + G::POFF);
        const double* Cn = reinterpret_cast<const double*>(smem + sn * G::STAGE);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const double2 t = ld2(Cn + cb + r * CW);
            un[2 * r] = t.x;
            un[2 * r + 1] = t.y;
        }
        const int gzq = a.zoff + q;
        double* Wq = (q & 1) ? Wb1 : Wb0;
        const double dgz = BCM ? diag - (gzq == 0 ? a.ecor[4] : 0.0) - (gzq == a.mz - 1 ? a.ecor[5] : 0.0) : diag;
        const double cf = fma(sa, dgz, sb);  // coefficient of u_i in w (this plane, no x/y face)
        if (INIT) {
#pragma unroll
            for (int c = 0; c < NC; ++c) wc[c] = uc[c];
        } else {
            const double2 ym = ld2(Cq + cb - CW), yp = ld2(Cq + cb + R * CW);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double xm = Cq[cb + r * CW - 1], xp = Cq[cb + r * CW + 2];
                double ydn0, ydn1, yup0, yup1;
                if (r == 0) {
                    ydn0 = ym.x;
                    ydn1 = ym.y;
                } else {
                    ydn0 = uc[2 * r - 2];
                    ydn1 = uc[2 * r - 1];
                }
                if (r == R - 1) {
                    yup0 = yp.x;
                    yup1 = yp.y;
                } else {
                    yup0 = uc[2 * r + 2];
                    yup1 = uc[2 * r + 3];
                }
                const int c0 = 2 * r, c1 = 2 * r + 1;
                const double cf0 = BCM == 2 ? fma(sa, dgz - exy[c0], sb) : cf;
                const double cf1 = BCM == 2 ? fma(sa, dgz - exy[c1], sb) : cf;
                // w = s_i (off-diagonal part of A u_i) - (s_i diag + alpha_i s_i) u_i - beta_{i-1} s_{i-1} u_{i-1}
                wc[c0] = fma(scx, xm + uc[c1], fma(scy, ydn0 + yup0, fma(scz, up[c0] + un[c0], -cf0 * uc[c0])));
                wc[c1] = fma(scx, uc[c0] + xp, fma(scy, ydn1 + yup1, fma(scz, up[c1] + un[c1], -cf1 * uc[c1])));
            }
            if (has_prev) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const double2 pv = ld2(Pq + pb + r * PW);
                    wc[2 * r] = fma(-sp, pv.x, wc[2 * r]);
                    wc[2 * r + 1] = fma(-sp, pv.y, wc[2 * r + 1]);
                }
            }
        }
        if (!FULL) {
#pragma unroll
            for (int c = 0; c < NC; ++c)
                if (!in[c]) wc[c] = 0.0;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) st2(Wq + wb + r * WW, wc[2 * r], wc[2 * r + 1]);
        if (ring) {
            rn = Cn[rcb];
            double r0 = rc;
            if (!INIT) {
                const double c0 = BCM ? fma(sa, dgz - rex, sb) : cf;
                r0 = fma(scx, Cq[rcb - 1] + Cq[rcb + 1],
                         fma(scy, Cq[rcb - CW] + Cq[rcb + CW], fma(scz, rp + rn, -c0 * rc)));
                if (has_prev) r0 = fma(-sp, Pq[rpb], r0);
            }
            if (!FULL && !rin) r0 = 0.0;
            Wq[rwb] = r0;
        }
        if (!FIRST && (UNROLL || q > zc0)) {  // products of plane q - 1 (its x+2 / row+R neighbours: last iteration)
            const double* Wp = ((q & 1) ? Wb0 : Wb1) + wb;
            const int gzp = gzq - 1;
            const double2 yu = ld2(Wp + R * WW);
            // neighbour products over the forward edges: w beyond the grid (cells outside a ragged tile, ring
            // cells outside the grid) is stored as 0, so edges to the x / y ghosts drop out without face code
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double xr = Wp[r * WW + 2];
                const double yn0 = r == R - 1 ? yu.x : wp[2 * r + 2], yn1 = r == R - 1 ? yu.y : wp[2 * r + 3];
                A.px = fma(wp[2 * r], wp[2 * r + 1], A.px);
                A.px = fma(wp[2 * r + 1], xr, A.px);
                A.py = fma(wp[2 * r], yn0, A.py);
                A.py = fma(wp[2 * r + 1], yn1, A.py);
            }
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                A.ww = fma(wp[c], wp[c], A.ww);
                A.sum += wp[c];
            }
            const bool ztop = gzp == a.mz - 1;  // uniform: the z+1 neighbour is the ghost above the grid (its w is
            if (!ztop) {                        // not a state value): no edge
#pragma unroll
                for (int c = 0; c < NC; ++c) A.pz = fma(wp[c], wc[c], A.pz);
            }
            if (BCM) {  // face cells: (d_c - diag) w_c^2 = -(sum of the cell's face corrections ecor) w_c^2
                if (gzp == 0 || ztop) {  // uniform, rare
                    double s2 = 0.0;
#pragma unroll
                    for (int c = 0; c < NC; ++c) s2 = fma(wp[c], wp[c], s2);
                    const double ez = (gzp == 0 ? a.ecor[4] : 0.0) + (ztop ? a.ecor[5] : 0.0);
                    A.face = fma(-ez, s2, A.face);
                }
                if (BCM == 2) {
#pragma unroll
                    for (int c = 0; c < NC; ++c) A.face = fma(-exy[c] * wp[c], wp[c], A.face);
                }
            }
            const bool wr = !INIT && dyn.write_out;
            if (wr) {
#pragma unroll
                for (int r = 0; r < R; ++r)
                    if (FULL || (gx < a.mx && gy + r < a.my)) st2(optr + r * a.pitch, wp[2 * r], wp[2 * r + 1]);
            }
            if (cta_box) {  // box output rows meeting this tile and plane (uniform, rare)
                uint32_t zmask = 0;
                for (int r = 0; r < a.nbox; ++r)
                    if (gzp >= a.box[r].lo[2] && gzp < a.box[r].hi[2]) zmask |= 1u << r;
                for (int r = 0; r < a.nbox; ++r) {  // uniform loop: a warp tree per box row meeting this plane
                    if (!((zmask >> r) & 1u)) continue;
                    double v = 0.0;
#pragma unroll
                    for (int c = 0; c < NC; ++c)
                        if ((bm[c] >> r) & 1u) v += wp[c];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
                    if (lane == 0) wbox[wid][r] += v;
                }
            }
            // halo planes for the neighbours, stored where they will be read (uniform per plane, rare): owned
            // planes 0, 1 -> the lower neighbour, the last owned plane -> the upper neighbour
            const int qq = q - 1;
            if (HALO && wr && ((a.rlo && qq < 2) || (a.rhi && qq == a.nz - 1))) {
                const int64_t off = (optr - dyn.out) - (int64_t)(qq + 1) * a.plane;  // in-plane offset of cell 0
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if (!(FULL || (gx < a.mx && gy + r < a.my))) continue;
                    if (a.rlo && qq < 2)
                        st2(a.rlo + a.rlo_plane0 + (int64_t)qq * a.plane + off + r * a.pitch, wp[2 * r], wp[2 * r + 1]);
                    if (a.rhi && qq == a.nz - 1) st2(a.rhi + off + r * a.pitch, wp[2 * r], wp[2 * r + 1]);
                }
            }
            optr += a.plane;
        }
        __syncthreads();
        if (tid == ISSUER) {
            if (q == zc0 && pfirst + S <= plast) issue(pfirst + S);
            if (q + S <= plast) issue(q + S);
        }
        sq = sn;
        if (++sn == S) {
            sn = 0;
            ph ^= 1u;
        }
    };
    using F1 = std::integral_constant<bool, true>;
    using F0 = std::integral_constant<bool, false>;
    if (UNROLL) {  // the first plane peeled (no products), then six planes per turn of the register rotation
        plane(U0, U1, U2, R0, R1, R2, WA, WB, zc0, F1{});
        for (int q = zc0 + 1; q <= zc1;) {
            plane(U1, U2, U0, R1, R2, R0, WB, WA, q, F0{});
            if (++q > zc1) break;
            plane(U2, U0, U1, R2, R0, R1, WA, WB, q, F0{});
            if (++q > zc1) break;
            plane(U0, U1, U2, R0, R1, R2, WB, WA, q, F0{});
            if (++q > zc1) break;
            plane(U1, U2, U0, R1, R2, R0, WA, WB, q, F0{});
            if (++q > zc1) break;
            plane(U2, U0, U1, R2, R0, R1, WB, WA, q, F0{});
            if (++q > zc1) break;
            plane(U0, U1, U2, R0, R1, R2, WA, WB, q, F0{});
            if (++q > zc1) break;
        }
    } else {
#pragma unroll 1
        for (int q = zc0; q <= zc1; ++q) {
            plane(U0, U1, U2, R0, R1, R2, WA, WB, q, F0{});
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                U0[c] = U1[c];
                U1[c] = U2[c];
                WA[c] = WB[c];
            }
            R0 = R1;
            R1 = R2;
        }
    }
}

// Work item -> (x-tile, y-tile, z-chunk). win = 0: z-chunk-major (all tiles of chunk 0, then chunk 1, ...).
// win = W (the resident CTAs of the launch): the tiles in groups of W, and within a group the z-chunks one after
// the other, so chunk z + 1 of a tile column is dispatched W items (one wave of resident CTAs) after chunk z: it
// starts as chunk z ends, and the three u_i planes and one u_{i-1} plane the two chunks share are still in L2
// (z-chunk-major order re-reads them from DRAM one pass over all tiles later: ~2 % of a step's bytes at C5).
__device__ __forceinline__ void lz_item_coords(const StepArgs& a, int item, int& xt, int& yt, int& zt) {
    const int T = a.gx * a.gy;
    int tile;
    if (a.win > 0 && a.win < T) {
        const int Z = a.nitems / T;
        const int g = item / (a.win * Z), rem = item - g * a.win * Z;
        const int gw = min(a.win, T - g * a.win);  // tiles in this group (the last one may be smaller)
        zt = rem / gw;
        tile = g * a.win + (rem - zt * gw);
    } else {
        tile = item % T;
        zt = item / T;
    }
    xt = a.ix0 + tile % a.gx;
    yt = a.iy0 + tile / a.gx;
    zt += a.iz0;
}

// The work items (x-tile, y-tile, z-chunk) of one step, dealt round-robin over the CTAs (fixed assignment,
// deterministic): the march of each item, accumulating the CTA's sums in A and wbox.
template <int TX, int TY, int S, bool INIT, bool BC, bool HALO, int R>
__device__ __forceinline__ void lz_items2(const CUtensorMap* tmC, const CUtensorMap* tmP, const StepArgs& a,
                                          const StepDyn& dy, unsigned char* smem, double* Wb0, double* Wb1,
                                          uint64_t* bar, Acc2& A, double (*wbox)[KR_MAX_BOX]) {
    const int tid = threadIdx.x;
    // Persistent CTAs: work items (x-tile, y-tile, z-chunk) dealt round-robin (fixed assignment, deterministic)
    for (int item = blockIdx.x; item < a.nitems; item += gridDim.x) {
        int xt, yt, zt;
        lz_item_coords(a, item, xt, yt, zt);
        const int x0 = xt * TX, y0 = yt * TY;
        const int zc0 = zt * a.zchunk;
        const int zc1 = min(zc0 + a.zchunk, a.nz);
        if (tid == 0) {
#pragma unroll
            for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        bool cta_box = false;
        for (int r = 0; r < a.nbox; ++r)
            if (!((a.all_mask >> r) & 1u) && a.box[r].lo[0] < x0 + TX && a.box[r].hi[0] > x0 &&
                a.box[r].lo[1] < y0 + TY && a.box[r].hi[1] > y0 && a.box[r].lo[2] < a.zoff + zc1 &&
                a.box[r].hi[2] > a.zoff + zc0)
                cta_box = true;
#define KR_M2(FULL_, BCM_) \
    lz_march2<TX, TY, R, S, INIT, FULL_, BCM_, HALO>(tmC, tmP, a, dy, smem, Wb0, Wb1, bar, x0, y0, zc0, zc1, cta_box, \
                                                            A, wbox)
        if (x0 + TX < a.mx && y0 + TY < a.my) {
            if constexpr (BC) {
                // a tile whose cells and forward ring (x0 + TX, y0 + TY) avoid the x / y faces and whose planes
                // zc0 .. zc1 (w of zc1 is formed too) avoid the z faces has the Dirichlet diagonal everywhere: the
                // plain march (no per-plane face logic; the paper model at 10^9: 15 of 17 z-chunks)
                if (x0 > 0 && y0 > 0 && x0 + TX + 1 < a.mx && y0 + TY + 1 < a.my && a.zint && a.zoff + zc0 >= 1 &&
                    a.zoff + zc1 <= a.mz - 2)
                    KR_M2(true, 0);
                else if (x0 > 0 && y0 > 0)
                    KR_M2(true, 1);
                else
                    KR_M2(true, 2);
            } else {
                KR_M2(true, 0);  // Dirichlet: no face terms, every full tile takes the unrolled march
            }
        } else {
            KR_M2(false, BC ? 2 : 0);
        }
#undef KR_M2
        __syncthreads();  // every issued plane was consumed: the barriers can be recycled for the next item
        if (tid == 0) {
#pragma unroll
            for (int s = 0; s < S; ++s)
                asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&bar[s])) : "memory");
        }
    }

}

template <int TX, int TY, int S, bool INIT, bool BC, bool HALO = false, int R = 2>
__global__ void __launch_bounds__(Geo2<TX, TY, R>::NT, (TY >= 32 && R == 2) ? 1 : 2)
    lz_step_kernel2(const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmP, const StepArgs a) {
    using G = Geo2<TX, TY, R>;
    if (a.sc->done) return;  // breakdown happened earlier: uniform early exit

    extern __shared__ __align__(128) unsigned char smem[];
    double* Wb0 = reinterpret_cast<double*>(smem + S * G::STAGE);
    double* Wb1 = Wb0 + G::WW * G::WH;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S * G::STAGE + G::WBYTES);

    const int tid = threadIdx.x;
    StepDyn dy{a.out, 1.0, 0.0, 0.0, a.has_prev, a.write_out};
    if (!INIT) {
        const LzScalars* sc = a.sc;
        const int i = a.step;
        dy.sa = sc->s[i];
        dy.sb = sc->alpha[i] * sc->s[i];
        dy.sp = (i > 1) ? sc->beta[i - 1] * sc->s[i - 1] : 0.0;
    }
    Acc2 A{0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    __shared__ double wbox[G::NT / 32][KR_MAX_BOX];  // per-warp box-row sums (lane 0 of each warp)
    if ((tid & 31) == 0)
        for (int r = 0; r < KR_MAX_BOX; ++r) wbox[tid >> 5][r] = 0.0;
    lz_items2<TX, TY, S, INIT, BC, HALO, R>(&tmC, &tmP, a, dy, smem, Wb0, Wb1, bar, A, wbox);

    if (HALO && a.rfence) __threadfence_system();  // peer-memory halo stores visible before the collective that follows
    __syncthreads();
    double acc[3 + KR_MAX_BOX];
    acc[0] = A.ww;
    acc[1] = acc2_wAw(a, A);  // -w^T A w
    acc[2] = A.sum;
#pragma unroll
    for (int r = 0; r < KR_MAX_BOX; ++r) acc[3 + r] = (tid & 31) == 0 ? wbox[tid >> 5][r] : 0.0;
    lz_epilogue<G::NT>(a, acc, reinterpret_cast<double*>(smem), a.plane);
}

// Scalar update after the (global) reduction: fixed-order sum over the R rank/slab vectors, then
// beta_i, alpha_{i+1}, s_{i+1}, H and P entries, breakdown test.
__device__ void lz_finalize_dev(const double* rankvec, int R, int nq, int n_out, int step, int k, LzScalars* sc,
                                double* H, double* P, double* beta0_out, double* hnext_out, int32_t* keff_out) {
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
        if (H) H[0] = a1;
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
    if (H) H[(int64_t)i * k + (i - 1)] = b;  // h_{i+1,i}: row i of the (k+1) x k Hessenberg (dense only for small k)
    if (b == 0.0 || b <= 16.0 * DBL_EPSILON * sc->hmax || i == k) {
        sc->done = 1;
        sc->k_eff = i;
        sc->h_next = b;
        *keff_out = i;
        *hnext_out = b;
        return;
    }
    if (H) H[(int64_t)(i - 1) * k + i] = b;
    sc->s[i + 1] = 1.0 / b;
    const double an = -SD / Sww;
    sc->alpha[i + 1] = an;
    if (H) H[(int64_t)i * k + i] = an;
    for (int r = 0; r < n_out; ++r) P[(int64_t)r * k + i] = sc->s[i + 1] * S[2 + r];
    sc->hmax = fmax(sc->hmax, fmax(b, fabs(an)));
    sc->k_eff = i + 1;
    *keff_out = i + 1;
}

__global__ void lz_finalize(const double* rankvec, int R, int nq, int n_out, int step, int k, LzScalars* sc,
                            double* H, double* P, double* beta0_out, double* hnext_out, int32_t* keff_out) {
    if (threadIdx.x != 0 || sc->done) return;
    lz_finalize_dev(rankvec, R, nq, n_out, step, k, sc, H, P, beta0_out, hnext_out, keff_out);
}

// Per-CTA partial sums, quantity-major [nqp][nblk]: [0] sum w^2, [1] sum D, [2 + r] box row r (all-grid
// rows take sum w). No fence or atomic: the CTA exits immediately; lz_reduce_kernel (next launch)
// reduces them in a fixed order.
template <int NT>
__device__ void lz_epilogue(const StepArgs& a, const double* acc, double* red, int64_t plane_elems) {
    (void)red;
    (void)plane_elems;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    __shared__ double wred[NT / 32][3 + KR_MAX_BOX];
#pragma unroll
    for (int r = 0; r < 3 + KR_MAX_BOX; ++r) {
        if (r < 3 + a.nbox) {
            double v = acc[r];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
            if (lane == 0) wred[wid][r] = v;
        }
    }
    __syncthreads();
    if (tid < a.nqp) {
        const int src = tid < 2 ? tid : (((a.all_mask >> (tid - 2)) & 1u) ? 2 : tid + 1);
        double s = 0.0;
        for (int w = 0; w < NT / 32; ++w) s += wred[w][src];
        const int64_t nblk = (int64_t)gridDim.x * gridDim.y * gridDim.z;
        const int64_t blk = blockIdx.x + (int64_t)gridDim.x * (blockIdx.y + (int64_t)gridDim.y * blockIdx.z);
        a.partials[(int64_t)tid * nblk + blk] = s;
    }
}

// Fixed-order reduction of a slab's partials over G CTAs: CTA g sums the contiguous block range
// [g*seg, (g+1)*seg) (per-thread strided sums with nqp independent loads in flight, warp trees, warps in
// order) and stores its nqp sums; the last CTA to arrive (arrival counter, reset by it for the next graph
// replay) adds the G sums in CTA order, gathers the sparse output rows from the new vector, writes the
// slab's vector [2 + n_out] to rankvec and — for a single slab on a single rank — does the scalar update.
// Same result for every run (fixed segments and order; the counter only elects the CTA, no float atomics).
constexpr int RT = 512;
__global__ void __launch_bounds__(RT) lz_reduce_kernel(const StepArgs a, int64_t nblk) {
    if (a.sc->done) return;
    __shared__ double red[KR_MAX_BOX + 2][RT / 32];
    __shared__ double res[2 + KR_MAX_OUT];
    __shared__ int last;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int nqp = a.nqp;
    const int G = (int)gridDim.x;
    const int64_t seg = (nblk + G - 1) / G;
    const int64_t b0 = (int64_t)blockIdx.x * seg, b1 = b0 + seg < nblk ? b0 + seg : nblk;
    double v[2 + KR_MAX_BOX];
#pragma unroll
    for (int q = 0; q < 2 + KR_MAX_BOX; ++q) v[q] = 0.0;
    for (int64_t b = b0 + tid; b < b1; b += RT) {
#pragma unroll
        for (int q = 0; q < 2 + KR_MAX_BOX; ++q)
            if (q < nqp) v[q] += a.partials[(int64_t)q * nblk + b];
    }
#pragma unroll
    for (int q = 0; q < 2 + KR_MAX_BOX; ++q) {
        if (q < nqp) {
            double t = v[q];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
            if (lane == 0) red[q][wid] = t;
        }
    }
    __syncthreads();
    if (G > 1) {
        double* gsum = a.partials + (int64_t)nqp * nblk;  // [G][nqp] behind the per-CTA partials
        if (tid < nqp) {
            double s = 0.0;
            for (int w = 0; w < RT / 32; ++w) s += red[tid][w];
            gsum[(int64_t)blockIdx.x * nqp + tid] = s;
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) last = atomicAdd(a.counter, 1) == G - 1;
        __syncthreads();
        if (!last) return;
        __threadfence();
        if (tid == 0) *a.counter = 0;
        if (tid < nqp) {
            double s = 0.0;
            for (int g = 0; g < G; ++g) s += __ldcg(gsum + (int64_t)g * nqp + tid);
            red[tid][0] = s;
            for (int w = 1; w < RT / 32; ++w) red[tid][w] = 0.0;
        }
        __syncthreads();
    }
    for (int r = tid; r < 2 + a.n_out; r += RT) res[r] = 0.0;
    __syncthreads();
    if (tid < nqp) {
        double s = 0.0;
        for (int w = 0; w < RT / 32; ++w) s += red[tid][w];
        if (tid < 2)
            res[tid] = s;
        else
            res[2 + a.box_slot[tid - 2]] = s * a.box_val[tid - 2];
    }
    __syncthreads();
    if (a.gather_u || a.gc) {  // sparse output rows from the freshly written vector (owned planes)
        __shared__ double gred[RT / 32];
        const int64_t mxy = (int64_t)a.mx * a.my;
        for (int r = 0; r < a.n_out; ++r) {
            const DVec o = a.outs[r];
            if (o.kind != KR_VEC_SPARSE) continue;
            double t = 0.0;
            for (int64_t e = tid; e < o.nnz; e += RT) {
                const int64_t idx = o.idx[e];
                const int64_t z = idx / mxy, rem = idx - z * mxy;
                const int64_t y = rem / a.mx, x = rem - y * a.mx;
                const int64_t zl = z - a.zoff;
                if (zl < 0 || zl >= a.nz) continue;
                if (a.gc) {  // compact u_1: zero outside the stored region
                    const int64_t cx_ = x - a.gcx0, cy_ = y - a.gcy0, cp_ = zl + 1 - a.gcp0;
                    if (cx_ >= 0 && cx_ < a.gcw && cy_ >= 0 && cy_ < a.gch && cp_ >= 0 && cp_ < a.gcd)
                        t += o.val[e] * a.gc[(cp_ * a.gch + cy_) * a.gcpitch + cx_];
                } else {
                    t += o.val[e] * a.gather_u[(zl + 1) * a.plane + y * a.pitch + x];
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) t += __shfl_down_sync(0xffffffffu, t, off);
            if (lane == 0) gred[wid] = t;
            __syncthreads();
            if (tid == 0) {
                double s2 = 0.0;
                for (int w = 0; w < RT / 32; ++w) s2 += gred[w];
                res[2 + r] = s2;
            }
            __syncthreads();
        }
    }
    for (int r = tid; r < 2 + a.n_out; r += RT) a.rankvec[r] = res[r];
    __syncthreads();
    if (tid == 0 && a.fin)
        lz_finalize_dev(res, 1, 2 + a.n_out, a.n_out, a.step, a.k, a.scw, a.H, a.P, a.beta0_out, a.hnext_out,
                        a.keff_out);
}

// ---- persistent multi-step Lanczos (small grids) --------------------------------------------------------------
// Steps i0..i1 of Alg. 3 / 4 in ONE cooperative launch, for a single slab on a single rank whose three
// state vectors stay in the 126 MB L2 (10^6 cells: 24 MB): per step the same march as lz_step_kernel2 over the
// CTA's work items, its partial sums, one grid barrier, then EVERY CTA reduces all partials in the same fixed order
// and updates the scalars itself (identical values everywhere, so the breakdown / k test exits all CTAs at the
// same step and no second barrier is needed). Replaces a step launch + a reduce launch per step (~21 us at 10^6
// cells, latency-bound) by ~one barrier. The scalars (alpha, beta, s, P, H, k_eff, h_next, done) are written to
// global memory by every CTA with the same bits; hmax lives in shared memory (a CTA must not read another CTA's
// newer global hmax, which could flip its breakdown test).
struct MultiArgs {
    double* u[3];   // the slab's state buffers
    double* part;   // [2][nqp][gridDim.x] per-CTA partial sums, double-buffered by step parity
    int32_t i0, i1; // steps
    uint64_t* prof; // KR_MS_PROF=1: %globaltimer per CTA at step start / march end / after the grid barrier / step
                    // end for the first KR_MS_PROF_STEPS steps of the launch, [step][CTA][4]; else NULL
};

__device__ __forceinline__ uint64_t kr_globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
constexpr int KR_MS_PROF_STEPS = 8;

template <int TX, int TY, int S, bool BC, int R>
__global__ void __launch_bounds__(Geo2<TX, TY, R>::NT, (TY >= 32 && R == 2) ? 1 : 2)
    lz_multistep_kernel(const __grid_constant__ CUtensorMap tmC0, const __grid_constant__ CUtensorMap tmC1,
                        const __grid_constant__ CUtensorMap tmC2, const __grid_constant__ CUtensorMap tmP0,
                        const __grid_constant__ CUtensorMap tmP1, const __grid_constant__ CUtensorMap tmP2,
                        const StepArgs a, const MultiArgs m) {
    using G = Geo2<TX, TY, R>;
    constexpr int NWp = G::NT / 32;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(128) unsigned char smem[];
    double* Wb0 = reinterpret_cast<double*>(smem + S * G::STAGE);
    double* Wb1 = Wb0 + G::WW * G::WH;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S * G::STAGE + G::WBYTES);
    __shared__ double wbox[NWp][KR_MAX_BOX];
    __shared__ double wred[NWp][3 + KR_MAX_BOX];
    __shared__ double qsum[2 + KR_MAX_BOX];
    __shared__ double coef[3];
    __shared__ double hmax;
    __shared__ int done;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int nblk = (int)gridDim.x, nqp = a.nqp, k = a.k;
    LzScalars* sc = a.scw;
    if (tid == 0) {  // read before the first barrier: no CTA has written step i0's scalars yet
        const int i = m.i0;
        done = sc->done;
        hmax = sc->hmax;
        coef[0] = sc->s[i];
        coef[1] = sc->alpha[i] * sc->s[i];
        coef[2] = i > 1 ? sc->beta[i - 1] * sc->s[i - 1] : 0.0;
    }
    __syncthreads();
    for (int i = m.i0; i <= m.i1; ++i) {
        if (done) break;  // uniform over the grid
        uint64_t* pr = (m.prof && i - m.i0 < KR_MS_PROF_STEPS && tid == 0)
                           ? m.prof + ((size_t)(i - m.i0) * nblk + blockIdx.x) * 4 : nullptr;
        if (pr) pr[0] = kr_globaltimer();
        const int cur = (i - 1) % 3, nxt = i % 3, prev = i >= 2 ? (i - 2) % 3 : cur;
        const CUtensorMap* tc = cur == 0 ? &tmC0 : (cur == 1 ? &tmC1 : &tmC2);
        const CUtensorMap* tp = prev == 0 ? &tmP0 : (prev == 1 ? &tmP1 : &tmP2);
        const StepDyn dy{m.u[nxt], coef[0], coef[1], coef[2], i > 1 ? 1 : 0, i < k ? 1 : 0};
        Acc2 A{0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        if (lane == 0)
            for (int r = 0; r < KR_MAX_BOX; ++r) wbox[wid][r] = 0.0;
        lz_items2<TX, TY, S, false, BC, false, R>(tc, tp, a, dy, smem, Wb0, Wb1, bar, A, wbox);
        __syncthreads();
        // the CTA's sums (as lz_epilogue), into the partials of this step's parity
        {
            double acc[3 + KR_MAX_BOX];
            acc[0] = A.ww;
            acc[1] = acc2_wAw(a, A);  // -w^T A w
            acc[2] = A.sum;
#pragma unroll
            for (int r = 0; r < KR_MAX_BOX; ++r) acc[3 + r] = lane == 0 ? wbox[wid][r] : 0.0;
#pragma unroll
            for (int r = 0; r < 3 + KR_MAX_BOX; ++r) {
                if (r < 3 + a.nbox) {
                    double v = acc[r];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
                    if (lane == 0) wred[wid][r] = v;
                }
            }
        }
        __syncthreads();
        double* part = m.part + (size_t)(i & 1) * nqp * nblk;
        if (tid < nqp) {
            const int src = tid < 2 ? tid : (((a.all_mask >> (tid - 2)) & 1u) ? 2 : tid + 1);
            double s = 0.0;
            for (int w = 0; w < NWp; ++w) s += wred[w][src];
            part[(size_t)tid * nblk + blockIdx.x] = s;
        }
        // u_{i+1} was written by generic stores; the next step reads it through TMA (async proxy)
        asm volatile("fence.proxy.async.global;" ::: "memory");
        if (pr) pr[1] = kr_globaltimer();
        grid.sync();
        if (pr) pr[2] = kr_globaltimer();
        // all partials, fixed order (lane-strided sums, xor tree): the same bits in every CTA
        for (int q = wid; q < nqp; q += NWp) {
            // every partial of the lane in flight at once (one L2 round trip for grids up to 32 x 12 CTAs; the
            // round trips, not the adds, bound this), summed in a fixed order
            constexpr int U = 12;
            double vu[U];
            const double* pq = part + (size_t)q * nblk;
#pragma unroll
            for (int u = 0; u < U; ++u) vu[u] = lane + 32 * u < nblk ? __ldcg(pq + lane + 32 * u) : 0.0;
            for (int b = lane + 32 * U; b < nblk; b += 32) vu[U - 1] += __ldcg(pq + b);  // larger grids
#pragma unroll
            for (int w = 1; w < U; w *= 2)
#pragma unroll
                for (int u = 0; u + w < U; u += 2 * w) vu[u] += vu[u + w];
            double v = vu[0];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) qsum[q] = v;
        }
        __syncthreads();
        if (tid == 0) {
            // the scalar update of lz_finalize_dev for step i >= 1 (beta_i, alpha_{i+1}, s_{i+1}, P column, breakdown)
            const double Sww = qsum[0], SD = qsum[1];
            const double b = sqrt(Sww);
            if (!isfinite(b)) {
                sc->status = KR_ENONFINITE;
                sc->done = 1;
                done = 1;
            } else {
                sc->beta[i] = b;
                if (a.H) a.H[(int64_t)i * k + (i - 1)] = b;
                if (b == 0.0 || b <= 16.0 * DBL_EPSILON * hmax || i == k) {
                    sc->done = 1;
                    sc->k_eff = i;
                    sc->h_next = b;
                    *a.keff_out = i;
                    *a.hnext_out = b;
                    done = 1;
                } else {
                    if (a.H) a.H[(int64_t)(i - 1) * k + i] = b;
                    const double sn = 1.0 / b;
                    sc->s[i + 1] = sn;
                    const double an = -SD / Sww;
                    sc->alpha[i + 1] = an;
                    if (a.H) a.H[(int64_t)i * k + i] = an;
                    for (int r = 0; r < a.n_out; ++r) a.P[(int64_t)r * k + i] = 0.0;
                    for (int q = 2; q < nqp; ++q) a.P[(int64_t)a.box_slot[q - 2] * k + i] = sn * (qsum[q] * a.box_val[q - 2]);
                    hmax = fmax(hmax, fmax(b, fabs(an)));
                    sc->hmax = hmax;
                    sc->k_eff = i + 1;
                    *a.keff_out = i + 1;
                    coef[2] = b * coef[0];  // beta_i s_i
                    coef[0] = sn;
                    coef[1] = an * sn;
                }
            }
        }
        __syncthreads();
        if (pr) pr[3] = kr_globaltimer();
    }
}

// Init pass for an analytic generator (KR_VEC_BOX / KR_VEC_ALL): writes u_1 = v over the slab buffer
// (owned planes, plus the ghost/halo planes from the global description) and, in the same pass,
// accumulates ||v||^2, -v^T A v (summation-by-parts edge form) and the box-row projections C v (Alg. 4 lines 1-2,
// P:782-783). One 8n-byte write instead of a fill (8n write) followed by a read pass (8n).
// v = value * [x in X][y in Y][z in Z] with X, Y, Z the box ranges clipped to the grid (ALL = whole grid),
// so membership is precomputed per axis.
template <int TX, int TY>
__global__ void __launch_bounds__(Geo<TX, TY>::NT) lz_fillinit_kernel(const StepArgs a) {
    using G = Geo<TX, TY>;
    if (a.sc->done) return;
    double* red_s = nullptr;  // the epilogue needs no scratch
    constexpr int RS = G::NT / TX;
    const int tid = threadIdx.x;
    const double cx = a.cx, cy = a.cy, cz = a.cz;
    const DVec g = a.gen;
    const bool all = g.kind == KR_VEC_ALL;
    auto clip = [](int64_t v, int64_t lo, int64_t hi) { return (int)(v < lo ? lo : (v > hi ? hi : v)); };
    const int lx = all ? 0 : clip(g.lo[0], 0, a.mx), hx = all ? a.mx : clip(g.hi[0], 0, a.mx);
    const int ly = all ? 0 : clip(g.lo[1], 0, a.my), hy = all ? a.my : clip(g.hi[1], 0, a.my);
    const int lz = all ? 0 : clip(g.lo[2], 0, a.mz), hz = all ? a.mz : clip(g.hi[2], 0, a.mz);
    const double val = g.value;
    double acc[3 + KR_MAX_BOX];
#pragma unroll
    for (int r = 0; r < 3 + KR_MAX_BOX; ++r) acc[r] = 0.0;
    for (int item = blockIdx.x; item < a.nitems; item += gridDim.x) {
        const int xt = item % a.gx, yt = (item / a.gx) % a.gy, zt = item / (a.gx * a.gy);
        const int x0 = xt * TX, y0 = yt * TY;
        const int zc0 = zt * a.zchunk;
        const int zc1 = min(zc0 + a.zchunk, a.nz);
        {
            // Tiles none of whose cells (or +1 neighbours) touch the generator box hold zeros and add nothing
            // to the sums: plain 16-byte stores (the C5 start vector is 0.1% of the grid).
            const int qa = (zt == 0) ? -1 : zc0, qb = (zc1 == a.nz) ? a.nz + 2 : zc1;
            const bool tx_ = x0 < hx && x0 + TX > lx - 1, ty_ = y0 < hy && y0 + TY > ly - 1;
            const bool tz_ = a.zoff + qa < hz && a.zoff + qb - 1 >= lz - 1;
            if (!(tx_ && ty_ && tz_)) {
                static_assert(TX % 4 == 0, "zero-store map: 4 cells per store pair");
                for (int e = tid; e < (TX / 4) * TY; e += G::NT) {
                    const int xx = x0 + (e % (TX / 4)) * 4, yy = y0 + e / (TX / 4);
                    if (yy >= a.my) continue;
                    for (int q = qa; q < qb; ++q) {
                        double* row = a.out + (int64_t)(q + 1) * a.plane + (int64_t)yy * a.pitch;
                        if (xx + 3 < a.mx) {
                            reinterpret_cast<double2*>(row + xx)[0] = make_double2(0.0, 0.0);
                            reinterpret_cast<double2*>(row + xx)[1] = make_double2(0.0, 0.0);
                        } else {
                            for (int c = 0; c < 4; ++c)
                                if (xx + c < a.mx) row[xx + c] = 0.0;
                        }
                    }
                }
                continue;
            }
        }
        const int x = tid % TX, ty = tid / TX, gx = x0 + x;
        const bool fx0 = gx >= lx && gx < hx, fx1 = gx + 1 >= lx && gx + 1 < hx;
        // face terms of -v^T A v (gq = c_a on Dirichlet faces, 0 insulated, gamma Robin): low faces as ghost
        // terms, high faces replace the edge coefficient (the value beyond the grid is 0)
        const double gex = gx == 0 ? a.gq[0] : 0.0;
        const double kx = gx == a.mx - 1 ? a.gq[1] : cx;
        bool fy0[G::TS], fy1[G::TS], okc[G::TS];
        uint32_t bm[G::TS];
#pragma unroll
        for (int m = 0; m < G::TS; ++m) {
            const int gy = y0 + ty + m * RS;
            fy0[m] = gy >= ly && gy < hy;
            fy1[m] = gy + 1 >= ly && gy + 1 < hy;
            okc[m] = gx < a.mx && gy < a.my;
            uint32_t bb = 0;
            for (int r = 0; r < a.nbox; ++r)
                if (!((a.all_mask >> r) & 1u) && gx >= a.box[r].lo[0] && gx < a.box[r].hi[0] &&
                    gy >= a.box[r].lo[1] && gy < a.box[r].hi[1])
                    bb |= 1u << r;
            bm[m] = bb;
        }
        double* optr = a.out + (int64_t)(y0 + ty) * a.pitch + gx;
        const int64_t rowstep = (int64_t)RS * a.pitch;
        const int qa = (zt == 0) ? -1 : zc0;
        const int qb = (zc1 == a.nz) ? a.nz + 2 : zc1;  // exclusive
        for (int q = qa; q < qb; ++q) {
            const int gz = a.zoff + q;
            const bool own = q >= zc0 && q < zc1;
            const bool fz0 = gz >= lz && gz < hz, fz1 = gz + 1 >= lz && gz + 1 < hz;
            const double gez = gex + (gz == 0 ? a.gq[4] : 0.0);
            const double kz = gz == a.mz - 1 ? a.gq[5] : cz;
            uint32_t zmask = 0;
            if (own)
                for (int r = 0; r < a.nbox; ++r)
                    if (!((a.all_mask >> r) & 1u) && gz >= a.box[r].lo[2] && gz < a.box[r].hi[2]) zmask |= 1u << r;
            double* orow = optr + (int64_t)(q + 1) * a.plane;
#pragma unroll
            for (int m = 0; m < G::TS; ++m) {
                if (!okc[m]) continue;
                const double v = (fx0 && fy0[m] && fz0) ? val : 0.0;
                orow[m * rowstep] = v;
                if (!own) continue;
                const double dx = ((fx1 && fy0[m] && fz0) ? val : 0.0) - v;
                const double dy = ((fx0 && fy1[m] && fz0) ? val : 0.0) - v;
                const double dz = ((fx0 && fy0[m] && fz1) ? val : 0.0) - v;
                const int gy = y0 + ty + m * RS;
                const double ge = gez + (gy == 0 ? a.gq[2] : 0.0);
                const double ky = gy == a.my - 1 ? a.gq[3] : cy;
                const double v2 = v * v;
                acc[0] += v2;
                acc[1] = fma(kx, dx * dx, fma(ky, dy * dy, fma(kz, dz * dz, fma(ge, v2, acc[1]))));
                acc[2] += v;
                const uint32_t mk = bm[m] & zmask;
                if (mk) {
#pragma unroll
                    for (int r = 0; r < KR_MAX_BOX; ++r)
                        if ((mk >> r) & 1u) acc[3 + r] += v;
                }
            }
        }
    }
    lz_epilogue<G::NT>(a, acc, red_s, a.plane);
}

// Compact u_1 (Slab::CompactU1): the generator's value on the stored region (indicator of the box clipped
// to the grid; cells beyond the grid or the row length are 0, like the Dirichlet ghosts of the full maps).
__global__ void lz_fill_compact_kernel(double* g, int64_t x0, int64_t y0, int64_t p0, int64_t w, int64_t hh, int64_t d,
                                       int64_t pitch, int64_t zoff, int64_t mx, int64_t my, int64_t mz, DVec gen) {
    const int64_t tot = pitch * hh * d;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t cx = e % pitch, cy = (e / pitch) % hh, cp = e / (pitch * hh);
        const int64_t X = x0 + cx, Y = y0 + cy, Z = zoff + p0 + cp - 1;  // buffer plane p <-> z = zoff + p - 1
        bool in = cx < w && X < mx && Y < my && Z >= 0 && Z < mz;
        if (gen.kind == KR_VEC_BOX)
            in = in && X >= gen.lo[0] && X < gen.hi[0] && Y >= gen.lo[1] && Y < gen.hi[1] && Z >= gen.lo[2] &&
                 Z < gen.hi[2];
        g[e] = in ? gen.value : 0.0;
    }
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

template <int TX, int TY>
struct Stages {
#ifdef KR_STAGES
    static constexpr int S = KR_STAGES;
#else
    static constexpr int S = (TX * TY > 512) ? 4 : 5;
#endif
};

}  // namespace

size_t kr_lz_step_smem(int TX, int TY) {
    if (TX == 64 && TY == 16) return step2_smem_bytes<64, 16, Stages<64, 16>::S>();
    if (TX == 64 && TY == 8) return step2_smem_bytes<64, 8, Stages<64, 8>::S>();
    return 0;
}

void kr_lz_encode_maps(kr_handle* h) {
    for (auto& sl : h->slabs)
        for (int b = 0; b < 3; ++b) {
            encode(&sl.tmC[b], sl.u[b], h->mx, h->my, sl.nz + 3, h->pitch, h->TX + 4, h->TY + 3);
            encode(&sl.tmP[b], sl.u[b], h->mx, h->my, sl.nz + 3, h->pitch, h->TX + 2, h->TY + 1);
        }
}

// Compact u_1 for analytic generators (box / all-grid): the stored region is the generator box clipped
// to the slab's buffer planes, x start even (16-byte aligned TMA starts), at least one TMA box in x and y.
// Skipped (full fill + init pass instead) for sparse generators, for regions above max(1/8 of a state
// buffer, 8 MB) and with KR_NO_COMPACT=1.
void kr_lz_setup_compact(kr_handle* h) {
    const bool off = getenv("KR_NO_COMPACT") != nullptr;
    const int ndl = (int)h->my_dirs.size();
    auto clip = [](int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); };
    for (auto& sl : h->slabs) {
        sl.cu1.assign(ndl, Slab::CompactU1{});
        int64_t maxe = 0;
        for (int dl = 0; dl < ndl; ++dl) {
            Slab::CompactU1& c = sl.cu1[dl];
            const DVec& g = h->dirs_h[h->my_dirs[dl]];
            if (off || (g.kind != KR_VEC_BOX && g.kind != KR_VEC_ALL)) continue;
            const bool all = g.kind == KR_VEC_ALL;
            const int64_t lx = all ? 0 : clip(g.lo[0], 0, h->mx), hx = all ? h->mx : clip(g.hi[0], 0, h->mx);
            const int64_t ly = all ? 0 : clip(g.lo[1], 0, h->my), hy = all ? h->my : clip(g.hi[1], 0, h->my);
            const int64_t lz = all ? 0 : clip(g.lo[2], 0, h->mz), hz = all ? h->mz : clip(g.hi[2], 0, h->mz);
            // buffer plane p holds z = z0 + p - 1, p = 0 .. nz + 2
            const int64_t p_lo = std::max<int64_t>(lz, sl.z0 - 1) - sl.z0 + 1;
            const int64_t p_hi = std::min<int64_t>(hz, sl.z0 + sl.nz + 2) - sl.z0 + 1;
            const bool empty = hx <= lx || hy <= ly || p_hi <= p_lo;
            c.x0 = empty ? 0 : (lx & ~int64_t(1));
            c.y0 = empty ? 0 : ly;
            c.p0 = empty ? 0 : p_lo;
            c.w = std::max<int64_t>(empty ? 1 : hx - c.x0, h->TX + 4);
            c.h = std::max<int64_t>(empty ? 1 : hy - c.y0, h->TY + 3);
            c.d = empty ? 1 : p_hi - p_lo;
            // at least 64 rows and planes (where the slab has them): tensor maps of a few planes made the
            // out-of-bounds boxes slow (measured: a slab whose region was empty, d = 1, took 2x as long for
            // steps 1-2 as with the full u_1; d >= 64 restores the fast path); the extra cells hold zeros
            c.h = std::max(c.h, std::min<int64_t>(64, h->my));
            c.d = std::max(c.d, std::min<int64_t>(64, sl.nz + 3 - c.p0));
            c.pitch = (c.w + 1) & ~int64_t(1);
            const int64_t vol = c.pitch * c.h * c.d;
            if (vol * 8 > std::max<int64_t>((sl.nz + 3) * h->my * h->pitch, (int64_t)8 << 20)) continue;  // 1/8 of a buffer or 8 MB
            c.on = true;
            maxe = std::max(maxe, vol);
            // init-pass work items: tiles / z-chunks meeting the box dilated by one cell towards -x, -y, -z
            // (those cells' forward edges reach into the box), owned planes only
            const int64_t zq0 = std::max<int64_t>(0, lz - 1 - sl.z0), zq1 = std::min<int64_t>(sl.nz, hz - sl.z0);
            if (hx <= lx || hy <= ly || zq1 <= zq0) {
                c.nitems = 0;
                c.gx = c.gy = 0;
            } else {
                c.ix0 = (int32_t)(std::max<int64_t>(0, lx - 1) / h->TX);
                c.iy0 = (int32_t)(std::max<int64_t>(0, ly - 1) / h->TY);
                c.iz0 = (int32_t)(zq0 / sl.zchunk);
                c.gx = (int32_t)((hx - 1) / h->TX) - c.ix0 + 1;
                c.gy = (int32_t)((hy - 1) / h->TY) - c.iy0 + 1;
                const int64_t nch = (zq1 - 1) / sl.zchunk - c.iz0 + 1;
                c.nitems = (int64_t)c.gx * c.gy * nch;
            }
        }
        if (maxe == 0) continue;
        void* gp = nullptr;
        if (kr_dev_malloc(&gp, (size_t)maxe * 8) != cudaSuccess) KR_THROW(KR_ENOMEM, "compact u_1 buffer");
        h->extra_allocs.push_back(gp);  // freed with the handle
        sl.g1 = reinterpret_cast<double*>(gp);
        for (auto& c : sl.cu1) {
            if (!c.on) continue;
            encode(&c.tmC, sl.g1, c.w, c.h, c.d, c.pitch, h->TX + 4, h->TY + 3);
            encode(&c.tmP, sl.g1, c.w, c.h, c.d, c.pitch, h->TX + 2, h->TY + 1);
        }
    }
}

template <int TX, int TY, bool INIT, bool BC, bool HALO = false, int R = 2>
static void set_smem_attr2() {
    KR_CUDA(cudaFuncSetAttribute(lz_step_kernel2<TX, TY, Stages<TX, TY>::S, INIT, BC, HALO, R>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)step2_smem_bytes<TX, TY, Stages<TX, TY>::S>()));
}

template <int TX, int TY, int R>
static int occupancy_t() {
    set_smem_attr2<TX, TY, false, false, false, R>();
    set_smem_attr2<TX, TY, true, false, false, R>();
    set_smem_attr2<TX, TY, false, true, false, R>();
    set_smem_attr2<TX, TY, true, true, false, R>();
    set_smem_attr2<TX, TY, false, false, true, R>();
    set_smem_attr2<TX, TY, false, true, true, R>();
    int n1 = 0, n2 = 0;
    const size_t sm2 = step2_smem_bytes<TX, TY, Stages<TX, TY>::S>();
    KR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &n1, lz_step_kernel2<TX, TY, Stages<TX, TY>::S, false, false, false, R>, Geo2<TX, TY, R>::NT, sm2));
    KR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &n2, lz_step_kernel2<TX, TY, Stages<TX, TY>::S, false, true, false, R>, Geo2<TX, TY, R>::NT, sm2));
    return n1 < n2 ? n1 : n2;
}

int kr_lz_occupancy(int TX, int TY) {
    if (TX == 64 && TY == 16) return occupancy_t<64, 16, 2>();
    if (TX == 64 && TY == 8) return occupancy_t<64, 8, 2>();
    return 1;
}

void kr_lz_prepare(kr_handle* h) { (void)kr_lz_occupancy(h->TX, h->TY); }

// cmode: 0 = full state buffers; 1 = u_i is the compact u_1 (init pass / step 1); 2 = u_{i-1} is (step 2)
static StepArgs make_args(kr_handle* h, Slab& sl, int dl, int nxt, int step, bool init, bool write, int gather_buf,
                          int cmode = 0) {
    StepArgs a{};
    LzScalars* sc = h->d_sc + dl;
    const int k = h->k;
    a.out = sl.u[nxt];
    a.pitch = h->pitch;
    a.plane = h->pitch * h->my;
    a.mx = (int)h->mx;
    a.my = (int)h->my;
    a.mz = (int)h->mz;
    a.nz = (int)sl.nz;
    a.zoff = (int)sl.z0;
    a.zchunk = sl.zchunk;
    a.win = sl.win;
    static const bool no_zint = getenv("KR_NO_ZINT") != nullptr;  // A/B: the general-face march on every interior tile
    a.zint = no_zint ? 0 : 1;
    a.gx = sl.gx;
    a.gy = sl.gy;
    a.nitems = (int)sl.nitems;
    a.cx = h->cx;
    a.cy = h->cy;
    a.cz = h->cz;
    {
        const double c[3] = {h->cx, h->cy, h->cz};
        for (int f = 0; f < 6; ++f) {
            const double ca = c[f / 2];
            const int bc = h->bc[f];
            a.ecor[f] = (bc != KR_BC_DIRICHLET ? ca : 0.0) - (bc == KR_BC_ROBIN ? h->gamma[f] : 0.0);
            a.gq[f] = bc == KR_BC_DIRICHLET ? ca : (bc == KR_BC_ROBIN ? h->gamma[f] : 0.0);
        }
    }
    a.sc = sc;
    a.scw = sc;
    a.step = step;
    a.has_prev = (!init && step > 1) ? 1 : 0;
    a.write_out = write ? 1 : 0;
    a.rlo = a.rhi = nullptr;
    a.rlo_plane0 = 0;
    a.rfence = 0;
    if (write && !init && h->halo_inkernel) {
        a.rlo = sl.peer_lo[nxt];
        a.rhi = sl.peer_hi[nxt];
        a.rlo_plane0 = (sl.peer_lo_nz + 1) * (int64_t)h->pitch * h->my;
        a.rfence = h->p2p ? 1 : 0;
    }
    a.nqp = h->nqp;
    a.partials = sl.partials;
    a.nbox = (int)h->boxes.size();
    a.all_mask = 0;
    for (int r = 0; r < a.nbox; ++r) {
        a.box[r] = h->boxes[r];
        const BoxRow& b = h->boxes[r];
        if (b.lo[0] <= 0 && b.lo[1] <= 0 && b.lo[2] <= 0 && b.hi[0] >= h->mx && b.hi[1] >= h->my && b.hi[2] >= h->mz)
            a.all_mask |= 1u << r;
    }
    a.counter = sl.counter;
    const int S = (int)h->slabs.size();
    const int sidx = (int)(&sl - &h->slabs[0]);
    a.rankvec = h->d_rankvec + ((size_t)kr_zrank(h) * S + sidx) * h->nq;
    a.box_slot = h->d_box_slot;
    a.box_val = h->d_box_val;
    a.outs = h->d_outs;
    bool has_sparse = false;
    for (const DVec& o : h->outs_h) has_sparse |= o.kind == KR_VEC_SPARSE;
    a.gather_u = (gather_buf >= 0 && has_sparse) ? sl.u[gather_buf] : nullptr;
    a.n_out = h->n_out;
    a.fin = (S == 1 && kr_zworld(h) == 1) ? 1 : 0;
    a.k = k;
    a.H = h->d_H ? h->d_H + (size_t)dl * (k + 1) * k : nullptr;
    a.P = h->d_P + (size_t)dl * h->n_out * k;
    a.beta0_out = h->d_beta0 + dl;
    a.hnext_out = h->d_hnext + dl;
    a.keff_out = h->d_keff + dl;
    if (cmode) {
        const Slab::CompactU1& c = sl.cu1[dl];
        int32_t* sh = cmode == 1 ? a.shC : a.shP;
        sh[0] = (int32_t)c.x0;
        sh[1] = (int32_t)c.y0;
        sh[2] = (int32_t)c.p0;
        if (cmode == 1 && init) {  // the init pass only visits the tiles around the box
            a.ix0 = c.ix0;
            a.iy0 = c.iy0;
            a.iz0 = c.iz0;
            a.gx = c.gx;
            a.gy = c.gy;
            a.nitems = (int)c.nitems;
            if (a.gather_u) {
                a.gather_u = nullptr;
                a.gc = sl.g1;
                a.gcx0 = (int32_t)c.x0;
                a.gcy0 = (int32_t)c.y0;
                a.gcp0 = (int32_t)c.p0;
                a.gcw = (int32_t)c.w;
                a.gch = (int32_t)c.h;
                a.gcd = (int32_t)c.d;
                a.gcpitch = c.pitch;
            }
        }
    }
    return a;
}

template <int TX, int TY, int S, int R>
static void launch_step2(kr_handle* h, dim3 grid, size_t smem2, const CUtensorMap& tc, const CUtensorMap& tp,
                         const StepArgs& a, bool init, bool halo) {
    constexpr int NT2 = Geo2<TX, TY, R>::NT;
    if (h->gen_bc) {
        if (init)
            lz_step_kernel2<TX, TY, S, true, true, false, R><<<grid, NT2, smem2, h->stream>>>(tc, tp, a);
        else if (halo)
            lz_step_kernel2<TX, TY, S, false, true, true, R><<<grid, NT2, smem2, h->stream>>>(tc, tp, a);
        else
            lz_step_kernel2<TX, TY, S, false, true, false, R><<<grid, NT2, smem2, h->stream>>>(tc, tp, a);
    } else {
        if (init)
            lz_step_kernel2<TX, TY, S, true, false, false, R><<<grid, NT2, smem2, h->stream>>>(tc, tp, a);
        else if (halo)
            lz_step_kernel2<TX, TY, S, false, false, true, R><<<grid, NT2, smem2, h->stream>>>(tc, tp, a);
        else
            lz_step_kernel2<TX, TY, S, false, false, false, R><<<grid, NT2, smem2, h->stream>>>(tc, tp, a);
    }
}

template <int TX, int TY>
static void step_launch_t(kr_handle* h, Slab& sl, int dl, int cur, int prev, int nxt, int step, bool init,
                          bool write, bool fillinit, int cmode) {
    if (fillinit) {
        StepArgs a = make_args(h, sl, dl, cur, 0, true, false, cur);
        a.gen = h->dirs_h[h->my_dirs[dl]];
        lz_fillinit_kernel<TX, TY><<<sl.grid, Geo<TX, TY>::NT, 0, h->stream>>>(a);
    } else {
        StepArgs a = make_args(h, sl, dl, nxt, step, init, write, init ? cur : (write ? nxt : -1), cmode);
        const CUtensorMap& tc = cmode == 1 ? sl.cu1[dl].tmC : sl.tmC[cur];
        const CUtensorMap& tp = cmode == 2 ? sl.cu1[dl].tmP : sl.tmP[prev < 0 ? cur : prev];
        const dim3 grid = (cmode == 1 && init) ? dim3((unsigned)std::max<int64_t>(1, sl.cu1[dl].nitems), 1, 1) : sl.grid;
        constexpr int S = Stages<TX, TY>::S;
        const bool halo = a.rlo || a.rhi;  // this slab writes halo planes into a neighbour's buffer
        const size_t smem2 = step2_smem_bytes<TX, TY, S>();
        // two rows per thread (2 x 2 cells); four rows (2 x 4 cells, 128 threads) measured slower: C5 3.79-3.84 vs
        // 3.73 ms per step, C4 0.267 vs 0.251 ms (fewer warps to hide the shared-memory and TMA latencies)
        launch_step2<TX, TY, S, 2>(h, grid, smem2, tc, tp, a, init, halo);
    }
    KR_CUDA(cudaGetLastError());
    h->launches++;
}

// CTAs of the slab reduction: ~512 per-CTA partials each, at most one per 64 partials (the [G][nqp] sums
// live in the ngrp * nqp doubles behind the partials) and at most 148.
static int kr_reduce_ctas(int64_t nblk) {
    const int64_t ngrp = (nblk + 63) / 64;
    int64_t g = (nblk + 511) / 512;
    g = std::min<int64_t>(std::min<int64_t>(g, 148), ngrp);
    return (int)std::max<int64_t>(1, g);
}

// The slab reduction (+ scalar update when fin) after a step / init launch on slab sl.
static void reduce_launch(kr_handle* h, Slab& sl, int dl, int nxt, int step, bool init, bool write, int gather_buf,
                          int cmode = 0) {
    StepArgs a = make_args(h, sl, dl, nxt, step, init, write, gather_buf, cmode);
    // partial-sum slots = CTAs of the step launch (the compact init pass runs on the box's tiles only)
    const int64_t nblk = (cmode == 1 && init) ? std::max<int64_t>(1, sl.cu1[dl].nitems) : sl.nblk;
    lz_reduce_kernel<<<kr_reduce_ctas(nblk), RT, 0, h->stream>>>(a, nblk);
    KR_CUDA(cudaGetLastError());
    h->launches++;
}

static void step_launch(kr_handle* h, Slab& sl, int dl, int cur, int prev, int nxt, int step, bool init, bool write,
                        bool fillinit = false, int cmode = 0) {
    if (h->TX == 64 && h->TY == 16)
        step_launch_t<64, 16>(h, sl, dl, cur, prev, nxt, step, init, write, fillinit, cmode);
    else if (h->TX == 64 && h->TY == 8)
        step_launch_t<64, 8>(h, sl, dl, cur, prev, nxt, step, init, write, fillinit, cmode);
    else
        KR_THROW(KR_EINVAL, "unsupported tile");
}

static void halo_exchange_virtual(kr_handle* h, int buf) {
    // the same schedule as the NCCL transport (krylov_zslab_halo_plan), executed as device copies: each
    // receive of slab s is served by the matching send of its peer
    const size_t plane = (size_t)h->pitch * h->my;
    const int S = (int)h->slabs.size();
    for (int s = 0; s < S; ++s) {
        kr_halo_op ops[4];
        int32_t n = 0;
        if (krylov_zslab_halo_plan(h->mz, S, s, ops, &n) != KR_OK) KR_THROW(KR_EINVAL, "halo plan");
        for (int i = 0; i < n; ++i) {
            if (ops[i].is_send) continue;
            const Slab& peer = h->slabs[ops[i].peer];
            kr_halo_op pops[4];
            int32_t pn = 0;
            krylov_zslab_halo_plan(h->mz, S, ops[i].peer, pops, &pn);
            for (int j = 0; j < pn; ++j)
                if (pops[j].is_send && pops[j].peer == s) {
                    if (pops[j].nplanes != ops[i].nplanes) KR_THROW(KR_EINVAL, "halo plan mismatch");
                    KR_CUDA(cudaMemcpyAsync(h->slabs[s].u[buf] + ops[i].plane * plane, peer.u[buf] + pops[j].plane * plane,
                                            ops[i].nplanes * plane * sizeof(double), cudaMemcpyDeviceToDevice,
                                            h->stream));
                }
        }
    }
}

// After the per-slab step kernels (whose last CTA wrote each slab's reduced vector): combine slabs /
// ranks and update the scalars — unless a single slab on a single rank already did it in-kernel.
static void combine_and_finalize(kr_handle* h, int dl, int step) {
    const int S = (int)h->slabs.size();
    const int zw = kr_zworld(h);
    if (S == 1 && zw == 1) return;
    LzScalars* sc = h->d_sc + dl;
    const int R = S * zw;
    double* rv_local = h->d_rankvec + (size_t)kr_zrank(h) * S * h->nq;
    if (zw > 1) kr_nccl_allgather(h->comm, rv_local, h->d_rankvec, (size_t)S * h->nq, h->stream);
    const int k = h->k;
    lz_finalize<<<1, 32, 0, h->stream>>>(h->d_rankvec, R, h->nq, h->n_out, step, k, sc,
                                         h->d_H ? h->d_H + (size_t)dl * (k + 1) * k : nullptr,
                                         h->d_P + (size_t)dl * h->n_out * k,
                                         h->d_beta0 + dl, h->d_hnext + dl, h->d_keff + dl);
    KR_CUDA(cudaGetLastError());
    h->launches++;
}

// Start of a Lanczos run for local direction dl on h->stream (capturable): reset, u_1, init pass.
void kr_lz_enqueue_init(kr_handle* h, int dl) {
    const int d = h->my_dirs[dl];
    LzScalars* sc = h->d_sc + dl;
    lz_reset<<<1, 32, 0, h->stream>>>(sc);
    KR_CUDA(cudaGetLastError());
    h->launches++;
    // u_1 = v_d on every slab including halo planes (analytic: no exchange needed); init pass: beta0,
    // alpha_1, P_{.,1}. Box/all generators: one fused fill+init pass; sparse: fill then the init pass.
    // Compact u_1 (analytic generator, small box): store only the box region; the init pass visits only
    // the tiles around it, and steps 1 and 2 read u_1 through the shifted compact tensor maps (TMA zero
    // fill elsewhere) — no 8n-byte fill pass, no full read of u_1.
    const DVec& g = h->dirs_h[d];
    for (auto& sl : h->slabs) {
        const bool cmp = !sl.cu1.empty() && sl.cu1[dl].on;
        if (cmp) {
            const Slab::CompactU1& c = sl.cu1[dl];
            const int64_t tot = c.pitch * c.h * c.d;
            const unsigned nb = (unsigned)std::min<int64_t>((tot + 255) / 256, 4096);
            lz_fill_compact_kernel<<<nb, 256, 0, h->stream>>>(sl.g1, c.x0, c.y0, c.p0, c.w, c.h, c.d, c.pitch, sl.z0,
                                                              h->mx, h->my, h->mz, g);
            KR_CUDA(cudaGetLastError());
            h->launches++;
            step_launch(h, sl, dl, 0, -1, 0, 0, true, false, false, 1);
        } else if (g.kind == KR_VEC_BOX || g.kind == KR_VEC_ALL) {
            step_launch(h, sl, dl, 0, -1, 0, 0, true, false, true);
        } else {
            kr_fill_grid(h->stream, sl.u[0], h->mx, h->my, h->pitch, sl.nz + 3, sl.z0 - 1, h->mz, g, &h->launches);
            step_launch(h, sl, dl, 0, -1, 0, 0, true, false);
        }
    }
    for (auto& sl : h->slabs) {
        const bool cmp = !sl.cu1.empty() && sl.cu1[dl].on;
        reduce_launch(h, sl, dl, 0, 0, true, false, 0, cmp ? 1 : 0);
    }
    combine_and_finalize(h, dl, 0);
}

// Lanczos step i (1-based: computes beta_i, alpha_{i+1}, u_{i+1}) for local direction dl. Steps whose
// direction already stopped (breakdown / k reached) exit at once on the device flag.
void kr_lz_enqueue_step(kr_handle* h, int dl, int i, bool capture_events) {
    const int k = h->k;
    const int cur = (i - 1) % 3, prev = (i >= 2) ? (i - 2) % 3 : -1, nxt = i % 3;
    const bool write = i < k;
    const int evp = (capture_events && dl == 0 && i < (int)h->ev_pair_of_step.size()) ? h->ev_pair_of_step[(size_t)i] : -1;
    const bool ev = evp >= 0;
    if (ev) KR_CUDA(kr_event_record(h->ev[2 * evp], h->stream));
    if (ev && (size_t)evp < h->ev_rec.size()) h->ev_rec[(size_t)evp] = 1;
    for (auto& sl : h->slabs) {
        const bool cmp = !sl.cu1.empty() && sl.cu1[dl].on && i <= 2;  // u_1 compact: u_i at step 1, u_{i-1} at 2
        step_launch(h, sl, dl, cur, prev, nxt, i, false, write, false, cmp ? i : 0);
    }
    if (ev) KR_CUDA(kr_event_record(h->ev[2 * evp + 1], h->stream));
    for (auto& sl : h->slabs) reduce_launch(h, sl, dl, nxt, i, false, write, write ? nxt : -1);
    if (write && !h->halo_inkernel) {  // message transport: copies / NCCL send-recv after the step
        if (h->slabs.size() > 1) halo_exchange_virtual(h, nxt);
        if (kr_zworld(h) > 1) kr_nccl_halo(h->comm, h, nxt, h->stream);
    }
    combine_and_finalize(h, dl, i);
}

// ---- the multi-step route ---------------------------------------------------------------------------------------
template <int TX, int TY, bool BC>
static void* multistep_fn() {
    return (void*)lz_multistep_kernel<TX, TY, Stages<TX, TY>::S, BC, 2>;
}

template <int TX, int TY>
static void multistep_setup_t(kr_handle* h) {
    constexpr int S = Stages<TX, TY>::S;
    const size_t smem = step2_smem_bytes<TX, TY, S>();
    void* fn = h->gen_bc ? multistep_fn<TX, TY, true>() : multistep_fn<TX, TY, false>();
    KR_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, sms = 148, per_sm = 0;
    KR_CUDA(cudaGetDevice(&dev));
    KR_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    KR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, Geo2<TX, TY, 2>::NT, smem));
    if (const char* e = getenv("KR_MS_PER_SM")) per_sm = std::min(per_sm, std::max(1, atoi(e)));
    h->ms_grid = (int)std::min<int64_t>(h->slabs[0].nitems, (int64_t)sms * per_sm);
    h->ms_one_per_sm = h->ms_grid <= sms;
    // both the multi-step kernel and the eigen-solve are half-SM CTAs (<= 128 registers x 256 threads): with the
    // multi-step grid at two per SM, the rest of the 2 x SMs slots can host the checkpoint evaluation beside it
    h->ms_free_slots = per_sm == 2 ? 2 * sms - h->ms_grid : 0;
    if (per_sm < 1 || h->ms_grid < 1) h->multistep = false;
}

// Decide the multi-step route (after the slabs exist): one slab on one rank, no sparse output rows (their
// gather needs the whole new vector after the step), state vectors small enough to stay in L2 (3 x 8 n bytes
// <= ~100 MB: n <= 2^22 cells). KR_MULTISTEP=0 / 1 forces it off / on (on: any single-slab grid).
void kr_lz_multistep_setup(kr_handle* h) {
    h->multistep = false;
    if (h->path != PATH_FUSED_LANCZOS || h->slabs.size() != 1 || kr_zworld(h) != 1 || h->halo_inkernel) return;
    for (const DVec& o : h->outs_h)
        if (o.kind == KR_VEC_SPARSE) return;
    const Slab& sl = h->slabs[0];
    const int64_t n = sl.nz * h->mx * h->my;
    bool on = n <= (int64_t(1) << 22);
    if (const char* e = getenv("KR_MULTISTEP")) on = atoi(e) != 0;
    if (!on) return;
    h->multistep = true;
    if (h->TX == 64 && h->TY == 16)
        multistep_setup_t<64, 16>(h);
    else if (h->TX == 64 && h->TY == 8)
        multistep_setup_t<64, 8>(h);
    else
        h->multistep = false;
}

template <int TX, int TY>
static void multistep_launch_t(kr_handle* h, Slab& sl, int dl, int i0, int i1) {
    constexpr int S = Stages<TX, TY>::S;
    StepArgs a = make_args(h, sl, dl, i0 % 3, i0, false, true, -1, 0);
    MultiArgs m{{sl.u[0], sl.u[1], sl.u[2]}, sl.mspart, i0, i1, nullptr};
    // KR_MS_PROF=1 (diagnostics, not inside graph capture): per-CTA phase times of the launch's first steps on stderr
    static const bool prof = getenv("KR_MS_PROF") != nullptr;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    KR_CUDA(cudaStreamIsCapturing(h->stream, &cs));
    const size_t np = (size_t)KR_MS_PROF_STEPS * h->ms_grid * 4;
    if (prof && cs == cudaStreamCaptureStatusNone) {
        KR_CUDA(cudaMalloc(&m.prof, np * 8));
        KR_CUDA(cudaMemsetAsync(m.prof, 0, np * 8, h->stream));
    }
    void* fn = h->gen_bc ? multistep_fn<TX, TY, true>() : multistep_fn<TX, TY, false>();
    void* args[] = {(void*)&sl.tmC[0], (void*)&sl.tmC[1], (void*)&sl.tmC[2], (void*)&sl.tmP[0],
                    (void*)&sl.tmP[1], (void*)&sl.tmP[2], (void*)&a, (void*)&m};
    KR_CUDA(cudaLaunchCooperativeKernel(fn, dim3((unsigned)h->ms_grid), dim3(Geo2<TX, TY, 2>::NT), args,
                                        step2_smem_bytes<TX, TY, S>(), h->stream));
    h->launches++;
    if (m.prof) {
        std::vector<uint64_t> t(np);
        KR_CUDA(cudaMemcpyAsync(t.data(), m.prof, np * 8, cudaMemcpyDeviceToHost, h->stream));
        KR_CUDA(cudaStreamSynchronize(h->stream));
        KR_CUDA(cudaFree(m.prof));
        const int G = h->ms_grid;
        for (int s = 0; s < KR_MS_PROF_STEPS && s <= i1 - i0; ++s) {
            const uint64_t* b = t.data() + (size_t)s * G * 4;
            if (b[0] == 0) break;
            uint64_t t0 = UINT64_MAX, t1max = 0, t2min = UINT64_MAX, t3max = 0;
            std::vector<double> march(G), wait(G);
            for (int c = 0; c < G; ++c) {
                const uint64_t* q = b + (size_t)c * 4;
                t0 = std::min(t0, q[0]);
                t1max = std::max(t1max, q[1]);
                t2min = std::min(t2min, q[2]);
                t3max = std::max(t3max, q[3]);
                march[c] = 1e-3 * (double)(q[1] - q[0]);
                wait[c] = 1e-3 * (double)(q[2] - q[1]);
            }
            std::vector<double> ms = march;
            std::sort(ms.begin(), ms.end());
            int slow = 0;
            for (int c = 1; c < G; ++c)
                if (march[c] > march[slow]) slow = c;
            fprintf(stderr,
                    "[kr ms prof] step %d: march min %.2f med %.2f max %.2f us (slowest CTA %d); last arrival -> first "
                    "release %.2f us; release -> step end %.2f us; step %.2f us\n",
                    i0 + s, ms[0], ms[G / 2], ms[G - 1], slow, 1e-3 * (double)((int64_t)t2min - (int64_t)t1max),
                    1e-3 * (double)(t3max - t2min), 1e-3 * (double)(t3max - t0));
        }
    }
}

// Enqueue Lanczos steps i0..i1 of local direction dl: the persistent multi-step kernel where it applies (steps
// past the compact-u_1 ones), else one step launch + one reduce launch per step.
void kr_lz_enqueue_steps(kr_handle* h, int dl, int i0, int i1, bool capture_events) {
    int i = i0;
    if (h->multistep) {
        Slab& sl = h->slabs[0];
        const bool cmp = !sl.cu1.empty() && sl.cu1[dl].on;
        while (i <= i1 && cmp && i <= 2) kr_lz_enqueue_step(h, dl, i++, capture_events);
        if (i > i1) return;
        const bool ev = capture_events && dl == 0;
        size_t pe = 0;
        if (ev) {
            pe = h->ms_ev.size();
            while (h->ms_events.size() < 2 * (pe + 1)) {
                cudaEvent_t e;
                KR_CUDA(cudaEventCreate(&e));
                h->ms_events.push_back(e);
            }
            h->ms_ev.push_back({(int)pe, i, i1 - i + 1});
            KR_CUDA(kr_event_record(h->ms_events[2 * pe], h->stream));
        }
        if (h->TX == 64 && h->TY == 16)
            multistep_launch_t<64, 16>(h, sl, dl, i, i1);
        else
            multistep_launch_t<64, 8>(h, sl, dl, i, i1);
        if (ev) KR_CUDA(kr_event_record(h->ms_events[2 * pe + 1], h->stream));
        return;
    }
    for (; i <= i1; ++i) kr_lz_enqueue_step(h, dl, i, capture_events);
}

// Enqueue the complete fixed-k Lanczos run for local direction dl on h->stream (capturable).
void kr_lz_enqueue_direction(kr_handle* h, int dl, bool capture_events) {
    kr_lz_enqueue_init(h, dl);
    kr_lz_enqueue_steps(h, dl, 1, h->k, capture_events);
}
