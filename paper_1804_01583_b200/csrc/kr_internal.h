// kr_internal.h — internal types shared by the CUDA translation units of libkrylov_reach.so.
// Not part of the ABI (include/krylov_reach.h is). sm_100a only.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/krylov_reach.h"

#define KR_KMAX KR_K_MAX   // max Krylov dimension (stencil Lanczos; Arnoldi <= KR_K_MAX_FIXED_PADE)
#define KR_MAX_BOX 8       // box-kind output rows handled inside the fused stencil kernel
#define KR_MAX_OUT 64      // output rows
#define KR_ORTHO_ONE_CTA_MAX 27648  // stored-basis N up to which one CTA per direction runs MGS on chip
#define KR_LONG_ROW 256             // CSR rows longer than this get a CTA of their own in the SpMM

// ------------------------------------------------------------------------------------------------
// error plumbing
// ------------------------------------------------------------------------------------------------
void kr_set_error(const std::string& msg);
// record an event on s: an external event node inside stream capture, a plain record otherwise
cudaError_t kr_event_record(cudaEvent_t e, cudaStream_t s);
struct KrError {
    kr_status st;
    std::string msg;
};
#define KR_THROW(st, msg) throw KrError{(st), (msg)}
#define KR_CUDA(call)                                                                                   \
    do {                                                                                                \
        cudaError_t e_ = (call);                                                                        \
        if (e_ != cudaSuccess)                                                                          \
            KR_THROW(KR_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_) + " @" + __FILE__ + ":" + \
                                   std::to_string(__LINE__));                                          \
    } while (0)

// ------------------------------------------------------------------------------------------------
// device-side descriptors
// ------------------------------------------------------------------------------------------------
// A compact vector on the device (kr_vec with device idx/val; sparse entries sorted and merged on host)
struct DVec {
    int32_t kind;
    int64_t nnz;
    const int64_t* idx;
    const double* val;
    int64_t lo[3], hi[3];
    double value;
    uint64_t seed;  // KR_VEC_RAND
};

// KR_VEC_RAND entry c (include/krylov_reach.h): value * (splitmix64(seed + (c + 1) G) >> 11) * 2^-53
__host__ __device__ __forceinline__ double kr_rand_entry(uint64_t seed, int64_t c, double value) {
    uint64_t z = seed + (uint64_t)(c + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return value * ((double)(z >> 11) * 0x1.0p-53);
}

struct BoxRow {  // a KR_VEC_BOX / KR_VEC_ALL output row as seen by the fused kernel (global coords)
    int32_t lo[3], hi[3];
    int32_t slot;  // output row index r
};

// Per-direction Lanczos scalars of the fused path (device memory, written by lz_finalize).
// Index convention (1-based as in Alg. 3): alpha[i] = H_{i,i}, beta[i] = H_{i+1,i}, s[i] = 1/||u_i||.
// The three arrays (k + 2 entries each) are the 3k of Eq. 6: H is kept tridiagonal.
struct LzScalars {
    double* alpha;
    double* beta;
    double* s;
    double hmax;
    double beta0;
    double h_next;
    int32_t done;
    int32_t k_eff;
    int32_t status;  // KR_OK or KR_EZERO / KR_ENONFINITE detected on device
    int32_t pad;
};

// One z-slab of the fused Lanczos path. Vector buffers hold (nz + 3) planes of my x pitch doubles:
// buffer plane 0 = global plane z0-1 (ghost / halo), planes 1..nz = owned z0..z1-1, planes nz+1, nz+2 =
// halo z1, z1+1 (zero ghosts where outside the global grid).
struct Slab {
    int64_t z0, z1, nz;
    double* u[3];
    CUtensorMap tmC[3];  // "center" role box (TX+4, TY+3, 1)
    CUtensorMap tmP[3];  // "previous" role box (TX+2, TY+1, 1)
    double* partials;    // [nblk][nqp]
    double* mspart = nullptr;  // multi-step kernel partials [2][nqp][ms grid]
    int32_t* counter;    // last-CTA arrival counter of the fused reduction
    int64_t nblk;        // persistent CTAs (= number of partial-sum slots)
    double* peer_lo[3];  // the lower / upper neighbour's state buffers (peer memory or a sibling slab), or NULL
    double* peer_hi[3];
    int64_t peer_lo_nz;  // owned planes of the lower neighbour
    int32_t gx, gy;      // tiles per x / y
    int64_t nitems;      // work items = gx * gy * z-chunks
    dim3 grid;
    int zchunk;
    int32_t win = 0;     // item order window (resident CTAs of the step kernel; 0 = z-chunk-major order)
    // Compact start vector u_1 of an analytic (box / all-grid) generator, per local direction: only the
    // generator box clipped to this slab's buffer planes is stored (cells x0 .. x0+w, y0 .. y0+h, buffer
    // planes p0 .. p0+d); the step kernels read it through tensor maps over that small array with shifted
    // coordinates, and TMA's out-of-bounds zero fill supplies every other cell (exact: u_1 is 0 there).
    struct CompactU1 {
        bool on = false;
        int64_t x0 = 0, y0 = 0, p0 = 0, w = 1, h = 1, d = 1, pitch = 2;
        CUtensorMap tmC, tmP;
        int32_t ix0 = 0, iy0 = 0, iz0 = 0, gx = 0, gy = 0;  // init-pass work items: tiles around the box only
        int64_t nitems = 0;
    };
    std::vector<CompactU1> cu1;  // [local direction]
    double* g1 = nullptr;        // compact u_1 buffer (largest region over the directions)
};

struct SlabInfo {  // device-visible copy for the local-reduce sparse gather
    int64_t z0, z1, nz;
    const double* u[3];
};

// ------------------------------------------------------------------------------------------------
// handle
// ------------------------------------------------------------------------------------------------
enum { PATH_FUSED_LANCZOS = 0, PATH_GENERIC = 1 };

struct kr_comm {
    void* nccl;  // ncclComm_t (NCCL transport), or NULL (host transport)
    int32_t rank, world, device;
    // host transport (krylov_comm_create_host): every collective is an all-gather of host buffers done by the
    // caller's function; the library stages through a pinned buffer and synchronises its stream around it
    kr_allgather_fn host_fn = nullptr;
    void* host_ctx = nullptr;
    double* pinned = nullptr;
    size_t pinned_doubles = 0;
};

struct FaceCor {  // per-face diagonal correction of face cells relative to Dirichlet (x-, x+, y-, y+, z-, z+)
    double e[6];
};

struct kr_handle {
    // problem (host copies of scalars)
    int32_t op, method, path, part;
    int64_t mx, my, mz, pitch;
    double alpha, cx, cy, cz;
    int32_t bc[6];      // stencil face boundary conditions (kr_bc), x-, x+, y-, y+, z-, z+
    double gamma[6];    // Robin coefficients (units of A)
    bool gen_bc;        // any non-Dirichlet face
    double eps;         // adaptive error target (0 = fixed k)
    int64_t n;  // unlifted state count
    int64_t N;  // operator dimension (n or n+1)
    bool lifted;
    int32_t n_gen, n_dir, n_out, k;  // simulation view: n_dir simulations, n_out projection rows each
    // final basis-matrix layout [(N+1)][cf_nout][cf_ndir] (= n_out / n_dir, swapped in transpose mode)
    bool transposed = false;
    int32_t n_gen_cf = 0;    // generator directions of the final layout (the fixed direction, if any, is last)
    int32_t cf_nout = 0, cf_ndir = 0;
    double* d_cf = nullptr;  // final coefficients (= d_coeff unless transposed)
    int64_t n_steps;
    double step;
    double mu;  // Gershgorin upper bound of lambda_max(sym A)
    int32_t device;
    cudaStream_t stream;
    bool own_stream;
    kr_comm* comm;
    int32_t rank, world;
    std::vector<int32_t> my_dirs;  // global direction indices handled by this rank
    std::vector<double> zlo, zhi;  // per global direction (fixed direction: 1,1)

    // device memory
    char* ws;
    size_t ws_bytes, ws_used;
    bool own_ws;
    std::vector<void*> extra_allocs;
    char* arena = nullptr;  // small device allocations are carved from 4 MB chunks (dalloc)
    size_t arena_used = 0, arena_cap = 0;

    // descriptors
    std::vector<DVec> dirs_h;          // per global direction: up to 2 pieces (gen/center + lifted one)
    std::vector<int32_t> dir_lift1;    // per global direction: 1 if the lifted coordinate is 1
    DVec* d_outs;                      // [n_out]
    DVec* d_gdirs = nullptr;           // stored-basis paths: the local directions' start vectors [ndl]
    int32_t* d_glift = nullptr;        // ... and their lifted coordinate (1 for v_f = [c; 1]) [ndl]
    std::vector<DVec> outs_h;
    double* d_O;                       // generic path: dense [n_out][N]
    // CSR
    int64_t* d_rp;
    int32_t* d_ci;
    double* d_val;
    double* d_b;

    // results [local dirs]
    double* d_H;      // [ndl][k+1][k]
    double* d_P;      // [ndl][n_out][k]
    double* d_beta0;  // [ndl]
    double* d_hnext;  // [ndl]
    int32_t* d_keff;  // [ndl]
    int32_t* d_done;  // [ndl]
    double* d_hmax;   // [ndl]
    double* d_coeff;  // [(n_steps+1)][n_out][n_dir]  (full, after gather)
    double* d_coeff_loc;  // [(n_steps+1)][n_out][ndl]
    double* d_hlast;  // [ndl][n_steps+1]
    double* d_lemma;  // [ndl]
    double* d_zlo;    // [n_dir]
    double* d_zhi;
    double* d_box;    // box-check outputs: lo, hi [(N+1)][n_out]
    void* d_cex;      // device cex + witness
    double* d_gather; // dirs partition gather scratch
    int32_t* d_status;
    int32_t* d_box_slot;  // [n_box] output row of each fused box row
    double* d_box_val;    // [n_box] value of each fused box row
    int32_t* d_sense;     // [n_out] check_box scratch
    double* d_thr;        // [n_out]

    // fused path
    std::vector<Slab> slabs;
    SlabInfo* d_slabinfo;
    LzScalars* d_sc;       // [ndl]
    double* d_rankvec;     // [world*nslabs][nq]
    int32_t nq, nqp;       // 2 + n_out ; 2 + n_box
    std::vector<BoxRow> boxes;
    int32_t TX, TY;

    double* d_lzarr;       // [ndl][3][k+2] alpha / beta / s arrays of d_sc
    int steps_run0 = 0;
    double large_ms = 0.0;  // device time of the large-k route (exponentials + bounds) in the last project
    int32_t large_evals = 0;
    cudaEvent_t ev_lg0 = nullptr, ev_lg1 = nullptr;
    cudaStream_t stream2 = nullptr;  // adaptive runs: checkpoint evaluations beside the next checkpoint's steps
    cudaEvent_t ev_spec = nullptr;    // Lanczos steps run for local direction 0 by the last large-route project
    bool halo_inkernel = false;  // halo planes written by the step kernel into the neighbours' buffers
    bool p2p = false;            // ... across processes through CUDA IPC peer memory (NVLink)
    void* p2p_base[2] = {nullptr, nullptr};  // opened IPC bases (lower, upper neighbour)
    int32_t p2p_rank = 0, p2p_world = 1;
    bool expm_doubling = false;  // small-k exponentials: doubling over the time grid (else Pade per step)
    double* d_xt = nullptr;      // doubling trajectories [ndl][64][xt_ld] (one-CTA doubling, KR_EXPM_ONECTA=1)
    bool expm_onecta = false;
    double* d_pw = nullptr;      // powers E^{2^q} of e^{H delta}, [ndl][pw_q][64][65] (multi-CTA march)
    int pw_q = 0;
    int xt_ld = 0;
    bool large_route;      // exponentials through the large-k route (kr_large.cu) instead of per-step Pade
    // large-k route scratch (allocated at the first project that needs it, for kcap = k)
    double* d_big;         // 6 x kcap^2 doubles: X, X^2, X^3, X^4, Y, Y'
    double* d_traj;        // [(n_steps+1)][kcap] x_j = e^{H t_j} e_1
    int large_cap = 0;     // padded dimension the large-route scratch is sized for
    double* d_gpart = nullptr;      // split-K partial sums of the band GEMMs
    size_t large_part_doubles = 0;
    void* h_pin = nullptr;   // pinned host scratch (checkpoint bound + scalars in one round trip)
    bool multistep = false;  // Lanczos steps >= 3 by the persistent multi-step kernel (single L2-resident slab)
    int ms_grid = 0;         // its cooperative grid
    bool ms_one_per_sm = false;  // ... at most one CTA per SM (room for the eigen-solve's CTAs beside it)
    int ms_free_slots = 0;       // SM slots (half an SM each) a multi-step launch at two CTAs per SM leaves free
    int tdc_grid_cap = 0;        // > 0: the eigen-solve runs beside a multi-step launch on at most this many CTAs
    struct MsEv {
        int pair, i0, n;  // event pair index into ms_events, first step, steps
    };
    std::vector<MsEv> ms_ev;
    std::vector<char> ev_rec;  // per-step event pair recorded by the last enqueue (steps inside a multi-step launch are not)  // timed multi-step launches: (event pair index into ms_events, steps)
    std::vector<cudaEvent_t> ms_events;
    void* d_tdc = nullptr;  // divide-and-conquer eigen-solve workspace (kr_tridc.cu), for dimension tdc_cap
    int tdc_cap = 0;
    double* d_lbound;      // [ndl] unit-vector Lemma 1 bound of the accepted k
    double* d_scratch;     // small device scratch (norms, bound)
    std::vector<std::vector<std::pair<int32_t, double>>> checks;  // per local direction: (k, bound)

    // generic path
    double* d_bl = nullptr;   // stencil affine term b (dense, length n) when lifted, else NULL
    int64_t* d_long = nullptr;  // CSR rows with > KR_LONG_ROW entries
    int64_t n_long = 0;
    double* d_cgs = nullptr;  // CGS2 scratch (N > KR_ORTHO_ONE_CTA_MAX)
    bool use_cgs = false;     // stored-basis orthogonalisation by the multi-CTA CGS2 path
    double* d_V;  // [ndl][k+1][N]
    double* d_W;  // [ndl][N]

    // graph
    cudaGraphExec_t gexec;
    bool graph_ready;
    int64_t graph_launches;  // kernel nodes in the Krylov graph
    int64_t launches;
    bool projected;

    // timing
    bool timing;
    std::vector<cudaEvent_t> ev;  // pairs around the step kernel of the timed steps
    std::vector<int> ev_pair_of_step;  // [k + 1]: event pair of step i, or -1 (step not timed)
    std::vector<int> ev_step_of_pair;
    cudaEvent_t ev_it0, ev_it1;
    double last_iter_ms, last_step_ms_mean;
    std::vector<double> step_ms;  // per-step device times of the last project (first KR_MAX_EV steps, direction 0)
    int64_t last_step_launches;
    double step_bytes;  // algorithmic bytes per fused step launch (24 n_local)
    int64_t h2d_bytes, d2h_bytes;  // host<->device bytes moved by the ABI calls (create/project/check_box)
};

// ------------------------------------------------------------------------------------------------
// launchers (implemented in the .cu files)
// ------------------------------------------------------------------------------------------------
// fill: dst[(plane b, y, x)] for b in [0, nplanes) representing global plane zbase + b, pitch doubles per row
void kr_fill_grid(cudaStream_t s, double* dst, int64_t mx, int64_t my, int64_t pitch, int64_t nplanes,
                  int64_t zbase, int64_t mz, const DVec& v, int64_t* launches);
void kr_fill_dense(cudaStream_t s, double* dst, int64_t N, int64_t n, int64_t mx, int64_t my, bool stencil,
                   const DVec& v, int lift1, double scale, int accumulate, int64_t* launches);

// fused Lanczos
// Device memory owned by handles (kr_api.cu): a process-wide cache of freed blocks by (device, size class),
// so destroy / create do not pay cudaFree / cudaMalloc (blocks above the 1 GiB cache cap are freed).
cudaError_t kr_dev_malloc(void** p, size_t bytes);
void kr_dev_free(void* p);
void kr_dev_mark_exported(void* base);  // an IPC-exported block: cudaFree at its free, never cached

void kr_lz_encode_maps(kr_handle* h);
void kr_lz_setup_compact(kr_handle* h);
void kr_lz_enqueue_direction(kr_handle* h, int dl, bool capture_events);
size_t kr_lz_step_smem(int TX, int TY);

// generic
// the stencil operator's per-face diagonal correction (insulated / Robin faces, NEXT-1) relative to Dirichlet
inline FaceCor kr_face_cor(const kr_handle* h) {
    FaceCor fc{};
    const double c[3] = {h->cx, h->cy, h->cz};
    for (int f = 0; f < 6; ++f)
        fc.e[f] = (h->bc[f] != KR_BC_DIRICHLET ? c[f / 2] : 0.0) - (h->bc[f] == KR_BC_ROBIN ? h->gamma[f] : 0.0);
    return fc;
}
void kr_ge_enqueue_direction_set(kr_handle* h);
void kr_ge_enqueue_init(kr_handle* h);
void kr_ge_enqueue_step(kr_handle* h, int j);
size_t kr_cgs_scratch_doubles(const kr_handle* h, int ndl);
// One stored-basis Krylov step of the multi-CTA CGS2 path: j == 0 normalises the start vectors; j >= 1 applies
// the operator to v_{j-1} (fused with the first projection pass) and orthogonalises (kr_arnoldi.cu).
void kr_cgs_step(kr_handle* h, int j, int ndl, double* scratch);
// Y[d] = A' X[d] for the ndl local directions (CSR, lifted when b is set): block SpMM, each row read once (kr_generic.cu)
void kr_csr_spmm(kr_handle* h, const double* X, int64_t xstride, double* Y, int64_t ystride, int ndl);

// expm + projection + lemma
void kr_expm_enqueue(kr_handle* h);
void kr_expm_small_eval(kr_handle* h, int dl, int kc, const double* Hdense, int hstride, double* xt, int ldx);
// large-k route (kr_large.cu): x_j = e^{H t_j} e_1 for the tridiagonal of local direction dl at dimension
// kc, the coefficients c[j][.][d] of direction dl and the unit-vector Lemma 1 bound (returned; 0 with
// zero_bound, an exact breakdown); fin also writes the direction's stats. Synchronises the stream.
double kr_large_eval(kr_handle* h, int dl, int kc, bool fin, bool zero_bound, LzScalars* sc_out = nullptr);
void kr_large_alloc(kr_handle* h, int kc);
// kr_tridc.cu: the same for the symmetric Lanczos tridiagonal through a device divide-and-conquer eigen-solve
// (coefficients of direction dl and e_kc^T x_j into hl); kc up to kr_tridc_max_k()
void kr_tridc_eval(kr_handle* h, int dl, int kc, double* hl, int ndl_stride);
int kr_tridc_max_k();
// fused Lanczos building blocks for the adaptive (host-driven) loop
void kr_lz_enqueue_init(kr_handle* h, int dl);
void kr_lz_enqueue_steps(kr_handle* h, int dl, int i0, int i1, bool capture_events);
void kr_lz_multistep_setup(kr_handle* h);
void kr_lz_enqueue_step(kr_handle* h, int dl, int i, bool capture_events);
// box
void kr_box_enqueue(kr_handle* h, const int32_t* d_sense, const double* d_thr);

void kr_eval_outputs(kr_handle* h, int64_t step, const double* z_h, double* y_h);
// per-step LP (kr_lp.cu)
void kr_lp_run(kr_handle* h, int m_init, const double* IA, const double* Ib, int m_uns, const double* UA,
               const double* Ub, int32_t* feas_h, double* out_h);

// collectives (kr_comm.cu): NCCL, or the caller's host all-gather (host transport)
void kr_nccl_allgather(kr_comm* c, const double* send, double* recv, size_t count, cudaStream_t s);
void kr_nccl_check(kr_comm* c);
void kr_nccl_halo(kr_comm* c, kr_handle* h, int buf, cudaStream_t s);
inline bool kr_comm_is_host(const kr_comm* c) { return c && c->host_fn; }
// ranks that share one state vector: the z-slab partition's world (direction sharding keeps each direction on one
// rank, so its Lanczos scalars are reduced locally)
inline int kr_zworld(const kr_handle* h);
inline int kr_zrank(const kr_handle* h);
// peer-memory halo transport (kr_comm.cu)
void kr_p2p_blob(kr_handle* h, void* out);
void kr_p2p_open(kr_handle* h, const void* blobs, int32_t rank, int32_t world);
void kr_p2p_verify(kr_handle* h, int32_t* ok);
void kr_p2p_close(kr_handle* h);

inline int kr_zworld(const kr_handle* h) { return h->part == KR_PART_ZSLAB ? h->world : 1; }
inline int kr_zrank(const kr_handle* h) { return h->part == KR_PART_ZSLAB ? h->rank : 0; }
