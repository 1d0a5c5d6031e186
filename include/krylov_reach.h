/*
 * krylov_reach.h — C ABI of the B200-native Krylov projected-reachability hot path
 * (arXiv 1804.01583; PAPER.md cited as P:<line>; SURVEY.md §8(b) is the design note).
 *
 * What the library computes. For the affine system x' = Ax + b, an initial set
 * x0 = c + sum_d z_d g_d with a box z_lo <= z <= z_hi (initial space E, §3.2), output rows
 * C (o x n, §3.1), a step delta and N steps (t_j = j*delta, j = 0..N), it returns the
 * basis-matrix sequence C e^{A t_j} E by Krylov simulation of one direction per column of E
 * (§4.1; Eq. 2) — Arnoldi (Alg. 1) or Lanczos with projection
 * (Alg. 3/4) — and, per step, the interval bounds of every output over the box together
 * with the first violating step and a witness (Fig. 2(c)).
 *
 * Conventions (all functions):
 *  - Every pointer argument of kr_problem is HOST memory, borrowed for the duration of
 *    krylov_reach_create only: the library deep-copies what it needs to the device.
 *  - Output arrays are caller-allocated HOST buffers whose sizes follow from the problem:
 *    n_dir = n_gen + has_fixed, has_fixed = (center != NULL || b != NULL).
 *  - Errors: every call returns a kr_status; krylov_last_error() returns a thread-local message for
 *    the last non-OK status. After KR_ECUDA or KR_ENCCL the handle is unusable (destroy it).
 *  - No C++ types, exceptions or torch types cross this ABI.
 *  - Numerics: fp64 throughout. Results are bit-reproducible for identical inputs
 *    and identical partitioning (fixed-order reductions, no floating-point atomics).
 */
#ifndef KRYLOV_REACH_H
#define KRYLOV_REACH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    KR_OK = 0,
    KR_EINVAL = 1,      /* invalid argument: k < 1, step <= 0, n_steps < 0, z_lo > z_hi, bad enum, NULL */
    KR_EDIM = 2,        /* dimension mismatch / index out of range                          */
    KR_ENOMEM = 3,      /* device allocation failed or caller workspace too small                      */
    KR_ECUDA = 4,       /* CUDA runtime / driver failure                                               */
    KR_ENCCL = 5,       /* NCCL failure                                                                */
    KR_ENOTSYM = 6,     /* Lanczos requested on a non-symmetric operator (Alg. 3 needs A = A^T, §4.3)  */
    KR_EZERO = 7,       /* a direction vector is zero: ||v|| = 0 cannot be normalised (Alg. 1 line 1)  */
    KR_ENONFINITE = 8,  /* non-finite input value                                                      */
    KR_ESTATE = 9       /* call out of order (check_box before project)                               */
} kr_status;

typedef enum { KR_OP_STENCIL7 = 0, KR_OP_CSR = 1 } kr_op;
typedef enum { KR_AUTO = 0, KR_ARNOLDI = 1, KR_LANCZOS = 2 } kr_method;
typedef enum { KR_PART_NONE = 0, KR_PART_ZSLAB = 1, KR_PART_DIRS = 2 } kr_partition;
typedef enum { KR_GE = 0, KR_LE = 1, KR_EQ = 2, KR_NONE = 3 } kr_sense;
typedef enum { KR_VEC_SPARSE = 0, KR_VEC_BOX = 1, KR_VEC_ALL = 2, KR_VEC_RAND = 3 } kr_vec_kind;
/* Stencil boundary condition of one grid face (the paper's heat model, §5.3: all faces insulated
 * except x = 1, which exchanges heat with constant 0.5; SURVEY A1/A2 reconstruction, DESIGN R18):
 *  KR_BC_DIRICHLET: zero ghost value beyond the face (BASELINE configs; A = alpha L_h).
 *  KR_BC_INSULATED: the missing neighbour is dropped (zero flux): a face cell's diagonal is -(#neighbours) c_a.
 *  KR_BC_ROBIN:     insulated plus exchange with a zero ambient: the face cell's diagonal also gets -gamma
 *                   (gamma in units of A, e.g. 0.01 * 0.5 / h for the paper's x = 1 face).             */
typedef enum { KR_BC_DIRICHLET = 0, KR_BC_INSULATED = 1, KR_BC_ROBIN = 2 } kr_bc;
/* Which simulations compute the basis matrix C e^{A t} E (§4.1):
 *  KR_SIM_FORWARD:   one Krylov simulation of x' = A x per direction (generator columns of E + v_f);
 *  KR_SIM_TRANSPOSE: one simulation of x' = A'^T x per output row C_r^T, projected with E^T and
 *                    transposed back ("(E^T e^{A^T t} C^T)^T") — o simulations instead of i;
 *                    with an affine term the lifted A' = [[A, b], [0, 0]] is transposed explicitly;
 *  KR_SIM_AUTO:      the smaller of the two counts, min(i, o).                           */
typedef enum { KR_SIM_FORWARD = 0, KR_SIM_TRANSPOSE = 1, KR_SIM_AUTO = 2 } kr_sim_dir;
#define KR_K_MAX_FIXED_PADE 64   /* fixed k up to this uses per-step Pade-13 exponentials            */
#define KR_K_MAX 16384           /* Lanczos (stencil) Krylov dimension cap                          */
#define KR_K_MAX_ARNOLDI 2048    /* stored-basis (Arnoldi) Krylov dimension cap                     */

/* An n-vector given compactly: a generator column of E, the center c, or an output row of C
 * (P:447). Linear index of stencil cell (x,y,z) is x + mx*(y + my*z) (x fastest).
 *  KR_VEC_SPARSE: entries val[e] at idx[e] (e < nnz; duplicates add).
 *  KR_VEC_BOX:    value on the index box [lo, hi) (stencil: 3D; CSR: axis 0 only, lo[1..2]/hi[1..2] ignored).
 *  KR_VEC_ALL:    value everywhere (e.g. total heat). Never includes the lifted coordinate.
 *  KR_VEC_RAND:   a seeded dense field value * u_c over all n states, u_c = (mix(seed + (c+1) G) >> 11) 2^-53 in
 *                 [0, 1) with c the linear index, G = 0x9E3779B97F4A7C15 and mix the splitmix64 finaliser
 *                 (z ^= z >> 30; z *= 0xBF58476D1CE4E5B9; z ^= z >> 27; z *= 0x94D049BB133111EB; z ^= z >> 31),
 *                 all mod 2^64. A synthetic dense start vector (the dense-data bench workload); only
 *                 for generators and the center, forward simulations, no affine term (else KR_EINVAL). */
typedef struct {
    int32_t kind;
    int64_t nnz;
    const int64_t* idx;
    const double* val;
    int64_t lo[3], hi[3];
    double value;
    uint64_t seed;              /* KR_VEC_RAND only */
} kr_vec;

/* Opaque multi-GPU communicator (one process per GPU; NCCL over NVLink/NVSwitch). */
typedef struct kr_comm kr_comm;

typedef struct {
    /* Operator A. */
    int32_t op;                 /* kr_op */
    int64_t mx, my, mz;         /* STENCIL7: grid; A = alpha * L_h, Dirichlet, h_a = 1/(m_a+1) */
    double alpha;
    int64_t n, nnz;             /* CSR: n x n, row_ptr[n+1] (int64), col_idx[nnz] (int32), val[nnz]   */
    const int64_t* row_ptr;
    const int32_t* col_idx;
    const double* val;
    const double* b;            /* CSR only: affine term (length n) or NULL. Lifted into A' = [[A,b],[0,0]]
                                   with the extra coordinate fixed at 1. Must be NULL for STENCIL7. */
    const kr_vec* b_vec;        /* STENCIL7 only: the affine term as a compact vector (e.g. the permanent heater
                                   patch of P:1136-1138), lifted the same way (the system becomes nonsymmetric:
                                   Arnoldi); NULL = none. Must be NULL for CSR.                            */
    /* Initial set. */
    int32_t n_gen;              /* generator directions g_d, d < n_gen                                  */
    const kr_vec* gen;
    const double* z_lo;         /* box on z, length n_gen                                               */
    const double* z_hi;
    const kr_vec* center;       /* c, or NULL for 0. With b != NULL or center != NULL one fixed direction
                                   v_f = [c; 1] (or c) with z_f = 1 is appended             */
    /* Output space. */
    int32_t n_out;
    const kr_vec* out;          /* rows of C; entries at the lifted coordinate are 0                   */
    /* Time grid: t_j = (double)j * step, j = 0..n_steps. */
    double step;
    int64_t n_steps;
    /* Krylov iteration. */
    int32_t k;                  /* Krylov dimension (max; k_eff < k on breakdown). Stored-basis
                                   paths (Arnoldi, CSR): 1..KR_K_MAX_ARNOLDI. Stencil Lanczos: 1..KR_K_MAX.
                                   k > 64 or eps > 0 use the large-k exponential route (krylov_project)   */
    int32_t method;             /* kr_method. AUTO: Lanczos for STENCIL7 or exactly symmetric CSR (b=NULL) */
    /* Adaptive Krylov dimension, Alg. 2/4: eps > 0 runs the stencil Lanczos with
       error control — the Lemma 1 bound (unit start vector, tau = T, trapezoid on the t_j grid)
       is evaluated at the checkpoints k = 4, ceil(1.1 k), ... (fp64) and the first checkpoint
       whose bound is < eps is accepted; `k` is then the maximum (k_max). An exact breakdown before k_max
       is accepted with bound 0. If no checkpoint up to k_max meets eps, the k_max result is returned and
       kr_dir_stats.lemma1_bound reports its (too large) bound. eps = 0: fixed k. Stencil Lanczos only.  */
    double eps;
    /* Stencil boundary conditions per face, order x-, x+, y-, y+, z-, z+ (kr_bc; all zero = Dirichlet,
       the BASELINE configs) and the Robin exchange coefficients (used where bc = KR_BC_ROBIN, >= 0).   */
    int32_t bc[6];
    double gamma[6];
    /* Simulation direction (kr_sim_dir; 0 = forward). TRANSPOSE needs n_dir <= 64 (the directions become
       the projection rows) and is not combined with eps > 0.                                          */
    int32_t sim_dir;
    /* Partitioning. */
    int32_t part;               /* kr_partition. ZSLAB: STENCIL7 + LANCZOS only; DIRS: any             */
    int32_t virtual_slabs;      /* ZSLAB without a comm: emulate P = virtual_slabs slabs in this process
                                   on one device (halo copies instead of NCCL); 0/1 = off                */
    kr_comm* comm;              /* NULL = single process; otherwise create/project/check are collective */
    int32_t device;             /* CUDA device ordinal                                                  */
    void* stream;               /* cudaStream_t to run on, or NULL for a library-owned stream           */
    void* workspace;            /* optional caller-owned device buffer for the state vectors (e.g. a torch
                                   uint8 tensor) of at least krylov_workspace_bytes; NULL = library
                                   allocates. Must outlive the handle. Small descriptors and results are
                                   always library-allocated.                                             */
    size_t workspace_bytes;
} kr_problem;

typedef struct kr_handle kr_handle;

/* Per-simulation diagnostics (Lemma 1): one per direction (forward) or per output row
 * (transpose mode); krylov_sim_info gives the count. */
typedef struct {
    int32_t k_eff;              /* Krylov dimension actually used                                       */
    double beta0;               /* ||v_d||                                                              */
    double h_next;              /* h_{k_eff+1,k_eff} (0 on exact breakdown)                             */
    double lemma1_bound;        /* beta0 * h_next * e^{max(mu,0) T} * int_0^T |e_k^T e^{Ht} e_1| dt, with
                                   mu a Gershgorin upper bound of lambda_max((A+A^T)/2) and the integral
                                   by the trapezoid rule on the t_j grid                                 */
} kr_dir_stats;

/* Counter-example. */
typedef struct {
    int32_t found;              /* 1 = UNSAFE (some row violates at some step), 0 = SAFE               */
    int64_t step;               /* first violating j (first-hit semantics)                 */
    double time;                /* (double)step * delta                                                */
    int32_t row;                /* lowest violating output row at that step                            */
    double y;                   /* output value at the witness: sum_d c[j][row][d] z*_d                 */
} kr_cex;

/* Device bytes this rank needs for p (3 slab vectors + halos + scratch for the Lanczos stencil path;
 * (k+1) vectors per direction for Arnoldi). Host-only, no GPU work. */
kr_status krylov_workspace_bytes(const kr_problem* p, size_t* bytes);

/* Validate p, select the device, allocate (or bind the caller workspace), upload the operator and
 * descriptors, and prepare the per-step launch graph. Collective when p->comm != NULL. */
kr_status krylov_reach_create(const kr_problem* p, kr_handle** out);

/* Run the hot path: start vectors, k Krylov steps per direction (fused stencil Lanczos in one HBM pass
 * per step, or batched SpMM + Gram-Schmidt Arnoldi: one-CTA MGS below 4096 states, multi-CTA CGS2 above),
 * the k x k exponentials x_j = e^{H t_j} e_1 for every t_j (Eq. 2; "squaring and scaling and Pade",
 * e^{H delta} by Pade-13 scaling and squaring, then the uniform grid by doubling,
 * x_{2^q+j} = e^{H 2^q delta} x_j; for k > 64 or eps > 0 the large-k route with fp64 tensor-core GEMMs and,
 * with eps > 0, the Alg. 2/4 checkpoints) and the projection through P = C V_k (Alg. 4).
 * coeff: HOST [(n_steps+1)][n_out][n_dir] basis-matrix entries c[j][r][d] ~= C_r e^{A t_j} v_d (same
 * layout in transpose mode). stats: HOST [n_sim] (krylov_sim_info) or NULL. Either output may be NULL to
 * leave the results on the device only (then krylov_check_box still works). Synchronises the stream
 * before returning. */
kr_status krylov_project(kr_handle* h, double* coeff, kr_dir_stats* stats);

/* Per-step safety check over the box initial set (the exact LP optimum of Fig. 2(c) for a box and one
 * output half-space per row): lo/hi[j][r] = c_f + sum_d min/max(c z_lo_d, c z_hi_d); row r is unsafe at
 * step j if (GE) hi >= thr, (LE) lo <= thr, (EQ) lo <= thr <= hi; KR_NONE rows are never unsafe.
 * sense, thr: HOST [n_out]. lo, hi: HOST [(n_steps+1)][n_out] or NULL. cex: HOST, required.
 * z_witness: HOST [n_dir] or NULL: GE -> z_hi where c >= 0 else z_lo; LE mirrored; EQ interpolates
 * lambda = (thr-lo)/(hi-lo) along that vertex path. Requires a prior krylov_project. */
kr_status krylov_check_box(kr_handle* h, const int32_t* sense, const double* thr, double* lo, double* hi,
                           kr_cex* cex, double* z_witness);

/* Destroys the handle after its stream has finished. Its device blocks (everything but a caller workspace)
 * go to a process-wide cache, keyed by device and size class and capped at 1 GiB, from which the next
 * handles allocate: create / destroy then pay no cudaMalloc / cudaFree. */
void krylov_reach_destroy(kr_handle* h);

/* Returns every cached device block (see krylov_reach_destroy) to the driver, e.g. before cudaDeviceReset
 * or when the memory is needed elsewhere. Live handles are unaffected. Returns the bytes released.        */
size_t krylov_release_cached_memory(void);

const char* krylov_last_error(void);

/* The general per-step LP (NEXT-3; §2.1 P:145-152 in the initial / output spaces of §3; the LP
 * of Fig. 2(c), for polytopes): at every step j, is there z with
 *     z_lo <= z <= z_hi,   init_A z <= init_b,   unsafe_A (B_j z + c_f,j) <= unsafe_b ?
 * B_j = c[j][.][0..n_gen) (generator columns), c_f,j = c[j][.][n_gen] (fixed direction, z_f = 1) or 0.
 * init_A: HOST [m_init][n_gen] row-major (on the generator coordinates only), init_b [m_init];
 * unsafe_A: HOST [m_unsafe][n_out], unsafe_b [m_unsafe] (an equality is two rows). All N+1 LPs are solved
 * independently on the device (dense Phase-I simplex, Bland's rule, feasibility tolerance 1e-9 after row
 * normalisation). feasible: HOST [(n_steps+1)] or NULL: 1 feasible, 0 infeasible, -1 iteration cap.
 * cex: first feasible step (found, step, time; row = -1, y = first output at the witness). z_witness
 * [n_dir] (fixed coordinate 1) and y_witness [n_out] receive the solver's assignment, or may be NULL.
 * Requires krylov_project. KR_EINVAL if m_init + m_unsafe + n_gen exceeds the one-CTA tableau (~100).  */
kr_status krylov_check_lp(kr_handle* h, int32_t m_init, const double* init_A, const double* init_b, int32_t m_unsafe,
                          const double* unsafe_A, const double* unsafe_b, int32_t* feasible, kr_cex* cex,
                          double* z_witness, double* y_witness);

/* The outputs at one initial-space point: y[r] = sum_d c[step][r][d] z[d] (the basis matrix of P:481
 * applied to z; z HOST [n_dir] including z_f = 1 for the fixed direction, y HOST [n_out]). Used to check a
 * counter-example against an independent higher-accuracy re-simulation. */
kr_status krylov_eval_outputs(kr_handle* h, int64_t step, const double* z, double* y);

/* Simulation layout of h: *transposed = 1 in transpose mode (KR_SIM_TRANSPOSE, or AUTO with n_out < n_dir),
 * *n_sim = number of Krylov simulations (= length of the stats array of krylov_project): n_dir forward,
 * n_out transposed. Either pointer may be NULL. */
kr_status krylov_sim_info(const kr_handle* h, int32_t* transposed, int32_t* n_sim);

/* Number of this library's kernel launches issued so far on h (graph nodes counted per replay). */
int64_t krylov_launch_count(const kr_handle* h);

/* Host<->device bytes moved so far by this handle's ABI calls (create uploads, project/check_box
 * downloads and threshold uploads). */
kr_status krylov_transfer_bytes(const kr_handle* h, int64_t* h2d, int64_t* d2h);

/* Device-side duration in ms of the last krylov_project's Krylov iteration phase and of its dominant
 * kernel (mean per launch), measured with CUDA events on the library stream. */
kr_status krylov_last_timing(const kr_handle* h, double* iter_ms, double* step_kernel_ms_mean,
                             int64_t* step_kernel_launches, double* step_kernel_bytes);

/* Per-step device times (ms, CUDA events around the Krylov step's operator/step kernel of local direction 0)
 * of the last krylov_project: ms HOST [cap] or NULL, ms[i] for step i + 1 of the *n steps run. Timed steps:
 * the first min(k, KR_MAX_EV) if that environment variable is set, else steps 1, 2 and six steps spread over
 * 3..k-1 (k <= 64) or every 16th step from 3 on (k > 64, adaptive runs); event nodes around every step cost
 * ~8 us per step in the CUDA graph. Other entries are NaN. */
kr_status krylov_step_times(const kr_handle* h, double* ms, int32_t cap, int32_t* n);

/* Device time in ms spent by the last krylov_project in the large-k exponential route (all checkpoint
 * evaluations: e^{H delta} by scaling and squaring, the time march, projection and Lemma 1 bound;
 * CUDA events on the library stream) and the number of evaluations. 0 / 0 on the small-k route.    */
kr_status krylov_last_timing_large(const kr_handle* h, double* expm_ms, int32_t* n_evals);

/* Copy direction `dir`'s Krylov data to the host: H [(k+1)][k] row-major (the (k+1) x k Hessenberg
 * of Alg. 1 / tridiagonal of Alg. 3, entries beyond k_eff are 0) and P = C V [n_out][k] (Alg. 4).
 * Either pointer may be NULL. KR_EDIM if `dir` is not handled by this rank. Requires krylov_project. */
kr_status krylov_krylov_data(const kr_handle* h, int32_t dir, double* H, double* P);

/* Lanczos tridiagonal of direction `dir` (Alg. 3/4 keep H as 3 arrays, Eq. 6): alpha[i] =
 * H_{i+1,i+1}, beta[i] = H_{i+2,i+1} for i < k_eff (beta[k_eff-1] = h_{k_eff+1,k_eff}). HOST buffers of
 * `cap` doubles, either may be NULL; *k_eff receives k_eff. Stencil Lanczos path only (else KR_EINVAL). */
kr_status krylov_tridiag(const kr_handle* h, int32_t dir, double* alpha, double* beta, int32_t cap, int32_t* k_eff);

/* Adaptive error control trace of direction `dir` (eps > 0): the checkpoints evaluated, in order, with
 * the Lemma 1 bound of each (unit start vector). HOST buffers of `cap` entries; *n receives
 * the number of checkpoints evaluated (the last one evaluated is the accepted one unless breakdown).   */
kr_status krylov_adaptive_checks(const kr_handle* h, int32_t dir, int32_t* ks, double* bounds, int32_t cap,
                                 int32_t* n);

/* ---- multi-GPU plumbing (one process per GPU) -------------------------------------------------- */
/* Rank 0 calls krylov_comm_unique_id (128 bytes out), the caller broadcasts it (torch.distributed),
 * then every rank calls krylov_comm_create. Collective. */
kr_status krylov_comm_unique_id(void* id128);
kr_status krylov_comm_create(const void* id128, int32_t rank, int32_t world, int32_t device, kr_comm** out);
void krylov_comm_destroy(kr_comm* c);
/* Health check of a communicator as the fixed-k run uses it: the per-step all-gather of rank vectors (z-slab
 * partition) issued inside a CUDA graph capture on `stream` (a cudaStream_t; NULL = a library stream), replayed
 * `reps` times; every rank's slot must arrive. *ok = 1 on success. Collective. KR_ENCCL / KR_ECUDA on failure. */
kr_status krylov_comm_selftest(kr_comm* c, void* stream, int32_t reps, int32_t* ok);

/* Direction sharding (KR_PART_DIRS): the global directions (generator columns of E, then the
 * fixed direction v_f) that rank `rank` of `world` simulates — round robin, d = rank, rank + world,
 * ... — written to HOST dirs[cap], count in *n. Its local direction dl is global direction rank + dl * world;
 * the final gather places local block dl of rank w at global direction w + dl * world. Host only. KR_EINVAL on
 * bad arguments (cap too small included). */
kr_status krylov_dirs_of_rank(int32_t n_dir, int32_t world, int32_t rank, int32_t* dirs, int32_t cap, int32_t* n);

/* Host transport: a communicator whose collectives are all-gathers of HOST buffers performed by the caller's
 * function — fn(ctx, send, recv, bytes) must gather `bytes` bytes from every rank into recv in rank order
 * (recv holds world * bytes; e.g. torch.distributed.all_gather_into_tensor over gloo) and return 0 (non-zero:
 * the library call fails with KR_ENCCL). For several ranks sharing one GPU (NCCL needs one GPU per rank)
 * and for testing the multi-rank path: the per-step scalar all-gather, the halo exchange (an all-gather of
 * each rank's three boundary planes) and the direction-sharding gather are staged through pinned host memory
 * with a stream synchronisation around each; no kernel ever waits on another process; the fixed-k run is
 * not captured into a CUDA graph. The peer-memory halo transport (krylov_ipc_blob ...) works on top of it:
 * the host all-gather that follows every step orders the halo stores. fn is called from the thread that
 * calls krylov_project / krylov_check_box. Collective (every rank, same world).                         */
typedef int32_t (*kr_allgather_fn)(void* ctx, const void* send, void* recv, size_t bytes);
kr_status krylov_comm_create_host(int32_t rank, int32_t world, int32_t device, kr_allgather_fn fn, void* ctx,
                                  kr_comm** out);

/* ---- peer-memory halo transport (NVLink P2P through CUDA IPC; one process per GPU) --------------
 * With it the fused step kernel stores the halo planes of u_{i+1} straight into the neighbouring ranks'
 * state buffers (the compute and the exchange in one kernel), instead of a halo message after each step;
 * the per-step scalar all-gather, which follows every step anyway, orders those stores before any read.
 * Protocol (every rank, in this order, before the first krylov_project; the caller provides the
 * all-gather and the barrier, e.g. torch.distributed):
 *   krylov_ipc_blob(h, blob)                     this rank's export, KR_IPC_BLOB_BYTES bytes (HOST)
 *   all-gather the blobs in rank order          -> blobs [world][KR_IPC_BLOB_BYTES]
 *   krylov_p2p_open(h, blobs, rank, world)       opens the neighbours' buffers, writes a test pattern
 *   barrier
 *   krylov_p2p_verify(h, &ok)                    checks the pattern the neighbours wrote into my halos
 *   all-reduce ok (min) over ranks
 *   krylov_p2p_enable(h, ok_all)                 1: switch to the peer-memory transport; 0: close, keep NCCL
 * Stencil Lanczos path with one slab per rank only (KR_EINVAL otherwise). Collective.              */
#define KR_IPC_BLOB_BYTES 512
kr_status krylov_ipc_blob(kr_handle* h, void* blob);
kr_status krylov_p2p_open(kr_handle* h, const void* blobs, int32_t rank, int32_t world);
kr_status krylov_p2p_verify(kr_handle* h, int32_t* ok);
kr_status krylov_p2p_enable(kr_handle* h, int32_t on);

/* ---- host utilities (no GPU work) --------------------------------------------------------------- */
/* log10 of the a priori Krylov error bound of Eq. 3 for ||v|| = 1: ||At||^k e^{||At||} / k!
 * (the bound the paper shows to be unusable: 10^16182319 at ||At|| = 32771611, k = 10^6).
 * norm_At > 0, k >= 1; returns NaN otherwise. */
double krylov_a_priori_bound_log10(double norm_At, int32_t k);

/* Memory of the Krylov iteration in bytes: method KR_ARNOLDI (or a plain Lanczos storing V), Eq. 4
 * (P:604-607): k (n + k) doubles; KR_LANCZOS with projection (Alg. 4), Eq. 6:
 * (3k + n min(i, o) + 3n) doubles. -1 on bad arguments. (The GPU path's own footprint is
 * krylov_workspace_bytes.) */
int64_t krylov_memory_bytes(int64_t n, int32_t k, int32_t i, int32_t o, int32_t method);

/* z-slab partition of the stencil grid (host logic, no GPU): rank r of world owns global planes
 * [z0, z1). Balanced: the first mz % world ranks own one extra plane. KR_EINVAL if a rank would own
 * fewer than 2 planes (the depth-2 halo comes from one neighbour). */
kr_status krylov_zslab_range(int64_t mz, int32_t world, int32_t rank, int64_t* z0, int64_t* z1);

/* One halo transfer of the z-slab decomposition (host logic, no GPU). Buffer planes of a rank holding
 * nz owned planes: 0 = halo below (global z0-1), 1..nz = owned, nz+1 and nz+2 = halo above (z1, z1+1).
 * The fused step needs u_i at depth 2 above and depth 1 below, u_{i-1} at depth 1 above. */
typedef struct {
    int32_t is_send;   /* 1 = send my planes [plane, plane+nplanes) to peer; 0 = receive into them */
    int32_t peer;      /* neighbouring rank                                                          */
    int64_t plane;     /* first buffer plane (of this rank's buffer)                                  */
    int64_t nplanes;   /* 2 towards the lower neighbour, 1 towards the upper neighbour                */
} kr_halo_op;

/* The exchange schedule of rank `rank` after each Krylov step, in issue order (sends and receives
 * paired as one NCCL group): to rank-1 send planes [1,3) and receive into plane 0; to rank+1 send plane
 * nz and receive into [nz+1, nz+3). ops must hold 4 entries; *n_ops receives the count. */
kr_status krylov_zslab_halo_plan(int64_t mz, int32_t world, int32_t rank, kr_halo_op* ops, int32_t* n_ops);

#ifdef __cplusplus
}
#endif
#endif /* KRYLOV_REACH_H */
