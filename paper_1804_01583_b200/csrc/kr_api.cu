// kr_api.cu — the C ABI of include/krylov_reach.h: validation, device memory, descriptor upload,
// CUDA-graph capture of the hot path, results download. See the header for the contract.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <utility>

#include "kr_internal.h"

namespace {
// KR_TRACE=1: host wall-clock of the create phases on stderr (diagnostics only).
struct PhaseTrace {
    bool on = getenv("KR_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        const auto n = std::chrono::steady_clock::now();
        fprintf(stderr, "[kr trace] %-28s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
        t = n;
    }
};
}  // namespace

static thread_local std::string g_err;
void kr_set_error(const std::string& m) { g_err = m; }

cudaError_t kr_event_record(cudaEvent_t e, cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaError_t r = cudaStreamIsCapturing(s, &cs);
    if (r != cudaSuccess) return r;
    return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal)
                                               : cudaEventRecord(e, s);
}

kr_status kr_comm_unique_id_impl(void* id128);
kr_comm* kr_comm_create_impl(const void* id128, int32_t rank, int32_t world, int32_t device);
void kr_comm_destroy_impl(kr_comm* c);
void kr_comm_selftest_impl(kr_comm* c, cudaStream_t s, int reps, int32_t* ok);
kr_comm* kr_comm_create_host_impl(int32_t rank, int32_t world, int32_t device, kr_allgather_fn fn, void* ctx);
size_t kr_box_cex_bytes();
int kr_lz_occupancy(int TX, int TY);
void kr_lz_prepare(kr_handle* h);
void kr_expm_prepare(kr_handle* h);
void kr_ge_prepare();

namespace {

bool finite(double v) { return std::isfinite(v); }

// an affine term lifts the system: CSR b (dense) or the stencil's compact b_vec
bool has_affine(const kr_problem* p) { return p->b != nullptr || (p->op == KR_OP_STENCIL7 && p->b_vec != nullptr); }

int64_t n_state(const kr_problem* p) { return p->op == KR_OP_STENCIL7 ? p->mx * p->my * p->mz : p->n; }

void validate_vec(const kr_problem* p, const kr_vec& v, const char* what) {
    const int64_t n = n_state(p);
    if (v.kind == KR_VEC_SPARSE) {
        if (v.nnz < 0 || (v.nnz > 0 && (!v.idx || !v.val))) KR_THROW(KR_EINVAL, std::string(what) + ": bad sparse vector");
        for (int64_t e = 0; e < v.nnz; ++e) {
            if (v.idx[e] < 0 || v.idx[e] >= n) KR_THROW(KR_EDIM, std::string(what) + ": index out of range");
            if (!finite(v.val[e])) KR_THROW(KR_ENONFINITE, std::string(what) + ": non-finite value");
        }
    } else if (v.kind == KR_VEC_BOX || v.kind == KR_VEC_ALL || v.kind == KR_VEC_RAND) {
        if (!finite(v.value)) KR_THROW(KR_ENONFINITE, std::string(what) + ": non-finite value");
        if (v.kind == KR_VEC_BOX) {
            const int axes = p->op == KR_OP_STENCIL7 ? 3 : 1;
            const int64_t ext[3] = {p->op == KR_OP_STENCIL7 ? p->mx : p->n, p->my, p->mz};
            for (int a = 0; a < axes; ++a)
                if (v.lo[a] < 0 || v.hi[a] > ext[a] || v.lo[a] > v.hi[a])
                    KR_THROW(KR_EDIM, std::string(what) + ": box out of range");
        }
    } else {
        KR_THROW(KR_EINVAL, std::string(what) + ": bad vector kind");
    }
}

bool vec_is_zero(const kr_problem* p, const kr_vec& v) {
    if (v.kind == KR_VEC_SPARSE) {
        for (int64_t e = 0; e < v.nnz; ++e)
            if (v.val[e] != 0.0) return false;
        return true;
    }
    if (v.value == 0.0) return true;
    if (v.kind == KR_VEC_ALL || v.kind == KR_VEC_RAND) return n_state(p) == 0;
    const int axes = p->op == KR_OP_STENCIL7 ? 3 : 1;
    for (int a = 0; a < axes; ++a)
        if (v.hi[a] <= v.lo[a]) return true;
    return false;
}

// CSR rows with ascending columns and duplicates summed (host, O(nnz log row length)), and its transpose
// by a counting sort (rows of A^T then also have ascending columns).
struct RowsCsr {
    std::vector<int64_t> rp, ci;
    std::vector<double> v;
};

RowsCsr merged_rows(const kr_problem* p) {
    RowsCsr m;
    m.rp.assign((size_t)p->n + 1, 0);
    m.ci.reserve((size_t)p->nnz);
    m.v.reserve((size_t)p->nnz);
    std::vector<std::pair<int64_t, double>> row;
    for (int64_t r = 0; r < p->n; ++r) {
        row.clear();
        for (int64_t e = p->row_ptr[r]; e < p->row_ptr[r + 1]; ++e) row.push_back({p->col_idx[e], p->val[e]});
        if (row.size() > 32) {
            std::stable_sort(row.begin(), row.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        } else {  // stable insertion sort: no temporary buffer for the typical short row
            for (size_t i = 1; i < row.size(); ++i) {
                const auto x = row[i];
                size_t j = i;
                for (; j > 0 && row[j - 1].first > x.first; --j) row[j] = row[j - 1];
                row[j] = x;
            }
        }
        for (size_t i = 0; i < row.size();) {
            size_t j = i;
            double acc = 0.0;
            while (j < row.size() && row[j].first == row[i].first) acc += row[j++].second;
            m.ci.push_back(row[i].first);
            m.v.push_back(acc);
            i = j;
        }
        m.rp[(size_t)r + 1] = (int64_t)m.ci.size();
    }
    return m;
}

RowsCsr transpose_rows(const RowsCsr& a, int64_t n) {
    RowsCsr t;
    t.rp.assign((size_t)n + 1, 0);
    for (int64_t c : a.ci) t.rp[(size_t)c + 1]++;
    for (int64_t r = 0; r < n; ++r) t.rp[(size_t)r + 1] += t.rp[(size_t)r];
    t.ci.resize(a.ci.size());
    t.v.resize(a.v.size());
    std::vector<int64_t> next(t.rp.begin(), t.rp.end() - 1);
    for (int64_t r = 0; r < n; ++r)
        for (int64_t e = a.rp[(size_t)r]; e < a.rp[(size_t)r + 1]; ++e) {
            const int64_t pos = next[(size_t)a.ci[(size_t)e]]++;
            t.ci[(size_t)pos] = r;
            t.v[(size_t)pos] = a.v[(size_t)e];
        }
    return t;
}

bool csr_exactly_symmetric(const kr_problem* p) {
    const RowsCsr a = merged_rows(p);
    const RowsCsr t = transpose_rows(a, p->n);
    return a.rp == t.rp && a.ci == t.ci && a.v == t.v;
}

// Gershgorin upper bound of lambda_max((A+A^T)/2) (Lemma 1's nu(B) = -mu(A), B = -A).
double gershgorin_mu(const kr_problem* p) {
    if (p->op == KR_OP_STENCIL7) {
        const int64_t m[3] = {p->mx, p->my, p->mz};
        double s = 0.0;
        for (int a = 0; a < 3; ++a) {
            const double ih = (double)(m[a] + 1) * (double)(m[a] + 1);
            s += (double)(std::min<int64_t>(2, m[a] - 1) - 2) * ih;
        }
        double mu = p->alpha * s;
        if (p->b_vec) {  // lifted: row r gains |b_r|/2, the lifted row sum_r |b_r|/2
            const kr_vec& v = *p->b_vec;
            double bmax = 0.0, bsum = 0.0;
            if (v.kind == KR_VEC_SPARSE) {
                std::map<int64_t, double> acc;
                for (int64_t e = 0; e < v.nnz; ++e) acc[v.idx[e]] += v.val[e];
                for (auto& kv : acc) {
                    bmax = std::max(bmax, std::fabs(kv.second));
                    bsum += std::fabs(kv.second);
                }
            } else {
                int64_t cnt = p->mx * p->my * p->mz;
                if (v.kind == KR_VEC_BOX)
                    cnt = (v.hi[0] - v.lo[0]) * (v.hi[1] - v.lo[1]) * (v.hi[2] - v.lo[2]);
                bmax = cnt > 0 ? std::fabs(v.value) : 0.0;
                bsum = std::fabs(v.value) * (double)cnt;
            }
            mu = std::max(mu + 0.5 * bmax, 0.5 * bsum);
        }
        return mu;
    }
    // s_rc = (a_rc + a_cr) / 2 over rows with ascending columns and no duplicates (the caller's rows when they
    // already are, else merged copies). Each pair {r, c} is visited once, from its entry with c > r: the mirror
    // a_cr is found by binary search in row c and marked, |s_rc| goes to both radii; entries with c < r whose
    // mirror was not marked (a_cr absent) add |a_rc| / 2 to both. O(nnz log row length), no transpose.
    const int64_t n = p->n, N = n + (p->b ? 1 : 0);
    bool sorted = true;
    for (int64_t r = 0; r < n && sorted; ++r)
        for (int64_t e = p->row_ptr[r] + 1; e < p->row_ptr[r + 1]; ++e)
            if (p->col_idx[e] <= p->col_idx[e - 1]) {
                sorted = false;
                break;
            }
    std::vector<double> diag(N, 0.0), rad(N, 0.0);
    // Row blocks on T host threads (C2: 240k entries, ~2.7 ms on one thread), two phases: (1) the pairs {r, c} from
    // their entry with c > r (mirror found, marked, |s_rc| to both radii), (2) after all marks, the unmarked entries
    // with c < r. Each thread adds into its own radius array; the arrays are summed in thread order (deterministic).
    auto run = [&](const int64_t* rp, const auto* ci, const double* v) {
        const int64_t nnz = rp[n];
        // at most 8 threads, ~16k entries per thread, and T per-thread radius arrays within 256 MB of host memory
        const int T = (int)std::max<int64_t>(1, std::min<int64_t>({8, (int64_t)std::thread::hardware_concurrency(),
                                                                    nnz / 16384, (int64_t(256) << 20) / (8 * N)}));
        std::vector<uint8_t> paired((size_t)nnz, 0);
        std::vector<std::vector<double>> radt((size_t)T, std::vector<double>(N, 0.0));
        auto rows = [&](int t) { return std::make_pair(n * t / T, n * (t + 1) / T); };
        auto phase1 = [&](int t) {
            std::vector<double>& rd = radt[(size_t)t];
            const auto [r0, r1] = rows(t);
            for (int64_t r = r0; r < r1; ++r) {
                for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
                    const int64_t c = ci[e];
                    if (c == r) {
                        diag[(size_t)r] += v[e];  // 0.5 a_rr + 0.5 a_rr
                        continue;
                    }
                    if (c < r) continue;  // phase 2
                    int64_t lo = rp[c], hi = rp[c + 1];  // binary search of column r in row c
                    while (lo < hi) {
                        const int64_t mid = (lo + hi) >> 1;
                        if (ci[mid] < r) lo = mid + 1; else hi = mid;
                    }
                    double s;
                    if (lo < rp[c + 1] && ci[lo] == r) {
                        s = std::fabs(0.5 * v[e] + 0.5 * v[lo]);
                        paired[(size_t)lo] = 1;  // the only writer of this byte (pair {r, c} is visited from r)
                    } else {
                        s = std::fabs(0.5 * v[e]);
                    }
                    rd[(size_t)r] += s;
                    rd[(size_t)c] += s;
                }
                if (p->b && p->b[r] != 0.0) {  // lifted column b and (zero) lifted row: s_{r,n} = s_{n,r} = b_r / 2
                    rd[(size_t)r] += std::fabs(0.5 * p->b[r]);
                    rd[(size_t)n] += std::fabs(0.5 * p->b[r]);
                }
            }
        };
        auto phase2 = [&](int t) {
            std::vector<double>& rd = radt[(size_t)t];
            const auto [r0, r1] = rows(t);
            for (int64_t r = r0; r < r1; ++r)
                for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
                    const int64_t c = ci[e];
                    if (c >= r || paired[(size_t)e]) continue;  // counted from row c
                    const double s = std::fabs(0.5 * v[e]);
                    rd[(size_t)r] += s;
                    rd[(size_t)c] += s;
                }
        };
        for (int ph = 0; ph < 2; ++ph) {
            auto f = [&](int t) {
                if (ph == 0)
                    phase1(t);
                else
                    phase2(t);
            };
            std::vector<std::thread> th;
            int t_next = 1;
            try {  // this may itself run on a helper thread: no exception may escape (threads that fail to start
                   // are run inline below)
                for (; t_next < T; ++t_next) th.emplace_back(f, t_next);
            } catch (...) {
            }
            f(0);
            for (int t = t_next; t < T; ++t) f(t);
            for (auto& x : th) x.join();
        }
        for (int t = 0; t < T; ++t)
            for (int64_t r = 0; r < N; ++r) rad[(size_t)r] += radt[(size_t)t][(size_t)r];
    };
    if (sorted) {
        run(p->row_ptr, p->col_idx, p->val);
    } else {
        const RowsCsr m = merged_rows(p);
        run(m.rp.data(), m.ci.data(), m.v.data());
    }
    double mu = -INFINITY;
    for (int64_t r = 0; r < N; ++r) mu = std::max(mu, diag[r] + rad[r]);
    return mu;
}

// Process-wide cache of device blocks released by destroyed handles, keyed by (device, size class): size
// classes are 256-byte multiples up to 1 MiB and 1 MiB multiples above; at most 1 GiB stays cached (larger
// releases go back to the driver). The cache object is never destroyed (no teardown ordering at exit).
struct DevCache {
    std::mutex mu;
    std::map<std::pair<int, size_t>, std::vector<void*>> free_blocks;
    std::unordered_map<void*, std::pair<int, size_t>> live;
    std::unordered_set<void*> exported;  // blocks exported over CUDA IPC: never recycled (peers may map them)
    size_t cached = 0;
};
DevCache& dev_cache() {
    static DevCache* c = new DevCache();
    return *c;
}
size_t size_class(size_t b) {
    b = std::max<size_t>(b, 256);
    return b <= (size_t(1) << 20) ? (b + 255) & ~size_t(255) : (b + (size_t(1) << 20) - 1) & ~((size_t(1) << 20) - 1);
}
constexpr size_t kCacheCap = size_t(1) << 30;

// Device allocations owned by the handle: requests up to 1 MB are carved (256-byte aligned) from 4 MB
// chunks, larger ones get their own cudaMalloc — a handle makes a few dozen small allocations, and each
// cudaMalloc / cudaFree pair costs tens of microseconds to milliseconds of create / destroy time.
void* dalloc(kr_handle* h, size_t bytes) {
    constexpr size_t kChunk = size_t(4) << 20;
    bytes = (std::max<size_t>(bytes, 8) + 255) & ~size_t(255);
    auto device_alloc = [&](size_t b) {
        void* p = nullptr;
        cudaError_t e = kr_dev_malloc(&p, b);
        if (e != cudaSuccess) KR_THROW(KR_ENOMEM, "cudaMalloc(" + std::to_string(b) + "): " + cudaGetErrorString(e));
        h->extra_allocs.push_back(p);
        return p;
    };
    if (bytes > kChunk / 4) return device_alloc(bytes);
    if (h->arena_used + bytes > h->arena_cap) {
        h->arena = reinterpret_cast<char*>(device_alloc(kChunk));
        h->arena_used = 0;
        h->arena_cap = kChunk;
    }
    void* p = h->arena + h->arena_used;
    h->arena_used += bytes;
    return p;
}

void* carve(kr_handle* h, size_t bytes) {
    const size_t off = (h->ws_used + 255) & ~size_t(255);
    if (off + bytes > h->ws_bytes) KR_THROW(KR_ENOMEM, "workspace too small");
    h->ws_used = off + bytes;
    return h->ws + off;
}

template <class T>
T* upload(kr_handle* h, const T* src, size_t count) {
    T* d = reinterpret_cast<T*>(dalloc(h, count * sizeof(T)));
    // on the handle's (non-blocking) stream: a pageable source is staged before the call returns, and every
    // consumer enqueued later on h->stream is ordered after the copy (a legacy-stream cudaMemcpy is not)
    if (count) {
        if (h->stream)
            KR_CUDA(cudaMemcpyAsync(d, src, count * sizeof(T), cudaMemcpyHostToDevice, h->stream));
        else
            KR_CUDA(cudaMemcpy(d, src, count * sizeof(T), cudaMemcpyHostToDevice));
    }
    h->h2d_bytes += (int64_t)(count * sizeof(T));
    return d;
}

// Sort + merge duplicate sparse entries on the host, upload; box/all copied as is.
DVec make_dvec(kr_handle* h, const kr_vec& v) {
    DVec d{};
    d.kind = v.kind;
    d.value = v.value;
    d.seed = v.seed;
    for (int a = 0; a < 3; ++a) {
        d.lo[a] = v.lo[a];
        d.hi[a] = v.hi[a];
    }
    if (v.kind == KR_VEC_SPARSE) {
        bool sorted = true;  // strictly ascending indices (no duplicates): upload as is
        for (int64_t i = 1; i < v.nnz && sorted; ++i) sorted = v.idx[i] > v.idx[i - 1];
        if (sorted) {
            d.nnz = v.nnz;
            d.idx = upload(h, v.idx, (size_t)v.nnz);
            d.val = upload(h, v.val, (size_t)v.nnz);
            return d;
        }
        std::vector<std::pair<int64_t, double>> e((size_t)v.nnz);
        for (int64_t i = 0; i < v.nnz; ++i) e[i] = {v.idx[i], v.val[i]};
        std::stable_sort(e.begin(), e.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        std::vector<int64_t> idx;
        std::vector<double> val;
        for (size_t i = 0; i < e.size();) {
            size_t j = i;
            double s = 0.0;
            while (j < e.size() && e[j].first == e[i].first) s += e[j++].second;
            idx.push_back(e[i].first);
            val.push_back(s);
            i = j;
        }
        d.nnz = (int64_t)idx.size();
        d.idx = upload(h, idx.data(), idx.size());
        d.val = upload(h, val.data(), val.size());
    }
    return d;
}

struct Sizes {
    int path, method;
    int64_t N;
    int ndl;
    size_t state_bytes;
};

int resolve_method(const kr_problem* p) {
    if (p->method == KR_ARNOLDI || p->method == KR_LANCZOS) return p->method;
    if (p->op == KR_OP_STENCIL7) return p->b_vec ? KR_ARNOLDI : KR_LANCZOS;
    if (!p->b && csr_exactly_symmetric(p)) return KR_LANCZOS;
    return KR_ARNOLDI;
}

int local_dirs(const kr_problem* p, int n_dir, int rank, int world) {
    if (p->part != KR_PART_DIRS || world <= 1) return n_dir;
    int32_t c = 0;
    if (krylov_dirs_of_rank(n_dir, world, rank, nullptr, 0, &c) != KR_OK) KR_THROW(KR_EINVAL, "direction partition");
    return c;
}

void validate(const kr_problem* p) {
    if (!p) KR_THROW(KR_EINVAL, "NULL problem");
    if (p->op != KR_OP_STENCIL7 && p->op != KR_OP_CSR) KR_THROW(KR_EINVAL, "bad op");
    if (p->op == KR_OP_STENCIL7) {
        if (p->mx < 1 || p->my < 1 || p->mz < 1) KR_THROW(KR_EDIM, "stencil grid must be >= 1 per axis");
        if (p->mx > (1 << 30) || p->my > (1 << 30) || p->mz > (1 << 30)) KR_THROW(KR_EDIM, "grid too large");
        if (!finite(p->alpha)) KR_THROW(KR_ENONFINITE, "alpha");
        if (p->b) KR_THROW(KR_EINVAL, "stencil affine term: pass it as b_vec (compact), not b");
        if (p->b_vec) validate_vec(p, *p->b_vec, "b_vec");
    } else {
        if (p->n < 1 || !p->row_ptr || (p->nnz > 0 && (!p->col_idx || !p->val))) KR_THROW(KR_EINVAL, "bad CSR");
        if (p->row_ptr[0] != 0 || p->row_ptr[p->n] != p->nnz) KR_THROW(KR_EDIM, "row_ptr inconsistent with nnz");
        for (int64_t r = 0; r < p->n; ++r)
            if (p->row_ptr[r + 1] < p->row_ptr[r]) KR_THROW(KR_EDIM, "row_ptr not monotone");
        for (int64_t e = 0; e < p->nnz; ++e) {
            if (p->col_idx[e] < 0 || p->col_idx[e] >= p->n) KR_THROW(KR_EDIM, "col_idx out of range");
            if (!finite(p->val[e])) KR_THROW(KR_ENONFINITE, "non-finite matrix value");
        }
        if (p->b_vec) KR_THROW(KR_EINVAL, "b_vec is for the stencil operator; CSR takes a dense b");
        if (p->b)
            for (int64_t r = 0; r < p->n; ++r)
                if (!finite(p->b[r])) KR_THROW(KR_ENONFINITE, "non-finite b");
    }
    if (p->n_gen < 0 || (p->n_gen > 0 && (!p->gen || !p->z_lo || !p->z_hi))) KR_THROW(KR_EINVAL, "bad generators");
    if (p->n_out < 1 || p->n_out > KR_MAX_OUT || !p->out) KR_THROW(KR_EINVAL, "n_out must be 1..64");
    if (!(p->step > 0.0) || !finite(p->step)) KR_THROW(KR_EINVAL, "step must be > 0");
    if (p->n_steps < 0) KR_THROW(KR_EINVAL, "n_steps must be >= 0");
    if (p->method < 0 || p->method > 2) KR_THROW(KR_EINVAL, "bad method");
    {
        const bool stencil_lz = p->op == KR_OP_STENCIL7 && p->method != KR_ARNOLDI && !p->b_vec;
        const int kmax = stencil_lz ? KR_K_MAX : KR_K_MAX_ARNOLDI;
        if (p->k < 1 || p->k > kmax)
            KR_THROW(KR_EINVAL, "k must be 1.." + std::to_string(kmax) + (stencil_lz ? "" : " (Arnoldi / CSR)"));
        if (!(p->eps >= 0.0) || !finite(p->eps)) KR_THROW(KR_EINVAL, "eps must be >= 0");
        if (p->sim_dir < KR_SIM_FORWARD || p->sim_dir > KR_SIM_AUTO) KR_THROW(KR_EINVAL, "bad sim_dir");
        if (p->eps > 0.0 && p->method == KR_LANCZOS && p->op != KR_OP_STENCIL7)
            KR_THROW(KR_EINVAL, "adaptive k (eps > 0): stencil Lanczos (Alg. 4) or Arnoldi (Alg. 2)");
        for (int f = 0; f < 6; ++f) {
            if (p->bc[f] < KR_BC_DIRICHLET || p->bc[f] > KR_BC_ROBIN) KR_THROW(KR_EINVAL, "bad boundary condition");
            if (p->bc[f] != KR_BC_DIRICHLET && p->op != KR_OP_STENCIL7)
                KR_THROW(KR_EINVAL, "boundary conditions apply to the stencil operator only");
            if (p->bc[f] == KR_BC_ROBIN && (!finite(p->gamma[f]) || p->gamma[f] < 0.0))
                KR_THROW(KR_EINVAL, "Robin gamma must be finite and >= 0");
        }
    }
    if (p->part < 0 || p->part > 2) KR_THROW(KR_EINVAL, "bad partition");
    for (int d = 0; d < p->n_gen; ++d) {
        validate_vec(p, p->gen[d], "generator");
        if (!finite(p->z_lo[d]) || !finite(p->z_hi[d])) KR_THROW(KR_ENONFINITE, "z bounds");
        if (p->z_lo[d] > p->z_hi[d]) KR_THROW(KR_EINVAL, "z_lo > z_hi");
        if (vec_is_zero(p, p->gen[d])) KR_THROW(KR_EZERO, "generator " + std::to_string(d) + " is zero");
    }
    if (p->center) validate_vec(p, *p->center, "center");
    if (p->center && !has_affine(p) && vec_is_zero(p, *p->center)) KR_THROW(KR_EZERO, "center is zero (pass NULL)");
    for (int r = 0; r < p->n_out; ++r) validate_vec(p, p->out[r], "output row");
    {  // the seeded dense field: a start vector of forward simulations only (no lifting, no transpose, no rows)
        bool rnd = p->center && p->center->kind == KR_VEC_RAND;
        for (int d = 0; d < p->n_gen; ++d) rnd |= p->gen[d].kind == KR_VEC_RAND;
        for (int r = 0; r < p->n_out; ++r)
            if (p->out[r].kind == KR_VEC_RAND) KR_THROW(KR_EINVAL, "KR_VEC_RAND is not allowed for output rows");
        if (p->b_vec && p->b_vec->kind == KR_VEC_RAND) KR_THROW(KR_EINVAL, "KR_VEC_RAND is not allowed for b_vec");
        if (rnd && (has_affine(p) || p->sim_dir == KR_SIM_TRANSPOSE))
            KR_THROW(KR_EINVAL, "KR_VEC_RAND start vectors need forward simulations without an affine term");
    }
    const int n_dir = p->n_gen + ((p->center || has_affine(p)) ? 1 : 0);
    if (n_dir < 1) KR_THROW(KR_EINVAL, "no directions");
}

Sizes plan(const kr_problem* p, int rank, int world) {
    Sizes s{};
    s.method = resolve_method(p);
    if (s.method == KR_LANCZOS) {
        if (has_affine(p)) KR_THROW(KR_ENOTSYM, "lifted affine system is not symmetric; use Arnoldi");
        if (p->op == KR_OP_CSR && !csr_exactly_symmetric(p)) KR_THROW(KR_ENOTSYM, "CSR matrix is not symmetric");
    }
    s.N = (p->op == KR_OP_STENCIL7 ? p->mx * p->my * p->mz : p->n) + (has_affine(p) ? 1 : 0);
    const int n_dir = p->n_gen + ((p->center || has_affine(p)) ? 1 : 0);
    s.ndl = local_dirs(p, n_dir, rank, world);
    s.path = (p->op == KR_OP_STENCIL7 && s.method == KR_LANCZOS) ? PATH_FUSED_LANCZOS : PATH_GENERIC;
    if (s.path == PATH_GENERIC && (p->part == KR_PART_ZSLAB || p->virtual_slabs > 1))
        KR_THROW(KR_EINVAL, "z-slab partition needs the stencil Lanczos path");
    if (s.path == PATH_FUSED_LANCZOS) {
        const int64_t pitch = (p->mx + 1) & ~int64_t(1);
        int nsl = 1, W = 1, R = 0;
        if (p->part == KR_PART_ZSLAB && world > 1) {
            W = world;
            R = rank;
        } else if (p->virtual_slabs > 1) {
            nsl = p->virtual_slabs;
        }
        size_t b = 0;
        for (int s2 = 0; s2 < nsl; ++s2) {
            int64_t z0, z1;
            if (krylov_zslab_range(p->mz, nsl > 1 ? nsl : W, nsl > 1 ? s2 : R, &z0, &z1) != KR_OK)
                KR_THROW(KR_EINVAL, "each slab needs >= 2 planes");
            b += (size_t)3 * (size_t)(z1 - z0 + 3) * (size_t)p->my * (size_t)pitch * sizeof(double);
        }
        s.state_bytes = b + (size_t)3 * 256 * (size_t)nsl;  // + 256-byte alignment of each carved buffer
    } else {
        if (s.N > KR_ORTHO_ONE_CTA_MAX && s.method == KR_LANCZOS)
            KR_THROW(KR_EINVAL, "stored-basis Lanczos needs operator dimension <= 27648 (use the stencil path or Arnoldi)");
        s.state_bytes = (size_t)s.ndl * (size_t)(p->k + 2) * (size_t)s.N * sizeof(double) + 2 * 256;
    }
    return s;
}

__global__ void reorder_dirs_kernel(const double* g, double* coeff, int64_t np1, int n_out, int n_dir, int world,
                                    int ndl_max) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= np1 * n_out * n_dir) return;
    const int d = (int)(e % n_dir);
    const int64_t jr = e / n_dir;
    const int w = d % world, dl = d / world;
    coeff[e] = g[((int64_t)w * np1 * n_out + jr) * ndl_max + dl];
}

__global__ void pack_stats_kernel(const double* beta0, const double* hnext, const double* lemma, const int32_t* keff,
                                  int ndl, double* out) {
    const int d = threadIdx.x;
    if (d < ndl) {
        out[d * 4 + 0] = beta0[d];
        out[d * 4 + 1] = hnext[d];
        out[d * 4 + 2] = lemma[d];
        out[d * 4 + 3] = (double)keff[d];
    }
}

template <class F>
kr_status guarded(F&& f) {
    try {
        f();
        return KR_OK;
    } catch (const KrError& e) {
        kr_set_error(e.msg);
        return e.st;
    } catch (const std::exception& e) {
        kr_set_error(e.what());
        return KR_EINVAL;
    }
}

int n_dirs_of(const kr_problem* p) { return p->n_gen + ((p->center || has_affine(p)) ? 1 : 0); }

bool transposed_mode(const kr_problem* p) {
    if (p->sim_dir == KR_SIM_TRANSPOSE) return true;
    if (p->center && p->center->kind == KR_VEC_RAND) return false;  // dense seeded start: forward only
    for (int d = 0; d < p->n_gen; ++d)
        if (p->gen[d].kind == KR_VEC_RAND) return false;
    if (p->sim_dir == KR_SIM_AUTO) return p->n_out < n_dirs_of(p);
    return false;
}

// Host storage of the transposed problem (borrowed by create, like the caller's arrays).
struct TransposeStore {
    std::vector<int64_t> rp;
    std::vector<int32_t> ci;
    std::vector<double> val;
    std::vector<kr_vec> gens, outs;
    std::vector<int64_t> fidx;
    std::vector<double> fval, zlo, zhi;
};

// The transpose-dynamics problem of §4.1: simulate x' = A'^T x from each output row C_r^T
// and project with E^T. A'^T of the lifted CSR is built explicitly: A'^T = [[A^T, 0], [b^T, 0]]
// (counting sort by column, rows of A' scanned in order, so each row of A'^T has ascending columns).
// The stencil operator is symmetric (also with insulated / Robin faces) and is kept as is.
void build_transposed(const kr_problem* p, TransposeStore& T, kr_problem& q) {
    q = *p;
    const int nd = n_dirs_of(p);
    if (nd > KR_MAX_OUT) KR_THROW(KR_EINVAL, "transpose mode: at most 64 directions (they become projection rows)");
    if (p->op == KR_OP_STENCIL7 && p->b_vec) KR_THROW(KR_EINVAL, "transpose mode: lifted stencil not supported");
    if (p->eps > 0.0) KR_THROW(KR_EINVAL, "transpose mode is not combined with adaptive k (eps > 0)");
    const bool csr = p->op == KR_OP_CSR;
    const int64_t n = n_state(p);
    const bool lifted = csr && p->b;
    if (csr) {
        const int64_t N = n + (lifted ? 1 : 0);
        T.rp.assign((size_t)N + 1, 0);
        for (int64_t e = 0; e < p->nnz; ++e) T.rp[(size_t)p->col_idx[e] + 1]++;
        if (lifted)
            for (int64_t r = 0; r < n; ++r)
                if (p->b[r] != 0.0) T.rp[(size_t)n + 1]++;
        for (int64_t r = 0; r < N; ++r) T.rp[(size_t)r + 1] += T.rp[(size_t)r];
        T.ci.resize((size_t)T.rp[(size_t)N]);
        T.val.resize((size_t)T.rp[(size_t)N]);
        std::vector<int64_t> next(T.rp.begin(), T.rp.end() - 1);
        for (int64_t r = 0; r < n; ++r) {
            for (int64_t e = p->row_ptr[r]; e < p->row_ptr[r + 1]; ++e) {
                const int64_t pos = next[(size_t)p->col_idx[e]]++;
                T.ci[(size_t)pos] = (int32_t)r;
                T.val[(size_t)pos] = p->val[e];
            }
            if (lifted && p->b[r] != 0.0) {  // A'[r][n] = b_r  ->  A'^T[n][r] = b_r
                const int64_t pos = next[(size_t)n]++;
                T.ci[(size_t)pos] = (int32_t)r;
                T.val[(size_t)pos] = p->b[r];
            }
        }
        q.n = N;
        q.nnz = T.rp[(size_t)N];
        q.row_ptr = T.rp.data();
        q.col_idx = T.ci.data();
        q.val = T.val.data();
        q.b = nullptr;
    }
    auto unlifted = [&](kr_vec v) {  // an ALL vector of the unlifted space stays off the lifted coordinate
        if (lifted && v.kind == KR_VEC_ALL) {
            v.kind = KR_VEC_BOX;
            v.lo[0] = 0;
            v.hi[0] = n;
        }
        return v;
    };
    for (int r = 0; r < p->n_out; ++r) T.gens.push_back(unlifted(p->out[r]));
    T.zlo.assign(p->n_out, 0.0);
    T.zhi.assign(p->n_out, 0.0);
    for (int d = 0; d < p->n_gen; ++d) T.outs.push_back(unlifted(p->gen[d]));
    if (nd > p->n_gen) {  // v_f = [c; 1] (lifted) or c
        if (!lifted) {
            T.outs.push_back(*p->center);
        } else {
            if (p->center) {
                const kr_vec& c = *p->center;
                if (c.kind == KR_VEC_SPARSE) {
                    for (int64_t e = 0; e < c.nnz; ++e) {
                        T.fidx.push_back(c.idx[e]);
                        T.fval.push_back(c.val[e]);
                    }
                } else {
                    const int64_t lo = c.kind == KR_VEC_ALL ? 0 : c.lo[0], hi = c.kind == KR_VEC_ALL ? n : c.hi[0];
                    for (int64_t i = lo; i < hi; ++i) {
                        T.fidx.push_back(i);
                        T.fval.push_back(c.value);
                    }
                }
            }
            T.fidx.push_back(n);
            T.fval.push_back(1.0);
            kr_vec f{};
            f.kind = KR_VEC_SPARSE;
            f.nnz = (int64_t)T.fidx.size();
            f.idx = T.fidx.data();
            f.val = T.fval.data();
            T.outs.push_back(f);
        }
    }
    q.n_gen = p->n_out;
    q.gen = T.gens.data();
    q.z_lo = T.zlo.data();
    q.z_hi = T.zhi.data();
    q.center = nullptr;
    q.n_out = nd;
    q.out = T.outs.data();
    q.sim_dir = KR_SIM_FORWARD;
}

// final layout c[j][r][d] = simulation layout s[j][d][r]
__global__ void transpose_coeff_kernel(const double* sim, double* cf, int64_t np1, int cf_nout, int cf_ndir) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= np1 * cf_nout * cf_ndir) return;
    const int d = (int)(e % cf_ndir);
    const int64_t jr = e / cf_ndir;
    const int r = (int)(jr % cf_nout);
    const int64_t j = jr / cf_nout;
    cf[e] = sim[(j * cf_ndir + d) * cf_nout + r];
}

void free_handle(kr_handle* h) {
    if (!h) return;
    if (h->stream) cudaStreamSynchronize(h->stream);  // the blocks go back to the cache: no work may still use them
    PhaseTrace tr;
    kr_p2p_close(h);
    if (h->graph_ready) cudaGraphExecDestroy(h->gexec);
    tr.mark("destroy: p2p + graph");
    for (auto e : h->ev) cudaEventDestroy(e);
    for (auto e : h->ms_events) cudaEventDestroy(e);
    if (h->h_pin) cudaFreeHost(h->h_pin);
    if (h->ev_it0) cudaEventDestroy(h->ev_it0);
    if (h->ev_it1) cudaEventDestroy(h->ev_it1);
    if (h->ev_lg0) cudaEventDestroy(h->ev_lg0);
    if (h->ev_lg1) cudaEventDestroy(h->ev_lg1);
    if (h->ev_spec) cudaEventDestroy(h->ev_spec);
    if (h->stream2) {
        cudaStreamSynchronize(h->stream2);
        cudaStreamDestroy(h->stream2);
    }
    tr.mark("destroy: events");
    for (void* p : h->extra_allocs) kr_dev_free(p);
    if (h->own_ws && h->ws) kr_dev_free(h->ws);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    tr.mark("destroy: frees");
    delete h;
}

}  // namespace

cudaError_t kr_dev_malloc(void** p, size_t bytes) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const std::pair<int, size_t> key{dev, size_class(bytes)};
    DevCache& c = dev_cache();
    {
        std::lock_guard<std::mutex> lk(c.mu);
        auto it = c.free_blocks.find(key);
        if (it != c.free_blocks.end() && !it->second.empty()) {
            *p = it->second.back();
            it->second.pop_back();
            c.cached -= key.second;
            c.live[*p] = key;
            return cudaSuccess;
        }
    }
    e = cudaMalloc(p, key.second);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(c.mu);
    c.live[*p] = key;
    return cudaSuccess;
}

void kr_dev_free(void* p) {
    if (!p) return;
    DevCache& c = dev_cache();
    {
        std::lock_guard<std::mutex> lk(c.mu);
        auto it = c.live.find(p);
        if (it != c.live.end()) {
            const auto key = it->second;
            c.live.erase(it);
            if (c.exported.erase(p) == 0 && c.cached + key.second <= kCacheCap) {
                c.free_blocks[key].push_back(p);
                c.cached += key.second;
                return;
            }
        }
    }
    cudaFree(p);
}

// A block whose IPC handle was given to peer processes goes straight back to the driver at its free (no reuse
// by a new handle while a peer may still store halo planes into it). No-op for memory the library does not own.
void kr_dev_mark_exported(void* base) {
    DevCache& c = dev_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    if (c.live.count(base)) c.exported.insert(base);
}

extern "C" {

size_t krylov_release_cached_memory(void) {
    DevCache& c = dev_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    size_t released = 0;
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& kv : c.free_blocks) {
        cudaSetDevice(kv.first.first);
        for (void* p : kv.second) {
            cudaFree(p);
            released += kv.first.second;
        }
    }
    cudaSetDevice(cur);
    c.free_blocks.clear();
    c.cached = 0;
    return released;
}

const char* krylov_last_error(void) { return g_err.c_str(); }

kr_status krylov_dirs_of_rank(int32_t n_dir, int32_t world, int32_t rank, int32_t* dirs, int32_t cap, int32_t* n) {
    if (world < 1 || rank < 0 || rank >= world || n_dir < 0 || !n) {
        kr_set_error("krylov_dirs_of_rank: bad arguments");
        return KR_EINVAL;
    }
    int32_t c = 0;
    for (int32_t d = rank; d < n_dir; d += world) {
        if (dirs) {
            if (c >= cap) {
                kr_set_error("krylov_dirs_of_rank: cap too small");
                return KR_EINVAL;
            }
            dirs[c] = d;
        }
        ++c;
    }
    *n = c;
    return KR_OK;
}

kr_status krylov_zslab_range(int64_t mz, int32_t world, int32_t rank, int64_t* z0, int64_t* z1) {
    if (world < 1 || rank < 0 || rank >= world || mz < 1 || !z0 || !z1) {
        kr_set_error("krylov_zslab_range: bad arguments");
        return KR_EINVAL;
    }
    const int64_t base = mz / world, rem = mz % world;
    const int64_t nz = base + (rank < rem ? 1 : 0);
    *z0 = rank * base + std::min<int64_t>(rank, rem);
    *z1 = *z0 + nz;
    if (world > 1 && nz < 2) {
        kr_set_error("krylov_zslab_range: each rank needs >= 2 planes");
        return KR_EINVAL;
    }
    return KR_OK;
}

kr_status krylov_zslab_halo_plan(int64_t mz, int32_t world, int32_t rank, kr_halo_op* ops, int32_t* n_ops) {
    if (!ops || !n_ops) {
        kr_set_error("krylov_zslab_halo_plan: NULL output");
        return KR_EINVAL;
    }
    int64_t z0, z1;
    const kr_status st = krylov_zslab_range(mz, world, rank, &z0, &z1);
    if (st != KR_OK) return st;
    const int64_t nz = z1 - z0;
    int n = 0;
    if (rank > 0) {  // lower neighbour: it needs my first two planes (its depth-2 upper halo)
        ops[n++] = kr_halo_op{1, rank - 1, 1, 2};
        ops[n++] = kr_halo_op{0, rank - 1, 0, 1};
    }
    if (rank + 1 < world) {  // upper neighbour: it needs my last plane (its depth-1 lower halo)
        ops[n++] = kr_halo_op{1, rank + 1, nz, 1};
        ops[n++] = kr_halo_op{0, rank + 1, nz + 1, 2};
    }
    *n_ops = n;
    return KR_OK;
}

kr_status krylov_workspace_bytes(const kr_problem* p, size_t* bytes) {
    return guarded([&] {
        validate(p);
        if (!bytes) KR_THROW(KR_EINVAL, "NULL bytes");
        const int rank = p->comm ? p->comm->rank : 0, world = p->comm ? p->comm->world : 1;
        if (transposed_mode(p)) {
            TransposeStore T;
            kr_problem q;
            build_transposed(p, T, q);
            validate(&q);
            *bytes = plan(&q, rank, world).state_bytes;
        } else {
            *bytes = plan(p, rank, world).state_bytes;
        }
    });
}

kr_status krylov_comm_unique_id(void* id128) {
    if (!id128) return KR_EINVAL;
    return kr_comm_unique_id_impl(id128);
}

kr_status krylov_comm_create(const void* id128, int32_t rank, int32_t world, int32_t device, kr_comm** out) {
    return guarded([&] {
        if (!id128 || !out || world < 1 || rank < 0 || rank >= world) KR_THROW(KR_EINVAL, "bad comm arguments");
        *out = kr_comm_create_impl(id128, rank, world, device);
    });
}

void krylov_comm_destroy(kr_comm* c) { kr_comm_destroy_impl(c); }

kr_status krylov_comm_selftest(kr_comm* c, void* stream, int32_t reps, int32_t* ok) {
    return guarded([&] {
        if (!c || !ok || reps < 1) KR_THROW(KR_EINVAL, "krylov_comm_selftest: bad arguments");
        KR_CUDA(cudaSetDevice(c->device));
        cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
        bool own = false;
        if (!s) {
            KR_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            own = true;
        }
        try {
            kr_comm_selftest_impl(c, s, reps, ok);
        } catch (...) {
            if (own) cudaStreamDestroy(s);
            throw;
        }
        if (own) cudaStreamDestroy(s);
    });
}

kr_status krylov_comm_create_host(int32_t rank, int32_t world, int32_t device, kr_allgather_fn fn, void* ctx,
                                  kr_comm** out) {
    return guarded([&] {
        if (!fn || !out || world < 1 || rank < 0 || rank >= world) KR_THROW(KR_EINVAL, "bad comm arguments");
        *out = kr_comm_create_host_impl(rank, world, device, fn, ctx);
    });
}

static kr_status create_impl(const kr_problem* p, kr_handle** out);

kr_status krylov_reach_create(const kr_problem* p, kr_handle** out) {
    if (!p || !transposed_mode(p)) return create_impl(p, out);
    TransposeStore T;
    kr_problem q;
    kr_status st = guarded([&] {
        PhaseTrace tr;
        validate(p);
        build_transposed(p, T, q);
        tr.mark("transpose lowering");
    });
    if (st != KR_OK) return st;
    st = create_impl(&q, out);
    if (st != KR_OK) return st;
    kr_handle* h = *out;
    st = guarded([&] {  // final layout: the caller's outputs and directions
        h->transposed = true;
        h->cf_nout = p->n_out;
        h->cf_ndir = n_dirs_of(p);
        h->n_gen_cf = p->n_gen;
        h->zlo.clear();
        h->zhi.clear();
        for (int d = 0; d < p->n_gen; ++d) {
            h->zlo.push_back(p->z_lo[d]);
            h->zhi.push_back(p->z_hi[d]);
        }
        if (h->cf_ndir > p->n_gen) {
            h->zlo.push_back(1.0);
            h->zhi.push_back(1.0);
        }
        h->d_zlo = upload(h, h->zlo.data(), h->zlo.size());
        h->d_zhi = upload(h, h->zhi.data(), h->zhi.size());
        const int64_t np1 = h->n_steps + 1;
        h->d_cf = reinterpret_cast<double*>(dalloc(h, (size_t)np1 * h->cf_nout * h->cf_ndir * 8));
        h->d_box = reinterpret_cast<double*>(dalloc(h, (size_t)np1 * h->cf_nout * (8 + 8 + 4) + 16));
        h->d_cex = dalloc(h, 64 + (size_t)h->cf_ndir * 8);
        h->d_sense = reinterpret_cast<int32_t*>(dalloc(h, (size_t)h->cf_nout * 4));
        h->d_thr = reinterpret_cast<double*>(dalloc(h, (size_t)h->cf_nout * 8));
    });
    if (st != KR_OK) {
        free_handle(h);
        *out = nullptr;
    }
    return st;
}

static kr_status create_impl(const kr_problem* p, kr_handle** out) {
    kr_handle* h = nullptr;
    kr_status st = guarded([&] {
        PhaseTrace tr;
        if (!out) KR_THROW(KR_EINVAL, "NULL out");
        *out = nullptr;
        validate(p);
        tr.mark("validate");
        h = new kr_handle();
        h->comm = p->comm;
        h->rank = p->comm ? p->comm->rank : 0;
        h->world = p->comm ? p->comm->world : 1;
        if (p->comm && p->comm->device != p->device) KR_THROW(KR_EINVAL, "comm device != problem device");
        if (p->virtual_slabs > 1 && h->world > 1) KR_THROW(KR_EINVAL, "virtual slabs need world == 1");
        const Sizes sz = plan(p, h->rank, h->world);
        tr.mark("plan");
        h->op = p->op;
        h->method = sz.method;
        h->path = sz.path;
        h->part = p->part;
        h->mx = p->op == KR_OP_STENCIL7 ? p->mx : p->n;
        h->my = p->op == KR_OP_STENCIL7 ? p->my : 1;
        h->mz = p->op == KR_OP_STENCIL7 ? p->mz : 1;
        h->pitch = (h->mx + 1) & ~int64_t(1);
        h->alpha = p->alpha;
        h->gen_bc = false;
        for (int f = 0; f < 6; ++f) {
            h->bc[f] = p->op == KR_OP_STENCIL7 ? p->bc[f] : KR_BC_DIRICHLET;
            h->gamma[f] = h->bc[f] == KR_BC_ROBIN ? p->gamma[f] : 0.0;
            h->gen_bc |= h->bc[f] != KR_BC_DIRICHLET;
        }
        h->eps = p->eps;
        if (p->op == KR_OP_STENCIL7) {
            h->cx = p->alpha * (double)(p->mx + 1) * (double)(p->mx + 1);
            h->cy = p->alpha * (double)(p->my + 1) * (double)(p->my + 1);
            h->cz = p->alpha * (double)(p->mz + 1) * (double)(p->mz + 1);
        }
        h->n = n_state(p);
        h->N = sz.N;
        h->lifted = has_affine(p);
        h->n_gen = p->n_gen;
        h->n_dir = p->n_gen + ((p->center || has_affine(p)) ? 1 : 0);
        h->n_out = p->n_out;
        h->k = p->k;
        h->n_steps = p->n_steps;
        h->step = p->step;
        // Gershgorin mu of a CSR matrix (O(nnz log), 2.6 ms at C2's 240k entries) on a host thread beside the rest
        // of the set-up; joined before create returns (the guard joins on every exit path)
        struct Joiner {
            std::thread t;
            ~Joiner() {
                if (t.joinable()) t.join();
            }
        } mu_job;
        double mu_val = 0.0;
        if (p->op == KR_OP_CSR && p->nnz > 20000)
            mu_job.t = std::thread([&mu_val, p] { mu_val = gershgorin_mu(p); });
        else
            h->mu = gershgorin_mu(p);
        tr.mark("gershgorin mu");
        h->device = p->device;
        KR_CUDA(cudaSetDevice(p->device));
        if (p->stream) {
            h->stream = reinterpret_cast<cudaStream_t>(p->stream);
        } else {
            KR_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
            h->own_stream = true;
        }
        if (p->part == KR_PART_DIRS && h->world > 1) {  // round robin (krylov_dirs_of_rank)
            int32_t cnt = 0;
            krylov_dirs_of_rank(h->n_dir, h->world, h->rank, nullptr, 0, &cnt);
            h->my_dirs.resize((size_t)cnt);
            if (krylov_dirs_of_rank(h->n_dir, h->world, h->rank, h->my_dirs.data(), cnt, &cnt) != KR_OK)
                KR_THROW(KR_EINVAL, "direction partition");
        } else {
            for (int d = 0; d < h->n_dir; ++d) h->my_dirs.push_back(d);
        }
        const int ndl = (int)h->my_dirs.size();
        // directions and box bounds
        for (int d = 0; d < p->n_gen; ++d) {
            h->dirs_h.push_back(make_dvec(h, p->gen[d]));
            h->dir_lift1.push_back(0);
            h->zlo.push_back(p->z_lo[d]);
            h->zhi.push_back(p->z_hi[d]);
        }
        if (h->n_dir > p->n_gen) {
            if (p->center) {
                h->dirs_h.push_back(make_dvec(h, *p->center));
            } else {
                DVec z{};
                z.kind = KR_VEC_ALL;
                z.value = 0.0;
                h->dirs_h.push_back(z);
            }
            h->dir_lift1.push_back(has_affine(p) ? 1 : 0);
            h->zlo.push_back(1.0);
            h->zhi.push_back(1.0);
        }
        for (int r = 0; r < p->n_out; ++r) h->outs_h.push_back(make_dvec(h, p->out[r]));
        h->d_outs = upload(h, h->outs_h.data(), h->outs_h.size());
        h->d_zlo = upload(h, h->zlo.data(), h->zlo.size());
        h->d_zhi = upload(h, h->zhi.data(), h->zhi.size());
        tr.mark("stream + dirs + outs");
        // workspace (state vectors)
        if (p->workspace) {
            if (p->workspace_bytes < sz.state_bytes) KR_THROW(KR_ENOMEM, "caller workspace too small");
            h->ws = reinterpret_cast<char*>(p->workspace);
            h->ws_bytes = p->workspace_bytes;
        } else {
            h->ws_bytes = sz.state_bytes + 256 * 8;
            cudaError_t e = kr_dev_malloc(reinterpret_cast<void**>(&h->ws), h->ws_bytes);
            if (e != cudaSuccess) KR_THROW(KR_ENOMEM, std::string("workspace cudaMalloc: ") + cudaGetErrorString(e));
            h->own_ws = true;
        }
        const int k = h->k;
        const int64_t np1 = h->n_steps + 1;
        h->large_route = h->eps > 0.0 || k > KR_K_MAX_FIXED_PADE;
        h->checks.assign(ndl, {});
        h->d_scratch = reinterpret_cast<double*>(dalloc(h, 64));
        if (!h->large_route || h->path == PATH_GENERIC) {  // dense H: per-step Pade, or Arnoldi's Hessenberg
            h->d_H = reinterpret_cast<double*>(dalloc(h, (size_t)ndl * (k + 1) * k * 8));
            KR_CUDA(cudaMemsetAsync(h->d_H, 0, (size_t)ndl * (k + 1) * k * 8, h->stream));
        }
        h->d_P = reinterpret_cast<double*>(dalloc(h, (size_t)ndl * h->n_out * k * 8));
        h->d_beta0 = reinterpret_cast<double*>(dalloc(h, (size_t)ndl * 8));
        h->d_hnext = reinterpret_cast<double*>(dalloc(h, (size_t)ndl * 8));
        h->d_hmax = reinterpret_cast<double*>(dalloc(h, (size_t)ndl * 8));
        h->d_lemma = reinterpret_cast<double*>(dalloc(h, (size_t)ndl * 8));
        h->d_keff = reinterpret_cast<int32_t*>(dalloc(h, (size_t)ndl * 4));
        h->d_done = reinterpret_cast<int32_t*>(dalloc(h, (size_t)ndl * 4));
        h->d_status = reinterpret_cast<int32_t*>(dalloc(h, (size_t)ndl * 4 + 64));
        KR_CUDA(cudaMemsetAsync(h->d_P, 0, (size_t)ndl * h->n_out * k * 8, h->stream));
        KR_CUDA(cudaMemsetAsync(h->d_hnext, 0, (size_t)ndl * 8, h->stream));
        KR_CUDA(cudaMemsetAsync(h->d_status, 0, (size_t)ndl * 4 + 64, h->stream));
        h->d_coeff = reinterpret_cast<double*>(dalloc(h, (size_t)np1 * h->n_out * h->n_dir * 8));
        h->d_cf = h->d_coeff;
        h->cf_nout = h->n_out;
        h->cf_ndir = h->n_dir;
        h->n_gen_cf = h->n_gen;
        if (p->part == KR_PART_DIRS && h->world > 1) {
            const int ndl_max = (h->n_dir + h->world - 1) / h->world;
            h->d_coeff_loc = reinterpret_cast<double*>(dalloc(h, (size_t)np1 * h->n_out * ndl_max * 8 * h->world));
            h->d_gather = reinterpret_cast<double*>(dalloc(h, (size_t)ndl_max * 4 * 8 * h->world));
        } else {
            h->d_coeff_loc = h->d_coeff;
        }
        h->d_hlast = reinterpret_cast<double*>(dalloc(h, (size_t)ndl * np1 * 8));
        h->d_box = reinterpret_cast<double*>(dalloc(h, (size_t)np1 * h->n_out * (8 + 8 + 4) + 16));
        h->d_cex = dalloc(h, 64 + (size_t)h->n_dir * 8);
        tr.mark("result buffers");
        if (h->path == PATH_FUSED_LANCZOS) {
            // box-kind output rows are reduced inside the fused kernel, sparse rows gathered after it
            std::vector<int32_t> slots;
            for (int r = 0; r < h->n_out; ++r) {
                const kr_vec& o = p->out[r];
                if (o.kind == KR_VEC_SPARSE) continue;
                BoxRow b{};
                if (o.kind == KR_VEC_ALL) {
                    b.lo[0] = b.lo[1] = b.lo[2] = 0;
                    b.hi[0] = (int32_t)h->mx;
                    b.hi[1] = (int32_t)h->my;
                    b.hi[2] = (int32_t)h->mz;
                } else {
                    for (int a = 0; a < 3; ++a) {
                        b.lo[a] = (int32_t)o.lo[a];
                        b.hi[a] = (int32_t)o.hi[a];
                    }
                }
                b.slot = r;
                if (h->boxes.size() >= KR_MAX_BOX) KR_THROW(KR_EINVAL, "at most 8 box/all output rows on the stencil path");
                h->boxes.push_back(b);
                slots.push_back(r);
            }
            // the fused kernel accumulates sum(w) over the box; the row value multiplies in finalize:
            // fold the value into the slot table by scaling in the reduce (value kept in outs_h)
            h->d_box_slot = upload(h, slots.data(), slots.size());
            std::vector<double> bvals;
            for (int32_t r : slots) bvals.push_back(p->out[r].kind == KR_VEC_ALL || p->out[r].kind == KR_VEC_BOX ? p->out[r].value : 1.0);
            h->d_box_val = upload(h, bvals.data(), bvals.size());
            h->nq = 2 + h->n_out;
            h->nqp = 2 + (int)h->boxes.size();
            // tile: 64 x 16 cells (one x-pair per lane, a warp per row pair: 256 threads), 64 x 8 below 64 rows
            h->TX = 64;
            h->TY = h->my >= 64 ? 16 : 8;
            if (const char* e = getenv("KR_TY")) h->TY = atoi(e) == 8 ? 8 : 16;  // diagnostic: tile height
            int nsl = 1, W = h->world, R = h->rank;
            if (p->virtual_slabs > 1) {
                nsl = p->virtual_slabs;
                W = nsl;
            }
            if (p->part != KR_PART_ZSLAB && nsl == 1) {
                W = 1;
                R = 0;
            }
            const int occ = std::max(1, kr_lz_occupancy(h->TX, h->TY));
            int dev_sms = 148;
            KR_CUDA(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, p->device));
            const char* env_zc = getenv("KR_ZCHUNK");
            for (int s = 0; s < nsl; ++s) {
                Slab sl{};
                if (krylov_zslab_range(h->mz, W, nsl > 1 ? s : R, &sl.z0, &sl.z1) != KR_OK)
                    KR_THROW(KR_EINVAL, "each slab needs >= 2 planes");
                sl.nz = sl.z1 - sl.z0;
                const size_t vb = (size_t)(sl.nz + 3) * h->my * h->pitch * sizeof(double);
                // Only the ghost / halo planes need zeros up front (global Dirichlet ghosts; neighbour halos
                // are rewritten every step before they are read, u_1 is written on all planes by the init
                // pass, and every later vector on all owned planes before its first read): 3 planes per
                // buffer instead of the whole 24 GB at C5 (create time 4 ms shorter).
                const size_t pb = (size_t)h->my * h->pitch * sizeof(double);
                for (int b = 0; b < 3; ++b) {
                    sl.u[b] = reinterpret_cast<double*>(carve(h, vb));
                    if (getenv("KR_ZERO_ALL")) {
                        KR_CUDA(cudaMemsetAsync(sl.u[b], 0, vb, h->stream));
                    } else {
                        KR_CUDA(cudaMemsetAsync(sl.u[b], 0, pb, h->stream));
                        KR_CUDA(cudaMemsetAsync(reinterpret_cast<char*>(sl.u[b]) + (size_t)(sl.nz + 1) * pb, 0, 2 * pb,
                                                h->stream));
                    }
                }
                const int64_t gx = (h->mx + h->TX - 1) / h->TX, gy = (h->my + h->TY - 1) / h->TY;
                const int64_t slots_total = (int64_t)dev_sms * occ;
                // z-chunking: enough CTAs for ~full waves; each chunk re-reads 3 halo planes. Chunks of at most
                // 80 planes: many short CTAs keep neighbouring tiles co-resident, so their halo rows are L2 hits
                // (C5, v2 kernel: 143-plane chunks 3.89 ms per step, 72-plane 3.70 ms; profiles/r02_zchunk.txt)
                int best_zc = (int)sl.nz;
                double best_cost = 1e300;
                const int64_t zc_max = 80;
                for (int nzc = 1; nzc <= 256 && nzc <= sl.nz; ++nzc) {
                    const int64_t zc = (sl.nz + nzc - 1) / nzc;
                    if (zc > zc_max && nzc < 256 && nzc < sl.nz) continue;
                    const int64_t nch = (sl.nz + zc - 1) / zc;
                    const int64_t nb = gx * gy * nch;
                    const double waves = (double)nb / (double)slots_total;
                    const double eff = waves / std::ceil(waves);
                    const double cost = (1.0 + 1.5 / (double)zc) / eff;
                    if (cost < best_cost - 1e-9) {
                        best_cost = cost;
                        best_zc = (int)zc;
                    }
                }
                if (env_zc) best_zc = std::max(1, atoi(env_zc));
                sl.zchunk = best_zc;
                // items in windows of the resident CTAs (KR_WIN=0: z-chunk-major order, KR_WIN=n: window n)
                sl.win = (int32_t)slots_total;
                if (const char* e = getenv("KR_WIN")) sl.win = std::max(0, atoi(e));
                const int64_t nch = (sl.nz + sl.zchunk - 1) / sl.zchunk;
                sl.gx = (int32_t)gx;
                sl.gy = (int32_t)gy;
                sl.nitems = gx * gy * nch;
                sl.nblk = sl.nitems;  // one work item per CTA: the block scheduler keeps neighbours co-resident
                sl.grid = dim3((unsigned)sl.nblk, 1, 1);
                const int64_t ngrp = (sl.nblk + 63) / 64;
                sl.partials = reinterpret_cast<double*>(dalloc(h, (size_t)(sl.nblk + ngrp) * h->nqp * 8));
                sl.counter = reinterpret_cast<int32_t*>(dalloc(h, (size_t)(1 + ngrp) * 4));
                KR_CUDA(cudaMemsetAsync(sl.counter, 0, (size_t)(1 + ngrp) * 4, h->stream));
                h->slabs.push_back(sl);
            }
            // virtual slabs: halos are written by the step kernel straight into the sibling slabs (the same
            // code path as NVLink peer memory across processes); KR_HALO_COPY=1 keeps the copy transport
            if (h->slabs.size() > 1 && !getenv("KR_HALO_COPY")) {
                for (size_t si = 0; si < h->slabs.size(); ++si)
                    for (int b = 0; b < 3; ++b) {
                        h->slabs[si].peer_lo[b] = si > 0 ? h->slabs[si - 1].u[b] : nullptr;
                        h->slabs[si].peer_hi[b] = si + 1 < h->slabs.size() ? h->slabs[si + 1].u[b] : nullptr;
                    }
                for (size_t si = 1; si < h->slabs.size(); ++si) h->slabs[si].peer_lo_nz = h->slabs[si - 1].nz;
                h->halo_inkernel = true;
            }
            kr_lz_encode_maps(h);
            kr_lz_setup_compact(h);
            kr_lz_multistep_setup(h);
            if (h->multistep) {  // the multi-step kernel's partials, double-buffered by step parity
                Slab& s0 = h->slabs[0];
                s0.mspart = reinterpret_cast<double*>(dalloc(h, (size_t)2 * h->nqp * h->ms_grid * 8));
            }
            kr_lz_prepare(h);
            const int R_total = (int)h->slabs.size() * kr_zworld(h);
            h->d_rankvec = reinterpret_cast<double*>(dalloc(h, (size_t)R_total * h->nq * 8));
            h->d_sc = reinterpret_cast<LzScalars*>(dalloc(h, (size_t)ndl * sizeof(LzScalars)));
            h->d_lzarr = reinterpret_cast<double*>(dalloc(h, (size_t)ndl * 3 * (k + 2) * 8));
            KR_CUDA(cudaMemsetAsync(h->d_lzarr, 0, (size_t)ndl * 3 * (k + 2) * 8, h->stream));
            {
                std::vector<LzScalars> scs(ndl);
                for (int dl = 0; dl < ndl; ++dl) {
                    std::memset(&scs[dl], 0, sizeof(LzScalars));
                    double* base = h->d_lzarr + (size_t)dl * 3 * (k + 2);
                    scs[dl].alpha = base;
                    scs[dl].beta = base + (k + 2);
                    scs[dl].s = base + 2 * (k + 2);
                }
                KR_CUDA(cudaMemcpyAsync(h->d_sc, scs.data(), (size_t)ndl * sizeof(LzScalars), cudaMemcpyHostToDevice,
                                        h->stream));
                KR_CUDA(cudaStreamSynchronize(h->stream));
            }
            int64_t nloc = 0;
            for (auto& sl : h->slabs) nloc += sl.nz * h->mx * h->my;
            h->step_bytes = 24.0 * (double)nloc;
        } else {
            if (p->op == KR_OP_CSR) {
                h->d_rp = upload(h, p->row_ptr, (size_t)p->n + 1);
                h->d_ci = upload(h, p->col_idx, (size_t)p->nnz);
                h->d_val = upload(h, p->val, (size_t)p->nnz);
                h->d_b = p->b ? upload(h, p->b, (size_t)p->n) : nullptr;
                std::vector<int64_t> lr;
                for (int64_t r = 0; r < p->n; ++r)
                    if (p->row_ptr[r + 1] - p->row_ptr[r] > KR_LONG_ROW) lr.push_back(r);
                h->n_long = (int64_t)lr.size();
                if (h->n_long) h->d_long = upload(h, lr.data(), lr.size());
            }
            kr_ge_prepare();
            {  // the local start vectors for the one-launch fill of kr_ge_enqueue_init
                std::vector<DVec> gd;
                std::vector<int32_t> gl;
                for (int dl = 0; dl < ndl; ++dl) {
                    gd.push_back(h->dirs_h[h->my_dirs[dl]]);
                    gl.push_back(h->dir_lift1[h->my_dirs[dl]]);
                }
                if (ndl > 0) {
                    h->d_gdirs = upload(h, gd.data(), gd.size());
                    h->d_glift = upload(h, gl.data(), gl.size());
                }
            }
            h->d_V = reinterpret_cast<double*>(carve(h, (size_t)ndl * (k + 1) * h->N * 8));
            h->d_W = reinterpret_cast<double*>(carve(h, (size_t)ndl * h->N * 8));
            h->d_O = reinterpret_cast<double*>(dalloc(h, (size_t)h->n_out * h->N * 8));
            int64_t dummy = 0;
            for (int r = 0; r < h->n_out; ++r)
                kr_fill_dense(h->stream, h->d_O + (int64_t)r * h->N, h->N, h->n, h->mx, h->my,
                              h->op == KR_OP_STENCIL7, h->outs_h[r], 0, 1.0, 0, &dummy);
            if (p->op == KR_OP_STENCIL7 && p->b_vec) {  // dense affine term for the lifted stencil apply
                h->d_bl = reinterpret_cast<double*>(dalloc(h, (size_t)h->n * 8));
                const DVec bv = make_dvec(h, *p->b_vec);
                kr_fill_dense(h->stream, h->d_bl, h->n, h->n, h->mx, h->my, true, bv, 0, 1.0, 0, &dummy);
            }
            // CGS2 across the GPU beyond one CTA's reach, and already from 4096 states for Arnoldi, where one
            // CTA per direction serialises j block-wide reductions per step (C2: 8.1 -> 6.1 ms); small systems
            // (C1, the oscillator) keep the one-CTA MGS of Alg. 1. KR_FORCE_CGS=0/1 overrides.
            h->use_cgs = h->N > KR_ORTHO_ONE_CTA_MAX || (h->method == KR_ARNOLDI && h->N >= 4096);
            if (const char* e = getenv("KR_FORCE_CGS")) h->use_cgs = h->N > KR_ORTHO_ONE_CTA_MAX || (atoi(e) != 0 && h->method == KR_ARNOLDI);
            if (h->use_cgs) h->d_cgs = reinterpret_cast<double*>(dalloc(h, kr_cgs_scratch_doubles(h, ndl) * 8));
            KR_CUDA(cudaStreamSynchronize(h->stream));
            // bytes per batched operator launch: A once + X and Y per direction (context only)
            h->step_bytes = (h->op == KR_OP_CSR ? (double)p->nnz * 12.0 + (double)(p->n + 1) * 8.0 : 0.0) +
                            16.0 * (double)h->N * ndl;
        }
        tr.mark("path set-up");
        kr_expm_prepare(h);  // also for the large-k route: its checkpoints with k <= 64 use the powers + march kernels
        tr.mark("expm prepare");
        h->d_sense = reinterpret_cast<int32_t*>(dalloc(h, (size_t)h->n_out * 4));
        h->d_thr = reinterpret_cast<double*>(dalloc(h, (size_t)h->n_out * 8));
        h->timing = true;
        {
            // timed steps: with KR_MAX_EV = c the first min(k, c) steps; for k <= 64 steps 1, 2 and six steps
            // spread over 3..k-1, above (adaptive / large k) steps 1, 2 and every 16th step — event nodes around
            // every step cost ~8 us per step inside the CUDA graph (C3: 1.03 -> 0.70 ms per 40-step run)
            std::vector<int> steps;
            if (const char* e = getenv("KR_MAX_EV")) {
                for (int i = 1; i <= std::min(k, std::max(1, atoi(e))); ++i) steps.push_back(i);
            } else if (k > 64) {  // adaptive / large k: steps 1, 2 and every 16th step from 3 on (clock drifts)
                for (int i = 1; i <= k; i = i < 3 ? i + 1 : i + 16) steps.push_back(i);
            } else {
                for (int i = 1; i <= std::min(k, 2); ++i) steps.push_back(i);
                const int lo = 3, hi = k - 1, ns = 6;
                for (int t = 0; t < ns && hi >= lo; ++t) {
                    const int s = lo + (int)(((int64_t)(hi - lo) * t + (ns - 1) / 2) / (ns - 1));
                    if (steps.back() < s) steps.push_back(s);
                }
            }
            h->ev_pair_of_step.assign((size_t)k + 1, -1);
            h->ev_step_of_pair = steps;
            for (size_t p = 0; p < steps.size(); ++p) h->ev_pair_of_step[(size_t)steps[p]] = (int)p;
            h->ev.resize(2 * steps.size());
        }
        for (auto& e : h->ev) KR_CUDA(cudaEventCreate(&e));
        KR_CUDA(cudaEventCreate(&h->ev_it0));
        KR_CUDA(cudaEventCreate(&h->ev_it1));
        tr.mark("events");
        // all set-up work (zeroing of the state buffers, descriptors) ran on h->stream, which does not
        // synchronise with the legacy default stream: finish it before the handle is used
        KR_CUDA(cudaStreamSynchronize(h->stream));
        if (mu_job.t.joinable()) {
            mu_job.t.join();
            h->mu = mu_val;
        }
        tr.mark("final sync");
        *out = h;
    });
    if (st != KR_OK) free_handle(h);
    return st;
}

kr_status krylov_project(kr_handle* h, double* coeff, kr_dir_stats* stats) {
    return guarded([&] {
        if (!h) KR_THROW(KR_EINVAL, "NULL handle");
        KR_CUDA(cudaSetDevice(h->device));
        const int ndl = (int)h->my_dirs.size();
        const bool dirs_gather = h->part == KR_PART_DIRS && h->world > 1;
        const int ndl_max = dirs_gather ? (h->n_dir + h->world - 1) / h->world : ndl;
        const int64_t np1 = h->n_steps + 1;
        auto post = [&]() {
            if (dirs_gather) {
                double* loc = h->d_coeff_loc + (size_t)h->rank * np1 * h->n_out * ndl_max;
                // expm wrote rank-local slots at the start of d_coeff_loc; move into the rank's block
                if (h->rank != 0)
                    KR_CUDA(cudaMemcpyAsync(loc, h->d_coeff_loc, (size_t)np1 * h->n_out * ndl_max * 8,
                                            cudaMemcpyDeviceToDevice, h->stream));
                kr_nccl_allgather(h->comm, loc, h->d_coeff_loc, (size_t)np1 * h->n_out * ndl_max, h->stream);
                const int64_t tot = np1 * h->n_out * h->n_dir;
                reorder_dirs_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, h->stream>>>(
                    h->d_coeff_loc, h->d_coeff, np1, h->n_out, h->n_dir, h->world, ndl_max);
                KR_CUDA(cudaGetLastError());
                h->launches++;
                pack_stats_kernel<<<1, 256, 0, h->stream>>>(h->d_beta0, h->d_hnext, h->d_lemma, h->d_keff, ndl,
                                                             h->d_gather + (size_t)h->rank * ndl_max * 4);
                KR_CUDA(cudaGetLastError());
                h->launches++;
                kr_nccl_allgather(h->comm, h->d_gather + (size_t)h->rank * ndl_max * 4, h->d_gather,
                                  (size_t)ndl_max * 4, h->stream);
            }
            if (h->transposed) {
                const int64_t tot = np1 * h->cf_nout * h->cf_ndir;
                transpose_coeff_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, h->stream>>>(h->d_coeff, h->d_cf, np1,
                                                                                            h->cf_nout, h->cf_ndir);
                KR_CUDA(cudaGetLastError());
                h->launches++;
            }
        };
        auto enqueue = [&](bool ev) {
            KR_CUDA(kr_event_record(h->ev_it0, h->stream));
            h->ms_ev.clear();  // timed multi-step launches of this enqueue (a captured graph replays them)
            h->ev_rec.assign(h->ev.size() / 2, 0);
            if (h->path == PATH_FUSED_LANCZOS) {
                for (int dl = 0; dl < ndl; ++dl) kr_lz_enqueue_direction(h, dl, ev);
            } else {
                kr_ge_enqueue_direction_set(h);
            }
            KR_CUDA(kr_event_record(h->ev_it1, h->stream));
            kr_expm_enqueue(h);
            post();
        };
        // Large-k route (eps > 0: Alg. 4 with Lemma 1 checkpoints; or fixed k > 64): host-driven, since the
        // number of Krylov steps depends on the bounds. Each checkpoint synchronises once (a few per run).
        auto run_large = [&]() {
            auto read_sc = [&](int dl) {
                LzScalars sc;
                KR_CUDA(cudaMemcpyAsync(&sc, h->d_sc + dl, sizeof(LzScalars), cudaMemcpyDeviceToHost, h->stream));
                KR_CUDA(cudaStreamSynchronize(h->stream));
                return sc;
            };
            h->large_ms = 0.0;
            h->large_evals = 0;
            KR_CUDA(cudaEventRecord(h->ev_it0, h->stream));
            h->ms_ev.clear();
            h->ev_rec.assign(h->ev.size() / 2, 0);
            if (h->path == PATH_GENERIC && h->eps > 0.0) {
                // Alg. 2: all local directions step together (one SpMM per step); each direction is
                // checked at the checkpoints 4, ceil(1.1 k), ... until its Lemma-1 bound is below eps, then
                // stopped (its first kc basis vectors and H entries are final)
                kr_ge_enqueue_init(h);
                std::vector<int> acc(ndl, -1);
                std::vector<int32_t> ke(ndl), dn(ndl), stv(ndl);
                int j = 0, left = ndl;
                auto readback = [&]() {
                    KR_CUDA(cudaMemcpyAsync(ke.data(), h->d_keff, ndl * 4, cudaMemcpyDeviceToHost, h->stream));
                    KR_CUDA(cudaMemcpyAsync(dn.data(), h->d_done, ndl * 4, cudaMemcpyDeviceToHost, h->stream));
                    KR_CUDA(cudaMemcpyAsync(stv.data(), h->d_status, ndl * 4, cudaMemcpyDeviceToHost, h->stream));
                    KR_CUDA(cudaStreamSynchronize(h->stream));
                };
                const int32_t one = 1;
                for (int kc = 4; kc <= h->k && left > 0; kc = (int)std::ceil(1.1 * (double)kc)) {
                    while (j < kc) kr_ge_enqueue_step(h, ++j);
                    readback();
                    for (int dl = 0; dl < ndl; ++dl) {
                        if (acc[dl] >= 0 || stv[dl]) continue;
                        if (dn[dl] && ke[dl] < h->k) {  // exact breakdown: accepted, bound 0
                            kr_large_eval(h, dl, std::max(1, (int)ke[dl]), true, true);
                            acc[dl] = ke[dl];
                            --left;
                            continue;
                        }
                        const double b = kr_large_eval(h, dl, kc, true, false);
                        h->checks[dl].push_back({kc, b});
                        if (b < h->eps) {
                            acc[dl] = kc;
                            --left;
                            KR_CUDA(cudaMemcpyAsync(h->d_done + dl, &one, 4, cudaMemcpyHostToDevice, h->stream));
                        }
                    }
                }
                if (left > 0) {  // k_max reached for some directions
                    while (j < h->k) kr_ge_enqueue_step(h, ++j);
                    readback();
                    for (int dl = 0; dl < ndl; ++dl) {
                        if (acc[dl] >= 0 || stv[dl]) continue;
                        const bool brk = dn[dl] && ke[dl] < h->k;
                        const double b = kr_large_eval(h, dl, std::max(1, (int)ke[dl]), true, brk);
                        if (!brk) h->checks[dl].push_back({ke[dl], b});
                    }
                }
                h->steps_run0 = j;
                KR_CUDA(cudaEventRecord(h->ev_it1, h->stream));
                KR_CUDA(cudaStreamSynchronize(h->stream));
                post();
                return;
            }
            if (h->path == PATH_GENERIC) {  // stored-basis Arnoldi with k > 64: all steps, then the exponentials
                kr_ge_enqueue_direction_set(h);
                KR_CUDA(cudaEventRecord(h->ev_it1, h->stream));
                std::vector<int32_t> ke(ndl), stv(ndl);
                KR_CUDA(cudaMemcpyAsync(ke.data(), h->d_keff, ndl * 4, cudaMemcpyDeviceToHost, h->stream));
                KR_CUDA(cudaMemcpyAsync(stv.data(), h->d_status, ndl * 4, cudaMemcpyDeviceToHost, h->stream));
                KR_CUDA(cudaStreamSynchronize(h->stream));
                h->steps_run0 = ndl > 0 ? ke[0] : 0;
                for (int dl = 0; dl < ndl; ++dl)
                    if (!stv[dl]) kr_large_eval(h, dl, std::max(1, (int)ke[dl]), true, false);
                post();
                return;
            }
            for (int dl = 0; dl < ndl; ++dl) {
                h->checks[dl].clear();
                kr_lz_enqueue_init(h, dl);
                int i = 0, accepted = -1;
                bool failed = false;
                if (h->eps > 0.0) {
                    // checkpoints k = 4, ceil(1.1 k), ... in fp64 (Alg. 2 lines 11-16).
                    // Pipelined: while checkpoint kc is evaluated on a second stream (it reads only alpha_1..kc,
                    // beta_1..kc, which later steps do not touch), the steps up to the next checkpoint already run
                    // on the main stream; if kc is accepted they are discarded (k_eff, h_next reset to kc below).
                    if (!h->stream2) {
                        KR_CUDA(cudaStreamCreateWithFlags(&h->stream2, cudaStreamNonBlocking));
                        KR_CUDA(cudaEventCreateWithFlags(&h->ev_spec, cudaEventDisableTiming));
                    }
                    // only where the steps are latency-bound (slabs up to 2^24 cells): on large grids the step
                    // kernels fill the GPU and concurrent checkpoint GEMMs slow both (paper heat 10^9: 28.9 -> 31.6 s)
                    int64_t ncell = 0;
                    for (const auto& sl : h->slabs) ncell = std::max<int64_t>(ncell, sl.nz * h->mx * h->my);
                    bool pipe = ncell <= (int64_t(1) << 24);
                    if (getenv("KR_NO_SPECULATE")) pipe = false;
                    if (getenv("KR_SPECULATE")) pipe = true;
                    // two cooperative kernels (the multi-step steps and the eigen-solve) run side by side only when
                    // both grids fit the GPU together (the multi-step kernel at one CTA per SM, KR_MS_PIPE=1)
                    // (the multi-step grid at one CTA per SM with KR_MS_PIPE=1, or at two per SM when it leaves >= 8
                    // half-SM slots free for the evaluation, which then runs on those slots only)
                    const bool ms_pipe = h->ms_free_slots >= 8 && !getenv("KR_MS_SEQ");
                    if (h->multistep && !(h->ms_one_per_sm && getenv("KR_MS_PIPE")) && !ms_pipe) pipe = false;
                    bool by_bound = false;
                    int kc = 4;
                    while (kc <= h->k) {
                        if (i < kc) kr_lz_enqueue_steps(h, dl, i + 1, kc, h->timing);
                        i = std::max(i, kc);
                        // sequential schedule: the checkpoint's evaluation is enqueued right behind the steps and
                        // its bound and the scalars come back in one round trip (a breakdown found there discards
                        // the evaluation below); pipelined: the scalars first, the evaluation beside the next steps
                        LzScalars sc;
                        double b_seq = 0.0;
                        if (!pipe || kc >= h->k)
                            b_seq = kr_large_eval(h, dl, kc, true, false, &sc);
                        else
                            sc = read_sc(dl);
                        const bool have_b = !pipe || kc >= h->k;
                        if (sc.status) {
                            failed = true;
                            break;
                        }
                        if (dl == 0) h->steps_run0 = std::min(i, std::max(1, sc.k_eff));
                        if (sc.done && sc.k_eff < h->k) {  // exact breakdown: the approximation is exact
                            kr_large_eval(h, dl, std::max(1, sc.k_eff), true, true);
                            accepted = sc.k_eff;
                            break;
                        }
                        const int kn = (int)std::ceil(1.1 * (double)kc);
                        double b;
                        if (pipe && kn <= h->k) {
                            KR_CUDA(cudaEventRecord(h->ev_spec, h->stream));
                            if (i < kn) kr_lz_enqueue_steps(h, dl, i + 1, kn, h->timing);  // speculative
                            i = std::max(i, kn);
                            std::swap(h->stream, h->stream2);
                            h->tdc_grid_cap = (h->multistep && !h->ms_one_per_sm) ? h->ms_free_slots : 0;
                            try {
                                KR_CUDA(cudaStreamWaitEvent(h->stream, h->ev_spec, 0));
                                b = kr_large_eval(h, dl, kc, true, false);
                            } catch (...) {
                                h->tdc_grid_cap = 0;
                                std::swap(h->stream, h->stream2);
                                throw;
                            }
                            h->tdc_grid_cap = 0;
                            std::swap(h->stream, h->stream2);
                        } else {
                            b = have_b ? b_seq : kr_large_eval(h, dl, kc, true, false);
                        }
                        h->checks[dl].push_back({kc, b});
                        if (b < h->eps) {
                            accepted = kc;
                            by_bound = true;
                            break;
                        }
                        kc = kn;
                    }
                    if (by_bound && i > accepted) {  // speculative steps past the accepted checkpoint
                        // the direction's state becomes that of the sequential schedule stopped at kc: k_eff = kc,
                        // h_next = beta_kc, done; a status (non-finite) set by a discarded step is dropped with it
                        // (a status of the steps up to kc was caught by read_sc before the evaluation)
                        LzScalars sc = read_sc(dl);
                        const int32_t ka = accepted;
                        double hn = 0.0;
                        KR_CUDA(cudaMemcpy(&hn, h->d_lzarr + (size_t)dl * 3 * (h->k + 2) + (h->k + 2) + ka, 8,
                                           cudaMemcpyDeviceToHost));
                        sc.status = 0;
                        sc.done = 1;
                        sc.k_eff = ka;
                        sc.h_next = hn;
                        KR_CUDA(cudaMemcpyAsync(h->d_sc + dl, &sc, sizeof(LzScalars), cudaMemcpyHostToDevice, h->stream));
                        KR_CUDA(cudaMemcpyAsync(h->d_keff + dl, &ka, 4, cudaMemcpyHostToDevice, h->stream));
                        KR_CUDA(cudaMemcpyAsync(h->d_hnext + dl, &hn, 8, cudaMemcpyHostToDevice, h->stream));
                        KR_CUDA(cudaStreamSynchronize(h->stream));
                        if (dl == 0) h->steps_run0 = i;
                    }
                }
                if (accepted < 0 && !failed) {  // fixed k, or k_max reached without meeting eps
                    if (i < h->k) kr_lz_enqueue_steps(h, dl, i + 1, h->k, h->timing);
                    i = std::max(i, h->k);
                    if (dl == 0) h->steps_run0 = i;
                    const LzScalars sc = read_sc(dl);
                    if (!sc.status) {
                        const int ke = std::max(1, sc.k_eff);
                        const bool brk = h->eps > 0.0 && sc.done && sc.k_eff < h->k;
                        const double b = kr_large_eval(h, dl, ke, true, brk);
                        if (h->eps > 0.0 && !brk) h->checks[dl].push_back({ke, b});
                    }
                }
            }
            KR_CUDA(cudaEventRecord(h->ev_it1, h->stream));
            post();
        };
        // host transport: its collectives synchronise the stream on the host (no stream capture)
        const bool use_graph = getenv("KR_NO_GRAPH") == nullptr && !h->large_route && !kr_comm_is_host(h->comm);
        if (h->large_route) {
            run_large();
        } else if (use_graph && !h->graph_ready) {
            const int64_t before = h->launches;
            cudaGraph_t g;
            KR_CUDA(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
            try {
                enqueue(h->timing);
            } catch (...) {
                cudaStreamEndCapture(h->stream, &g);
                throw;
            }
            KR_CUDA(cudaStreamEndCapture(h->stream, &g));
            KR_CUDA(cudaGraphInstantiate(&h->gexec, g, 0));
            KR_CUDA(cudaGraphDestroy(g));
            h->graph_launches = h->launches - before;
            h->launches = before;
            h->graph_ready = true;
        }
        if (h->large_route) {
        } else if (use_graph) {
            KR_CUDA(cudaGraphLaunch(h->gexec, h->stream));
            h->launches += h->graph_launches;
        } else {
            enqueue(h->timing);
        }
        KR_CUDA(cudaStreamSynchronize(h->stream));
        if (h->world > 1) kr_nccl_check(h->comm);
        // device-side status (zero direction / non-finite)
        int32_t worst = 0;
        if (h->path == PATH_FUSED_LANCZOS) {
            std::vector<LzScalars> sc(ndl);
            KR_CUDA(cudaMemcpy(sc.data(), h->d_sc, ndl * sizeof(LzScalars), cudaMemcpyDeviceToHost));
            for (auto& s : sc)
                if (s.status) worst = s.status;
        } else {
            std::vector<int32_t> stv(ndl);
            KR_CUDA(cudaMemcpy(stv.data(), h->d_status, ndl * 4, cudaMemcpyDeviceToHost));
            for (auto s : stv)
                if (s) worst = s;
        }
        if (worst) KR_THROW((kr_status)worst, worst == KR_EZERO ? "zero direction vector" : "non-finite value in iteration");
        if (h->timing) {
            float ms = 0.f;
            KR_CUDA(cudaEventElapsedTime(&ms, h->ev_it0, h->ev_it1));
            h->last_iter_ms = ms;
            double tot = 0.0;
            int64_t cnt = 0;
            int keff0 = h->k;
            if (ndl > 0) KR_CUDA(cudaMemcpy(&keff0, h->d_keff, 4, cudaMemcpyDeviceToHost));
            if (h->large_route) keff0 = h->steps_run0;  // Lanczos steps enqueued for direction 0
            const int nrun = std::min(h->k, std::max(1, keff0));  // steps enqueued for direction 0 this run
            FILE* trace = nullptr;
            if (const char* tp = getenv("KR_STEP_TRACE")) trace = fopen(tp, "w");  // diagnostics: per-step ms
            h->step_ms.assign((size_t)nrun, NAN);  // NaN: step not timed
            for (size_t p = 0; p < h->ev_step_of_pair.size(); ++p) {
                const int s = h->ev_step_of_pair[p];
                if (s > nrun) break;
                if (p >= h->ev_rec.size() || !h->ev_rec[p]) continue;  // ran inside a multi-step launch
                float t = 0.f;
                KR_CUDA(cudaEventElapsedTime(&t, h->ev[2 * p], h->ev[2 * p + 1]));
                tot += t;
                cnt++;
                h->step_ms[(size_t)s - 1] = t;
                if (trace) {
                    float g = 0.f;
                    if (p + 1 < h->ev_step_of_pair.size() && h->ev_step_of_pair[p + 1] == s + 1 && s + 1 <= nrun)
                        KR_CUDA(cudaEventElapsedTime(&g, h->ev[2 * p], h->ev[2 * p + 2]));
                    fprintf(trace, "%d %.6f %.6f\n", s, t, g);
                }
            }
            if (trace) fclose(trace);
            // multi-step launches: their time spread evenly over the steps they ran (steps past k_eff exit at once)
            for (const auto& pe : h->ms_ev) {
                float t = 0.f;
                KR_CUDA(cudaEventElapsedTime(&t, h->ms_events[2 * pe.pair], h->ms_events[2 * pe.pair + 1]));
                const int n = std::min(pe.n, nrun - pe.i0 + 1);
                if (n <= 0) continue;
                const double per = (double)t / pe.n;
                for (int s = pe.i0; s < pe.i0 + n; ++s) h->step_ms[(size_t)s - 1] = per;
                tot += per * n;
                cnt += n;
            }
            h->last_step_ms_mean = cnt ? tot / cnt : 0.0;
            h->last_step_launches = (int64_t)nrun * (h->path == PATH_FUSED_LANCZOS ? (int64_t)h->slabs.size() : 1);
        }
        if (coeff) {
            KR_CUDA(cudaMemcpy(coeff, h->d_cf, (size_t)np1 * h->cf_nout * h->cf_ndir * 8, cudaMemcpyDeviceToHost));
            h->d2h_bytes += (int64_t)np1 * h->cf_nout * h->cf_ndir * 8;
        }
        if (stats) h->d2h_bytes += (int64_t)ndl * 28;
        if (stats) {
            if (dirs_gather) {
                std::vector<double> g((size_t)ndl_max * 4 * h->world);
                KR_CUDA(cudaMemcpy(g.data(), h->d_gather, g.size() * 8, cudaMemcpyDeviceToHost));
                for (int d = 0; d < h->n_dir; ++d) {
                    const int w = d % h->world, dl = d / h->world;
                    const double* s = &g[((size_t)w * ndl_max + dl) * 4];
                    stats[d].beta0 = s[0];
                    stats[d].h_next = s[1];
                    stats[d].lemma1_bound = s[2];
                    stats[d].k_eff = (int32_t)s[3];
                }
            } else {
                std::vector<double> b0(ndl), hn(ndl), lm(ndl);
                std::vector<int32_t> ke(ndl);
                KR_CUDA(cudaMemcpy(b0.data(), h->d_beta0, ndl * 8, cudaMemcpyDeviceToHost));
                KR_CUDA(cudaMemcpy(hn.data(), h->d_hnext, ndl * 8, cudaMemcpyDeviceToHost));
                KR_CUDA(cudaMemcpy(lm.data(), h->d_lemma, ndl * 8, cudaMemcpyDeviceToHost));
                KR_CUDA(cudaMemcpy(ke.data(), h->d_keff, ndl * 4, cudaMemcpyDeviceToHost));
                for (int dl = 0; dl < ndl; ++dl) {
                    const int d = h->my_dirs[dl];
                    stats[d].beta0 = b0[dl];
                    stats[d].h_next = hn[dl];
                    stats[d].lemma1_bound = lm[dl];
                    stats[d].k_eff = ke[dl];
                }
            }
        }
        h->projected = true;
    });
}

kr_status krylov_check_box(kr_handle* h, const int32_t* sense, const double* thr, double* lo, double* hi,
                           kr_cex* cex, double* z_witness) {
    return guarded([&] {
        if (!h || !sense || !thr || !cex) KR_THROW(KR_EINVAL, "NULL argument");
        if (!h->projected) KR_THROW(KR_ESTATE, "krylov_check_box before krylov_project");
        for (int r = 0; r < h->cf_nout; ++r) {
            if (sense[r] < 0 || sense[r] > KR_NONE) KR_THROW(KR_EINVAL, "bad sense");
            if (sense[r] != KR_NONE && !std::isfinite(thr[r])) KR_THROW(KR_ENONFINITE, "non-finite threshold");
        }
        KR_CUDA(cudaSetDevice(h->device));
        const int64_t np1 = h->n_steps + 1;
        const int64_t total = np1 * h->cf_nout;
        int32_t* ds = h->d_sense;
        double* dt = h->d_thr;
        KR_CUDA(cudaMemcpyAsync(ds, sense, (size_t)h->cf_nout * 4, cudaMemcpyHostToDevice, h->stream));
        KR_CUDA(cudaMemcpyAsync(dt, thr, (size_t)h->cf_nout * 8, cudaMemcpyHostToDevice, h->stream));
        h->h2d_bytes += (int64_t)h->cf_nout * 12;
        kr_box_enqueue(h, ds, dt);
        h->d2h_bytes += (lo ? total * 8 : 0) + (hi ? total * 8 : 0) + 32 + (int64_t)h->cf_ndir * 8;
        if (lo) KR_CUDA(cudaMemcpyAsync(lo, h->d_box, total * 8, cudaMemcpyDeviceToHost, h->stream));
        if (hi) KR_CUDA(cudaMemcpyAsync(hi, h->d_box + total, total * 8, cudaMemcpyDeviceToHost, h->stream));
        struct {
            int32_t found;
            int64_t step;
            int32_t row;
            double y;
        } dc;
        static_assert(sizeof(dc) <= 64, "cex");
        KR_CUDA(cudaMemcpyAsync(&dc, h->d_cex, sizeof(dc), cudaMemcpyDeviceToHost, h->stream));
        std::vector<double> zw(h->cf_ndir);
        KR_CUDA(cudaMemcpyAsync(zw.data(), reinterpret_cast<char*>(h->d_cex) + 64, (size_t)h->cf_ndir * 8,
                                cudaMemcpyDeviceToHost, h->stream));
        KR_CUDA(cudaStreamSynchronize(h->stream));
        cex->found = dc.found;
        cex->step = dc.step;
        cex->row = dc.row;
        cex->y = dc.y;
        cex->time = dc.found ? (double)dc.step * h->step : 0.0;
        if (z_witness)
            for (int d = 0; d < h->cf_ndir; ++d) z_witness[d] = zw[d];
    });
}

void krylov_reach_destroy(kr_handle* h) {
    if (!h) return;
    cudaSetDevice(h->device);
    cudaStreamSynchronize(h->stream);
    free_handle(h);
}

kr_status krylov_krylov_data(const kr_handle* h, int32_t dir, double* H, double* P) {
    return guarded([&] {
        if (!h) KR_THROW(KR_EINVAL, "NULL handle");
        if (!h->projected) KR_THROW(KR_ESTATE, "krylov_krylov_data before krylov_project");
        int dl = -1;
        for (size_t i = 0; i < h->my_dirs.size(); ++i)
            if (h->my_dirs[i] == dir) dl = (int)i;
        if (dl < 0) KR_THROW(KR_EDIM, "direction not handled by this rank");
        const int k = h->k;
        if (H && h->d_H) {
            KR_CUDA(cudaMemcpy(H, h->d_H + (size_t)dl * (k + 1) * k, (size_t)(k + 1) * k * 8, cudaMemcpyDeviceToHost));
        } else if (H) {  // large-k route keeps H tridiagonal (Eq. 6): expand alpha / beta
            LzScalars sc;
            KR_CUDA(cudaMemcpy(&sc, h->d_sc + dl, sizeof(LzScalars), cudaMemcpyDeviceToHost));
            int ke = 0;
            KR_CUDA(cudaMemcpy(&ke, h->d_keff + dl, 4, cudaMemcpyDeviceToHost));
            std::vector<double> al(k + 2), be(k + 2);
            KR_CUDA(cudaMemcpy(al.data(), sc.alpha, (size_t)(k + 2) * 8, cudaMemcpyDeviceToHost));
            KR_CUDA(cudaMemcpy(be.data(), sc.beta, (size_t)(k + 2) * 8, cudaMemcpyDeviceToHost));
            std::memset(H, 0, (size_t)(k + 1) * k * 8);
            for (int i = 0; i < ke; ++i) {
                H[(size_t)i * k + i] = al[i + 1];
                H[(size_t)(i + 1) * k + i] = be[i + 1];
                if (i + 1 < ke) H[(size_t)i * k + i + 1] = be[i + 1];
            }
        }
        if (P) KR_CUDA(cudaMemcpy(P, h->d_P + (size_t)dl * h->n_out * k, (size_t)h->n_out * k * 8, cudaMemcpyDeviceToHost));
    });
}

kr_status krylov_tridiag(const kr_handle* h, int32_t dir, double* alpha, double* beta, int32_t cap, int32_t* k_eff) {
    return guarded([&] {
        if (!h || !k_eff || cap < 0) KR_THROW(KR_EINVAL, "bad arguments");
        if (h->path != PATH_FUSED_LANCZOS) KR_THROW(KR_EINVAL, "krylov_tridiag: stencil Lanczos path only");
        if (!h->projected) KR_THROW(KR_ESTATE, "krylov_tridiag before krylov_project");
        int dl = -1;
        for (size_t i = 0; i < h->my_dirs.size(); ++i)
            if (h->my_dirs[i] == dir) dl = (int)i;
        if (dl < 0) KR_THROW(KR_EDIM, "direction not handled by this rank");
        int ke = 0;
        KR_CUDA(cudaMemcpy(&ke, h->d_keff + dl, 4, cudaMemcpyDeviceToHost));
        *k_eff = ke;
        LzScalars sc;
        KR_CUDA(cudaMemcpy(&sc, h->d_sc + dl, sizeof(LzScalars), cudaMemcpyDeviceToHost));
        const int n = std::min(ke, cap);
        if (alpha && n > 0) KR_CUDA(cudaMemcpy(alpha, sc.alpha + 1, (size_t)n * 8, cudaMemcpyDeviceToHost));
        if (beta && n > 0) KR_CUDA(cudaMemcpy(beta, sc.beta + 1, (size_t)n * 8, cudaMemcpyDeviceToHost));
    });
}

kr_status krylov_adaptive_checks(const kr_handle* h, int32_t dir, int32_t* ks, double* bounds, int32_t cap,
                                 int32_t* n) {
    return guarded([&] {
        if (!h || !n || cap < 0) KR_THROW(KR_EINVAL, "bad arguments");
        if (!h->projected) KR_THROW(KR_ESTATE, "krylov_adaptive_checks before krylov_project");
        int dl = -1;
        for (size_t i = 0; i < h->my_dirs.size(); ++i)
            if (h->my_dirs[i] == dir) dl = (int)i;
        if (dl < 0) KR_THROW(KR_EDIM, "direction not handled by this rank");
        const auto& c = h->checks[dl];
        *n = (int32_t)c.size();
        for (int i = 0; i < (int)c.size() && i < cap; ++i) {
            if (ks) ks[i] = c[i].first;
            if (bounds) bounds[i] = c[i].second;
        }
    });
}

kr_status krylov_last_timing_large(const kr_handle* h, double* expm_ms, int32_t* n_evals) {
    if (!h) return KR_EINVAL;
    if (expm_ms) *expm_ms = h->large_ms;
    if (n_evals) *n_evals = h->large_evals;
    return KR_OK;
}

kr_status krylov_check_lp(kr_handle* h, int32_t m_init, const double* init_A, const double* init_b, int32_t m_unsafe,
                          const double* unsafe_A, const double* unsafe_b, int32_t* feasible, kr_cex* cex,
                          double* z_witness, double* y_witness) {
    return guarded([&] {
        if (!h || !cex || m_init < 0 || m_unsafe < 0) KR_THROW(KR_EINVAL, "bad arguments");
        if (!h->projected) KR_THROW(KR_ESTATE, "krylov_check_lp before krylov_project");
        const int ng = h->n_gen_cf, o = h->cf_nout;
        if ((m_init > 0 && (!init_A || !init_b)) || (m_unsafe > 0 && (!unsafe_A || !unsafe_b)))
            KR_THROW(KR_EINVAL, "NULL constraint block");
        for (int64_t e = 0; e < (int64_t)m_init * ng; ++e)
            if (!std::isfinite(init_A[e])) KR_THROW(KR_ENONFINITE, "init_A");
        for (int r = 0; r < m_init; ++r)
            if (!std::isfinite(init_b[r])) KR_THROW(KR_ENONFINITE, "init_b");
        for (int64_t e = 0; e < (int64_t)m_unsafe * o; ++e)
            if (!std::isfinite(unsafe_A[e])) KR_THROW(KR_ENONFINITE, "unsafe_A");
        for (int r = 0; r < m_unsafe; ++r)
            if (!std::isfinite(unsafe_b[r])) KR_THROW(KR_ENONFINITE, "unsafe_b");
        KR_CUDA(cudaSetDevice(h->device));
        std::vector<double> out((size_t)2 + h->cf_ndir + o);
        kr_lp_run(h, m_init, init_A, init_b, m_unsafe, unsafe_A, unsafe_b, feasible, out.data());
        cex->found = out[0] != 0.0;
        cex->step = (int64_t)out[1];
        cex->time = cex->found ? (double)cex->step * h->step : 0.0;
        cex->row = -1;
        cex->y = cex->found ? out[(size_t)2 + h->cf_ndir] : 0.0;
        if (cex->found) {
            if (z_witness)
                for (int d = 0; d < h->cf_ndir; ++d) z_witness[d] = out[(size_t)2 + d];
            if (y_witness)
                for (int q = 0; q < o; ++q) y_witness[q] = out[(size_t)2 + h->cf_ndir + q];
        }
    });
}

kr_status krylov_eval_outputs(kr_handle* h, int64_t step, const double* z, double* y) {
    return guarded([&] {
        if (!h || !z || !y) KR_THROW(KR_EINVAL, "NULL argument");
        if (!h->projected) KR_THROW(KR_ESTATE, "krylov_eval_outputs before krylov_project");
        if (step < 0 || step > h->n_steps) KR_THROW(KR_EDIM, "step out of range");
        for (int d = 0; d < h->cf_ndir; ++d)
            if (!std::isfinite(z[d])) KR_THROW(KR_ENONFINITE, "z");
        KR_CUDA(cudaSetDevice(h->device));
        kr_eval_outputs(h, step, z, y);
    });
}

kr_status krylov_ipc_blob(kr_handle* h, void* blob) {
    return guarded([&] {
        if (!h || !blob) KR_THROW(KR_EINVAL, "NULL argument");
        KR_CUDA(cudaSetDevice(h->device));
        kr_p2p_blob(h, blob);
    });
}

kr_status krylov_p2p_open(kr_handle* h, const void* blobs, int32_t rank, int32_t world) {
    return guarded([&] {
        if (!h || !blobs) KR_THROW(KR_EINVAL, "NULL argument");
        KR_CUDA(cudaSetDevice(h->device));
        kr_p2p_open(h, blobs, rank, world);
    });
}

kr_status krylov_p2p_verify(kr_handle* h, int32_t* ok) {
    return guarded([&] {
        if (!h || !ok) KR_THROW(KR_EINVAL, "NULL argument");
        KR_CUDA(cudaSetDevice(h->device));
        kr_p2p_verify(h, ok);
    });
}

kr_status krylov_p2p_enable(kr_handle* h, int32_t on) {
    return guarded([&] {
        if (!h) KR_THROW(KR_EINVAL, "NULL handle");
        KR_CUDA(cudaSetDevice(h->device));
        if (h->graph_ready) {  // kernel arguments change: recapture at the next project
            KR_CUDA(cudaGraphExecDestroy(h->gexec));
            h->graph_ready = false;
        }
        if (on) {
            if (!h->p2p_base[0] && !h->p2p_base[1] && h->p2p_world > 1)
                KR_THROW(KR_ESTATE, "krylov_p2p_enable before krylov_p2p_open");
            h->p2p = h->halo_inkernel = h->p2p_world > 1;
        } else {
            kr_p2p_close(h);
            h->p2p = h->halo_inkernel = false;
        }
    });
}

double krylov_a_priori_bound_log10(double norm_At, int32_t k) {
    if (!(norm_At > 0.0) || !std::isfinite(norm_At) || k < 1) return NAN;
    // log10(x^k e^x / k!) = k log10 x + x / ln 10 - lgamma(k + 1) / ln 10
    const double ln10 = std::log(10.0);
    return (double)k * std::log10(norm_At) + norm_At / ln10 - std::lgamma((double)k + 1.0) / ln10;
}

int64_t krylov_memory_bytes(int64_t n, int32_t k, int32_t i, int32_t o, int32_t method) {
    if (n < 1 || k < 1 || i < 1 || o < 1) return -1;
    if (method == KR_LANCZOS) return (3 * (int64_t)k + n * (int64_t)std::min(i, o) + 3 * n) * 8;
    return (int64_t)k * (n + (int64_t)k) * 8;
}

kr_status krylov_step_times(const kr_handle* h, double* ms, int32_t cap, int32_t* n) {
    if (!h || !n || cap < 0) return KR_EINVAL;
    *n = (int32_t)h->step_ms.size();
    for (int i = 0; i < (int)h->step_ms.size() && i < cap; ++i)
        if (ms) ms[i] = h->step_ms[(size_t)i];
    return KR_OK;
}

kr_status krylov_sim_info(const kr_handle* h, int32_t* transposed, int32_t* n_sim) {
    if (!h) return KR_EINVAL;
    if (transposed) *transposed = h->transposed ? 1 : 0;
    if (n_sim) *n_sim = h->n_dir;
    return KR_OK;
}

int64_t krylov_launch_count(const kr_handle* h) { return h ? h->launches : 0; }

kr_status krylov_transfer_bytes(const kr_handle* h, int64_t* h2d, int64_t* d2h) {
    if (!h) return KR_EINVAL;
    if (h2d) *h2d = h->h2d_bytes;
    if (d2h) *d2h = h->d2h_bytes;
    return KR_OK;
}

kr_status krylov_last_timing(const kr_handle* h, double* iter_ms, double* step_kernel_ms_mean,
                             int64_t* step_kernel_launches, double* step_kernel_bytes) {
    if (!h) return KR_EINVAL;
    if (iter_ms) *iter_ms = h->last_iter_ms;
    if (step_kernel_ms_mean) *step_kernel_ms_mean = h->last_step_ms_mean;
    if (step_kernel_launches) *step_kernel_launches = h->last_step_launches;
    if (step_kernel_bytes) *step_kernel_bytes = h->step_bytes;
    return KR_OK;
}

}  // extern "C"
