"""Thin Python binding over the C ABI (include/krylov_reach.h). Same names as the ABI; argument
marshalling only. Problems are the dicts of workloads/ (see its docstring)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi as A

_METHOD = {"auto": A.KR_AUTO, "arnoldi": A.KR_ARNOLDI, "lanczos": A.KR_LANCZOS}
_PART = {None: A.KR_PART_NONE, "none": A.KR_PART_NONE, "zslab": A.KR_PART_ZSLAB, "dirs": A.KR_PART_DIRS}
_KIND = {"sparse": A.KR_VEC_SPARSE, "box": A.KR_VEC_BOX, "all": A.KR_VEC_ALL, "rand": A.KR_VEC_RAND}
_SIM = {None: A.KR_SIM_FORWARD, "forward": A.KR_SIM_FORWARD, "transpose": A.KR_SIM_TRANSPOSE, "auto": A.KR_SIM_AUTO}


def _p(a):
    return None if a is None else a.ctypes.data


class _Marshal:
    """Builds a kr_problem and keeps every numpy buffer alive while the C call borrows it."""

    def __init__(self, prob, device=0, stream=None, workspace=None, workspace_bytes=0, comm=None, part=None,
                 virtual_slabs=0, method=None, sim=None):
        self.keep = []
        p = A.kr_problem()
        if prob["op"] == "stencil":
            p.op = A.KR_OP_STENCIL7
            p.mx, p.my, p.mz = int(prob["mx"]), int(prob["my"]), int(prob["mz"])
            p.alpha = float(prob["alpha"])
            bc = prob.get("bc") or [A.KR_BC_DIRICHLET] * 6
            gm = prob.get("gamma") or [0.0] * 6
            p.bc = (C.c_int32 * 6)(*[int(b) for b in bc])
            p.gamma = (C.c_double * 6)(*[float(g) for g in gm])
            if prob.get("b") is not None:  # compact affine term of the stencil (lifted)
                bv = prob["b"] if isinstance(prob["b"], dict) else {"kind": "sparse", "idx": np.nonzero(prob["b"])[0],
                                                                    "val": np.asarray(prob["b"])[np.nonzero(prob["b"])[0]]}
                kb = self._vec(bv)
                self.keep.append(kb)
                p.b_vec = C.addressof(kb)
        else:
            p.op = A.KR_OP_CSR
            rp = self._arr(prob["row_ptr"], np.int64)
            ci = self._arr(prob["col_idx"], np.int32)
            va = self._arr(prob["val"], np.float64)
            p.n, p.nnz = int(prob["n"]), int(ci.size)
            p.row_ptr, p.col_idx, p.val = _p(rp), _p(ci), _p(va)
            if prob.get("b") is not None:
                p.b = _p(self._arr(prob["b"], np.float64))
        gens = prob["gens"]
        p.n_gen = len(gens)
        if gens:
            gv = (A.kr_vec * len(gens))(*[self._vec(g) for g in gens])
            self.keep.append(gv)
            p.gen = gv
            p.z_lo = _p(self._arr(prob["z_lo"], np.float64))
            p.z_hi = _p(self._arr(prob["z_hi"], np.float64))
        if prob.get("center") is not None:
            cv = self._vec(prob["center"])
            self.keep.append(cv)
            p.center = C.pointer(cv)
        outs = prob["outs"]
        ov = (A.kr_vec * len(outs))(*[self._vec(o) for o in outs])
        self.keep.append(ov)
        p.n_out, p.out = len(outs), ov
        p.step, p.n_steps = float(prob["step"]), int(prob["n_steps"])
        p.k = int(prob["k"])
        p.eps = float(prob.get("eps", 0.0) or 0.0)
        p.sim_dir = _SIM[sim or prob.get("sim")]
        p.method = _METHOD[method or prob.get("method", "auto")]
        p.part = _PART[part]
        p.virtual_slabs = int(virtual_slabs)
        p.comm = comm.ptr if comm is not None else None
        p.device = int(device)
        p.stream = stream
        p.workspace = workspace
        p.workspace_bytes = int(workspace_bytes)
        self.p = p

    def _arr(self, a, dt):
        a = np.ascontiguousarray(a, dtype=dt)
        self.keep.append(a)
        return a

    def _vec(self, v):
        kv = A.kr_vec()
        kv.kind = _KIND[v["kind"]]
        if v["kind"] == "sparse":
            idx = self._arr(v["idx"], np.int64)
            val = self._arr(v["val"], np.float64)
            kv.nnz, kv.idx, kv.val = idx.size, _p(idx), _p(val)
        else:
            kv.value = float(v["value"])
            if v["kind"] == "rand":
                kv.seed = int(v["seed"])
            if v["kind"] == "box":
                lo, hi = list(v["lo"]) + [0] * (3 - len(v["lo"])), list(v["hi"]) + [0] * (3 - len(v["hi"]))
                kv.lo = (C.c_int64 * 3)(*lo)
                kv.hi = (C.c_int64 * 3)(*hi)
        return kv


def n_dirs(prob):
    return len(prob["gens"]) + (1 if (prob.get("center") is not None or prob.get("b") is not None) else 0)


def krylov_workspace_bytes(prob, **kw):
    m = _Marshal(prob, **kw)
    out = C.c_size_t()
    A.check(A.lib().krylov_workspace_bytes(C.byref(m.p), C.byref(out)))
    return out.value


class KrylovReach:
    """One handle = one problem on one device (krylov_reach_create). project() runs the hot path,
    check_box() the per-step safety check."""

    def __init__(self, prob, device=0, stream=None, workspace=None, workspace_bytes=0, comm=None, part=None,
                 virtual_slabs=0, method=None, sim=None):
        self.prob = prob
        m = _Marshal(prob, device, stream, workspace, workspace_bytes, comm, part, virtual_slabs, method, sim)
        h = C.c_void_p()
        A.check(A.lib().krylov_reach_create(C.byref(m.p), C.byref(h)))
        self.h = h
        self.n_out = len(prob["outs"])
        self.n_dir = n_dirs(prob)
        self.n_steps = int(prob["n_steps"])
        tr, ns = C.c_int32(), C.c_int32()
        A.check(A.lib().krylov_sim_info(h, C.byref(tr), C.byref(ns)))
        self.transposed, self.n_sim = bool(tr.value), int(ns.value)

    def project(self, want=True):
        if not want:
            A.check(A.lib().krylov_project(self.h, None, None))
            return None, None
        coeff = np.empty((self.n_steps + 1, self.n_out, self.n_dir))
        st = (A.kr_dir_stats * self.n_sim)()
        A.check(A.lib().krylov_project(self.h, _p(coeff), st))
        stats = [{"k_eff": s.k_eff, "beta0": s.beta0, "h_next": s.h_next, "lemma1": s.lemma1_bound} for s in st]
        return coeff, stats

    def check_box(self, thresholds=None, want_bounds=True):
        """thresholds: list of (row, sense, theta) with sense 0=GE, 1=LE, 2=EQ (rows not listed: none)."""
        thresholds = self.prob.get("thresholds", []) if thresholds is None else thresholds
        sense = np.full(self.n_out, A.KR_NONE, dtype=np.int32)
        thr = np.zeros(self.n_out)
        for r, s, t in thresholds:
            sense[r] = s
            thr[r] = t
        lo = hi = None
        if want_bounds:
            lo = np.empty((self.n_steps + 1, self.n_out))
            hi = np.empty((self.n_steps + 1, self.n_out))
        cex = A.kr_cex()
        z = np.empty(self.n_dir)
        A.check(A.lib().krylov_check_box(self.h, _p(sense), _p(thr), _p(lo), _p(hi), C.byref(cex), _p(z)))
        return {"lo": lo, "hi": hi, "found": bool(cex.found), "step": int(cex.step), "time": cex.time,
                "row": int(cex.row), "y": cex.y, "z": z if cex.found else None}

    def check_lp(self, init_A=None, init_b=None, unsafe_A=None, unsafe_b=None, want_feasible=True):
        """Per-step LP feasibility for a polytope initial set (rows on the generator coordinates) and a
        polytope unsafe set in output space (krylov_check_lp)."""
        ng = len(self.prob["gens"])
        IA = np.ascontiguousarray(np.zeros((0, ng)) if init_A is None else init_A, dtype=np.float64).reshape(-1, ng)
        Ib = np.ascontiguousarray(np.zeros(0) if init_b is None else init_b, dtype=np.float64).reshape(-1)
        UA = np.ascontiguousarray(np.zeros((0, self.n_out)) if unsafe_A is None else unsafe_A,
                                  dtype=np.float64).reshape(-1, self.n_out)
        Ub = np.ascontiguousarray(np.zeros(0) if unsafe_b is None else unsafe_b, dtype=np.float64).reshape(-1)
        feas = np.zeros(self.n_steps + 1, dtype=np.int32) if want_feasible else None
        cex = A.kr_cex()
        z = np.zeros(self.n_dir)
        y = np.zeros(self.n_out)
        A.check(A.lib().krylov_check_lp(self.h, IA.shape[0], _p(IA), _p(Ib), UA.shape[0], _p(UA), _p(Ub), _p(feas),
                                        C.byref(cex), _p(z), _p(y)))
        return {"feasible": feas, "found": bool(cex.found), "step": int(cex.step), "time": cex.time,
                "z": z if cex.found else None, "y": y if cex.found else None}

    def eval_outputs(self, step, z):
        """y = c[step] z on the device (krylov_eval_outputs); z has n_dir entries (fixed direction: 1)."""
        z = np.ascontiguousarray(z, dtype=np.float64)
        y = np.zeros(self.n_out)
        A.check(A.lib().krylov_eval_outputs(self.h, int(step), _p(z), _p(y)))
        return y

    def attach_peers(self, rank, world, allgather, barrier):
        """Peer-memory halo transport (krylov_ipc_blob / p2p_open / p2p_verify / p2p_enable): the z-slab step
        kernel then stores its halo planes straight into the neighbours' buffers over NVLink. allgather(bytes)
        -> list of bytes in rank order and barrier() are collectives the caller provides (torch.distributed).
        Every rank takes part even if its own part fails, and the transport is switched on only if every
        rank verified the test pattern; otherwise the NCCL halo exchange stays. Returns True if enabled."""
        ok = 0
        blobs = None
        self.p2p_error = None
        try:
            blob = (C.c_ubyte * A.KR_IPC_BLOB_BYTES)()
            A.check(A.lib().krylov_ipc_blob(self.h, blob))
            mine = bytes(blob)
        except A.KrylovError as e:
            self.p2p_error = repr(e)
            mine = bytes(A.KR_IPC_BLOB_BYTES)
        blobs = allgather(mine)
        try:
            allb = (C.c_ubyte * (A.KR_IPC_BLOB_BYTES * world)).from_buffer_copy(b"".join(blobs))
            A.check(A.lib().krylov_p2p_open(self.h, allb, int(rank), int(world)))
            opened = True
        except A.KrylovError as e:
            self.p2p_error = self.p2p_error or repr(e)
            opened = False
        barrier()
        if opened:
            v = C.c_int32()
            try:
                A.check(A.lib().krylov_p2p_verify(self.h, C.byref(v)))
                ok = int(v.value)
                if not ok:
                    self.p2p_error = "test pattern mismatch"
            except A.KrylovError as e:
                self.p2p_error = self.p2p_error or repr(e)
                ok = 0
        oks = allgather(bytes([ok]))
        on = all(len(o) == 1 and o[0] == 1 for o in oks)
        A.check(A.lib().krylov_p2p_enable(self.h, 1 if on else 0))
        return on

    def krylov_data(self, d=0):
        """(H [(k+1) x k], P [n_out x k]) of direction d (Hessenberg / tridiagonal and P = C V)."""
        k = int(self.prob["k"])
        H = np.zeros((k + 1, k))
        P = np.zeros((self.n_out, k))
        A.check(A.lib().krylov_krylov_data(self.h, int(d), _p(H), _p(P)))
        return H, P

    def tridiag(self, d=0):
        """(alpha [k_eff], beta [k_eff]) of the Lanczos tridiagonal of direction d (stencil Lanczos path)."""
        k = int(self.prob["k"])
        al, be = np.zeros(k), np.zeros(k)
        ke = C.c_int32()
        A.check(A.lib().krylov_tridiag(self.h, int(d), _p(al), _p(be), k, C.byref(ke)))
        return al[:ke.value].copy(), be[:ke.value].copy()

    def adaptive_checks(self, d=0):
        """[(k, unit-vector Lemma 1 bound)] at the Alg. 4 checkpoints evaluated for direction d."""
        cap = 512
        ks = np.zeros(cap, dtype=np.int32)
        bs = np.zeros(cap)
        n = C.c_int32()
        A.check(A.lib().krylov_adaptive_checks(self.h, int(d), _p(ks), _p(bs), cap, C.byref(n)))
        return [(int(ks[i]), float(bs[i])) for i in range(min(n.value, cap))]

    def transfer_bytes(self):
        h2d, d2h = C.c_int64(), C.c_int64()
        A.check(A.lib().krylov_transfer_bytes(self.h, C.byref(h2d), C.byref(d2h)))
        return h2d.value, d2h.value

    def step_times(self):
        """Per-step device times (ms) of the last project (krylov_step_times)."""
        n = C.c_int32()
        A.check(A.lib().krylov_step_times(self.h, None, 0, C.byref(n)))
        ms = np.zeros(max(n.value, 1))
        A.check(A.lib().krylov_step_times(self.h, _p(ms), n.value, C.byref(n)))
        return ms[:n.value]

    def launch_count(self):
        return int(A.lib().krylov_launch_count(self.h))

    def last_timing(self):
        it, st, bytes_ = C.c_double(), C.c_double(), C.c_double()
        n = C.c_int64()
        A.check(A.lib().krylov_last_timing(self.h, C.byref(it), C.byref(st), C.byref(n), C.byref(bytes_)))
        lg, ne = C.c_double(), C.c_int32()
        A.check(A.lib().krylov_last_timing_large(self.h, C.byref(lg), C.byref(ne)))
        return {"iter_ms": it.value, "step_ms_mean": st.value, "step_launches": n.value, "step_bytes": bytes_.value,
                "large_ms": lg.value, "large_evals": ne.value}

    def close(self):
        if getattr(self, "h", None):
            A.lib().krylov_reach_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def validate_counterexample(prob, step, z, y, k=None, **kw):
    """Counter-example check by an independent, higher-accuracy re-simulation: the
    problem is simulated again with a larger Krylov dimension (2k, capped at the path's maximum; for the
    stencil Lanczos path an adaptive run to eps = 1e-12 when k is not given), the outputs at the witness
    z are evaluated on the device, and the relative error against the LP's / box check's outputs y is
    returned as (rel_err, y_resim)."""
    q = dict(prob)
    lanczos_stencil = (prob["op"] == "stencil" and prob.get("method", "lanczos") != "arnoldi"
                       and prob.get("b") is None)
    cap = A.KR_K_MAX if lanczos_stencil else A.KR_K_MAX_ARNOLDI
    q["k"] = int(k) if k else min(2 * int(prob["k"]), cap)
    with KrylovReach(q, **kw) as h:
        h.project(want=False)
        yr = h.eval_outputs(step, z)
    y = np.atleast_1d(np.asarray(y, dtype=np.float64))
    rel = float(np.max(np.abs(yr[:y.size] - y)) / max(np.max(np.abs(yr[:y.size])), 1e-300))
    return rel, yr


# ABI-named functional wrappers
def krylov_reach_create(prob, **kw):
    return KrylovReach(prob, **kw)


def krylov_project(handle):
    return handle.project()


def krylov_check_box(handle, thresholds=None):
    return handle.check_box(thresholds)


def krylov_reach_destroy(handle):
    handle.close()


def krylov_release_cached_memory():
    """Return the device blocks cached from destroyed handles to the driver; bytes released."""
    return int(A.lib().krylov_release_cached_memory())


def krylov_zslab_range(mz, world, rank):
    z0, z1 = C.c_int64(), C.c_int64()
    A.check(A.lib().krylov_zslab_range(int(mz), int(world), int(rank), C.byref(z0), C.byref(z1)))
    return z0.value, z1.value


def krylov_dirs_of_rank(n_dir, world, rank):
    """Global directions simulated by `rank` under direction sharding (round robin; host only)."""
    n = C.c_int32()
    A.check(A.lib().krylov_dirs_of_rank(int(n_dir), int(world), int(rank), None, 0, C.byref(n)))
    out = (C.c_int32 * max(1, n.value))()
    A.check(A.lib().krylov_dirs_of_rank(int(n_dir), int(world), int(rank), out, n.value, C.byref(n)))
    return [int(x) for x in out[:n.value]]


def krylov_zslab_halo_plan(mz, world, rank):
    """Halo schedule of a z-slab rank: list of (is_send, peer, first_buffer_plane, nplanes)."""
    ops = (A.kr_halo_op * 4)()
    n = C.c_int32()
    A.check(A.lib().krylov_zslab_halo_plan(int(mz), int(world), int(rank), ops, C.byref(n)))
    return [(bool(o.is_send), int(o.peer), int(o.plane), int(o.nplanes)) for o in ops[:n.value]]


class KrComm:
    """NCCL communicator for one process per GPU. The 128-byte ncclUniqueId is produced by rank 0
    (krylov_comm_unique_id) and broadcast with torch.distributed (any backend)."""

    def __init__(self, rank, world, device, broadcast):
        """broadcast(bytes_or_None) -> bytes: rank 0 passes the id, every rank gets it back."""
        idbuf = (C.c_ubyte * 128)()
        if rank == 0:
            A.check(A.lib().krylov_comm_unique_id(idbuf))
            data = bytes(idbuf)
        else:
            data = None
        data = broadcast(data)
        idbuf = (C.c_ubyte * 128).from_buffer_copy(data)
        ptr = C.c_void_p()
        A.check(A.lib().krylov_comm_create(idbuf, int(rank), int(world), int(device), C.byref(ptr)))
        self.ptr = ptr
        self.rank, self.world = rank, world

    @classmethod
    def host(cls, rank, world, device, allgather=None):
        """Host-transport communicator (krylov_comm_create_host): the library's collectives become all-gathers
        of host buffers done by `allgather(bytes) -> list of bytes` (default: torch.distributed over the
        default group, e.g. gloo) — several ranks may share one GPU. Marshalling only: the callback moves
        bytes, the library stages them."""
        self = cls.__new__(cls)
        gather = allgather or torch_allgather_raw

        def fn(ctx, send, recv, nbytes):
            try:
                parts = gather(C.string_at(send, nbytes))
                blob = b"".join(parts)
                if len(blob) != nbytes * world:
                    return 1
                C.memmove(recv, blob, len(blob))
                return 0
            except Exception:  # noqa: BLE001 - reported to the library as a failed collective
                return 1

        self._fn = A.ALLGATHER_FN(fn)  # kept alive with the communicator
        ptr = C.c_void_p()
        A.check(A.lib().krylov_comm_create_host(int(rank), int(world), int(device), self._fn, None, C.byref(ptr)))
        self.ptr = ptr
        self.rank, self.world = rank, world
        return self

    def selftest(self, stream=None, reps=3):
        """krylov_comm_selftest: the per-step all-gather inside a captured CUDA graph, replayed; True if every slot
        arrived (collective)."""
        ok = C.c_int32()
        A.check(A.lib().krylov_comm_selftest(self.ptr, stream, int(reps), C.byref(ok)))
        return bool(ok.value)

    def close(self):
        if self.ptr:
            A.lib().krylov_comm_destroy(self.ptr)
            self.ptr = None


def torch_allgather_raw(data):
    """All-gather equal-length bytes over the default torch.distributed group (CPU tensors: gloo), rank order."""
    import torch
    import torch.distributed as dist
    t = torch.frombuffer(bytearray(data), dtype=torch.uint8)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [o.numpy().tobytes() for o in out]


def torch_allgather_bytes(data):
    """All-gather a bytes object over the default torch.distributed group (rank order)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, data)
    return out


def torch_broadcast_id(data):
    """Broadcast the 128-byte NCCL id from rank 0 over the default torch.distributed group."""
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.zeros(128, dtype=torch.uint8, device=dev)
    if data is not None:
        t.copy_(torch.frombuffer(bytearray(data), dtype=torch.uint8))
    dist.broadcast(t, src=0)
    return bytes(t.cpu().numpy().tobytes())
