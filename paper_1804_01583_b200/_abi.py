"""ctypes mirror of include/krylov_reach.h (argument marshalling only — every step of the hot path runs
inside libkrylov_reach.so). Loading fails loudly if the CUDA library has not been built: there is no
CPU fallback."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libkrylov_reach.so")  # the in-tree build, nothing else

KR_OK, KR_EINVAL, KR_EDIM, KR_ENOMEM, KR_ECUDA, KR_ENCCL, KR_ENOTSYM, KR_EZERO, KR_ENONFINITE, KR_ESTATE = range(10)
STATUS_NAMES = ["KR_OK", "KR_EINVAL", "KR_EDIM", "KR_ENOMEM", "KR_ECUDA", "KR_ENCCL", "KR_ENOTSYM", "KR_EZERO",
                "KR_ENONFINITE", "KR_ESTATE"]
KR_OP_STENCIL7, KR_OP_CSR = 0, 1
KR_AUTO, KR_ARNOLDI, KR_LANCZOS = 0, 1, 2
KR_PART_NONE, KR_PART_ZSLAB, KR_PART_DIRS = 0, 1, 2
KR_GE, KR_LE, KR_EQ, KR_NONE = 0, 1, 2, 3
KR_VEC_SPARSE, KR_VEC_BOX, KR_VEC_ALL, KR_VEC_RAND = 0, 1, 2, 3
KR_BC_DIRICHLET, KR_BC_INSULATED, KR_BC_ROBIN = 0, 1, 2
KR_K_MAX_FIXED_PADE, KR_K_MAX, KR_K_MAX_ARNOLDI = 64, 16384, 2048
KR_SIM_FORWARD, KR_SIM_TRANSPOSE, KR_SIM_AUTO = 0, 1, 2
KR_IPC_BLOB_BYTES = 512


class kr_vec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("nnz", C.c_int64), ("idx", C.c_void_p), ("val", C.c_void_p),
                ("lo", C.c_int64 * 3), ("hi", C.c_int64 * 3), ("value", C.c_double), ("seed", C.c_uint64)]


class kr_problem(C.Structure):
    _fields_ = [
        ("op", C.c_int32), ("mx", C.c_int64), ("my", C.c_int64), ("mz", C.c_int64), ("alpha", C.c_double),
        ("n", C.c_int64), ("nnz", C.c_int64), ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p),
        ("val", C.c_void_p), ("b", C.c_void_p), ("b_vec", C.c_void_p),
        ("n_gen", C.c_int32), ("gen", C.POINTER(kr_vec)), ("z_lo", C.c_void_p), ("z_hi", C.c_void_p),
        ("center", C.POINTER(kr_vec)),
        ("n_out", C.c_int32), ("out", C.POINTER(kr_vec)),
        ("step", C.c_double), ("n_steps", C.c_int64),
        ("k", C.c_int32), ("method", C.c_int32), ("eps", C.c_double),
        ("bc", C.c_int32 * 6), ("gamma", C.c_double * 6), ("sim_dir", C.c_int32),
        ("part", C.c_int32), ("virtual_slabs", C.c_int32), ("comm", C.c_void_p), ("device", C.c_int32),
        ("stream", C.c_void_p), ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t),
    ]


class kr_dir_stats(C.Structure):
    _fields_ = [("k_eff", C.c_int32), ("beta0", C.c_double), ("h_next", C.c_double), ("lemma1_bound", C.c_double)]


class kr_halo_op(C.Structure):
    _fields_ = [("is_send", C.c_int32), ("peer", C.c_int32), ("plane", C.c_int64), ("nplanes", C.c_int64)]


class kr_cex(C.Structure):
    _fields_ = [("found", C.c_int32), ("step", C.c_int64), ("time", C.c_double), ("row", C.c_int32),
                ("y", C.c_double)]


EXPORTS = ["krylov_workspace_bytes", "krylov_reach_create", "krylov_project", "krylov_check_box",
           "krylov_reach_destroy", "krylov_last_error", "krylov_launch_count", "krylov_last_timing",
           "krylov_comm_unique_id", "krylov_comm_create", "krylov_comm_destroy", "krylov_zslab_range",
           "krylov_krylov_data", "krylov_transfer_bytes", "krylov_zslab_halo_plan", "krylov_tridiag",
           "krylov_adaptive_checks", "krylov_last_timing_large", "krylov_sim_info", "krylov_check_lp",
           "krylov_eval_outputs", "krylov_ipc_blob", "krylov_p2p_open", "krylov_p2p_verify", "krylov_p2p_enable",
           "krylov_a_priori_bound_log10", "krylov_memory_bytes", "krylov_step_times",
           "krylov_release_cached_memory", "krylov_comm_create_host", "krylov_dirs_of_rank",
           "krylov_comm_selftest"]

# int32_t fn(void* ctx, const void* send, void* recv, size_t bytes): the host transport's all-gather
ALLGATHER_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)

_lib = None


def lib():
    """Load libkrylov_reach.so (raises if it is missing — build it with python -m paper_1804_01583_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built: run `python -m paper_1804_01583_b200.build` "
                          "(there is no CPU fallback for the Krylov hot path)")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    L.krylov_workspace_bytes.argtypes = [C.POINTER(kr_problem), C.POINTER(C.c_size_t)]
    L.krylov_reach_create.argtypes = [C.POINTER(kr_problem), C.POINTER(vp)]
    L.krylov_project.argtypes = [vp, vp, C.POINTER(kr_dir_stats)]
    L.krylov_check_box.argtypes = [vp, vp, vp, vp, vp, C.POINTER(kr_cex), vp]
    L.krylov_reach_destroy.argtypes = [vp]
    L.krylov_reach_destroy.restype = None
    L.krylov_release_cached_memory.argtypes = []
    L.krylov_release_cached_memory.restype = C.c_size_t
    L.krylov_last_error.restype = C.c_char_p
    L.krylov_launch_count.argtypes = [vp]
    L.krylov_launch_count.restype = C.c_int64
    L.krylov_last_timing.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                     C.POINTER(C.c_double)]
    L.krylov_comm_unique_id.argtypes = [vp]
    L.krylov_comm_create.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32, C.POINTER(vp)]
    L.krylov_comm_create_host.argtypes = [C.c_int32, C.c_int32, C.c_int32, ALLGATHER_FN, vp, C.POINTER(vp)]
    L.krylov_comm_destroy.argtypes = [vp]
    L.krylov_comm_selftest.argtypes = [vp, vp, C.c_int32, C.POINTER(C.c_int32)]
    L.krylov_dirs_of_rank.argtypes = [C.c_int32, C.c_int32, C.c_int32, vp, C.c_int32, C.POINTER(C.c_int32)]
    L.krylov_comm_destroy.restype = None
    L.krylov_krylov_data.argtypes = [vp, C.c_int32, vp, vp]
    L.krylov_check_lp.argtypes = [vp, C.c_int32, vp, vp, C.c_int32, vp, vp, vp, C.POINTER(kr_cex), vp, vp]
    L.krylov_eval_outputs.argtypes = [vp, C.c_int64, vp, vp]
    L.krylov_ipc_blob.argtypes = [vp, vp]
    L.krylov_step_times.argtypes = [vp, vp, C.c_int32, C.POINTER(C.c_int32)]
    L.krylov_a_priori_bound_log10.argtypes = [C.c_double, C.c_int32]
    L.krylov_a_priori_bound_log10.restype = C.c_double
    L.krylov_memory_bytes.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32]
    L.krylov_memory_bytes.restype = C.c_int64
    L.krylov_p2p_open.argtypes = [vp, vp, C.c_int32, C.c_int32]
    L.krylov_p2p_verify.argtypes = [vp, C.POINTER(C.c_int32)]
    L.krylov_p2p_enable.argtypes = [vp, C.c_int32]
    L.krylov_sim_info.argtypes = [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    L.krylov_last_timing_large.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_int32)]
    L.krylov_tridiag.argtypes = [vp, C.c_int32, vp, vp, C.c_int32, C.POINTER(C.c_int32)]
    L.krylov_adaptive_checks.argtypes = [vp, C.c_int32, vp, vp, C.c_int32, C.POINTER(C.c_int32)]
    L.krylov_zslab_halo_plan.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.POINTER(kr_halo_op),
                                         C.POINTER(C.c_int32)]
    L.krylov_transfer_bytes.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    L.krylov_zslab_range.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    for name in EXPORTS:
        if name not in ("krylov_reach_destroy", "krylov_last_error", "krylov_launch_count", "krylov_comm_destroy",
                        "krylov_a_priori_bound_log10", "krylov_memory_bytes"):
            getattr(L, name).restype = C.c_int
    _lib = L
    return L


class KrylovError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")


def check(status):
    if status != KR_OK:
        raise KrylovError(status, lib().krylov_last_error().decode(errors="replace"))
