"""CPU-only checks of the C ABI library: it loads, exports every function include/krylov_reach.h declares,
and its host-only logic (partitioning, validation / error mapping, workspace sizing) behaves. No GPU
compute is called here."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1804_01583_b200 import build
    build.build()
    from paper_1804_01583_b200 import _abi
    return _abi.lib()


def header_functions():
    src = open(os.path.join(ROOT, "include", "krylov_reach.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(krylov_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    from paper_1804_01583_b200 import _abi
    names = header_functions()
    assert len(names) >= 12
    out = subprocess.run(["nm", "-D", "--defined-only", _abi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (krylov_\w+)", out))
    for n in names:
        assert n in exported, n
        assert hasattr(lib, n)
    assert set(_abi.EXPORTS) == set(names)


def test_library_is_sm100a(lib):
    from paper_1804_01583_b200 import _abi
    out = subprocess.run(["cuobjdump", "--list-elf", _abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_zslab_range_partition():
    from paper_1804_01583_b200 import krylov_zslab_range, KrylovError
    for mz, world in [(1000, 8), (400, 8), (1000, 3), (26, 4), (7, 3), (100, 1)]:
        spans = [krylov_zslab_range(mz, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == mz
        for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
            assert a1 == b0
        sizes = [b - a for a, b in spans]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(KrylovError):
        krylov_zslab_range(5, 4, 3)  # rank 3 would own 1 plane
    assert krylov_zslab_range(1000, 8, 7) == (875, 1000)


def test_workspace_bytes_host_only():
    from paper_1804_01583_b200 import krylov_workspace_bytes
    p = W.config5()
    b = krylov_workspace_bytes(p)
    pitch = 1000
    assert b == 3 * (1000 + 3) * 1000 * pitch * 8 + 3 * 256  # 3 vectors + ghost planes (Eq. 6's 3n) + alignment
    p4 = W.heat(401, 40, 40)
    assert krylov_workspace_bytes(p4) == 3 * (401 + 3) * 401 * 402 * 8 + 3 * 256  # pitch padded to even
    q = W.config2()
    assert krylov_workspace_bytes(q) == 21 * 42 * 20001 * 8 + 512  # Arnoldi stores k+1 vectors (+W) per direction


@pytest.mark.parametrize("mutate,code", [
    (lambda p: p.update(k=0), "KR_EINVAL"),
    (lambda p: p.update(k=16385), "KR_EINVAL"),
    (lambda p: p.update(k=2049, method="arnoldi"), "KR_EINVAL"),
    (lambda p: p.update(eps=-1e-6), "KR_EINVAL"),
    (lambda p: p.update(bc=[3, 0, 0, 0, 0, 0]), "KR_EINVAL"),
    (lambda p: p.update(bc=[2, 0, 0, 0, 0, 0], gamma=[-1.0, 0, 0, 0, 0, 0]), "KR_EINVAL"),
    (lambda p: p.update(step=0.0), "KR_EINVAL"),
    (lambda p: p.update(n_steps=-1), "KR_EINVAL"),
    (lambda p: p.update(z_lo=np.array([2.0])), "KR_EINVAL"),
    (lambda p: p.update(gens=[W.box((0, 0, 0), (2, 2, 0))]), "KR_EZERO"),
    (lambda p: p.update(gens=[W.box((0, 0, 0), (20, 2, 2))]), "KR_EDIM"),
    (lambda p: p.update(outs=[W.sparse([10 ** 6], [1.0])]), "KR_EDIM"),
    (lambda p: p.update(alpha=float("nan")), "KR_ENONFINITE"),
    (lambda p: p.update(outs=[]), "KR_EINVAL"),
])
def test_validation_errors(mutate, code):
    from paper_1804_01583_b200 import KrylovError, krylov_workspace_bytes
    p = W.heat(10, 2, 5)
    mutate(p)
    with pytest.raises(KrylovError) as e:
        krylov_workspace_bytes(p)
    assert code in str(e.value)


def test_large_k_and_boundaries_accepted_host_side():
    """NEXT-1: stencil Lanczos takes k up to KR_K_MAX, adaptive eps and per-face boundaries (host-only sizing)."""
    from paper_1804_01583_b200 import krylov_workspace_bytes
    p = W.heat_paper(20, eps=1e-6, k_max=16384)
    assert krylov_workspace_bytes(p) == 3 * (20 + 3) * 20 * 20 * 8 + 3 * 256
    p = W.heat(10, 2, 5)
    p.update(k=500, bc=[1, 2, 1, 1, 0, 1], gamma=[0, 0.3, 0, 0, 0, 0])
    assert krylov_workspace_bytes(p) > 0


def test_lanczos_on_nonsymmetric_rejected():
    from paper_1804_01583_b200 import KrylovError, krylov_workspace_bytes
    with pytest.raises(KrylovError) as e:
        krylov_workspace_bytes(W.oscillator(), method="lanczos")
    assert "KR_ENOTSYM" in str(e.value)
    rp, ci, va, dense = W.random_csr(50, 4, seed=1)
    q = {"op": "csr", "n": 50, "row_ptr": rp, "col_idx": ci, "val": va, "b": None, "gens": [W.sparse([0], [1.0])],
         "z_lo": [0.0], "z_hi": [1.0], "center": None, "outs": [W.allv()], "step": 0.1, "n_steps": 3, "k": 4}
    with pytest.raises(KrylovError):
        krylov_workspace_bytes(q, method="lanczos")
    rp, ci, va, dense = W.random_csr(50, 4, seed=1, symmetric=True)
    q.update(row_ptr=rp, col_idx=ci, val=va)
    assert krylov_workspace_bytes(q, method="lanczos") > 0


def test_product_fails_loudly_without_library(tmp_path, monkeypatch):
    """No CPU fallback: a missing .so raises on load."""
    from paper_1804_01583_b200 import _abi
    monkeypatch.setattr(_abi, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_abi, "_lib", None)
    with pytest.raises(ImportError):
        _abi.lib()


def test_transpose_mode_host_side():
    """NEXT-2: the transposed problem's workspace is sized for o simulations of the lifted A'^T."""
    from paper_1804_01583_b200 import KrylovError, krylov_workspace_bytes
    q = W.config2()
    assert krylov_workspace_bytes(q, sim="transpose") == 3 * 42 * 20001 * 8 + 512
    assert krylov_workspace_bytes(q, sim="auto") == 3 * 42 * 20001 * 8 + 512
    p = W.heat_paper(20)
    with pytest.raises(KrylovError) as e:
        krylov_workspace_bytes(p, sim="transpose")  # not combined with adaptive k
    assert "KR_EINVAL" in str(e.value)


def test_lifted_stencil_host_side():
    """NEXT-4: the heater's compact affine term lifts the stencil (N = n + 1, one fixed direction, Arnoldi);
    beyond one CTA the stored basis is orthogonalised by the CGS2 path (no dimension cap)."""
    from paper_1804_01583_b200 import KrylovError, krylov_workspace_bytes
    p = W.heat_heater(10)
    assert krylov_workspace_bytes(p) == 1 * (64 + 2) * 1001 * 8 + 512
    q = W.heat_heater(100, k=400)
    assert krylov_workspace_bytes(q) == 1 * 402 * 1000001 * 8 + 512
    with pytest.raises(KrylovError) as e:
        krylov_workspace_bytes(q, method="lanczos")
    assert "KR_ENOTSYM" in str(e.value)


def test_adaptive_validation():
    """eps > 0: stencil Lanczos (Alg. 4) or Arnoldi (Alg. 2); not stored-basis Lanczos on a CSR matrix."""
    from paper_1804_01583_b200 import KrylovError, krylov_workspace_bytes
    q = W.csr_stable_nonsym()
    assert krylov_workspace_bytes(q) == 3 * (200 + 2) * 400 * 8 + 512
    rp, ci, va, dense = W.random_csr(50, 4, seed=1, symmetric=True)
    r = {"op": "csr", "n": 50, "row_ptr": rp, "col_idx": ci, "val": va, "b": None, "gens": [W.sparse([0], [1.0])],
         "z_lo": [0.0], "z_hi": [1.0], "center": None, "outs": [W.allv()], "step": 0.1, "n_steps": 3, "k": 4,
         "eps": 1e-6}
    with pytest.raises(KrylovError) as e:
        krylov_workspace_bytes(r, method="lanczos")
    assert "KR_EINVAL" in str(e.value)


def test_host_utilities_match_oracle():
    """Eq. 3 a priori bound and Eq. 4 / Eq. 6 memory (host utilities of the ABI) against the oracle's
    definitions and the paper's printed values (10^16182319; 46 TB)."""
    import oracle
    from paper_1804_01583_b200 import _abi as A
    L = A.lib()
    for x, k in [(32771611.0, 10 ** 6), (2.5, 10), (100.0, 40)]:
        assert abs(L.krylov_a_priori_bound_log10(x, k) - oracle.a_priori_bound_log10(x, k)) <= 1e-9 * abs(
            oracle.a_priori_bound_log10(x, k)) + 1e-9
    assert round(L.krylov_a_priori_bound_log10(32771611.0, 10 ** 6)) == 16182319
    assert L.krylov_memory_bytes(10 ** 9, 5932, 1, 1, A.KR_ARNOLDI) == oracle.memory_bytes(10 ** 9, 5932)
    assert L.krylov_memory_bytes(10923, 63, 10, 2, A.KR_LANCZOS) == oracle.memory_bytes(10923, 63, 10, 2, "lanczos")
    assert L.krylov_memory_bytes(0, 5, 1, 1, A.KR_ARNOLDI) == -1


def test_release_cached_memory_without_gpu(lib):
    """The block cache is empty without a GPU: releasing it is a no-op returning 0 bytes."""
    from paper_1804_01583_b200 import krylov_release_cached_memory
    assert krylov_release_cached_memory() == 0
