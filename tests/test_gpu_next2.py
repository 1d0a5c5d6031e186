"""GPU parity for SURVEY §8(f) NEXT-2: the basis matrix by transpose dynamics (§4.1) — o
Krylov simulations of x' = A'^T x from the output rows, projected with E^T — against the oracle's
transpose mode (tolerance tests/parity.py), verdicts identical, and against the forward mode where both
are exact."""
import math

import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import assert_coeff, bounds_close

pytestmark = pytest.mark.gpu


def run(p, **kw):
    from paper_1804_01583_b200 import KrylovReach
    with KrylovReach(p, **kw) as h:
        coeff, stats = h.project()
        cb = h.check_box()
        info = (h.transposed, h.n_sim, h.launch_count())
    assert info[2] > 0
    return coeff, stats, cb, info


def test_transpose_oscillator_paper_example():
    p = W.oscillator()
    coeff, stats, cb, (tr, ns, _) = run(p, sim="transpose")
    assert tr and ns == 1  # o = 1 simulation
    res = oracle.krylov_project_transpose(p)
    assert_coeff(coeff, res["coeff"], "oscillator^T")
    assert np.allclose(coeff[3, 0], [0.707, 3.54], atol=5e-3)
    assert cb["found"] and cb["step"] == 3 and abs(cb["z"][0] - (4 * math.sqrt(2) - 5)) <= 1e-12


def test_transpose_config1_one_simulation():
    """C1: 1 simulation from the center cell instead of 8; equal to the forward result (both exact)."""
    p = W.config1()
    coeff, stats, cb, (tr, ns, _) = run(p, sim="transpose")
    assert tr and ns == 1
    assert_coeff(coeff, oracle.krylov_project_transpose(p)["coeff"], "C1^T")
    assert_coeff(coeff, oracle.krylov_project(p)["coeff"], "C1^T vs forward")
    assert not cb["found"]
    _, _, cb2, _ = run(dict(p, thresholds=[(0, W.GE, 0.02)]), sim="transpose")
    assert cb2["found"] and cb2["step"] == 74


def test_transpose_config2_full_size():
    """BASELINE configs[1] at full size: 3 simulations of the lifted A'^T (n' = 20001) instead of 21,
    against the oracle's transpose mode on every step; AUTO picks the transpose (o = 3 < i = 21)."""
    p = W.config2()
    coeff, stats, cb, (tr, ns, _) = run(p, sim="auto")
    assert tr and ns == 3
    res = oracle.krylov_project_transpose(p)
    assert_coeff(coeff, res["coeff"], "C2^T")
    for s, r in zip(stats, res["per_dir"]):
        assert s["k_eff"] == r["k_eff"]
    ocb = oracle.check_box(p, res["coeff"], [])
    zlo, zhi = oracle.z_bounds(p)
    for side in ("lo", "hi"):
        ok, worst = bounds_close(cb[side], ocb[side], res["coeff"], zlo, zhi)
        assert ok, (side, worst)
    # the Lemma-1 diagnostic of each transposed simulation (+inf on both sides: mu > 0 for the lifted A'^T)
    from tests.test_gpu_parity import assert_lemma1, hmax_of
    assert_lemma1(stats, res["lemma1"], "C2^T", T=p["n_steps"] * p["step"], mu=res["mu"], hmax=hmax_of(res["per_dir"]))


@pytest.mark.parametrize("vs", [0, 2])
def test_transpose_stencil_lanczos(vs):
    """Fused stencil Lanczos in transpose mode: simulations start at the 4 output rows (center, total heat,
    two cells), projected on the corner-block generator; 1 and 2 virtual z-slabs."""
    p = W.heat(30, 4, 30, n_steps=150, my=21, mz=13)
    coeff, stats, cb, (tr, ns, _) = run(p, sim="transpose", virtual_slabs=vs)
    assert tr and ns == 4
    assert_coeff(coeff, oracle.krylov_project_transpose(p)["coeff"], f"heat^T vs={vs}")


def test_auto_keeps_forward_when_fewer_directions():
    p = W.heat(20, 3, 20, n_steps=40)
    _, stats, _, (tr, ns, _) = run(p, sim="auto")
    assert not tr and ns == 1


def test_transpose_more_simulations_than_directions():
    """Forced transpose with o = 4 > i = 1 (AUTO would stay forward): still the oracle's transpose result."""
    p = W.heat(14, 3, 20, n_steps=40)
    coeff, stats, cb, (tr, ns, _) = run(p, sim="transpose")
    assert tr and ns == 4 and len(stats) == 4
    assert_coeff(coeff, oracle.krylov_project_transpose(p)["coeff"], "heat^T o>i")


def test_transpose_combinations():
    """Transpose mode with a center but no affine term (the fixed direction is c itself, not lifted), on CSR
    and on the stencil; every output against the oracle's transpose mode, verdicts as in forward mode."""
    rp, ci, va, dense = W.random_csr(300, 5, seed=11, scale=0.3)
    p = {"name": "csr_center", "op": "csr", "n": 300, "row_ptr": rp, "col_idx": ci, "val": va, "b": None,
         "gens": [W.sparse([0], [1.0]), W.box((10,), (40,), 0.5), W.sparse([7, 8], [1.0, -1.0])],
         "z_lo": np.array([-1.0, 0.0, -0.5]), "z_hi": np.array([1.0, 2.0, 0.5]), "center": W.sparse([3, 5], [2.0, 1.0]),
         "outs": [W.allv(1.0), W.sparse(np.arange(300), np.linspace(-1, 1, 300))], "step": 0.05, "n_steps": 120,
         "k": 30, "method": "arnoldi", "thresholds": [(0, W.GE, 1.5)]}
    coeff, stats, cb, (tr, ns, _) = run(p, sim="transpose")
    assert tr and ns == 2
    ref = oracle.krylov_project_transpose(p)["coeff"]
    assert_coeff(coeff, ref, "csr center^T")
    ocb = oracle.check_box(p, ref)
    assert cb["found"] == ocb["found"] and cb["step"] == ocb["step"]
    q = W.heat(16, 3, 24, n_steps=60)
    q["center"] = W.box((2, 2, 2), (5, 6, 7), 0.3)
    coeff, stats, cb, (tr, ns, _) = run(q, sim="transpose")
    assert tr and ns == 4
    assert_coeff(coeff, oracle.krylov_project_transpose(q)["coeff"], "heat center^T")
