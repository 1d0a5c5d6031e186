"""GPU parity for SURVEY §8(f) NEXT-4: the nonsymmetric heat variant with a permanent heater —
a lifted stencil (compact affine term) simulated by Arnoldi, on the one-CTA MGS path, the
multi-CTA CGS2 path (large N), and with k > 64 through the large-k route on the dense Hessenberg —
against the oracle's literal MGS Arnoldi (tolerance tests/parity.py)."""
import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import assert_coeff

pytestmark = pytest.mark.gpu


def gpu(p, **kw):
    from paper_1804_01583_b200 import KrylovReach
    with KrylovReach(p, **kw) as h:
        coeff, stats = h.project()
        assert h.launch_count() > 0
    return coeff, stats


@pytest.mark.parametrize("cgs", [False, True])
def test_heater_m10(cgs, monkeypatch):
    """The paper's 10x10x10 version, k = 64 (per-step Pade), one-CTA MGS and forced CGS2."""
    if cgs:
        monkeypatch.setenv("KR_FORCE_CGS", "1")
    p = W.heat_heater(10)
    res = oracle.krylov_project(p)
    coeff, stats = gpu(p)
    assert_coeff(coeff, res["coeff"], f"heater10 cgs={cgs}")
    assert stats[0]["k_eff"] == res["per_dir"][0]["k_eff"]
    assert abs(stats[0]["beta0"] - 1.0) == 0.0  # the lifted start e_{n+1}


def test_heater_large_k_dense_hessenberg():
    """k = 100 > 64: the Arnoldi Hessenberg through the large-k route (Taylor scaling-squaring + doubling)."""
    p = W.heat_heater(10, k=100, n_steps=200, step=2.5)
    res = oracle.krylov_project(p)
    coeff, stats = gpu(p)
    assert stats[0]["k_eff"] == res["per_dir"][0]["k_eff"]
    assert_coeff(coeff, res["coeff"], "heater10 k=100")


def test_heater_cgs2_path_large_n():
    """m = 32: N = 32769 > 27648 lifts the basis out of one CTA: the CGS2 multi-CTA path."""
    p = W.heat_heater(32, k=48, n_steps=200, step=2.5)
    res = oracle.krylov_project(p)
    coeff, stats = gpu(p)
    assert_coeff(coeff, res["coeff"], "heater32 (CGS2)")


def test_cgs2_forced_on_config1():
    """CGS2 on the BASELINE configs[0] (8 directions, stencil Arnoldi) equals the oracle's MGS."""
    import os
    os.environ["KR_FORCE_CGS"] = "1"
    try:
        p = W.config1()
        coeff, _ = gpu(p)
    finally:
        del os.environ["KR_FORCE_CGS"]
    assert_coeff(coeff, oracle.krylov_project(p)["coeff"], "C1 CGS2")


def test_new_paths_bitwise_deterministic():
    """Fixed-order reductions everywhere: repeated runs of the adaptive large-k route, the CGS2 Arnoldi, the
    transpose mode and the batched LP are bitwise identical."""
    from paper_1804_01583_b200 import KrylovReach

    def run_all():
        out = []
        with KrylovReach(W.heat_paper(20, k_max=400)) as h:
            out.append(h.project()[0])
        with KrylovReach(W.heat_heater(32, k=48, n_steps=100, step=2.5)) as h:
            out.append(h.project()[0])
        with KrylovReach(W.config2(n=3000, n_gen=6, n_steps=200, k=30), sim="transpose") as h:
            c, _ = h.project()
            out.append(c)
            lp = h.check_lp(np.ones((1, 6)), [0.5], [[1.0, 0, 0]], [float(np.median(c[:, 0, :].sum(axis=1)))])
            out.append(lp["feasible"].astype(np.float64))
        return out

    a, b = run_all(), run_all()
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
