"""GPU parity for SURVEY §8(f) NEXT-3: the general per-step LP (polytope initial set on z, polytope unsafe
set on the outputs; §2.1, Fig. 2(c)) solved for all time steps at once on the device,
against the oracle's LP (HiGHS) on the oracle's own basis matrices. Feasibility verdicts must agree on
every step whose LP is not degenerate within 1e-7 (margin computed by the oracle side); the first unsafe
step must agree; the GPU witness must satisfy the constraints (witnesses are not unique)."""
import math

import numpy as np
import pytest
from scipy.optimize import linprog

import oracle
import workloads as W

pytestmark = pytest.mark.gpu


def margins(p, coeff, IA, Ib, UA, Ub):
    """Per step: max t such that every row holds with slack t * ||row|| (t > 0: feasible with margin)."""
    ng = len(p["gens"])
    zlo, zhi = np.asarray(p["z_lo"], float)[:ng], np.asarray(p["z_hi"], float)[:ng]
    out = []
    for j in range(coeff.shape[0]):
        B = coeff[j, :, :ng]
        cf = coeff[j, :, ng] if coeff.shape[2] > ng else np.zeros(coeff.shape[1])
        A = np.vstack([IA, UA @ B]) if len(IA) else UA @ B
        b = np.concatenate([Ib, Ub - UA @ cf]) if len(IA) else Ub - UA @ cf
        nr = np.linalg.norm(A, axis=1) + 1e-300
        Ab = np.hstack([A, nr[:, None]])
        r = linprog(np.r_[np.zeros(ng), -1.0], A_ub=Ab, b_ub=b, bounds=list(zip(zlo, zhi)) + [(-1e3, 1e3)],
                    method="highs")
        out.append(-r.fun if r.status == 0 else -np.inf)
    return np.array(out)


def gpu_lp(p, IA, Ib, UA, Ub, **kw):
    from paper_1804_01583_b200 import KrylovReach
    with KrylovReach(p, **kw) as h:
        coeff, _ = h.project()
        lp = h.check_lp(IA, Ib, UA, Ub)
    return coeff, lp


def check(p, ocoeff, IA, Ib, UA, Ub, **kw):
    IA, Ib, UA, Ub = (np.asarray(x, dtype=float) for x in (IA, Ib, UA, Ub))
    ref = oracle.check_lp(p, ocoeff, IA, Ib, UA, Ub)
    coeff, lp = gpu_lp(p, IA, Ib, UA, Ub, **kw)
    m = margins(p, ocoeff, IA.reshape(-1, len(p["gens"])), Ib, UA, Ub)
    clear = np.abs(m) > 1e-7
    assert np.all(lp["feasible"] >= 0)
    assert np.array_equal(lp["feasible"][clear] == 1, ref["feasible"][clear]), np.nonzero(
        (lp["feasible"] == 1) != ref["feasible"])
    assert lp["found"] == ref["found"]
    if lp["found"]:
        assert lp["step"] == ref["step"]
        ng = len(p["gens"])
        z = lp["z"][:ng]
        j = lp["step"]
        B = coeff[j, :, :ng]
        cf = coeff[j, :, ng] if coeff.shape[2] > ng else 0.0
        y = B @ z + cf
        assert np.allclose(lp["y"], y, rtol=1e-9, atol=1e-12)
        tol = 1e-7 * (1 + np.abs(Ub).max())
        assert np.all(UA @ y <= Ub + tol)
        if len(Ib):
            assert np.all(IA.reshape(-1, ng) @ z <= Ib + 1e-7 * (1 + np.abs(Ib).max()))
        assert np.all(z >= np.asarray(p["z_lo"])[:ng] - 1e-9) and np.all(z <= np.asarray(p["z_hi"])[:ng] + 1e-9)
    return lp, ref


def test_lp_oscillator_paper():
    p = W.oscillator()
    lp, ref = check(p, oracle.krylov_project(p)["coeff"], np.zeros((0, 1)), [], [[1.0], [-1.0]], [4.0, -4.0])
    assert list(lp["feasible"][:4] == 1) == [False, False, False, True]
    assert abs(lp["z"][0] - (4 * math.sqrt(2) - 5)) < 1e-9 and abs(lp["y"][0] - 4.0) < 1e-9


def test_lp_config1_halfspace_equals_box_check():
    p = W.config1()
    lp, ref = check(p, oracle.krylov_project(p)["coeff"], np.zeros((0, 8)), [], [[-1.0]], [-0.02])
    assert lp["step"] == 74  # the interval check's first unsafe step


def test_lp_config1_polytope_initial_set():
    """C1 with a polytope initial set: sum of the 8 cell temperatures <= 7.6 and cell (0,0,0) - cell (1,1,1)
    <= 0.05 — the interval check no longer applies; threshold on the center chosen mid-trajectory."""
    p = W.config1()
    oc = oracle.krylov_project(p)["coeff"]
    IA = np.zeros((2, 8))
    IA[0] = 1.0
    IA[1, 0], IA[1, 7] = 1.0, -1.0
    Ib = [7.6, 0.05]
    check(p, oc, IA, Ib, [[-1.0]], [-0.0275])


def test_lp_config2_transposed_polytopes():
    """C2 (transpose mode, 3 simulations): the 20 generators are further restricted by 41 rows (|z_d| <= 0.01
    and sum z <= 0.1) so the outputs follow the affine term's trajectory; unsafe: y_0 <= theta_0 (crossed
    mid-trajectory, placed by the oracle) and y_1 <= theta_1 (a second row that binds part of the time)."""
    p = W.config2()
    oc = oracle.krylov_project_transpose(p)["coeff"]
    IA = np.vstack([np.eye(20), -np.eye(20), np.ones((1, 20))])
    Ib = np.r_[np.full(40, 0.01), 0.1]
    yf = oc[:, :, 20]  # fixed-term outputs
    th0 = 0.5 * (yf[0, 0] + yf[-1, 0])
    th1 = 0.5 * (yf[:, 1].min() + yf[:, 1].max())
    UA = np.array([[1.0 if yf[-1, 0] < yf[0, 0] else -1.0, 0, 0], [0, 1.0, 0]])
    Ub = np.array([th0 * UA[0, 0], th1])
    lp, ref = check(p, oc, IA, Ib, UA, Ub, sim="transpose")
    assert ref["found"] and 0 < ref["step"] < p["n_steps"]


def test_counterexample_resimulation():
    """the LP counter-example of C2 (transpose mode, k = 40) re-simulated independently — forward
    mode, one simulation per direction, k = 64 — agrees to well under the paper's 1e-6 LP tolerance
    (the paper reports 6.17e-9 on MNA5); krylov_eval_outputs equals c[j] z."""
    from paper_1804_01583_b200 import KrylovReach, validate_counterexample
    p = W.config2()
    IA = np.vstack([np.eye(20), -np.eye(20), np.ones((1, 20))])
    Ib = np.r_[np.full(40, 0.01), 0.1]
    with KrylovReach(p, sim="transpose") as h:
        coeff, _ = h.project()
        yf = coeff[:, :, 20]
        th0 = 0.5 * (yf[0, 0] + yf[-1, 0])
        lp = h.check_lp(IA, Ib, [[1.0 if yf[-1, 0] < yf[0, 0] else -1.0, 0, 0]],
                        [th0 * (1.0 if yf[-1, 0] < yf[0, 0] else -1.0)])
        assert lp["found"]
        y_dev = h.eval_outputs(lp["step"], lp["z"])
        assert np.allclose(y_dev, coeff[lp["step"]] @ lp["z"], rtol=1e-12, atol=1e-14)
        assert np.allclose(y_dev, lp["y"], rtol=1e-12, atol=1e-14)
    rel, y_re = validate_counterexample(p, lp["step"], lp["z"], lp["y"], k=64, sim="forward")
    assert rel < 1e-9, rel


def test_lp_degenerate_cases():
    """No constraints at all (every step feasible: first unsafe step 0, witness in the box); an empty initial
    polytope (z_0 <= -2 with z_0 in [0.9, 1.1]: never feasible); n_steps = 0."""
    from paper_1804_01583_b200 import KrylovReach
    p = W.heat(12, 2, 10, n_steps=20)
    with KrylovReach(p) as h:
        h.project()
        lp = h.check_lp()
        assert lp["found"] and lp["step"] == 0 and 0.9 <= lp["z"][0] <= 1.1
        assert np.all(lp["feasible"] == 1)
        lp = h.check_lp([[1.0]], [-2.0], None, None)
        assert not lp["found"] and np.all(lp["feasible"] == 0)
    q = W.heat(12, 2, 10, n_steps=0)
    with KrylovReach(q) as h:
        c, _ = h.project()
        lp = h.check_lp(None, None, [[-1.0, 0, 0, 0]], [-1e9])  # center >= 1e9: infeasible
        assert not lp["found"] and lp["feasible"].shape == (1,)
