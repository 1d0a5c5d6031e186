"""Pins for the CPU oracle (oracle/) against things other than itself: the paper's printed worked
example, closed forms, library routines (scipy) on special cases, invariants and brute force.
Each test names what it pins and where the expected value comes from. CPU only (-m "not gpu")."""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp
from scipy.optimize import linprog

import oracle
import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def kron_laplacian(mx, my, mz, alpha):
    """Independent construction of A = alpha * L_h (Dirichlet, h_a = 1/(m_a+1)) as a Kronecker sum
    of 1-D second-difference matrices (textbook), x fastest."""
    def t1(m):
        return sp.diags([np.ones(m - 1), -2 * np.ones(m), np.ones(m - 1)], [-1, 0, 1]) * float(m + 1) ** 2
    Ix, Iy, Iz = sp.identity(mx), sp.identity(my), sp.identity(mz)
    L = sp.kron(Iz, sp.kron(Iy, t1(mx))) + sp.kron(Iz, sp.kron(t1(my), Ix)) + sp.kron(t1(mz), sp.kron(Iy, Ix))
    return (alpha * L).tocsr()


def sine_mode(m, p):
    x = np.arange(m)
    return np.sin((x + 1) * p * np.pi / (m + 1))


def lam1(m, p, alpha):
    """1-D Dirichlet eigenvalue of alpha*T_h: -4 alpha (m+1)^2 sin^2(p pi / (2(m+1)))."""
    return -4.0 * alpha * (m + 1) ** 2 * math.sin(p * math.pi / (2 * (m + 1))) ** 2


# ---------------------------------------------------------------------------------------------
# Operators
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("mx,my,mz", [(5, 5, 5), (6, 4, 7), (1, 3, 2), (12, 12, 12)])
def test_stencil_sine_modes_closed_form(mx, my, mz):
    """Sine modes are exact eigenvectors of the Dirichlet 7-point Laplacian (closed form)."""
    alpha = 0.01
    p = W.heat(mx, 1, 1, my=my, mz=mz, extras=False)
    op = oracle.Operator(p)
    rng = np.random.default_rng(0)
    for _ in range(4):
        px, py, pz = rng.integers(1, mx + 1), rng.integers(1, my + 1), rng.integers(1, mz + 1)
        phi = np.einsum("k,j,i->kji", sine_mode(mz, pz), sine_mode(my, py), sine_mode(mx, px)).ravel()
        lam = lam1(mx, px, alpha) + lam1(my, py, alpha) + lam1(mz, pz, alpha)
        y = op.apply(phi)
        assert np.max(np.abs(y - lam * phi)) <= 1e-13 * abs(lam) * np.max(np.abs(phi)) + 1e-300


def test_stencil_matches_kronecker_sum():
    p = W.heat(7, 2, 1, my=5, mz=6, extras=False)
    A = kron_laplacian(7, 5, 6, 0.01)
    u = np.random.default_rng(1).standard_normal(7 * 5 * 6)
    y = oracle.Operator(p).apply(u)
    assert np.allclose(y, A @ u, rtol=1e-14, atol=1e-14 * np.abs(A @ u).max())


def test_csr_apply_examples_and_scipy():
    # SPEC example: [[0,1],[-1,0]] (3,4) = (4,-3)
    p = {"op": "csr", "n": 2, "row_ptr": np.array([0, 1, 2]), "col_idx": np.array([1, 0], dtype=np.int32),
         "val": np.array([1.0, -1.0]), "b": None}
    assert np.array_equal(oracle.Operator(p).apply(np.array([3.0, 4.0])), np.array([4.0, -3.0]))
    rp, ci, va, dense = W.random_csr(40, 6, seed=3)
    p = {"op": "csr", "n": 40, "row_ptr": rp, "col_idx": ci, "val": va, "b": None}
    x = np.random.default_rng(2).standard_normal(40)
    assert np.allclose(oracle.Operator(p).apply(x), dense @ x, rtol=1e-14, atol=1e-13)


def test_lifting_is_augmented_matrix():
    """A' = [[A, b], [0, 0]]; the extra coordinate stays 1."""
    rp, ci, va, dense = W.random_csr(10, 4, seed=5)
    b = np.random.default_rng(6).uniform(-1, 1, 10)
    p = {"op": "csr", "n": 10, "row_ptr": rp, "col_idx": ci, "val": va, "b": b}
    Ap = np.zeros((11, 11))
    Ap[:10, :10] = dense
    Ap[:10, 10] = b
    x = np.random.default_rng(7).standard_normal(11)
    y = oracle.Operator(p).apply(x)
    assert y[10] == 0.0
    assert np.allclose(y, Ap @ x, rtol=1e-14, atol=1e-13)


# ---------------------------------------------------------------------------------------------
# Small expm
# ---------------------------------------------------------------------------------------------
def test_expm_identities_and_scipy():
    k = 9
    assert np.array_equal(oracle.expm(np.zeros((k, k))), np.eye(k))  # e^0 = I exactly
    d = np.array([-3.0, -0.5, 0.0, 1.0, 2.5])
    assert np.allclose(oracle.expm(np.diag(d)), np.diag(np.exp(d)), rtol=1e-14, atol=0)
    rng = np.random.default_rng(0)
    for scale in (0.1, 3.0, 50.0):
        M = rng.standard_normal((k, k)) * scale / k
        F = oracle.expm(M)
        S = sla.expm(M)
        assert np.max(np.abs(F - S)) <= 1e-12 * np.max(np.abs(S))
        assert np.allclose(oracle.expm(M.T), F.T, rtol=1e-12, atol=1e-12 * np.abs(F).max())
        if scale <= 3.0:
            assert np.allclose(F @ oracle.expm(-M), np.eye(k), atol=1e-12)


def test_expm_large_norm_symmetric_mpmath():
    """Symmetric negative definite H with eigenvalues over 7 decades, ||H t|| up to 2e6 (C5 scale):
    against a 40-digit mpmath expm. Scaling and squaring with ||.|| <= 1/2 needs up to 23 squarings
    here; the rounding error grows ~2^s eps, measured 1.2e-10 at t=20 (scipy's Pade-13, 3 fewer
    squarings: 1.0e-11), so the pin is 2e-10 of max(1, |ref|)."""
    import mpmath as mp
    rng = np.random.default_rng(1)
    Q, _ = np.linalg.qr(rng.standard_normal((30, 30)))
    lam = -np.logspace(-2, 5, 30)
    H = (Q * lam) @ Q.T
    H = 0.5 * (H + H.T)
    mp.mp.dps = 40
    for t, tol in ((0.02, 2e-12), (1.0, 5e-11), (20.0, 2e-10)):
        E = mp.expm(mp.matrix(H * t))
        ref = np.array([float(E[i, 0]) for i in range(30)])
        x = oracle.expm(H * t)[:, 0]
        assert np.max(np.abs(x - ref)) <= tol * max(1.0, np.abs(ref).max())


def test_expm_semigroup():
    """e^{H(t+s)} = e^{Hs} e^{Ht}."""
    rng = np.random.default_rng(4)
    H = rng.standard_normal((12, 12))
    X = oracle.expm_e1_times(H, 0.05, 40)
    E = oracle.expm(H * 0.05)
    for j in range(40):
        assert np.allclose(E @ X[j], X[j + 1], rtol=1e-12, atol=1e-12 * np.abs(X[j + 1]).max())


# ---------------------------------------------------------------------------------------------
# Lanczos / Arnoldi
# ---------------------------------------------------------------------------------------------
def identity_rows(n):
    return [W.sparse([i], [1.0]) for i in range(n)]


def test_arnoldi_krylov_relation_and_orthonormality():
    rp, ci, va, dense = W.random_csr(60, 8, seed=11)
    p = {"op": "csr", "n": 60, "row_ptr": rp, "col_idx": ci, "val": va, "b": None, "outs": identity_rows(60)}
    v = np.random.default_rng(12).standard_normal(60)
    k = 20
    r = oracle.arnoldi(p, v, k)
    V = r["P"]  # C = I so P = V_k
    Hf = r["Hfull"]
    # single-pass MGS loses orthogonality ~ eps * cond(Krylov basis) (measured 1.4e-8 here)
    assert np.allclose(V.T @ V, np.eye(k), atol=1e-7)
    R = dense @ V - V @ Hf[:k, :k]
    # the residual lives only in the last column with norm h_{k+1,k}
    assert np.max(np.abs(R[:, :-1])) <= 1e-12 * (1 + np.abs(dense).sum(axis=0).max())
    assert abs(np.linalg.norm(R[:, -1]) - Hf[k, k - 1]) <= 1e-12 * (1 + Hf[k, k - 1])
    assert np.allclose(V[:, 0], v / np.linalg.norm(v), atol=1e-15)
    assert np.allclose(np.triu(Hf[:k, :k].T, 2), 0.0)  # Hessenberg


def test_lanczos_equals_arnoldi_on_symmetric_input():
    p = W.heat(6, 2, 10, extras=False)
    p["outs"] = identity_rows(216)
    v = np.random.default_rng(5).standard_normal(216)
    la = oracle.lanczos(p, v, 10)
    ar = oracle.arnoldi(p, v, 10)
    assert np.allclose(la["H"], ar["H"], rtol=1e-9, atol=1e-9 * np.abs(ar["H"]).max())
    assert np.allclose(la["P"], ar["P"], atol=1e-9)
    assert np.allclose(la["H"], la["H"].T)


def test_lanczos_eigenvector_start_breaks_down():
    """Start = sine mode -> breakdown after one step with H = [lambda]."""
    m = 8
    p = W.heat(m, 1, 10, extras=False)
    p["outs"] = [W.allv()]
    phi = np.einsum("k,j,i->kji", sine_mode(m, 2), sine_mode(m, 1), sine_mode(m, 3)).ravel()
    lam = lam1(m, 3, 0.01) + lam1(m, 1, 0.01) + lam1(m, 2, 0.01)
    for fn in (oracle.lanczos, oracle.arnoldi):
        r = fn(p, phi, 10)
        assert r["k_eff"] == 1
        assert abs(r["H"][0, 0] - lam) <= 1e-13 * abs(lam)


def test_lanczos_diag_exact_at_full_dimension():
    """diag(1,2,3), v=(1,1,1)/sqrt(3), k=3: exact vs diagonal expm."""
    p = {"op": "csr", "n": 3, "row_ptr": np.array([0, 1, 2, 3]), "col_idx": np.array([0, 1, 2], dtype=np.int32),
         "val": np.array([1.0, 2.0, 3.0]), "b": None, "outs": identity_rows(3),
         "gens": [W.sparse([0, 1, 2], [1 / math.sqrt(3)] * 3)], "z_lo": [0.0], "z_hi": [1.0],
         "center": None, "step": 0.1, "n_steps": 10, "k": 3, "method": "lanczos", "thresholds": []}
    res = oracle.krylov_project(p)
    for j, t in enumerate(res["times"]):
        exact = np.exp(np.array([1.0, 2.0, 3.0]) * t) / math.sqrt(3)
        assert np.allclose(res["coeff"][j, :, 0], exact, rtol=1e-12)


def test_scale_invariance():
    p = W.heat(5, 2, 8, extras=True)
    v = W.dense_vec(p["gens"][0], p)
    a = oracle.lanczos(p, v, 8)
    b = oracle.lanczos(p, 4.0 * v, 8)  # power-of-two scale: bitwise identical basis
    assert np.array_equal(a["H"], b["H"]) and np.array_equal(a["P"], b["P"])
    assert b["beta0"] == 4.0 * a["beta0"]


def test_first_lanczos_step_closed_form():
    """Corner block b^3, Dirichlet stencil, c = alpha (m+1)^2: alpha_1 = -6c/b and
    beta_1^2 = c^2 [sum_{s=0..3} C(3,s) 2^s (b-2)^{3-s} (6/b - s)^2 + 3 b^2] / b^3 (cell counting,
    SURVEY A.16); first projections: total heat b^1.5, corner b^-1.5, cell (b,b,b) 0."""
    for m, b in [(20, 4), (40, 4), (100, 10), (12, 3)]:
        p = W.heat(m, b, 2)
        v = W.dense_vec(p["gens"][0], p)
        r = oracle.lanczos(p, v, 2)
        c = 0.01 * (m + 1) ** 2
        a1 = -6 * c / b
        s = sum(math.comb(3, q) * 2 ** q * (b - 2) ** (3 - q) * (6 / b - q) ** 2 for q in range(4))
        b1 = math.sqrt(c * c * (s + 3 * b * b) / b ** 3)
        assert abs(r["alpha"][0] - a1) <= 1e-13 * abs(a1)
        assert abs(r["beta"][0] - b1) <= 1e-13 * b1
        P1 = r["P"][:, 0]
        assert P1[0] == 0.0  # center cell far from the block
        assert abs(P1[1] - b ** 1.5) <= 1e-13 * b ** 1.5
        assert P1[2] == 0.0
        assert abs(P1[3] - b ** -1.5) <= 1e-15


# ---------------------------------------------------------------------------------------------
# Krylov approximant against the plain definition where they coincide
# ---------------------------------------------------------------------------------------------
def test_config1_matches_dense_expm():
    """C1 (n=125, only 25 distinct eigenvalues): k=30 >= Krylov dimension, so the Arnoldi result
    equals O e^{At} v_d; dense expm by scipy (library routine) on the Kronecker-sum matrix."""
    p = W.config1()
    res = oracle.krylov_project(p)
    A = kron_laplacian(5, 5, 5, 0.01).toarray()
    O = np.array([W.dense_vec(o, p) for o in p["outs"]])
    E = np.array([W.dense_vec(g, p) for g in p["gens"]]).T
    scale = np.abs(res["coeff"]).max()
    for j in range(0, p["n_steps"] + 1, 7):
        ref = O @ sla.expm(A * (j * p["step"])) @ E
        assert np.max(np.abs(res["coeff"][j] - ref)) <= 1e-12 * scale


def test_config1_verdicts():
    """C1: exact hi peak 0.0298306499842393895 at step 145 (mpmath); theta=0.05 SAFE;
    theta=0.02 UNSAFE first at step 74. Cross-checked here against scipy dense expm."""
    p = W.config1()
    res = oracle.krylov_project(p)
    cb = oracle.check_box(p, res["coeff"])
    assert not cb["found"]
    assert int(np.argmax(cb["hi"][:, 0])) == 145
    assert abs(cb["hi"][:, 0].max() - 0.0298306499842393895) <= 1e-14
    cb2 = oracle.check_box(p, res["coeff"], [(0, W.GE, 0.02)])
    assert cb2["found"] and cb2["step"] == 74
    A = kron_laplacian(5, 5, 5, 0.01).toarray()
    O = np.array([W.dense_vec(o, p) for o in p["outs"]])
    E = np.array([W.dense_vec(g, p) for g in p["gens"]]).T
    hi = lambda j: np.sum(np.maximum(0.9 * (O @ sla.expm(A * j * 0.02) @ E), 1.1 * (O @ sla.expm(A * j * 0.02) @ E)))
    assert hi(73) < 0.02 <= hi(74)
    assert abs(hi(145) - 0.0298306499842393895) <= 1e-14


def dst_heat_projection(m, b, t, alpha=0.01):
    """Closed form for a tensor-product start on the Dirichlet stencil: e^{At}(1_b x 1_b x 1_b) is
    the tensor product of 1-D solutions u(t) = S diag(e^{lam t}) S^T 1_b, S = orthonormal DST-I
    basis (separable eigendecomposition)."""
    x = np.arange(m)
    S = np.sqrt(2.0 / (m + 1)) * np.sin(np.outer(x + 1, np.arange(1, m + 1)) * np.pi / (m + 1))
    lam = np.array([lam1(m, q, alpha) for q in range(1, m + 1)])
    v = np.zeros(m)
    v[:b] = 1.0
    return S @ (np.exp(lam * t) * (S.T @ v))


def test_lanczos_converges_to_dst_closed_form():
    """Lanczos reaches the separable closed form at 1e-12 with k=60 (m=10)."""
    m, b = 10, 3
    p = W.heat(m, b, 60, n_steps=50, step=0.2)
    res = oracle.krylov_project(p)
    c = W.center_index(m)
    for j in range(0, 51, 5):
        u = dst_heat_projection(m, b, j * 0.2)
        exact = [u[c] ** 3, u.sum() ** 3, u[b] ** 3, u[0] ** 3]
        got = res["coeff"][j, :, 0]
        assert np.max(np.abs(got - np.array(exact))) <= 1e-11 * max(1.0, abs(exact[1]))


def test_t0_identity():
    """c[0][r][d] = C_r v_d: e^0 = I exactly."""
    p = W.config3(n_steps=3)
    p = dict(p, mx=30, my=30, mz=30, gens=[W.box((0, 0, 0), (5, 5, 5))], k=12,
             outs=[W.point(14, 14, 14), W.allv(), W.point(5, 5, 5), W.point(0, 0, 0), W.box((2, 2, 2), (9, 9, 9), 0.5)])
    res = oracle.krylov_project(p)
    assert res["coeff"][0, 0, 0] == 0.0 and res["coeff"][0, 2, 0] == 0.0
    assert abs(res["coeff"][0, 1, 0] - 125.0) <= 1e-12 * 125
    assert abs(res["coeff"][0, 3, 0] - 1.0) <= 1e-14
    assert abs(res["coeff"][0, 4, 0] - 0.5 * 27) <= 1e-13 * 13.5


def test_heat_invariants_dense():
    """Physics of P:973 on the converged path: 0 <= e^{At}v <= max v and total heat decreasing."""
    m, b = 8, 2
    p = W.heat(m, b, 100, n_steps=40, step=0.5)
    p["outs"] = [W.allv()] + [W.point(x, y, z) for (x, y, z) in [(0, 0, 0), (3, 3, 3), (7, 7, 7)]]
    res = oracle.krylov_project(p)
    tot = res["coeff"][:, 0, 0]
    assert np.all(np.diff(tot) <= 1e-12 * tot[0])
    pts = res["coeff"][:, 1:, 0]
    assert np.all(pts >= -1e-13) and np.all(pts <= 1 + 1e-13)


# ---------------------------------------------------------------------------------------------
# The paper's worked example (Fig. 2, §2.2, §3, §4.1)
# ---------------------------------------------------------------------------------------------
def test_oscillator_paper_example():
    g = json.load(open(os.path.join(GOLD, "oscillator.json")))
    p = W.oscillator()
    res = oracle.krylov_project(p)
    # basis row at 3pi/4 (Fig. 2c): columns (i_y, i_f)
    row = res["coeff"][3, 0, :]
    assert np.allclose(row, g["basis_row_3pi4"]["value"], atol=g["basis_row_3pi4"]["printed_digits_tol"])
    cb = oracle.check_box(p, res["coeff"])
    assert cb["found"] and cb["step"] == g["first_unsafe_step"]["value"]
    for j in g["infeasible_steps"]["value"]:
        assert not (cb["lo"][j, 0] <= 4.0 <= cb["hi"][j, 0])
    # x0 = (-5, y0, 0, 1): y0 = z_y
    assert abs(cb["z"][0] - g["x0"]["value"][1]) <= g["x0"]["printed_digits_tol"]
    assert abs(cb["z"][0] - (4 * math.sqrt(2) - 5)) <= 1e-12  # exact: y0 = 4 sqrt2 - 5
    # unsafe state (4, 3.07, 2.36, 1): simulate from x0 with full-state outputs
    q = dict(p, outs=[W.sparse([i], [1.0]) for i in range(4)])
    full = oracle.krylov_project(q)["coeff"][3]  # 4 x 2
    state = full @ cb["z"]
    assert np.allclose(state, g["unsafe_state"]["value"], atol=g["unsafe_state"]["printed_digits_tol"])
    # expm block of Fig. 2a: e^{A 3pi/4} columns from unit directions (full state, 4 simulations)
    Ap = np.array([[0, 1, 0, 0], [-1, 0, 0, 0], [0, 0, 0, 1], [0, 0, 0, 0]], dtype=float)
    F = oracle.expm(Ap * 3 * math.pi / 4)
    assert np.allclose(F[:2, :2], g["expAt_3pi4_block"]["value"], atol=g["expAt_3pi4_block"]["printed_digits_tol"])
    assert abs(F[2, 3] - g["expAt_3pi4_t_row_a_entry"]["value"]) <= g["expAt_3pi4_t_row_a_entry"]["printed_digits_tol"]
    # transpose simulation: simulate A^T from C^T = e_1
    assert np.allclose(F.T[:, 0], g["transpose_state_3pi4"]["value"], atol=g["transpose_state_3pi4"]["printed_digits_tol"])
    # Arnoldi from the y0 generator breaks down exactly (h_32 = 0, k_eff = 2)
    assert res["per_dir"][0]["k_eff"] == 2 and res["per_dir"][0]["h_next"] == 0.0


# ---------------------------------------------------------------------------------------------
# Box check = the LP of Fig. 2(c) for a box initial set and one output half-space
# ---------------------------------------------------------------------------------------------
def test_box_check_equals_lp():
    rng = np.random.default_rng(9)
    for trial in range(20):
        nd = int(rng.integers(1, 6))
        c = rng.standard_normal((1, 1, nd))
        zlo = rng.uniform(-2, 0, nd)
        zhi = zlo + rng.uniform(0, 2, nd)
        p = {"z_lo": zlo, "z_hi": zhi, "b": None, "center": None, "step": 1.0}
        cb = oracle.check_box(p, c, [])
        for sgn, key in ((1, "lo"), (-1, "hi")):
            r = linprog(sgn * c[0, 0], bounds=list(zip(zlo, zhi)), method="highs")
            assert abs(sgn * r.fun - cb[key][0, 0]) <= 1e-9 * (1 + np.abs(c).sum())
        # verdict + witness feasibility for each sense
        th = float(rng.uniform(cb["lo"][0, 0] - 1, cb["hi"][0, 0] + 1))
        for s in (W.GE, W.LE, W.EQ):
            cbs = oracle.check_box(p, c, [(0, s, th)])
            A_eq = c[0]
            if s == W.EQ:
                r = linprog(np.zeros(nd), A_eq=A_eq, b_eq=[th], bounds=list(zip(zlo, zhi)), method="highs")
            else:
                sign = -1.0 if s == W.GE else 1.0  # GE: -c z <= -th ; LE: c z <= th
                r = linprog(np.zeros(nd), A_ub=sign * A_eq, b_ub=[sign * th], bounds=list(zip(zlo, zhi)), method="highs")
            feasible = r.status == 0
            assert cbs["found"] == feasible
            if feasible:
                z = cbs["z"]
                assert np.all(z >= zlo - 1e-12) and np.all(z <= zhi + 1e-12)
                y = float(c[0, 0] @ z)
                assert abs(y - cbs["y"]) <= 1e-12 * (1 + abs(y))
                if s == W.GE:
                    assert y >= th - 1e-12
                elif s == W.LE:
                    assert y <= th + 1e-12
                else:
                    assert abs(y - th) <= 1e-9 * (1 + abs(th))


# ---------------------------------------------------------------------------------------------
# Lemma 1 diagnostic
# ---------------------------------------------------------------------------------------------
def test_lemma1_sound_on_heat():
    """bound >= actual full-state error (+ a rounding floor: the lemma is exact arithmetic)."""
    m, b = 12, 3
    for k in (10, 20, 40):
        p = W.heat(m, b, k, n_steps=100, step=0.05)
        n = m ** 3
        p["outs"] = identity_rows(n)
        res = oracle.krylov_project(p)
        A = kron_laplacian(m, m, m, 0.01).toarray()
        v = W.dense_vec(p["gens"][0], p)
        T = 100 * 0.05
        err = np.linalg.norm(sla.expm(A * T) @ v - res["coeff"][-1, :, 0])
        assert res["mu"] <= 0.0
        assert err <= res["lemma1"][0] + 1e-13 * np.linalg.norm(v)


def test_rand_field_splitmix64_reference_values():
    """The seeded dense field (include/krylov_reach.h KR_VEC_RAND): u_c is the (c+1)-th output of SplitMix64
    started at state `seed`, top 53 bits. Pinned to the generator's published first outputs for state 0
    (0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F, 0xF88BB8A8724C81EC), the stream property
    (seed + G shifts the stream by one), and uniformity on [0, 1)."""
    ref = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F, 0xF88BB8A8724C81EC]
    u = oracle._rand_field(0, 4, 1.0)
    assert [float(r >> 11) * 2.0 ** -53 for r in ref] == list(u)
    G = 0x9E3779B97F4A7C15
    a = oracle._rand_field(0, 1001, 2.5)
    b = oracle._rand_field(G, 1000, 2.5)
    assert np.array_equal(a[1:], b)
    big = oracle._rand_field(12345, 1 << 20, 1.0)
    assert big.min() >= 0.0 and big.max() < 1.0 and abs(big.mean() - 0.5) < 2e-3
    p = W.heat(6, 2, 3)
    assert np.array_equal(oracle.directions(dict(p, gens=[W.rand(7, 0.5)]))[0], oracle._rand_field(7, 216, 0.5))


def _diag_csr(lams):
    n = len(lams)
    return {"op": "csr", "n": n, "row_ptr": np.arange(n + 1, dtype=np.int64), "col_idx": np.arange(n, dtype=np.int32),
            "val": np.asarray(lams, dtype=np.float64), "b": None}


@pytest.mark.parametrize("lams,v,k", [((-1.0, -2.0), (3.0, 4.0), 1), ((-1.0, -2.5, 0.3), (1.0, -2.0, 0.5), 2),
                                      ((-0.5, -3.0, -1.2), (2.0, 1.0, -1.0), 2)])
def test_lemma1_closed_form_value(lams, v, k):
    """Lemma 1 as krylov_project reports it, against its value in closed form: A = diag(lams)
    (so mu = max lams exactly), start v with ||v|| != 1. Lanczos is written out here from its definition
    (alpha_1 = q1'Aq1, beta_1 = ||Aq1 - alpha_1 q1||, ...); for k = 1, x(t) = e^{alpha_1 t}; for k = 2 the
    2 x 2 symmetric H has x_2(t) = beta_1 (e^{th1 t} - e^{th2 t}) / (th1 - th2) >= 0, integrated exactly.
    bound = ||v|| h_{k+1,k} e^{max(mu,0) T} int_0^T |x_k| dt; the trapezoid rule is within ~d^2 |H|^2 / 12."""
    A = np.diag(lams)
    v = np.asarray(v, dtype=np.float64)
    q1 = v / np.linalg.norm(v)
    a1 = q1 @ A @ q1
    r1 = A @ q1 - a1 * q1
    b1 = np.linalg.norm(r1)
    T, N = 2.0, 4000
    if k == 1:
        h_next = b1
        integral = (math.exp(a1 * T) - 1.0) / a1
    else:
        q2 = r1 / b1
        a2 = q2 @ A @ q2
        h_next = np.linalg.norm(A @ q2 - a2 * q2 - b1 * q1)
        tr, det = a1 + a2, a1 * a2 - b1 * b1
        th1 = 0.5 * (tr + math.sqrt(tr * tr - 4 * det))
        th2 = 0.5 * (tr - math.sqrt(tr * tr - 4 * det))
        integral = b1 / (th1 - th2) * ((math.exp(th1 * T) - 1) / th1 - (math.exp(th2 * T) - 1) / th2)
    exact = np.linalg.norm(v) * h_next * math.exp(max(max(lams), 0.0) * T) * integral
    p = dict(_diag_csr(lams), name="diag", gens=[W.sparse(np.arange(len(v)), v)], z_lo=[1.0], z_hi=[1.0], center=None,
             outs=[W.sparse([0], [1.0])], step=T / N, n_steps=N, k=k, method="lanczos", thresholds=[])
    res = oracle.krylov_project(p)
    assert res["per_dir"][0]["k_eff"] == k
    assert abs(res["lemma1"][0] - exact) <= 2e-7 * exact, (res["lemma1"][0], exact)


def test_output_rows_csr_box_all_sparse():
    """P_{r,i} = C_r V_{*,i} (Alg. 4) with compact rows on a CSR operator, lifted and not: a box row
    [lo, hi) (clipped to the unlifted length n: the lifted coordinate never belongs to an output row), an
    all-ones row and a sparse row, against the dense row vector dotted with v by numpy."""
    import ctypes as C
    n = 50
    rp, ci, va, _ = W.random_csr(n, 4, seed=5)
    v = np.random.default_rng(9).standard_normal(n + 1)
    rows = [W.box((3,), (17,), 0.5), W.box((-4,), (9,), 2.0), W.box((40,), (n + 7,), -1.5), W.box((20,), (20,), 1.0),
            W.allv(0.25), W.sparse([0, 7, n - 1], [1.0, -2.0, 3.0])]
    for b in (None, np.linspace(-0.1, 0.1, n)):
        p = {"op": "csr", "n": n, "row_ptr": rp, "col_idx": ci, "val": va, "b": b, "outs": rows}
        op = oracle.Operator(p)
        N = n + (b is not None)
        crow, keep = oracle._rows(p)
        for r, row in enumerate(rows):
            dense = np.zeros(N)
            if row["kind"] == "box":
                dense[max(row["lo"][0], 0):min(row["hi"][0], n)] = row["value"]
            elif row["kind"] == "all":
                dense[:n] = row["value"]
            else:
                dense[np.asarray(row["idx"])] = row["val"]
            got = oracle.lib().oracle_row_dot(C.byref(op.s), C.byref(crow[r]), v[:N].ctypes.data)
            assert abs(got - dense @ v[:N]) <= 1e-14 * (1 + np.abs(dense) @ np.abs(v[:N])), (r, b is None)


def test_gershgorin_mu_upper_bounds_symmetric_part():
    rp, ci, va, dense = W.random_csr(30, 5, seed=21)
    b = np.random.default_rng(3).uniform(-0.1, 0.1, 30)
    p = {"op": "csr", "n": 30, "row_ptr": rp, "col_idx": ci, "val": va, "b": b}
    Ap = np.zeros((31, 31))
    Ap[:30, :30] = dense
    Ap[:30, 30] = b
    lam = np.linalg.eigvalsh(0.5 * (Ap + Ap.T)).max()
    assert oracle.gershgorin_mu(p) >= lam - 1e-12
    ph = W.heat(6, 2, 3)
    lamh = np.linalg.eigvalsh(kron_laplacian(6, 6, 6, 0.01).toarray()).max()
    assert oracle.gershgorin_mu(ph) >= lamh


# ---------------------------------------------------------------------------------------------
# NEXT-1: the paper's heat benchmark (insulated faces + Robin exchange at x = 1) and adaptive k
# ---------------------------------------------------------------------------------------------
def paper_matrix(m):
    """Independent construction of the SURVEY A2 reading: Neumann (dropped neighbour) Laplacian,
    x = 1 face diagonal -0.5/h, times 0.01."""
    h = 1.0 / (m + 1)

    def t1n(k):
        d = -2 * np.ones(k)
        d[0] = d[-1] = -1
        return sp.diags([np.ones(k - 1), d, np.ones(k - 1)], [-1, 0, 1]) / h ** 2
    I = sp.identity(m)
    L = sp.kron(I, sp.kron(I, t1n(m))) + sp.kron(I, sp.kron(t1n(m), I)) + sp.kron(t1n(m), sp.kron(I, I))
    rob = np.zeros(m)
    rob[-1] = 0.5 / h
    return (0.01 * (L - sp.kron(I, sp.kron(I, sp.diags(rob))))).tocsr()


def frobenius_by_coloring(op, m):
    """||A||_F^2 = sum_s ||A v_s||^2 with v_s the indicator of colour s of the perfect-code 7-colouring
    (x + 2y + 3z) mod 7 of the 7-point stencil graph: same-colour cells have disjoint closed
    neighbourhoods, so the columns A e_c of one colour do not overlap."""
    z, y, x = np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij")
    col = ((x + 2 * y + 3 * z) % 7).ravel()
    return math.sqrt(sum(np.sum(op.apply((col == s).astype(float)) ** 2) for s in range(7)))


def test_paper_heat_operator():
    p = W.heat_paper(9)
    A = paper_matrix(9)
    u = np.random.default_rng(3).standard_normal(9 ** 3)
    assert np.allclose(oracle.Operator(p).apply(u), A @ u, rtol=1e-13, atol=1e-13 * np.abs(A @ u).max())
    assert abs(frobenius_by_coloring(oracle.Operator(p), 9) - sp.linalg.norm(A)) <= 1e-12 * sp.linalg.norm(A)


def test_paper_heat_norm_at_t50():
    """'At time 50, this system has matrix norm ||At|| = 32771611' (m = 100; Frobenius norm,
    SURVEY A2). The oracle operator reproduces it to 3.2e-8 relative."""
    nrm = 50 * frobenius_by_coloring(oracle.Operator(W.heat_paper(100)), 100)
    assert abs(nrm - 32771611) <= 1e-7 * 32771611


def test_checkpoint_sequence():
    """fp64 ceil(1.1 k) from 4 (Alg. 2): contains the paper's k = 63, 544,
    5932; the exact-rational sequence would not contain 544."""
    ks = oracle.checkpoints(7000)
    assert ks[:10] == [4, 5, 6, 7, 8, 9, 10, 11, 13, 15]
    for k in (63, 544, 5932):
        assert k in ks


def test_eig_route_equals_pade_route():
    """The large-k exponential route (tridiagonal eigendecomposition) equals the per-step Pade route."""
    p = W.heat(20, 3, 30, n_steps=100, step=0.05)
    r = oracle.lanczos(p, oracle.directions(p)[0], 30)
    X1 = oracle.eig_e1_times(r["alpha"], r["beta"], 0.05, 100)
    X2 = oracle.expm_e1_times(r["H"], 0.05, 100)
    assert np.array_equal(X1[0], X2[0])  # t = 0 exactly e_1 on both routes
    assert np.max(np.abs(X1 - X2)) <= 1e-12


def test_lemma1_sound_on_paper_operator():
    p = W.heat_paper(12, n_steps=100, step=0.05)  # m >= 10 so the heated region is non-empty in z
    A = paper_matrix(12).toarray()
    v = oracle.directions(p)[0]
    v = v / np.linalg.norm(v)
    for k in (8, 16, 24):
        r = oracle.lanczos(dict(p, outs=identity_rows(12 ** 3)), v, k)
        X = oracle.eig_e1_times(r["alpha"], r["beta"], 0.05, 100)
        b = oracle.lemma1_bound(r["h_next"], X, 0.05, oracle.gershgorin_mu(p))
        err = np.linalg.norm(sla.expm(A * 5.0) @ v - r["P"] @ X[-1])
        assert err <= b + 1e-13


def test_adaptive_k_reproduces_paper_m100():
    """P:1032-1033 (Fig. 6): 'Once k = 544 iterations have been performed, the computed error bound is
    5.8e-7, which is below the desired error threshold of 1e-6' (m = 100). The oracle stops at k = 544
    exactly; its bound is 5.90e-7 (quadrature-converged — the 1.7% gap to the printed value is a reading
    difference of the unstated discretisation details, DESIGN R18); the previous checkpoint (494) is 8.2e-6."""
    p = W.heat_paper(100, k_max=560)
    r = oracle.lanczos_adaptive(p, oracle.directions(p)[0], 1e-6, 560)
    assert r["k_eff"] == 544
    assert abs(r["bound"] - 5.8e-7) <= 0.02 * 5.8e-7
    assert r["checks"][-2][0] == 494 and r["checks"][-2][1] > 1e-6


# ---------------------------------------------------------------------------------------------
# NEXT-2: transpose dynamics, min(i, o) simulations (§4.1)
# ---------------------------------------------------------------------------------------------
def test_transpose_oscillator_paper_example():
    """one simulation of A^T from the output direction, projected with E^T, gives the basis
    row (0.707, 3.54) at 3pi/4; same verdict (unsafe at step 3) and witness y0 = 4 sqrt2 - 5."""
    g = json.load(open(os.path.join(GOLD, "oscillator.json")))
    p = W.oscillator()
    res = oracle.krylov_project_transpose(p)
    assert len(res["per_dir"]) == 1  # o = 1 simulation instead of i + 1 = 2
    row = res["coeff"][3, 0, :]
    assert np.allclose(row, g["basis_row_3pi4"]["value"], atol=g["basis_row_3pi4"]["printed_digits_tol"])
    cb = oracle.check_box(p, res["coeff"])
    assert cb["found"] and cb["step"] == g["first_unsafe_step"]["value"]
    assert abs(cb["z"][0] - (4 * math.sqrt(2) - 5)) <= 1e-12


def test_transpose_problem_matrix_is_lifted_transpose():
    """The explicit A'^T equals the transpose of the augmented matrix [[A, b], [0, 0]], built
    independently with numpy."""
    rp, ci, va, dense = W.random_csr(30, 4, seed=3)
    b = np.random.default_rng(4).uniform(-1, 1, 30)
    p = {"op": "csr", "n": 30, "row_ptr": rp, "col_idx": ci, "val": va, "b": b, "gens": [W.sparse([0], [1.0])],
         "z_lo": [0.0], "z_hi": [1.0], "center": None, "outs": [W.allv()], "step": 0.1, "n_steps": 3, "k": 4,
         "method": "arnoldi"}
    q = oracle.transpose_problem(p)
    Aq = sp.csr_matrix((q["val"], q["col_idx"], q["row_ptr"]), shape=(31, 31)).toarray()
    Ap = np.zeros((31, 31))
    Ap[:30, :30] = dense
    Ap[:30, 30] = b
    assert np.array_equal(Aq, Ap.T)


@pytest.mark.parametrize("seed", [0, 1])
def test_transpose_equals_dense_expm_when_exact(seed):
    """Random affine CSR system (n = 24, lifted to 25), 5 generators + center, 3 output rows, k = 25 >= the
    Krylov dimension: forward (6 simulations) and transpose (3 simulations) both equal C' e^{A' t} E (scipy)."""
    n = 24
    rp, ci, va, dense = W.random_csr(n, 4, seed=seed, scale=0.5)
    rng = np.random.default_rng(seed + 10)
    b = rng.uniform(-1, 1, n)
    p = {"name": "rnd", "op": "csr", "n": n, "row_ptr": rp, "col_idx": ci, "val": va, "b": b,
         "gens": [W.sparse([i], [1.0]) for i in range(5)], "z_lo": -np.ones(5), "z_hi": np.ones(5),
         "center": W.sparse([7, 9], [0.5, -1.0]),
         "outs": [W.sparse(list(range(n)), list(rng.standard_normal(n))) for _ in range(3)],
         "step": 0.05, "n_steps": 40, "k": n + 1, "method": "arnoldi", "thresholds": []}
    fw = oracle.krylov_project(p)["coeff"]
    tr = oracle.krylov_project_transpose(p)["coeff"]
    Ap = np.zeros((n + 1, n + 1))
    Ap[:n, :n] = dense
    Ap[:n, n] = b
    C = np.zeros((3, n + 1))
    for r, o in enumerate(p["outs"]):
        C[r, o["idx"]] = o["val"]
    E = np.array(oracle.directions(p)).T
    scale = np.abs(fw).max()
    for j in range(0, 41, 5):
        ref = C @ sla.expm(Ap * (j * 0.05)) @ E
        assert np.max(np.abs(fw[j] - ref)) <= 1e-11 * scale
        assert np.max(np.abs(tr[j] - ref)) <= 1e-11 * scale


def test_transpose_config1_equals_dense_expm():
    """C1: o = 1 simulation of the (symmetric) stencil from the center cell, projected on the 8 unit
    generators, equals O e^{At} E (scipy) — one simulation instead of eight."""
    p = W.config1()
    res = oracle.krylov_project_transpose(p)
    assert len(res["per_dir"]) == 1
    A = kron_laplacian(5, 5, 5, 0.01).toarray()
    O = np.array([W.dense_vec(o, p) for o in p["outs"]])
    E = np.array([W.dense_vec(g, p) for g in p["gens"]]).T
    scale = np.abs(res["coeff"]).max()
    for j in range(0, p["n_steps"] + 1, 9):
        assert np.max(np.abs(res["coeff"][j] - O @ sla.expm(A * (j * p["step"])) @ E)) <= 1e-12 * scale


# ---------------------------------------------------------------------------------------------
# NEXT-3: general per-step LP (polytope initial set in z, polytope unsafe set in y)
# ---------------------------------------------------------------------------------------------
def brute_force_feasible(A, b, lo, hi, tol=1e-9):
    """Nonempty {z : A z <= b, lo <= z <= hi} by vertex enumeration (the box makes it bounded, so it is
    nonempty iff it has a vertex: i tight constraints with a nonsingular system)."""
    import itertools
    i = len(lo)
    G = np.vstack([A, np.eye(i), -np.eye(i)])
    h = np.concatenate([b, hi, -lo])
    for rows in itertools.combinations(range(len(h)), i):
        M = G[list(rows)]
        if abs(np.linalg.det(M)) < 1e-12:
            continue
        z = np.linalg.solve(M, h[list(rows)])
        if np.all(G @ z <= h + tol * (1 + np.abs(h))):
            return True, z
    return False, None


def test_lp_box_halfspace_equals_interval_check():
    """A box initial set with one output half-space: the LP verdict per step equals the closed-form
    interval check (the LP optimum of Fig. 2(c) for a box is sum max(c lo, c hi)) — C1, theta = 0.02."""
    p = W.config1()
    coeff = oracle.krylov_project(p)["coeff"]
    lp = oracle.check_lp(p, coeff, unsafe_A=[[-1.0]], unsafe_b=[-0.02])  # y >= 0.02  <=>  -y <= -0.02
    cb = oracle.check_box(p, coeff, [(0, W.GE, 0.02)])
    hi = cb["hi"][:, 0]
    margin = np.abs(hi - 0.02) > 1e-9
    assert np.array_equal(lp["feasible"][margin], (hi >= 0.02)[margin])
    assert lp["found"] and lp["step"] == cb["step"] == 74


def test_lp_oscillator_paper_constraints():
    """Fig. 2(c): z_y in [0, 1], fixed term, unsafe x = 4 as x <= 4 and -x <= -4: infeasible at
    steps 0-2, feasible at 3pi/4 with the witness output x = 4."""
    p = W.oscillator()
    coeff = oracle.krylov_project(p)["coeff"]
    lp = oracle.check_lp(p, coeff, unsafe_A=[[1.0], [-1.0]], unsafe_b=[4.0, -4.0])
    assert list(lp["feasible"][:4]) == [False, False, False, True]
    assert lp["step"] == 3 and abs(lp["y"][0] - 4.0) < 1e-7
    assert abs(lp["z"][0] - (4 * math.sqrt(2) - 5)) < 1e-7  # the only feasible z_y


@pytest.mark.parametrize("seed", range(4))
def test_lp_matches_vertex_enumeration(seed):
    """Random 3-generator problems with a polytope initial set (2 extra rows) and a 2-row unsafe polytope
    in a 2-output space: per-step feasibility equals brute-force vertex enumeration (tiny instances)."""
    rng = np.random.default_rng(100 + seed)
    ng, o, N = 3, 2, 30
    coeff = rng.standard_normal((N + 1, o, ng + 1))
    p = {"gens": [W.sparse([d], [1.0]) for d in range(ng)], "z_lo": -np.ones(ng), "z_hi": np.ones(ng)}
    IA = rng.standard_normal((2, ng))
    Ib = np.abs(rng.standard_normal(2)) * 0.5
    UA = rng.standard_normal((2, o))
    Ub = rng.standard_normal(2)
    lp = oracle.check_lp(p, coeff, IA, Ib, UA, Ub)
    for j in range(N + 1):
        B, cf = coeff[j, :, :ng], coeff[j, :, ng]
        ok, _ = brute_force_feasible(np.vstack([IA, UA @ B]), np.concatenate([Ib, Ub - UA @ cf]), -np.ones(ng),
                                     np.ones(ng))
        assert ok == lp["feasible"][j], j
    if lp["found"]:
        z, j = lp["z"], lp["step"]
        B, cf = coeff[j, :, :ng], coeff[j, :, ng]
        assert np.all(IA @ z <= Ib + 1e-7) and np.all(UA @ (B @ z + cf) <= Ub + 1e-7)


# ---------------------------------------------------------------------------------------------
# NEXT-4: nonsymmetric heat with a permanent heater: lifted stencil, Arnoldi
# ---------------------------------------------------------------------------------------------
def heater_augmented(m):
    """[[A, b], [0, 0]] built independently: the paper heat matrix (Kronecker sum + face terms) and the
    heater column b = 0.01 (m+1) on the z = 0 cells with x_i <= 0.4, y_j <= 0.2 (DESIGN R19)."""
    A = paper_matrix(m).toarray()
    n = m ** 3
    b = np.zeros(n)
    nx, ny = int(np.floor(0.4 * (m + 1) + 1e-9)), int(np.floor(0.2 * (m + 1) + 1e-9))
    for y in range(ny):
        for x in range(nx):
            b[x + m * y] = 0.01 * (m + 1)
    M = np.zeros((n + 1, n + 1))
    M[:n, :n] = A
    M[:n, n] = b
    return M


def test_heater_lifted_operator():
    p = W.heat_heater(6)
    op = oracle.Operator(p)
    M = heater_augmented(6)
    rng = np.random.default_rng(5)
    for _ in range(3):
        x = rng.standard_normal(op.dim)
        assert np.allclose(op.apply(x), M @ x, rtol=1e-13, atol=1e-12)


def test_heater_equals_dense_expm():
    """m = 4 (n' = 65), k = 65 >= the Krylov dimension: Arnoldi from e_{n'} equals C e^{A' t} e_{n'} (scipy)
    at every step up to T = 500; the lifted coordinate stays 1."""
    p = W.heat_heater(4, k=65)
    res = oracle.krylov_project(p)
    M = heater_augmented(4)
    C = np.array([W.dense_vec(o, p) for o in p["outs"]])
    e = np.zeros(65)
    e[64] = 1.0
    E1 = sla.expm(M * p["step"])
    x = e.copy()
    scale = np.abs(res["coeff"]).max()
    for j in range(p["n_steps"] + 1):
        if j % 50 == 0:
            assert np.max(np.abs(res["coeff"][j, :, 0] - C @ x[:64])) <= 1e-10 * scale, j
            assert abs(x[64] - 1.0) < 1e-12
        x = E1 @ x


def test_adaptive_arnoldi_sound_against_dense_expm():
    """Alg. 2 on a nonsymmetric system with mu < 0: the accepted approximation is within its Lemma-1 bound
    (x ||v||, unit-vector bound) of the exact C e^{At} v (scipy dense expm, n = 400), at every 20th step;
    the accepted k is the first checkpoint below eps."""
    p = W.csr_stable_nonsym(n_steps=100, step=0.05, scale=5.0, shift=0.01)
    assert oracle.gershgorin_mu(p) < 0
    res = oracle.krylov_project_adaptive(p)
    A = sp.csr_matrix((p["val"], p["col_idx"], p["row_ptr"]), shape=(400, 400)).toarray()
    C = np.zeros((2, 400))
    for r, o in enumerate(p["outs"]):
        C[r, o["idx"]] = o["val"]
    dirs = oracle.directions(p)
    for d, r in enumerate(res["per_dir"]):
        ks = [k for k, _ in r["checks"]]
        assert ks == oracle.checkpoints(ks[-1])[:len(ks)] and r["checks"][-1][1] < p["eps"]
        assert all(b >= p["eps"] for _, b in r["checks"][:-1])
        for j in range(0, p["n_steps"] + 1, 20):
            exact = C @ sla.expm(A * (j * p["step"])) @ dirs[d]
            err = np.abs(res["coeff"][j, :, d] - exact)
            # ||C (x - x_k)|| <= ||C|| ||x - x_k|| <= ||C||_2 ||v|| bound
            assert np.max(err) <= np.linalg.norm(C, 2) * r["beta0"] * r["bound"] + 1e-12, (d, j)


def test_a_priori_bound_and_memory_formulas():
    """at ||At|| = 32771611 even k = 10^6 gives an a priori bound of 10^16182319 (the printed value;
    SURVEY A.1: 16182318.694); storing V for k = 5932 at n = 10^9 needs 46 TB (Eq. 4); Alg. 4's
    Eq. 6 memory for the same run is three vectors (24 GB)."""
    v = oracle.a_priori_bound_log10(32771611, 10 ** 6)
    assert abs(v - 16182318.694) < 1e-3 and round(v) == 16182319
    m = oracle.memory_bytes(10 ** 9, 5932, method="arnoldi")
    assert m == 5932 * (10 ** 9 + 5932) * 8 and round(m / 2 ** 40) == 43 and round(m / 1e12) == 47  # "46 TB"
    assert 45.5e12 < m < 47.5e12
    assert oracle.memory_bytes(10 ** 9, 5932, 1, 1, "lanczos") == (3 * 5932 + 4 * 10 ** 9) * 8
