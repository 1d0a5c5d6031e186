"""CPU fp64 oracle for the Krylov projected-reachability hot path of arXiv 1804.01583.

TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package. The product path (paper_1804_01583_b200/) never
imports it, and the two share no code: the numerics live in oracle/krylov_oracle.c (plain C, fp64,
single thread, -ffp-contract=off) and in the plain numpy orchestration below.

What it computes (PAPER.md, "P:<line>"):
  * directions v_d: generator columns of E (§3.2), plus the fixed-term direction
    v_f = [c; 1] when there is a center c or an affine term b (lifting P:157-165, superposition of
    fixed terms P:1197-1225);
  * per direction, k steps of Arnoldi (Alg. 1) or Lanczos (Alg. 3/4) with the
    projection P = C V (Alg. 4);
  * per time point t_j = j*step, x_{d,j} = e^{H t_j} e_1 (Eq. 2) by Pade scaling and
    squaring and the basis-matrix entries c[j][r][d] = ||v_d|| (P_d x_{d,j})_r
    (= C e^{A t_j} E in the Krylov approximation, §3);
  * the per-step safety check specialised to a box initial set and one output half-space, i.e. the
    exact LP value max/min over the box (Fig. 2(c)), first violating step
    and witness;
  * the Lemma 1 a posteriori bound as a diagnostic.
Readings of ambiguous passages are SURVEY.md §8(c) A1-A20 and are listed in DESIGN.md.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "krylov_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

GE, LE, EQ = 0, 1, 2


def build(force=False):
    """Compile the C oracle with gcc (plain -O2, no FMA contraction, no vectorised reassociation)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c99",
                               "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Op(C.Structure):
    _fields_ = [("op", C.c_int32), ("mx", C.c_int64), ("my", C.c_int64), ("mz", C.c_int64),
                ("alpha", C.c_double), ("n", C.c_int64), ("row_ptr", C.c_void_p),
                ("col_idx", C.c_void_p), ("val", C.c_void_p), ("b", C.c_void_p),
                ("bc", C.c_int32 * 6), ("gamma", C.c_double * 6)]


class _Row(C.Structure):
    _fields_ = [("kind", C.c_int32), ("nnz", C.c_int64), ("idx", C.c_void_p), ("val", C.c_void_p),
                ("lo", C.c_int64 * 3), ("hi", C.c_int64 * 3), ("value", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        dp = C.POINTER(C.c_double)
        _lib.oracle_sum.restype = C.c_double
        _lib.oracle_sum.argtypes = [C.c_void_p, C.c_int64]
        _lib.oracle_dot.restype = C.c_double
        _lib.oracle_dot.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        _lib.oracle_op_dim.restype = C.c_int64
        _lib.oracle_op_dim.argtypes = [C.POINTER(_Op)]
        _lib.oracle_op_apply.argtypes = [C.POINTER(_Op), C.c_void_p, C.c_void_p]
        _lib.oracle_row_dot.restype = C.c_double
        _lib.oracle_row_dot.argtypes = [C.POINTER(_Op), C.POINTER(_Row), C.c_void_p]
        _lib.oracle_lanczos.argtypes = [C.POINTER(_Op), C.c_void_p, C.c_int32, C.c_int32, C.POINTER(_Row),
                                        C.c_void_p, C.c_void_p, C.c_void_p, dp, C.POINTER(C.c_int32)]
        _lib.oracle_arnoldi.argtypes = [C.POINTER(_Op), C.c_void_p, C.c_int32, C.c_int32, C.POINTER(_Row),
                                        C.c_void_p, C.c_void_p, dp, C.POINTER(C.c_int32)]
        _lib.oracle_expm.argtypes = [C.c_int32, C.c_void_p, C.c_void_p]
        _lib.oracle_expm_e1_times.argtypes = [C.c_int32, C.c_void_p, C.c_double, C.c_int64, C.c_void_p]
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


class Operator:
    """Keeps the numpy arrays alive next to the ctypes struct."""

    def __init__(self, p):
        self.p = p
        self.keep = []
        if p["op"] == "stencil":
            b = None if p.get("b") is None else np.ascontiguousarray(_dense(p["b"], p, p["mx"] * p["my"] * p["mz"])
                                                                     if isinstance(p["b"], dict) else p["b"],
                                                                     dtype=np.float64)
            self.keep.append(b)
            self.s = _Op(0, p["mx"], p["my"], p["mz"], p["alpha"], 0, None, None, None, _ptr(b),
                         (C.c_int32 * 6)(*p.get("bc", [0] * 6)), (C.c_double * 6)(*p.get("gamma", [0.0] * 6)))
        else:
            rp = np.ascontiguousarray(p["row_ptr"], dtype=np.int64)
            ci = np.ascontiguousarray(p["col_idx"], dtype=np.int32)
            va = np.ascontiguousarray(p["val"], dtype=np.float64)
            b = None if p.get("b") is None else np.ascontiguousarray(p["b"], dtype=np.float64)
            self.keep += [rp, ci, va, b]
            self.s = _Op(1, 0, 0, 0, 0.0, p["n"], _ptr(rp), _ptr(ci), _ptr(va), _ptr(b))
        self.dim = int(lib().oracle_op_dim(C.byref(self.s)))

    def apply(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.dim)
        lib().oracle_op_apply(C.byref(self.s), _ptr(x), _ptr(y))
        return y


def _rows(p):
    rows = (_Row * max(1, len(p["outs"])))()
    keep = []
    for r, v in enumerate(p["outs"]):
        if v["kind"] == "sparse":
            idx = np.ascontiguousarray(v["idx"], dtype=np.int64)
            val = np.ascontiguousarray(v["val"], dtype=np.float64)
            keep += [idx, val]
            rows[r] = _Row(0, idx.size, _ptr(idx), _ptr(val), (C.c_int64 * 3)(0, 0, 0),
                           (C.c_int64 * 3)(0, 0, 0), 0.0)
        elif v["kind"] == "all":
            rows[r] = _Row(2, 0, None, None, (C.c_int64 * 3)(0, 0, 0), (C.c_int64 * 3)(0, 0, 0), v["value"])
        else:
            rows[r] = _Row(1, 0, None, None, (C.c_int64 * 3)(*v["lo"]), (C.c_int64 * 3)(*v["hi"]), v["value"])
    return rows, keep


def _rand_field(seed, n, value, chunk=1 << 24):
    """The seeded dense field of include/krylov_reach.h KR_VEC_RAND, written out with numpy uint64 arithmetic
    (mod 2^64): u_c = (splitmix64 finaliser of seed + (c+1) G) >> 11, times 2^-53, times value."""
    out = np.empty(n)
    G = np.uint64(0x9E3779B97F4A7C15)
    M1, M2 = np.uint64(0xBF58476D1CE4E5B9), np.uint64(0x94D049BB133111EB)
    s30, s27, s31, s11 = np.uint64(30), np.uint64(27), np.uint64(31), np.uint64(11)
    for c0 in range(0, n, chunk):
        c = np.arange(c0 + 1, min(n, c0 + chunk) + 1, dtype=np.uint64)
        z = np.uint64(seed) + c * G
        z = (z ^ (z >> s30)) * M1
        z = (z ^ (z >> s27)) * M2
        z = z ^ (z >> s31)
        out[c0:c0 + len(c)] = (z >> s11).astype(np.float64) * (2.0 ** -53) * value
    return out


def _dense(v, p, n):
    """Dense materialisation of a compact vector (box / all / sparse entries / seeded field) of length n."""
    if v["kind"] == "rand":
        return _rand_field(int(v["seed"]), n, float(v["value"]))
    out = np.zeros(n)
    if v["kind"] == "all":
        out[:] = v["value"]
    elif v["kind"] == "sparse":
        for i, x in zip(v["idx"], v["val"]):
            out[int(i)] += x
    elif p["op"] == "stencil":
        g = out.reshape(p["mz"], p["my"], p["mx"])
        (x0, y0, z0), (x1, y1, z1) = v["lo"], v["hi"]
        g[z0:z1, y0:y1, x0:x1] = v["value"]
    else:
        out[v["lo"][0]:v["hi"][0]] = v["value"]
    return out


def directions(p):
    """Simulation directions: generator columns of E, plus the fixed-term direction
    v_f = [c; 1] (lifted) or v_f = c (no affine term) — superposition."""
    op = Operator(p)
    n = op.dim
    nb = n - 1 if p.get("b") is not None else n
    dirs = []
    for g in p["gens"]:
        v = np.zeros(n)
        v[:nb] = _dense(g, p, nb)
        dirs.append(v)
    if p.get("b") is not None or p.get("center") is not None:
        v = np.zeros(n)
        if p.get("center") is not None:
            v[:nb] = _dense(p["center"], p, nb)
        if n != nb:
            v[nb] = 1.0
        dirs.append(v)
    return dirs


def lanczos(p, v, k):
    """Alg. 3 + projection of Alg. 4 (see krylov_oracle.c). Returns dict(alpha, beta, P, beta0, k_eff)."""
    op = Operator(p)
    rows, keep = _rows(p)
    o = len(p["outs"])
    alpha = np.zeros(k)
    beta = np.zeros(k)
    P = np.zeros((max(o, 1), k))
    b0 = C.c_double()
    ke = C.c_int32()
    v = np.ascontiguousarray(v, dtype=np.float64)
    st = lib().oracle_lanczos(C.byref(op.s), _ptr(v), k, o, rows, _ptr(alpha), _ptr(beta), _ptr(P),
                              C.byref(b0), C.byref(ke))
    if st != 0:
        raise ValueError("zero start vector")
    kk = ke.value
    H = np.diag(alpha[:kk]) + np.diag(beta[:kk - 1], 1) + np.diag(beta[:kk - 1], -1)
    return {"alpha": alpha[:kk], "beta": beta[:kk], "H": H, "P": P[:o, :kk], "beta0": b0.value,
            "k_eff": kk, "h_next": beta[kk - 1]}


def arnoldi(p, v, k):
    """Alg. 1 with MGS (see krylov_oracle.c). Returns dict(H (k_eff x k_eff), P, beta0, k_eff, h_next)."""
    op = Operator(p)
    rows, keep = _rows(p)
    o = len(p["outs"])
    H = np.zeros((k + 1, k))
    P = np.zeros((max(o, 1), k))
    b0 = C.c_double()
    ke = C.c_int32()
    v = np.ascontiguousarray(v, dtype=np.float64)
    st = lib().oracle_arnoldi(C.byref(op.s), _ptr(v), k, o, rows, _ptr(H), _ptr(P), C.byref(b0), C.byref(ke))
    if st != 0:
        raise ValueError("zero start vector")
    kk = ke.value
    return {"H": H[:kk, :kk].copy(), "Hfull": H, "P": P[:o, :kk], "beta0": b0.value, "k_eff": kk,
            "h_next": H[kk, kk - 1]}


def expm(M):
    """Moler-Van Loan / Golub-Van Loan diagonal Pade (q=8) with scaling and squaring."""
    M = np.ascontiguousarray(M, dtype=np.float64)
    F = np.zeros_like(M)
    lib().oracle_expm(M.shape[0], _ptr(M), _ptr(F))
    return F


def expm_e1_times(H, step, n_steps):
    """x_j = e^{H t_j} e_1, t_j = (double)j*step, j = 0..n_steps (Eq. 2)."""
    H = np.ascontiguousarray(H, dtype=np.float64)
    k = H.shape[0]
    X = np.zeros((n_steps + 1, k))
    lib().oracle_expm_e1_times(k, _ptr(H), step, n_steps, _ptr(X))
    return X


def _exp_or_inf(x):
    """e^x, +inf past the fp64 range: Lemma 1's e^{max(mu,0) T} factor for lifted affine systems, whose
    Gershgorin mu is large (DESIGN R16: the bound is then astronomically loose, diagnostic only)."""
    return math.exp(x) if x < 709.0 else math.inf


def a_priori_bound_log10(norm_At, k):
    """log10 of the a priori Krylov error bound of Eq. 3, ||v|| ||At||^k e^{||At||} / k! for
    ||v|| = 1: k log10 x + x log10 e - log10 k! (lgamma)."""
    x = float(norm_At)
    return k * math.log10(x) + x * math.log10(math.e) - math.lgamma(k + 1) / math.log(10.0)


def memory_bytes(n, k, i=1, o=1, method="arnoldi"):
    """Memory of the Krylov iteration in bytes: Eq. 4 k (n + k) doubles for Arnoldi / plain
    Lanczos; Eq. 6 (3k + n min(i, o) + 3n) doubles for Lanczos with projection (Alg. 4)."""
    if method == "arnoldi":
        return k * (n + k) * 8
    return (3 * k + n * min(i, o) + 3 * n) * 8


def checkpoints(k_max):
    """Alg. 2/4 error-check points: k = 4, then k <- ceil(1.1 k) evaluated in
    fp64 (the paper's k = 63, 544, 5932 lie on this sequence, not on the exact-rational one)."""
    ks, k = [], 4
    while k <= k_max:
        ks.append(k)
        k = int(math.ceil(1.1 * k))
    return ks


def eig_e1_times(alpha, beta, step, n_steps):
    """x_j = e^{H t_j} e_1 for the symmetric tridiagonal H = tridiag(beta; alpha; beta) through its
    eigendecomposition (numpy eigh = LAPACK, a library primitive): x_j = Q e^{Lambda t_j} Q^T e_1 — the
    large-k route (k up to thousands, where per-step Pade is O(k^3) per t). t = 0 returns e_1 exactly
    (eigh's Q Q^T = I only to rounding)."""
    k = len(alpha)
    H = np.diag(alpha) + np.diag(beta[:k - 1], 1) + np.diag(beta[:k - 1], -1)
    lam, Q = np.linalg.eigh(H)
    t = np.arange(n_steps + 1) * step
    X = (np.exp(np.outer(t, lam)) * Q[0]) @ Q.T  # row j: sum_l e^{lam_l t_j} Q[0,l] Q[:,l]
    X[0] = 0.0
    X[0, 0] = 1.0
    return X


def lemma1_bound(h_next, X, step, mu=0.0):
    """Lemma 1 for a unit start vector at tau = T: h_{k+1,k} e^{max(mu,0) T}
    int_0^T |e_k^T e^{H t} e_1| dt, trapezoid on the t_j grid (reading: DESIGN R16)."""
    h = np.abs(X[:, -1])
    T = (X.shape[0] - 1) * step
    base = h_next * float(np.sum(0.5 * step * (h[1:] + h[:-1])))
    return 0.0 if base == 0.0 else base * _exp_or_inf(max(mu, 0.0) * T)


def lanczos_adaptive(p, v, eps, k_max):
    """Alg. 4 with error control: Lanczos with projection, error checked at the checkpoint
    sequence k = 4, ceil(1.1 k), ... (Alg. 2 lines 11-16), stopping at the first k whose Lemma-1 bound for
    the unit start vector is below eps. The first k steps of Lanczos do not depend on later steps, so
    one literal Alg. 3 run to k_max is cut at the accepted checkpoint. Returns the lanczos() dict for
    k_eff = accepted k, plus 'bound' (unit-vector bound) and 'checks' [(k, bound)]."""
    full = lanczos(p, v, k_max)
    mu = gershgorin_mu(p)
    checks = []
    kk = full["k_eff"]
    for k in checkpoints(kk):
        if k == kk and kk < k_max:  # exact breakdown before k_max: the approximation is exact
            break
        X = eig_e1_times(full["alpha"][:k], full["beta"][:k], p["step"], p["n_steps"])
        b = lemma1_bound(full["beta"][k - 1], X, p["step"], mu)
        checks.append((k, b))
        if b < eps:
            kk = k
            break
    else:
        if kk == k_max and (not checks or checks[-1][1] >= eps):
            raise RuntimeError("adaptive Krylov: k_max reached before the error target")
    r = {"alpha": full["alpha"][:kk], "beta": full["beta"][:kk], "P": full["P"][:, :kk], "beta0": full["beta0"],
         "k_eff": kk, "h_next": full["beta"][kk - 1], "checks": checks,
         "bound": checks[-1][1] if checks and checks[-1][0] == kk else 0.0}
    r["H"] = np.diag(r["alpha"]) + np.diag(r["beta"][:kk - 1], 1) + np.diag(r["beta"][:kk - 1], -1)
    return r


def arnoldi_adaptive(p, v, eps, k_max):
    """Alg. 2: Arnoldi (Alg. 1, MGS) with the error checked at the checkpoints k = 4, ceil(1.1 k),
    ... (fp64) by Lemma 1 for the unit start vector; x(t_j) = e^{H_k t_j} e_1 by the oracle's
    per-step Pade. As in lanczos_adaptive, one Arnoldi run to k_max is cut at the accepted
    checkpoint (its first k columns do not depend on later steps)."""
    full = arnoldi(p, v, k_max)
    mu = gershgorin_mu(p)
    Hf = full["Hfull"]
    checks = []
    kk = full["k_eff"]
    for k in checkpoints(kk):
        if k == kk and kk < k_max:  # exact breakdown before k_max
            break
        X = expm_e1_times(Hf[:k, :k], p["step"], p["n_steps"])
        b = lemma1_bound(Hf[k, k - 1], X, p["step"], mu)
        checks.append((k, b))
        if b < eps:
            kk = k
            break
    else:
        if kk == k_max and (not checks or checks[-1][1] >= eps):
            raise RuntimeError("adaptive Krylov: k_max reached before the error target")
    return {"H": Hf[:kk, :kk].copy(), "P": full["P"][:, :kk], "beta0": full["beta0"], "k_eff": kk,
            "h_next": Hf[kk, kk - 1], "checks": checks,
            "bound": checks[-1][1] if checks and checks[-1][0] == kk else 0.0}


def krylov_project_adaptive(p):
    """Basis-matrix sequence with adaptive k (p['eps'], p['k_max']): Lanczos (Alg. 4) through the
    eigendecomposition route, or Arnoldi (Alg. 2, p['method'] == 'arnoldi') through per-step Pade:
    coeff[j][r][d] = ||v_d|| (P_d e^{H_d t_j} e_1)_r."""
    dirs = directions(p)
    o, N = len(p["outs"]), p["n_steps"]
    coeff = np.zeros((N + 1, o, len(dirs)))
    per = []
    for d, v in enumerate(dirs):
        if p.get("method") == "arnoldi":
            r = arnoldi_adaptive(p, v, p["eps"], p["k_max"])
            X = expm_e1_times(r["H"], p["step"], N)
        else:
            r = lanczos_adaptive(p, v, p["eps"], p["k_max"])
            X = eig_e1_times(r["alpha"], r["beta"], p["step"], N)
        coeff[:, :, d] = r["beta0"] * (X @ r["P"].T)
        r["X"] = X
        per.append(r)
    return {"coeff": coeff, "per_dir": per, "times": np.arange(N + 1) * p["step"]}


def gershgorin_mu(p):
    """Upper bound on mu(A) = lambda_max((A+A^T)/2) by Gershgorin discs (reading for Lemma 1's
    nu(B) = -mu(A) with B = -A). Lifted matrix when b is present."""
    if p["op"] == "stencil":
        best = -math.inf
        ih = [float(p[a] + 1) ** 2 for a in ("mx", "my", "mz")]
        nb = [min(2, p[a] - 1) for a in ("mx", "my", "mz")]
        # the most interior cell maximises diag + sum |offdiag| (all off-diagonals are positive)
        best = p["alpha"] * sum((nb[a] - 2) * ih[a] for a in range(3))
        if p.get("b") is not None:  # lifted: row r gains |b_r|/2, the lifted row sum_r |b_r|/2
            bd = np.abs(_dense(p["b"], p, p["mx"] * p["my"] * p["mz"]) if isinstance(p["b"], dict) else p["b"])
            best = max(best + 0.5 * float(bd.max()), 0.5 * float(bd.sum()))
        return best
    n = p["n"]
    rp, ci, va = p["row_ptr"], p["col_idx"], p["val"]
    N = n + (1 if p.get("b") is not None else 0)
    diag = np.zeros(N)
    off = {}
    for r in range(n):
        for e in range(rp[r], rp[r + 1]):
            c = int(ci[e])
            if c == r:
                diag[r] += va[e]
            else:
                off[(r, c)] = off.get((r, c), 0.0) + 0.5 * va[e]
                off[(c, r)] = off.get((c, r), 0.0) + 0.5 * va[e]
        if p.get("b") is not None and p["b"][r] != 0.0:
            off[(r, n)] = off.get((r, n), 0.0) + 0.5 * p["b"][r]
            off[(n, r)] = off.get((n, r), 0.0) + 0.5 * p["b"][r]
    rad = np.zeros(N)
    for (r, c), s in off.items():
        rad[r] += abs(s)
    return float(np.max(diag + rad))


def krylov_project(p, method=None):
    """The whole basis-matrix sequence: coeff[j][r][d] ~= C_r e^{A t_j} v_d for j = 0..N.
    Returns dict(coeff, per_dir=[...], lemma1[d], times)."""
    method = method or p["method"]
    dirs = directions(p)
    o = len(p["outs"])
    N = p["n_steps"]
    nd = len(dirs)
    coeff = np.zeros((N + 1, o, nd))
    per_dir = []
    mu = gershgorin_mu(p)
    lemma = np.zeros(nd)
    for d, v in enumerate(dirs):
        r = lanczos(p, v, p["k"]) if method == "lanczos" else arnoldi(p, v, p["k"])
        X = expm_e1_times(r["H"], p["step"], N)  # (N+1) x k_eff
        coeff[:, :, d] = r["beta0"] * (X @ r["P"].T)  # c[j][r] = ||v|| (P x_j)_r
        r["X"] = X
        # Lemma 1 for the start vector v: ||v|| times the unit-vector bound
        # h_{k+1,k} e^{max(mu,0) T} int_0^T |e_k^T e^{Ht} e_1| dt (trapezoid) of lemma1_bound
        lemma[d] = r["beta0"] * lemma1_bound(r["h_next"], X, p["step"], mu) if N > 0 else 0.0
        per_dir.append(r)
    return {"coeff": coeff, "per_dir": per_dir, "lemma1": lemma, "mu": mu,
            "times": np.arange(N + 1) * p["step"]}


def transpose_problem(p):
    """The transpose-dynamics problem of §4.1: C e^{At} E = (E^T e^{A^T t} C^T)^T, so the basis
    matrix can be computed from o simulations of x' = A^T x started at the output rows C_r^T, each then
    projected with E^T (the "(or the transpose of the initial space matrix E^T)" of Alg. 4).
    With an affine term the lifted matrix A' = [[A, b], [0, 0]] is transposed explicitly:
    A'^T = [[A^T, 0], [b^T, 0]]; the output rows have 0 in the lifted coordinate and the projection rows
    are the forward directions (generators and v_f = [c; 1]). The stencil operator is symmetric."""
    fwd = directions(p)
    n_lift = len(fwd[0])
    q = dict(p)
    if p["op"] == "csr":
        n = p["n"]
        rp, ci, va = p["row_ptr"], p["col_idx"], p["val"]
        b = p.get("b")
        ent = []  # (row, col, value) of A'^T, in the order met while scanning A' row by row
        for r in range(n):
            for e in range(int(rp[r]), int(rp[r + 1])):
                ent.append((int(ci[e]), r, float(va[e])))
            if b is not None and b[r] != 0.0:
                ent.append((n, r, float(b[r])))
        ent.sort(key=lambda t: (t[0], t[1]))
        row_ptr = np.zeros(n_lift + 1, dtype=np.int64)
        for (r, c, v) in ent:
            row_ptr[r + 1] += 1
        row_ptr = np.cumsum(row_ptr)
        q.update(n=n_lift, row_ptr=row_ptr, col_idx=np.array([c for (_, c, _) in ent], dtype=np.int32),
                 val=np.array([v for (_, _, v) in ent]), b=None)
    # simulation directions: the output rows (as explicit vectors, 0 in the lifted coordinate)
    nb = n_lift - 1 if (p["op"] == "csr" and p.get("b") is not None) else n_lift
    gens = []
    for o in p["outs"]:
        v = _dense(o, p, nb)
        nz = np.nonzero(v)[0]
        gens.append({"kind": "sparse", "idx": nz.astype(np.int64), "val": v[nz]})
    outs = []
    for v in fwd:
        nz = np.nonzero(v)[0]
        outs.append({"kind": "sparse", "idx": nz.astype(np.int64), "val": v[nz]})
    q.update(gens=gens, outs=outs, center=None, z_lo=np.zeros(len(gens)), z_hi=np.zeros(len(gens)),
             thresholds=[], name=p.get("name", "") + "_T")
    return q


def krylov_project_transpose(p, method=None):
    """Basis-matrix sequence by the transpose dynamics: one Krylov simulation per output row,
    projected with E^T, transposed back: coeff[j][r][d] ~= C_r e^{A t_j} v_d. Same return layout as
    krylov_project; per_dir / lemma1 are per simulation (output row)."""
    q = transpose_problem(p)
    res = krylov_project(q, method=method or ("arnoldi" if q["op"] == "csr" else p["method"]))
    res["coeff"] = np.ascontiguousarray(np.transpose(res["coeff"], (0, 2, 1)))
    return res


def z_bounds(p):
    """Box bounds per direction; the fixed-term direction has z_f = 1."""
    lo = list(np.asarray(p["z_lo"], dtype=np.float64))
    hi = list(np.asarray(p["z_hi"], dtype=np.float64))
    if p.get("b") is not None or p.get("center") is not None:
        lo.append(1.0)
        hi.append(1.0)
    return np.array(lo), np.array(hi)


def check_lp(p, coeff, init_A=None, init_b=None, unsafe_A=None, unsafe_b=None):
    """The per-step LP of §2.1 in the initial / output spaces (Fig. 2(c); §3,
    P:467-496) for a general polytope: at step j the constraints are
        z_lo <= z <= z_hi,   I_z z <= iota            (initial set, "I_x x0 <= iota_x" on z)
        U_y (B_j z + c_f,j) <= upsilon                 (unsafe set, "U_x x <= upsilon_x" on y = C x)
    with B_j the generator columns of the basis matrix and c_f,j the fixed-term column (z_f = 1,
    P:1221-1225). The system is unsafe at the first j where the LP is feasible; the witness is
    the solver's assignment. Solver: scipy linprog / HiGHS (a library routine), zero objective.
    Returns dict(feasible [(N+1)] bool, found, step, z, y)."""
    from scipy.optimize import linprog
    ng = len(p["gens"])
    has_fixed = coeff.shape[2] > ng
    zlo = np.asarray(p["z_lo"], dtype=np.float64)[:ng]
    zhi = np.asarray(p["z_hi"], dtype=np.float64)[:ng]
    IA = np.zeros((0, ng)) if init_A is None else np.asarray(init_A, dtype=np.float64).reshape(-1, ng)
    Ib = np.zeros(0) if init_b is None else np.asarray(init_b, dtype=np.float64).reshape(-1)
    o = coeff.shape[1]
    UA = np.zeros((0, o)) if unsafe_A is None else np.asarray(unsafe_A, dtype=np.float64).reshape(-1, o)
    Ub = np.zeros(0) if unsafe_b is None else np.asarray(unsafe_b, dtype=np.float64).reshape(-1)
    Np1 = coeff.shape[0]
    feas = np.zeros(Np1, dtype=bool)
    res = {"feasible": feas, "found": False, "step": -1, "z": None, "y": None}
    for j in range(Np1):
        B = coeff[j, :, :ng]
        cf = coeff[j, :, ng] if has_fixed else np.zeros(o)
        A_ub = np.vstack([IA, UA @ B])
        b_ub = np.concatenate([Ib, Ub - UA @ cf])
        r = linprog(np.zeros(ng), A_ub=A_ub if A_ub.size else None, b_ub=b_ub if A_ub.size else None,
                    bounds=list(zip(zlo, zhi)), method="highs")
        feas[j] = r.status == 0
        if feas[j] and not res["found"]:
            res.update(found=True, step=j, z=np.array(r.x), y=B @ np.array(r.x) + cf)
    return res


def check_box(p, coeff, thresholds=None):
    """Per-step interval bounds of each output over the box initial set, the exact LP optimum for a
    box (Fig. 2(c)), the first violating step and a witness.
    thresholds: list of (row, sense, theta). Returns dict(lo, hi, found, step, row, y, z)."""
    thresholds = p["thresholds"] if thresholds is None else thresholds
    zlo, zhi = z_bounds(p)
    Np1, o, nd = coeff.shape
    lo = np.zeros((Np1, o))
    hi = np.zeros((Np1, o))
    for j in range(Np1):
        for r in range(o):
            a = 0.0
            b = 0.0
            for d in range(nd):
                c = coeff[j, r, d]
                a += min(c * zlo[d], c * zhi[d])
                b += max(c * zlo[d], c * zhi[d])
            lo[j, r] = a
            hi[j, r] = b
    res = {"lo": lo, "hi": hi, "found": False, "step": -1, "row": -1, "y": 0.0, "z": None}
    sense_of = {r: (s, th) for (r, s, th) in thresholds}
    for j in range(Np1):
        for r in range(o):
            if r not in sense_of:
                continue
            s, th = sense_of[r]
            bad = (hi[j, r] >= th) if s == GE else (lo[j, r] <= th) if s == LE else (lo[j, r] <= th <= hi[j, r])
            if not bad:
                continue
            c = coeff[j, r]
            if s == GE:
                z = np.where(c >= 0, zhi, zlo)
            elif s == LE:
                z = np.where(c >= 0, zlo, zhi)
            else:
                lam = 0.0 if hi[j, r] == lo[j, r] else (th - lo[j, r]) / (hi[j, r] - lo[j, r])
                z = np.where(c >= 0, zlo + lam * (zhi - zlo), zhi - lam * (zhi - zlo))
            y = float(np.sum(c * z))
            res.update(found=True, step=j, row=r, y=y, z=z, time=j * p["step"])
            return res
    return res
