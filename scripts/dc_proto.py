"""Prototype (numpy, loops) of the carried-rows divide-and-conquer eigen-solve of a symmetric tridiagonal that
kr_tridc.cu implements: leaves of size 1, Cuppen rank-one merges bottom-up, LAPACK-style deflation, secular roots
by the two-pole rational interpolation, Gu-Eisenstat z, and only the rows R Q carried (R = e_1^T, e_k^T, P).
Not product code, not the oracle: a design check against numpy eigh. Usage: python scripts/dc_proto.py"""
import numpy as np

EPS = np.finfo(float).eps / 2


def secular_root(d, z, rho, j):
    """Root j of 1 + rho sum z_i^2/(d_i - lam) (d strictly increasing), returned as (origin index, tau)."""
    K = len(d)
    if K == 1:
        return 0, rho * z[0] ** 2
    if j < K - 1:
        gap = d[j + 1] - d[j]
        mid = 0.5 * gap
        fm = 1.0 + rho * np.sum(z ** 2 / ((d - d[j]) - mid))
        if fm > 0:
            org, lo, hi = j, 0.0, mid
        else:
            org, lo, hi = j + 1, -mid, 0.0
        p1, p2 = j, j + 1
    else:
        org, lo, hi = K - 1, 0.0, rho
        p1, p2 = K - 2, K - 1
    dl = d - d[org]
    tau = 0.5 * (lo + hi)
    for it in range(80):
        den = dl - tau
        t = rho * z ** 2 / den
        f = 1.0 + np.sum(t)
        erretm = 1.0 + np.sum(np.abs(t))
        if abs(f) <= 8 * EPS * erretm:
            break
        if f > 0:
            hi = tau
        else:
            lo = tau
        g1 = np.arange(K) <= p1
        s1, s2 = np.sum(t[g1]), np.sum(t[~g1])
        ds1 = np.sum((t / den)[g1])
        ds2 = np.sum((t / den)[~g1])
        D1, D2 = dl[p1] - tau, dl[p2] - tau
        b1 = ds1 * D1 * D1
        b2 = ds2 * D2 * D2
        a1 = s1 - b1 / D1
        a2 = s2 - b2 / D2
        c = 1.0 + a1 + a2
        A = c
        B = c * (D1 + D2) + b1 + b2
        C = D1 * D2 * f
        if A == 0.0:
            eta = C / B
        else:
            disc = max(B * B - 4 * A * C, 0.0)
            eta = 2 * C / (B + np.copysign(np.sqrt(disc), B))
        tn = tau + eta
        if not (lo < tn < hi):
            tn = 0.5 * (lo + hi)
        if tn == tau:
            break
        tau = tn
    return org, tau


def merge(lam1, W1, lam2, W2, beta, rows_first_last=(0, 1)):
    """Children (eigenvalues, carried rows [first, last, P...] x n_c) -> parent."""
    n1, n2 = len(lam1), len(lam2)
    n = n1 + n2
    rho = abs(beta)
    s = 1.0 if beta >= 0 else -1.0
    D = np.concatenate([lam1, lam2])
    z = np.concatenate([W1[1], s * W2[0]]) / np.sqrt(2.0)
    rho = 2 * rho
    R = W1.shape[0]
    Wp = np.zeros((R, n))
    Wp[0, :n1] = W1[0]
    Wp[1, n1:] = W2[1]
    Wp[2:, :n1] = W1[2:]
    Wp[2:, n1:] = W2[2:]
    perm = np.argsort(D, kind="stable")
    D = D[perm].copy()
    z = z[perm].copy()
    Wp = Wp[:, perm].copy()
    tol = 8 * EPS * max(np.max(np.abs(D)), np.max(np.abs(z)))
    keep, defl = [], []
    pj = -1
    for nj in range(n):
        if rho * abs(z[nj]) <= tol:
            defl.append(nj)
            continue
        if pj < 0:
            pj = nj
            continue
        ss, cc = z[pj], z[nj]
        tau = np.hypot(cc, ss)
        t = D[nj] - D[pj]
        cc /= tau
        ss = -ss / tau
        if abs(t * cc * ss) <= tol:
            z[nj] = tau
            z[pj] = 0.0
            a, b = Wp[:, pj].copy(), Wp[:, nj].copy()
            Wp[:, pj] = cc * a + ss * b  # deflated column
            Wp[:, nj] = -ss * a + cc * b
            dp = D[pj] * cc * cc + D[nj] * ss * ss
            D[nj] = D[pj] * ss * ss + D[nj] * cc * cc
            D[pj] = dp
            defl.append(pj)
            pj = nj
        else:
            keep.append(pj)
            pj = nj
    if pj >= 0:
        keep.append(pj)
    keep = np.array(keep, dtype=int)
    K = len(keep)
    d = D[keep]
    zz = z[keep]
    roots = [secular_root(d, zz, rho, j) for j in range(K)]
    # Gu-Eisenstat z
    zh = np.zeros(K)
    for i in range(K):
        o, t = roots[i]
        prod = ((d[o] - d[i]) + t) / rho
        for j in range(K):
            if j == i:
                continue
            oj, tj = roots[j]
            prod *= ((d[oj] - d[i]) + tj) / (d[j] - d[i])
        zh[i] = np.copysign(np.sqrt(prod), zz[i])
    lam_new = np.zeros(n)
    W = np.zeros((R, n))
    Wk = Wp[:, keep]
    for j in range(K):
        o, t = roots[j]
        u = zh / ((d - d[o]) - t)
        u /= np.linalg.norm(u)
        lam_new[j] = d[o] + t
        W[:, j] = Wk @ u
    for q, c in enumerate(defl):
        lam_new[K + q] = D[c]
        W[:, K + q] = Wp[:, c]
    return lam_new, W, K


def dc(alpha, beta, P):
    """Eigenvalues and rows [e_1^T Q, e_k^T Q, P Q] of tridiag(beta; alpha; beta) by bottom-up D&C."""
    k = len(alpha)
    o = P.shape[0]
    a = alpha.astype(float).copy()
    for i in range(k - 1):
        a[i] -= abs(beta[i])
        a[i + 1] -= abs(beta[i])
    nodes = [(a[i:i + 1].copy(), np.vstack([np.ones(1), np.ones(1), P[:, i:i + 1]])) for i in range(k)]
    lo = list(range(k))
    s = 1
    stats = []
    while len(nodes) > 1:
        nn, nl = [], []
        for q in range(0, len(nodes), 2):
            if q + 1 == len(nodes):
                nn.append(nodes[q])
                nl.append(lo[q])
                continue
            l1, W1 = nodes[q]
            l2, W2 = nodes[q + 1]
            m = lo[q + 1]
            lam, W, K = merge(l1, W1, l2, W2, beta[m - 1])
            stats.append((len(lam), K))
            nn.append((lam, W))
            nl.append(lo[q])
        nodes, lo = nn, nl
        s *= 2
    return nodes[0][0], nodes[0][1], stats


def e1_times_dc(alpha, beta, P, step, N):
    lam, W, _ = dc(alpha, beta, P)
    t = np.arange(N + 1) * step
    E = np.exp(np.outer(t, lam)) * W[0]
    last = E @ W[1]
    c = E @ W[2:].T
    last[0] = 1.0 if len(alpha) == 1 else 0.0
    c[0] = P[:, 0]
    return last, c


if __name__ == "__main__":
    rng = np.random.default_rng(1)
    import sys
    sys.path.insert(0, ".")
    for k in (1, 2, 3, 7, 64, 100, 301):
        al = rng.standard_normal(k)
        be = rng.standard_normal(k - 1) if k > 1 else np.zeros(0)
        P = rng.standard_normal((2, k))
        H = np.diag(al) + np.diag(be, 1) + np.diag(be, -1)
        lam, Q = np.linalg.eigh(H)
        l2, W, st = dc(al, be, P)
        i = np.argsort(l2)
        print(k, np.max(np.abs(l2[i] - lam)), np.max(np.abs(np.abs(W[0][i]) - np.abs(Q[0]))),
              np.max(np.abs(W[0][i] * W[1][i] - Q[0] * Q[-1])), np.max(np.abs(W[2:, i] * W[0][i] - (P @ Q) * Q[0])))
    # Lanczos tridiagonal of a heat operator (ghost eigenvalues)
    import workloads as Wk
    import oracle
    p = Wk.heat_paper(20, k_max=400)
    r = oracle.lanczos(p, oracle.directions(p)[0], 300)
    for k in (70, 150, 300):
        al, be = r["alpha"][:k], r["beta"][:k]
        X = oracle.eig_e1_times(al, be, p["step"], p["n_steps"])
        last, c = e1_times_dc(al, be[:k - 1], r["P"][:, :k], p["step"], p["n_steps"])
        ref = X @ r["P"][:, :k].T
        lam, W, st = dc(al, be[:k - 1], r["P"][:, :k])
        print("heat k", k, "defl", sum(n - K for n, K in st), "last err", np.max(np.abs(last - X[:, -1])) / np.max(np.abs(X[:, -1])),
              "c err", np.max(np.abs(c - ref)) / np.max(np.abs(ref)))
