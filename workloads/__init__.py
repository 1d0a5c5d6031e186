"""Seeded synthetic workloads shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no operator application, no Krylov iteration, no
exponential, no interval sums). It only describes problems: grid sizes, generator / output vectors
given compactly, time grids, and — for the CSR workload — seeded random matrix entries. Both the
oracle (oracle/) and the CUDA path (paper_1804_01583_b200/) consume the same descriptions, so the two
sides see identical inputs without sharing any code of the method.

Problem statement (§2): x' = Ax + b, initial set I, unsafe set U, step δ, bound T.
Initial space E (n x i, §3.2) is given by generator vectors; output space C (o x n,
§3.1) by output rows.

A vector is a dict:
  {"kind": "box", "lo": (x,y,z), "hi": (x,y,z), "value": v}   value on the index box [lo, hi)
  {"kind": "all", "value": v}                                   value everywhere
  {"kind": "sparse", "idx": int64[], "val": float64[]}          explicit entries (linear index)
For CSR problems a box uses only axis 0 (linear index range [lo[0], hi[0])).
Linear index of a stencil cell (x, y, z) is x + mx*(y + my*z) (x fastest).

Configs follow BASELINE.json "configs" and SURVEY.md §8(d); the readings of ambiguous points are
SURVEY.md §8(c) A1-A17 and are listed in DESIGN.md.
"""
from __future__ import annotations

import math
import numpy as np

GE, LE, EQ = 0, 1, 2  # unsafe if y >= θ, y <= θ, y == θ


def box(lo, hi, value=1.0):
    return {"kind": "box", "lo": tuple(int(v) for v in lo), "hi": tuple(int(v) for v in hi),
            "value": float(value)}


def point(x, y=0, z=0, value=1.0):
    return box((x, y, z), (x + 1, y + 1, z + 1), value)


def allv(value=1.0):
    return {"kind": "all", "value": float(value)}


def rand(seed, value=1.0):
    """A seeded dense field value * u_c, u_c in [0, 1) from a counter-based generator (include/krylov_reach.h
    KR_VEC_RAND; each side implements it). Synthetic dense start vectors: the dense-data bench workload."""
    return {"kind": "rand", "seed": int(seed), "value": float(value)}


def sparse(idx, val):
    return {"kind": "sparse", "idx": np.ascontiguousarray(idx, dtype=np.int64),
            "val": np.ascontiguousarray(val, dtype=np.float64)}


def center_index(m):
    """Center cell for a side-m grid: floor((m-1)/2) per axis."""
    return (m - 1) // 2


def heat(m, block, k, n_steps=1000, step=0.02, alpha=0.01, method="lanczos", extras=True,
         thresholds=None, my=None, mz=None):
    """3D heat diffusion, Dirichlet 7-point stencil, A = alpha * L_h, h = 1/(m+1) per axis
    (BASELINE.json configs 3-5). Initial set: corner block [0,block)^3 in [0.9, 1.1]
    as ONE generator direction with z in [0.9, 1.1]. Outputs: center cell, plus the
    supplementary non-vacuous rows of SURVEY A11: total heat, cell (b,b,b), corner (0,0,0)."""
    mx = m
    my = m if my is None else my
    mz = m if mz is None else mz
    c = (center_index(mx), center_index(my), center_index(mz))
    outs = [point(*c)]
    if extras:
        b = min(block, mx - 1, my - 1, mz - 1)
        outs += [allv(1.0), point(b, b, b), point(0, 0, 0)]
    return {
        "name": f"heat{mx}x{my}x{mz}_b{block}",
        "op": "stencil", "mx": mx, "my": my, "mz": mz, "alpha": float(alpha),
        "gens": [box((0, 0, 0), (block, block, block), 1.0)],
        "z_lo": np.array([0.9]), "z_hi": np.array([1.1]),
        "center": None, "b": None,
        "outs": outs,
        "step": float(step), "n_steps": int(n_steps), "k": int(k), "method": method,
        "thresholds": list(thresholds or []),
    }


def config1():
    """BASELINE.json configs[0]: 5x5x5 heat (n=125), 8 generator directions e_(x,y,z), x,y,z in {0,1},
    z in [0.9,1.1], O = center cell (2,2,2), unsafe if y >= 0.05, step 0.02, 200 steps, Arnoldi k=30."""
    m = 5
    gens = [point(x, y, z) for z in (0, 1) for y in (0, 1) for x in (0, 1)]
    c = center_index(m)
    return {
        "name": "C1_heat5", "op": "stencil", "mx": m, "my": m, "mz": m, "alpha": 0.01,
        "gens": gens, "z_lo": np.full(8, 0.9), "z_hi": np.full(8, 1.1),
        "center": None, "b": None, "outs": [point(c, c, c)],
        "step": 0.02, "n_steps": 200, "k": 30, "method": "arnoldi",
        "thresholds": [(0, GE, 0.05)],
    }


def csr_banded_random(n=20000, seed=0, band=50, n_band=9, n_rand=2):
    """BASELINE.json configs[1] matrix under SURVEY §8(c) A16: per row i, the diagonal; n_band distinct
    off-diagonal columns uniform without replacement from [i-band, i+band] \\ {i} ∩ [0,n); n_rand
    columns uniform over [0,n) (self dropped, duplicates merged); off-diagonal values U[-1,1];
    a_ii = -(sum|a_ij| + U[0.1,1]). Then b ~ U[-0.1,0.1]. RNG numpy default_rng(seed), this draw order.
    Returns (row_ptr int64[n+1], col_idx int32[nnz], val float64[nnz], b float64[n], rng)."""
    rng = np.random.default_rng(seed)
    rows_c, rows_v = [], []
    for i in range(n):
        lo, hi = max(0, i - band), min(n - 1, i + band)
        cand = np.array([j for j in range(lo, hi + 1) if j != i], dtype=np.int64)
        bc = rng.choice(cand, size=min(n_band, cand.size), replace=False)
        rc = rng.integers(0, n, size=n_rand)
        cols = np.unique(np.concatenate([bc, rc[rc != i]]))
        vals = rng.uniform(-1.0, 1.0, size=cols.size)
        diag = -(np.abs(vals).sum() + rng.uniform(0.1, 1.0))
        allc = np.concatenate([cols, [i]])
        allv_ = np.concatenate([vals, [diag]])
        order = np.argsort(allc, kind="stable")
        rows_c.append(allc[order])
        rows_v.append(allv_[order])
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    row_ptr[1:] = np.cumsum([c.size for c in rows_c])
    col_idx = np.concatenate(rows_c).astype(np.int32)
    val = np.concatenate(rows_v).astype(np.float64)
    b = rng.uniform(-0.1, 0.1, size=n)
    return row_ptr, col_idx, val, b, rng


def config2(n=20000, n_gen=20, n_steps=2000, k=40, seed=0):
    """BASELINE.json configs[1]: nonsymmetric sparse affine system, CSR ~12 nnz/row, b ~ U[-0.1,0.1],
    initial box over the first 20 states in [-1,1], O = 3 Gaussian rows, step 0.005, 2000 steps,
    Arnoldi k=40 batched over the directions. Lifting adds the fixed direction
    v_f = e_{n'} (center 0, b != 0) — SURVEY A5."""
    row_ptr, col_idx, val, b, rng = csr_banded_random(n, seed)
    O = rng.standard_normal((3, n))
    outs = [sparse(np.arange(n, dtype=np.int64), O[r]) for r in range(3)]
    return {
        "name": f"C2_csr{n}", "op": "csr", "n": n,
        "row_ptr": row_ptr, "col_idx": col_idx, "val": val, "b": b,
        "gens": [sparse([d], [1.0]) for d in range(n_gen)],
        "z_lo": np.full(n_gen, -1.0), "z_hi": np.full(n_gen, 1.0),
        "center": None, "outs": outs,
        "step": 0.005, "n_steps": int(n_steps), "k": int(k), "method": "arnoldi",
        "thresholds": [],
    }


def config3(**kw):
    """BASELINE.json configs[2]: 100^3 heat, 10^3 corner block, Lanczos k=40, 1000 steps."""
    return dict(heat(100, 10, 40, **kw), name="C3_heat100")


def config4(**kw):
    """BASELINE.json configs[3]: 400^3 heat, 40^3 corner block, Lanczos k=40, 1000 steps."""
    return dict(heat(400, 40, 40, **kw), name="C4_heat400")


def config5(**kw):
    """BASELINE.json configs[4]: 1000^3 heat (10^9 states), 100^3 corner block, Lanczos k=30,
    1000 steps of 0.02; unsafe if center y >= 0.012."""
    p = heat(1000, 100, 30, **kw)
    p["thresholds"] = [(0, GE, 0.012)]
    return dict(p, name="C5_heat1000")


def config5_dense(**kw):
    """C5 with a dense start: the corner-block generator replaced by a seeded dense field over the whole 10^9
    grid (rand(seed 5), z in [0.9, 1.1]). Every Krylov vector is dense from step 1, as in the paper's own
    10^9-state run after its first ~1000 steps, so the step kernel is measured on data with
    realistic bit toggling (the C5 vectors are >= 99.8% zeros at k = 30). The center row is non-vacuous here."""
    p = heat(1000, 100, 30, **kw)
    p["gens"] = [rand(5)]
    p["thresholds"] = [(0, GE, 0.012)]
    return dict(p, name="C5D_heat1000_dense")


def oscillator():
    """Timed harmonic oscillator, PAPER.md:175-214 (§2.2): x'=y, y'=-x, t'=1; x0=-5, y0 in [0,1],
    t0=0; unsafe x = 4; δ=π/4, T=π. As an affine system: A 3x3, b=(0,0,1), center (-5,0,0),
    one generator e_y with z in [0,1], output row x, EQ threshold 4."""
    row_ptr = np.array([0, 1, 2, 2], dtype=np.int64)
    col_idx = np.array([1, 0], dtype=np.int32)
    val = np.array([1.0, -1.0])
    return {
        "name": "oscillator", "op": "csr", "n": 3,
        "row_ptr": row_ptr, "col_idx": col_idx, "val": val, "b": np.array([0.0, 0.0, 1.0]),
        "gens": [sparse([1], [1.0])], "z_lo": np.array([0.0]), "z_hi": np.array([1.0]),
        "center": sparse([0], [-5.0]), "outs": [sparse([0], [1.0])],
        "step": math.pi / 4, "n_steps": 4, "k": 4, "method": "arnoldi",
        "thresholds": [(0, EQ, 4.0)],
    }


def random_csr(n, nnz_per_row, seed, symmetric=False, scale=1.0):
    """Small seeded random CSR matrices for property tests (diagonally dominant, negative diagonal)."""
    rng = np.random.default_rng(seed)
    dense = np.zeros((n, n))
    for i in range(n):
        cols = rng.choice(n, size=min(nnz_per_row, n), replace=False)
        dense[i, cols] = rng.uniform(-1, 1, size=cols.size)
    if symmetric:
        dense = 0.5 * (dense + dense.T)
    np.fill_diagonal(dense, 0.0)
    dense[np.diag_indices(n)] = -(np.abs(dense).sum(axis=1) + rng.uniform(0.1, 1.0, size=n))
    dense *= scale
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    cols_l, vals_l = [], []
    for i in range(n):
        nz = np.nonzero(dense[i])[0]
        cols_l.append(nz)
        vals_l.append(dense[i, nz])
        row_ptr[i + 1] = row_ptr[i] + nz.size
    return row_ptr, np.concatenate(cols_l).astype(np.int32), np.concatenate(vals_l), dense


BC_DIRICHLET, BC_NEUMANN, BC_ROBIN = 0, 1, 2


def heat_paper(m, eps=1e-6, k_max=8000, n_steps=1000, step=0.02):
    """The paper's own 3D heat benchmark (§5.3): unit cube, all faces
    insulated except x = 1, which exchanges heat with constant 0.5; heated region
    x in [0,0.4], y in [0,0.2], z in [0,0.1] at [0.9,1.1], rest 0; u_t = alpha^2 Lap u with
    'alpha = 0.01'. Reading (DESIGN R18): grid points x_i = (i+1) h, h = 1/(m+1);
    insulated faces drop the missing neighbour; the x = 1 face adds -0.5/h to the diagonal; the whole
    operator is scaled by 0.01 (this reproduces ||A 50|| = 32771611 of P:674 to 3e-8). Heated cells:
    (i+1) h <= bound. Output: center point. T = 20, delta = 0.02. Adaptive k with
    Lemma 1 to eps = 1e-6."""
    h = 1.0 / (m + 1)
    n_x = int(math.floor(0.4 * (m + 1) + 1e-9))
    n_y = int(math.floor(0.2 * (m + 1) + 1e-9))
    n_z = int(math.floor(0.1 * (m + 1) + 1e-9))
    c = center_index(m)
    gamma = 0.01 * 0.5 / h
    return {
        "name": f"heat_paper{m}", "op": "stencil", "mx": m, "my": m, "mz": m, "alpha": 0.01,
        "bc": [BC_NEUMANN, BC_ROBIN, BC_NEUMANN, BC_NEUMANN, BC_NEUMANN, BC_NEUMANN],
        "gamma": [0.0, gamma, 0.0, 0.0, 0.0, 0.0],
        "gens": [box((0, 0, 0), (n_x, n_y, n_z), 1.0)],
        "z_lo": np.array([0.9]), "z_hi": np.array([1.1]),
        "center": None, "b": None, "outs": [point(c, c, c), allv(1.0)],
        "step": float(step), "n_steps": int(n_steps), "k": int(k_max), "method": "lanczos",
        "eps": float(eps), "k_max": int(k_max), "thresholds": [],
    }


def heat_heater(m, k=64, n_steps=1000, step=0.5):
    """The paper's nonsymmetric 3D heat variant: the heat model of
    heat_paper (insulated faces, Robin 0.5 at x = 1, 'alpha = 0.01' as A = 0.01 L) with the initially heated
    region replaced by a permanent heater on the bottom face z = 0 over x in [0, 0.4], y in [0, 0.2]
    (P:1136-1138); T = 500, delta = 0.5. Reading (DESIGN R19): the heater is a unit heat flux
    through the z = 0 face into the first cell layer, i.e. the affine term b = 0.01 * 1/h on those cells
    (the same scaling as the Robin term 0.01 * 0.5/h); the initial temperature is 0, so the only Krylov
    simulation is the lifted fixed direction e_{n+1} and the reachable output is one trajectory
    (the paper plots "the temperature reachable at the center"). Lifting makes the system
    nonsymmetric: Arnoldi."""
    h = 1.0 / (m + 1)
    n_x = int(math.floor(0.4 * (m + 1) + 1e-9))
    n_y = int(math.floor(0.2 * (m + 1) + 1e-9))
    c = center_index(m)
    return {
        "name": f"heat_heater{m}", "op": "stencil", "mx": m, "my": m, "mz": m, "alpha": 0.01,
        "bc": [BC_NEUMANN, BC_ROBIN, BC_NEUMANN, BC_NEUMANN, BC_NEUMANN, BC_NEUMANN],
        "gamma": [0.0, 0.01 * 0.5 / h, 0.0, 0.0, 0.0, 0.0],
        "b": box((0, 0, 0), (n_x, n_y, 1), 0.01 / h),
        "gens": [], "z_lo": np.zeros(0), "z_hi": np.zeros(0), "center": None,
        "outs": [point(c, c, c), allv(1.0)],
        "step": float(step), "n_steps": int(n_steps), "k": int(k), "method": "arnoldi", "thresholds": [],
    }


def csr_stable_nonsym(n=400, nnz_per_row=6, seed=7, n_gen=3, eps=1e-6, k_max=200, n_steps=200, step=0.02,
                      scale=1.0, shift=1.0):
    """A nonsymmetric sparse system whose symmetric part is negative definite by Gershgorin (diagonal =
    -(row + column off-diagonal mass)/2 - 1), so Lemma 1's e^{-min(nu, 0) tau} factor is 1 and the adaptive
    Arnoldi of Alg. 2 can meet eps: random off-diagonals scale * U[-1,1], diagonal
    -(row + column off-diagonal mass)/2 - shift, no affine term, unit generators in [-1, 1], two Gaussian
    output rows."""
    rng = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    for i in range(n):
        js = rng.choice(np.delete(np.arange(n), i), size=nnz_per_row, replace=False)
        for j in js:
            rows.append(i)
            cols.append(int(j))
            vals.append(float(scale * rng.uniform(-1.0, 1.0)))
    rows, cols, vals = np.array(rows), np.array(cols), np.array(vals)
    rmass = np.bincount(rows, weights=np.abs(vals), minlength=n)
    cmass = np.bincount(cols, weights=np.abs(vals), minlength=n)
    diag = -(rmass + cmass) / 2.0 - shift
    rows = np.concatenate([rows, np.arange(n)])
    cols = np.concatenate([cols, np.arange(n)])
    vals = np.concatenate([vals, diag])
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    outs = [sparse(np.arange(n), rng.standard_normal(n)) for _ in range(2)]
    return {"name": f"csr_stable{n}", "op": "csr", "n": n, "row_ptr": row_ptr, "col_idx": cols.astype(np.int32),
            "val": vals, "b": None, "gens": [sparse([d * 7], [1.0]) for d in range(n_gen)],
            "z_lo": -np.ones(n_gen), "z_hi": np.ones(n_gen), "center": None, "outs": outs,
            "step": float(step), "n_steps": int(n_steps), "k": int(k_max), "method": "arnoldi",
            "eps": float(eps), "k_max": int(k_max), "thresholds": []}


def paper1000_dense(k=30):
    """The paper's 10^9-state heat model (insulated faces, Robin at x = 1; heat_paper(1000)) with a fixed k and the
    dense start rand(5): the general-boundary step kernel on dense data, as in steps 1000+ of the paper's own run
    (timing workload for A/B runs, not a bench line)."""
    p = heat_paper(1000, k_max=k)
    p["eps"] = 0.0
    p["gens"] = [rand(5)]
    return dict(p, name="P1000D_heat_paper1000_dense")


CONFIGS = {"C1": config1, "C2": config2, "C3": config3, "C4": config4, "C5": config5, "C5D": config5_dense,
           "P1000D": paper1000_dense,
           "P100": lambda: heat_paper(100), "P1000": lambda: heat_paper(1000),
           "H10": lambda: heat_heater(10), "H100": lambda: heat_heater(100, k=800),
           "C2T": lambda: dict(config2(), sim="transpose")}


def n_state(p):
    return p["mx"] * p["my"] * p["mz"] if p["op"] == "stencil" else p["n"]


def n_dirs(p):
    return len(p["gens"]) + (1 if (p.get("center") is not None or p.get("b") is not None) else 0)


def dense_vec(v, p):
    """Materialize a compact vector as a dense float64 array of the (unlifted) state length.
    Pure indexing (no arithmetic of the method); used by tests on small problems."""
    n = n_state(p)
    out = np.zeros(n)
    if v["kind"] == "all":
        out[:] = v["value"]
    elif v["kind"] == "sparse":
        np.add.at(out, v["idx"], v["val"])
    else:
        if p["op"] == "stencil":
            g = out.reshape(p["mz"], p["my"], p["mx"])
            (x0, y0, z0), (x1, y1, z1) = v["lo"], v["hi"]
            g[z0:z1, y0:y1, x0:x1] = v["value"]
        else:
            out[v["lo"][0]:v["hi"][0]] = v["value"]
    return out
