"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.
Tolerance: tests/parity.py (north_star's 1e-9 relative, floored per series). Verdicts and violation
steps must be identical."""
import math

import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import assert_coeff, bounds_close

pytestmark = pytest.mark.gpu


def gpu_run(prob, thresholds=None, **kw):
    from paper_1804_01583_b200 import KrylovReach
    with KrylovReach(prob, **kw) as h:
        coeff, stats = h.project()
        cb = h.check_box(thresholds)
        launches = h.launch_count()
    return coeff, stats, cb, launches


def compare_full(prob, thresholds=None, method=None, res=None, **kw):
    res = res if res is not None else oracle.krylov_project(prob, method=method)
    coeff, stats, cb, launches = gpu_run(prob, thresholds, method=method, **kw)
    assert launches > 0
    worst = assert_coeff(coeff, res["coeff"], prob["name"])
    ocb = oracle.check_box(prob, res["coeff"], thresholds)
    zlo, zhi = oracle.z_bounds(prob)
    ok, wb = bounds_close(cb["lo"], ocb["lo"], res["coeff"], zlo, zhi)
    assert ok, f"lo bounds worst {wb}"
    ok, wb = bounds_close(cb["hi"], ocb["hi"], res["coeff"], zlo, zhi)
    assert ok, f"hi bounds worst {wb}"
    assert cb["found"] == ocb["found"]
    if cb["found"]:
        assert cb["step"] == ocb["step"] and cb["row"] == ocb["row"]
        c = res["coeff"][cb["step"], cb["row"]]
        sig = np.abs(c) > 1e-9 * np.abs(c).sum()
        assert np.allclose(cb["z"][sig], ocb["z"][sig], rtol=1e-9, atol=1e-12)
        assert abs(cb["y"] - ocb["y"]) <= 1e-9 * max(1.0, abs(ocb["y"]))
    for d, (s, r) in enumerate(zip(stats, res["per_dir"])):
        assert s["k_eff"] == r["k_eff"], (d, s["k_eff"], r["k_eff"])
        assert abs(s["beta0"] - r["beta0"]) <= 1e-12 * r["beta0"]
    assert_lemma1(stats, res["lemma1"], prob["name"], T=prob["n_steps"] * prob["step"], mu=res["mu"],
                  hmax=hmax_of(res["per_dir"]))
    return coeff, res, cb, ocb, stats, worst


def assert_lemma1(stats, orc, what="", T=None, mu=0.0, hmax=None, floor=1e-6):
    """Lemma 1 diagnostic per direction: the same value to 1e-9 relative, floored like the parity metric
    at floor * beta0 T e^{max(mu,0) T} max|H| (the bound's rounding envelope: h_{k+1,k} carries absolute rounding of
    order u max|H| and the integrand |e_k^T e^{Ht} e_1| of order u on both sides, so near-breakdown bounds — the
    oscillator's h_54 = 2e-17 — and bounds far below the envelope — C1 at k = 30: 1e-36 — are compared to that
    floor); both +inf where e^{mu T} overflows, both 0 on an exact breakdown. hmax: per direction."""
    for d, (s, o) in enumerate(zip(stats, orc)):
        g = s["lemma1"]
        assert not math.isnan(g), (what, d)
        if math.isinf(o) or o == 0.0:
            assert g == o, (what, d, g, o)
        else:
            hm = max(s["h_next"], hmax[d] if hmax is not None else 0.0)
            env = s["beta0"] * (T or 0.0) * math.exp(min(max(mu, 0.0) * (T or 0.0), 700.0)) * hm
            assert abs(g - o) <= 1e-9 * max(abs(o), floor * env), (what, d, g, o, env)


def hmax_of(per_dir):
    return [float(np.max(np.abs(r["H"]))) if np.size(r["H"]) else 0.0 for r in per_dir]


# ---------------------------------------------------------------------------------------------
# BASELINE configs
# ---------------------------------------------------------------------------------------------
def test_config1_arnoldi_parity_and_verdicts():
    p = W.config1()
    coeff, res, cb, ocb, stats, _ = compare_full(p)
    assert not cb["found"]  # theta = 0.05: SAFE (BASELINE configs[0])
    _, _, cb2, _ = gpu_run(p, [(0, W.GE, 0.02)])
    assert cb2["found"] and cb2["step"] == 74


def test_oscillator_paper_example():
    p = W.oscillator()
    coeff, res, cb, ocb, stats, _ = compare_full(p)
    assert cb["found"] and cb["step"] == 3
    assert abs(cb["z"][0] - (4 * math.sqrt(2) - 5)) <= 1e-12  # y0 = 0.66
    assert np.allclose(coeff[3, 0], [0.707, 3.54], atol=5e-3)  # Fig. 2(c)
    assert stats[0]["k_eff"] == 2 and stats[0]["h_next"] == 0.0  # exact breakdown


def test_config2_full_size_parity():
    """BASELINE configs[1] at full size (n = 20000 lifted to 20001, 21 directions, k = 40, 2001 steps): every
    coefficient, both bounds, the Lemma-1 diagnostic and the verdict of an oracle-chosen threshold (SURVEY A11 iv:
    first violation mid-trajectory, >= 1e-6 relative margin from every step's bound) against the full oracle run."""
    p = W.config2()
    res = oracle.krylov_project(p)
    prop = choose_property(oracle.check_box(p, res["coeff"], []))
    coeff, res2, cb, ocb, stats, _ = compare_full(p, [prop], res=res)
    assert cb["found"]  # C2 contracts from the initial box: every bound starts at its extreme, first violation at 0


def choose_threshold(series, sense, margin=1e-6):
    """A threshold whose first violation falls as late as possible after step 0 and at least margin (relative to the
    series scale) away from the bound of every step, so no step is within the parity tolerance of it (SURVEY §8(c)
    C-parity, A11 iv): the midpoint of the bounds of steps j-1 and j. None if the series allows none."""
    s = np.asarray(series, dtype=np.float64)
    scale = float(np.max(np.abs(s)))
    for j in range(len(s) - 1, 0, -1):
        th = 0.5 * (s[j - 1] + s[j])
        bad = s >= th if sense == W.GE else s <= th
        if bad.any() and int(np.argmax(bad)) == j and np.min(np.abs(s - th)) >= margin * scale:
            return float(th)
    return None


def choose_property(bounds):
    """(row, sense, threshold) over all output rows: GE on the upper bounds or LE on the lower bounds, the latest
    first violation."""
    best = None
    for r in range(bounds["hi"].shape[1]):
        for sense, ser in ((W.GE, bounds["hi"][:, r]), (W.LE, bounds["lo"][:, r])):
            th = choose_threshold(ser, sense)
            if th is None:
                continue
            bad = ser >= th if sense == W.GE else ser <= th
            j = int(np.argmax(bad))
            if best is None or j > best[0]:
                best = (j, (r, sense, th))
    if best is None:  # every bound starts at its extreme (a contracting system): a violation at step 0 only
        for r in range(bounds["hi"].shape[1]):
            hi = bounds["hi"][:, r]
            scale = float(np.max(np.abs(hi)))
            if len(hi) > 1 and hi[0] - np.max(hi[1:]) >= 2e-6 * scale:
                return (r, W.GE, float(0.5 * (hi[0] + np.max(hi[1:]))))
    assert best is not None, "no threshold with margin"
    return best[1]


@pytest.mark.parametrize("cgs", ["0", "1"])
def test_config2_small_full_parity(cgs, monkeypatch):
    """Config-2 recipe at n=2000, 5 generators, 300 steps: every output, bound and verdict — with the one-CTA
    MGS of Alg. 1 and with the multi-CTA CGS2 orthogonalisation."""
    monkeypatch.setenv("KR_FORCE_CGS", cgs)
    p = W.config2(n=2000, n_gen=5, n_steps=300, k=30)
    res = oracle.krylov_project(p)
    th = float(np.median(res["coeff"][:, 0, :].sum(axis=1)))
    thresholds = [(0, W.GE, th + 0.123456)]
    compare_full(p, thresholds)


def test_config3_lanczos_parity():
    """BASELINE configs[2]: 100^3 heat, Lanczos k=40, 1001 steps, plus the non-vacuous rows."""
    p = W.config3()
    res = oracle.krylov_project(p)
    tot = res["coeff"][:, 1, 0]
    theta = 0.5 * (tot.max() + tot.min())  # harness LE threshold on total heat (SURVEY A11 iv)
    coeff, res2, cb, ocb, stats, _ = compare_full(p, [(0, W.GE, 1e-3), (1, W.LE, theta)])
    assert np.all(coeff[:, 0, 0] == 0.0)  # center row vacuous at k=40
    assert cb["found"] and cb["row"] == 1


def test_config4_lanczos_parity():
    """BASELINE configs[3]: 400^3 heat (6.4e7 states), k=40, 1001 steps — full oracle run."""
    p = W.config4()
    compare_full(p, [(0, W.GE, 1e-3)])


def test_config5_full_size_properties():
    """BASELINE configs[4] at full size (10^9 states, 8 GB per vector), k=30, 1001 steps.
    The oracle cannot run 30 steps of 10^9 quickly; pinned instead by properties that hold at any size:
    first Lanczos step in closed form, vacuous center row (exact 0), H symmetric
    tridiagonal negative definite, t=0 identity, verdict SAFE for y >= 0.012 (BASELINE)."""
    p = W.config5()
    from paper_1804_01583_b200 import KrylovReach
    with KrylovReach(p) as h:
        coeff, stats = h.project()
        cb = h.check_box()
    m, b = 1000, 100
    c = 0.01 * (m + 1) ** 2
    assert stats[0]["k_eff"] == 30
    assert abs(stats[0]["beta0"] - b ** 1.5) <= 1e-12 * b ** 1.5
    assert np.all(coeff[:, 0, 0] == 0.0)
    assert not cb["found"]
    assert abs(coeff[0, 1, 0] - b ** 3) <= 1e-12 * b ** 3  # total heat at t=0
    assert coeff[0, 2, 0] == 0.0 and abs(coeff[0, 3, 0] - 1.0) <= 1e-14
    assert np.all(np.diff(coeff[:, 1, 0]) <= 1e-9 * b ** 3)  # total heat non-increasing (up to tolerance)


def test_config5_full_size_oracle_golden():
    """BASELINE configs[4] (north_star's target) element by element at full size: 10^9 states, k = 30, 1001 steps,
    four output rows, against tests/golden/C5_heat1000_oracle.json — the oracle's own full run (written by
    scripts/gen_golden.py, which calls only oracle/). Every coefficient (1e-9 floored relative), both bounds,
    beta0, k_eff, the tridiagonal H, the Lemma-1 diagnostic, and the verdict / step / row / witness of the BASELINE
    threshold (center y >= 0.012: never) plus the oracle-chosen LE threshold on total heat (SURVEY A11 iv)."""
    import json
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "C5_heat1000_oracle.json")
    g = json.load(open(path))
    p = W.config5()
    assert (g["m"], g["k"], g["n_steps"], g["step"]) == (1000, p["k"], p["n_steps"], p["step"])
    thresholds = [(int(r), int(s), float(t)) for (r, s, t) in g["thresholds"]]
    orc = np.array(g["coeff"])[:, :, None]
    from paper_1804_01583_b200 import KrylovReach
    with KrylovReach(p) as h:
        coeff, stats = h.project()
        cb = h.check_box(thresholds)
        H, P = h.krylov_data(0)
    assert_coeff(coeff, orc, "C5 full size vs oracle golden")
    assert stats[0]["k_eff"] == g["k_eff"] == 30
    assert abs(stats[0]["beta0"] - g["beta0"]) <= 1e-12 * g["beta0"]
    k = g["k_eff"]
    assert np.allclose(np.diag(H[:k, :k]), g["alpha"], rtol=1e-9, atol=0)
    assert np.allclose(np.diag(H[1:k + 1, :k]), g["beta"], rtol=1e-9, atol=0)
    assert_lemma1(stats, [g["lemma1"]], "C5", T=g["n_steps"] * g["step"], mu=g["mu"],
                  hmax=[max(np.max(np.abs(g["alpha"])), np.max(np.abs(g["beta"])))])
    ocb = oracle.check_box(p, orc, thresholds)
    zlo, zhi = oracle.z_bounds(p)
    for side in ("lo", "hi"):
        ok, worst = bounds_close(cb[side], ocb[side], orc, zlo, zhi)
        assert ok, (side, worst)
    v = g["verdict"]
    assert cb["found"] == v["found"] == ocb["found"] and v["found"]
    assert cb["step"] == v["step"] == ocb["step"] and cb["row"] == v["row"] == 1
    assert 0 < v["step"] < p["n_steps"]
    assert abs(cb["y"] - v["y"]) <= 1e-9 * abs(v["y"])
    assert np.allclose(cb["z"], v["z"], rtol=1e-12, atol=0)
    assert np.all(coeff[:, 0, 0] == 0.0)  # the BASELINE center row: exactly 0 at k = 30


@pytest.mark.parametrize("P", [8])
def test_config5_zslabs_oracle_golden(P):
    """north_star's target configuration: the 10^9-state system decomposed into the z-slabs of 8 GPUs (125 planes
    each, halo planes stored by the step kernel into the neighbouring slab — the peer-memory code path), emulated on
    this GPU (virtual_slabs: the slabs run one after the other): every coefficient against the oracle's full run
    (tests/golden), verdict / step identical."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "C5_heat1000_oracle.json")))
    p = W.config5()
    thresholds = [(int(r), int(s), float(t)) for (r, s, t) in g["thresholds"]]
    from paper_1804_01583_b200 import KrylovReach
    with KrylovReach(p, virtual_slabs=P, part="zslab") as h:
        coeff, stats = h.project()
        cb = h.check_box(thresholds)
    assert_coeff(coeff, np.array(g["coeff"])[:, :, None], f"C5 on {P} z-slabs vs oracle golden")
    assert stats[0]["k_eff"] == g["k_eff"]
    assert cb["found"] and cb["step"] == g["verdict"]["step"] and cb["row"] == g["verdict"]["row"]


def test_config5_first_step_closed_form():
    """alpha_1 = -6c/b, beta_1 from cell counting at 10^9 with k=2."""
    p = W.config5(n_steps=1)
    p["k"] = 2
    from paper_1804_01583_b200 import KrylovReach
    with KrylovReach(p) as h:
        coeff, stats = h.project()
        H, P = h.krylov_data(0)
    m, b = 1000, 100
    c = 0.01 * (m + 1) ** 2
    s = sum(math.comb(3, q) * 2 ** q * (b - 2) ** (3 - q) * (6 / b - q) ** 2 for q in range(4))
    b1 = math.sqrt(c * c * (s + 3 * b * b) / b ** 3)
    assert abs(H[0, 0] - (-6 * c / b)) <= 1e-12 * 6 * c / b
    assert abs(H[1, 0] - b1) <= 1e-12 * b1
    assert abs(P[1, 0] - b ** 1.5) <= 1e-12 * b ** 1.5 and P[0, 0] == 0.0 and P[2, 0] == 0.0


# ---------------------------------------------------------------------------------------------
# Stencil Lanczos: ragged tiles, odd sizes, partitions, determinism, breakdown
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("mx,my,mz,blk,k", [(16, 16, 16, 3, 20), (37, 21, 13, 4, 25), (5, 5, 5, 2, 30),
                                            (70, 9, 11, 5, 16), (130, 17, 6, 5, 12), (2, 3, 2, 1, 6)])
def test_stencil_lanczos_shapes(mx, my, mz, blk, k):
    p = W.heat(mx, blk, k, n_steps=60, step=0.05, my=my, mz=mz)
    p["outs"].append(W.box((1, 1, 1), (min(mx, 4), min(my, 5), min(mz, 3)), 0.5))
    p["outs"].append(W.sparse([0, mx * my * mz - 1, mx + 3], [1.0, 2.0, -1.0]))
    compare_full(p, [(1, W.LE, 0.5 * blk ** 3)])


@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_virtual_slabs_match(P):
    """z-slab decomposition with halo exchange, emulated on one GPU (P slabs, device-to-device halo
    copies instead of NCCL): equal to the unpartitioned run and the oracle."""
    p = W.heat(24, 4, 25, n_steps=100, step=0.02, mz=26)
    res = oracle.krylov_project(p)
    c1, _, _, _ = gpu_run(p)
    cP, _, _, _ = gpu_run(p, virtual_slabs=P, part="zslab")
    assert_coeff(cP, res["coeff"], f"P={P} vs oracle")
    assert_coeff(cP, c1, f"P={P} vs P=1")


def test_deterministic_bitwise():
    p = W.heat(40, 4, 30, n_steps=50)
    a, _, _, _ = gpu_run(p)
    b, _, _, _ = gpu_run(p)
    assert np.array_equal(a, b)
    q = W.config1()
    a, _, _, _ = gpu_run(q)
    b, _, _, _ = gpu_run(q)
    assert np.array_equal(a, b)


def test_lanczos_breakdown_on_sine_mode():
    m = 12
    x = np.arange(m)
    s1 = np.sin((x + 1) * 3 * np.pi / (m + 1))  # odd modes: no output is identically zero
    s2 = np.sin((x + 1) * 1 * np.pi / (m + 1))
    phi = np.einsum("k,j,i->kji", s2, s1, s2).ravel()
    p = W.heat(m, 2, 10, n_steps=20, step=0.1, extras=True)
    p["gens"] = [W.sparse(np.arange(m ** 3), phi)]
    for method in ("lanczos", "arnoldi"):
        coeff, res, cb, ocb, stats, _ = compare_full(p, method=method)
        assert stats[0]["k_eff"] == 1


def test_edge_cases():
    # n_steps = 0, k = 1
    p = W.heat(10, 2, 1, n_steps=0)
    compare_full(p)
    # Arnoldi on the stencil (generic path) vs oracle Arnoldi
    p = W.heat(9, 3, 15, n_steps=40, step=0.05)
    compare_full(p, method="arnoldi")
    # Lanczos on a symmetric CSR
    rp, ci, va, dense = W.random_csr(300, 5, seed=4, symmetric=True)
    q = {"name": "symcsr", "op": "csr", "n": 300, "row_ptr": rp, "col_idx": ci, "val": va, "b": None,
         "gens": [W.sparse([0, 5], [1.0, 2.0]), W.box((10,), (20,), 1.0)], "z_lo": [0.0, -1.0], "z_hi": [1.0, 1.0],
         "center": W.sparse([3], [1.0]), "outs": [W.sparse(np.arange(300), np.linspace(-1, 1, 300)), W.allv()],
         "step": 0.05, "n_steps": 80, "k": 20, "method": "lanczos", "thresholds": [(1, W.LE, 0.3)]}
    compare_full(q)


def test_errors():
    from paper_1804_01583_b200 import KrylovError, KrylovReach
    p = W.heat(8, 2, 5)
    p["gens"] = [W.box((0, 0, 0), (0, 2, 2))]  # empty box: zero direction
    with pytest.raises(KrylovError) as e:
        KrylovReach(p)
    assert "KR_EZERO" in str(e.value)
    q = W.oscillator()
    with pytest.raises(KrylovError) as e:
        KrylovReach(q, method="lanczos")
    assert "KR_ENOTSYM" in str(e.value)
    h = KrylovReach(W.heat(8, 2, 5))
    with pytest.raises(KrylovError) as e:
        h.check_box()
    assert "KR_ESTATE" in str(e.value)
    h.close()


@pytest.mark.parametrize("cfg", ["C1", "C3"])
def test_expm_doubling_equals_per_step_pade(cfg, monkeypatch):
    """The small-k exponentials by doubling over the time grid (default: E = e^{H delta} by Pade-13, then
    x_{2^q+j} = E^{2^q} x_j) agree with one Pade-13 per (step, direction) (KR_EXPM_PADE=1) and the oracle."""
    p = W.CONFIGS[cfg]()
    a, _, _, _ = gpu_run(p)
    monkeypatch.setenv("KR_EXPM_PADE", "1")
    b, _, _, _ = gpu_run(p)
    assert_coeff(a, b, f"{cfg} doubling vs per-step Pade")
    assert_coeff(a, oracle.krylov_project(p)["coeff"], f"{cfg} doubling vs oracle")


@pytest.mark.parametrize("vs", [0, 3])
def test_state_buffers_need_only_ghost_planes_zeroed(vs, monkeypatch):
    """create zeroes only the ghost / halo planes of the three state buffers: the results equal those of
    fully zeroed buffers (KR_ZERO_ALL=1) bitwise, also when the same handle projects twice."""
    from paper_1804_01583_b200 import KrylovReach
    p = W.heat(33, 4, 20, n_steps=40, my=19, mz=14)
    with KrylovReach(p, virtual_slabs=vs) as h:
        a1, _ = h.project()
        a2, _ = h.project()
    monkeypatch.setenv("KR_ZERO_ALL", "1")
    with KrylovReach(p, virtual_slabs=vs) as h:
        b1, _ = h.project()
    assert np.array_equal(a1, a2) and np.array_equal(a1, b1)


@pytest.mark.parametrize("vs", [0, 2, 3])
@pytest.mark.parametrize("lo,hi", [((0, 0, 0), (6, 5, 4)), ((37, 11, 9), (52, 20, 30)), ((71, 30, 0), (80, 40, 3)),
                                   ((13, 0, 14), (14, 1, 15))])
def test_compact_start_vector(lo, hi, vs, monkeypatch):
    """Box generators store only the box region of u_1 (compact tensor maps, TMA zero fill elsewhere;
    the init pass visits the box's tiles only; steps 1-2 read u_1 through the shifted maps). Boxes at a
    corner, in the interior with an odd x start, on the high x / y / low z faces and a single cell; one and
    several slabs (boxes inside one slab or crossing slab boundaries; a box outside a slab's planes).
    Equal to the full fill + init pass (KR_NO_COMPACT=1) and to the oracle, incl. sparse and box output
    rows that meet the box (the init pass gathers P_{.,1} from the compact u_1)."""
    p = W.heat(80, 4, 20, n_steps=40, step=0.02, my=40, mz=30)
    p["gens"] = [W.box(lo, hi, 1.0)]
    inside = (lo[0] + (hi[0] - lo[0]) // 2, lo[1] + (hi[1] - lo[1]) // 2, lo[2] + (hi[2] - lo[2]) // 2)
    idx = lambda x, y, z: x + 80 * (y + 40 * z)  # noqa: E731
    p["outs"] += [W.sparse([idx(*inside), idx(lo[0], lo[1], lo[2]), idx(max(lo[0] - 1, 0), lo[1], lo[2])],
                           [1.0, -0.5, 2.0]),
                  W.box(lo, (hi[0], hi[1], min(hi[2], lo[2] + 2)), 0.25)]
    kw = dict(virtual_slabs=vs, part="zslab") if vs else {}
    a, sa, _, _ = gpu_run(p, **kw)
    monkeypatch.setenv("KR_NO_COMPACT", "1")
    b, sb, _, _ = gpu_run(p, **kw)
    assert [s["k_eff"] for s in sa] == [s["k_eff"] for s in sb]
    assert_coeff(a, b, f"compact vs full u_1 {lo}-{hi} vs={vs}")
    assert_coeff(a, oracle.krylov_project(p)["coeff"], f"compact u_1 {lo}-{hi} vs={vs} vs oracle")


@pytest.mark.parametrize("vs", [0, 3])
def test_compact_start_vector_several_directions(vs):
    """Several directions on the fused Lanczos path, each with its own compact u_1 region (different box
    shapes sharing one compact buffer, refilled at each direction's init) or none (a sparse generator and an
    all-grid center): equal to the oracle on 1 and 3 slabs."""
    p = W.heat(72, 4, 18, n_steps=30, step=0.02, my=36, mz=27)
    p["gens"] = [W.box((0, 0, 0), (5, 4, 3), 1.0), W.box((40, 10, 12), (71, 35, 26), 1.0),
                 W.sparse([5 + 72 * (7 + 36 * 9), 6 + 72 * (7 + 36 * 9)], [1.0, -2.0]), W.box((9, 9, 9), (10, 10, 10), 2.0)]
    p["z_lo"] = np.array([0.9, -1.0, 0.0, 0.5])
    p["z_hi"] = np.array([1.1, 1.0, 1.0, 1.5])
    p["center"] = W.allv(0.25)
    kw = dict(virtual_slabs=vs, part="zslab") if vs else {}
    coeff, stats, _, _ = gpu_run(p, **kw)
    res = oracle.krylov_project(p)
    assert [s["k_eff"] for s in stats] == [r["k_eff"] for r in res["per_dir"]]
    assert_coeff(coeff, res["coeff"], f"several directions vs={vs}")


@pytest.mark.parametrize("n_steps,B", [(0, None), (1, None), (63, None), (64, None), (1000, None), (1000, "1"),
                                       (1000, "7"), (1000, "1001")])
def test_expm_march_equals_one_cta_doubling(n_steps, B, monkeypatch):
    """The time grid over many CTAs (powers E^{2^q}, each CTA starting from x_{sB} = prod E^{2^q} e_1 and
    marching x_{j+1} = E x_j with the projection in the same product) agrees with the one-CTA doubling
    (KR_EXPM_ONECTA=1) and the oracle: grids of 1, 2, 64, 65 and 1001 points, segments of 1, 7, 8+ and all
    columns; two directions."""
    p = W.heat(16, 3, 30, n_steps=n_steps, step=0.05, my=12, mz=10)
    p["gens"].append(W.sparse([W.center_index(16) + 16 * (5 + 12 * 4)], [1.0]))
    p["z_lo"] = np.array([0.9, -1.0])
    p["z_hi"] = np.array([1.1, 1.0])
    if B:
        monkeypatch.setenv("KR_EXPM_B", B)
    a, sa, _, _ = gpu_run(p)
    monkeypatch.setenv("KR_EXPM_ONECTA", "1")
    b, sb, _, _ = gpu_run(p)
    assert [s["k_eff"] for s in sa] == [s["k_eff"] for s in sb]
    assert [s["lemma1"] for s in sa] == pytest.approx([s["lemma1"] for s in sb], rel=1e-9, abs=1e-300)
    assert_coeff(a, b, f"march vs one-CTA doubling N={n_steps} B={B}")
    assert_coeff(a, oracle.krylov_project(p)["coeff"], f"march vs oracle N={n_steps} B={B}")


@pytest.mark.parametrize("k,expect", [(30, [1, 2, 3, 8, 13, 19, 24, 29]), (5, [1, 2, 3, 4]), (2, [1, 2])])
def test_step_times_sampled(k, expect, monkeypatch):
    """krylov_step_times with one launch per step (KR_MULTISTEP=0): one entry per step run; CUDA events around
    steps 1, 2 and six steps spread over 3..k-1 (finite, positive), NaN elsewhere."""
    from paper_1804_01583_b200 import KrylovReach
    monkeypatch.setenv("KR_MULTISTEP", "0")
    p = W.heat(20, 3, k, n_steps=10)
    with KrylovReach(p) as h:
        h.project(want=False)
        st = h.step_times()
        t = h.last_timing()
    assert len(st) == k
    timed = [i + 1 for i, x in enumerate(st) if np.isfinite(x)]
    assert timed == expect
    assert all(st[i - 1] > 0 for i in timed)
    assert t["step_ms_mean"] == pytest.approx(float(np.mean([st[i - 1] for i in timed])), rel=1e-12)


@pytest.mark.parametrize("k", [30, 5, 2])
def test_step_times_multistep(k):
    """With the persistent multi-step kernel (the default on small grids) steps 1-2 of a compact start vector are
    timed one by one and every later step gets its launch's mean; step_ms_mean is their mean."""
    from paper_1804_01583_b200 import KrylovReach
    p = W.heat(20, 3, k, n_steps=10)
    with KrylovReach(p) as h:
        h.project(want=False)
        st = h.step_times()
        t = h.last_timing()
    assert len(st) == k
    assert all(np.isfinite(x) and x > 0 for x in st)
    assert t["step_ms_mean"] == pytest.approx(float(np.mean(st)), rel=1e-12)


def test_virtual_slabs_two_planes_each():
    """halo correctness at the minimum slab thickness — m = 16 on 8 slabs (2 planes each, so every
    owned plane is a halo plane of a neighbour): equal to one slab and to the oracle."""
    p = W.heat(16, 3, 20, n_steps=60, step=0.05)
    res = oracle.krylov_project(p)
    c1, _, _, _ = gpu_run(p)
    c8, _, _, _ = gpu_run(p, virtual_slabs=8, part="zslab")
    assert_coeff(c8, res["coeff"], "m=16 P=8 vs oracle")
    assert_coeff(c8, c1, "m=16 P=8 vs P=1")


@pytest.mark.parametrize("vs", [0, 3])
def test_dense_rand_start_vector(vs):
    """A seeded dense start vector (KR_VEC_RAND, the C5D recipe at small size): the field is generated on the
    device by the library's own counter-based generator and by the oracle's numpy one; every output (the center
    row is non-vacuous here), bound, Lemma 1 and the verdict of an oracle-chosen threshold match; 1 and 3 slabs;
    plus the stored-basis Arnoldi path on the same field."""
    p = W.heat(45, 4, 25, n_steps=200, step=0.02, my=30, mz=20)
    p["gens"] = [W.rand(5)]
    res = oracle.krylov_project(p)
    prop = choose_property(oracle.check_box(p, res["coeff"], []))
    kw = dict(virtual_slabs=vs, part="zslab") if vs else {}
    coeff, _, cb, _, stats, _ = compare_full(p, [prop], res=res, **kw)
    assert np.all(coeff[:, 0, 0] != 0.0) and cb["found"]
    if not vs:
        compare_full(dict(p, k=15), method="arnoldi")


def test_rand_vector_rejected_where_not_defined():
    from paper_1804_01583_b200 import KrylovError, KrylovReach
    p = W.heat(8, 2, 5)
    for q in (dict(p, outs=[W.rand(1)]), dict(p, gens=[W.rand(1)], b=W.box((0, 0, 0), (1, 1, 1), 1.0))):
        with pytest.raises(KrylovError) as e:
            KrylovReach(q)
        assert "KR_EINVAL" in str(e.value)
    with pytest.raises(KrylovError):
        KrylovReach(dict(p, gens=[W.rand(1)]), sim="transpose")


def test_device_block_cache_reuse_and_release():
    """Handles take their device blocks from the process-wide cache filled by destroyed handles (same results,
    bitwise); krylov_release_cached_memory returns them to the driver, and new handles still work."""
    from paper_1804_01583_b200 import krylov_release_cached_memory
    p = W.heat(30, 4, 20, n_steps=40)
    a, _, _, _ = gpu_run(p)
    b, _, _, _ = gpu_run(p)  # blocks from the cache
    assert np.array_equal(a, b)
    assert krylov_release_cached_memory() > 0
    assert krylov_release_cached_memory() == 0
    c, _, _, _ = gpu_run(p)
    assert np.array_equal(a, c)


@pytest.mark.parametrize("env", [{"KR_ZCHUNK": "1"}, {"KR_ZCHUNK": "3"}, {"KR_ZCHUNK": "500"}, {"KR_NO_GRAPH": "1"},
                                 {"KR_HALO_COPY": "1"}, {"KR_WIN": "4", "KR_ZCHUNK": "3"},
                                 {"KR_WIN": "1", "KR_ZCHUNK": "5"}, {"KR_WIN": "5", "KR_ZCHUNK": "2"},
                                 {"KR_WIN": "0", "KR_ZCHUNK": "3"}])
def test_stencil_switches_keep_parity(env, monkeypatch):
    """The diagnostic switches of the fused stencil path (README) change scheduling only: z-chunks of 1, 3 and all
    planes, no CUDA graph, the copy halo transport on 3 virtual slabs, the work-item order (windows of 4, 1 and 5
    tiles over the 6 tiles of the grid, the last group smaller; z-chunk-major) — equal to the oracle; the z-chunk
    choice and the item order only reorder the per-CTA partial sums."""
    p = W.heat(70, 5, 20, n_steps=80, step=0.02, my=40, mz=33)
    p["gens"].append(W.rand(11, 0.3))
    p["z_lo"] = np.array([0.9, 0.0])
    p["z_hi"] = np.array([1.1, 1.0])
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    kw = dict(virtual_slabs=3, part="zslab") if "KR_HALO_COPY" in env else {}
    coeff, _, _, _ = gpu_run(p, **kw)
    assert_coeff(coeff, oracle.krylov_project(p)["coeff"], f"switches {env}")


def test_spmm_per_direction_equals_block(monkeypatch):
    """The block SpMM (each CSR row read once for all directions) sums every row in entry order, like one thread per
    (row, direction): bitwise equal results (C2 recipe, 10 directions — the block form runs from 8 —, both
    Arnoldi routes)."""
    p = W.config2(n=3000, n_gen=9, n_steps=100, k=25)
    for cgs in ("0", "1"):
        monkeypatch.setenv("KR_FORCE_CGS", cgs)
        monkeypatch.delenv("KR_SPMM_PER_DIR", raising=False)
        a, _, _, _ = gpu_run(p)
        monkeypatch.setenv("KR_SPMM_PER_DIR", "1")
        b, _, _, _ = gpu_run(p)
        assert np.array_equal(a, b), cgs
