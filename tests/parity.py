"""Parity metric between the CUDA path and the oracle (SURVEY §8(c) C-parity).

Floating point: north_star's 1e-9 relative tolerance, floored per (row, direction) series at 1e-3 of
that series' scale S = max_j |oracle|, because early-time values that the method itself produces at
the 1e-14 level carry summation-order noise far above 1e-9 of themselves (1.46e-9 at a
value of 1.7e-14 when S = 8.7e-4). A series that is identically zero in the oracle must be exactly
zero on the GPU (vacuous rows)."""
import numpy as np

RTOL = 1e-9
FLOOR = 1e-3


def projection_envelope(beta0, P, c=64.0):
    """Rounding envelope of c = beta0 P x for ||x||_inf <= 1 (e^{Ht} e_1 of a dissipative H) in ANY evaluation
    order: c u beta0 sum_l |P_rl| per output row (DESIGN R28). beta0: [d]; P: [d][o][k] (or [o][k] for d = 1).
    Returns [1][o][d] for coeff_close's atol."""
    P = np.asarray(P, dtype=float)
    if P.ndim == 2:
        P = P[None]
    b = np.atleast_1d(np.asarray(beta0, dtype=float))
    env = c * np.finfo(float).eps / 2 * b[:, None] * np.sum(np.abs(P), axis=2)  # [d][o]
    return env.T[None]


def coeff_close(gpu, orc, rtol=RTOL, floor=FLOOR, atol=None):
    """gpu, orc: [(N+1)][o][d]. atol: an optional absolute floor broadcastable to [1][o][d] (a rounding
    envelope, projection_envelope). Returns (ok, worst_ratio, where)."""
    gpu = np.asarray(gpu)
    orc = np.asarray(orc)
    assert gpu.shape == orc.shape, (gpu.shape, orc.shape)
    S = np.max(np.abs(orc), axis=0, keepdims=True)  # per (r, d)
    vac = S == 0
    if np.any(vac):
        m = np.broadcast_to(vac, orc.shape)
        if np.any(gpu[m] != 0.0):
            return False, np.inf, "vacuous series not exactly zero"
    tol = rtol * np.maximum(np.abs(orc), floor * S)
    if atol is not None:
        tol = np.maximum(tol, atol)
    err = np.abs(gpu - orc)
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = np.where(tol > 0, err / np.where(tol > 0, tol, 1.0), np.where(err > 0, np.inf, 0.0))
    worst = float(np.max(ratio)) if ratio.size else 0.0
    idx = np.unravel_index(int(np.argmax(ratio)), ratio.shape) if ratio.size else None
    return worst <= 1.0, worst, idx


def bounds_close(gpu, orc, coeff_orc, zlo, zhi, rtol=RTOL, floor=FLOOR):
    """Bounds lo/hi [(N+1)][o]; scale S_r = max_j sum_d |c| max(|zlo|,|zhi|) (magnitude sum)."""
    mag = np.abs(coeff_orc) * np.maximum(np.abs(zlo), np.abs(zhi))[None, None, :]
    S = np.max(np.sum(mag, axis=2), axis=0, keepdims=True)
    tol = rtol * np.maximum(np.abs(orc), floor * S)
    err = np.abs(np.asarray(gpu) - np.asarray(orc))
    ok = np.all((err <= tol) | ((S == 0) & (err == 0)))
    worst = float(np.max(np.where(tol > 0, err / np.where(tol > 0, tol, 1), 0)))
    return bool(ok), worst


def assert_coeff(gpu, orc, what="", atol=None):
    ok, worst, where = coeff_close(gpu, orc, atol=atol)
    assert ok, f"{what}: parity fails, worst err/tol = {worst:.3g} at {where}"
    return worst
