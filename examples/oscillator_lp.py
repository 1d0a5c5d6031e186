"""The timed harmonic oscillator of PAPER.md §2.2 (x' = y, y' = -x, t' = 1; x0 = -5, y0 in [0, 1]; unsafe
x = 4; delta = pi/4): one simulation of the transpose dynamics (the output space is one-dimensional,
§4.1), the per-step LP of Fig. 2(c) with the unsafe set as two inequalities, the counter-example, and its
check by an independent higher-accuracy re-simulation.

    python examples/oscillator_lp.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1804_01583_b200 import KrylovReach, validate_counterexample  # noqa: E402

p = W.oscillator()
with KrylovReach(p, sim="auto") as h:
    coeff, _ = h.project()
    print("transpose dynamics:", h.transposed, "simulations:", h.n_sim)
    print("basis row at 3pi/4 (P:352: 0.707, 3.54):", coeff[3, 0])
    lp = h.check_lp(None, None, [[1.0], [-1.0]], [4.0, -4.0])  # x <= 4 and -x <= -4
print("feasible steps:", [j for j, f in enumerate(lp["feasible"]) if f == 1])
print(f"counter-example: step {lp['step']} (t = {lp['time']:.4f}), y0 = {lp['z'][0]:.6f} (P:416: 0.66), "
      f"x = {lp['y'][0]:.6f}")
rel, _ = validate_counterexample(p, lp["step"], lp["z"], lp["y"], k=8, sim="forward")
print(f"re-simulation relative error {rel:.2e}")
