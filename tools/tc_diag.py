"""Full-size diagnostic: tf32x3 vs fp32 vs fp64 operators on config B."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2604_09233_b200._native import Plan
from paper_2604_09233_b200 import simulate

prob = simulate.make_problem("B")
K, L = prob.temporal.shape[0], prob.spatial.shape[1]
rng = np.random.default_rng(0)
p = rng.standard_normal(L) + 1j * rng.standard_normal(L)
sig = rng.standard_normal((K, 32)) + 1j * rng.standard_normal((K, 32))
out = {}
for prec in ("fp64", "fp32", "tf32x3", "f16x3"):
    plan = Plan(K, L, 32, 16, prec)
    plan.set_tables(prob.temporal, prob.spatial)
    plan.set_sens(prob.sens, prob.intensity)
    out[prec] = (plan.apply_E(p), plan.apply_EH(sig))
    print(prec, plan.describe()[-120:])
    plan.close()
ye, qe = out["fp64"]
for prec in ("fp32", "tf32x3", "f16x3"):
    y, q = out[prec]
    print(prec, "E rel", np.linalg.norm(y - ye) / np.linalg.norm(ye), "EH rel", np.linalg.norm(q - qe) / np.linalg.norm(qe))
    ey = np.linalg.norm(y - ye, axis=1) / np.linalg.norm(ye, axis=1)
    eq = np.abs(q - qe) / np.abs(qe)
    blk = ey[: (K // 128) * 128].reshape(-1, 128).max(1)
    print("  E per-128-tile max rel: worst tiles", np.argsort(blk)[-5:], np.sort(blk)[-5:])
    blq = eq[: (L // 128) * 128].reshape(-1, 128).max(1)
    print("  EH per-128-tile max rel: worst tiles", np.argsort(blq)[-5:], np.sort(blq)[-5:])
    print("  EH median rel", np.median(eq), "E median rel", np.median(ey))
