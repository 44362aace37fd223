"""Operator error vs FP64 for the benchmark configs (all precisions), incl. masked config A."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2604_09233_b200._native import Plan
from paper_2604_09233_b200 import simulate
for name in ("A", "A_mask"):
    prob = simulate.make_problem(name)
    K, L = prob.temporal.shape[0], prob.spatial.shape[1]
    G, P1 = prob.sens.shape[1], prob.spatial.shape[0]
    rng = np.random.default_rng(0)
    p = rng.standard_normal(L) + 1j * rng.standard_normal(L)
    sig = rng.standard_normal((K, G)) + 1j * rng.standard_normal((K, G))
    out = {}
    for prec in ("fp64", "fp32", "f16x3", "tf32x3"):
        plan = Plan(K, L, G, P1, prec)
        plan.set_tables(prob.temporal, prob.spatial)
        plan.set_sens(prob.sens, prob.intensity)
        out[prec] = (plan.apply_E(p), plan.apply_EH(sig), plan.describe()[-90:])
        plan.close()
    for prec in ("fp32", "f16x3", "tf32x3"):
        e = np.linalg.norm(out[prec][0] - out["fp64"][0]) / np.linalg.norm(out["fp64"][0])
        eh = np.linalg.norm(out[prec][1] - out["fp64"][1]) / np.linalg.norm(out["fp64"][1])
        rows = np.linalg.norm(out[prec][0] - out["fp64"][0], axis=1) / np.linalg.norm(out["fp64"][0], axis=1)
        vox = np.abs(out[prec][1] - out["fp64"][1]) / np.abs(out["fp64"][1])
        print(name, prec, f"E {e:.2e} EH {eh:.2e} worst E row {rows.argmax()} {rows.max():.2e} worst EH vox {vox.argmax()} {vox.max():.2e}", out[prec][2])
