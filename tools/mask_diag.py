import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from conftest import golden
from paper_2604_09233_b200 import engine, simulate
from paper_2604_09233_b200._native import Plan
g = golden("config_a"); pm = simulate.make_problem("A_mask")
K, L = pm.temporal.shape[0], pm.spatial.shape[1]
q0 = {}
for prec in ("fp64", "fp32", "f16x3"):
    plan = Plan(K, L, 8, 3, prec); plan.set_tables(pm.temporal, pm.spatial); plan.set_sens(pm.sens, pm.intensity)
    q0[prec] = plan.apply_EH(g["sigma"]); plan.close()
    inputs = engine.EncodingInputs(sigma=g["sigma"], spatial=pm.spatial, temporal=pm.temporal, sens=pm.sens,
                                   intensity=pm.intensity, kfilter=None, mask_r=pm.mask_r, grid=pm.grid, n_iter=10)
    img, log = engine.recon_full(inputs, precision=prec)
    print(prec, "res", " ".join(f"{(a-b)/b:+.1e}" for a, b in zip(log.residual_norms, g["res_mask"][:10])))
    print(prec, "res abs", " ".join(f"{a:.3e}" for a in log.residual_norms))
for prec in ("fp32", "f16x3"):
    print(prec, "q0 rel", np.linalg.norm(q0[prec]-q0["fp64"])/np.linalg.norm(q0["fp64"]))
