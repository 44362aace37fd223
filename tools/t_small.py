import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2604_09233_b200._native import Plan
rng = np.random.default_rng(3)
for (L, K, G, P1) in [(100, 50, 8, 3), (300, 500, 8, 3), (1000, 2000, 32, 16)]:
    spatial = rng.standard_normal((P1, L)) * 0.5
    temporal = rng.standard_normal((K, P1)) * 2.0
    sens = rng.standard_normal((L, G)) + 1j * rng.standard_normal((L, G))
    p = rng.standard_normal(L) + 1j * rng.standard_normal(L)
    plan = Plan(K, L, G, P1, "f16x3"); plan.set_tables(temporal, spatial); plan.set_sens(sens)
    print((L, K), "E", np.linalg.norm(plan.apply_E(p)), plan.describe()[-60:], flush=True)
