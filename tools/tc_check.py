"""Quick operator check of the fast modes against the FP64 device path (small shapes).

(The oracle is test infrastructure: only tests/, smoke() and bench.py's CPU legs use it.)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2604_09233_b200._native import Plan

rng = np.random.default_rng(3)
for (L, K, G, P1) in [(300, 500, 8, 3), (301, 777, 40, 17), (1000, 2000, 32, 16), (129, 33, 3, 5)]:
    spatial = rng.standard_normal((P1, L)) * 0.5
    temporal = rng.standard_normal((K, P1)) * 2.0
    sens = rng.standard_normal((L, G)) + 1j * rng.standard_normal((L, G))
    p = rng.standard_normal(L) + 1j * rng.standard_normal(L)
    sig = rng.standard_normal((K, G)) + 1j * rng.standard_normal((K, G))
    ref = Plan(K, L, G, P1, "fp64")
    ref.set_tables(temporal, spatial)
    ref.set_sens(sens)
    ref_e, ref_eh = ref.apply_E(p), ref.apply_EH(sig)
    ref.close()
    for prec in ("fp32", "tf32x3", "f16x3"):
        plan = Plan(K, L, G, P1, prec)
        plan.set_tables(temporal, spatial)
        plan.set_sens(sens)
        e = plan.apply_E(p)
        eh = plan.apply_EH(sig)
        print(prec, (L, K, G, P1), "E rel", np.linalg.norm(e - ref_e) / np.linalg.norm(ref_e),
              "EH rel", np.linalg.norm(eh - ref_eh) / np.linalg.norm(ref_eh), plan.describe()[-80:])
        plan.close()
