"""Small-shape driver for compute-sanitizer (racecheck / synccheck / memcheck) over every kernel
family of the path: the tcgen05 operators (f16x3 tci_kernel, tf32x3 tc kernel), the CUDA-core
contraction (fp32, fp64), the table / B-image prep kernels and the device CG kernels.

    compute-sanitizer --tool racecheck python tools/sanitize_small.py > profiles/...log

Shapes are the smallest that still exercise multi-chunk pipelines, split-K and the 2-CTA
multicast clusters (config B shrunk 8x in-plane: 32^2, K = 1024, 32 coils, P+1 = 16).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2604_09233_b200 import _native, simulate  # noqa: E402

precs = sys.argv[1:] or ["f16x3", "tf32x3", "fp32", "fp64"]
prob = simulate.make_problem("B", scale=8)
K, L = prob.temporal.shape[0], prob.spatial.shape[1]
for prec in precs:
    plan = _native.Plan(K, L, prob.sens.shape[1], prob.spatial.shape[0], prec, 0)
    plan.set_tables(prob.temporal, prob.spatial)
    plan.set_sens(prob.sens, prob.intensity)
    sigma = plan.apply_E(prob.rho_true / prob.intensity)
    plan.set_samples(sigma)
    q = plan.apply_EHE(prob.rho_true)
    rho, res, sol, tim, n = plan.cg_solve(3)
    print(prec, plan.describe()[:80], "EHE norm", float(np.linalg.norm(q)), "cg", n, res[-1])
    plan.close()
print("done")
