"""Per-iteration device time of the CG loop vs bare E^H E applies on config B (one process).

    python tools/cg_overhead.py [precision]
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2604_09233_b200 import _native, simulate

prec = sys.argv[1] if len(sys.argv) > 1 else "f16x3"
prob = simulate.make_problem("B")
K, L, G, P1 = prob.temporal.shape[0], prob.spatial.shape[1], prob.sens.shape[1], prob.spatial.shape[0]
plan = _native.Plan(K, L, G, P1, prec, 0)
plan.set_tables(prob.temporal, prob.spatial)
plan.set_sens(prob.sens, prob.intensity)
sig = plan.apply_E(prob.rho_true / prob.intensity)
plan.set_samples(sig)
for rep in range(3):
    rho, res, sol, tim, n = plan.cg_solve(20)
    print(f"cg: initial adjoint {tim[0]*1e3:.3f} ms, iterations mean {np.mean(tim[2:2+n])*1e3:.3f} ms "
          f"(min {np.min(tim[2:2+n])*1e3:.3f}, max {np.max(tim[2:2+n])*1e3:.3f})")
plan.apply_EHE_resident(3)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    plan.apply_EHE_resident(20)
    torch.cuda.synchronize()
    print(f"bare E^H E x20: {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms each (wall)")
print("kernel_times", plan.kernel_times(3))
