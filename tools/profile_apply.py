"""Run a few E^H E applies of a benchmark config for ncu capture (no timing printed)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2604_09233_b200 import _native, simulate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="B")
ap.add_argument("--precision", default="fp32")
ap.add_argument("--applies", type=int, default=2)
ap.add_argument("--scale", type=int, default=1)
a = ap.parse_args()
prob = simulate.make_problem(a.config, scale=a.scale)
K, L = prob.temporal.shape[0], prob.spatial.shape[1]
plan = _native.Plan(K, L, prob.sens.shape[1], prob.spatial.shape[0], a.precision, 0)
plan.set_tables(prob.temporal, prob.spatial)
plan.set_sens(prob.sens, prob.intensity)
print(plan.describe())
q = plan.apply_EHE(prob.rho_true)
plan.apply_EHE_resident(a.applies)
print("ok", float(np.linalg.norm(q)))
