"""A/B helper: one apply_E / apply_EH / 5-iteration CG of a config through the library in
NFS_B200_LIB, saved to an .npz, so two builds can be compared bit for bit.

    NFS_B200_LIB=tools/variants/lib_x.so python tools/ab_check.py --config B --out gpurun_out/ab_x.npz
    python tools/ab_check.py --compare gpurun_out/ab_a.npz gpurun_out/ab_b.npz
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="B")
ap.add_argument("--scale", type=int, default=1)
ap.add_argument("--precision", default="f16x3")
ap.add_argument("--out")
ap.add_argument("--compare", nargs=2)
a = ap.parse_args()
if a.compare:
    x, y = np.load(a.compare[0]), np.load(a.compare[1])
    for k in x.files:
        same = np.array_equal(x[k], y[k])
        rel = float(np.linalg.norm(x[k] - y[k]) / max(np.linalg.norm(x[k]), 1e-300))
        print(f"{k}: identical={same} rel={rel:.3e}")
    sys.exit(0)
from paper_2604_09233_b200 import _native, simulate  # noqa: E402

prob = simulate.make_problem(a.config, scale=a.scale)
K, L = prob.temporal.shape[0], prob.spatial.shape[1]
plan = _native.Plan(K, L, prob.sens.shape[1], prob.spatial.shape[0], a.precision, 0)
plan.set_tables(prob.temporal, prob.spatial)
plan.set_sens(prob.sens, prob.intensity)
rng = np.random.default_rng(11)
x = rng.standard_normal(L) + 1j * rng.standard_normal(L)
y = plan.apply_E(x)
q = plan.apply_EH(y)
plan.set_samples(y)
rho, res, *_ = plan.cg_solve(5)
import hashlib  # noqa: E402

# digests (bit identity) + a small slice (the size of the difference) keep the file small
np.savez(a.out, **{k: np.frombuffer(hashlib.sha256(np.ascontiguousarray(v).tobytes()).digest(), np.uint8)
                   for k, v in (("y_sha", y), ("q_sha", q), ("rho_sha", rho))},
         y=y.ravel()[:4096], q=q[:4096], rho=rho[:4096], res=np.asarray(res))
print("saved", a.out)
