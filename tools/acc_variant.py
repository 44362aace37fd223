"""Accuracy and speed of one library build (NFS_B200_LIB selects a variant) in f16x3 mode.

    NFS_B200_LIB=tools/variants/lib_X.so python tools/acc_variant.py [PREC]

Prints one JSON line: config-A CG iterate errors vs the reference goldens (unmasked and
masked + j + k-filter, iterations 5 / 10, residual norms over the first 10), the E^H sigma error
of the masked config A vs the FP64 device path, and the config-B per-operator device times.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import golden  # noqa: E402
from paper_2604_09233_b200 import _native, engine, simulate  # noqa: E402

PREC = sys.argv[1] if len(sys.argv) > 1 else "f16x3"


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def cg_errors(name, g):
    prob = simulate.make_problem(name)
    seen = {}
    kf = g["kfilter"] if name == "A_mask" else None
    inputs = engine.EncodingInputs(sigma=g["sigma"], spatial=prob.spatial, temporal=prob.temporal,
                                   sens=prob.sens, intensity=prob.intensity, kfilter=kf,
                                   mask_r=prob.mask_r, grid=prob.grid, n_iter=20)
    _, log = engine.recon_full(inputs, callback=lambda n, r: seen.__setitem__(n, r), precision=PREC)
    key = "rho_iters_mask" if name == "A_mask" else "rho_iters"
    res_ref = g["res_mask" if name == "A_mask" else "res"]
    out = {f"it{int(i)}": rel(seen[int(i)], ref) for i, ref in zip(g["iters"], g[key]) if i <= 15}
    out["res10"] = float(np.max(np.abs(np.array(log.residual_norms[:10]) - res_ref[:10]) / res_ref[:10]))
    return out


def op_error(g):
    prob = simulate.make_problem("A_mask")
    K, L = prob.temporal.shape[0], prob.spatial.shape[1]
    res = {}
    for prec in ("fp64", PREC):
        plan = _native.Plan(K, L, 8, 3, prec)
        plan.set_tables(prob.temporal, prob.spatial)
        plan.set_sens(prob.sens, prob.intensity)
        res[prec] = plan.apply_EH(g["sigma"])
        plan.close()
    return rel(res[PREC], res["fp64"])


def main():
    g = golden("config_a")
    out = {"lib": os.path.basename(os.environ.get("NFS_B200_LIB", "default")), "prec": PREC}
    out["A"] = cg_errors("A", g)
    out["A_mask"] = cg_errors("A_mask", g)
    out["EH_sigma_A_mask"] = op_error(g)
    prob = simulate.make_problem("B")
    K, L = prob.temporal.shape[0], prob.spatial.shape[1]
    plan = _native.Plan(K, L, 32, 16, PREC, 0)
    plan.set_tables(prob.temporal, prob.spatial)
    plan.set_sens(prob.sens, prob.intensity)
    plan.apply_EHE(prob.rho_true)
    kt = plan.kernel_times(5)
    out["B_fwd_ms"], out["B_adj_ms"] = round(float(kt[0]), 4), round(float(kt[2]), 4)
    out["describe"] = plan.describe()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
