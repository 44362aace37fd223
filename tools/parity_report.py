"""Parity report: GPU CG iterates vs the reference's golden iterates, per precision mode.

    python tools/parity_report.py > profiles/parity_r1.md

Config A (unmasked and masked/j/k-filter) against tests/golden/config_a.npz (produced by the
real reference), relative-L2 of the restricted iterate at iterations 5/10/15/20 and of the
final image; plus the full-size config-B operator error vs the FP64 path.
"""

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import golden  # noqa: E402
from paper_2604_09233_b200 import engine, simulate  # noqa: E402
from paper_2604_09233_b200._native import Plan  # noqa: E402

PRECS = ["fp64", "fp32", "f16x3", "tf32x3"]


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def run_a(name, prec, g):
    prob = simulate.make_problem(name)
    seen = {}
    kf = g["kfilter"] if name == "A_mask" else None
    inputs = engine.EncodingInputs(sigma=g["sigma"], spatial=prob.spatial, temporal=prob.temporal,
                                   sens=prob.sens, intensity=prob.intensity, kfilter=kf,
                                   mask_r=prob.mask_r, grid=prob.grid, n_iter=20)
    img, log = engine.recon_full(inputs, callback=lambda n, r: seen.__setitem__(n, r), precision=prec)
    key = "rho_iters_mask" if name == "A_mask" else "rho_iters"
    its = {int(i): rel(seen[int(i)], ref) for i, ref in zip(g["iters"], g[key])}
    final = rel(img.values, g["values_mask" if name == "A_mask" else "values"])
    res_ref = g["res_mask" if name == "A_mask" else "res"]
    res10 = float(np.max(np.abs(np.array(log.residual_norms[:10]) - res_ref[:10]) / res_ref[:10]))
    return {"iterate_rel_l2": its, "final_image_rel_l2": final, "residual_norm_rel_err_first10": res10}


def run_b_operator():
    prob = simulate.make_problem("B")
    K, L = prob.temporal.shape[0], prob.spatial.shape[1]
    rng = np.random.default_rng(0)
    p = rng.standard_normal(L) + 1j * rng.standard_normal(L)
    out = {}
    for prec in PRECS:
        plan = Plan(K, L, 32, 16, prec)
        plan.set_tables(prob.temporal, prob.spatial)
        plan.set_sens(prob.sens, prob.intensity)
        out[prec] = plan.apply_EHE(p)
        plan.close()
    return {prec: rel(out[prec], out["fp64"]) for prec in PRECS if prec != "fp64"}


def main():
    g = golden("config_a")
    report = {"config_A": {}, "config_A_mask_j_kfilter": {}}
    for prec in PRECS:
        report["config_A"][prec] = run_a("A", prec, g)
        report["config_A_mask_j_kfilter"][prec] = run_a("A_mask", prec, g)
    report["config_B_EHE_vs_fp64_rel_l2"] = run_b_operator()
    print("# Parity report (GPU vs reference golden vectors)\n")
    print("Relative-L2 of the restricted CG iterate vs the reference (nfs/engine.py recon_full, FP64 "
          "numpy) at identical iteration counts; golden vectors from tests/golden/make_golden.py.\n")
    for cfg in ("config_A", "config_A_mask_j_kfilter"):
        print(f"## {cfg}\n\n| mode | it 5 | it 10 | it 15 | it 20 | final image | residual norms (first 10) |")
        print("|---|---|---|---|---|---|---|")
        for prec in PRECS:
            r = report[cfg][prec]
            it = r["iterate_rel_l2"]
            print(f"| {prec} | {it[5]:.1e} | {it[10]:.1e} | {it[15]:.1e} | {it[20]:.1e} | "
                  f"{r['final_image_rel_l2']:.1e} | {r['residual_norm_rel_err_first10']:.1e} |")
        print()
    print("## config B, one E^H E apply at full size vs the FP64 device path\n")
    for k, v in report["config_B_EHE_vs_fp64_rel_l2"].items():
        print(f"- {k}: {v:.2e}")
    print("\n```json\n" + json.dumps(report, indent=1) + "\n```")


if __name__ == "__main__":
    main()
