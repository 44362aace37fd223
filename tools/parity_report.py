"""Parity report: GPU CG iterates vs the reference's golden iterates, every precision mode.

    python tools/parity_report.py > profiles/parity_r2.md

Relative-L2 of the restricted CG iterate vs the REAL reference (tests/golden/make_golden.py) at
identical iteration counts, and the worst relative error of the residual norms over the first
10 iterations, for: config A (unmasked; masked + intensity correction + k-filter), config B
(full size, recon_split with 2^28-byte blocks, 10 it), config C (an off-centre slice, z = +39 mm,
scaled 64^2, 10 it) and config D (3D, 32 coils, P+1 = 16, scaled 32x32x16, 50 it); plus the
reference's own split-vs-full drift on config D (the FP64 floor).
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
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def device_sigma(prob, rho):
    k, l = prob.temporal.shape[0], prob.spatial.shape[1]
    plan = Plan(k, l, prob.sens.shape[1], prob.spatial.shape[0], "fp64")
    plan.set_tables(prob.temporal, prob.spatial)
    plan.set_sens(prob.sens)
    out = plan.apply_E(rho)
    plan.close()
    return out


def solve(prob, sigma, prec, n_iter, kfilter=None, starts=None):
    seen = {}
    inputs = engine.EncodingInputs(sigma=sigma, spatial=prob.spatial, temporal=prob.temporal,
                                   sens=prob.sens, intensity=prob.intensity, kfilter=kfilter,
                                   mask_r=prob.mask_r, grid=prob.grid, n_iter=n_iter, block_starts=starts)
    run = engine.recon_split if starts is not None else engine.recon_full
    img, log = run(inputs, callback=lambda n, r: seen.__setitem__(n, r), precision=prec)
    return img, log, seen


def case(name, prob, sigma, g, n_iter, key_it="rho_iters", key_res="res", key_val="values", **kw):
    out = {}
    for prec in PRECS:
        img, log, seen = solve(prob, sigma, prec, n_iter, **kw)
        its = {int(i): rel(seen[int(i)], ref) for i, ref in zip(g["iters"], g[key_it])}
        res_ref = g[key_res][:10]
        res = float(np.max(np.abs(np.array(log.residual_norms[:10]) - res_ref) / res_ref))
        out[prec] = {"iterate_rel_l2": its, "final_image_rel_l2": rel(img.values, g[key_val]),
                     "residual_norm_rel_err_first10": res}
    return name, out


def main():
    report = {}
    ga = golden("config_a")
    pa = simulate.make_problem("A")
    pm = simulate.make_problem("A_mask")
    for name, prob, kf, kit, kres, kval in (("config A", pa, None, "rho_iters", "res", "values"),
                                             ("config A masked + j + k-filter", pm, ga["kfilter"],
                                              "rho_iters_mask", "res_mask", "values_mask")):
        n, r = case(name, prob, ga["sigma"], ga, 20, kit, kres, kval, kfilter=kf)
        report[n] = r
    gb = golden("config_b_cg")
    pb = simulate.make_problem("B")
    n, r = case("config B (full size, recon_split 2^28-byte blocks)", pb, device_sigma(pb, gb["rho_true"]),
                gb, 10, starts=gb["starts"])
    report[n] = r
    gc = golden("config_c_slice")
    pc = simulate.make_slices(40, scale=4, which=[39])[0]
    n, r = case("config C slice z=+39 mm (64^2)", pc, device_sigma(pc, gc["rho_true"]), gc, 10)
    report[n] = r
    gd = golden("config_d_small")
    pd = simulate.make_problem("D", scale=4)
    n, r = case("config D 3D 32x32x16, 32 coils, P+1=16", pd, device_sigma(pd, gd["rho_true"]), gd, 50)
    report[n] = r
    drift = golden("config_d_small_split")
    report["reference split-vs-full drift, config D"] = {
        int(i): rel(s, f) for i, s, f in zip(drift["iters"], drift["rho_iters"], gd["rho_iters"])}

    print("# Parity report (GPU vs the reference's golden iterates)\n")
    print("Relative-L2 of the restricted CG iterate vs the reference (FP64 numpy, `nfs/engine.py`) at "
          "identical iteration counts; golden vectors from `tests/golden/make_golden.py` (run against "
          "the real reference). `res10` = worst relative error of the residual norms over the first 10 "
          "iterations. Stated bounds: fast modes <= 1e-5 at <= 10 iterations (SURVEY 8d); FP64 <= 1e-8.\n")
    for name, r in report.items():
        if name.startswith("reference split"):
            continue
        its = sorted(next(iter(r.values()))["iterate_rel_l2"])
        print(f"## {name}\n\n| mode | " + " | ".join(f"it {i}" for i in its) + " | final image | res10 |")
        print("|---|" + "---|" * (len(its) + 2))
        for prec, v in r.items():
            print(f"| {prec} | " + " | ".join(f"{v['iterate_rel_l2'][i]:.1e}" for i in its)
                  + f" | {v['final_image_rel_l2']:.1e} | {v['residual_norm_rel_err_first10']:.1e} |")
        print()
    d = report["reference split-vs-full drift, config D"]
    print("Reference's own recon_split (4 blocks) vs recon_full on config D, same iterations: "
          + ", ".join(f"it {k}: {v:.1e}" for k, v in d.items()) + "\n")
    print("```json\n" + json.dumps(report, indent=1) + "\n```")


if __name__ == "__main__":
    main()
