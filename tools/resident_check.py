"""Resident phase vs on the fly: bit-identity and timing (config A masked, scaled D, full B).

    python tools/resident_check.py [--configs A_mask,D4,B] [--steps 20]

For each problem: apply_E, apply_EH and a 10-iteration CG solve through one f16x3 plan with
the phase regenerated per apply, then again after nfs_plan_set_phase_resident(1) -- the
results must be identical bit for bit -- and the E^H E time of both modes (nfs_bench_applies,
L2 flushed before every step) plus the build time of the resident phase.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

FLUSH = 256 << 20


def problem(name):
    from paper_2604_09233_b200 import simulate
    if name == "D4":
        return simulate.make_problem("D", scale=4)
    return simulate.make_problem(name)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="A_mask,D4,B")
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    import torch
    from paper_2604_09233_b200._native import Plan

    for name in args.configs.split(","):
        prob = problem(name)
        K, L = prob.temporal.shape[0], prob.spatial.shape[1]
        G, P1 = prob.sens.shape[1], prob.spatial.shape[0]
        plan = Plan(K, L, G, P1, "f16x3")
        plan.set_tables(prob.temporal, prob.spatial)
        plan.set_sens(prob.sens, prob.intensity)
        rng = np.random.default_rng(5)
        x = rng.standard_normal(L) + 1j * rng.standard_normal(L)
        outs = {}
        for mode in (0, 1):
            t_build = None
            if mode:
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                nbytes = plan.set_phase_resident(1)
                torch.cuda.synchronize()
                t_build = time.perf_counter() - t0
            y = plan.apply_E(x)
            q = plan.apply_EH(y)
            plan.set_samples(y)
            rho, res, *_ = plan.cg_solve(10)
            plan.apply_EHE(x)
            step_ms, kern_ms = plan.bench_applies(args.steps, FLUSH)
            outs[mode] = dict(y=y, q=q, rho=rho, res=np.asarray(res), step=float(np.mean(step_ms)),
                              kern=[k / args.steps for k in kern_ms], build_s=t_build)
        same = {k: bool(np.array_equal(outs[0][k], outs[1][k])) for k in ("y", "q", "rho", "res")}
        rec = {"config": name, "K": K, "L_R": L, "coils": G, "P1": P1, "bit_identical": same,
               "ehe_ms_on_the_fly": outs[0]["step"], "ehe_ms_resident": outs[1]["step"],
               "kernel_ms_on_the_fly": outs[0]["kern"], "kernel_ms_resident": outs[1]["kern"],
               "resident_build_s": outs[1]["build_s"], "resident_bytes": nbytes,
               "describe": plan.describe()}
        if not all(same.values()):
            for k in ("y", "q", "rho"):
                a, b = outs[0][k], outs[1][k]
                rec[f"rel_diff_{k}"] = float(np.linalg.norm(a - b) / max(np.linalg.norm(a), 1e-300))
        print(json.dumps(rec), flush=True)
        plan.close()


if __name__ == "__main__":
    main()
