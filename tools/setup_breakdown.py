"""Wall time of each host-side step of a recon_full at config B (what `e2e` pays besides the
applies): plan creation, S' upload, table upload + image build, samples upload, the solve,
the finalize, the plan release.  python tools/setup_breakdown.py [--config B] [--reps 3]"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="B")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    import torch
    from paper_2604_09233_b200 import _native, engine, simulate

    prob = simulate.make_problem(args.config)
    K, L = prob.temporal.shape[0], prob.spatial.shape[1]
    G, P1 = prob.sens.shape[1], prob.spatial.shape[0]
    p0 = _native.Plan(K, L, G, P1, "f16x3")
    p0.set_tables(prob.temporal, prob.spatial)
    p0.set_sens(prob.sens, prob.intensity)
    sigma = p0.apply_E(prob.rho_true / prob.intensity)
    p0.close()
    for _ in range(args.reps):
        t = {}
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan = _native.Plan(K, L, G, P1, "f16x3")
        t["plan_create"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        plan.set_sens(prob.sens, prob.intensity)
        t["set_sens"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        plan.set_tables(prob.temporal, prob.spatial)
        t["set_tables"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        plan.set_samples(sigma)
        t["set_samples"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        rho, res, sol, tim, n = plan.cg_solve(args.iters)
        t["cg_solve"] = time.perf_counter() - t0
        t["cg_device_initial_adjoint"] = float(tim[0])
        t["cg_device_iterations"] = float(np.sum(tim[2:2 + n]))
        t0 = time.perf_counter()
        full = np.zeros(prob.mask_r.size, dtype=complex)
        full[prob.mask_r] = rho * prob.intensity
        t["finalize"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        plan.close()
        t["plan_close"] = time.perf_counter() - t0
        print(json.dumps({k: round(v * 1e3, 3) for k, v in t.items()}), flush=True)


if __name__ == "__main__":
    main()
