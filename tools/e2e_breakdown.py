"""Where the end-to-end time of a recon_full goes (config B by default).

    python tools/e2e_breakdown.py [--config B] [--precision f16x3] [--reps 3]

Prints the CGLog timing labels of `engine.recon_full` (plan + table upload, S' upload, samples
upload, initial adjoint, per-iteration device times) next to the wall time of the whole call,
so the part of the e2e number that is not E^H E applies is visible.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="B")
    ap.add_argument("--precision", default="f16x3")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    import torch
    from paper_2604_09233_b200 import _native, engine, simulate

    prob = simulate.make_problem(args.config)
    K, L = prob.temporal.shape[0], prob.spatial.shape[1]
    plan = _native.Plan(K, L, prob.sens.shape[1], prob.spatial.shape[0], args.precision)
    plan.set_tables(prob.temporal, prob.spatial)
    plan.set_sens(prob.sens, prob.intensity)
    sigma = plan.apply_E(prob.rho_true / prob.intensity)
    plan.close()
    inputs = engine.EncodingInputs(sigma=sigma, spatial=prob.spatial, temporal=prob.temporal, sens=prob.sens,
                                   intensity=prob.intensity, kfilter=None, mask_r=prob.mask_r, grid=prob.grid,
                                   n_iter=args.iters)
    out = []
    for _ in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        img, log = engine.recon_full(inputs, precision=args.precision)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        tim = dict(log.timings)
        it = [v for k, v in log.timings if k.startswith("cg_iteration_")]
        rec = {"wall_s": wall, "iterations_s": float(np.sum(it)), "iteration_mean_ms": 1e3 * float(np.mean(it)),
               **{k: v for k, v in tim.items() if not k.startswith("cg_iteration_")}}
        rec["unlabelled_s"] = wall - sum(v for k, v in tim.items() if not k.startswith("cg_iteration_")) \
            - rec["iterations_s"]
        out.append(rec)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
