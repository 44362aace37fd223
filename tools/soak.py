"""Soak test: many back-to-back f16x3 E^H E applies on fresh and reused plans must be bitwise
identical (a rare scheduling race would show as a mismatch).

    python tools/soak.py [--reps 300] [--scales 8,2,1]
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=300)
    ap.add_argument("--scales", default="8,2,1")
    ap.add_argument("--precision", default="f16x3")
    args = ap.parse_args()
    from paper_2604_09233_b200 import simulate
    from paper_2604_09233_b200._native import Plan

    for scale in (int(s) for s in args.scales.split(",")):
        prob = simulate.make_problem("B", scale=scale)
        k, l = prob.temporal.shape[0], prob.spatial.shape[1]
        rng = np.random.default_rng(3)
        p = rng.standard_normal(l) + 1j * rng.standard_normal(l)
        digests = set()
        t0 = time.perf_counter()
        n = 0
        for plan_i in range(3):
            plan = Plan(k, l, 32, 16, args.precision)
            plan.set_tables(prob.temporal, prob.spatial)
            plan.set_sens(prob.sens, prob.intensity)
            for _ in range(args.reps // 3):
                q = plan.apply_EHE(p)
                digests.add(hashlib.sha256(q.tobytes()).hexdigest())
                n += 1
            plan.close()
        print(json.dumps({"scale": scale, "K": k, "L_R": l, "applies": n, "distinct_results": len(digests),
                          "seconds": round(time.perf_counter() - t0, 1)}), flush=True)


if __name__ == "__main__":
    main()
