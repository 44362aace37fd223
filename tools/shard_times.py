"""Per-rank E^H E time of the sample-sharded decomposition, on one GPU.

    python tools/shard_times.py [--config B] [--worlds 1,2,4,8] [--precision f16x3]

Rank r of a world of N runs the operator on its engine.shard_rows(K, r, N) sample rows; the
slowest rank's apply plus the adjoint-image all-reduce is the sharded apply.  This times every
rank's plan (bench_applies: L2 flushed, events per step) so the strong-scaling ceiling of the
decomposition -- before the all-reduce -- is known without N GPUs.
"""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="B")
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--precision", default="f16x3")
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    from paper_2604_09233_b200 import _native, engine, simulate

    prob = simulate.make_problem(args.config)
    K, L = prob.temporal.shape[0], prob.spatial.shape[1]
    G, P1 = prob.sens.shape[1], prob.spatial.shape[0]
    base = None
    for world in (int(w) for w in args.worlds.split(",")):
        ranks = sorted({engine.shard_rows(K, r, world) for r in range(world)}, key=lambda lh: lh[1] - lh[0])
        times, kern, desc = [], [], ""
        for lo, hi in (ranks[0], ranks[-1]):   # the smallest and the largest shard
            plan = _native.Plan(hi - lo, L, G, P1, args.precision, 0)
            plan.set_tables(prob.temporal[lo:hi], prob.spatial)
            plan.set_sens(prob.sens, prob.intensity)
            plan.apply_EHE(prob.rho_true)
            step_ms, kern_ms = plan.bench_applies(args.steps, 256 << 20)
            times.append(float(np.mean(step_ms)))
            kern.append([k / args.steps for k in kern_ms])
            desc = plan.describe()
            plan.close()
        worst = max(times)
        base = worst if world == 1 else base
        print(json.dumps({"config": args.config, "world": world, "rows_per_rank": [r[1] - r[0] for r in (ranks[0], ranks[-1])],
                          "apply_ms_slowest_rank": worst, "kernel_ms_fwd_adj": kern[-1],
                          "efficiency_before_allreduce": base / (world * worst) if base else None,
                          "plan": desc}), flush=True)


if __name__ == "__main__":
    main()
